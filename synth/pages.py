"""Synthetic page batches (BASELINE.json configs[1]).

All batches are returned in the struct-of-arrays layout of include/vb.h:
numpy shape (cols, rows, N), so entry (i, j) of page k is ``x[j, i, k]``
(column-major entries, page-contiguous planes, ld = N).
"""
import numpy as np

from .rng import normal, uniform01

A_STREAM = 10
B_STREAM = 11
INV_STREAM = 12
INT_STREAM = 13


def normal_pages(rows, cols, npages, seed=0, stream=A_STREAM):
    """Entries i.i.d. N(0,1)."""
    return normal(seed, stream, rows * cols * npages).reshape(cols, rows, npages)


def inverse_pages(n, npages, seed=0, cond_max=1e4, max_rounds=64):
    """A = 3 I + N(0,1) noise; pages with 2-norm condition number > cond_max
    are re-drawn from later counters of the same stream until none remain.

    The condition number is an input-selection criterion (BASELINE.json
    configs[1]: "rejecting pages with cond>1e4"), taken from numpy's SVD;
    nothing here computes a determinant or an inverse.
    Returns (pages (n, n, N), number of pages that were re-drawn).
    """
    per = n * n
    x = normal(seed, INV_STREAM, per * npages).reshape(npages, n, n)   # x[k, j, i]
    eye = np.eye(n)
    a = x + 3.0 * eye
    redrawn = 0
    offset = per * npages
    for _ in range(max_rounds):
        bad = np.nonzero(np.linalg.cond(a) > cond_max)[0]
        if bad.size == 0:
            break
        redrawn += bad.size
        y = normal(seed, INV_STREAM, per * bad.size, offset).reshape(bad.size, n, n)
        offset += per * bad.size
        a[bad] = y + 3.0 * eye
    else:
        raise RuntimeError("inverse_pages: rejection did not converge")
    # a[k, j, i] holds entry (i, j) of page k; planes are (j, i)
    return np.ascontiguousarray(a.transpose(1, 2, 0)), redrawn


def integer_pages(rows, cols, npages, seed=0, stream=INT_STREAM, bound=16):
    """Entries uniform integers in [-bound, bound] stored as float64 (products
    and small determinants of such pages are exact in fp64)."""
    u = uniform01(seed, stream, rows * cols * npages)
    v = np.floor(u * (2 * bound + 1)) - bound
    return v.reshape(cols, rows, npages)
