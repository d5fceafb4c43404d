"""Pins of the P2 oracle (NEXT-3: stiffness_matrixP2 / mass_matrixP2,
P:1009-1049): the paper's printed P2 error columns, reproduction of
quadratic functions, K 1 = 0, sum M = |Omega|, degree-4 quadrature exactness."""
import math

import numpy as np
import pytest

import oracle
import synth


def quad_form(rp, ci, vals, u):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    return math.fsum(u[rows] * vals * u[ci])


def within_last_digit(x, printed, units=1.0):
    e = math.floor(math.log10(abs(printed)))
    return abs(x - printed) <= units * 10 ** (e - 2) * 1.0001


def p2_mesh(dim, level, jitter=0.0):
    if dim == 2:
        return synth.p2_from_p1(*synth.square_crossed_p1(2 ** level))
    return synth.p2_from_p1(*synth.cube_kuhn_p1(2 ** level, jitter=jitter, flip=(0, 0, 1)))


@pytest.mark.parametrize("dim,level", [(2, 6), (3, 2), (3, 3), (3, 4)])
def test_paper_p2_tables(golden, dim, level):
    g1 = golden("paper_tables_p1.json")
    g2 = golden("paper_tables_p2.json")
    row = [r for r in g2["p2_%dd" % dim] if r["level"] == level][0]
    coords, elems = p2_mesh(dim, level)
    assert coords.shape[1] == row["size"]
    rp, ci = oracle.pattern(elems, coords.shape[1])
    K, M = oracle.p2_assemble_coef(coords, elems, rp, ci, gqo=4)
    if dim == 2:
        v = np.sin(np.pi * coords[0]) * np.sin(np.pi * coords[1])
    else:
        v = np.cos(np.pi * coords[0]) * np.cos(np.pi * coords[1]) * np.cos(np.pi * coords[2])
    eK = abs(quad_form(rp, ci, K, v) - g1["I_K_%dd" % dim])
    eM = abs(quad_form(rp, ci, M, v) - g1["I_M_%dd" % dim])
    assert within_last_digit(eK, row["e_K"]) and within_last_digit(eM, row["e_M"])


@pytest.mark.parametrize("dim", [2, 3])
def test_p2_reproduces_quadratics_and_invariants(dim):
    coords, elems = p2_mesh(dim, 2 if dim == 3 else 3)
    # jittered P1 vertices keep straight edges (midpoints are recomputed)
    rp, ci = oracle.pattern(elems, coords.shape[1])
    K, M = oracle.p2_assemble_coef(coords, elems, rp, ci, gqo=4, cK=(1.0, (0, 0, 0)), cM=(1.0, (0, 0, 0)))
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    Kone = np.zeros(coords.shape[1])
    np.add.at(Kone, rows, K)
    assert np.max(np.abs(Kone)) <= 1e-13 * np.max(np.abs(K))              # K 1 = 0
    assert abs(math.fsum(M) - 1.0) <= 1e-13                                  # sum M = |Omega|
    x = coords
    u = x[0] ** 2 + 0.5 * x[0] * x[1] - x[1] ** 2 + (x[2] ** 2 if dim == 3 else 0.0)
    # int |grad u|^2 over the unit square / cube, exact
    # grad u = (2x + y/2, x/2 - 2y[, 2z]): |grad u|^2 = 17/4 (x^2 + y^2) [+ 4 z^2]
    exact = 17.0 / 6.0 + (4.0 / 3.0 if dim == 3 else 0.0)
    assert abs(quad_form(rp, ci, K, u) - exact) <= 1e-12 * exact


@pytest.mark.parametrize("dim", [2, 3])
def test_degree4_rules_exact(dim):
    lam, w = oracle.quad_rule(dim, 4)
    assert abs(w.sum() - 1.0 / math.factorial(dim)) < 1e-15
    # int lam^alpha = d! alpha! / (d + |alpha|)! |T| for all |alpha| <= 4
    nv = dim + 1
    import itertools
    for deg in range(5):
        for alpha in itertools.product(range(deg + 1), repeat=nv):
            if sum(alpha) != deg:
                continue
            num = math.factorial(dim) * math.prod(math.factorial(a) for a in alpha)
            exact = num / math.factorial(dim + deg) / math.factorial(dim)
            got = float(np.dot(w, np.prod(lam ** np.array(alpha), axis=1)))
            assert abs(got - exact) < 1e-15
