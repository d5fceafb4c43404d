"""Counter-based splitmix64 generator (vectorised numpy).

Value i of stream s under seed S is ``mix(key(S, s) + (i + 1) * GOLDEN)``,
i.e. the i-th output of a splitmix64 generator seeded with ``key(S, s)``.
Streams are named by small integers so every array draws from its own
sequence ("separate streams").
"""
import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _key(seed, stream):
    with np.errstate(over="ignore"):
        base = np.array([(int(seed) * 0x100000001B3 + int(stream) * 0x1F3) & 0xFFFFFFFFFFFFFFFF],
                        dtype=np.uint64)
        return _mix(base + GOLDEN)[0]


def splitmix64_u64(seed, stream, n, offset=0):
    """n raw 64-bit outputs of stream ``stream`` starting at counter ``offset``."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        return _mix(_key(seed, stream) + i * GOLDEN)


def uniform01(seed, stream, n, offset=0):
    """U[0,1) with 53 random mantissa bits."""
    return (splitmix64_u64(seed, stream, n, offset) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(seed, stream, n, offset=0):
    """U[-1,1)."""
    return 2.0 * uniform01(seed, stream, n, offset) - 1.0


def normal(seed, stream, n, offset=0):
    """N(0,1) by Box-Muller on two consecutive uniforms per output."""
    u = uniform01(seed, stream, 2 * n, 2 * offset)
    u1 = 1.0 - u[0::2]          # (0, 1]
    u2 = u[1::2]
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
