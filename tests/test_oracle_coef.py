"""Pins of the coefficient-weighted P1 oracle (NEXT-1: eq:K_M with c_K, c_M,
Code stiff_scalar_P1 with gqo = 2): the paper's own printed error columns of
Tables tab:KM_P1_2D and tab:KM_P1_3D, the printed closed forms I_K, I_M,
reduction to the c = 1 oracle, quadrature-rule exactness."""
import math

import numpy as np
import pytest

import oracle
import synth


def quad_form(rp, ci, vals, u):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    return math.fsum(u[rows] * vals * u[ci])


def printed_close(x, printed):
    """x rounds to the printed 3-significant-digit value (half a unit in the last place)."""
    e = math.floor(math.log10(abs(printed)))
    return abs(x - printed) <= 0.5 * 10 ** (e - 2) * 1.0001


def test_closed_forms_match_printed_values(golden):
    g = golden("paper_tables_p1.json")
    pi, e = math.pi, math.e
    assert abs(4 * pi ** 4 * (e - 1) ** 2 * (1 + 2 * pi ** 2) / (1 + 4 * pi ** 2) ** 2 - g["I_K_2d"]) < 1e-10
    assert abs(4 * pi ** 4 * (e - 1) ** 2 / (1 + 4 * pi ** 2) ** 2 - g["I_M_2d"]) < 1e-10
    assert abs(6 * pi ** 4 * (e - 1) ** 3 * (1 + 2 * pi ** 2) ** 2 / (1 + 4 * pi ** 2) ** 3 - g["I_K_3d"]) < 1e-10
    assert abs((e - 1) ** 3 * (1 + 2 * pi ** 2) ** 3 / (1 + 4 * pi ** 2) ** 3 - g["I_M_3d"]) < 1e-10


@pytest.mark.parametrize("row", [0, 1])
def test_paper_table_2d_errors(golden, row):
    g = golden("paper_tables_p1.json")
    t = g["p1_2d"][row]
    coords, elems = synth.square_crossed_p1(2 ** t["level"])
    assert coords.shape[1] == t["size"]
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    K, M = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2)
    v = np.sin(np.pi * coords[0]) * np.sin(np.pi * coords[1])
    assert printed_close(abs(quad_form(rp, ci, K, v) - g["I_K_2d"]), t["e_K"])
    assert printed_close(abs(quad_form(rp, ci, M, v) - g["I_M_2d"]), t["e_M"])


@pytest.mark.parametrize("row", [0, 1, 2, 3])
def test_paper_table_3d_errors(golden, row):
    g = golden("paper_tables_p1.json")
    t = g["p1_3d"][row]
    coords, elems = synth.cube_kuhn_p1(2 ** t["level"], jitter=0.0, flip=(0, 0, 1))
    assert coords.shape[1] == t["size"]
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    K, M = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2)
    v = np.cos(np.pi * coords[0]) * np.cos(np.pi * coords[1]) * np.cos(np.pi * coords[2])
    assert printed_close(abs(quad_form(rp, ci, K, v) - g["I_K_3d"]), t["e_K"])
    assert printed_close(abs(quad_form(rp, ci, M, v) - g["I_M_3d"]), t["e_M"])


@pytest.mark.parametrize("dim", [2, 3])
def test_constant_coefficient_reduces_to_c1(dim):
    coords, elems = synth.square_p1(5) if dim == 2 else synth.cube_kuhn_p1(3)
    rp, ci = oracle.p1_pattern(elems, coords.shape[1])
    K1, M1 = oracle.p1_assemble(coords, elems, rp, ci)
    K, M = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=2, cK=(2.5, (0, 0, 0)), cM=(0.5, (0, 0, 0)))
    assert np.max(np.abs(K - 2.5 * K1)) <= 1e-13 * np.max(np.abs(K1))
    assert np.max(np.abs(M - 0.5 * M1)) <= 1e-13 * np.max(np.abs(M1))       # degree-2 rule is exact for phi phi
    Kc, _ = oracle.p1_assemble_coef(coords, elems, rp, ci, gqo=1, cK=(2.5, (0, 0, 0)), cM=(0.5, (0, 0, 0)))
    assert np.max(np.abs(Kc - 2.5 * K1)) <= 1e-13 * np.max(np.abs(K1))      # c const: one point is exact


@pytest.mark.parametrize("dim", [2, 3])
def test_quadrature_rules_exact_to_degree_2(dim):
    """intquad rules integrate monomials of barycentrics exactly: the simplex
    formula int lam^alpha = d! alpha! / (d + |alpha|)! * |T|."""
    for gqo, deg in ((1, 1), (2, 2)):
        lam, w = oracle.quad_rule(dim, gqo)
        assert abs(w.sum() - 1.0 / math.factorial(dim)) < 1e-16
        nv = dim + 1
        for a in range(nv):
            exact1 = 1.0 / math.factorial(dim + 1)
            assert abs(np.dot(w, lam[:, a]) - exact1) < 1e-16
            if deg >= 2:
                for b in range(nv):
                    exact2 = (2.0 if a == b else 1.0) / math.factorial(dim + 2)
                    assert abs(np.dot(w, lam[:, a] * lam[:, b]) - exact2) < 1e-16
