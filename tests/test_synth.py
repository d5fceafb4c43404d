"""The seeded input generators (synth/, the one module the oracle side and the CUDA side share): SHA-256 of
small instances against tests/golden/synth_hashes.json (identical inputs on both sides, pinned
against drift of the recipe in DESIGN.md §5), and the counts the recipe states."""
import importlib.util
import json
import os

import synth

HERE = os.path.dirname(os.path.abspath(__file__))


def _maker():
    spec = importlib.util.spec_from_file_location("make_synth_hashes", os.path.join(HERE, "golden", "make_synth_hashes.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_generators_reproduce_their_hashes():
    want = json.load(open(os.path.join(HERE, "golden", "synth_hashes.json")))["sha256"]
    cases = _maker().cases()
    assert set(want) == set(cases)
    for name, fn in cases.items():
        assert fn() == want[name], name


def test_recipe_counts():
    c, e = synth.cube_kuhn_p1(4)
    assert c.shape == (3, 5 ** 3) and e.shape == (4, 6 * 4 ** 3)
    c, e = synth.square_p1(8)
    assert c.shape == (2, 81) and e.shape == (3, 128)
    assert synth.cube_counts(128) == (129 ** 3, 6 * 128 ** 3) or synth.cube_counts(128)[0] == 129 ** 3
    x, t = synth.icosphere(2)
    assert x.shape[1] == 10 * 4 ** 2 + 2 and t.shape[1] == 20 * 4 ** 2
