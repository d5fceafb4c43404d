"""Writes tests/golden/synth_hashes.json: SHA-256 of small instances of every seeded input generator (calls only
synth/; run from the repo root: python tests/golden/make_synth_hashes.py).  tests/test_synth.py recomputes them."""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402


def sha(*arrs):
    h = hashlib.sha256()
    for a in arrs:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def cases():
    return {
        "square_p1(8, 0.1, 0)": lambda: sha(*synth.square_p1(8, jitter=0.1, seed=0)),
        "rect_p1(7, 4, 0.1, 1, flip=1)": lambda: sha(*synth.rect_p1(7, 4, jitter=0.1, seed=1, flip=1)),
        "cube_kuhn_p1(4, 0.05, 0)": lambda: sha(*synth.cube_kuhn_p1(4, jitter=0.05, seed=0)),
        "box_kuhn_p1(3, 4, 5, 0.05, 3, flip=(0,1,1))": lambda: sha(*synth.box_kuhn_p1(3, 4, 5, jitter=0.05, seed=3, flip=(0, 1, 1))),
        "square_crossed_p1(5)": lambda: sha(*synth.square_crossed_p1(5)),
        "icosphere(2, 0.01, 0)": lambda: sha(*synth.icosphere(2, perturb=0.01, seed=0)),
        "normal_pages(3, 3, 100, stream=10)": lambda: sha(synth.normal_pages(3, 3, 100, stream=10)),
        "inverse_pages(3, 50, seed=0)": lambda: sha(synth.inverse_pages(3, 50, seed=0)[0]),
        "integer_pages(2, 2, 64, seed=0)": lambda: sha(synth.integer_pages(2, 2, 64, seed=0)),
        "p2_from_p1(cube_kuhn_p1(2, 0))": lambda: sha(*synth.p2_from_p1(*synth.cube_kuhn_p1(2, jitter=0.0))),
        "uniform01(0, 1, 16)": lambda: sha(synth.uniform01(0, 1, 16)),
    }


if __name__ == "__main__":
    out = {k: f() for k, f in cases().items()}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "synth_hashes.json")
    json.dump({"what": "SHA-256 of small instances of every seeded input generator (dtype, shape and bytes of each "
                       "array, in order): the recipe of DESIGN.md 5 pinned against drift; written by "
                       "tests/golden/make_synth_hashes.py, which calls only synth/", "sha256": out},
              open(path, "w"), indent=1)
    print("wrote", path)
