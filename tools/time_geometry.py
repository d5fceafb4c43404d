"""vb_simplex_geometry alone on the config-5 mesh (12.58 M tets): sizes, normals, both; ALG bytes and GB/s."""
import statistics
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import synth  # noqa: E402
from paper_2404_16039_b200 import vb  # noqa: E402

dev = torch.device("cuda:0")


def tm(fn, reps=20):
    for _ in range(3):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(5):
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b) / reps)
    return statistics.median(out)


coords, elems = synth.cube_kuhn_p1(128, jitter=0.05, seed=0)
cd, ed = torch.from_numpy(coords).to(dev), torch.from_numpy(elems).to(dev)
nn, ne = coords.shape[1], elems.shape[1]
m = torch.empty(ne, dtype=torch.float64, device=dev)
N = torch.empty((4, 3, ne), dtype=torch.float64, device=dev)
for name, kw, nbytes in (("meass", dict(want_normals=False, meass=m), ne * 24 + nn * 24),
                         ("normals3D", dict(want_meass=False, normals=N), ne * 112 + nn * 24),
                         ("both", dict(meass=m, normals=N), ne * 120 + nn * 24)):
    ms = tm(lambda: vb.vb_simplex_geometry(cd, ed, **kw))
    print("vb_simplex_geometry %-9s ne=%d: %.4f ms, ALG %.0f MB, %.0f GB/s" % (name, ne, ms, nbytes / 1e6, nbytes / ms / 1e6))
