"""Device Delaunay (sof_tetrahedralize) vs the reference on one point set, with timings:
    python tools/dl_check.py random3000|random10k|clustered_small"""
import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2506_19139_b200 as sof
from oracle import refpy
r = refpy.RefLib()
rng = np.random.default_rng(7)
case = sys.argv[1]
if case == "random3000":
    pts = rng.normal(size=(3000, 3))
elif case == "clustered":
    pts = np.concatenate([rng.normal(scale=1e-3, size=(300, 3)), rng.normal(scale=10.0, size=(300, 3))])
elif case == "clustered_small":
    pts = np.concatenate([rng.normal(scale=1e-3, size=(40, 3)), rng.normal(scale=10.0, size=(40, 3))])
elif case == "random10k":
    pts = rng.random((10000, 3))
t = time.time(); want = r.delaunay(pts); tr = time.time() - t
ctx = sof.Context(0)
t = time.time(); got = sof.delaunay_tetrahedralize(pts, ctx); tg = time.time() - t
print(case, "ref", round(tr, 2), "s", want.shape, "gpu", round(tg, 2), "s", got.tetrahedra.shape,
      "equal", got.tetrahedra.shape == want.shape and bool((got.tetrahedra == want).all()), flush=True)
