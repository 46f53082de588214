"""One C5 meshing step on the unbounded scene with the host debug report
(SOF_DEBUG_HOST=1 prints the bisection-cache summary): where refine time goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_19139_b200 as sof  # noqa: E402
from paper_2506_19139_b200.workloads import config_inputs  # noqa: E402

scene, cams, (verts, tets) = config_inputs("C5")
ctx = sof.Context(0)
ctx.set_scene(scene)
ctx.set_views(cams)
ctx.set_tets(verts, tets)
for step in range(int(os.environ.get("STEPS", "1"))):
    st = {}
    t0 = time.perf_counter()
    sof.extract_resident(ctx, sof.ExtractOptions(profile=True), st, fetch=False)
    print(step, round(time.perf_counter() - t0, 2), "s", {k: st[k] for k in st if k.startswith("ms_") or k in ("crossing_edges",)}, flush=True)
