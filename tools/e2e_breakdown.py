"""Host-side breakdown of bench.py's e2e step (C3): scene / views / tets upload,
extract, mesh fetch."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_19139_b200 as sof  # noqa: E402
from paper_2506_19139_b200.workloads import config_inputs  # noqa: E402


def pinned(a):
    import torch
    t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def main():
    scene, cams, (verts, tets) = config_inputs("C3")
    scene = sof.GaussianScene(*(pinned(np.ascontiguousarray(getattr(scene, k))) for k in
                                ("pos", "scale", "rot", "opacity", "dc")))
    verts, tets = pinned(verts), pinned(tets)
    ctx = sof.Context(0)
    opt = sof.ExtractOptions()
    for step in range(3):
        t = [time.perf_counter()]
        ctx.set_scene(scene)
        t.append(time.perf_counter())
        ctx.set_views(cams)
        t.append(time.perf_counter())
        ctx.set_tets(verts, tets, async_copy=os.environ.get("SYNC_TETS") is None)
        t.append(time.perf_counter())
        st = {}
        sof.extract_resident(ctx, opt, st, fetch=False)
        t.append(time.perf_counter())
        mesh = ctx.result(4, np.float64, 3), ctx.result(5, np.int32, 3)
        t.append(time.perf_counter())
        d = np.diff(t) * 1e3
        print(f"step {step}: scene {d[0]:.1f} views {d[1]:.1f} tets {d[2]:.1f} extract {d[3]:.1f} "
              f"fetch {d[4]:.1f} total {sum(d):.1f} ms | device label {st['ms_label']:.1f} "
              f"march {st['ms_march']:.1f} refine {st['ms_refine']:.1f} weld {st['ms_weld']:.1f}")


if __name__ == "__main__":
    main()
