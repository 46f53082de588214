"""A short C3 meshing run for ncu captures (same scene, lattice and kernels as bench.py,
with the views subsampled so a profiled run stays short).

    python tools/profile_case.py --views 8 --steps 2
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2506_19139_b200 as sof  # noqa: E402
from paper_2506_19139_b200.workloads import CONFIGS, kuhn_lattice, orbit_cameras, synthetic_scene  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--lattice", type=int, default=0, help="override the config's lattice size")
    ap.add_argument("--render", action="store_true", help="render one view instead of meshing")
    ap.add_argument("--timed", type=int, default=0, help="also time this many unprofiled steps (wall clock)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    scene = synthetic_scene(cfg["gaussians"], int(args.config[1:]))
    cams = orbit_cameras(cfg["views"], cfg["width"], cfg["height"])
    cams = cams.subset(np.linspace(0, cfg["views"] - 1, args.views).astype(int))
    ctx = sof.Context(0)
    ctx.set_scene(scene)
    ctx.set_views(cams)
    if args.render:
        import ctypes
        views = sof.ViewSet(ctx, ctx.scene, ctx.cams, 0.0)
        stats = np.zeros(4, np.uint64)
        lib, ms, best = ctx.lib, ctypes.c_float(), float("inf")
        for _ in range(args.steps):  # device time of the render alone (no output copies)
            ctx.check(lib.sof_event_record(ctx.h, 0))
            ctx.check(lib.sof_render_view(ctx.h, 0, sof.DEPTH_EXACT, 16, None, None, None, None,
                                          stats.ctypes.data))
            ctx.check(lib.sof_event_record(ctx.h, 1))
            ctx.check(lib.sof_event_elapsed(ctx.h, 0, 1, ctypes.byref(ms)))
            best = min(best, ms.value)
        w, h = (int(x) for x in cams.wh[0])
        print(f"render {w}x{h}: {best:.1f} ms device ({w * h / best / 1e3:.1f} Mpix/s) stats "
              f"[tested, contributing, sorted-path pixels, exact-depth fallbacks] = {stats.tolist()}")
        return
    verts, tets = kuhn_lattice(args.lattice or cfg["lattice"])
    ctx.set_tets(verts, tets)
    for _ in range(args.steps):
        st = {}
        sof.extract_resident(ctx, sof.ExtractOptions(profile=True), st, fetch=False)
    print({k: st[k] for k in ("ms_label", "ms_refine", "ms_eval_kernel", "ms_prep", "ms_sched", "exact_pairs", "contrib_pairs", "point_view_evals", "host_ms_prep",
                               "host_ms_sched", "pairs", "crossing_edges", "kernel_launches")})
    import time
    walls = []
    for _ in range(args.timed):  # unprofiled steps (no per-launch events): wall time
        t0 = time.perf_counter()
        st = {}
        sof.extract_resident(ctx, sof.ExtractOptions(), st, fetch=False)
        walls.append((time.perf_counter() - t0) * 1e3)
    if walls:
        print("unprofiled step ms:", [round(w, 1) for w in walls], "label", round(st["ms_label"], 1), "refine",
              round(st["ms_refine"], 1))


if __name__ == "__main__":
    main()
