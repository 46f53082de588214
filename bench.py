#!/usr/bin/env python
"""Benchmark of the SOF hot path on B200: one step = one full meshing pass
(label -> Marching Tetrahedra -> 8-step bisection -> weld) of the tetra input.

Metric (BASELINE.json): opacity-field point queries/sec, a query being one full
O(x) = min over all views for one point (the label pass answers one per tetra
vertex, the bisection one per crossing edge per iteration), with meshing
wall-seconds reported beside it. Workload: BASELINE.json configs[2] (C3: 3M
Gaussians, 200 views at 1600x1064, 300^3 jittered Kuhn lattice = 27M vertices,
160M tets), synthetic (paper_2506_19139_b200/workloads.py).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

One JSON line on rank 0. Under torchrun (N>1) views are sharded across ranks and
merged exactly (paper_2506_19139_b200/sharded.py). --impl reference times the
reference's own CPU code (oracle/_ref, compiled in place) on a bounded sample.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ITER = 8  # refine_iterations (extract.hpp:16)
# algorithmic FP64 FLOPs of one evaluated (point, Gaussian) pair of view_opacity
# (field_eval.hpp:95-103) as the bit-exact reference arithmetic performs it:
# abc_cached 24 (A: 13 mul + 5 add, B: 4 mul + 2 add), peak_t 2 + IEEE division ~8,
# eval_1d argument 5, exp (sof_exp: rint-scaled reduction 6, 13-term Horner 24,
# reconstruction 2) 32, alpha / clamp / survive 5 -> 76. The kernel
# skips the division and the exp where it can prove them irrelevant, so this is the
# algorithmic (reference) work, not the executed instruction count.
FLOP_PER_PAIR = 76.0


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for k, name in enumerate(names):
                    if r[5 + k].lower() == "active":
                        reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}


def ncu_traffic() -> float | None:
    """dram bytes per launch of the opacity-eval kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "k_eval_traffic.json")
    try:
        return float(json.load(open(p))["dram_bytes_per_launch"])
    except Exception:
        return None


# ---- sorted rasterizer sample (secondary: not the headline metric) -------------------------

def render_sample(device: int, views=(0, 1, 2)):
    """C2 (1M Gaussians, 1920x1080) exact-depth render of a few views through
    sof_render_view, device-timed with events; outputs stay on the device."""
    import paper_2506_19139_b200 as sof
    from paper_2506_19139_b200.workloads import CONFIGS, orbit_cameras, synthetic_scene
    cfg = CONFIGS["C2"]
    scene = synthetic_scene(cfg["gaussians"], 2)
    cams = orbit_cameras(cfg["views"], cfg["width"], cfg["height"]).subset(np.array(views))
    ctx = sof.Context(device)
    ctx.set_scene(scene)
    ctx.set_views(cams)
    stats = np.zeros(4, np.uint64)
    ms, res = ctypes.c_float(), []
    for rep in range(2):  # pass 0 warms up (spill-pool and binning allocations), pass 1 is timed
        for v in range(len(views)):
            ctx.check(ctx.lib.sof_event_record(ctx.h, 0))
            ctx.check(ctx.lib.sof_render_view(ctx.h, v, sof.DEPTH_EXACT, 16, None, None, None, None,
                                              stats.ctypes.data))
            ctx.check(ctx.lib.sof_event_record(ctx.h, 1))
            ctx.check(ctx.lib.sof_event_elapsed(ctx.h, 0, 1, ctypes.byref(ms)))
            if rep == 1:
                res.append((ms.value, stats.copy()))
    timed = res
    t = float(np.mean([r[0] for r in timed]))
    tested = float(np.mean([float(r[1][0]) for r in timed]))
    contrib = float(np.mean([float(r[1][1]) for r in timed]))
    px = cfg["width"] * cfg["height"]
    ctx.close()
    return {"config": "C2: 1M Gaussians, 1920x1080, exact depth + colour + T + opacity at depth, bit-exact",
            "views_timed": len(timed), "ms_per_view": t, "mpix_per_s": px / (t * 1e-3) / 1e6,
            "tested_pairs_per_s": tested / (t * 1e-3), "contributing_pairs_per_s": contrib / (t * 1e-3),
            "sorted_path_pixels": int(np.mean([float(r[1][2]) for r in timed]))}


# ---- CPU reference (oracle/_ref): bounded sample -----------------------------------------------

def cpu_reference_sample(scene, cams, verts, sample_views=(0, 1), threads=None, vertex_stride=1):
    """The reference's own FieldEvaluator (all strategies) on a 2-view ViewSet:
    ViewSet::build + FieldEvaluator ctor (tile bindings) + label_grid over the
    vertices with ThreadPool(threads). Returns seconds and the per-view-query rate
    extrapolated linearly to all V views (pruning makes later views cheaper, so
    this is an upper bound on CPU time)."""
    from oracle import refpy
    ref = refpy.RefLib()
    threads = threads or len(os.sched_getaffinity(0))
    sub = cams.subset(list(sample_views))
    xyz = np.ascontiguousarray(verts[::vertex_stride])
    t0 = time.perf_counter()
    rc = ref.context(scene, sub)
    ev = rc.evaluator(refpy.ALL)
    ev.label_grid(xyz, True, threads)
    dt = time.perf_counter() - t0
    k = len(sample_views)
    per_query = dt * (cams.v / k) / len(xyz)
    return {"seconds": dt, "queries_per_s": 1.0 / per_query, "threads": threads, "views": k,
            "vertices": len(xyz), "pairs": ev.counters()["pairs"]}


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    from paper_2506_19139_b200.workloads import CONFIGS, config_inputs, kuhn_lattice
    cfg = CONFIGS[args.config]
    scene, cams, _ = config_inputs(args.config, lattice=False)
    verts, _ = kuhn_lattice(cfg["lattice"]) if cfg["lattice"] else (None, None)
    for _ in range(args.warmup):  # warm-up: a small sample (threads, page cache)
        cpu_reference_sample(scene, cams, verts, vertex_stride=64)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_reference_sample(scene, cams, verts)
        vals.append(r["queries_per_s"])
        secs.append(r["seconds"])
    v = float(np.median(vals))
    sample = (f"reference label_grid (all strategies, ThreadPool({r['threads']})) over all {r['vertices']} "
              f"lattice vertices with views {{0,1}} incl. ViewSet::build + tile bindings, "
              f"{np.median(secs):.1f} s/step, extrapolated x{cams.v // 2} in views")
    line = {"metric": "opacity-field point queries/sec", "value": v, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(secs)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: meshing step (label + 8-step bisection queries)",
                       "gaussians": cfg["gaussians"], "views": cfg["views"],
                       "resolution": [cfg["width"], cfg["height"]], "lattice": cfg["lattice"]},
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": r["threads"], "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---- ours ---------------------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-render", action="store_true", help="skip the C2 render sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_2506_19139_b200 as sof
    from paper_2506_19139_b200 import _lib
    from paper_2506_19139_b200.workloads import CONFIGS, config_inputs

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    # one GPU per rank; SOF_DIST_BACKEND=gloo (host collectives, ranks may share a GPU)
    # exists only to exercise the multi-rank path where fewer GPUs than ranks exist
    backend = os.environ.get("SOF_DIST_BACKEND", "nccl")
    if backend == "gloo" and local >= torch.cuda.device_count():
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = CONFIGS[args.config]
    scene, cams, (verts, tets) = config_inputs(args.config)
    V = cams.v
    v0, v1 = rank * V // world, (rank + 1) * V // world

    ctx = sof.Context(local)
    lib = ctx.lib
    # pinned host buffers (the e2e leg copies from these every step)
    host_arrays = [scene.pos, scene.scale, scene.rot, scene.opacity, scene.dc, verts, tets]
    for a in host_arrays:
        ctx.check(lib.sof_host_register(a.ctypes.data, a.nbytes))
    ctx.set_scene(scene)
    ctx.set_views(cams)
    ctx.set_tets(verts, tets)
    opt = sof.ExtractOptions(view_begin=v0, view_end=v1)
    if world > 1:
        from paper_2506_19139_b200.sharded import ShardedMesher
        mesher = ShardedMesher(ctx, rank, world)
        step = lambda st: mesher.extract(sof.ExtractOptions(), st, fetch=False)  # noqa: E731
    else:
        step = lambda st: sof.extract_resident(ctx, opt, st, fetch=False)  # noqa: E731

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        ctx.check(lib.sof_sync(ctx.h))
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step({})
    barrier()
    launches0 = ctx.kernel_launches
    stats = []
    with Clocks(local) as clk:
        ctx.check(lib.sof_event_record(ctx.h, 0))
        for _ in range(args.steps):
            st = {}
            step(st)
            stats.append(st)
        ctx.check(lib.sof_event_record(ctx.h, 1))
        ms = ctypes.c_float()
        ctx.check(lib.sof_event_elapsed(ctx.h, 0, 1, ctypes.byref(ms)))
        barrier()
    launches = ctx.kernel_launches - launches0
    total_ms = ms.value
    # one more step with per-kernel device timings, outside the timed region, for the
    # roofline (the timed steps run without the per-launch events)
    prof_stats = {}
    if world == 1:
        sof.extract_resident(ctx, sof.ExtractOptions(view_begin=v0, view_end=v1, profile=True), prof_stats,
                             fetch=False)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda" if backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    last = stats[-1]
    E = int(last["crossing_edges"])
    queries = len(verts) + ITER * E
    value = queries / (ms_step * 1e-3)

    # roofline of the dominant kernel (opacity evaluation, FP64 pipe); the fused
    # single-GPU step reports per-launch kernel times, the sharded step does not
    def mean(k, default=None):
        vals = [s[k] for s in stats if k in s]
        return float(np.mean(vals)) if vals else default

    pairs = mean("pairs", mean("rank_pairs", 0.0))
    roof = None
    if prof_stats.get("ms_eval_kernel"):
        eval_ms = float(prof_stats["ms_eval_kernel"])
        eval_launches = float(prof_stats["eval_launches"])
        prof_step_ms = sum(float(prof_stats[k]) for k in ("ms_label", "ms_march", "ms_refine", "ms_weld"))
        fp64 = ctypes.c_double()
        ctx.check(lib.sof_fp64_peak(ctx.h, ctypes.byref(fp64)))
        achieved = pairs * FLOP_PER_PAIR / (eval_ms * 1e-3) / 1e12
        roof = {"bound": "fp64", "kernel": "k_eval (opacity evaluation, FP64 parity path)",
                "achieved": achieved, "peak": fp64.value, "unit": "TFLOP/s", "frac": achieved / fp64.value,
                "traffic": ncu_traffic(), "flop_per_pair": FLOP_PER_PAIR,
                "pairs_per_s": pairs / (eval_ms * 1e-3), "kernel_share_of_step": eval_ms / prof_step_ms,
                "avg_launch_ms": eval_ms / max(eval_launches, 1),
                "peak_note": "FP64 FMA-pipe throughput measured in-process (sof_fp64_peak, 2 FLOP/DFMA); "
                             "MEASURED_PEAKS.json has no FP64 figure"}

    # e2e: the public C-ABI with host buffers: upload scene/views/tets, extract, fetch mesh
    e2e = None
    if args.e2e_steps > 0 and world == 1:
        h2d = sum(a.nbytes for a in host_arrays) + cams.R.nbytes + cams.t.nbytes + cams.intr.nbytes + cams.wh.nbytes
        times, d2h = [], 0
        for k in range(args.e2e_steps + 1):
            barrier()
            t0 = time.perf_counter()
            ctx.set_scene(scene)
            ctx.set_views(cams)
            ctx.set_tets(verts, tets, async_copy=True)  # tets upload overlaps the label pass
            mesh = sof.extract_resident(ctx, opt, {}, fetch=True)
            dt = time.perf_counter() - t0
            d2h = mesh.vertices.nbytes + mesh.triangles.nbytes
            if k > 0:
                times.append(dt)
        e2e = {"value": queries / float(np.median(times)), "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(np.median(times)) * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_sample(scene, cams, verts)
            cpu = {"value": r["queries_per_s"], "unit": "queries/s", "cores": r["threads"], "kind": "reference",
                   "sample": f"reference label_grid over all {r['vertices']} vertices with views {{0,1}} "
                             f"(incl. ViewSet::build + bindings), {r['seconds']:.1f} s, extrapolated x{V // 2} in views"}
        except Exception as e:  # the reference build is absent
            cpu = {"value": None, "unit": "queries/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": "opacity-field point queries/sec", "value": value, "unit": "queries/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                # one C3 job; its views are split across the ranks: total work is fixed
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"{args.config}: meshing step (label + march + {ITER}-step bisection + weld)",
                           "gaussians": cfg["gaussians"], "views": V, "resolution": [cfg["width"], cfg["height"]],
                           "lattice": cfg["lattice"], "tets": int(len(tets)), "vertices": int(len(verts)),
                           "parallelism": f"views sharded x{world}" if world > 1 else "single GPU",
                           "l2": f"inputs ({verts.nbytes / 1e9:.2f} GB vertices + {tets.nbytes / 1e9:.2f} GB tets + "
                                 f"per-view records of {cfg['gaussians'] * 128 / 1e9:.2f} GB) exceed the 126 MB L2"},
                "meshing_wall_s": ms_step / 1e3, "queries_per_step": queries,
                "stages_ms": {k: mean(k) for k in ("ms_label", "ms_march", "ms_refine", "ms_weld") if k in last},
                "profiled_step_ms": {k: float(prof_stats[k]) for k in ("ms_label", "ms_march", "ms_refine", "ms_weld",
                                                                      "ms_prep", "ms_sched", "ms_eval_kernel")
                                     if k in prof_stats},
                "point_view_evals_per_step": int(mean("point_view_evals", mean("rank_point_view_evals", 0))),
                "label_queries_per_s": (len(verts) / (mean("ms_label") * 1e-3)) if "ms_label" in last else None,
                "crossing_edges": E, "mesh_vertices": int(last["mesh_vertices"]),
                "mesh_triangles": int(last["mesh_triangles"]), "pairs_per_step": int(pairs),
                "gpu_launches": int(launches), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk.summary()}
    for a in host_arrays:
        lib.sof_host_unregister(a.ctypes.data)
    ctx.close()  # the render sample gets the whole device (the meshing cache holds ~half of HBM)
    if rank == 0:
        render = None
        if world == 1 and not args.no_render:
            try:
                render = render_sample(local)
            except Exception as e:
                render = {"unavailable": str(e)[:200]}
        line["render"] = render
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
