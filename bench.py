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
# Algorithmic FP64 FLOPs of one evaluated (point, Gaussian) pair of view_opacity
# (field_eval.hpp:95-103) as the reference arithmetic performs it (no contraction):
# abc_cached A 18 (13 mul + 5 add), B 6, 2a 1, the division t* = -b / 2a ~8 (Newton
# sequence), eval_1d's exponent 5, exp 18 (sof_exp: rint-scaled reduction 1 mul + 2 fma,
# degree-6 polynomial 4 fma + 1 mul + 1 fma, table reconstruction 1 fma + 1 add, scaling
# 1 mul; fma = 2 FLOP), alpha 1, survive 2 -> 59. The kernel skips the
# division and the exp where it can prove them irrelevant, so this is the reference's work,
# not the executed instruction count.
FLOP_PER_PAIR = 59.0
# SURVEY.md §8(d) issue roofline of an FP32 fast path: 148 SM x 4 warp-instr/clk x 32 x
# 1.965 GHz / 21 issue slots per pair (reported beside the FP64-pipe fraction)
ISSUE_PAIRS_PER_S = 148 * 4 * 32 * 1.965e9 / 21
# render (K5) issue roofline, §8(d): 17 issue slots per tested (pixel, Gaussian) pair
RENDER_TESTED_PAIRS_PER_S = 148 * 4 * 32 * 1.965e9 / 17


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


def ncu_k_eval() -> dict:
    """dram bytes per launch and pipe utilisation of the opacity-eval kernel from the
    committed ncu capture (profiles/k_eval_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "k_eval_traffic.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def ncu_render() -> dict:
    """Issue activity of the render kernels from the committed ncu captures
    (profiles/k_render_issue.json)."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "k_render_issue.json")))
    except Exception:
        return {}


# ---- sorted rasterizer sample (secondary: not the headline metric) -------------------------

def render_sample(device: int, views=(0, 1, 2), rows=(135, 540, 945), threads=None):
    """C2 (1M Gaussians, 1920x1080) exact-depth render of a few views through
    sof_render_view, device-timed with events (outputs stay on the device), then a CPU
    baseline and a parity check on the same rows: the reference's collect_contributions +
    render_pixel (oracle/_ref, ThreadPool-like host threads) for every pixel of `rows` of
    view 0, compared bit for bit (colour, T, depth, opacity, contribution counts)."""
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
    for rep in range(2):  # pass 0 warms up (scratch allocations), pass 1 is timed
        for v in range(len(views)):
            ctx.check(ctx.lib.sof_event_record(ctx.h, 0))
            ctx.check(ctx.lib.sof_render_view(ctx.h, v, sof.DEPTH_EXACT, 16, None, None, None, None,
                                              stats.ctypes.data))
            ctx.check(ctx.lib.sof_event_record(ctx.h, 1))
            ctx.check(ctx.lib.sof_event_elapsed(ctx.h, 0, 1, ctypes.byref(ms)))
            if rep == 1:
                res.append((ms.value, stats.copy()))
    t = float(np.mean([r[0] for r in res]))
    tested = float(np.mean([float(r[1][0]) for r in res]))
    contrib = float(np.mean([float(r[1][1]) for r in res]))
    px = cfg["width"] * cfg["height"]
    out = {"config": "C2: 1M Gaussians, 1920x1080, exact depth + colour + T + opacity at depth",
           "views_timed": len(res), "ms_per_view": t, "mpix_per_s": px / (t * 1e-3) / 1e6,
           "tested_pairs_per_s": tested / (t * 1e-3), "contributing_pairs_per_s": contrib / (t * 1e-3),
           "contributions_per_pixel": contrib / px,
           "roofline": {"bound": "issue", "kernel": "K5 (R1-R4, whole render)", "achieved": tested / (t * 1e-3),
                        "peak": RENDER_TESTED_PAIRS_PER_S, "unit": "tested pairs/s",
                        "frac": tested / (t * 1e-3) / RENDER_TESTED_PAIRS_PER_S,
                        "ncu_issue_active_weighted": ncu_render().get("issue_active_time_weighted_pct"),
                        "note": "SURVEY.md 8(d): 17 issue slots per tested (pixel, Gaussian) pair; the binning's "
                                "tile cull removes tested pairs, so this counts work not done. "
                                "ncu_issue_active_weighted: issue activity of R0-R4 weighted by kernel time "
                                "(profiles/k_render_issue.json)"}}
    # the rows of view 0 on the device, then on the CPU reference
    full = sof.render_view(sof.ViewSet(ctx, ctx.scene, ctx.cams, 0.0), 0, sof.DEPTH_EXACT, counts=True)
    ctx.close()
    try:
        from oracle import refpy
        ref = refpy.RefLib()
        threads = threads or len(os.sched_getaffinity(0))
        rc = ref.context(scene, cams.subset(np.array([0])))
        w = cfg["width"]
        pix = np.array([(x, y) for y in rows for x in range(w)], np.int32)
        t0 = time.perf_counter()
        want = rc.render_pixels(0, pix, True, threads=threads)
        dt = time.perf_counter() - t0
        ys, xs = pix[:, 1], pix[:, 0]
        bad = {k: int((full[kk][ys, xs].reshape(len(pix), -1).view(np.uint64) !=
                       want[k].reshape(len(pix), -1).view(np.uint64)).any(axis=1).sum())
               for k, kk in (("color", "rgb"), ("tfinal", "t_final"), ("depth", "depth"), ("acc", "opacity"))}
        bad["counts"] = int((full["counts"][ys, xs] != want["ncontrib"]).sum())
        out["parity"] = {"pixels": len(pix), "rows": list(rows), "mismatched_pixels": bad,
                         "bit_identical": all(v == 0 for v in bad.values())}
        cpu_mpix = len(pix) / dt / 1e6
        out["cpu_baseline"] = {"value": cpu_mpix, "unit": "Mpix/s", "cores": threads, "kind": "reference",
                               "sample": f"reference collect_contributions + render_pixel over {len(pix)} pixels "
                                         f"(rows {list(rows)} of view 0), {dt:.1f} s"}
    except Exception as e:  # the reference build is absent
        out["parity"] = {"unavailable": str(e)[:200]}
        out["cpu_baseline"] = {"value": None, "unit": "Mpix/s", "cores": 0, "kind": "reference",
                               "sample": f"unavailable: {e}"[:200]}
    return out


# ---- CPU reference (oracle/_ref): bounded sample -----------------------------------------------

def crossing_edge_sample(verts, labels, n_lattice, count, seed=0):
    """Up to `count` lattice edges (x, y and z neighbours) whose endpoints are on
    opposite sides of the level set of `labels`, oriented (inside, outside)."""
    inside = labels >= 0.5
    rng = np.random.default_rng(seed)
    out = []
    for step in (1, n_lattice, n_lattice * n_lattice):
        i = np.arange(len(verts) - step)
        i = i[inside[i] != inside[i + step]]
        if step == 1:
            i = i[(i % n_lattice) != n_lattice - 1]
        elif step == n_lattice:
            i = i[(i // n_lattice) % n_lattice != n_lattice - 1]
        a, b = i, i + step
        e = np.where(inside[a][:, None], np.stack([a, b], 1), np.stack([b, a], 1))
        out.append(e)
    e = np.concatenate(out)
    return e[rng.permutation(len(e))[:count]].astype(np.int64)


def cpu_reference_sample(scene, cams, verts, n_lattice, edges_total, sample_views=(0, 1), threads=None,
                         vertex_stride=1, refine_edges=10_000):
    """The reference's own code (oracle/_ref, all strategies) on a ViewSet of
    `sample_views`: ViewSet::build + FieldEvaluator ctor (tile bindings) + label_grid over
    the vertices with ThreadPool(threads), then binary_search_refine (8 iterations, the
    serial classify_point callback as in extract_mesh) over `refine_edges` crossing
    lattice edges of that label. Per-query times are scaled by V / k views, and the
    label and bisection queries are combined in the step's own mix (N_v + 8 E)."""
    from oracle import refpy
    ref = refpy.RefLib()
    threads = threads or len(os.sched_getaffinity(0))
    sub = cams.subset(list(sample_views))
    xyz = np.ascontiguousarray(verts[::vertex_stride])
    t0 = time.perf_counter()
    rc = ref.context(scene, sub)
    ev = rc.evaluator(refpy.ALL)
    labels = ev.label_grid(xyz, True, threads)
    t_label = time.perf_counter() - t0
    out = {"seconds_label": t_label, "threads": threads, "views": len(sample_views), "vertices": len(xyz),
           "labels": labels, "pairs": ev.counters()["pairs"], "evaluator": ev, "context": rc}
    k = len(sample_views)
    per_label_query = t_label * (cams.v / k) / len(xyz)
    out["label_queries_per_s"] = 1.0 / per_label_query
    if vertex_stride == 1 and refine_edges > 0:
        e = crossing_edge_sample(xyz, labels, n_lattice, refine_edges)
        used, inv = np.unique(e.ravel(), return_inverse=True)
        ev2 = rc.evaluator(refpy.ALL)
        sub_xyz = np.ascontiguousarray(xyz[used])
        sub_e = inv.reshape(-1, 2).astype(np.int32)
        t1 = time.perf_counter()
        ev2.refine(sub_xyz, sub_e, 0.5 * (sub_xyz[sub_e[:, 0]] + sub_xyz[sub_e[:, 1]]), ITER)
        t_ref = time.perf_counter() - t1
        per_bisect_query = t_ref * (cams.v / k) / (ITER * len(e))
        out.update(seconds_refine=t_ref, refine_edges=len(e), bisection_queries_per_s=1.0 / per_bisect_query)
        q_label, q_bis = len(xyz), ITER * edges_total
        out["queries_per_s"] = (q_label + q_bis) / (q_label * per_label_query + q_bis * per_bisect_query)
    else:
        out["queries_per_s"] = out["label_queries_per_s"]
    return out


def describe_cpu(r, V):
    s = (f"reference label_grid (all strategies, ThreadPool({r['threads']})) over {r['vertices']} lattice vertices "
         f"with views {{0,1}} incl. ViewSet::build + tile bindings ({r['seconds_label']:.1f} s)")
    if "seconds_refine" in r:
        s += (f" + binary_search_refine (8 iterations, serial classify_point) of {r['refine_edges']} crossing "
              f"edges ({r['seconds_refine']:.1f} s); per-query times x{V // r['views']} in views, "
              f"combined as N_v label + 8 E bisection queries")
    return s


def run_reference(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    from paper_2506_19139_b200.workloads import CONFIGS, config_inputs, kuhn_lattice
    cfg = CONFIGS[args.config]
    scene, cams, _ = config_inputs(args.config, lattice=False)
    verts, _ = kuhn_lattice(cfg["lattice"]) if cfg["lattice"] else (None, None)
    for _ in range(args.warmup):  # warm-up: a small sample (threads, page cache)
        cpu_reference_sample(scene, cams, verts, cfg["lattice"], cfg["edges"], vertex_stride=64, refine_edges=0)
    vals, secs = [], []
    for _ in range(args.steps):
        r = cpu_reference_sample(scene, cams, verts, cfg["lattice"], cfg["edges"])
        vals.append(r["queries_per_s"])
        secs.append(r["seconds_label"] + r.get("seconds_refine", 0.0))
    v = float(np.median(vals))
    sample = describe_cpu(r, cams.v) + f", {np.median(secs):.1f} s/step"
    line = {"metric": "opacity-field point queries/sec", "value": v, "unit": "queries/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.median(secs)) * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: meshing step (label + {ITER}-step bisection queries)",
                       "gaussians": cfg["gaussians"], "views": cfg["views"],
                       "resolution": [cfg["width"], cfg["height"]], "lattice": cfg["lattice"]},
            "cpu_baseline": {"value": v, "unit": "queries/s", "cores": r["threads"], "kind": "reference",
                             "sample": sample},
            "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def c3_parity(device, scene, cams, verts, n_lattice, cpu_run, classify_points=10_000):
    """Parity of the benchmark configuration itself, outside the timed region: the GPU
    label over views {0, 1} of every lattice vertex against the reference's label_grid on
    the same 2-view ViewSet (the cpu_baseline run above: values bit for bit, pairs and
    point-view counters equal), and classify_point on a 10^4-point sample (crossing-edge
    midpoints and uniform points) against the reference's classify_point."""
    import paper_2506_19139_b200 as sof
    want = cpu_run["labels"]
    rev = cpu_run["evaluator"]
    sub = cams.subset([0, 1])
    ctx = sof.Context(device)
    views = sof.ViewSet.build(scene, sub, ctx=ctx)
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    got = ev.label_grid(verts)
    label_bad = int((got.view(np.uint64) != want.view(np.uint64)).sum())
    label_counters = ev.counters() == rev.counters()
    e = crossing_edge_sample(verts, want, n_lattice, classify_points // 2, seed=1)
    rng = np.random.default_rng(2)
    mid = np.concatenate([0.5 * (verts[e[:, 0]] + verts[e[:, 1]]),
                          rng.uniform(verts.min(0), verts.max(0), (classify_points - len(e), 3))])
    ev.reset_counters()
    rev.reset_counters()
    g = ev.classify_points(mid)
    r = rev.classify_points(mid).astype(bool)
    cls_bad = int((g != r).sum())
    cls_counters = ev.counters() == rev.counters()
    ctx.close()
    return {"label_views01": {"vertices": int(len(verts)), "mismatched_values": label_bad,
                              "counters_equal": bool(label_counters), "pairs": int(rev.counters()["pairs"] or 0)},
            "classify_sample": {"points": int(len(mid)), "crossing_edge_midpoints": int(len(e)),
                                "mismatched": cls_bad, "counters_equal": bool(cls_counters)},
            "reference": "oracle/_ref (reference headers compiled in place)",
            "bit_identical": label_bad == 0 and cls_bad == 0 and label_counters and cls_counters}


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
    # SOF_BENCH_COMM=1 (under torchrun) attaches the library communicator even at one rank,
    # so the multi-GPU code path can be exercised where only one GPU exists
    force_comm = os.environ.get("SOF_BENCH_COMM") == "1" and "RANK" in os.environ
    if world > 1 or force_comm:
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
    opt = sof.ExtractOptions()
    comm_kind = "single GPU"
    if (world > 1 or force_comm) and backend == "nccl":
        # the library owns the communicator: rank 0 draws the NCCL id, torch.distributed
        # only carries it; sof_extract then shards views and tets with NCCL collectives on
        # the library stream (k_comm.cu)
        obj = [sof.Context.comm_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        ctx.comm_init(obj[0], world, rank)
        comm_kind = f"library NCCL communicator, views and tets sharded x{world}"
        step = lambda st: sof.extract_resident(ctx, opt, st, fetch=False)  # noqa: E731
    elif world > 1:  # SOF_DIST_BACKEND=gloo: ranks may share a GPU; host-driven protocol (sharded.py)
        from paper_2506_19139_b200.sharded import ShardedMesher
        mesher = ShardedMesher(ctx, rank, world)
        comm_kind = f"host protocol over gloo, views sharded x{world}"
        step = lambda st: mesher.extract(sof.ExtractOptions(), st, fetch=False)  # noqa: E731
    else:
        step = lambda st: sof.extract_resident(ctx, opt, st, fetch=False)  # noqa: E731

    def barrier():
        if world > 1 or force_comm:
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
    if world == 1 or backend == "nccl":
        sof.extract_resident(ctx, sof.ExtractOptions(profile=True), prof_stats, fetch=False)
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
    # the kernels' own work: list entries scanned (the reference's pair counter adds the
    # Gaussians counted without listing -- behind or crossing the camera plane -- which
    # only unbounded scenes have; scanned_pairs is 0 otherwise and the pairs are the work)
    scanned = mean("scanned_pairs", 0.0) or pairs
    roof = None
    if prof_stats.get("ms_eval_kernel"):
        eval_ms = float(prof_stats["ms_eval_kernel"])
        eval_launches = float(prof_stats["eval_launches"])
        prof_step_ms = sum(float(prof_stats[k]) for k in ("ms_label", "ms_march", "ms_refine", "ms_weld"))
        fp64 = ctypes.c_double()
        ctx.check(lib.sof_fp64_peak(ctx.h, ctypes.byref(fp64)))
        achieved = scanned * FLOP_PER_PAIR / (eval_ms * 1e-3) / 1e12
        nk = ncu_k_eval()
        pps = scanned / (eval_ms * 1e-3)
        roof = {"bound": "fp64", "kernel": "k_eval (opacity evaluation, FP64 parity path)",
                "achieved": achieved, "peak": fp64.value, "unit": "TFLOP/s", "frac": achieved / fp64.value,
                "traffic": nk.get("dram_bytes_per_launch"), "flop_per_pair": FLOP_PER_PAIR,
                "pairs_per_s": pps, "scanned_pairs_per_step": scanned, "kernel_share_of_step": eval_ms / prof_step_ms,
                "avg_launch_ms": eval_ms / max(eval_launches, 1),
                "issue_roofline_frac": pps / ISSUE_PAIRS_PER_S,
                "ncu_fp64_pipe_active": nk.get("fp64_pipe_active_pct"),
                "ncu_issue_active": nk.get("issue_active_pct"),
                "peak_note": "FP64 FMA-pipe throughput measured in-process (sof_fp64_peak, 2 FLOP/DFMA); "
                             "MEASURED_PEAKS.json has no FP64 figure. issue_roofline_frac: pairs/s against "
                             "SURVEY.md 8(d)'s FP32 fast-path issue roofline (1.77e12 pairs/s)"}

    # e2e: the public C-ABI with host buffers: upload scene/views/tets, extract, fetch mesh
    e2e = None
    if args.e2e_steps > 0 and (world == 1 or backend == "nccl"):
        h2d = sum(a.nbytes for a in host_arrays) + cams.R.nbytes + cams.t.nbytes + cams.intr.nbytes + cams.wh.nbytes
        times, d2h = [], 0
        for k in range(args.e2e_steps + 1):
            barrier()
            t0 = time.perf_counter()
            ctx.set_scene(scene)
            ctx.set_views(cams)
            ctx.set_tets(verts, tets, async_copy=True)  # tets upload overlaps the label pass
            # every rank holds the merged mesh; rank 0 delivers it to the host
            mesh = sof.extract_resident(ctx, opt, {}, fetch=(rank == 0))
            dt = time.perf_counter() - t0
            if world > 1:  # the job ends when the slowest rank is done
                tt = torch.tensor([dt], device="cuda")
                torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
                dt = float(tt.item())
            if mesh is not None:
                d2h = mesh.vertices.nbytes + mesh.triangles.nbytes
            if k > 0:
                times.append(dt)
        # job totals: every rank uploads the inputs, rank 0 downloads the mesh
        e2e = {"value": queries / float(np.median(times)), "unit": "queries/s",
               "h2d_bytes_per_step": int(h2d) * world, "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(np.median(times)) * 1e3}

    cpu, cpu_run = None, None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu_run = cpu_reference_sample(scene, cams, verts, cfg["lattice"], E)
            cpu = {"value": cpu_run["queries_per_s"], "unit": "queries/s", "cores": cpu_run["threads"],
                   "kind": "reference", "sample": describe_cpu(cpu_run, V)}
            if world > 1:
                cpu["note"] = "measured on rank 0's host cores once; the same CPU job for every N"
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
                           "parallelism": comm_kind,
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
    ok = True
    if rank == 0 and cpu_run is not None:
        line["parity"] = c3_parity(local, scene, cams, verts, cfg["lattice"], cpu_run)
        ok = line["parity"].get("bit_identical", True)
    if rank == 0:
        render = None
        if world == 1 and not args.no_render:
            try:
                render = render_sample(local)
            except Exception as e:
                render = {"unavailable": str(e)[:200]}
        line["render"] = render
        if render and render.get("parity", {}).get("bit_identical") is False:
            ok = False
        print(json.dumps(line), flush=True)
    if world > 1 or force_comm:
        torch.distributed.destroy_process_group()
    if not ok:
        print("PARITY FAILURE: the GPU results differ from the reference (see the parity objects)", file=sys.stderr)
        return 3
    return 0


if __name__ == "__main__":
    sys.exit(main())
