"""Generates tests/golden/*.npz from the reference compiled in place (oracle/_ref).

Run in the build container (needs /root/reference + `make -C oracle ref`):
    python tests/golden/make_golden.py
The fixtures pin the C restatement (oracle/sof_oracle.c) without the reference
being present, e.g. on the GPU box. Inputs come from the reference's own
fixture helpers (tests/test_util.hpp via oracle/ref_capi.cpp) plus numpy points.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refpy  # noqa: E402
from paper_2506_19139_b200.workloads import kuhn_lattice  # noqa: E402


def scene_dict(prefix, s):
    return {f"{prefix}_pos": s.pos, f"{prefix}_scale": s.scale, f"{prefix}_rot": s.rot,
            f"{prefix}_opacity": s.opacity, f"{prefix}_dc": s.dc}


def cams_dict(prefix, c):
    return {f"{prefix}_R": c.R, f"{prefix}_t": c.t, f"{prefix}_intr": c.intr, f"{prefix}_wh": c.wh}


def main():
    ref = refpy.RefLib()
    # ---- field: tu::random_scene(mt19937(52), 300) + tu::orbit_cameras(6, 4, 1.8, 64)
    scene = ref.random_scene(52, 300, 1.0)
    cams = ref.orbit_cameras(6, 4.0, 1.8, 64)
    rc = ref.context(scene, cams)
    pts = np.random.default_rng(7).uniform(-1.3, 1.3, (800, 3))
    g = {**scene_dict("scene", scene), **cams_dict("cams", cams), "pts": pts, "precompute": rc.precompute()}
    for v in (0, 3):
        b = rc.tile_binding(v, 16)
        g[f"bind{v}_offsets"], g[f"bind{v}_entries"] = b["offsets"], b["entries"]
    for mask in (0, 31, 9):
        ev = rc.evaluator(mask)
        g[f"label{mask}"] = ev.label_grid(pts, True)
        g[f"label{mask}_counters"] = np.array(list(ev.counters().values()), np.uint64)
    for mask, classify in ((31, True), (0, False), (7, True)):
        ev = rc.evaluator(mask)
        o, ob, co = ev.view_opacity(2, pts, classify)
        g[f"vo{mask}_o"], g[f"vo{mask}_observed"], g[f"vo{mask}_complete"] = o, ob, co
        g[f"vo{mask}_counters"] = np.array(list(ev.counters().values()), np.uint64)
    ev = rc.evaluator(31)
    g["classify31"] = ev.classify_points(pts)
    g["classify31_counters"] = np.array(list(ev.counters().values()), np.uint64)
    ev = rc.evaluator(19)
    g["value19"] = ev.value_at(pts)
    np.savez_compressed(os.path.join(HERE, "field.npz"), **g)

    # ---- mesh: tu::random_scene(mt19937(55), 40) + 5 orbit cameras, jittered 10^3 Kuhn lattice
    scene = ref.random_scene(55, 40, 1.0)
    cams = ref.orbit_cameras(5, 4.0, 1.8, 64)
    verts, tets = kuhn_lattice(10, -1.3, 1.3)
    rc = ref.context(scene, cams)
    out = rc.extract_tetgrid(verts, tets, strategies=31, iterations=8)
    m = {**scene_dict("scene", scene), **cams_dict("cams", cams), "verts": verts, "tets": tets}
    for k in ("grid_opacity", "edges", "refined", "march_triangles", "vertices", "triangles", "counters"):
        m[k] = out[k]
    np.savez_compressed(os.path.join(HERE, "mesh.npz"), **m)

    # ---- render: tu::random_scene(mt19937(21), 60), 2 orbit cameras at 32x32
    scene = ref.random_scene(21, 60, 1.0)
    cams = ref.orbit_cameras(2, 4.0, 1.8, 32)
    rc = ref.context(scene, cams)
    yy, xx = np.mgrid[0:32, 0:32]
    pix = np.stack([xx.ravel(), yy.ravel()], 1).astype(np.int32)
    r = {**scene_dict("scene", scene), **cams_dict("cams", cams), "pix": pix}
    for exact in (True, False):
        p = rc.render_pixels(1, pix, exact)
        for k, val in p.items():
            r[f"{'exact' if exact else 'median'}_{k}"] = val
    d, o = rc.render_depth_map(1, True)
    r["depth_map"], r["opacity_map"] = d, o
    np.savez_compressed(os.path.join(HERE, "render.npz"), **r)
    print("wrote", sorted(f for f in os.listdir(HERE) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
