"""Appendix B's unbounded layout with the cameras INSIDE the background shell.

About half of the shell lies behind every camera; the reference binds those Gaussians
to every tile (tiles.hpp:116-126) ahead of all other entries, and counts them as pairs
for every evaluated point (field_eval.hpp:94) although they never contribute. The fast
evaluation loop leaves them out of the tile lists and counts them (gauss_behind,
Binding::nb, behind_pairs in k_field.cu); the extraction must still equal the
reference's mesh byte for byte with identical pair / point-view counters — in the label
pass, the per-view bisection and the truncated bisection caches.
"""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from paper_2506_19139_b200.workloads import kuhn_lattice, orbit_cameras, unbounded_scene
from oracle.refpy import Cameras, Scene

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def case(ref):
    c = orbit_cameras(8, 64, 48, radius=4.0)
    s = unbounded_scene(4000, 5, c)
    scene = Scene(s.pos, s.scale, s.rot, s.opacity, s.dc)
    cams = Cameras(c.R, c.t, c.intr, c.wh, c.nearfar)
    verts, tets = kuhn_lattice(16)
    rc = ref.context(scene, cams)
    # behind the cameras in Mahalanobis terms: centre depth beyond the bound
    zc = np.einsum("vj,nj->vn", cams.R[:, 2, :], s.pos) + cams.t[:, 2:3]
    assert (zc < -1.0).sum(axis=1).min() > 50  # shell Gaussians behind every camera
    return scene, cams, verts, tets, rc


@pytest.mark.parametrize("budget", [None, 0])
@pytest.mark.parametrize("mask", [31, 27, 23])
def test_unbounded_extract_matches_reference(case, tmp_path, mask, budget):
    scene, cams, verts, tets, rc = case
    want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
    assert len(want["triangles"]) > 100
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    if budget is not None:  # bisection through truncated caches
        ctx.check(ctx.lib.sof_set_cache_budget(ctx.h, budget))
    st = {}
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets),
                            sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask)), st)
    np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, want["triangles"])
    assert st["pairs"] == int(want["counters"][0])
    assert st["point_view_evals"] == int(want["counters"][1])
    ctx.close()


@pytest.mark.parametrize("classify", [True, False])
def test_unbounded_label_and_views(case, classify):
    """label_grid in both modes and view_opacity per view (early stop and value mode)."""
    from oracle.refpy import ALL
    scene, cams, verts, tets, rc = case
    rev = rc.evaluator(ALL)
    want = rev.label_grid(verts, classify)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    got = ev.label_grid(verts, classify)
    np.testing.assert_array_equal(bits(got), bits(want))
    assert ev.counters() == rev.counters()
    for v in range(cams.v):
        rev.reset_counters()
        ev.reset_counters()
        o, ob, co = ev.view_opacity(v, verts[::7], classify)
        wo, wob, wco = rev.view_opacity(v, verts[::7], classify)
        np.testing.assert_array_equal(bits(o), bits(wo))
        np.testing.assert_array_equal(ob, wob.astype(bool))
        np.testing.assert_array_equal(co, wco.astype(bool))
        assert ev.counters() == rev.counters()
    ctx.close()


def _stats(ctx, v):
    st = np.zeros(3, np.int64)
    ctx.check(ctx.lib.sof_live_binding_stats(ctx.h, v, 16, st.ctypes.data_as(__import__("ctypes").c_void_p)))
    return st


@pytest.fixture(scope="module")
def crossing_case(ref):
    """The unbounded case plus Gaussians straddling camera planes right in front of the
    cameras (the reference lists them in every tile; they reach part of the image)."""
    c = orbit_cameras(6, 64, 48, radius=4.0)
    s = unbounded_scene(3000, 7, c)
    rng = np.random.default_rng(9)
    extra_pos, extra_scale = [], []
    for v in range(c.R.shape[0]):
        R, t = c.R[v], c.t[v]
        centre = -R.T @ t
        for k in range(4):
            off = R.T @ np.array([rng.uniform(-0.4, 0.4), rng.uniform(-0.3, 0.3), rng.uniform(-0.05, 0.25)])
            extra_pos.append(centre + off)
            extra_scale.append(rng.uniform(0.05, 0.3, 3))
    m = len(extra_pos)
    pos = np.concatenate([s.pos, np.array(extra_pos)])
    scale = np.concatenate([s.scale, np.array(extra_scale)])
    rot = np.concatenate([s.rot, np.tile([1.0, 0, 0, 0], (m, 1))])
    op = np.concatenate([s.opacity, rng.uniform(0.2, 0.9, m)])
    dc = np.concatenate([s.dc, rng.uniform(0, 1, (m, 3))])
    scene = Scene(pos, scale, rot, op, dc)
    cams = Cameras(c.R, c.t, c.intr, c.wh, c.nearfar)
    verts, tets = kuhn_lattice(14, -4.5, 4.5)
    return scene, cams, verts, tets, ref.context(scene, cams)


def test_crossing_binding_counts(crossing_case):
    scene, cams, verts, tets, rc = crossing_case
    ctx = sof.Context(0)
    sof.ViewSet.build(scene, cams, ctx=ctx)
    st = np.array([_stats(ctx, v) for v in range(cams.v)])
    assert (st[:, 1] > 0).all()       # counted Gaussians in every view
    assert st[:, 2].sum() > 0         # crossing Gaussians listed where they reach
    # far fewer entries than the every-tile binding (4 x 3 tiles x counted)
    ctx.close()


@pytest.mark.parametrize("budget", [None, 0])
@pytest.mark.parametrize("mask", [31, 27])
def test_crossing_extract_matches_reference(crossing_case, mask, budget):
    scene, cams, verts, tets, rc = crossing_case
    want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    if budget is not None:
        ctx.check(ctx.lib.sof_set_cache_budget(ctx.h, budget))
    st = {}
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets),
                            sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask)), st)
    np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, want["triangles"])
    assert st["pairs"] == int(want["counters"][0])
    assert st["point_view_evals"] == int(want["counters"][1])
    ctx.close()


@pytest.mark.parametrize("classify", [True, False])
def test_crossing_label_and_views(crossing_case, classify):
    from oracle.refpy import ALL
    scene, cams, verts, tets, rc = crossing_case
    rev = rc.evaluator(ALL)
    want = rev.label_grid(verts, classify)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    got = ev.label_grid(verts, classify)
    np.testing.assert_array_equal(bits(got), bits(want))
    assert ev.counters() == rev.counters()
    for v in range(cams.v):
        rev.reset_counters()
        ev.reset_counters()
        o, ob, co = ev.view_opacity(v, verts[::5], classify)
        wo, wob, wco = rev.view_opacity(v, verts[::5], classify)
        np.testing.assert_array_equal(bits(o), bits(wo))
        assert ev.counters() == rev.counters()


def test_unbounded_medium_label_matches_reference(ref):
    """A larger unbounded case at C5's resolution (200k Gaussians, two 1600x1064 views with
    the cameras inside the shell, a 32^3 lattice reaching out to the cameras): label
    opacities and the reference's pair / point-view counters, with counted Gaussians listed
    only where they reach."""
    from oracle.refpy import ALL
    c = orbit_cameras(2, 1600, 1064, radius=4.0)
    s = unbounded_scene(200000, 5, c)
    scene = Scene(s.pos, s.scale, s.rot, s.opacity, s.dc)
    cams = Cameras(c.R, c.t, c.intr, c.wh, c.nearfar)
    verts, _ = kuhn_lattice(32, -4.5, 4.5)
    rev = ref.context(scene, cams).evaluator(ALL)
    want = rev.label_grid(verts, True)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    st = np.array([_stats(ctx, v) for v in range(cams.v)])
    assert (st[:, 1] > 100).all()  # counted Gaussians in every view
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    got = ev.label_grid(verts, True)
    np.testing.assert_array_equal(bits(got), bits(want))
    assert ev.counters() == rev.counters()
    ctx.close()
