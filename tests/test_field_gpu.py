"""GPU parity of the opacity-field path against the reference compiled in place.

Bit-exact (uint64 view of every double) for PrecomputedGaussian, tile lists,
point schedules, view_opacity / label_grid / classify / value_at outputs and the
reference's exact pair / point-view counters, over all 32 strategy subsets.
Reference functions: precompute.hpp:57-78, tiles.hpp:29-146, field_eval.hpp:59-176.
"""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from oracle.refpy import ALL

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def assert_bits(got, want, what=""):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape, what
    bad = bits(got) != bits(want)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} differ, first at {tuple(i)}: "
                             f"{got[tuple(i)]!r} vs {want[tuple(i)]!r}")


@pytest.fixture(scope="module")
def case(ref):
    scene = ref.random_scene(52, 300, 1.0)
    cams = ref.orbit_cameras(6, 4.0, 1.8, 64)
    rc = ref.context(scene, cams)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    rng = np.random.default_rng(7)
    pts = rng.uniform(-1.3, 1.3, (3000, 3))
    return scene, cams, rc, views, pts


def test_precompute_bitexact(case):
    scene, cams, rc, views, _ = case
    want = rc.precompute()
    for v in range(cams.v):
        assert_bits(views.ctx.precompute_view(v), want[v], f"view {v}")


@pytest.mark.parametrize("tile_size", [16, 8, 23])
def test_tile_binding_exact(case, tile_size):
    scene, cams, rc, views, _ = case
    for v in range(cams.v):
        off, ent = views.ctx.tile_binding(v, tile_size)
        want = rc.tile_binding(v, tile_size)
        np.testing.assert_array_equal(off, want["offsets"])
        np.testing.assert_array_equal(ent, want["entries"])


def test_schedule_points_exact(case):
    scene, cams, rc, views, pts = case
    for v in range(cams.v):
        got = views.ctx.schedule_points(v, pts, 16)
        want = rc.schedule_points(v, pts, 16)
        for k in ("tile_assignment", "order", "key_tile", "block_to_tile"):
            np.testing.assert_array_equal(got[k], want[k], err_msg=k)
        assert_bits(got["key_depth"], want["key_depth"], "key_depth")
        np.testing.assert_array_equal(got["block_ranges"], want["block_ranges"])


@pytest.mark.parametrize("mask", list(range(32)))
def test_view_opacity_all_strategies(case, mask):
    scene, cams, rc, views, pts = case
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
    rev = rc.evaluator(mask)
    for classify in (False, True):
        for v in range(cams.v):
            o, ob, co = ev.view_opacity(v, pts, classify)
            ro, rob, rco = rev.view_opacity(v, pts, classify)
            np.testing.assert_array_equal(ob, rob.astype(bool))
            np.testing.assert_array_equal(co, rco.astype(bool))
            assert_bits(o[ob], ro[rob.astype(bool)], f"mask {mask} view {v} classify {classify}")
    assert ev.counters() == rev.counters()


@pytest.mark.parametrize("mask", [0, 1, 3, 7, 15, 31, 16, 24, 17, 30])
@pytest.mark.parametrize("classify", [True, False])
def test_label_grid_bitexact(case, mask, classify):
    scene, cams, rc, views, pts = case
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
    rev = rc.evaluator(mask)
    got = ev.label_grid(pts, classify)
    want = rev.label_grid(pts, classify)
    assert_bits(got, want, f"mask {mask}")
    assert ev.counters() == rev.counters()


@pytest.mark.parametrize("mask", [8, 12, 15, 24, 31])
def test_label_grid_sched_lookahead_bitexact(case, mask, monkeypatch):
    """Schedule of view v + 1 built on the prep lane during view v's evaluation
    (SOF_SCHED_LOOKAHEAD): pruned points re-checked by the kernel, values and the
    reference counters unchanged."""
    scene, cams, rc, views, pts = case
    monkeypatch.setenv("SOF_SCHED_LOOKAHEAD", "1")
    for classify in (True, False):
        ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
        rev = rc.evaluator(mask)
        assert_bits(ev.label_grid(pts, classify), rev.label_grid(pts, classify), f"mask {mask}")
        assert ev.counters() == rev.counters()
        np.testing.assert_array_equal(ev.classify_points(pts), rev.classify_points(pts).astype(bool))
        assert ev.counters() == rev.counters()


@pytest.mark.parametrize("mask", [0, 31, 8, 12, 19])
def test_classify_and_value_at(case, mask):
    scene, cams, rc, views, pts = case
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
    rev = rc.evaluator(mask)
    np.testing.assert_array_equal(ev.classify_points(pts), rev.classify_points(pts).astype(bool))
    assert ev.counters() == rev.counters()
    if not mask & 4:  # value_at requires early_stop off (field_eval.hpp:127)
        ev.reset_counters()
        rev.reset_counters()
        assert_bits(ev.value_at(pts), rev.value_at(pts))
        assert ev.counters() == rev.counters()


def test_value_at_matches_point_oracle(case):
    """FieldEvaluator.MatchesPointOracle (test_mesher.cpp:155-169)."""
    scene, cams, rc, views, pts = case
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies(True, True, False, False, True))
    np.testing.assert_allclose(ev.value_at(pts[:500]), rc.opacity_at_point(pts[:500]), atol=1e-12, rtol=0)


def test_filter_scale_and_dead(ref):
    """Filtered opacity (gaussian.hpp:67-73) and dead-Gaussian culling stay bit-exact."""
    scene = ref.random_scene(11, 200, 1.0)
    scene.opacity[::7] = 0.002  # dead: below 1/255
    cams = ref.orbit_cameras(4, 4.0, 1.8, 48)
    rc = ref.context(scene, cams, filter_scale=0.003)
    views = sof.ViewSet.build(scene, cams, filter_scale=0.003, ctx=sof.Context(0))
    for v in range(cams.v):
        assert_bits(views.ctx.precompute_view(v), rc.precompute()[v])
    pts = np.random.default_rng(3).uniform(-1.2, 1.2, (2000, 3))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    rev = rc.evaluator(ALL)
    assert_bits(ev.label_grid(pts), rev.label_grid(pts))
    assert ev.counters() == rev.counters()


@pytest.mark.parametrize("mask", [31, 30, 19, 18, 23])
def test_dead_records_in_fast_loop(ref, mask):
    """Dead Gaussians (op < 1/255, incl. one ulp-scale below the threshold) inside the
    min-z-sorted lists: skipped before the pair counter, never ending the scan."""
    scene = ref.random_scene(29, 400, 1.0)
    scene.opacity[::5] = 0.002
    scene.opacity[2::9] = (1.0 / 255.0) * (1.0 - 1e-12)
    scene.opacity[4::13] = 1.0 / 255.0  # not dead (op < 1/255 is false)
    cams = ref.orbit_cameras(3, 4.0, 1.8, 48)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    pts = np.random.default_rng(5).uniform(-1.2, 1.2, (3000, 3))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
    rev = rc.evaluator(mask)
    for classify in (False, True):
        for v in range(cams.v):
            o, ob, co = ev.view_opacity(v, pts, classify)
            ro, rob, rco = rev.view_opacity(v, pts, classify)
            np.testing.assert_array_equal(co, rco.astype(bool))
            assert_bits(o[ob], ro[rob.astype(bool)], f"mask {mask} view {v}")
    assert_bits(ev.label_grid(pts), rev.label_grid(pts))
    assert ev.counters() == rev.counters()


def test_single_view_mahalanobis_ball(ref):
    """FieldEvaluator.SingleViewMahalanobisBall (test_mesher.cpp:171-188)."""
    from oracle.refpy import Scene
    scene = Scene(np.zeros((1, 3)), np.full((1, 3), 0.3), np.array([[1.0, 0, 0, 0]]), np.ones(1), np.zeros((1, 3)))
    eye = np.array([0, 0, 3.0])
    cams = ref.look_at(eye, [0, 0, 0], [0, 1, 0], 0.4 * 64 * 3.0, 0.4 * 64 * 3.0, 64, 64)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    rng = np.random.default_rng(53)
    x = rng.uniform(-0.5, 0.5, (400, 3))
    mahal = np.linalg.norm(x, axis=1) / 0.3
    iso = np.sqrt(2 * np.log(2))
    keep = (np.abs(mahal - iso) >= 0.02) & (x[:, 2] > 3.0 - 3.0 - 10)
    zview = (cams.R[0] @ x.T).T[:, 2] + cams.t[0][2]
    keep &= zview < 3.0
    got = ev.classify_points(x[keep])
    np.testing.assert_array_equal(got, mahal[keep] < iso)


def test_errors(ref):
    scene = ref.random_scene(1, 10, 1.0)
    scene.pos[3, 1] = np.nan
    ctx = sof.Context(0)
    with pytest.raises(ValueError, match="non-finite Gaussian parameters"):
        ctx.set_scene(scene)
    with pytest.raises(sof.SofError, match="no scene"):
        sof.FieldEvaluator(None, sof.ViewSet(ctx, None, None, 0.0)).label_grid(np.zeros((3, 3)))
    # the check runs on the device after the upload: a rejected scene replaces a valid one
    # with none (sof_cuda.h, sof_set_scene)
    good = ref.random_scene(1, 10, 1.0)
    ctx.set_scene(good)
    assert ctx.lib.sof_scene_size(ctx.h) == 10
    for field, k in (("opacity", (4,)), ("scale", (2, 0)), ("pos", (9, 2))):
        bad = ref.random_scene(1, 10, 1.0)
        getattr(bad, field)[k] = np.inf
        with pytest.raises(ValueError, match="non-finite Gaussian parameters"):
            ctx.set_scene(bad)
        assert ctx.lib.sof_scene_size(ctx.h) == -1
        ctx.set_scene(good)
        assert ctx.lib.sof_scene_size(ctx.h) == 10


def test_label_all_points_pruned_early(ref):
    """Points that are exterior in the first views are pruned from every later view
    (field_eval.hpp:147); when the candidate list empties, the remaining views have
    nothing to evaluate."""
    scene = ref.random_scene(52, 50, 0.3)
    cams = ref.orbit_cameras(24, 4.0, 1.8, 32)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    centre0 = -cams.R[0].T @ cams.t[0]
    # halfway between camera 0 and the scene: exterior in view 0, pruned afterwards
    pts = 0.5 * centre0 + np.random.default_rng(1).normal(0, 0.05, (500, 3))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    rev = rc.evaluator(ALL)
    got = ev.label_grid(pts)
    assert_bits(got, rev.label_grid(pts))
    assert ev.counters() == rev.counters()
    # every point exterior in view 0 and never evaluated again
    assert (got < 0.5).all() and ev.counters()["point_view_evals"] == len(pts)


@pytest.mark.parametrize("staging", [0, 1])
@pytest.mark.parametrize("mask", [31, 23, 19, 27])
def test_fast_loop_staging_bitexact(ref, mask, staging):
    """The fast loop (tile lists + min-z + dead cull) runs on live-only tile lists with
    either record staging (plain loads / TMA tile::gather4 into an mbarrier double
    buffer): values, exterior flags and the reference counters stay bit-exact, with
    dead Gaussians (field_eval.hpp:89) and lists longer than one staging chunk."""
    scene = ref.random_scene(31, 700, 1.0)
    scene.opacity[::6] = 0.003
    scene.opacity[3::11] = (1.0 / 255.0) * (1.0 - 1e-12)
    cams = ref.orbit_cameras(4, 4.0, 1.8, 40)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    views.ctx.check(views.ctx.lib.sof_set_staging(views.ctx.h, staging))
    pts = np.random.default_rng(17).uniform(-1.2, 1.2, (4000, 3))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
    rev = rc.evaluator(mask)
    for classify in (False, True):
        assert_bits(ev.label_grid(pts, classify), rev.label_grid(pts, classify), f"mask {mask}")
        assert ev.counters() == rev.counters()
    for v in (0, cams.v - 1):
        o, ob, co = ev.view_opacity(v, pts, True)
        ro, rob, rco = rev.view_opacity(v, pts, True)
        np.testing.assert_array_equal(co, rco.astype(bool))
        assert_bits(o[ob], ro[rob.astype(bool)], f"mask {mask} view {v}")
    np.testing.assert_array_equal(ev.classify_points(pts), rev.classify_points(pts).astype(bool))
    # the reference tile lists (with the dead Gaussians) are still what the binding API returns
    off, ent = views.ctx.tile_binding(0, 16)
    want = rc.tile_binding(0, 16)
    np.testing.assert_array_equal(off, want["offsets"])
    np.testing.assert_array_equal(ent, want["entries"])


@pytest.mark.parametrize("group", [5, 40])
def test_tile_binding_depth_key_ties(ref, group):
    """The tile lists' (min_z, index) order (tiles.hpp:139-144) survives the 32-bit key
    sort: clusters of Gaussians whose min_z differ only below float resolution (and some
    exactly equal) are re-sorted by the full key; clusters longer than the tie-run limit
    take the 64-bit fallback sort."""
    scene = ref.random_scene(61, 400, 1.0)
    rng = np.random.default_rng(group)
    for g in range(len(scene.opacity) // group):
        sl = slice(g * group, (g + 1) * group)
        scene.pos[sl] = scene.pos[g * group]
        scene.scale[sl] = scene.scale[g * group]
        scene.rot[sl] = scene.rot[g * group]
        eps = rng.permutation(group) * 1e-10 * (g % 3)  # g % 3 == 0: exact ties
        scene.pos[sl, 2] += eps
    cams = ref.orbit_cameras(3, 4.0, 1.8, 64)
    rc = ref.context(scene, cams)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    for v in range(cams.v):
        off, ent = ctx.tile_binding(v, 16)
        want = rc.tile_binding(v, 16)
        np.testing.assert_array_equal(off, want["offsets"])
        np.testing.assert_array_equal(ent, want["entries"])
    pts = np.random.default_rng(9).uniform(-1.2, 1.2, (3000, 3))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    rev = rc.evaluator(ALL)
    assert_bits(ev.label_grid(pts), rev.label_grid(pts))
    assert ev.counters() == rev.counters()


def test_rejected_views_leave_previous_cameras(ref):
    """sof_set_views validates every camera before replacing the set: a camera with a
    non-positive resolution is rejected and the cached per-view state of the previous
    cameras stays valid (results identical before and after the failed call)."""
    scene = ref.random_scene(52, 200, 1.0)
    cams = ref.orbit_cameras(3, 4.0, 1.8, 48)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    pts = np.random.default_rng(3).uniform(-1.2, 1.2, (500, 3))
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
    before = ev.label_grid(pts)
    bad = ref.orbit_cameras(3, 5.0, 1.8, 48)
    bad.wh[2] = (0, 48)
    with pytest.raises(ValueError, match="resolution"):
        ctx.set_views(bad)
    after = ev.label_grid(pts)
    assert_bits(after, before, "labels after a rejected sof_set_views")


def test_strategy_mask_outside_0_31_rejected(case):
    scene, cams, rc, views, pts = case
    for m in (32, 1 << 8, -1):
        ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.all())
        ev.mask = m
        with pytest.raises(ValueError, match="strategies"):
            ev.label_grid(pts[:10])
