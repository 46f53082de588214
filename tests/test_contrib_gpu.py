"""The per-ray API and the K-window resort mode against the compiled reference.

* collect_contributions (opacity_field.hpp:39-61) for arbitrary rays: same lists, same
  (t*, index) order, same six values, bit for bit.
* render_pixel (opacity_field.hpp:201-219) of given lists, and of lists passed through
  windowed_resort (:66-91).
* windowed_resort on the device: the reference's element order, ties included (its
  std::sort / std::push_heap / std::pop_heap tie behaviour, stl_order.cuh).
* sof_render_view with a window K: per pixel, contributions in view-space centre-depth
  order through the K-slot window, then blended; every output bit-identical to the
  reference composition collect_contributions -> order -> windowed_resort -> render_pixel.
"""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from oracle.refpy import Scene

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def tie_scene(n, seed=11):
    rng = np.random.default_rng(seed)
    pos = np.zeros((n, 3))
    pos[:, 2] = rng.uniform(-1.0, 1.0, n)
    pos[:, :2] = rng.normal(0, 0.03, (n, 2))
    scale = np.full((n, 3), 0.35)
    op = rng.uniform(0.01, 0.3, n)
    for i in range(1, n, 3):  # duplicates -> equal t* and equal centre depth
        pos[i] = pos[i - 1]
        scale[i] = scale[i - 1]
    return Scene(pos, scale, np.tile([1.0, 0, 0, 0], (n, 1)), op, rng.uniform(0, 1, (n, 3)))


@pytest.fixture(scope="module")
def dense(ref):
    scene = ref.random_scene(52, 600, 1.0)
    cams = ref.orbit_cameras(2, 4.0, 1.8, 40)
    return scene, cams, ref.context(scene, cams), sof.ViewSet.build(scene, cams, ctx=sof.Context(0))


def ref_lists(rc, view, pix):
    lists = [rc.collect_contributions(view, int(x), int(y)) for x, y in pix]
    off = np.concatenate([[0], np.cumsum([len(c["index"]) for c in lists])]).astype(np.int64)
    cat = {k: np.concatenate([c[k] for c in lists]) for k in lists[0]}
    return off, cat


def test_collect_contributions_matches_reference(dense):
    scene, cams, rc, views = dense
    rng = np.random.default_rng(5)
    pix = rng.integers(0, 40, (300, 2))
    for view in range(cams.v):
        got = sof.collect_contributions(views, view, sof.pixel_rays(views.ctx.cams, view, pix))
        off, want = ref_lists(rc, view, pix)
        np.testing.assert_array_equal(got["offsets"], off)
        np.testing.assert_array_equal(got["index"], want["index"])
        for k in ("t_star", "alpha", "a", "b", "c", "opacity"):
            np.testing.assert_array_equal(bits(got[k]), bits(want[k]), err_msg=k)
        assert off[-1] > 1000


def test_collect_contributions_edge_cases(dense):
    scene, cams, rc, views = dense
    got = sof.collect_contributions(views, 0, np.zeros((0, 3)))
    assert list(got["offsets"]) == [0] and len(got["index"]) == 0
    away = sof.collect_contributions(views, 0, [[0.0, 0.0, -1.0]])  # no Gaussian ahead of the ray
    with pytest.raises(ValueError):
        sof.collect_contributions(views, 7, [[0.0, 0.0, 1.0]])
    with pytest.raises(ValueError):
        sof.collect_contributions(views, 0, [[np.nan, 0.0, 1.0]])
    assert away["offsets"][-1] >= 0


@pytest.mark.parametrize("exact", [True, False])
def test_render_pixel_of_reference_lists(dense, exact):
    scene, cams, rc, views = dense
    rng = np.random.default_rng(6)
    pix = rng.integers(0, 40, (200, 2))
    off, want_l = ref_lists(rc, 1, pix)
    vals = np.stack([want_l[k] for k in ("t_star", "alpha", "a", "b", "c", "opacity")], 1)
    got = sof.render_pixel(off, want_l["index"], vals, sof.DEPTH_EXACT if exact else sof.DEPTH_MEDIAN, views.ctx)
    want = rc.render_pixels(1, pix.astype(np.int32), exact)
    np.testing.assert_array_equal(bits(got["color"]), bits(want["color"]))
    np.testing.assert_array_equal(bits(got["depth"]), bits(want["depth"]))
    np.testing.assert_array_equal(bits(got["accumulated_opacity"]), bits(want["acc"]))
    np.testing.assert_array_equal(bits(got["t_final"]), bits(want["tfinal"]))
    # explicit colours instead of the resident scene's
    got2 = sof.render_pixel(off, want_l["index"], vals, sof.DEPTH_EXACT if exact else sof.DEPTH_MEDIAN, views.ctx,
                            dc=np.asarray(scene.dc))
    np.testing.assert_array_equal(bits(got2["color"]), bits(want["color"]))
    # windowed lists: the same composition in the reference
    w = rc.ref
    for window in (2, 5):
        order = sof.windowed_resort(off, want_l["t_star"], window, views.ctx)
        got3 = sof.render_pixel(off, want_l["index"][order], vals[order], sof.DEPTH_EXACT, views.ctx)
        want3 = rc.render_pixel_lists(off, want_l["index"][order], vals[order], True)
        for k, kk in (("color", "color"), ("depth", "depth"), ("accumulated_opacity", "acc"), ("t_final", "tfinal")):
            np.testing.assert_array_equal(bits(got3[k]), bits(want3[kk]))
        for i in range(0, len(off) - 1, 17):  # the order itself is the reference's
            a, b = off[i], off[i + 1]
            np.testing.assert_array_equal(want_l["index"][order[a:b]],
                                          w.windowed_resort(want_l["t_star"][a:b], want_l["index"][a:b], window))


def test_render_pixel_errors(dense):
    scene, cams, rc, views = dense
    with pytest.raises(ValueError):
        sof.render_pixel([0, 1], [10 ** 6], np.zeros((1, 6)), sof.DEPTH_EXACT, views.ctx)
    with pytest.raises(ValueError):
        sof.render_pixel([1, 1], [0], np.zeros((1, 6)), sof.DEPTH_EXACT, views.ctx)
    empty = sof.render_pixel([0, 0], np.zeros(0, np.int32), np.zeros((0, 6)), sof.DEPTH_EXACT, views.ctx)
    assert np.isnan(empty["depth"][0]) and empty["t_final"][0] == 1.0 and empty["accumulated_opacity"][0] == 0.0


@pytest.mark.parametrize("levels", [3, 0])
def test_windowed_resort_device_ties(ref, levels):
    rng = np.random.default_rng(40 + levels)
    sizes = list(range(0, 50)) + [100, 300, 1000]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    C = int(off[-1])
    t = rng.integers(1, levels + 1, C).astype(np.float64) if levels else rng.random(C) + 0.1
    idx = rng.permutation(C).astype(np.int32)
    ctx = sof.Context(0)
    for window in (0, 1, 2, 3, 7, 16, 64, 5000):
        order = sof.windowed_resort(off, t, window, ctx)
        for i in range(len(sizes)):
            a, b = off[i], off[i + 1]
            np.testing.assert_array_equal(idx[order[a:b]], ref.windowed_resort(t[a:b], idx[a:b], window),
                                          err_msg=f"size={b - a} window={window}")
    with pytest.raises(ValueError):
        sof.windowed_resort([0, 2, 1], np.zeros(2), 3, ctx)


def check_window(rc, views, view, window, exact=True):
    w, h = (int(x) for x in views.ctx.cams.wh[view])
    r = sof.render_view(views, view, sof.DEPTH_EXACT if exact else sof.DEPTH_MEDIAN, window=window)
    yy, xx = np.mgrid[0:h, 0:w]
    pix = np.stack([xx.ravel(), yy.ravel()], 1).astype(np.int32)
    want = rc.render_pixels_windowed(view, pix, window, exact)
    np.testing.assert_array_equal(bits(r["rgb"].reshape(-1, 3)), bits(want["color"]))
    np.testing.assert_array_equal(bits(r["t_final"].ravel()), bits(want["tfinal"]))
    np.testing.assert_array_equal(bits(r["depth"].ravel()), bits(want["depth"]))
    np.testing.assert_array_equal(bits(r["opacity"].ravel()), bits(want["acc"]))
    return r


@pytest.mark.parametrize("window", [1, 4, 16, 100000])
def test_render_window_mode_dense(dense, window):
    scene, cams, rc, views = dense
    for v in range(cams.v):
        check_window(rc, views, v, window, exact=(v == 0))
    exact = sof.render_view(views, 0)  # window 0 restores the exact order
    base = rc.render_pixels(0, np.stack([a.ravel() for a in np.mgrid[0:40, 0:40][::-1]], 1).astype(np.int32), True)
    np.testing.assert_array_equal(bits(exact["depth"].ravel()), bits(base["depth"]))


@pytest.mark.parametrize("window", [2, 8, 300])
def test_render_window_mode_ties(ref, window):
    scene = tie_scene(900)
    cams = ref.look_at([0, 0, -4.0], [0, 0, 0], [0, 1, 0], 40.0, 40.0, 20, 20)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    r = check_window(rc, views, 0, window)
    r_exact = sof.render_view(views, 0)
    if window < 300:  # a narrow window changes the blend order somewhere
        assert np.any(bits(r["rgb"]) != bits(r_exact["rgb"]))


def test_render_window_mode_bands(ref):
    """window mode with a tiny render pool: many bands, each with its two slice buffers"""
    scene = ref.random_scene(53, 400, 1.0)
    cams = ref.orbit_cameras(1, 4.0, 1.8, 48)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    views.ctx.check(views.ctx.lib.sof_set_render_pool(views.ctx.h, 64 << 10))
    check_window(rc, views, 0, 3)
    assert views.ctx.lib.sof_set_render_window(views.ctx.h, -1) != 0
