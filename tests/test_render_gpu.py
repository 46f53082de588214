"""GPU parity of the sorted rasterizer against the compiled reference.

render_pixel / render_depth_map (opacity_field.hpp:192-219, render.hpp:26-51) over
collect_contributions' exhaustive, fully sorted per-pixel lists (:39-61). Colour,
final transmittance, depth (median and exact) and the accumulated opacity at the depth
are bit-identical.
"""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from oracle.refpy import Scene

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def check(ref_ctx, views, view, exact, stats_out=None):
    w, h = (int(x) for x in views.ctx.cams.wh[view])
    r = sof.render_view(views, view, sof.DEPTH_EXACT if exact else sof.DEPTH_MEDIAN, counts=True)
    yy, xx = np.mgrid[0:h, 0:w]
    pix = np.stack([xx.ravel(), yy.ravel()], 1).astype(np.int32)
    want = ref_ctx.render_pixels(view, pix, exact)
    np.testing.assert_array_equal(r["counts"].ravel(), want["ncontrib"])
    np.testing.assert_array_equal(bits(r["rgb"].reshape(-1, 3)), bits(want["color"]))
    np.testing.assert_array_equal(bits(r["t_final"].ravel()), bits(want["tfinal"]))
    np.testing.assert_array_equal(bits(r["depth"].ravel()), bits(want["depth"]))
    np.testing.assert_array_equal(bits(r["opacity"].ravel()), bits(want["acc"]))
    if stats_out is not None:
        stats_out.append(r["stats"])
    return r, want


@pytest.mark.parametrize("exact", [True, False])
def test_render_random_scene(ref, exact):
    scene = ref.random_scene(21, 60, 1.0)
    cams = ref.orbit_cameras(2, 4.0, 1.8, 32)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for v in range(cams.v):
        check(rc, views, v, exact)


def test_render_dense_scene_and_depth_map(ref):
    scene = ref.random_scene(52, 1500, 1.0)
    cams = ref.orbit_cameras(3, 4.0, 1.8, 48)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    st = []
    for v in range(cams.v):
        r, _ = check(rc, views, v, True, st)
        d, o = rc.render_depth_map(v, True)
        np.testing.assert_array_equal(bits(r["depth"]), bits(d))
        np.testing.assert_array_equal(bits(r["opacity"]), bits(o))
    assert sum(int(s[1]) for s in st) > 0


def test_render_long_slices_cta_sort(ref):
    """1500 Gaussians stacked along the optical axis: the centre pixels have more than
    1024 contributions, which take the CTA-wide sort (k_rsort_big); same bits."""
    n = 1500
    rng = np.random.default_rng(3)
    pos = np.zeros((n, 3))
    pos[:, 2] = rng.uniform(-1.0, 1.0, n)
    pos[:, :2] = rng.normal(0, 0.05, (n, 2))
    scene = Scene(pos, np.full((n, 3), 0.3), np.tile([1.0, 0, 0, 0], (n, 1)), rng.uniform(0.02, 0.2, n),
                  rng.uniform(0, 1, (n, 3)))
    cams = ref.look_at([0, 0, -4.0], [0, 0, 0], [0, 1, 0], 40.0, 40.0, 24, 24)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    st = []
    check(rc, views, 0, True, st)
    assert st[0][2] > 0  # some pixels took the CTA-wide sort


def test_render_single_gaussian_disk(ref):
    """RenderDepthMap.SingleGaussianDisk (test_opacity_field.cpp:263-279)."""
    scene = Scene(np.zeros((1, 3)), np.ones((1, 3)), np.array([[1.0, 0, 0, 0]]), np.ones(1), np.zeros((1, 3)))
    f = 0.4 * 32 * 5.0 / 2.0
    cams = ref.look_at([0, 0, -5.0], [0, 0, 0], [0, 1, 0], f, f, 32, 32)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    de, _ = sof.render_depth_map(views, 0, exact=True)
    dm, _ = sof.render_depth_map(views, 0, exact=False)
    assert abs(de[16, 16] - 3.82258) < 0.01 and abs(dm[16, 16] - 5.0) < 0.01
    np.testing.assert_array_equal(np.isnan(de), np.isnan(dm))


@pytest.mark.parametrize("n", [200, 1400, 5000])
def test_render_long_slices_with_ties(ref, n):
    """Hundreds to thousands of contributions per pixel with duplicated Gaussians (equal t*:
    the index breaks the tie, opacity_field.hpp:56-59): slices up to 256 take the warp sort
    and its exact equal-prefix fix-up, up to 4096 the CTA sort in shared memory, longer
    ones the CTA sort in global memory."""
    rng = np.random.default_rng(11)
    pos = np.zeros((n, 3))
    pos[:, 2] = rng.uniform(-1.0, 1.0, n)
    pos[:, :2] = rng.normal(0, 0.03, (n, 2))
    scale = np.full((n, 3), 0.35)
    op = rng.uniform(0.01, 0.05, n)
    for i in range(1, n, 3):  # duplicates -> ties in t*
        pos[i] = pos[i - 1]
        scale[i] = scale[i - 1]
    scene = Scene(pos, scale, np.tile([1.0, 0, 0, 0], (n, 1)), op, rng.uniform(0, 1, (n, 3)))
    cams = ref.look_at([0, 0, -4.0], [0, 0, 0], [0, 1, 0], 40.0, 40.0, 20, 20)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for exact in (True, False):
        st = []
        check(rc, views, 0, exact, st)
        assert st[0][1] > n // 3 * 20 * 4
        assert (st[0][2] > 0) == (n > 256)


@pytest.mark.parametrize("n", [40, 200, 900])
def test_render_near_ties_in_quantised_keys(ref, n):
    """Distinct t* a few ulp apart next to far-away Gaussians: the sort key keeps only the
    top bits of the t* span, so these share a key and the per-run exact (t*, index) fix-up
    orders them; indices run against t* (later Gaussians nearer) to make every run need it."""
    rng = np.random.default_rng(5)
    k = n - n // 8
    pos = np.zeros((n, 3))
    pos[:k, 2] = -np.arange(k) * 1e-13 + rng.integers(0, 3, k) * 1e-14
    pos[:k, :2] = rng.normal(0, 1e-3, (k, 2))
    pos[k:, 2] = rng.uniform(1.0, 3.0, n - k)
    pos[k:, :2] = rng.normal(0, 0.03, (n - k, 2))
    scale = np.full((n, 3), 0.35)
    op = rng.uniform(0.01, 0.05, n)
    scene = Scene(pos, scale, np.tile([1.0, 0, 0, 0], (n, 1)), op, rng.uniform(0, 1, (n, 3)))
    cams = ref.look_at([0, 0, -4.0], [0, 0, 0], [0, 1, 0], 40.0, 40.0, 20, 20)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for exact in (True, False):
        check(rc, views, 0, exact, [])


# ---- normals (render.hpp:58-107) and the `sof render` outputs (sof_cli.cpp:122-130) ------------

def _plain_cam(w, h, cx, cy, f):
    from oracle.refpy import Cameras
    c = Cameras.empty(1)
    c.R[0] = np.eye(3)
    c.intr[0] = (f, f, cx, cy)
    c.wh[0] = (w, h)
    c.nearfar[0] = (0.2, 100.0)
    return c


def _one_gaussian():
    return Scene(np.zeros((1, 3)), np.ones((1, 3)), np.array([[1.0, 0, 0, 0]]), np.ones(1), np.zeros((1, 3)))


def test_render_normals_bitexact(ref):
    scene = ref.random_scene(52, 1500, 1.0)
    cams = ref.orbit_cameras(2, 4.0, 1.8, 48)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for v in range(cams.v):
        r = sof.render_view(views, v, sof.DEPTH_EXACT, normals=True)
        d, _ = rc.render_depth_map(v, True)
        np.testing.assert_array_equal(bits(r["depth"]), bits(d))
        n_ref, ok_ref = rc.normal_from_depth(v, d)
        np.testing.assert_array_equal(r["normal_valid"], ok_ref)
        np.testing.assert_array_equal(bits(r["normal"]), bits(n_ref))
        assert ok_ref.sum() > 100
        # the same from a host depth map
        n2, ok2 = sof.normal_from_depth(views, v, d)
        np.testing.assert_array_equal(bits(n2), bits(n_ref))
        np.testing.assert_array_equal(ok2, ok_ref)


def test_normal_from_depth_known_answers(ref):
    """NormalFromDepth.FrontoParallelPlane / SlantedPlane / IsolatedPixelInvalid
    (test_opacity_field.cpp:285-327)."""
    ctx = sof.Context(0)
    cam = _plain_cam(16, 16, 8, 8, 20)
    views = sof.ViewSet.build(_one_gaussian(), cam, ctx=ctx)
    yy, xx = np.mgrid[0:16, 0:16]
    d = np.stack([(xx + 0.5 - 8) / 20, (yy + 0.5 - 8) / 20, np.ones_like(xx, float)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    n, ok = sof.normal_from_depth(views, 0, 5.0 / d[..., 2])
    assert ok[8, 8] and np.allclose(n[8, 8], (0, 0, -1), atol=1e-9)
    rc = ref.context(_one_gaussian(), cam)
    n_ref, ok_ref = rc.normal_from_depth(0, 5.0 / d[..., 2])
    np.testing.assert_array_equal(bits(n), bits(n_ref))
    np.testing.assert_array_equal(ok, ok_ref)

    cam = _plain_cam(32, 32, 16, 16, 60)
    views = sof.ViewSet.build(_one_gaussian(), cam, ctx=ctx)
    yy, xx = np.mgrid[0:32, 0:32]
    d = np.stack([(xx + 0.5 - 16) / 60, (yy + 0.5 - 16) / 60, np.ones_like(xx, float)], -1)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    npl = np.array([0.3, -0.2, -1.0]) / np.linalg.norm([0.3, -0.2, -1.0])
    n, ok = sof.normal_from_depth(views, 0, -5.0 / (d @ npl))
    assert ok[16, 16] and np.linalg.norm(n[16, 16] - npl) < 1e-3

    cam = _plain_cam(8, 8, 4, 4, 500)
    views = sof.ViewSet.build(_one_gaussian(), cam, ctx=ctx)
    depth = np.full((8, 8), np.nan)
    depth[3, 3] = 5.0
    n, ok = sof.normal_from_depth(views, 0, depth)
    assert ok.sum() == 0 and not n.any()


def test_gaussian_normal(ref):
    """GaussianNormal.RadialAndFallback / AlwaysFacesCamera (test_opacity_field.cpp:330-351)
    and bit-exact against the reference on random queries."""
    flat = Scene(np.zeros((2, 3)), np.array([[1.0, 1, 1], [1.0, 1.0, 0.2]]), np.tile([1.0, 0, 0, 0], (2, 1)),
                 np.ones(2), np.zeros((2, 3)))
    cam = _plain_cam(16, 16, 8, 8, 20)
    views = sof.ViewSet.build(flat, cam, ctx=sof.Context(0))
    o, dvec = np.array([[0, 0, -5.0]]), np.array([[0, 0, 1.0]])
    n = sof.gaussian_normal(views.ctx, [0], o, dvec, [6.0])
    assert np.allclose(n[0], (0, 0, -1), atol=1e-12)
    n = sof.gaussian_normal(views.ctx, [1], o, dvec, [5.0])
    assert abs(abs(n[0, 2]) - 1.0) < 1e-12 and n[0] @ dvec[0] <= 0.0

    scene = ref.random_scene(27, 300, 1.0)
    views = sof.ViewSet.build(scene, cam, ctx=sof.Context(0))
    rc = ref.context(scene, cam)
    rng = np.random.default_rng(9)
    m = 2000
    g = rng.integers(0, 300, m).astype(np.int32)
    o = np.column_stack([rng.uniform(-2, 2, (m, 2)), np.full(m, -6.0)])
    dv = np.column_stack([rng.uniform(-0.2, 0.2, (m, 2)), np.ones(m)])
    dv /= np.linalg.norm(dv, axis=1, keepdims=True)
    t = rng.uniform(2.0, 8.0, m)
    got = sof.gaussian_normal(views.ctx, g, o, dv, t)
    np.testing.assert_array_equal(bits(got), bits(rc.gaussian_normals(g, o, dv, t)))
    assert (np.einsum("ij,ij->i", got, dv) <= 1e-12).all()


def test_render_maps_files_byte_identical(ref, tmp_path):
    """`sof render` per-view outputs (sof_cli.cpp:122-130): depth + opacity map and
    normal map files, byte-identical to the reference's."""
    scene = ref.random_scene(21, 600, 1.0)
    cams = ref.orbit_cameras(2, 4.0, 1.8, 40)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for v in range(cams.v):
        for exact in (True, False):
            a, b = tmp_path / "a_d.sofmap", tmp_path / "a_n.sofmap"
            c, d = tmp_path / "b_d.sofmap", tmp_path / "b_n.sofmap"
            sof.render_maps(views, v, str(a), str(b), exact=exact)
            rc.render_maps(v, str(c), str(d), exact=exact)
            assert a.read_bytes() == c.read_bytes()
            assert b.read_bytes() == d.read_bytes()


@pytest.mark.parametrize("pool", [1 << 16, 3 << 20])
def test_render_bands_bit_identical(ref, pool):
    """A small scratch budget splits the frame into bands of tiles (one tile per band at
    64 KiB): every output bit-identical to the single-band render and to the reference."""
    scene = ref.random_scene(52, 1500, 1.0)
    cams = ref.orbit_cameras(1, 4.0, 1.8, 48)
    rc = ref.context(scene, cams)
    ctx = sof.Context(0)
    views = sof.ViewSet.build(scene, cams, ctx=ctx)
    whole = sof.render_view(views, 0, sof.DEPTH_EXACT)
    ctx.check(ctx.lib.sof_set_render_pool(ctx.h, pool))
    banded, _ = check(rc, views, 0, True)
    for k in ("rgb", "t_final", "depth", "opacity"):
        np.testing.assert_array_equal(bits(banded[k]), bits(whole[k]))
    ctx.check(ctx.lib.sof_set_render_pool(ctx.h, 0))


@pytest.mark.parametrize("dist", [1.2, 0.6])
def test_render_cameras_inside_scene(ref, dist):
    """Cameras inside the Gaussian cloud: boxes crossing the camera plane (every tile),
    Gaussians behind the camera (no tile) and non-elliptic conics (never culled) next to
    ordinary ellipses; every output bit-identical."""
    scene = ref.random_scene(71, 400, 1.0)
    cams = ref.orbit_cameras(3, dist, 1.8, 40)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for v in range(cams.v):
        for exact in (True, False):
            check(rc, views, v, exact)


def test_render_views_batch(ref):
    """sof_render_views: one call over several views equals the per-view renders (bits)."""
    scene = ref.random_scene(61, 300, 1.0)
    cams = ref.orbit_cameras(3, 4.0, 1.8, 40)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    batch = sof.render_views(views, 1, 2)
    for k, v in enumerate((1, 2)):
        one = sof.render_view(views, v)
        for key in ("depth", "opacity", "rgb", "t_final"):
            np.testing.assert_array_equal(bits(batch[k][key]), bits(one[key]), err_msg=key)
    with pytest.raises(ValueError):
        sof.render_views(views, 2, 2)
