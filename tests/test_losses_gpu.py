"""Training losses (losses.hpp) batched on the device against the
reference compiled in place, bit for bit: per-ray losses, per-sample gradients, the
image losses' scalars (summed in the reference's scan order) and per-pixel gradients.
Edge cases follow the reference's own tests (tests/test_losses.cpp): samples behind the
camera, empty rays, alpha at the clamp, empty visible segments, no median, no surface,
invalid normals, flat normal regions."""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def eq(got, want, what):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape, what
    bad = bits(got) != bits(want)
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} differ"


@pytest.fixture(scope="module")
def ctx():
    return sof.Context(0)


def ragged(rng, rays, max_len):
    lens = rng.integers(0, max_len + 1, rays)
    lens[:3] = [0, 1, max_len]
    return np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)


@pytest.mark.parametrize("attach", [True, False])
def test_distortion_loss(ref, ctx, attach):
    rng = np.random.default_rng(1)
    off = ragged(rng, 300, 40)
    S = int(off[-1])
    alpha = rng.uniform(1 / 255, 0.999, S)
    alpha[::17] = 0.999
    t = rng.uniform(0.3, 20.0, S)
    t[::11] = -rng.uniform(0, 1, len(t[::11]))  # peaks behind the camera
    got = sof.distortion_loss(ctx, off, alpha, t, 0.2, 100.0, attach)
    want = ref.distortion_loss(off, alpha, t, 0.2, 100.0, attach)
    eq(got["loss"], want["loss"], "loss")
    eq(got["d_t"], want["d_t"], "d_t")
    if attach:
        eq(got["d_alpha"], want["d_alpha"], "d_alpha")


def test_extent_loss(ref, ctx):
    rng = np.random.default_rng(2)
    off = ragged(rng, 200, 30)
    S = int(off[-1])
    w = rng.uniform(0, 1, S)
    a = rng.uniform(0.1, 4, S)
    b = rng.uniform(-6, 6, S)
    b[::13] = 1e-13  # singular B
    c = rng.uniform(0, 9, S)
    bound = rng.uniform(0, 3.4, S)
    got = sof.extent_loss(ctx, off, w, a, b, c, bound, 0.2, 100.0)
    want = ref.extent_loss(off, w, a, b, c, bound, 0.2, 100.0)
    assert (want["skipped"] > 0).any()
    np.testing.assert_array_equal(got["skipped"], want["skipped"])
    for k in ("loss", "d_a", "d_b", "d_c", "d_w"):
        eq(got[k], want[k], k)


def test_depth_normal_loss(ref, ctx):
    rng = np.random.default_rng(3)
    off = ragged(rng, 150, 20)
    S = int(off[-1])
    w = rng.uniform(0, 1, S)
    n = rng.normal(size=(S, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    pn = rng.normal(size=(len(off) - 1, 3))
    got = sof.depth_normal_loss(ctx, off, w, n, pn)
    want = ref.depth_normal_loss(off, w, n, pn)
    for k in ("loss", "d_w", "d_n"):
        eq(got[k], want[k], k)


def test_opacity_supervision_loss(ref, ctx):
    rng = np.random.default_rng(4)
    off = ragged(rng, 250, 25)
    S = int(off[-1])
    rc = np.empty((S, 6))
    rc[:, 0] = rng.uniform(0.5, 8, S)             # t*
    rc[:, 1] = rng.uniform(1 / 255, 0.6, S)       # alpha
    rc[:, 2] = rng.uniform(0.5, 3, S)             # a
    rc[:, 3] = -2 * rc[:, 2] * rc[:, 0]           # b (peak at t*)
    rc[:, 4] = rng.uniform(0, 4, S) + rc[:, 3] ** 2 / (4 * rc[:, 2])  # c
    rc[:, 5] = rng.uniform(0.05, 0.99, S)         # opacity
    for r in range(len(off) - 1):                 # sorted by t* inside each ray
        sl = slice(off[r], off[r + 1])
        rc[sl] = rc[sl][np.argsort(rc[sl, 0], kind="stable")]
    low = slice(off[5], off[6])
    rc[low, 1] = 0.01                             # no median on this ray
    depth = rng.uniform(0.5, 8, len(off) - 1)
    depth[::9] = np.nan                           # no surface
    got = sof.opacity_supervision_loss(ctx, off, rc, depth)
    want = ref.opacity_supervision_loss(off, rc, depth)
    np.testing.assert_array_equal(got["defined"], want["defined"])
    assert want["defined"].any() and not want["defined"].all()
    for k in ("loss", "field_value", "d_alpha"):
        eq(got[k], want[k], k)


@pytest.mark.parametrize("per_channel", [False, True])
def test_normal_smoothness_loss(ref, ctx, per_channel):
    rng = np.random.default_rng(5)
    H, W = 37, 53
    n = rng.normal(size=(H, W, 3))
    n /= np.linalg.norm(n, axis=2, keepdims=True)
    n[10:20, 10:30] = [0.0, 0.0, 1.0]             # flat region: |grad N| = 0
    valid = (rng.uniform(size=(H, W)) > 0.15).astype(np.uint8)
    img = rng.uniform(0, 1, (H, W, 3))
    got = sof.normal_smoothness_loss(ctx, n, valid, img, per_channel)
    want = ref.normal_smoothness_loss(n, valid, img, per_channel)
    assert got["pixels_used"] == want["pixels_used"] > 0
    eq(got["loss"], want["loss"], "loss")
    eq(got["d_normal"], want["d_normal"], "d_normal")


def test_l1_and_total(ref, ctx):
    rng = np.random.default_rng(6)
    a, b = rng.uniform(0, 1, (4000, 3)), rng.uniform(0, 1, (4000, 3))
    eq(sof.l1_rgb_loss(ctx, a, b), ref.l1_rgb_loss(a, b), "l1")
    terms = dict(rgb=0.1, distortion=0.2, normal=0.3, extent=0.4, opacity=0.5, smoothness=0.6)
    wts = sof.LossWeights()
    assert sof.total_loss(terms, wts, 100, True) == 0.1
    assert sof.total_loss(terms, wts, 20000, False) == (0.1 + 100.0 * 0.2 + 0.05 * 0.3 + 0.1 * 0.4 + 0.04 * 0.5 +
                                                        0.01 * 0.6)


def test_losses_reject_bad_offsets(ctx):
    with pytest.raises(ValueError, match="non-decreasing"):  # std::invalid_argument
        sof.distortion_loss(ctx, [0, 3, 2], np.ones(3) * 0.5, np.ones(3), 0.2, 100.0)
