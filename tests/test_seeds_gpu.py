"""build_seed_points (seed_points.hpp:41-87) on the device — the producer side of the
tetra input: centres + 8 oriented E-box corners, 1e-9-grid dedup in
insertion order, dead cutoff, bounding variants. Bit-exact against the reference."""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from oracle.refpy import Scene

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _scene(ref, seed, n):
    s = ref.random_scene(seed, n, 1.0)
    s.opacity[::6] = 0.002                 # dead (filtered opacity < 1/255)
    s.opacity[1::11] = 1.0 / 255.0         # exactly at the threshold
    s.pos[5::17] = s.pos[4::17][: len(s.pos[5::17])]      # duplicated centres
    s.scale[5::17] = s.scale[4::17][: len(s.scale[5::17])]
    s.rot[5::17] = s.rot[4::17][: len(s.rot[5::17])]
    s.pos[7::19] += 3e-10                  # within the 1e-9 grid of a neighbour? (key rounding)
    s.scale[9] = [1e300, 1e300, 1.0]       # corners overflow to inf: skipped
    return s


@pytest.mark.parametrize("variant", [sof.SEED_STP, sof.SEED_THREE_SIGMA, sof.SEED_STRETCHED_SIGMA])
@pytest.mark.parametrize("cutoff", [sof.SEED_CUT_NONE, sof.SEED_CUT_DEAD])
@pytest.mark.parametrize("filter_scale", [0.0, 0.003])
def test_seed_points_bitexact(ref, variant, cutoff, filter_scale):
    scene = _scene(ref, 31, 700)
    cams = ref.orbit_cameras(1, 4.0, 1.8, 32)
    rc = ref.context(scene, cams)
    ctx = sof.Context(0)
    ctx.set_scene(scene)
    got = sof.build_seed_points(ctx, variant, cutoff, filter_scale)
    pts, prov = rc.seed_points(variant, cutoff, filter_scale)
    assert len(pts) > 1000
    np.testing.assert_array_equal(bits(got.points), bits(pts))
    np.testing.assert_array_equal(got.provenance, prov)


def test_seed_points_no_live_gaussians(ref):
    n = 5
    scene = Scene(np.zeros((n, 3)), np.ones((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), np.full(n, 0.001),
                  np.zeros((n, 3)))
    ctx = sof.Context(0)
    ctx.set_scene(scene)
    with pytest.raises(RuntimeError, match="no live Gaussians"):
        sof.build_seed_points(ctx, sof.SEED_STP, sof.SEED_CUT_DEAD)
    got = sof.build_seed_points(ctx, sof.SEED_STP, sof.SEED_CUT_NONE)  # centres survive
    assert len(got.points) == 1 and got.provenance.tolist() == [0]
