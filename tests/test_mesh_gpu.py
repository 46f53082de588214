"""GPU parity of the Marching-Tetrahedra mesher against the compiled reference.

Bit-exact: crossing edges and their numbering (first appearance), lerp and refined
vertex positions, triangle indices and winding, welded mesh, and the PLY bytes of
write_mesh_ply (io_mesh.hpp:55-73). Reference: marching_tets.hpp:29-114,
mesh.hpp:36-79, extract.hpp:59-78.
"""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from paper_2506_19139_b200.workloads import kuhn_lattice
from oracle.refpy import ALL

pytestmark = pytest.mark.gpu

SINGLE = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1.0]])


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("opa", [[0.4, 0.4, 0.4, 0.6], [0.4, 0.4, 0.6, 0.6], [0.6, 0.7, 0.8, 0.9],
                                 [0.1, 0.2, 0.3, 0.4], [0.4, 0.6, 0.4, 0.4], [0.6, 0.6, 0.6, 0.4],
                                 [0.6, 0.4, 0.6, 0.4], [0.5, 0.4, 0.4, 0.4]])
def test_single_tet_cases(ref, opa):
    """MarchingTets.* (test_mesher.cpp:75-101) on every case shape."""
    grid = sof.TetGrid(SINGLE, np.array([[0, 1, 2, 3]], np.int32), np.array(opa))
    got = sof.marching_tets(grid)
    want = ref.marching_tets(SINGLE, grid.tetrahedra, grid.opacity)
    np.testing.assert_array_equal(got.edges, want["edges"])
    np.testing.assert_array_equal(bits(got.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(got.triangles, want["triangles"])


@pytest.fixture(scope="module")
def lattice_case(ref):
    scene = ref.random_scene(55, 40, 1.0)
    cams = ref.orbit_cameras(5, 4.0, 1.8, 64)
    verts, tets = kuhn_lattice(14, -1.3, 1.3)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    return scene, cams, rc, views, verts, tets


def test_march_random_field(ref, lattice_case):
    _, _, _, _, verts, tets = lattice_case
    rng = np.random.default_rng(5)
    opa = rng.uniform(0.2, 0.8, len(verts))
    opa[::17] = 0.5  # exact iso-value: inside (>= 0.5), s = 0 lerp
    got = sof.marching_tets(sof.TetGrid(verts, tets, opa))
    want = ref.marching_tets(verts, tets, opa)
    np.testing.assert_array_equal(got.edges, want["edges"])
    np.testing.assert_array_equal(bits(got.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(got.triangles, want["triangles"])


@pytest.mark.parametrize("mask", [31, 0, 9, 27])
def test_refine_bitexact(lattice_case, mask):
    scene, cams, rc, views, verts, tets = lattice_case
    rev = rc.evaluator(mask)
    opa = rev.label_grid(verts, True)
    m = sof.marching_tets(sof.TetGrid(verts, tets, opa), ctx=views.ctx)
    ev = sof.FieldEvaluator(scene, views, sof.EvalStrategies.from_mask(mask))
    rev.reset_counters()
    want = rev.refine(verts, m.edges, m.vertices, 8)
    sof.binary_search_refine(m, sof.TetGrid(verts, tets, opa), ev, 8)
    np.testing.assert_array_equal(bits(m.vertices), bits(want))
    assert ev.counters() == rev.counters()


def test_refine_zero_iterations_keeps_lerp(lattice_case):
    scene, cams, rc, views, verts, tets = lattice_case
    opa = rc.evaluator(ALL).label_grid(verts, True)
    m = sof.marching_tets(sof.TetGrid(verts, tets, opa), ctx=views.ctx)
    before = m.vertices.copy()
    sof.binary_search_refine(m, sof.TetGrid(verts, tets, opa), sof.FieldEvaluator(scene, views, sof.EvalStrategies.all()), 0)
    np.testing.assert_array_equal(bits(m.vertices), bits(before))


def test_assemble_weld_and_degenerate(ref):
    """AssembleMesh.WeldAndDegenerate / EmptyInput (test_mesher.cpp:139-153)."""
    verts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1 + 1e-9, 0, 0]], float)
    tris = np.array([[0, 1, 2], [0, 3, 2], [0, 1, 3]], np.int32)
    got = sof.assemble_mesh(verts, tris)
    want = ref.assemble(verts, tris)
    assert len(got.vertices) == 3 and len(got.triangles) == 2
    np.testing.assert_array_equal(bits(got.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(got.triangles, want["triangles"])
    empty = sof.assemble_mesh(np.zeros((0, 3)), np.zeros((0, 3), np.int32))
    assert len(empty.vertices) == 0 and len(empty.triangles) == 0


def test_assemble_random_duplicates(ref):
    rng = np.random.default_rng(9)
    base = rng.uniform(-1, 1, (500, 3))
    verts = np.concatenate([base, base[rng.integers(0, 500, 300)] + rng.normal(0, 2e-8, (300, 3))])
    verts = verts[rng.permutation(len(verts))]
    tris = rng.integers(0, len(verts), (2000, 3)).astype(np.int32)
    got = sof.assemble_mesh(verts, tris)
    want = ref.assemble(verts, tris)
    np.testing.assert_array_equal(bits(got.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(got.triangles, want["triangles"])


@pytest.mark.parametrize("mask", [31, 0, 23, 27, 19])
def test_extract_fused_ply_bytes(ref, lattice_case, tmp_path, mask):
    """The fused device pipeline reproduces extract_mesh's mesh byte for byte
    (Extract.DeterministicAcrossThreadCounts, test_mesher.cpp:242-257)."""
    scene, cams, rc, views, verts, tets = lattice_case
    want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
    stats = {}
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets),
                            sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask)), stats)
    assert len(want["triangles"]) > 0
    np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, want["triangles"])
    assert stats["pairs"] == int(want["counters"][0])
    assert stats["point_view_evals"] == int(want["counters"][1])
    p1, p2 = str(tmp_path / "gpu.ply"), str(tmp_path / "ref.ply")
    sof.write_mesh_ply(mesh, p1)
    ref.write_mesh_ply(want["vertices"], want["triangles"], p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()


def test_extract_delaunay_grid(ref):
    """The reference's own seeds + Delaunay tetra input (seed_points.hpp, delaunay.hpp)."""
    scene = ref.random_scene(55, 15, 1.0)
    cams = ref.orbit_cameras(3, 4.0, 1.8, 64)
    rc = ref.context(scene, cams)
    grid = rc.seed_delaunay()
    full = rc.extract_full(ALL)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(grid["vertices"], grid["tets"]))
    np.testing.assert_array_equal(bits(mesh.vertices), bits(full["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, full["triangles"])


def test_sharded_path_single_rank_matches_fused(ref, lattice_case):
    """The view-sharded step (sharded.py over the device primitives) on one rank equals
    the fused sof_extract bit for bit."""
    import torch
    from paper_2506_19139_b200.sharded import ShardedMesher
    scene, cams, rc, views, verts, tets = lattice_case
    views.ctx.set_tets(verts, tets)
    fused = sof.extract_resident(views.ctx, sof.ExtractOptions(), {})
    mesher = ShardedMesher(views.ctx, 0, 1)
    st = {}
    mesh = mesher.extract(sof.ExtractOptions(), st)
    np.testing.assert_array_equal(bits(mesh.vertices), bits(fused.vertices))
    np.testing.assert_array_equal(mesh.triangles, fused.triangles)
    torch.cuda.synchronize()


def test_async_tets_upload(lattice_case):
    """sof_set_tets_async: the same mesh as the synchronous upload; a bad index is
    reported by the extract that consumes the tets."""
    scene, cams, rc, views, verts, tets = lattice_case
    ctx = views.ctx
    ctx.set_tets(verts, tets)
    want = sof.extract_resident(ctx, sof.ExtractOptions(), {})
    for _ in range(2):  # twice: a pending upload is replaced cleanly
        ctx.set_tets(verts, tets, async_copy=True)
    got = sof.extract_resident(ctx, sof.ExtractOptions(), {})
    np.testing.assert_array_equal(bits(got.vertices), bits(want.vertices))
    np.testing.assert_array_equal(got.triangles, want.triangles)
    bad = tets.copy()
    bad[len(bad) // 2, 1] = len(verts)
    ctx.set_tets(verts, bad, async_copy=True)
    with pytest.raises(ValueError, match="out of range"):
        sof.extract_resident(ctx, sof.ExtractOptions(), {})
    ctx.set_tets(verts, tets)
    again = sof.extract_resident(ctx, sof.ExtractOptions(), {})
    np.testing.assert_array_equal(again.triangles, want.triangles)


def test_extract_many_views_grouped_bisection(ref):
    """More views than one classification group (kGroupViews = 32): the grouped bisection
    keeps the reference's per-point view order, counters included."""
    scene = ref.random_scene(57, 60, 1.0)
    cams = ref.orbit_cameras(70, 4.0, 1.8, 48)
    verts, tets = kuhn_lattice(12, -1.3, 1.3)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    for mask in (31, 23):
        want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
        stats = {}
        mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets),
                                sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask)), stats)
        assert len(want["triangles"]) > 0
        np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
        np.testing.assert_array_equal(mesh.triangles, want["triangles"])
        assert stats["pairs"] == int(want["counters"][0])
        assert stats["point_view_evals"] == int(want["counters"][1])
        # label: one launch per view; bisection: one per 32-view group and iteration
        assert stats["eval_launches"] == 70 + 8 * 3, stats["eval_launches"]


@pytest.mark.parametrize("budget", [0, 12_000])
def test_extract_past_cache_budget(ref, budget):
    """Views past the record / tile-list cache budget are rebuilt in two scratch slots
    while earlier views still evaluate (prep stream ahead of the eval stream): same mesh
    and counters as the reference."""
    scene = ref.random_scene(61, 40, 1.0)
    cams = ref.orbit_cameras(40, 4.0, 1.8, 48)
    verts, tets = kuhn_lattice(12, -1.3, 1.3)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    views.ctx.check(views.ctx.lib.sof_set_cache_budget(views.ctx.h, budget))
    want = rc.extract_tetgrid(verts, tets, strategies=31, iterations=8)
    stats = {}
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets), sof.ExtractOptions(), stats)
    np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, want["triangles"])
    assert stats["pairs"] == int(want["counters"][0])
    assert stats["point_view_evals"] == int(want["counters"][1])


def test_assemble_overflowing_weld_keys(ref):
    """llround(p * 1e7) beyond 2^63 is x86's 0x8000000000000000 for either sign in the
    reference binary (mesh.hpp:57-62): such vertices weld together on that axis."""
    rng = np.random.default_rng(8)
    verts = rng.normal(size=(300, 3))
    verts[::7, 0] = 2e12
    verts[1::7, 0] = -3e12
    verts[2::7, 1:] = verts[3::7, 1:][: len(verts[2::7])]
    verts[3::7, 0] = 5e12
    tris = rng.integers(0, len(verts), (500, 3)).astype(np.int32)
    got = sof.assemble_mesh(verts, tris)
    want = ref.assemble(verts, tris)
    np.testing.assert_array_equal(bits(got.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(got.triangles, want["triangles"])


@pytest.mark.parametrize("world", [2, 3, 7])
def test_tet_sharded_march_merge(lattice_case, world):
    """Tet-sharded Marching Tetrahedra (sharded.py): each shard marches a contiguous tet
    range (sof_march_range_resident) and the gathered lists are merged
    (sof_march_merge_dev) into exactly the whole-grid march: same first-appearance edge
    numbering, lerp vertex bits, triangles and winding (marching_tets.hpp:29-84)."""
    import torch
    from paper_2506_19139_b200 import _lib as L
    from paper_2506_19139_b200.sharded import GpuBackend, view_range
    scene, cams, rc, views, verts, tets = lattice_case
    ctx = views.ctx
    ctx.set_tets(verts, tets)
    sof.extract_resident(ctx, sof.ExtractOptions(), {})  # leaves the merged labels resident
    b = GpuBackend(ctx)
    b.march()
    want = (ctx.result(L.R_EDGES, np.int32, 2), ctx.result(L.R_EDGE_VERTS, np.float64, 3),
            ctx.result(L.R_TRIANGLES, np.int32, 3))
    assert len(want[2]) > 100
    es, ts, ec, tc = [], [], [], []
    for r in range(world):
        ne, nt = b.march_range(*view_range(r, world, len(tets)))
        e, t = b.march_local(ne, nt)
        es.append(e.clone())
        ts.append(t.clone())
        ec.append(ne)
        tc.append(nt)
    assert sum(ec) >= len(want[0])  # edges on shard boundaries appear in both shards
    ne, nt = b.march_merge(ec, torch.cat(es), tc, torch.cat(ts))
    got = (ctx.result(L.R_EDGES, np.int32, 2), ctx.result(L.R_EDGE_VERTS, np.float64, 3),
           ctx.result(L.R_TRIANGLES, np.int32, 3))
    assert (ne, nt) == (len(want[0]), len(want[2]))
    np.testing.assert_array_equal(got[0], want[0])
    np.testing.assert_array_equal(bits(got[1]), bits(want[1]))
    np.testing.assert_array_equal(got[2], want[2])


@pytest.mark.parametrize("dist", [4.0, 1.0])
def test_bisection_cache_truncated_lists(ref, dist):
    """Views past the cache budget get bisection caches: tile lists truncated to the
    depths the midpoints can reach, with compact records (bisect_cache_views). Same mesh
    and exact counters as the reference; with cameras inside the lattice (dist 1.0) some
    crossing edges reach the camera plane and those views keep the per-view path."""
    scene = ref.random_scene(63, 60, 1.0)
    cams = ref.orbit_cameras(12, dist, 1.8, 48)
    verts, tets = kuhn_lattice(12, -1.3, 1.3)
    rc = ref.context(scene, cams)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    views.ctx.check(views.ctx.lib.sof_set_cache_budget(views.ctx.h, 0))
    want = rc.extract_tetgrid(verts, tets, strategies=31, iterations=8)
    assert len(want["triangles"]) > 0
    stats = {}
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets), sof.ExtractOptions(), stats)
    np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, want["triangles"])
    assert stats["pairs"] == int(want["counters"][0])
    assert stats["point_view_evals"] == int(want["counters"][1])
    # later extracts on the same context rebuild the truncated caches into the buffers of
    # the first one (in place, no allocation) and still match, counters included
    for _ in range(2):
        st2 = {}
        mesh2 = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets), sof.ExtractOptions(), st2)
        np.testing.assert_array_equal(bits(mesh2.vertices), bits(want["vertices"]))
        np.testing.assert_array_equal(mesh2.triangles, want["triangles"])
        assert st2["pairs"] == int(want["counters"][0])
        assert st2["point_view_evals"] == int(want["counters"][1])


@pytest.mark.parametrize("mask", [31, 23])
def test_extract_residuals(ref, lattice_case, mask):
    """ExtractOptions::compute_residuals (extract.hpp:65-72): level_set_residuals with the
    naive exact evaluator at the refined vertices, carried through the weld (mesh.hpp:66);
    every residual bit-identical to the reference's."""
    from oracle.refpy import NAIVE
    scene, cams, rc, views, verts, tets = lattice_case
    want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
    exact = rc.evaluator(NAIVE)
    res = np.abs(exact.value_at(want["refined"]) - 0.5)
    wmesh = ref.assemble(want["refined"], want["march_triangles"], res)
    mesh = sof.extract_mesh(scene, views, sof.TetGrid(verts, tets),
                            sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask), compute_residuals=True))
    np.testing.assert_array_equal(bits(mesh.vertices), bits(wmesh["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, wmesh["triangles"])
    assert len(mesh.residuals) == len(mesh.vertices) > 0
    np.testing.assert_array_equal(bits(mesh.residuals), bits(wmesh["residuals"]))
    # the stand-alone weld with a residual passthrough
    m2 = sof.assemble_mesh(want["refined"], want["march_triangles"], residuals=res, ctx=views.ctx)
    np.testing.assert_array_equal(bits(m2.residuals), bits(wmesh["residuals"]))


@pytest.mark.parametrize("seed, count", [(55, 15), (56, 30)])
def test_extract_mesh_reference_signature(ref, seed, count, tmp_path):
    """extract_mesh(gaussians, views, opt) (extract.hpp:35-86) with its own producer:
    build_seed_points on the device, delaunay_tetrahedralize on the host (sof_tetrahedralize,
    the reference's Bowyer-Watson tet list exactly), then the device pipeline; the PLY
    bytes equal the reference's extract_mesh."""
    scene = ref.random_scene(seed, count, 1.0)
    cams = ref.orbit_cameras(3, 4.0, 1.8, 64)
    rc = ref.context(scene, cams)
    grid_ref = rc.seed_delaunay(bounding=0, cutoff=1)
    full = rc.extract_full(ALL)
    views = sof.ViewSet.build(scene, cams, ctx=sof.Context(0))
    seeds = sof.build_seed_points(views.ctx, sof.SEED_STP, sof.SEED_CUT_DEAD)
    grid = sof.delaunay_tetrahedralize(seeds.points, views.ctx)
    np.testing.assert_array_equal(bits(grid.vertices), bits(grid_ref["vertices"]))
    np.testing.assert_array_equal(grid.tetrahedra, grid_ref["tets"])
    st = {}
    mesh = sof.extract_mesh(scene, views, opt=sof.ExtractOptions(), stats=st)
    assert st["tetrahedra"] == len(grid_ref["tets"])
    np.testing.assert_array_equal(bits(mesh.vertices), bits(full["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, full["triangles"])
    p1, p2 = str(tmp_path / "gpu.ply"), str(tmp_path / "ref.ply")
    sof.write_mesh_ply(mesh, p1)
    ref.write_mesh_ply(full["vertices"], full["triangles"], p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()


def test_tetrahedralize_errors(ref):
    ctx = sof.Context(0)
    with pytest.raises(ValueError, match="need at least 4 points"):
        sof.delaunay_tetrahedralize(np.zeros((3, 3)), ctx)
    with pytest.raises(ValueError, match="degenerate"):
        sof.delaunay_tetrahedralize(np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0], [2, 3, 0.0]]), ctx)


def _sphere_points(n, seed):
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    return d / np.linalg.norm(d, axis=1, keepdims=True)


@pytest.mark.parametrize("case", ["random50", "random3000", "lattice6", "sphere400", "clustered", "uniform10k"])
def test_device_delaunay_matches_reference(ref, case):
    """sof_tetrahedralize (the device Bowyer-Watson) returns the reference's tet list
    (delaunay.hpp:52-142) in the reference's order, on random, cospherical (lattice,
    sphere) and clustered point sets."""
    rng = np.random.default_rng(7)
    if case == "random50":
        pts = rng.random((50, 3))
    elif case == "random3000":
        pts = rng.normal(size=(3000, 3))
    elif case == "lattice6":
        pts = np.stack(np.meshgrid(*[np.arange(6.0)] * 3, indexing="ij"), -1).reshape(-1, 3)
    elif case == "sphere400":
        pts = _sphere_points(400, 3)
    elif case == "uniform10k":
        pts = rng.random((10000, 3))
    else:
        # two scales 10^4 apart (the reference's slivers and holes; it slows down
        # super-linearly on such sets, so a small one)
        pts = np.concatenate([rng.normal(scale=1e-3, size=(40, 3)), rng.normal(scale=10.0, size=(40, 3))])
    want = ref.delaunay(pts)
    got = sof.delaunay_tetrahedralize(pts, sof.Context(0))
    np.testing.assert_array_equal(got.tetrahedra, want)
