"""The library-owned multi-GPU meshing step (k_comm.cu, include/sof_cuda.h sof_comm_*).

* NCCL, world size 1: a context with an attached NCCL communicator runs the sharded
  protocol (NCCL collectives on the library stream) and produces the single-GPU mesh bit
  for bit.
* The same C++ protocol with 2, 3 and 5 ranks on one GPU through the in-process
  communicator (sof_comm_init_local): one context per rank, one host thread per rank,
  collectives as device-side reductions between the contexts; every rank's mesh equals
  the single-context mesh and the reference's (with and without pruning).
"""
import threading

import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from paper_2506_19139_b200.workloads import kuhn_lattice

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def case(ref):
    scene = ref.random_scene(55, 60, 1.0)
    cams = ref.orbit_cameras(9, 4.0, 1.8, 64)
    verts, tets = kuhn_lattice(14, -1.3, 1.3)
    rc = ref.context(scene, cams)
    return scene, cams, verts, tets, rc


def make_ctx(scene, cams, verts, tets):
    ctx = sof.Context(0)
    ctx.set_scene(scene)
    ctx.set_views(cams)
    ctx.set_tets(verts, tets)
    return ctx


@pytest.mark.parametrize("mask", [31, 23])
def test_nccl_world1_matches_single_gpu(case, mask):
    scene, cams, verts, tets, rc = case
    want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
    ctx = make_ctx(scene, cams, verts, tets)
    ctx.comm_init(sof.Context.comm_unique_id(), 1, 0)
    assert ctx.comm_info() == ("nccl", 1, 0)
    st = {}
    mesh = sof.extract_resident(ctx, sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask)), st)
    np.testing.assert_array_equal(bits(mesh.vertices), bits(want["vertices"]))
    np.testing.assert_array_equal(mesh.triangles, want["triangles"])
    assert st["pairs"] == int(want["counters"][0])  # one rank: the reference's counters
    ctx.comm_destroy()
    assert ctx.comm_info()[0] == "none"
    ctx.close()


@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("mask", [31, 23])
def test_local_ranks_match_reference(case, world, mask):
    scene, cams, verts, tets, rc = case
    want = rc.extract_tetgrid(verts, tets, strategies=mask, iterations=8)
    ctxs = [make_ctx(scene, cams, verts, tets) for _ in range(world)]
    sof.Context.comm_init_local(ctxs)
    assert [c.comm_info() for c in ctxs] == [("local", world, r) for r in range(world)]
    meshes, stats, errors = [None] * world, [dict() for _ in range(world)], []

    def run(r):
        try:
            meshes[r] = sof.extract_resident(ctxs[r], sof.ExtractOptions(strategies=sof.EvalStrategies.from_mask(mask)),
                                             stats[r])
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errors, errors
    for r in range(world):
        np.testing.assert_array_equal(bits(meshes[r].vertices), bits(want["vertices"]))
        np.testing.assert_array_equal(meshes[r].triangles, want["triangles"])
        assert stats[r]["crossing_edges"] == len(want["edges"]) if "edges" in want else True
    # views are split: every rank evaluated only part of the pairs
    assert all(s["label_pairs"] < int(want["counters"][0]) for s in stats)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("world", [1, 3])
def test_local_ranks_residuals(case, world):
    """compute_residuals on the sharded step: the per-view |T-0.5| values are MIN-reduced
    across the view shards, then every rank welds the same residuals as one context."""
    scene, cams, verts, tets, rc = case
    opt = sof.ExtractOptions(compute_residuals=True)
    one = make_ctx(scene, cams, verts, tets)
    want = sof.extract_resident(one, opt, {})
    assert len(want.residuals) == len(want.vertices) > 0
    ctxs = [make_ctx(scene, cams, verts, tets) for _ in range(world)]
    sof.Context.comm_init_local(ctxs)
    meshes, errors = [None] * world, []

    def run(r):
        try:
            meshes[r] = sof.extract_resident(ctxs[r], opt, {})
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not errors, errors
    for m in meshes:
        np.testing.assert_array_equal(bits(m.vertices), bits(want.vertices))
        np.testing.assert_array_equal(bits(m.residuals), bits(want.residuals))
    for c in ctxs + [one]:
        c.close()
