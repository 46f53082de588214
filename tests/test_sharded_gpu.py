"""The multi-GPU meshing protocol (sharded.py) end to end on the device: two ranks
(processes) with their own contexts, views split for the label pass and the bisection,
tets split for Marching Tetrahedra with the all-gathered merge. This environment has
one GPU, so both ranks share it and the collectives run over gloo on the host (no
kernel waits on another rank); the driver's scaling run exercises NCCL. The merged mesh
must equal the single-process fused extraction bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _inputs():
    from oracle import restatement as R
    from paper_2506_19139_b200.workloads import Cams, kuhn_lattice
    scene = R.random_scene(57, 60)
    c = R.orbit_cameras(7, 4.0, 1.8, 48)
    cams = Cams(c.R, c.t, c.intr, c.wh, c.nearfar)
    verts, tets = kuhn_lattice(13, -1.3, 1.3)
    return scene, cams, verts, tets


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2506_19139_b200 as sof
        from paper_2506_19139_b200.sharded import ShardedMesher
        scene, cams, verts, tets = _inputs()
        ctx = sof.Context(0)
        ctx.set_scene(scene)
        ctx.set_views(cams)
        ctx.set_tets(verts, tets)
        st = {}
        mesh = ShardedMesher(ctx, rank, world).extract(sof.ExtractOptions(), st)
        out[rank] = (mesh.vertices.copy(), mesh.triangles.copy(), st["crossing_edges"])
        ctx.close()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_extract_on_device(world):
    import paper_2506_19139_b200 as sof
    scene, cams, verts, tets = _inputs()
    ctx = sof.Context(0)
    ctx.set_scene(scene)
    ctx.set_views(cams)
    ctx.set_tets(verts, tets)
    want = sof.extract_resident(ctx, sof.ExtractOptions(), {})
    ctx.close()
    assert len(want.triangles) > 0
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        v, t, ne = res[r]
        assert np.array_equal(v.view(np.uint64), want.vertices.view(np.uint64)), f"rank {r} vertices"
        assert np.array_equal(t, want.triangles), f"rank {r} triangles"
