"""View-sharded meshing step across GPUs (one process per GPU, torch.distributed).

The reference evaluates views sequentially (field_eval.hpp:145-176); here rank r
owns the contiguous view range [r V / R, (r + 1) V / R) and the per-view work never
crosses ranks. Two exchange points reproduce the sequential results exactly:

* label pass — with pruning, a vertex's value is the min over the views up to the
  first view in which it becomes exterior (later views are skipped,
  field_eval.hpp:147). Each rank labels its own range with local pruning; an
  all-reduce MIN of (exterior_r ? r : R) gives the first exterior rank r*; ranks
  after r* mask their minima to +inf; an all-reduce MIN of the minima is then the
  sequential min. Without pruning it is a plain MIN / MAX.
* bisection — classification only (marching_tets.hpp:107-110): each iteration every
  rank classifies all midpoints against its views, an all-reduce MAX merges the
  exterior flags, and every rank updates the brackets identically.

* Marching Tetrahedra — the tets are split into contiguous ranges: each rank marches
  its range (edges numbered by first appearance within it), the edge and triangle
  lists are all-gathered in rank order, and every rank merges them: an edge's global
  first appearance lies in the first range that contains it, so the global numbering
  is the first-appearance numbering of the concatenated lists (marching_tets.hpp:31-44).

The bisection brackets and the weld are replicated (each rank holds the merged march). The backend performs the per-rank device work
(GpuBackend: libsof_cuda.so on CUDA tensors; tests/test_sharded_cpu.py supplies a
CPU backend to exercise the same protocol over gloo).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from .api import Context, ExtractOptions, Mesh, _mask


def view_range(rank: int, world: int, views: int) -> tuple[int, int]:
    return rank * views // world, (rank + 1) * views // world


class GpuBackend:
    """Per-rank primitives over libsof_cuda.so; state lives in torch CUDA tensors."""

    def __init__(self, ctx: Context):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.dev = torch.device("cuda", ctx.device)
        p, nv = ctypes.c_void_p(), ctypes.c_int64()
        ctx.check(ctx.lib.sof_tets_vertices_dev(ctx.h, ctypes.byref(p), ctypes.byref(nv)))
        self.xyz, self.nv = p, nv.value
        self.counters = np.zeros(2, np.uint64)

    def _p(self, t):
        return ctypes.c_void_p(t.data_ptr())

    def sync(self):
        """Orders the library's stream after everything torch enqueued so far (no host
        synchronisation: sof_stream_wait records an event on torch's current stream)."""
        st = self.torch.cuda.current_stream(self.dev)
        self.ctx.check(self.ctx.lib.sof_stream_wait(self.ctx.h, ctypes.c_void_p(st.cuda_stream)))

    # torch fills and concatenations run on torch's current stream; the library works on
    # its own non-blocking stream, so every tensor torch wrote is ordered before a library
    # call reads it (the library calls themselves return with their stream idle)
    def new_state(self, n):
        t = self.torch
        out = t.ones(n, dtype=t.float64, device=self.dev), t.zeros(n, dtype=t.uint8, device=self.dev)
        self.sync()
        return out

    def zeros_u8(self, n):
        out = self.torch.zeros(max(n, 1), dtype=self.torch.uint8, device=self.dev)
        self.sync()
        return out

    def label_views(self, v0, v1, strategies, tile_size, min_op, ext):
        c = self.ctx
        c.check(c.lib.sof_label_views_dev(c.h, v0, v1, self.nv, self.xyz, strategies, tile_size, 1,
                                          self._p(min_op), self._p(ext), self.counters.ctypes.data_as(ctypes.c_void_p)))

    def ext_rank(self, ext, rank, world):
        out = self.torch.empty(self.nv, dtype=self.torch.int32, device=self.dev)  # written by the library only
        self.ctx.check(self.ctx.lib.sof_shard_ext_rank_dev(self.ctx.h, self.nv, self._p(ext), rank, world, self._p(out)))
        return out

    def mask_min(self, rstar, rank, min_op):
        self.ctx.check(self.ctx.lib.sof_shard_mask_min_dev(self.ctx.h, self.nv, self._p(rstar), rank, self._p(min_op)))

    def finalize(self, min_op, rstar, world):
        self.ctx.check(self.ctx.lib.sof_shard_finalize_dev(self.ctx.h, self.nv, self._p(min_op), self._p(rstar), world))

    def march(self):
        ne, nt = ctypes.c_int64(), ctypes.c_int64()
        self.ctx.check(self.ctx.lib.sof_march_resident(self.ctx.h, ctypes.byref(ne), ctypes.byref(nt)))
        return ne.value, nt.value

    def march_range(self, t0, t1):
        ne, nt = ctypes.c_int64(), ctypes.c_int64()
        self.ctx.check(self.ctx.lib.sof_march_range_resident(self.ctx.h, t0, t1, ctypes.byref(ne), ctypes.byref(nt)))
        return ne.value, nt.value

    def march_local(self, ne, nt):
        """This shard's march result as flat int32 tensors: edges [2 ne], triangles [3 nt]."""
        t = self.torch
        edges = t.empty(max(2 * ne, 1), dtype=t.int32, device=self.dev)
        tris = t.empty(max(3 * nt, 1), dtype=t.int32, device=self.dev)
        self.ctx.check(self.ctx.lib.sof_march_result_copy_dev(self.ctx.h, self._p(edges), self._p(tris)))
        return edges[: 2 * ne], tris[: 3 * nt]

    def march_merge(self, edge_counts, edges_all, tri_counts, tris_all):
        ec, tc = np.asarray(edge_counts, np.int64), np.asarray(tri_counts, np.int64)
        ne, nt = ctypes.c_int64(), ctypes.c_int64()
        edges_all, tris_all = edges_all.contiguous(), tris_all.contiguous()
        self.ctx.check(self.ctx.lib.sof_march_merge_dev(
            self.ctx.h, len(ec), ec.ctypes.data_as(ctypes.c_void_p), self._p(edges_all),
            tc.ctypes.data_as(ctypes.c_void_p), self._p(tris_all), ctypes.byref(ne), ctypes.byref(nt)))
        self.sync()
        return ne.value, nt.value

    def refine_phase(self, phase, ext, v0, v1, strategies, tile_size):
        self.ctx.check(self.ctx.lib.sof_refine_phase_dev(
            self.ctx.h, phase, self._p(ext) if ext is not None else None, v0, v1, strategies, tile_size,
            self.counters.ctypes.data_as(ctypes.c_void_p)))

    def assemble(self, weld_eps, min_area):
        nv, nt = ctypes.c_int64(), ctypes.c_int64()
        self.ctx.check(self.ctx.lib.sof_assemble_resident(self.ctx.h, weld_eps, min_area, ctypes.byref(nv),
                                                          ctypes.byref(nt)))
        return nv.value, nt.value

    def fetch_mesh(self) -> Mesh:
        return Mesh(self.ctx.result(L.R_MESH_VERTS, np.float64, 3), self.ctx.result(L.R_MESH_TRIS, np.int32, 3))


class ShardedMesher:
    """label -> march -> 8-step bisection -> weld with views sharded across ranks."""

    def __init__(self, backend_or_ctx, rank: int, world: int, n_views: int | None = None, group=None,
                 n_tets: int | None = None, shard_tets: bool = True):
        import torch.distributed as dist
        self.dist = dist
        self.b = GpuBackend(backend_or_ctx) if isinstance(backend_or_ctx, Context) else backend_or_ctx
        self.rank, self.world, self.group = rank, world, group
        if n_views is None:
            n_views = backend_or_ctx.cams.v
        self.n_views = n_views
        if n_tets is None:
            n_tets = backend_or_ctx.n_tets if isinstance(backend_or_ctx, Context) else backend_or_ctx.n_tets
        self.n_tets, self.shard_tets = n_tets, shard_tets

    def _allreduce(self, t, op):
        if self.world > 1:
            if t.is_cuda and self.dist.get_backend(self.group) == "gloo":  # host collective
                h = t.cpu()
                self.dist.all_reduce(h, op=op, group=self.group)
                t.copy_(h)
            else:
                self.dist.all_reduce(t, op=op, group=self.group)
            self.b.sync()  # the library runs on its own stream

    def _allgather_v(self, t, n):
        """All ranks' first n entries of the 1-D tensor t, concatenated in rank order,
        and the per-rank counts (collectives have no gatherv: pad to the largest)."""
        import torch
        dist = self.dist
        # gloo gathers host tensors only (NCCL gathers device tensors in place)
        stage = t.is_cuda and dist.get_backend(self.group) == "gloo"
        dev = torch.device("cpu") if stage else t.device
        cnt = torch.tensor([n], dtype=torch.int64, device=dev)
        cnts = [torch.zeros_like(cnt) for _ in range(self.world)]
        dist.all_gather(cnts, cnt, group=self.group)
        counts = [int(x.item()) for x in cnts]
        buf = torch.zeros(max(max(counts), 1), dtype=t.dtype, device=dev)
        buf[:n] = t[:n].to(dev)
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        out = torch.cat([o[:k] for o, k in zip(outs, counts)]).to(t.device)
        self.b.sync()  # the concatenation (torch's stream) is read by the library next
        return out, counts

    def _march(self, n_tets: int):
        """Marching Tetrahedra with the tets split across ranks: rank r marches the r-th
        contiguous tet range, the edge and triangle lists are gathered in rank (= tet)
        order, and every rank merges them into the whole-grid numbering
        (sof_march_merge_dev); identical to a single-rank march."""
        if self.world == 1 or not self.shard_tets:
            return self.b.march()
        t0, t1 = view_range(self.rank, self.world, n_tets)
        ne, nt = self.b.march_range(t0, t1)
        edges, tris = self.b.march_local(ne, nt)
        edges_all, ecnt = self._allgather_v(edges, 2 * ne)
        tris_all, tcnt = self._allgather_v(tris, 3 * nt)
        return self.b.march_merge([k // 2 for k in ecnt], edges_all, [k // 3 for k in tcnt], tris_all)

    def extract(self, opt: ExtractOptions | None = None, stats: dict | None = None, fetch: bool = True):
        opt = opt or ExtractOptions()
        R = self.dist.ReduceOp
        strategies = _mask(opt.strategies)
        prune = bool(strategies & 8)
        v0, v1 = view_range(self.rank, self.world, self.n_views)
        b = self.b
        b.counters[:] = 0
        min_op, ext = b.new_state(b.nv)
        b.label_views(v0, v1, strategies, opt.tile_size, min_op, ext)
        if prune:
            rstar = b.ext_rank(ext, self.rank, self.world)
            self._allreduce(rstar, R.MIN)
            b.mask_min(rstar, self.rank, min_op)
            self._allreduce(min_op, R.MIN)
        else:
            self._allreduce(min_op, R.MIN)
            self._allreduce(ext, R.MAX)
            rstar = b.ext_rank(ext, 0, self.world)
        b.finalize(min_op, rstar, self.world)
        label_counters = b.counters.copy()
        ne, ntri = self._march(self.n_tets)
        if opt.refine_iterations > 0 and ne > 0:
            ext_e = b.zeros_u8(ne)
            b.refine_phase(0, None, v0, v1, strategies, opt.tile_size)
            for _ in range(opt.refine_iterations):
                b.refine_phase(1, ext_e, v0, v1, strategies, opt.tile_size)
                self._allreduce(ext_e, R.MAX)
                b.refine_phase(2, ext_e, v0, v1, strategies, opt.tile_size)
            b.refine_phase(3, None, v0, v1, strategies, opt.tile_size)
        nv, nt = b.assemble(opt.weld_eps, opt.min_area)
        if stats is not None:
            stats.update(crossing_edges=ne, march_triangles=ntri, mesh_vertices=nv, mesh_triangles=nt,
                         rank_pairs=int(b.counters[0]), rank_point_view_evals=int(b.counters[1]),
                         rank_label_pairs=int(label_counters[0]))
        return b.fetch_mesh() if fetch else None

    def extract_resident(self, opt: ExtractOptions, stats: dict | None = None):
        return self.extract(ExtractOptions(strategies=opt.strategies, refine_iterations=opt.refine_iterations,
                                           tile_size=opt.tile_size, weld_eps=opt.weld_eps, min_area=opt.min_area),
                            stats, fetch=False)
