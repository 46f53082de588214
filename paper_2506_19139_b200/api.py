"""Host-side mirror of the reference's `sof::` API for the hot path, over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/sof:
  EvalStrategies / FieldEvaluator        field_eval.hpp:14-198
  ViewSet                                opacity_field.hpp:21-35 (lazy, device-resident)
  TetGrid                                delaunay.hpp:14-18
  marching_tets / binary_search_refine   marching_tets.hpp:29-114
  assemble_mesh / Mesh                   mesh.hpp:13-79
  extract_mesh (tetra-input overload)    extract.hpp:35-86
  render_depth_map / render_pixel        render.hpp:26-51, opacity_field.hpp:201-219
  write_mesh_ply                         io_mesh.hpp:55-73
Every computation runs in libsof_cuda.so on the GPU; numpy only holds host buffers.
Errors: std::invalid_argument -> ValueError, std::runtime_error -> RuntimeError.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

_P = ctypes.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a, shape_last=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape_last is not None:
        a = a.reshape(-1, shape_last)
    return a


class SofError(RuntimeError):
    pass


def _check(ctx_handle, status: int):
    if status == L.SOF_OK:
        return
    lib = L.load()
    msg = lib.sof_last_error(ctx_handle).decode() if ctx_handle else "error"
    if status == L.SOF_E_INVALID:
        raise ValueError(msg)
    if status == L.SOF_E_OOM:
        raise MemoryError(msg)
    raise SofError(f"[{status}] {msg}")


# ---- reference data types ------------------------------------------------------------------

@dataclass
class GaussianScene:
    """std::vector<GaussianPrimitive> as SoA arrays (gaussian.hpp:12-18)."""
    pos: np.ndarray
    scale: np.ndarray
    rot: np.ndarray  # (w, x, y, z)
    opacity: np.ndarray
    dc: np.ndarray

    @property
    def n(self) -> int:
        return int(np.asarray(self.opacity).shape[0])

    @staticmethod
    def of(obj) -> "GaussianScene":
        return GaussianScene(_f64(obj.pos, 3), _f64(obj.scale, 3), _f64(obj.rot, 4),
                             _f64(obj.opacity).reshape(-1), _f64(obj.dc, 3))


@dataclass
class CameraSet:
    """std::vector<Camera> as arrays (camera.hpp:10-21)."""
    R: np.ndarray
    t: np.ndarray
    intr: np.ndarray
    wh: np.ndarray
    nearfar: np.ndarray

    @property
    def v(self) -> int:
        return int(np.asarray(self.t).shape[0])

    @staticmethod
    def of(obj) -> "CameraSet":
        nf = getattr(obj, "nearfar", None)
        R = _f64(obj.R).reshape(-1, 9)
        return CameraSet(R, _f64(obj.t, 3), _f64(obj.intr, 4), np.ascontiguousarray(obj.wh, np.int32).reshape(-1, 2),
                         _f64(nf, 2) if nf is not None else np.tile([0.2, 100.0], (R.shape[0], 1)))


@dataclass
class EvalStrategies:
    tile_scheduling: bool = False
    min_z: bool = False
    early_stop: bool = False
    prune: bool = False
    dead_cull: bool = False

    @staticmethod
    def naive() -> "EvalStrategies":
        return EvalStrategies()

    @staticmethod
    def all() -> "EvalStrategies":
        return EvalStrategies(True, True, True, True, True)

    @staticmethod
    def from_mask(m: int) -> "EvalStrategies":
        return EvalStrategies(bool(m & 1), bool(m & 2), bool(m & 4), bool(m & 8), bool(m & 16))

    @property
    def mask(self) -> int:
        return (int(self.tile_scheduling) | int(self.min_z) << 1 | int(self.early_stop) << 2
                | int(self.prune) << 3 | int(self.dead_cull) << 4)


def _mask(s) -> int:
    return s if isinstance(s, int) else s.mask


@dataclass
class TetGrid:
    vertices: np.ndarray
    tetrahedra: np.ndarray
    opacity: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class MarchingResult:
    edges: np.ndarray      # [E, 2] (inside, outside)
    vertices: np.ndarray   # [E, 3]
    triangles: np.ndarray  # [T, 3]


@dataclass
class Mesh:
    vertices: np.ndarray
    triangles: np.ndarray
    residuals: np.ndarray = field(default_factory=lambda: np.zeros(0))


@dataclass
class ExtractOptions:
    strategies: EvalStrategies = field(default_factory=EvalStrategies.all)
    refine_iterations: int = 8
    tile_size: int = 16
    weld_eps: float = 1e-7
    min_area: float = 1e-14
    view_begin: int = -1
    view_end: int = -1
    profile: bool = False  # per-kernel device timings in the stats (adds host-side cost)
    compute_residuals: bool = False  # extract.hpp:19,65-72: |exact value_at - 0.5| per mesh vertex


# ---- device context ------------------------------------------------------------------------

class Context:
    """One GPU's sof_ctx: resident scene, cameras, tets and per-view caches."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = _P()
        st = self.lib.sof_ctx_create(device, ctypes.byref(h))
        if st != L.SOF_OK:
            raise SofError(f"sof_ctx_create(device={device}) failed with status {st} (no usable CUDA device?)")
        self.h = h
        self.device = device
        self.scene: GaussianScene | None = None
        self.cams: CameraSet | None = None
        self.nv = 0
        self.n_tets = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.sof_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def check(self, st):
        _check(self.h, st)

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.sof_kernel_launches(self.h))

    def set_scene(self, scene, filter_scale: float = 0.0):
        s = GaussianScene.of(scene)
        self.check(self.lib.sof_set_scene(self.h, s.n, _ptr(s.pos), _ptr(s.scale), _ptr(s.rot), _ptr(s.opacity),
                                          _ptr(s.dc), float(filter_scale)))
        self.scene = s

    def load_scene_ply(self, path: str, filter_scale: float = 0.0) -> "GaussianScene":
        """parse_scene (io_scene.hpp:54-134) decoded and activated on the device into this
        context's scene; returns the activated parameters."""
        n = ctypes.c_int64(0)
        self.scene = None
        self.check(self.lib.sof_load_scene_ply(self.h, str(path).encode(), float(filter_scale), ctypes.byref(n)))
        self.scene = self.get_scene(int(n.value))
        return self.scene

    def get_scene(self, n: int | None = None) -> "GaussianScene":
        """The context's scene as activated GaussianPrimitive fields (device -> host)."""
        if n is None:
            if self.scene is None:
                raise SofError("no scene: call set_scene or load_scene_ply first")
            n = self.scene.n
        s = GaussianScene(np.empty((n, 3)), np.empty((n, 3)), np.empty((n, 4)), np.empty(n), np.empty((n, 3)))
        self.check(self.lib.sof_get_scene(self.h, _ptr(s.pos), _ptr(s.scale), _ptr(s.rot), _ptr(s.opacity),
                                          _ptr(s.dc)))
        return s

    def write_scene_ply(self, path: str):
        """write_scene (io_scene.hpp:138-181) of this context's scene (inverse activations on
        the device); byte-identical to the reference writer."""
        self.check(self.lib.sof_write_scene_ply(self.h, str(path).encode()))

    def set_views(self, cams):
        c = CameraSet.of(cams)
        self.check(self.lib.sof_set_views(self.h, c.v, _ptr(c.R), _ptr(c.t), _ptr(c.intr), _ptr(c.wh), _ptr(c.nearfar)))
        self.cams = c

    def set_tets(self, vertices, tets, async_copy: bool = False):
        """TetGrid vertices + tetrahedra to the device. async_copy: the tets travel on a
        copy stream during the next label pass (sof_set_tets_async); keep `tets` alive and
        unchanged until the next extract returns."""
        v = _f64(vertices, 3)
        t = np.ascontiguousarray(tets, np.int32).reshape(-1, 4)
        fn = self.lib.sof_set_tets_async if async_copy else self.lib.sof_set_tets
        self.check(fn(self.h, len(v), _ptr(v), len(t), _ptr(t)))
        self._tets_keepalive = t if async_copy else None
        self.nv = len(v)
        self.n_tets = len(t)

    def result(self, kind: int, dtype, width: int):
        n = int(self.lib.sof_result_count(self.h, kind))
        if n < 0:
            raise SofError("no result of that kind")
        out = np.empty(n, dtype)
        if n:
            self.check(self.lib.sof_copy_result(self.h, kind, _ptr(out)))
        return out.reshape(-1, width) if width > 1 else out

    # -- multi-GPU: the context's communicator (include/sof_cuda.h, sof_comm_*) ------------
    @staticmethod
    def comm_unique_id() -> bytes:
        """A fresh NCCL unique id (rank 0 draws it, every rank receives it out of band)."""
        lib = L.load()
        buf = ctypes.create_string_buffer(L.SOF_COMM_ID_BYTES)
        st = lib.sof_comm_unique_id(buf)
        if st != L.SOF_OK:
            raise SofError(f"sof_comm_unique_id failed with status {st} (NCCL unavailable?)")
        return buf.raw

    def comm_init(self, uid: bytes, nranks: int, rank: int):
        """Attach an NCCL communicator: sof_extract then runs the sharded meshing step."""
        buf = ctypes.create_string_buffer(bytes(uid), L.SOF_COMM_ID_BYTES)
        self.check(self.lib.sof_comm_init(self.h, buf, int(nranks), int(rank)))

    @staticmethod
    def comm_init_local(ctxs) -> None:
        """Join contexts of this process (one device) into an in-process communicator;
        drive each from its own thread afterwards (tests of the sharded protocol)."""
        arr = (_P * len(ctxs))(*[c.h for c in ctxs])
        st = L.load().sof_comm_init_local(arr, len(ctxs))
        if st != L.SOF_OK:
            raise SofError(f"sof_comm_init_local failed with status {st}")

    def comm_info(self) -> tuple[str, int, int]:
        n, r = ctypes.c_int(), ctypes.c_int()
        kind = self.lib.sof_comm_info(self.h, ctypes.byref(n), ctypes.byref(r))
        return {0: "none", 1: "nccl", 2: "local"}.get(kind, "error"), n.value, r.value

    def comm_destroy(self):
        self.check(self.lib.sof_comm_destroy(self.h))

    # -- inspection / parity -------------------------------------------------------------
    def precompute_view(self, view: int) -> np.ndarray:
        out = np.empty((self.scene.n, 13))
        self.check(self.lib.sof_precompute_view(self.h, view, _ptr(out)))
        return out

    def tile_binding(self, view: int, tile_size: int = 16):
        nt, ne = ctypes.c_int64(), ctypes.c_int64()
        self.check(self.lib.sof_tile_binding(self.h, view, tile_size, ctypes.byref(nt), ctypes.byref(ne)))
        return self.result(L.R_TILE_OFFSETS, np.int64, 1), self.result(L.R_TILE_ENTRIES, np.int32, 1)

    def schedule_points(self, view: int, xyz, tile_size: int = 16) -> dict:
        xyz = _f64(xyz, 3)
        n = len(xyz)
        ns, nb = ctypes.c_int64(), ctypes.c_int64()
        ta = np.empty(n, np.int32)
        self.check(self.lib.sof_schedule_points(self.h, view, n, _ptr(xyz), tile_size, ctypes.byref(ns),
                                                ctypes.byref(nb), _ptr(ta), None, None, None, None, None))
        order, kt = np.empty(ns.value, np.int32), np.empty(ns.value, np.int32)
        kd = np.empty(ns.value)
        br, bt = np.empty((nb.value, 2), np.int32), np.empty(nb.value, np.int32)
        self.check(self.lib.sof_schedule_points(self.h, view, n, _ptr(xyz), tile_size, None, None, _ptr(ta),
                                                _ptr(order), _ptr(kt), _ptr(kd), _ptr(br), _ptr(bt)))
        return {"tile_assignment": ta, "order": order, "key_tile": kt, "key_depth": kd,
                "block_ranges": br, "block_to_tile": bt}


_default_ctx: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


class ViewSet:
    """ViewSet::build (opacity_field.hpp:26-34): the per-view caches are built lazily
    on the device instead of eagerly materialising V x N PrecomputedGaussians."""

    def __init__(self, ctx: Context, scene: GaussianScene, cams: CameraSet, filter_scale: float):
        self.ctx, self.scene, self.cameras, self.filter_scale = ctx, scene, cams, filter_scale

    @staticmethod
    def build(gaussians, cams, filter_scale: float = 0.0, ctx: Context | None = None) -> "ViewSet":
        ctx = ctx or Context(0)
        ctx.set_scene(gaussians, filter_scale)
        ctx.set_views(cams)
        return ViewSet(ctx, ctx.scene, ctx.cams, filter_scale)


class FieldEvaluator:
    """FieldEvaluator (field_eval.hpp:39-198), batched over points on the GPU."""

    def __init__(self, gaussians, views: ViewSet, strategies=None, tile_size: int = 16):
        self.views = views
        self.ctx = views.ctx
        self.strategies = EvalStrategies.naive() if strategies is None else strategies
        self.mask = _mask(self.strategies)
        self.tile_size = int(tile_size)
        if self.tile_size <= 0:
            raise ValueError("tile_size must be positive")
        self._counters = np.zeros(2, np.uint64)

    def counters(self) -> dict:
        return {"pairs": int(self._counters[0]), "point_view_evals": int(self._counters[1])}

    def reset_counters(self):
        self._counters[:] = 0

    def view_opacity(self, view: int, xyz, classify_mode: bool):
        xyz = _f64(xyz, 3)
        n = len(xyz)
        o, ob, co = np.empty(n), np.empty(n, np.uint8), np.empty(n, np.uint8)
        self.ctx.check(self.ctx.lib.sof_view_opacity(self.ctx.h, view, n, _ptr(xyz), self.mask, self.tile_size,
                                                     int(classify_mode), _ptr(o), _ptr(ob), _ptr(co),
                                                     _ptr(self._counters)))
        return o, ob.astype(bool), co.astype(bool)

    def classify_points(self, xyz) -> np.ndarray:
        xyz = _f64(xyz, 3)
        out = np.empty(len(xyz), np.uint8)
        self.ctx.check(self.ctx.lib.sof_classify_points(self.ctx.h, len(xyz), _ptr(xyz), self.mask, self.tile_size,
                                                        _ptr(out), _ptr(self._counters)))
        return out.astype(bool)

    def classify_point(self, x) -> bool:
        return bool(self.classify_points(np.asarray(x, np.float64).reshape(1, 3))[0])

    def value_at(self, xyz):
        a = _f64(xyz, 3)
        out = np.empty(len(a))
        self.ctx.check(self.ctx.lib.sof_value_at(self.ctx.h, len(a), _ptr(a), self.mask, self.tile_size,
                                                 _ptr(out), _ptr(self._counters)))
        return out if np.ndim(xyz) == 2 else float(out[0])

    def label_grid(self, grid, classify_mode: bool = True):
        """Labels every grid vertex; writes grid.opacity (field_eval.hpp:140-176)."""
        xyz = _f64(grid.vertices if hasattr(grid, "vertices") else grid, 3)
        out = np.empty(len(xyz))
        self.ctx.check(self.ctx.lib.sof_label_grid(self.ctx.h, len(xyz), _ptr(xyz), self.mask, self.tile_size,
                                                   int(classify_mode), _ptr(out), _ptr(self._counters)))
        if hasattr(grid, "vertices"):
            grid.opacity = out
        return out


def marching_tets(grid: TetGrid, ctx: Context | None = None) -> MarchingResult:
    """marching_tets (marching_tets.hpp:29-84) on the GPU."""
    ctx = ctx or default_context()
    ctx.set_tets(grid.vertices, grid.tetrahedra)
    opa = _f64(grid.opacity).reshape(-1)
    if len(opa) != ctx.nv:
        raise ValueError("grid.opacity must have one value per vertex")
    ne, nt = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(ctx.lib.sof_marching_tets(ctx.h, _ptr(opa), ctypes.byref(ne), ctypes.byref(nt)))
    return MarchingResult(ctx.result(L.R_EDGES, np.int32, 2), ctx.result(L.R_EDGE_VERTS, np.float64, 3),
                          ctx.result(L.R_TRIANGLES, np.int32, 3))


def binary_search_refine(m: MarchingResult, grid: TetGrid, evaluator: FieldEvaluator, iterations: int = 8):
    """Batched binary_search_refine (marching_tets.hpp:94-114): all edges x `iterations`
    device passes, classify_point as the interior test. Updates m.vertices in place."""
    ctx = evaluator.ctx
    ctx.set_tets(grid.vertices, grid.tetrahedra)
    edges = np.ascontiguousarray(m.edges, np.int32).reshape(-1, 2)
    v = np.array(m.vertices, np.float64, order="C").reshape(-1, 3)
    ctx.check(ctx.lib.sof_refine(ctx.h, len(edges), _ptr(edges), _ptr(v), int(iterations), evaluator.mask,
                                 evaluator.tile_size, _ptr(evaluator._counters)))
    m.vertices = v
    return m


def assemble_mesh(vertices, triangles, residuals=None, weld_eps: float = 1e-7, min_area: float = 1e-14,
                  ctx: Context | None = None) -> Mesh:
    """assemble_mesh (mesh.hpp:36-79) on the GPU."""
    ctx = ctx or default_context()
    v = _f64(vertices, 3) if len(vertices) else np.zeros((0, 3))
    t = np.ascontiguousarray(triangles, np.int32).reshape(-1, 3)
    r = None if residuals is None else _f64(residuals).reshape(-1)
    if r is not None and len(r) != len(v):
        raise ValueError("one residual per vertex")
    nv, nt = ctypes.c_int64(), ctypes.c_int64()
    ctx.check(ctx.lib.sof_assemble_residuals(ctx.h, len(v), _ptr(v), _ptr(r), len(t), _ptr(t), float(weld_eps),
                                             float(min_area), ctypes.byref(nv), ctypes.byref(nt)))
    res = ctx.result(L.R_MESH_RESIDUALS, np.float64, 1) if r is not None else np.zeros(0)
    return Mesh(ctx.result(L.R_MESH_VERTS, np.float64, 3), ctx.result(L.R_MESH_TRIS, np.int32, 3), res)


def delaunay_tetrahedralize(points, ctx: Context | None = None) -> TetGrid:
    """delaunay_tetrahedralize (delaunay.hpp:52-142): the reference's Bowyer-Watson tet
    list in the reference's order, on the device (sof_tetrahedralize)."""
    ctx = ctx or default_context()
    p = _f64(points, 3)
    nt = ctypes.c_int64()
    ctx.check(ctx.lib.sof_tetrahedralize(ctx.h, len(p), _ptr(p), ctypes.byref(nt)))
    return TetGrid(p.copy(), ctx.result(L.R_TETS, np.int32, 4), np.zeros(len(p)))


def extract_mesh(gaussians, views: ViewSet, grid: TetGrid | None = None, opt: ExtractOptions | None = None,
                 stats: dict | None = None, bounding: int = L.SEED_STP, cutoff: int = L.SEED_CUT_DEAD) -> Mesh:
    """extract_mesh (extract.hpp:35-86). With `grid`: label -> march -> refine -> weld on
    the given tetra input, fused on the device. Without: the reference's own producer
    first — build_seed_points and delaunay_tetrahedralize (both on the device), with the
    reference's defaults (BoundingVariant::kStp, SeedCutoff::kDeadGaussians)."""
    opt = opt or ExtractOptions()
    ctx = views.ctx
    if grid is None:
        seeds = build_seed_points(ctx, bounding, cutoff, views.filter_scale)
        grid = delaunay_tetrahedralize(seeds.points, ctx)
        if stats is not None:
            stats.update(seed_points=len(seeds.points), tetrahedra=len(grid.tetrahedra))
    ctx.set_tets(grid.vertices, grid.tetrahedra)
    return extract_resident(ctx, opt, stats)


def extract_resident(ctx: Context, opt: ExtractOptions, stats: dict | None = None, fetch: bool = True):
    o = L.ExtractOpts(_mask(opt.strategies), opt.tile_size, opt.refine_iterations, opt.weld_eps, opt.min_area,
                      opt.view_begin, opt.view_end, int(opt.profile), int(opt.compute_residuals))
    st = L.ExtractStats()
    ctx.check(ctx.lib.sof_extract(ctx.h, ctypes.byref(o), ctypes.byref(st)))
    if stats is not None:
        stats.update(st.as_dict())
    if not fetch:
        return None
    res = ctx.result(L.R_MESH_RESIDUALS, np.float64, 1) if opt.compute_residuals else np.zeros(0)
    return Mesh(ctx.result(L.R_MESH_VERTS, np.float64, 3), ctx.result(L.R_MESH_TRIS, np.int32, 3), res)


def render_view(views: ViewSet, view: int, depth_mode: int = L.DEPTH_EXACT, tile_size: int = 16,
                normals: bool = False, counts: bool = False, window: int = 0) -> dict:
    """render_depth_map (render.hpp:26-51) + render_pixel colour / T (opacity_field.hpp:201-219);
    with normals=True also normal_from_depth (render.hpp:60-88) of the depth, computed on
    the device from the resident depth map. window=K > 0 replaces the exact per-pixel
    (t*, index) order by windowed_resort's K-slot window (opacity_field.hpp:66-91) over
    the contributions in view-space centre-depth order (sof_set_render_window)."""
    ctx = views.ctx
    ctx.check(ctx.lib.sof_set_render_window(ctx.h, int(window)))
    w, h = (int(x) for x in ctx.cams.wh[view])
    out = {"depth": np.empty((h, w)), "opacity": np.empty((h, w)), "rgb": np.empty((h, w, 3)),
           "t_final": np.empty((h, w)), "stats": np.zeros(4, np.uint64)}
    ctx.check(ctx.lib.sof_render_view(ctx.h, view, depth_mode, tile_size, _ptr(out["depth"]), _ptr(out["opacity"]),
                                      _ptr(out["rgb"]), _ptr(out["t_final"]), _ptr(out["stats"])))
    if counts:  # per-pixel contribution counts (len(collect_contributions))
        out["counts"] = np.empty((h, w), np.uint32)
        ctx.check(ctx.lib.sof_render_counts(ctx.h, view, _ptr(out["counts"])))
    if normals:
        out["normal"] = np.empty((h, w, 3))
        out["normal_valid"] = np.empty((h, w), np.uint8)
        ctx.check(ctx.lib.sof_render_normals(ctx.h, view, _ptr(out["normal"]), _ptr(out["normal_valid"])))
    return out


def render_views(views: ViewSet, first: int, count: int, depth_mode: int = L.DEPTH_EXACT) -> list:
    """sof_render_views: the exact render of views [first, first + count) in one call;
    per view a dict of depth, opacity, rgb and t_final (as render_view)."""
    ctx = views.ctx
    wh = [(int(w), int(h)) for w, h in ctx.cams.wh[first:first + count]]
    px = sum(w * h for w, h in wh)
    rgb, depth, op, tf = np.empty((px, 3)), np.empty(px), np.empty(px), np.empty(px)
    ctx.check(ctx.lib.sof_set_render_window(ctx.h, 0))
    ctx.check(ctx.lib.sof_render_views(ctx.h, int(first), int(count), int(depth_mode), _ptr(rgb), _ptr(depth),
                                       _ptr(op), _ptr(tf)))
    out, at = [], 0
    for w, h in wh:
        sl = slice(at, at + w * h)
        out.append({"depth": depth[sl].reshape(h, w), "opacity": op[sl].reshape(h, w),
                    "rgb": rgb[sl].reshape(h, w, 3), "t_final": tf[sl].reshape(h, w)})
        at += w * h
    return out


def pixel_rays(cams: CameraSet, view: int, pix) -> np.ndarray:
    """ray_through_pixel(cam, x + 0.5, y + 0.5).direction (camera.hpp:42-48) for integer
    pixels pix[n, 2] = (x, y), in the reference's operation order (host)."""
    pix = np.asarray(pix, np.float64).reshape(-1, 2)
    R = np.asarray(cams.R[view], np.float64).reshape(3, 3)
    fx, fy, cx, cy = (float(v) for v in cams.intr[view])
    v0 = ((pix[:, 0] + 0.5) - cx) / fx
    v1 = ((pix[:, 1] + 0.5) - cy) / fy
    d = np.stack([(R[0, i] * v0 + R[1, i] * v1) + R[2, i] * 1.0 for i in range(3)], axis=1)
    sq = (d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2]
    nrm = np.sqrt(sq)
    return np.where(sq[:, None] > 0.0, d / np.where(nrm > 0, nrm, 1.0)[:, None], d)


def collect_contributions(views: ViewSet, view: int, directions) -> dict:
    """collect_contributions (opacity_field.hpp:39-61) for each ray of `view` (unit
    directions [n, 3]; the origin is the camera centre), on the device over ALL Gaussians.
    Returns offsets [n + 1] and, per contribution in (t*, index) order per ray, index and
    t_star / alpha / a / b / c / opacity (values [C, 6] holds the six columns)."""
    ctx = views.ctx
    d = _f64(directions, 3)
    off = np.zeros(len(d) + 1, np.int64)
    ctx.check(ctx.lib.sof_collect_contributions(ctx.h, int(view), len(d), _ptr(d), _ptr(off)))
    idx = ctx.result(L.R_CONTRIB_INDEX, np.int32, 1)
    val = ctx.result(L.R_CONTRIB_VALUES, np.float64, 6).reshape(-1, 6)
    out = {"offsets": off, "index": idx, "values": val}
    for k, name in enumerate(("t_star", "alpha", "a", "b", "c", "opacity")):
        out[name] = val[:, k]
    return out


def windowed_resort(offsets, t_star, window: int, ctx: Context | None = None) -> np.ndarray:
    """windowed_resort (opacity_field.hpp:66-91) of arrival-ordered lists on the device:
    returns order[C], the input position of the element at each output slot (ties as
    libstdc++ orders them)."""
    ctx = ctx or default_context()
    off = np.ascontiguousarray(offsets, np.int64)
    t = np.ascontiguousarray(t_star, np.float64)
    order = np.empty(len(t), np.int64)
    ctx.check(ctx.lib.sof_windowed_resort(ctx.h, len(off) - 1, _ptr(off), _ptr(t), int(window), _ptr(order)))
    return order


def render_pixel(offsets, index, values, depth_mode: int = L.DEPTH_EXACT, ctx: Context | None = None,
                 dc=None) -> dict:
    """render_pixel (opacity_field.hpp:201-219) of given contribution lists on the device;
    colours from `dc` [N, 3] or, when None, the resident scene of `ctx`."""
    ctx = ctx or default_context()
    off = np.ascontiguousarray(offsets, np.int64)
    idx = np.ascontiguousarray(index, np.int32)
    val = np.ascontiguousarray(values, np.float64).reshape(-1, 6)
    nl = len(off) - 1
    dcp = None if dc is None else _f64(dc, 3)
    out = {"color": np.empty((nl, 3)), "depth": np.empty(nl), "accumulated_opacity": np.empty(nl),
           "t_final": np.empty(nl)}
    ctx.check(ctx.lib.sof_render_pixel(ctx.h, nl, _ptr(off), _ptr(idx), _ptr(val), 0 if dcp is None else len(dcp),
                                       None if dcp is None else _ptr(dcp), int(depth_mode),
                                       *(_ptr(out[k]) for k in ("color", "depth", "accumulated_opacity", "t_final"))))
    return out


def render_depth_map(views: ViewSet, view: int, exact: bool = True):
    r = render_view(views, view, L.DEPTH_EXACT if exact else L.DEPTH_MEDIAN)
    return r["depth"], r["opacity"]


def normal_from_depth(views: ViewSet, view: int, depth):
    """normal_from_depth (render.hpp:60-88) of a depth map [h, w] (NaN = no surface) with the
    camera of `view`. Returns (normal [h, w, 3], valid [h, w] uint8)."""
    ctx = views.ctx
    w, h = (int(x) for x in ctx.cams.wh[view])
    depth = np.ascontiguousarray(depth, np.float64)
    if depth.shape != (h, w):
        raise ValueError(f"depth map must be {h}x{w}")
    normal, valid = np.empty((h, w, 3)), np.empty((h, w), np.uint8)
    ctx.check(ctx.lib.sof_normal_from_depth(ctx.h, view, _ptr(depth), _ptr(normal), _ptr(valid)))
    return normal, valid


def gaussian_normal(ctx: Context, gidx, origin, direction, t):
    """gaussian_normal (render.hpp:93-107), batched: Gaussian gidx[k], ray (origin[k],
    direction[k]) at parameter t[k]."""
    gidx = np.ascontiguousarray(np.atleast_1d(gidx), np.int32)
    o = np.ascontiguousarray(origin, np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(direction, np.float64).reshape(-1, 3)
    t = np.ascontiguousarray(np.atleast_1d(t), np.float64)
    if not (len(o) == len(d) == len(t) == len(gidx)):
        raise ValueError("gidx, origin, direction and t must have the same length")
    out = np.empty((len(gidx), 3))
    ctx.check(ctx.lib.sof_gaussian_normals(ctx.h, len(gidx), *(_ptr(a) for a in (gidx, o, d, t, out))))
    return out


# ---- float maps (io_maps.hpp) ----------------------------------------------------------------

@dataclass
class FloatMap:
    """`channels` interleaved float32 values per pixel, row-major (io_maps.hpp:17-29)."""
    width: int = 0
    height: int = 0
    channels: int = 1
    data: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))


def write_float_map(m: FloatMap, path: str):
    """write_float_map (io_maps.hpp:30-38): ASCII header "sofmap W H C\n" then the raw
    little-endian float32 payload; byte-identical to the reference writer."""
    data = np.ascontiguousarray(m.data, "<f4").ravel()
    if data.size != m.width * m.height * m.channels:
        raise RuntimeError("float map size mismatch")
    try:
        f = open(path, "wb")
    except OSError:
        raise RuntimeError(f"cannot write float map: {path}") from None
    with f:
        f.write(f"sofmap {m.width} {m.height} {m.channels}\n".encode())
        f.write(data.tobytes())


def read_float_map(path: str) -> FloatMap:
    """read_float_map (io_maps.hpp:40-58), same error messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot open float map: {path}") from None
    with f:
        line = f.readline()
        parts = line.decode("latin-1").split()
        try:
            magic, w, h, c = parts[0], int(parts[1]), int(parts[2]), int(parts[3])
        except (IndexError, ValueError):
            raise RuntimeError("malformed float map header") from None
        if magic != "sofmap" or w <= 0 or h <= 0 or c <= 0:
            raise RuntimeError("malformed float map header")
        payload = f.read(4 * w * h * c)
        if len(payload) != 4 * w * h * c:
            raise RuntimeError("truncated float map payload")
    return FloatMap(w, h, c, np.frombuffer(payload, "<f4").copy())


def depth_to_map(depth, opacity) -> FloatMap:
    """depth_to_map (io_maps.hpp:60-72): channels (depth, opacity at depth) as float32."""
    depth, opacity = np.asarray(depth, np.float64), np.asarray(opacity, np.float64)
    h, w = depth.shape
    return FloatMap(w, h, 2, np.stack([depth, opacity], -1).astype(np.float32).ravel())


def normals_to_map(normal) -> FloatMap:
    """normals_to_map (io_maps.hpp:74-84)."""
    normal = np.asarray(normal, np.float64)
    h, w, _ = normal.shape
    return FloatMap(w, h, 3, normal.astype(np.float32).ravel())


def render_maps(views: ViewSet, view: int, depth_path: str, normal_path: str, exact: bool = True):
    """The per-view output of the reference `sof render` (sof_cli.cpp:122-130): depth +
    opacity-at-depth map and normal map, rendered and differentiated on the device."""
    r = render_view(views, view, L.DEPTH_EXACT if exact else L.DEPTH_MEDIAN, normals=True)
    write_float_map(depth_to_map(r["depth"], r["opacity"]), depth_path)
    write_float_map(normals_to_map(r["normal"]), normal_path)
    return r


def write_mesh_ply(mesh: Mesh, path: str):
    """Binary little-endian PLY with double coordinates, byte-identical to
    write_mesh_ply (io_mesh.hpp:55-73)."""
    v = _f64(mesh.vertices, 3) if len(mesh.vertices) else np.zeros((0, 3))
    t = np.ascontiguousarray(mesh.triangles, np.int32).reshape(-1, 3)
    header = ("ply\nformat binary_little_endian 1.0\n"
              f"element vertex {len(v)}\n"
              "property double x\nproperty double y\nproperty double z\n"
              f"element face {len(t)}\n"
              "property list uchar int vertex_indices\nend_header\n").encode()
    faces = np.empty(len(t), dtype=[("n", "u1"), ("i", "<i4", 3)])
    faces["n"] = 3
    faces["i"] = t
    with open(path, "wb") as f:
        f.write(header)
        f.write(v.astype("<f8").tobytes())
        f.write(faces.tobytes())


def read_mesh_ply(path: str) -> Mesh:
    """read_mesh_ply (io_mesh.hpp:75-113), same error messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"cannot open mesh: {path}") from None
    with f:
        if f.readline().rstrip(b"\n") != b"ply":
            raise RuntimeError("malformed PLY header: missing magic")
        nv = nf = -1
        while True:
            line = f.readline()
            if not line:
                break
            tk = line.decode("latin-1").split()
            if not tk:
                continue
            if tk[0] == "format" and (len(tk) < 2 or tk[1] != "binary_little_endian"):
                raise RuntimeError("unsupported PLY format: " + (tk[1] if len(tk) > 1 else ""))
            if tk[0] == "element" and len(tk) > 2:
                if tk[1] == "vertex":
                    nv = int(tk[2])
                if tk[1] == "face":
                    nf = int(tk[2])
            if tk[0] == "end_header":
                break
        if nv < 0 or nf < 0:
            raise RuntimeError("malformed PLY header: incomplete")
        vb = f.read(24 * nv)
        if len(vb) != 24 * nv:
            raise RuntimeError("truncated PLY payload")
        fb = f.read(13 * nf)
    faces = np.frombuffer(fb[: 13 * (len(fb) // 13)], dtype=[("n", "u1"), ("i", "<i4", 3)])
    bad = np.nonzero(faces["n"] != 3)[0]
    full = len(faces)
    if len(bad) and bad[0] < full:
        raise RuntimeError("only triangle faces supported")
    if full < nf:
        # a short read: the count byte (if present) is checked before the indices
        rest = fb[13 * full:]
        if len(rest) == 0 or rest[0] != 3:
            raise RuntimeError("only triangle faces supported")
        raise RuntimeError("truncated PLY payload")
    return Mesh(np.frombuffer(vb, "<f8").reshape(-1, 3).copy(), faces["i"].astype(np.int32).copy())


def write_mesh_obj(mesh: Mesh, path: str):
    """write_mesh_obj (io_mesh.hpp:19-29): "v %.17g %.17g %.17g" and 1-based faces."""
    v = _f64(mesh.vertices, 3) if len(mesh.vertices) else np.zeros((0, 3))
    t = np.ascontiguousarray(mesh.triangles, np.int64).reshape(-1, 3)
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot write mesh: {path}") from None
    with f:
        f.writelines("v %.17g %.17g %.17g\n" % (x, y, z) for x, y, z in v.tolist())
        f.writelines(f"f {a + 1} {b + 1} {c + 1}\n" for a, b, c in t.tolist())


def read_mesh_obj(path: str) -> Mesh:
    """read_mesh_obj (io_mesh.hpp:31-51): v / f records, other lines ignored."""
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open mesh: {path}") from None
    vs, ts = [], []
    with f:
        for line in f:
            tk = line.split()
            if not tk:
                continue
            if tk[0] == "v":
                vs.append([float(x) for x in tk[1:4]])
            elif tk[0] == "f":
                ts.append([int(x) - 1 for x in tk[1:4]])
    return Mesh(np.array(vs, np.float64).reshape(-1, 3), np.array(ts, np.int32).reshape(-1, 3))


def write_mesh(mesh: Mesh, path: str, fmt: str = "ply"):
    """write_mesh (io_mesh.hpp:115-120): fmt "obj" or "ply" (binary)."""
    (write_mesh_obj if fmt == "obj" else write_mesh_ply)(mesh, path)


_CAM_REQUIRED = ("width", "height", "fx", "fy", "cx", "cy", "rotation", "translation")


def load_cameras(path: str) -> CameraSet:
    """load_cameras (io_camera.hpp:17-63): {"cameras": [{width, height, fx, fy, cx, cy,
    rotation (9, row-major world-to-view), translation (3), near?, far?}, ...]}, with the
    reference's checks and messages (RuntimeError)."""
    import json
    try:
        f = open(path)
    except OSError:
        raise RuntimeError(f"cannot open camera file: {path}") from None
    with f:
        try:
            root = json.load(f)
        except ValueError as e:
            raise RuntimeError(f"camera schema error: {e}") from None
    if not isinstance(root, dict) or not isinstance(root.get("cameras"), list):
        raise RuntimeError("camera schema error: missing field 'cameras'")
    v = len(root["cameras"])
    R, t, intr = np.empty((v, 9)), np.empty((v, 3)), np.empty((v, 4))
    wh, nf = np.empty((v, 2), np.int32), np.tile([0.2, 100.0], (v, 1))  # camera.hpp:16-17
    for k, jc in enumerate(root["cameras"]):
        for req in _CAM_REQUIRED:
            if req not in jc:
                raise RuntimeError(f"camera schema error: missing field '{req}'")
        wh[k] = int(jc["width"]), int(jc["height"])
        intr[k] = [float(jc[n]) for n in ("fx", "fy", "cx", "cy")]
        r, tt = jc["rotation"], jc["translation"]
        if not isinstance(r, list) or len(r) != 9:
            raise RuntimeError("camera schema error: rotation must have 9 entries")
        if not isinstance(tt, list) or len(tt) != 3:
            raise RuntimeError("camera schema error: translation must have 3 entries")
        R[k], t[k] = [float(x) for x in r], [float(x) for x in tt]
        if "near" in jc:
            nf[k, 0] = float(jc["near"])
        if "far" in jc:
            nf[k, 1] = float(jc["far"])
        m = R[k].reshape(3, 3)
        if np.abs(m @ m.T - np.eye(3)).max() > 1e-6:
            raise RuntimeError("degenerate rotation: not orthonormal")
        if wh[k, 0] <= 0 or wh[k, 1] <= 0 or intr[k, 0] <= 0.0 or intr[k, 1] <= 0.0:
            raise RuntimeError("camera schema error: non-positive intrinsics")
    return CameraSet(R, t, intr, wh, nf)


def save_cameras(cams, path: str):
    """save_cameras (io_camera.hpp:65-87): nlohmann::json::dump(2)'s layout (keys sorted,
    2-space indent) plus a newline. Doubles use Python's shortest round-trip repr, so the
    values read back bit-identically; the digits can differ from nlohmann's Grisu2 (and
    non-finite values, which nlohmann writes as null, are not representable here)."""
    import json
    c = CameraSet.of(cams)
    out = []
    for k in range(c.v):
        fx, fy, cx, cy = (float(x) for x in c.intr[k])
        out.append({"width": int(c.wh[k, 0]), "height": int(c.wh[k, 1]), "fx": fx, "fy": fy, "cx": cx, "cy": cy,
                    "rotation": [float(x) for x in c.R[k]], "translation": [float(x) for x in c.t[k]],
                    "near": float(c.nearfar[k, 0]), "far": float(c.nearfar[k, 1])})
    try:
        f = open(path, "w", newline="\n")
    except OSError:
        raise RuntimeError(f"cannot write camera file: {path}") from None
    with f:
        f.write(json.dumps({"cameras": out}, indent=2, sort_keys=True) + "\n")


@dataclass
class SeedPointSet:
    """seed_points.hpp:24-27: points and provenance (0 centre, 1 bounding-box corner)."""
    points: np.ndarray
    provenance: np.ndarray


def build_seed_points(ctx: Context, variant: int = L.SEED_STP, cutoff: int = L.SEED_CUT_NONE,
                      filter_scale: float = 0.0) -> SeedPointSet:
    """build_seed_points (seed_points.hpp:41-87) over ctx's scene, on the device: Gaussian
    centres + the 8 oriented bounding-box corners, deduplicated on the 1e-9 grid in
    insertion order. RuntimeError "no live Gaussians" when nothing survives."""
    n = ctypes.c_int64(0)
    ctx.check(ctx.lib.sof_seed_points(ctx.h, int(variant), int(cutoff), float(filter_scale), ctypes.byref(n)))
    return SeedPointSet(ctx.result(L.R_SEEDS, np.float64, 3), ctx.result(L.R_SEED_PROVENANCE, np.uint8, 1).ravel())


def parse_scene(path: str, ctx: Context | None = None, filter_scale: float = 0.0) -> GaussianScene:
    """parse_scene (io_scene.hpp:54-134), decoded and activated on the device of `ctx`
    (default context), which keeps the scene resident."""
    return (ctx or default_context()).load_scene_ply(path, filter_scale)


def write_scene(scene, path: str, ctx: Context | None = None):
    """write_scene (io_scene.hpp:138-181) via the device of `ctx`; byte-identical file."""
    c = ctx or default_context()
    c.set_scene(scene)
    c.write_scene_ply(path)


# ---- training losses (losses.hpp) ------------------------------------------------
# Batched over rays in CSR form: ray r owns samples [off[r], off[r + 1]). Each returns the
# reference's per-ray results (losses.hpp names and fields), computed on the device.

def _off(off):
    o = np.ascontiguousarray(off, np.int64)
    if o.ndim != 1 or len(o) < 1:
        raise ValueError("offsets must be a 1-D array of nrays + 1 entries")
    return o


def distortion_loss(ctx: Context, off, alpha, t, near: float, far: float, attach_w: bool = True) -> dict:
    """distortion_loss (losses.hpp:54-107): loss per ray, d_alpha / d_t per sample."""
    o = _off(off)
    a, tt = _f64(alpha), _f64(t)
    R, S = len(o) - 1, int(o[-1])
    loss, da, dt = np.empty(R), np.zeros(S), np.empty(S)
    ctx.check(ctx.lib.sof_distortion_loss(ctx.h, R, _ptr(o), _ptr(a), _ptr(tt), near, far, int(attach_w), _ptr(loss),
                                          _ptr(da), _ptr(dt)))
    return {"loss": loss, "d_alpha": da if attach_w else None, "d_t": dt}


def extent_loss(ctx: Context, off, w, a, b, c, bound, near: float, far: float) -> dict:
    """extent_loss (losses.hpp:152-179)."""
    o = _off(off)
    arrs = [_f64(x) for x in (w, a, b, c, bound)]
    R, S = len(o) - 1, int(o[-1])
    loss, skipped = np.empty(R), np.empty(R, np.int32)
    g = [np.empty(S) for _ in range(4)]
    ctx.check(ctx.lib.sof_extent_loss(ctx.h, R, _ptr(o), *(_ptr(x) for x in arrs), near, far, _ptr(loss),
                                      _ptr(skipped), *(_ptr(x) for x in g)))
    return {"loss": loss, "skipped": skipped, "d_a": g[0], "d_b": g[1], "d_c": g[2], "d_w": g[3]}


def depth_normal_loss(ctx: Context, off, w, normals, pixel_normals) -> dict:
    """depth_normal_loss (losses.hpp:119-133)."""
    o = _off(off)
    ww, nn, pn = _f64(w), _f64(normals, 3), _f64(pixel_normals, 3)
    R, S = len(o) - 1, int(o[-1])
    loss, dw, dn = np.empty(R), np.empty(S), np.empty((S, 3))
    ctx.check(ctx.lib.sof_depth_normal_loss(ctx.h, R, _ptr(o), _ptr(ww), _ptr(nn), _ptr(pn), _ptr(loss), _ptr(dw),
                                            _ptr(dn)))
    return {"loss": loss, "d_w": dw, "d_n": dn}


def opacity_supervision_loss(ctx: Context, off, contribs, depth) -> dict:
    """opacity_supervision_loss (losses.hpp:195-229); contribs: (S, 6) = t*, alpha, a, b, c,
    opacity per sample in each ray's sorted order; depth per ray (NaN = no surface)."""
    o = _off(off)
    rc, dep = _f64(contribs, 6), _f64(depth)
    R, S = len(o) - 1, int(o[-1])
    loss, fv, defined, da = np.empty(R), np.empty(R), np.empty(R, np.uint8), np.empty(S)
    ctx.check(ctx.lib.sof_opacity_supervision_loss(ctx.h, R, _ptr(o), _ptr(rc), _ptr(dep), _ptr(loss), _ptr(fv),
                                                   _ptr(defined), _ptr(da)))
    return {"loss": loss, "field_value": fv, "defined": defined.astype(bool), "d_alpha": da}


def normal_smoothness_loss(ctx: Context, normals, valid, image, per_channel: bool = False) -> dict:
    """normal_smoothness_loss (losses.hpp:247-293); normals / image (H, W, 3), valid (H, W)."""
    n = np.ascontiguousarray(normals, np.float64)
    img = np.ascontiguousarray(image, np.float64)
    v = np.ascontiguousarray(valid, np.uint8)
    H, W = v.shape
    if n.shape != (H, W, 3) or img.shape != (H, W, 3):
        raise SofError("normal map and image resolution mismatch")
    loss, used, dn = ctypes.c_double(), ctypes.c_int64(), np.empty((H, W, 3))
    ctx.check(ctx.lib.sof_normal_smoothness_loss(ctx.h, W, H, _ptr(n), _ptr(v), _ptr(img), int(per_channel),
                                                 ctypes.byref(loss), ctypes.byref(used), _ptr(dn)))
    return {"loss": loss.value, "pixels_used": used.value, "d_normal": dn}


def l1_rgb_loss(ctx: Context, rendered, reference) -> float:
    """l1_rgb_loss (losses.hpp:305-312)."""
    a = _f64(rendered, 3)
    b = _f64(reference, 3)
    if a.shape != b.shape:
        raise SofError("image resolution mismatch")
    out = ctypes.c_double()
    ctx.check(ctx.lib.sof_l1_rgb_loss(ctx.h, len(a), _ptr(a), _ptr(b), ctypes.byref(out)))
    return out.value


@dataclass
class LossWeights:
    """LossWeights (losses.hpp:12-25)."""
    lambda_dist_unbounded: float = 100.0
    lambda_dist_bounded: float = 1000.0
    lambda_normal: float = 0.05
    lambda_ext: float = 0.1
    lambda_opa: float = 0.04
    lambda_smooth: float = 0.01
    activation_iteration: int = 15000

    def lambda_dist(self, scene_bounded: bool) -> float:
        return self.lambda_dist_bounded if scene_bounded else self.lambda_dist_unbounded


def total_loss(terms: dict, weights: LossWeights, iteration: int, scene_bounded: bool) -> float:
    """total_loss (losses.hpp:315-324): auxiliary terms gated by the activation iteration."""
    if iteration < weights.activation_iteration:
        return terms["rgb"]
    return (terms["rgb"] + weights.lambda_dist(scene_bounded) * terms["distortion"] +
            weights.lambda_normal * terms["normal"] + weights.lambda_ext * terms["extent"] +
            weights.lambda_opa * terms["opacity"] + weights.lambda_smooth * terms["smoothness"])
