"""ctypes bindings for oracle/_ref/libsof_ref.so — the reference headers compiled in place.

TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs may import this module, and only as the checker or as the timed CPU
baseline. Nothing on the product path (paper_2506_19139_b200) imports oracle/.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsof_ref.so")
REF_GLIBC_SO = os.path.join(HERE, "_ref", "libsof_ref_glibc.so")

_P = ctypes.c_void_p
_D = ctypes.c_double
_I = ctypes.c_int
_L = ctypes.c_long

# strategy mask bits (same convention as include/sof_cuda.h, test_mesher.cpp:202-206)
TILE_SCHEDULING, MIN_Z, EARLY_STOP, PRUNE, DEAD_CULL = 1, 2, 4, 8, 16
ALL = 31
NAIVE = 0


def available(glibc: bool = False) -> bool:
    return os.path.exists(REF_GLIBC_SO if glibc else REF_SO)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


@dataclass
class Scene:
    pos: np.ndarray      # [n,3] f64
    scale: np.ndarray    # [n,3]
    rot: np.ndarray      # [n,4] (w,x,y,z)
    opacity: np.ndarray  # [n]
    dc: np.ndarray       # [n,3]

    @property
    def n(self) -> int:
        return int(self.opacity.shape[0])

    @staticmethod
    def empty(n: int) -> "Scene":
        return Scene(np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 4)), np.zeros(n), np.zeros((n, 3)))

    def subset(self, idx) -> "Scene":
        return Scene(*(np.ascontiguousarray(a[idx]) for a in (self.pos, self.scale, self.rot, self.opacity, self.dc)))


@dataclass
class Cameras:
    R: np.ndarray        # [V,3,3] world-to-view, row-major
    t: np.ndarray        # [V,3]
    intr: np.ndarray     # [V,4] fx, fy, cx, cy
    wh: np.ndarray       # [V,2] int32 width, height
    nearfar: np.ndarray  # [V,2]

    @property
    def v(self) -> int:
        return int(self.t.shape[0])

    @staticmethod
    def empty(v: int) -> "Cameras":
        return Cameras(np.zeros((v, 3, 3)), np.zeros((v, 3)), np.zeros((v, 4)),
                       np.zeros((v, 2), np.int32), np.zeros((v, 2)))

    def subset(self, idx) -> "Cameras":
        return Cameras(*(np.ascontiguousarray(a[idx]) for a in (self.R, self.t, self.intr, self.wh, self.nearfar)))

    @staticmethod
    def concat(cams) -> "Cameras":
        return Cameras(*(np.ascontiguousarray(np.concatenate([getattr(c, f) for c in cams]))
                         for f in ("R", "t", "intr", "wh", "nearfar")))


class RefLib:
    """Thin wrapper over the extern "C" surface in oracle/ref_capi.cpp."""

    def __init__(self, glibc: bool = False):
        path = REF_GLIBC_SO if glibc else REF_SO
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (needs /root/reference)")
        self.lib = ctypes.CDLL(path)
        L = self.lib
        L.sofref_last_error.restype = ctypes.c_char_p
        L.sofref_distortion_loss.argtypes = [_L, _P, _P, _P, _D, _D, _I, _P, _P, _P]
        L.sofref_extent_loss.argtypes = [_L] + [_P] * 6 + [_D, _D] + [_P] * 6
        L.sofref_depth_normal_loss.argtypes = [_L] + [_P] * 7
        L.sofref_opacity_supervision_loss.argtypes = [_L] + [_P] * 7
        L.sofref_normal_smoothness_loss.argtypes = [_I, _I, _P, _P, _P, _I, _P, _P, _P]
        L.sofref_l1_rgb_loss.restype = _D
        L.sofref_l1_rgb_loss.argtypes = [_L, _P, _P]
        L.sofref_exp_probe.restype = _D
        L.sofref_exp_probe.argtypes = [_D]
        L.sofref_log_probe.restype = _D
        L.sofref_log_probe.argtypes = [_D]
        L.sofref_random_scene.argtypes = [ctypes.c_uint, _I, _D] + [_P] * 5
        L.sofref_shell_scene.argtypes = [_I, _D, _D, _D] + [_P] * 5
        L.sofref_orbit_cameras.argtypes = [_I, _D, _D, _I] + [_P] * 5
        L.sofref_axis_cameras.argtypes = [_D, _D, _I] + [_P] * 5
        L.sofref_look_at.argtypes = [_P, _P, _P, _D, _D, _I, _I] + [_P] * 5
        L.sofref_bag_size.restype = _L
        L.sofref_bag_size.argtypes = [_P, ctypes.c_char_p]
        L.sofref_bag_copy.argtypes = [_P, ctypes.c_char_p, _P]
        L.sofref_bag_free.argtypes = [_P]
        L.sofref_create.restype = _P
        L.sofref_create.argtypes = [_I] + [_P] * 5 + [_I] + [_P] * 5 + [_D, _I]
        L.sofref_destroy.argtypes = [_P]
        L.sofref_precompute_dump.argtypes = [_P, _P]
        L.sofref_tile_binding.restype = _P
        L.sofref_tile_binding.argtypes = [_P, _I, _I]
        L.sofref_schedule_points.restype = _P
        L.sofref_schedule_points.argtypes = [_P, _I, _L, _P, _I]
        L.sofref_eval_create.restype = _P
        L.sofref_eval_create.argtypes = [_P, _I, _I]
        L.sofref_eval_destroy.argtypes = [_P]
        L.sofref_eval_counters.argtypes = [_P, _P]
        L.sofref_eval_reset_counters.argtypes = [_P]
        L.sofref_view_opacity.argtypes = [_P, _I, _L, _P, _I, _P, _P, _P]
        L.sofref_classify_points.argtypes = [_P, _L, _P, _P]
        L.sofref_value_at.argtypes = [_P, _L, _P, _P]
        L.sofref_opacity_at_point.argtypes = [_P, _L, _P, _P]
        L.sofref_label_grid.argtypes = [_P, _L, _P, _I, _I, _P]
        L.sofref_marching_tets.restype = _P
        L.sofref_marching_tets.argtypes = [_L, _P, _L, _P, _P]
        L.sofref_refine.argtypes = [_P, _L, _P, _L, _P, _P, _I]
        L.sofref_assemble.restype = _P
        L.sofref_assemble.argtypes = [_L, _P, _L, _P, _P, _D, _D]
        L.sofref_extract_tetgrid.restype = _P
        L.sofref_extract_tetgrid.argtypes = [_P, _L, _P, _L, _P, _I, _I, _I, _I]
        L.sofref_seed_points.restype = _P
        L.sofref_seed_points.argtypes = [_P, _I, _I, ctypes.c_double]
        L.sofref_seed_delaunay.restype = _P
        L.sofref_seed_delaunay.argtypes = [_P, _I, _I]
        L.sofref_extract_full.restype = _P
        L.sofref_extract_full.argtypes = [_P, _I, _I, _I, _I]
        L.sofref_write_mesh_obj.restype = _I
        L.sofref_write_mesh_obj.argtypes = [_L, _P, _L, _P, ctypes.c_char_p]
        L.sofref_read_mesh_ply.restype = _P
        L.sofref_read_mesh_ply.argtypes = [ctypes.c_char_p]
        L.sofref_parse_scene.restype = _P
        L.sofref_parse_scene.argtypes = [ctypes.c_char_p]
        L.sofref_write_scene.restype = _I
        L.sofref_write_scene.argtypes = [_I, _P, _P, _P, _P, _P, ctypes.c_char_p]
        L.sofref_write_mesh_ply.restype = _I
        L.sofref_write_mesh_ply.argtypes = [_L, _P, _L, _P, ctypes.c_char_p]
        L.sofref_save_cameras.restype = _I
        L.sofref_save_cameras.argtypes = [_I, _P, _P, _P, _P, _P, ctypes.c_char_p]
        L.sofref_load_cameras.restype = _I
        L.sofref_load_cameras.argtypes = [ctypes.c_char_p, _I, _P, _P, _P, _P, _P]
        L.sofref_render_depth_map.argtypes = [_P, _I, _I, _I, _I, _I, _P, _P]
        L.sofref_render_pixels.argtypes = [_P, _I, _I, _L, _P, _P, _P, _P, _P, _P]
        L.sofref_normal_from_depth.argtypes = [_P, _I, _P, _P, _P]
        L.sofref_gaussian_normals.argtypes = [_P, _L, _P, _P, _P, _P, _P]
        L.sofref_render_maps.argtypes = [_P, _I, _I, _I, ctypes.c_char_p, ctypes.c_char_p]
        L.sofref_write_float_map.argtypes = [_I, _I, _I, _P, ctypes.c_char_p]
        L.sofref_write_float_map.restype = _I
        L.sofref_collect_contributions.restype = _P
        L.sofref_collect_contributions.argtypes = [_P, _I, _I, _I]
        L.sofref_render_pixels_windowed.argtypes = [_P, _I, _I, _L, _L, _P, _P, _P, _P, _P, _P]
        L.sofref_windowed_resort.argtypes = [_L, _P, _P, _L, _P]
        L.sofref_delaunay.restype = _P
        L.sofref_delaunay.argtypes = [_L, _P]
        L.sofref_render_pixel_lists.argtypes = [_P, _I, _L, _P, _P, _P, _P, _P, _P, _P]

    # ---- fixtures ----
    def write_float_map(self, width: int, height: int, channels: int, data, path: str) -> int:
        """write_float_map (io_maps.hpp:30-38); returns 1 when the reference throws."""
        data = np.ascontiguousarray(data, np.float32)
        return self.lib.sofref_write_float_map(width, height, channels, _ptr(data), path.encode())

    def windowed_resort(self, t_star, index, window: int) -> np.ndarray:
        """windowed_resort (opacity_field.hpp:66-91) of one arrival-ordered list; returns
        the gaussian_index sequence."""
        t = np.ascontiguousarray(t_star, np.float64)
        i = np.ascontiguousarray(index, np.int32)
        out = np.empty(len(t), np.int32)
        self.lib.sofref_windowed_resort(len(t), _ptr(t), _ptr(i), int(window), _ptr(out))
        return out

    def delaunay(self, xyz) -> np.ndarray:
        """delaunay_tetrahedralize (delaunay.hpp:52-142) of arbitrary points: tets [T, 4]."""
        xyz = np.ascontiguousarray(xyz, np.float64).reshape(-1, 3)
        h = self.lib.sofref_delaunay(len(xyz), _ptr(xyz))
        if not h:
            raise ValueError(self.lib.sofref_last_error().decode())
        return self._bag(h, {"tets": np.int32})["tets"].reshape(-1, 4)

    def random_scene(self, seed: int, count: int, extent: float = 1.0) -> Scene:
        s = Scene.empty(count)
        self.lib.sofref_random_scene(seed, count, extent, *(_ptr(a) for a in (s.pos, s.scale, s.rot, s.opacity, s.dc)))
        return s

    def shell_scene(self, count: int, radius=1.0, scale=0.12, opacity=0.9) -> Scene:
        s = Scene.empty(count)
        self.lib.sofref_shell_scene(count, radius, scale, opacity, *(_ptr(a) for a in (s.pos, s.scale, s.rot, s.opacity, s.dc)))
        return s

    def orbit_cameras(self, count: int, dist: float, extent: float, res: int = 64) -> Cameras:
        c = Cameras.empty(count)
        self.lib.sofref_orbit_cameras(count, dist, extent, res, *(_ptr(a) for a in (c.R, c.t, c.intr, c.wh, c.nearfar)))
        return c

    def axis_cameras(self, dist: float, extent: float, res: int = 96) -> Cameras:
        c = Cameras.empty(3)
        self.lib.sofref_axis_cameras(dist, extent, res, *(_ptr(a) for a in (c.R, c.t, c.intr, c.wh, c.nearfar)))
        return c

    def look_at(self, eye, target, up, fx, fy, w, h) -> Cameras:
        c = Cameras.empty(1)
        e, t, u = (np.asarray(x, np.float64) for x in (eye, target, up))
        self.lib.sofref_look_at(_ptr(e), _ptr(t), _ptr(u), fx, fy, w, h,
                                *(_ptr(a) for a in (c.R, c.t, c.intr, c.wh, c.nearfar)))
        return c

    # ---- bags ----
    def _bag(self, h, spec: dict) -> dict:
        if not h:
            raise RuntimeError(self.lib.sofref_last_error().decode())
        out = {}
        for k, dt in spec.items():
            nbytes = self.lib.sofref_bag_size(h, k.encode())
            if nbytes < 0:
                continue
            a = np.empty(nbytes // np.dtype(dt).itemsize, dt)
            self.lib.sofref_bag_copy(h, k.encode(), _ptr(a))
            out[k] = a
        self.lib.sofref_bag_free(h)
        return out

    def context(self, scene: Scene, cams: Cameras, filter_scale: float = 0.0, z_mode: int = 0) -> "RefContext":
        return RefContext(self, scene, cams, filter_scale, z_mode)

    def marching_tets(self, verts, tets, opacity) -> dict:
        verts = np.ascontiguousarray(verts, np.float64)
        tets = np.ascontiguousarray(tets, np.int32)
        opacity = np.ascontiguousarray(opacity, np.float64)
        h = self.lib.sofref_marching_tets(len(verts), _ptr(verts), len(tets), _ptr(tets), _ptr(opacity))
        b = self._bag(h, {"edges": np.int32, "vertices": np.float64, "triangles": np.int32})
        return {"edges": b["edges"].reshape(-1, 2), "vertices": b["vertices"].reshape(-1, 3),
                "triangles": b["triangles"].reshape(-1, 3)}

    def assemble(self, verts, tris, residuals=None, weld_eps=1e-7, min_area=1e-14) -> dict:
        verts = np.ascontiguousarray(verts, np.float64)
        tris = np.ascontiguousarray(tris, np.int32)
        res = None if residuals is None else np.ascontiguousarray(residuals, np.float64)
        h = self.lib.sofref_assemble(len(verts), _ptr(verts), len(tris), _ptr(tris), _ptr(res), weld_eps, min_area)
        b = self._bag(h, {"vertices": np.float64, "triangles": np.int32, "residuals": np.float64})
        return {"vertices": b["vertices"].reshape(-1, 3), "triangles": b["triangles"].reshape(-1, 3),
                "residuals": b["residuals"]}

    def write_mesh_ply(self, verts, tris, path: str) -> None:
        verts = np.ascontiguousarray(verts, np.float64)
        tris = np.ascontiguousarray(tris, np.int32)
        if self.lib.sofref_write_mesh_ply(len(verts), _ptr(verts), len(tris), _ptr(tris), path.encode()):
            raise RuntimeError(self.lib.sofref_last_error().decode())


    def save_cameras(self, R, t, intr, wh, nearfar, path: str) -> None:
        a = [np.ascontiguousarray(x, np.float64) for x in (R, t, intr)]
        wh = np.ascontiguousarray(wh, np.int32)
        nf = np.ascontiguousarray(nearfar, np.float64)
        if self.lib.sofref_save_cameras(len(a[1]), *(_ptr(x) for x in a), _ptr(wh), _ptr(nf), path.encode()):
            raise RuntimeError(self.lib.sofref_last_error().decode())

    def load_cameras(self, path: str):
        """(R [V, 9], t [V, 3], intr [V, 4], wh [V, 2], nearfar [V, 2])."""
        v = self.lib.sofref_load_cameras(path.encode(), 0, None, None, None, None, None)
        if v < 0:
            raise RuntimeError(self.lib.sofref_last_error().decode())
        out = (np.empty((v, 9)), np.empty((v, 3)), np.empty((v, 4)), np.empty((v, 2), np.int32), np.empty((v, 2)))
        self.lib.sofref_load_cameras(path.encode(), v, *(_ptr(x) for x in out))
        return out

    def write_mesh_obj(self, verts, tris, path: str) -> None:
        verts = np.ascontiguousarray(verts, np.float64)
        tris = np.ascontiguousarray(tris, np.int32)
        if self.lib.sofref_write_mesh_obj(len(verts), _ptr(verts), len(tris), _ptr(tris), path.encode()):
            raise RuntimeError(self.lib.sofref_last_error().decode())

    def read_mesh_ply(self, path: str):
        b = self._bag(self.lib.sofref_read_mesh_ply(path.encode()), {"vertices": np.float64, "triangles": np.int32})
        return b["vertices"].reshape(-1, 3), b["triangles"].reshape(-1, 3)

    def parse_scene(self, path: str) -> Scene:
        """parse_scene (io_scene.hpp:54-134); RuntimeError with the reference's message."""
        b = self._bag(self.lib.sofref_parse_scene(path.encode()),
                      {k: np.float64 for k in ("pos", "scale", "rot", "opacity", "dc")})
        return Scene(b["pos"].reshape(-1, 3), b["scale"].reshape(-1, 3), b["rot"].reshape(-1, 4), b["opacity"],
                     b["dc"].reshape(-1, 3))

    def write_scene(self, scene: Scene, path: str) -> None:
        s = [np.ascontiguousarray(a, np.float64) for a in (scene.pos, scene.scale, scene.rot, scene.opacity, scene.dc)]
        if self.lib.sofref_write_scene(len(s[3]), *(_ptr(a) for a in s), path.encode()):
            raise RuntimeError(self.lib.sofref_last_error().decode())


    # ---- training losses (losses.hpp), per ray through the unmodified reference -----------
    def distortion_loss(self, off, alpha, t, near, far, attach_w=True):
        o = np.ascontiguousarray(off, np.int64)
        a, tt = np.ascontiguousarray(alpha, np.float64), np.ascontiguousarray(t, np.float64)
        R, S = len(o) - 1, int(o[-1])
        loss, da, dt = np.empty(R), np.zeros(S), np.empty(S)
        self.lib.sofref_distortion_loss(R, _ptr(o), _ptr(a), _ptr(tt), near, far, int(attach_w), _ptr(loss),
                                        _ptr(da), _ptr(dt))
        return {"loss": loss, "d_alpha": da if attach_w else None, "d_t": dt}

    def extent_loss(self, off, w, a, b, c, bound, near, far):
        o = np.ascontiguousarray(off, np.int64)
        arrs = [np.ascontiguousarray(x, np.float64) for x in (w, a, b, c, bound)]
        R, S = len(o) - 1, int(o[-1])
        loss, skipped = np.empty(R), np.empty(R, np.int32)
        g = [np.empty(S) for _ in range(4)]
        self.lib.sofref_extent_loss(R, _ptr(o), *(_ptr(x) for x in arrs), near, far, _ptr(loss), _ptr(skipped),
                                    *(_ptr(x) for x in g))
        return {"loss": loss, "skipped": skipped, "d_a": g[0], "d_b": g[1], "d_c": g[2], "d_w": g[3]}

    def depth_normal_loss(self, off, w, normals, pixel_normals):
        o = np.ascontiguousarray(off, np.int64)
        ww = np.ascontiguousarray(w, np.float64)
        nn = np.ascontiguousarray(normals, np.float64).reshape(-1, 3)
        pn = np.ascontiguousarray(pixel_normals, np.float64).reshape(-1, 3)
        R, S = len(o) - 1, int(o[-1])
        loss, dw, dn = np.empty(R), np.empty(S), np.empty((S, 3))
        self.lib.sofref_depth_normal_loss(R, _ptr(o), _ptr(ww), _ptr(nn), _ptr(pn), _ptr(loss), _ptr(dw), _ptr(dn))
        return {"loss": loss, "d_w": dw, "d_n": dn}

    def opacity_supervision_loss(self, off, contribs, depth):
        o = np.ascontiguousarray(off, np.int64)
        rc = np.ascontiguousarray(contribs, np.float64).reshape(-1, 6)
        dep = np.ascontiguousarray(depth, np.float64)
        R, S = len(o) - 1, int(o[-1])
        loss, fv, defined, da = np.empty(R), np.empty(R), np.empty(R, np.uint8), np.empty(S)
        self.lib.sofref_opacity_supervision_loss(R, _ptr(o), _ptr(rc), _ptr(dep), _ptr(loss), _ptr(fv),
                                                 _ptr(defined), _ptr(da))
        return {"loss": loss, "field_value": fv, "defined": defined.astype(bool), "d_alpha": da}

    def normal_smoothness_loss(self, normals, valid, image, per_channel=False):
        n = np.ascontiguousarray(normals, np.float64)
        img = np.ascontiguousarray(image, np.float64)
        v = np.ascontiguousarray(valid, np.uint8)
        H, W = v.shape
        loss, used, dn = np.zeros(1), np.zeros(1, np.int64), np.empty((H, W, 3))
        self.lib.sofref_normal_smoothness_loss(W, H, _ptr(n), _ptr(v), _ptr(img), int(per_channel), _ptr(loss),
                                               _ptr(used), _ptr(dn))
        return {"loss": float(loss[0]), "pixels_used": int(used[0]), "d_normal": dn}

    def l1_rgb_loss(self, rendered, reference):
        a = np.ascontiguousarray(rendered, np.float64).reshape(-1, 3)
        b = np.ascontiguousarray(reference, np.float64).reshape(-1, 3)
        return float(self.lib.sofref_l1_rgb_loss(len(a), _ptr(a), _ptr(b)))

class RefContext:
    """ViewSet::build over (scene, cameras) held by the reference library."""

    def __init__(self, ref: RefLib, scene: Scene, cams: Cameras, filter_scale=0.0, z_mode=0):
        self.ref, self.scene, self.cams = ref, scene, cams
        L = ref.lib
        self.h = L.sofref_create(scene.n, *(_ptr(a) for a in (scene.pos, scene.scale, scene.rot, scene.opacity, scene.dc)),
                                 cams.v, *(_ptr(a) for a in (cams.R, cams.t, cams.intr, cams.wh, cams.nearfar)),
                                 filter_scale, z_mode)
        if not self.h:
            raise ValueError(L.sofref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.sofref_destroy(self.h)
            self.h = None

    def precompute(self) -> np.ndarray:
        out = np.empty((self.cams.v, self.scene.n, 13))
        self.ref.lib.sofref_precompute_dump(self.h, _ptr(out))
        return out

    def tile_binding(self, view: int, tile_size: int = 16) -> dict:
        return self.ref._bag(self.ref.lib.sofref_tile_binding(self.h, view, tile_size),
                             {"offsets": np.int64, "entries": np.int32, "dims": np.int32})

    def schedule_points(self, view: int, xyz, tile_size: int = 16) -> dict:
        xyz = np.ascontiguousarray(xyz, np.float64)
        b = self.ref._bag(self.ref.lib.sofref_schedule_points(self.h, view, len(xyz), _ptr(xyz), tile_size),
                          {"tile_assignment": np.int32, "order": np.int32, "key_tile": np.int32,
                           "key_depth": np.float64, "block_counts": np.int32, "block_to_tile": np.int32,
                           "block_ranges": np.int32})
        b["block_ranges"] = b["block_ranges"].reshape(-1, 2)
        return b

    def evaluator(self, strategies: int, tile_size: int = 16) -> "RefEvaluator":
        return RefEvaluator(self, strategies, tile_size)

    def opacity_at_point(self, xyz) -> np.ndarray:
        xyz = np.ascontiguousarray(xyz, np.float64)
        out = np.empty(len(xyz))
        self.ref.lib.sofref_opacity_at_point(self.h, len(xyz), _ptr(xyz), _ptr(out))
        return out

    def seed_points(self, bounding: int = 0, cutoff: int = 1, filter_scale: float = 0.0):
        """build_seed_points (seed_points.hpp:41-87) -> (points [S, 3], provenance [S])."""
        b = self.ref._bag(self.ref.lib.sofref_seed_points(self.h, bounding, cutoff, filter_scale),
                          {"points": np.float64, "provenance": np.uint8})
        return b["points"].reshape(-1, 3), b["provenance"]

    def seed_delaunay(self, bounding: int = 0, cutoff: int = 1) -> dict:
        b = self.ref._bag(self.ref.lib.sofref_seed_delaunay(self.h, bounding, cutoff),
                          {"vertices": np.float64, "tets": np.int32})
        return {"vertices": b["vertices"].reshape(-1, 3), "tets": b["tets"].reshape(-1, 4)}

    def extract_tetgrid(self, verts, tets, strategies=ALL, tile_size=16, iterations=8, threads=0) -> dict:
        verts = np.ascontiguousarray(verts, np.float64)
        tets = np.ascontiguousarray(tets, np.int32)
        h = self.ref.lib.sofref_extract_tetgrid(self.h, len(verts), _ptr(verts), len(tets), _ptr(tets),
                                                strategies, tile_size, iterations, threads)
        b = self.ref._bag(h, {"grid_opacity": np.float64, "edges": np.int32, "refined": np.float64,
                              "march_triangles": np.int32, "vertices": np.float64, "triangles": np.int32,
                              "counters": np.uint64, "seconds": np.float64})
        for k, w in (("edges", 2), ("refined", 3), ("march_triangles", 3), ("vertices", 3), ("triangles", 3)):
            b[k] = b[k].reshape(-1, w)
        return b

    def extract_full(self, strategies=ALL, tile_size=16, iterations=8, threads=0) -> dict:
        h = self.ref.lib.sofref_extract_full(self.h, strategies, tile_size, iterations, threads)
        b = self.ref._bag(h, {"vertices": np.float64, "triangles": np.int32, "counters": np.uint64})
        b["vertices"] = b["vertices"].reshape(-1, 3)
        b["triangles"] = b["triangles"].reshape(-1, 3)
        return b

    def render_depth_map(self, view: int, exact: bool = True, rows=None, threads: int = 0):
        w, h = (int(x) for x in self.cams.wh[view])
        r0, r1 = (0, h) if rows is None else rows
        depth = np.full((h, w), np.nan)
        opac = np.zeros((h, w))
        self.ref.lib.sofref_render_depth_map(self.h, view, int(exact), r0, r1, threads, _ptr(depth), _ptr(opac))
        return depth, opac

    def normal_from_depth(self, view: int, depth):
        w, h = (int(x) for x in self.cams.wh[view])
        depth = np.ascontiguousarray(depth, np.float64).reshape(h, w)
        normal, valid = np.zeros((h, w, 3)), np.zeros((h, w), np.uint8)
        self.ref.lib.sofref_normal_from_depth(self.h, view, _ptr(depth), _ptr(normal), _ptr(valid))
        return normal, valid

    def gaussian_normals(self, gidx, origin, direction, t):
        gidx = np.ascontiguousarray(gidx, np.int32)
        o, d = (np.ascontiguousarray(a, np.float64).reshape(-1, 3) for a in (origin, direction))
        t = np.ascontiguousarray(t, np.float64)
        out = np.zeros((len(gidx), 3))
        self.ref.lib.sofref_gaussian_normals(self.h, len(gidx), *(_ptr(a) for a in (gidx, o, d, t, out)))
        return out

    def render_maps(self, view: int, depth_path: str, normal_path: str, exact: bool = True, threads: int = 0):
        self.ref.lib.sofref_render_maps(self.h, view, int(exact), threads, depth_path.encode(), normal_path.encode())

    def render_pixels(self, view: int, pix, exact: bool = True, threads: int = 1) -> dict:
        """collect_contributions + render_pixel per pixel. threads > 1 splits the pixels
        over host threads (ctypes releases the GIL; the reference call is const)."""
        pix = np.ascontiguousarray(pix, np.int32)
        n = len(pix)
        out = {"color": np.empty((n, 3)), "depth": np.empty(n), "acc": np.empty(n), "tfinal": np.empty(n),
               "ncontrib": np.empty(n, np.int32)}

        def run(a, b):
            if b > a:
                self.ref.lib.sofref_render_pixels(self.h, view, int(exact), b - a, _ptr(pix[a:b]),
                                                  *(_ptr(out[k][a:b]) for k in
                                                    ("color", "depth", "acc", "tfinal", "ncontrib")))
        if threads <= 1 or n < 2 * threads:
            run(0, n)
        else:
            from concurrent.futures import ThreadPoolExecutor
            cuts = np.linspace(0, n, 4 * threads + 1).astype(int)
            with ThreadPoolExecutor(threads) as ex:
                list(ex.map(lambda k: run(cuts[k], cuts[k + 1]), range(len(cuts) - 1)))
        return out

    def render_pixels_windowed(self, view: int, pix, window: int, exact: bool = True) -> dict:
        """collect_contributions, arrival order by view-space centre depth (ties: index),
        windowed_resort(window), render_pixel -- per pixel."""
        pix = np.ascontiguousarray(pix, np.int32)
        n = len(pix)
        out = {"color": np.empty((n, 3)), "depth": np.empty(n), "acc": np.empty(n), "tfinal": np.empty(n),
               "ncontrib": np.empty(n, np.int32)}
        self.ref.lib.sofref_render_pixels_windowed(self.h, view, int(exact), int(window), n, _ptr(pix),
                                                   *(_ptr(out[k]) for k in ("color", "depth", "acc", "tfinal",
                                                                            "ncontrib")))
        return out

    def render_pixel_lists(self, off, idx, vals, exact: bool = True) -> dict:
        """render_pixel (opacity_field.hpp:201-219) of given contribution lists."""
        off = np.ascontiguousarray(off, np.int64)
        idx = np.ascontiguousarray(idx, np.int32)
        vals = np.ascontiguousarray(vals, np.float64).reshape(-1, 6)
        nl = len(off) - 1
        out = {"color": np.empty((nl, 3)), "depth": np.empty(nl), "acc": np.empty(nl), "tfinal": np.empty(nl)}
        self.ref.lib.sofref_render_pixel_lists(self.h, int(exact), nl, _ptr(off), _ptr(idx), _ptr(vals),
                                               *(_ptr(out[k]) for k in ("color", "depth", "acc", "tfinal")))
        return out

    def collect_contributions(self, view: int, px: int, py: int) -> dict:
        return self.ref._bag(self.ref.lib.sofref_collect_contributions(self.h, view, px, py),
                             {"index": np.int32, "t_star": np.float64, "alpha": np.float64, "a": np.float64,
                              "b": np.float64, "c": np.float64, "opacity": np.float64})


class RefEvaluator:
    """FieldEvaluator(gaussians, views, strategies, tile_size) inside the reference library."""

    def __init__(self, ctx: RefContext, strategies: int, tile_size: int = 16):
        self.ctx = ctx
        self.L = ctx.ref.lib
        self.h = self.L.sofref_eval_create(ctx.h, strategies, tile_size)

    def __del__(self):
        if getattr(self, "h", None):
            self.L.sofref_eval_destroy(self.h)
            self.h = None

    def counters(self):
        out = np.zeros(2, np.uint64)
        self.L.sofref_eval_counters(self.h, _ptr(out))
        return {"pairs": int(out[0]), "point_view_evals": int(out[1])}

    def reset_counters(self):
        self.L.sofref_eval_reset_counters(self.h)

    def view_opacity(self, view: int, xyz, classify_mode: bool):
        xyz = np.ascontiguousarray(xyz, np.float64)
        n = len(xyz)
        o, ob, co = np.empty(n), np.empty(n, np.uint8), np.empty(n, np.uint8)
        self.L.sofref_view_opacity(self.h, view, n, _ptr(xyz), int(classify_mode), _ptr(o), _ptr(ob), _ptr(co))
        return o, ob, co

    def classify_points(self, xyz) -> np.ndarray:
        xyz = np.ascontiguousarray(xyz, np.float64)
        out = np.empty(len(xyz), np.uint8)
        self.L.sofref_classify_points(self.h, len(xyz), _ptr(xyz), _ptr(out))
        return out

    def value_at(self, xyz) -> np.ndarray:
        xyz = np.ascontiguousarray(xyz, np.float64)
        out = np.empty(len(xyz))
        self.L.sofref_value_at(self.h, len(xyz), _ptr(xyz), _ptr(out))
        return out

    def label_grid(self, xyz, classify_mode: bool = True, threads: int = 0) -> np.ndarray:
        xyz = np.ascontiguousarray(xyz, np.float64)
        out = np.empty(len(xyz))
        self.L.sofref_label_grid(self.h, len(xyz), _ptr(xyz), int(classify_mode), threads, _ptr(out))
        return out

    def refine(self, grid_xyz, edges, vertices, iterations: int = 8) -> np.ndarray:
        grid_xyz = np.ascontiguousarray(grid_xyz, np.float64)
        edges = np.ascontiguousarray(edges, np.int32)
        v = np.array(vertices, np.float64, copy=True, order="C")
        self.L.sofref_refine(self.h, len(grid_xyz), _ptr(grid_xyz), len(edges), _ptr(edges), _ptr(v), iterations)
        return v
