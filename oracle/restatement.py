"""ctypes bindings for oracle/_build/libsof_oracle.so — the C restatement of the
reference hot path (oracle/sof_oracle.c).

TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may call this, as the checker. Pinned against the reference
compiled in place (oracle/_ref) and against tests/golden/ (tests/test_oracle_cpu.py).
Scenes/cameras are plain objects with the array fields used everywhere
(pos, scale, rot, opacity, dc / R, t, intr, wh).
"""
from __future__ import annotations

import ctypes
import os
from types import SimpleNamespace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libsof_oracle.so")

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double


class _Scene(ctypes.Structure):
    _fields_ = [("n", _I64), ("pos", _P), ("scale", _P), ("rot", _P), ("opacity", _P), ("dc", _P),
                ("filter_scale", _D)]


class _Cams(ctypes.Structure):
    _fields_ = [("v", _I), ("R", _P), ("t", _P), ("intr", _P), ("wh", _P)]


_lib = None


def available() -> bool:
    return os.path.exists(SO)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise FileNotFoundError(f"{SO} missing: run `make -C oracle restatement`")
        L = ctypes.CDLL(SO)
        S, C = ctypes.POINTER(_Scene), ctypes.POINTER(_Cams)
        L.sofo_precompute.argtypes = [S, C, _I, _P]
        L.sofo_tile_binding.restype = _I64
        L.sofo_tile_binding.argtypes = [S, C, _I, _I, _P, _P, _I64]
        L.sofo_view_opacity.argtypes = [S, C, _I, _I, _I, _I64, _P, _I, _P, _P, _P, _P]
        L.sofo_label_grid.argtypes = [S, C, _I, _I, _I64, _P, _I, _P, _P]
        L.sofo_classify_points.argtypes = [S, C, _I, _I, _I64, _P, _P, _P]
        L.sofo_label_state.argtypes = [S, C, _I, _I, _I64, _P, _I, _P, _P, _P]
        L.sofo_value_at.argtypes = [S, C, _I, _I, _I64, _P, _P, _P]
        L.sofo_marching_tets.restype = _I64
        L.sofo_marching_tets.argtypes = [_I64, _P, _I64, _P, _P, _P, _P, _P, _P]
        L.sofo_refine.argtypes = [S, C, _I, _I, _P, _I64, _P, _P, _I, _P]
        L.sofo_assemble.restype = _I64
        L.sofo_assemble.argtypes = [_I64, _P, _I64, _P, _D, _D, _P, _P, _P]
        L.sofo_render_pixel.restype = _I64
        L.sofo_render_pixel.argtypes = [S, C, _I, _I, _I, _I, _P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class _Keep:
    """Holds contiguous copies alive while a struct points at them."""

    def __init__(self):
        self.refs = []

    def f64(self, a, w=None):
        a = np.ascontiguousarray(a, np.float64)
        if w:
            a = a.reshape(-1, w)
        self.refs.append(a)
        return a

    def i32(self, a, w=None):
        a = np.ascontiguousarray(a, np.int32)
        if w:
            a = a.reshape(-1, w)
        self.refs.append(a)
        return a


def _scene(k: _Keep, s, filter_scale=0.0):
    pos, sc, rot, op = k.f64(s.pos, 3), k.f64(s.scale, 3), k.f64(s.rot, 4), k.f64(s.opacity)
    dc = k.f64(s.dc, 3) if getattr(s, "dc", None) is not None else k.f64(np.zeros((len(op), 3)))
    return _Scene(len(op), _p(pos), _p(sc), _p(rot), _p(op), _p(dc), float(filter_scale))


def _cams(k: _Keep, c):
    R, t, intr, wh = k.f64(c.R, 9), k.f64(c.t, 3), k.f64(c.intr, 4), k.i32(c.wh, 2)
    return _Cams(len(t), _p(R), _p(t), _p(intr), _p(wh))


# ---- simple deterministic fixtures (numpy; no libstdc++ RNG needed) ----------------------------

def random_scene(seed: int, count: int, extent: float = 1.0):
    """Same distributions as tests/test_util.hpp:22-40 (positions U(-e,e), scales
    U(0.05e, 0.25e), opacity U(0.4, 0.95), random unit quaternion), numpy RNG."""
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(count, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return SimpleNamespace(pos=rng.uniform(-extent, extent, (count, 3)),
                           scale=rng.uniform(0.05 * extent, 0.25 * extent, (count, 3)), rot=q,
                           opacity=rng.uniform(0.4, 0.95, count), dc=rng.uniform(0, 1, (count, 3)))


def orbit_cameras(count: int, dist: float, extent: float, res: int = 64):
    """tests/test_util.hpp:63-84 (camera_towards + golden-spiral eyes) in numpy."""
    from paper_2506_19139_b200.workloads import look_at
    golden = np.pi * (3.0 - np.sqrt(5.0))
    R, t, intr = [], [], []
    for i in range(count):
        z = 0.8 - 1.6 * (i + 0.5) / count
        r = np.sqrt(max(0.0, 1.0 - z * z))
        eye = dist * np.array([r * np.cos(golden * i), r * np.sin(golden * i), z])
        fwd = -eye / np.linalg.norm(eye)
        up = np.array([1.0, 0, 0]) if abs(fwd[1]) > 0.9 else np.array([0, 1.0, 0])
        f = 0.4 * res * np.linalg.norm(eye) / extent
        Ri, ti, ii = look_at(eye, np.zeros(3), up, f, f, res, res)
        R.append(Ri)
        t.append(ti)
        intr.append(ii)
    return SimpleNamespace(R=np.array(R), t=np.array(t), intr=np.array(intr),
                           wh=np.tile(np.array([res, res], np.int32), (count, 1)),
                           nearfar=np.tile([0.2, 100.0], (count, 1)))


# ---- restated reference functions ---------------------------------------------------------------

def precompute(scene, cams, view: int, filter_scale=0.0) -> np.ndarray:
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    out = np.empty((s.n, 13))
    lib().sofo_precompute(ctypes.byref(s), ctypes.byref(c), view, _p(out))
    return out


def tile_binding(scene, cams, view: int, tile_size: int = 16, filter_scale=0.0):
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    w, h = (int(x) for x in np.asarray(cams.wh).reshape(-1, 2)[view])
    T = ((w + tile_size - 1) // tile_size) * ((h + tile_size - 1) // tile_size)
    off = np.empty(T + 1, np.int64)
    m = lib().sofo_tile_binding(ctypes.byref(s), ctypes.byref(c), view, tile_size, _p(off), None, 0)
    ent = np.empty(max(-m, 1), np.int32)
    lib().sofo_tile_binding(ctypes.byref(s), ctypes.byref(c), view, tile_size, _p(off), _p(ent), -m)
    return off, ent[:-m]


def view_opacity(scene, cams, strategies, view, xyz, classify_mode, tile_size=16, filter_scale=0.0):
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    xyz = k.f64(xyz, 3)
    n = len(xyz)
    o, ob, co, cnt = np.empty(n), np.empty(n, np.uint8), np.empty(n, np.uint8), np.zeros(2, np.uint64)
    lib().sofo_view_opacity(ctypes.byref(s), ctypes.byref(c), strategies, tile_size, view, n, _p(xyz),
                            int(classify_mode), _p(o), _p(ob), _p(co), _p(cnt))
    return o, ob, co, cnt


def label_grid(scene, cams, strategies, xyz, classify_mode=True, tile_size=16, filter_scale=0.0):
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    xyz = k.f64(xyz, 3)
    out, cnt = np.empty(len(xyz)), np.zeros(2, np.uint64)
    lib().sofo_label_grid(ctypes.byref(s), ctypes.byref(c), strategies, tile_size, len(xyz), _p(xyz),
                          int(classify_mode), _p(out), _p(cnt))
    return out, cnt


def label_state(scene, cams, strategies, xyz, min_op, ext, classify_mode=True, tile_size=16,
                filter_scale=0.0):
    """label_grid's view loop with caller state; min_op (f64) and ext (u8) updated in place."""
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    xyz = k.f64(xyz, 3)
    assert min_op.dtype == np.float64 and ext.dtype == np.uint8 and min_op.flags.c_contiguous
    cnt = np.zeros(2, np.uint64)
    if c.v:
        lib().sofo_label_state(ctypes.byref(s), ctypes.byref(c), strategies, tile_size, len(xyz), _p(xyz),
                               int(classify_mode), _p(min_op), _p(ext), _p(cnt))
    return cnt


def classify_points(scene, cams, strategies, xyz, tile_size=16, filter_scale=0.0):
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    xyz = k.f64(xyz, 3)
    out, cnt = np.empty(len(xyz), np.uint8), np.zeros(2, np.uint64)
    lib().sofo_classify_points(ctypes.byref(s), ctypes.byref(c), strategies, tile_size, len(xyz), _p(xyz),
                               _p(out), _p(cnt))
    return out, cnt


def value_at(scene, cams, strategies, xyz, tile_size=16, filter_scale=0.0):
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    xyz = k.f64(xyz, 3)
    out, cnt = np.empty(len(xyz)), np.zeros(2, np.uint64)
    lib().sofo_value_at(ctypes.byref(s), ctypes.byref(c), strategies, tile_size, len(xyz), _p(xyz), _p(out),
                        _p(cnt))
    return out, cnt


def marching_tets(verts, tets, opacity):
    k = _Keep()
    v, t, o = k.f64(verts, 3), k.i32(tets, 4), k.f64(opacity)
    cap = max(4 * len(t), 1)
    edges, ev, tris = np.empty((cap, 2), np.int32), np.empty((cap, 3)), np.empty((max(2 * len(t), 1), 3), np.int32)
    nt = ctypes.c_int64()
    ne = lib().sofo_marching_tets(len(v), _p(v), len(t), _p(t), _p(o), _p(edges), _p(ev), _p(tris), ctypes.byref(nt))
    return {"edges": edges[:ne].copy(), "vertices": ev[:ne].copy(), "triangles": tris[:nt.value].copy()}


def refine(scene, cams, strategies, grid_xyz, edges, vertices, iterations=8, tile_size=16, filter_scale=0.0):
    k = _Keep()
    s, c = _scene(k, scene, filter_scale), _cams(k, cams)
    g, e = k.f64(grid_xyz, 3), k.i32(edges, 2)
    v = np.array(vertices, np.float64, order="C").reshape(-1, 3)
    cnt = np.zeros(2, np.uint64)
    lib().sofo_refine(ctypes.byref(s), ctypes.byref(c), strategies, tile_size, _p(g), len(e), _p(e), _p(v),
                      iterations, _p(cnt))
    return v, cnt


def assemble(verts, tris, weld_eps=1e-7, min_area=1e-14):
    k = _Keep()
    v, t = k.f64(verts, 3), k.i32(tris, 3)
    ov, ot = np.empty((max(len(v), 1), 3)), np.empty((max(len(t), 1), 3), np.int32)
    ntr = ctypes.c_int64()
    nv = lib().sofo_assemble(len(v), _p(v), len(t), _p(t), weld_eps, min_area, _p(ov), _p(ot), ctypes.byref(ntr))
    return {"vertices": ov[:nv].copy(), "triangles": ot[:ntr.value].copy()}


def extract_tetgrid(scene, cams, verts, tets, strategies=31, iterations=8, tile_size=16, filter_scale=0.0):
    """extract_mesh's label -> march -> refine -> assemble (extract.hpp:59-78)."""
    opa, c1 = label_grid(scene, cams, strategies, verts, True, tile_size, filter_scale)
    m = marching_tets(verts, tets, opa)
    v, c2 = refine(scene, cams, strategies, verts, m["edges"], m["vertices"], iterations, tile_size, filter_scale)
    mesh = assemble(v, m["triangles"])
    mesh.update(grid_opacity=opa, edges=m["edges"], refined=v, march_triangles=m["triangles"],
                pairs=int(c1[0] + c2[0]), point_view_evals=int(c1[1] + c2[1]))
    return mesh


def render_pixels(scene, cams, view, pix, exact=True):
    k = _Keep()
    s, c = _scene(k, scene), _cams(k, cams)
    pix = np.asarray(pix, np.int32).reshape(-1, 2)
    out = np.empty((len(pix), 6))
    n = np.empty(len(pix), np.int64)
    for i, (px, py) in enumerate(pix):
        n[i] = lib().sofo_render_pixel(ctypes.byref(s), ctypes.byref(c), view, int(px), int(py), int(exact),
                                       _p(out[i]))
    return {"color": out[:, :3], "depth": out[:, 3], "acc": out[:, 4], "tfinal": out[:, 5], "ncontrib": n}
