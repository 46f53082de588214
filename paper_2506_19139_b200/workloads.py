"""Synthetic inputs for the benchmark configurations.

Deterministic generators for the tetra input (a jittered Kuhn/Freudenthal lattice)
and the C2-C5 scenes/cameras. These produce INPUT data only; nothing here is on
the compute path. The scene generator uses numpy's PCG64 with a fixed seed
(2506191390 + config index) instead of libstdc++'s mt19937_64 distributions, so
the same arrays are fed to the GPU path and to the CPU reference.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

SEED_BASE = 2506191390

# per-config sizes (BASELINE.json configs). `edges`: the
# crossing-edge count of one meshing step of the config (measured by bench.py's GPU arm,
# deterministic for the synthetic inputs); the CPU reference arm, which cannot run all
# views, uses it to weigh its bisection sample into the same query mix.
CONFIGS = {
    "C1": dict(gaussians=10_000, views=16, width=256, height=256, lattice=45, edges=22_750),
    "C2": dict(gaussians=1_000_000, views=100, width=1920, height=1080, lattice=0, edges=0),
    "C3": dict(gaussians=3_000_000, views=200, width=1600, height=1064, lattice=300, edges=564_638),
    "C4": dict(gaussians=5_000_000, views=300, width=1920, height=1080, lattice=345, edges=199_568),
    "C5": dict(gaussians=10_000_000, views=500, width=1600, height=1064, lattice=436, edges=1_223_734,
               unbounded=True),
}


@dataclass
class Scene:
    pos: np.ndarray
    scale: np.ndarray
    rot: np.ndarray
    opacity: np.ndarray
    dc: np.ndarray

    @property
    def n(self):
        return len(self.opacity)


@dataclass
class Cams:
    R: np.ndarray
    t: np.ndarray
    intr: np.ndarray
    wh: np.ndarray
    nearfar: np.ndarray

    @property
    def v(self):
        return len(self.t)

    def subset(self, idx):
        return Cams(*(np.ascontiguousarray(a[idx]) for a in (self.R, self.t, self.intr, self.wh, self.nearfar)))


# ---- tetra input -------------------------------------------------------------------------------

_PERMS = list(itertools.permutations(range(3)))  # xyz, xzy, yxz, yzx, zxy, zyx


def _hash3(ids: np.ndarray) -> np.ndarray:
    """Three deterministic uniforms in [0,1) per id (splitmix64)."""
    out = np.empty((len(ids), 3))
    for c in range(3):
        z = (ids.astype(np.uint64) * np.uint64(3) + np.uint64(c + 1)) * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        out[:, c] = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return out


def kuhn_lattice(n: int, lo: float = -2.5, hi: float = 2.5, jitter: float = 0.25):
    """n^3 vertices (id = i + n (j + n k)), 6 (n-1)^3 tets (per cell the 6 Kuhn
    permutations in fixed order, each positively oriented), vertices jittered by
    jitter * cell * (hash3(id) - 0.5)."""
    cell = (hi - lo) / (n - 1)
    g = np.arange(n, dtype=np.float64) * cell + lo
    k, j, i = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    verts = np.stack([g[i.ravel()], g[j.ravel()], g[k.ravel()]], axis=1)
    ids = np.arange(n ** 3, dtype=np.int64)
    if jitter:
        verts += jitter * cell * (_hash3(ids) - 0.5)
    m = n - 1
    ck, cj, ci = np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij")
    base = (ci + n * (cj + n * ck)).ravel().astype(np.int64)
    step = np.array([1, n, n * n], dtype=np.int64)
    tets = np.empty((len(base), 6, 4), dtype=np.int32)
    for p, perm in enumerate(_PERMS):
        v0 = base
        v1 = v0 + step[perm[0]]
        v2 = v1 + step[perm[1]]
        v3 = v2 + step[perm[2]]
        # even permutations are positively oriented; swap the last two otherwise
        parity = sum(1 for a in range(3) for b in range(a + 1, 3) if perm[a] > perm[b]) % 2
        if parity == 0:
            tets[:, p] = np.stack([v0, v1, v2, v3], 1)
        else:
            tets[:, p] = np.stack([v0, v1, v3, v2], 1)
    return verts, tets.reshape(-1, 4)


# ---- cameras --------------------------------------------------------------------------------------

def look_at(eye, target, up, fx, fy, w, h):
    """camera.hpp:62-79 in numpy (same formula; inputs only)."""
    eye = np.asarray(eye, float)
    fwd = np.asarray(target, float) - eye
    fwd = fwd / np.sqrt(fwd @ fwd)
    right = np.cross(fwd, up)
    right = right / np.sqrt(right @ right)
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    t = -R @ eye
    return R, t, np.array([fx, fy, w * 0.5, h * 0.5])


def orbit_cameras(count: int, width: int, height: int, radius: float = 6.0, focal_scale: float = 0.8) -> Cams:
    """Golden-spiral band z in [-0.8, 0.8] looking at the origin (test_util.hpp:72-84
    pattern), f = focal_scale * W; radius 6 (bounded scenes: the whole scene in front) or
    4 (Appendix B's unbounded scene: inside the background shell)."""
    golden = np.pi * (3.0 - np.sqrt(5.0))
    R = np.empty((count, 3, 3))
    t = np.empty((count, 3))
    intr = np.empty((count, 4))
    for i in range(count):
        z = 0.8 - 1.6 * (i + 0.5) / count
        r = np.sqrt(max(0.0, 1.0 - z * z))
        phi = golden * i
        eye = radius * np.array([r * np.cos(phi), r * np.sin(phi), z])
        fwd = -eye / np.linalg.norm(eye)
        up = np.array([1.0, 0, 0]) if abs(fwd[1]) > 0.9 else np.array([0, 1.0, 0])
        f = focal_scale * width
        R[i], t[i], intr[i] = look_at(eye, np.zeros(3), up, f, f, width, height)
    wh = np.tile(np.array([width, height], np.int32), (count, 1))
    nf = np.tile([0.2, 100.0], (count, 1))
    return Cams(R, t, intr, wh, nf)


# ---- scenes ----------------------------------------------------------------------------------------

def _rot_z_to(normals: np.ndarray) -> np.ndarray:
    """Unit quaternions (w,x,y,z) rotating +z onto each normal."""
    z = np.array([0.0, 0.0, 1.0])
    axis = np.cross(np.broadcast_to(z, normals.shape), normals)
    s = np.linalg.norm(axis, axis=1)
    c = normals @ z
    half = np.arctan2(s, c) * 0.5
    axis = np.where(s[:, None] > 1e-12, axis / np.maximum(s, 1e-300)[:, None], np.array([1.0, 0, 0]))
    return np.concatenate([np.cos(half)[:, None], axis * np.sin(half)[:, None]], axis=1)


def synthetic_scene(n: int, config_index: int) -> Scene:
    """Appendix B layout, kept in front of every camera: 85% surface Gaussians on
    3 spheres + a ground disk (z = -1, radius 3.2) + 2 boxes, 7% volumetric
    background in a shell of radius 2.8..4.2 around the objects, 8% dead (opacity
    below 1/255). Everything lies within radius ~4.5 of the origin while the cameras
    orbit at radius 6, so no E-box corner comes near a camera plane: the reference
    bins any Gaussian with a corner behind the camera into EVERY tile
    (tiles.hpp:116-126), which a surrounding background shell would trigger for
    ~half the shell in every view."""
    rng = np.random.default_rng(SEED_BASE + config_index)
    n_bg = int(round(0.07 * n))
    n_dead = int(round(0.08 * n))
    n_surf = n - n_bg - n_dead
    n_on = n_surf + n_dead
    spheres = [((-0.9, 0.2, 0.0), 0.8), ((0.9, -0.3, 0.3), 0.6), ((0.0, 0.9, -0.4), 0.5)]
    boxes = [((-1.8, -1.6, -1.0), (-1.0, -0.8, -0.2)), ((1.0, 1.0, -1.0), (1.7, 1.8, 0.1))]
    disk_r = 3.2
    areas = [4 * np.pi * r * r for _, r in spheres] + [np.pi * disk_r ** 2]
    for lo, hi in boxes:
        d = np.subtract(hi, lo)
        areas.append(2 * (d[0] * d[1] + d[1] * d[2] + d[0] * d[2]))
    areas = np.array(areas)
    which = rng.choice(len(areas), size=n_on, p=areas / areas.sum())
    pos = np.empty((n_on, 3))
    nrm = np.empty((n_on, 3))
    for k, (c, r) in enumerate(spheres):
        m = which == k
        d = rng.normal(size=(m.sum(), 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        pos[m] = np.asarray(c) + r * d
        nrm[m] = d
    m = which == 3
    rr = disk_r * np.sqrt(rng.uniform(0, 1, m.sum()))
    th = rng.uniform(0, 2 * np.pi, m.sum())
    pos[m] = np.stack([rr * np.cos(th), rr * np.sin(th), np.full(m.sum(), -1.0)], 1)
    nrm[m] = (0, 0, 1)
    for b, (lo, hi) in enumerate(boxes):
        m = which == 4 + b
        cnt = int(m.sum())
        lo, hi = np.asarray(lo), np.asarray(hi)
        p = rng.uniform(lo, hi, size=(cnt, 3))
        face = rng.integers(0, 6, cnt)
        ax = face // 2
        side = face % 2
        p[np.arange(cnt), ax] = np.where(side == 1, hi[ax], lo[ax])
        nn = np.zeros((cnt, 3))
        nn[np.arange(cnt), ax] = np.where(side == 1, 1.0, -1.0)
        pos[m] = p
        nrm[m] = nn
    s = 1.5 * np.sqrt(areas.sum() / max(n_on, 1))
    scale_on = np.tile([s, s, 0.1 * s], (n_on, 1)) * rng.uniform(0.7, 1.3, (n_on, 1))
    rot_on = _rot_z_to(nrm)
    opa_on = rng.uniform(0.5, 0.99, n_on)
    dead = np.zeros(n_on, bool)
    dead[rng.choice(n_on, n_dead, replace=False)] = True
    opa_on[dead] = rng.uniform(0.3 / 255, 0.99 / 255, n_dead)
    d = rng.normal(size=(n_bg, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pos_bg = d * rng.uniform(2.8, 4.2, (n_bg, 1))
    scale_bg = np.repeat(rng.uniform(0.01, 0.06, (n_bg, 1)), 3, axis=1) * rng.uniform(0.5, 1.5, (n_bg, 3))
    q = rng.normal(size=(n_bg, 4))
    rot_bg = q / np.linalg.norm(q, axis=1, keepdims=True)
    opa_bg = rng.uniform(0.05, 0.6, n_bg)
    pos = np.concatenate([pos, pos_bg])
    scale = np.concatenate([scale_on, scale_bg])
    rot = np.concatenate([rot_on, rot_bg])
    opa = np.concatenate([opa_on, opa_bg])
    dc = rng.uniform(0, 1, (n, 3))
    perm = rng.permutation(n)
    return Scene(*(np.ascontiguousarray(a[perm]) for a in (pos, scale, rot, opa, dc)))


def _quat_rot(q: np.ndarray) -> np.ndarray:
    """Rotation matrices of unit quaternions (w, x, y, z) (Eigen's formula)."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((len(q), 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def near_camera_plane(pos, scale, rot, opacity, cams: Cams, lo=1e-9, hi=1e-3, chunk=None) -> np.ndarray:
    """Gaussians with an E-box corner (tiles.hpp:104-117: E = tight bound, unclamped
    scales) at view z in (lo, hi] for some camera: Appendix B's rejection rule, which
    keeps the int(floor(px)) overflow window of tiles.hpp:127-130 out of the inputs. On
    the GPU through torch when one is present (input generation only)."""
    n = len(opacity)
    with np.errstate(divide="ignore", invalid="ignore"):
        v = 2.0 * np.log(255.0 * opacity)
    E = np.where(opacity >= 1.0 / 255.0, np.sqrt(np.maximum(v, 0.0)), 0.0)
    signs = np.array([[(m & 1) * 2 - 1, ((m >> 1) & 1) * 2 - 1, ((m >> 2) & 1) * 2 - 1] for m in range(8)], float)
    bad = np.zeros(n, bool)
    chunk = chunk or max(1024, int(2e8) // (8 * max(cams.v, 1)))  # <= 1.6 GB of corner depths per chunk
    try:
        import torch
        dev = "cuda" if torch.cuda.is_available() else None
    except Exception:
        dev = None
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        R = _quat_rot(rot[a:b])
        half = (E[a:b, None] * scale[a:b])[:, None, :] * signs[None]          # [m, 8, 3] local
        corners = pos[a:b, None, :] + np.einsum("mij,mkj->mki", R, half)       # [m, 8, 3] world
        if dev:
            Ct = torch.as_tensor(corners, device=dev)
            Rc = torch.as_tensor(cams.R[:, 2, :], device=dev)                  # [V, 3]
            tz = torch.as_tensor(cams.t[:, 2], device=dev)                     # [V]
            z = torch.einsum("mkj,vj->mkv", Ct, Rc) + tz
            hit = ((z > lo) & (z <= hi)).reshape(b - a, -1).any(1).cpu().numpy()
        else:
            z = np.einsum("mkj,vj->mkv", corners, cams.R[:, 2, :]) + cams.t[:, 2]
            hit = ((z > lo) & (z <= hi)).reshape(b - a, -1).any(1)
        bad[a:b] = hit & (E[a:b] > 0)
    return bad


def unbounded_scene(n: int, config_index: int, cams: Cams, max_rounds: int = 20) -> Scene:
    """SURVEY.md Appendix B as written: 85% surface Gaussians on 3 spheres, the ground
    plane z = -1 within |x|, |y| <= 3 and 2 boxes (scales (s, s, 0.1 s), normal-aligned,
    opacity U(0.5, 0.99)); 7% background uniform in the shell of radii 5..20 around the
    origin (isotropic scale U(0.05, 0.5), opacity U(0.05, 0.6)) — the cameras orbit at
    radius 4, INSIDE the shell, so about half of it lies behind every camera (bound to
    every tile by the reference, tiles.hpp:116-126); 8% dead (surface-like, opacity
    U(0.3/255, 0.99/255)). Gaussians with an E-box corner at view z in (1e-9, 1e-3] for
    any camera are redrawn. numpy PCG64 (seed 2506191390 + config index) instead of
    libstdc++'s mt19937_64: the inputs are generated once and fed to both arms."""
    rng = np.random.default_rng(SEED_BASE + config_index)
    n_bg = int(round(0.07 * n))
    n_dead = int(round(0.08 * n))
    n_on = n - n_bg
    spheres = [((-0.9, 0.2, 0.0), 0.8), ((0.9, -0.3, 0.3), 1.2), ((0.0, 0.9, -0.4), 0.5)]
    boxes = [((-1.8, -1.6, -1.0), (-1.0, -0.8, -0.2)), ((1.0, 1.0, -1.0), (1.7, 1.8, 0.1))]
    areas = [4 * np.pi * r * r for _, r in spheres] + [36.0]
    for blo, bhi in boxes:
        d = np.subtract(bhi, blo)
        areas.append(2 * (d[0] * d[1] + d[1] * d[2] + d[0] * d[2]))
    areas = np.array(areas)
    s_on = 1.5 * np.sqrt(areas.sum() / max(n_on, 1))

    def surface(m):
        which = rng.choice(len(areas), size=m, p=areas / areas.sum())
        p, nn = np.empty((m, 3)), np.empty((m, 3))
        for k, (c, r) in enumerate(spheres):
            sel = which == k
            d = rng.normal(size=(sel.sum(), 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            p[sel], nn[sel] = np.asarray(c) + r * d, d
        sel = which == 3
        p[sel] = np.stack([rng.uniform(-3, 3, sel.sum()), rng.uniform(-3, 3, sel.sum()), np.full(sel.sum(), -1.0)], 1)
        nn[sel] = (0, 0, 1)
        for bb, (blo, bhi) in enumerate(boxes):
            sel = which == 4 + bb
            cnt = int(sel.sum())
            blo, bhi = np.asarray(blo), np.asarray(bhi)
            q = rng.uniform(blo, bhi, size=(cnt, 3))
            face = rng.integers(0, 6, cnt)
            ax, side = face // 2, face % 2
            q[np.arange(cnt), ax] = np.where(side == 1, bhi[ax], blo[ax])
            nq = np.zeros((cnt, 3))
            nq[np.arange(cnt), ax] = np.where(side == 1, 1.0, -1.0)
            p[sel], nn[sel] = q, nq
        scale = np.tile([s_on, s_on, 0.1 * s_on], (m, 1)) * rng.uniform(0.7, 1.3, (m, 1))
        return p, scale, _rot_z_to(nn)

    def background(m):
        d = rng.normal(size=(m, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        r = np.cbrt(rng.uniform(5.0 ** 3, 20.0 ** 3, (m, 1)))  # uniform in the shell's volume
        q = rng.normal(size=(m, 4))
        return d * r, np.repeat(rng.uniform(0.05, 0.5, (m, 1)), 3, axis=1), q / np.linalg.norm(q, axis=1, keepdims=True)

    pos_on, scale_on, rot_on = surface(n_on)
    opa_on = rng.uniform(0.5, 0.99, n_on)
    dead = np.zeros(n_on, bool)
    dead[rng.choice(n_on, n_dead, replace=False)] = True
    opa_on[dead] = rng.uniform(0.3 / 255, 0.99 / 255, n_dead)
    pos_bg, scale_bg, rot_bg = background(n_bg)
    opa_bg = rng.uniform(0.05, 0.6, n_bg)
    pos = np.concatenate([pos_on, pos_bg])
    scale = np.concatenate([scale_on, scale_bg])
    rot = np.concatenate([rot_on, rot_bg])
    opa = np.concatenate([opa_on, opa_bg])
    is_bg = np.arange(n) >= n_on
    for _ in range(max_rounds):  # redraw the Gaussians the rejection rule hits
        bad = near_camera_plane(pos, scale, rot, opa, cams)
        if not bad.any():
            break
        i_on, i_bg = np.flatnonzero(bad & ~is_bg), np.flatnonzero(bad & is_bg)
        if len(i_on):
            pos[i_on], scale[i_on], rot[i_on] = surface(len(i_on))
        if len(i_bg):
            pos[i_bg], scale[i_bg], rot[i_bg] = background(len(i_bg))
    dc = rng.uniform(0, 1, (n, 3))
    perm = rng.permutation(n)
    return Scene(*(np.ascontiguousarray(a[perm]) for a in (pos, scale, rot, opa, dc)))


def config_inputs(name: str, lattice: bool = True, unbounded: bool | None = None):
    """(scene, cameras, (vertices, tets)) of a BASELINE.json config. unbounded (default:
    the config's own setting, C5 on) selects Appendix B's unbounded layout with the
    cameras at radius 4 inside the background shell."""
    cfg = CONFIGS[name]
    idx = int(name[1:])
    if unbounded is None:
        unbounded = cfg.get("unbounded", False)
    if unbounded:
        cams = orbit_cameras(cfg["views"], cfg["width"], cfg["height"], radius=4.0)
        scene = unbounded_scene(cfg["gaussians"], idx, cams)
    else:
        scene = synthetic_scene(cfg["gaussians"], idx)
        cams = orbit_cameras(cfg["views"], cfg["width"], cfg["height"])
    grid = kuhn_lattice(cfg["lattice"]) if (lattice and cfg["lattice"]) else None
    return scene, cams, grid
