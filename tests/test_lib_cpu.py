"""Host-side checks that need no GPU: the C-ABI library loads, exports every symbol
declared in include/sof_cuda.h, fails cleanly without a device, and the synthetic
workload generators produce valid tetra inputs."""
import ctypes
import subprocess

import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from paper_2506_19139_b200 import _lib
from paper_2506_19139_b200.workloads import kuhn_lattice, orbit_cameras, synthetic_scene


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _lib.declared_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_null_and_missing_device_paths():
    lib = _lib.load()
    assert lib.sof_version() == 1
    assert lib.sof_set_scene(None, 0, None, None, None, None, None, 0.0) == _lib.SOF_E_INVALID
    assert lib.sof_result_count(None, _lib.R_EDGES) == -1
    assert lib.sof_last_error(None) == b"null context"
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        h = ctypes.c_void_p()
        assert lib.sof_ctx_create(0, ctypes.byref(h)) == _lib.SOF_E_CUDA
        with pytest.raises(sof.SofError):
            sof.Context(0)


def test_loss_entry_points_reject_null_context():
    """Every batched loss entry point returns SOF_E_INVALID on a null context instead of
    dereferencing it (no device needed)."""
    lib = _lib.load()
    off = np.zeros(2, np.int64)
    z = np.zeros(4)
    p = lambda a: a.ctypes.data  # noqa: E731
    assert lib.sof_distortion_loss(None, 1, p(off), p(z), p(z), 0.2, 100.0, 1, p(z), p(z), p(z)) == _lib.SOF_E_INVALID
    assert lib.sof_extent_loss(None, 1, p(off), *([p(z)] * 5), 0.2, 100.0, *([p(z)] * 6)) == _lib.SOF_E_INVALID
    assert lib.sof_depth_normal_loss(None, 1, p(off), *([p(z)] * 6)) == _lib.SOF_E_INVALID
    assert lib.sof_opacity_supervision_loss(None, 1, p(off), *([p(z)] * 6)) == _lib.SOF_E_INVALID
    assert lib.sof_normal_smoothness_loss(None, 1, 1, p(z), p(z), p(z), 0, p(z), p(z), p(z)) == _lib.SOF_E_INVALID
    assert lib.sof_l1_rgb_loss(None, 1, p(z), p(z), p(z)) == _lib.SOF_E_INVALID


def test_comm_entry_points_without_device():
    """The communicator ABI: null checks, and a unique id from NCCL (resolved at run time)
    or a clean SOF_E_NCCL where no NCCL library exists."""
    lib = _lib.load()
    assert lib.sof_comm_info(None, None, None) == _lib.SOF_E_INVALID
    assert lib.sof_comm_init(None, None, 1, 0) == _lib.SOF_E_INVALID
    assert lib.sof_comm_init_local(None, 0) == _lib.SOF_E_INVALID
    assert lib.sof_comm_unique_id(None) == _lib.SOF_E_INVALID
    buf = ctypes.create_string_buffer(_lib.SOF_COMM_ID_BYTES)
    st = lib.sof_comm_unique_id(buf)
    assert st in (_lib.SOF_OK, _lib.SOF_E_NCCL)
    if st == _lib.SOF_OK:
        assert any(buf.raw)


def test_kuhn_lattice_valid():
    v, t = kuhn_lattice(6, -1, 1)
    assert v.shape == (216, 3) and t.shape == (6 * 125, 4)
    a, b, c, d = (v[t[:, k]] for k in range(4))
    vol = np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a)
    assert (vol > 0).all()  # every tet positively oriented
    # the 6 Kuhn tets tile each (jittered) cell: total volume = box volume without jitter
    v0, t0 = kuhn_lattice(6, -1, 1, jitter=0.0)
    a, b, c, d = (v0[t0[:, k]] for k in range(4))
    assert abs(np.einsum("ij,ij->i", np.cross(b - a, c - a), d - a).sum() / 6 - 8.0) < 1e-9


def test_synthetic_scene_shape():
    s = synthetic_scene(20000, 3)
    assert s.pos.shape == (20000, 3) and np.isfinite(s.pos).all()
    dead = (s.opacity < 1 / 255).mean()
    assert 0.07 < dead < 0.09
    assert np.allclose(np.linalg.norm(s.rot, axis=1), 1.0)
    cams = orbit_cameras(10, 160, 100)
    assert np.allclose(np.einsum("vij,vkj->vik", cams.R, cams.R), np.eye(3), atol=1e-12)
