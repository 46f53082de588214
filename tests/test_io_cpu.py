"""Mesh file IO on the host (io_mesh.hpp:19-120): byte-identical writers and readers
with the reference's error messages (tests/test_io.cpp:142-203)."""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof


def _mesh(seed=3, nv=50, nt=80):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(nv, 3)) * 10 ** rng.uniform(-8, 3, (nv, 1))
    t = rng.integers(0, nv, (nt, 3)).astype(np.int32)
    return sof.Mesh(v, t)


def test_obj_and_ply_writers_byte_identical(ref, tmp_path):
    m = _mesh()
    for fmt, theirs in (("obj", ref.write_mesh_obj), ("ply", ref.write_mesh_ply)):
        a, b = tmp_path / f"a.{fmt}", tmp_path / f"b.{fmt}"
        sof.write_mesh(m, str(a), fmt)
        theirs(m.vertices, m.triangles, str(b))
        assert a.read_bytes() == b.read_bytes(), fmt


def test_mesh_readers_round_trip(ref, tmp_path):
    m = _mesh(5)
    p = str(tmp_path / "m.ply")
    ref.write_mesh_ply(m.vertices, m.triangles, p)
    got = sof.read_mesh_ply(p)
    rv, rt = ref.read_mesh_ply(p)
    np.testing.assert_array_equal(got.vertices.view(np.uint64), rv.view(np.uint64))
    np.testing.assert_array_equal(got.triangles, rt)
    o = str(tmp_path / "m.obj")
    sof.write_mesh_obj(m, o)
    back = sof.read_mesh_obj(o)  # %.17g round-trips doubles exactly
    np.testing.assert_array_equal(back.vertices.view(np.uint64), m.vertices.view(np.uint64))
    np.testing.assert_array_equal(back.triangles, m.triangles)


def test_mesh_ply_errors(ref, tmp_path):
    m = _mesh(7, 4, 2)
    p = tmp_path / "t.ply"
    sof.write_mesh_ply(m, str(p))
    good = p.read_bytes()
    cases = {
        "trunc_faces": good[:-4],
        "trunc_verts": good[: good.index(b"end_header\n") + 11 + 30],
        "quad": good[:-26] + b"\x04" + good[-25:],
        "ascii": good.replace(b"binary_little_endian", b"ascii"),
        "nomagic": b"plx\n" + good[4:],
        "noface": good.replace(b"element face 2\n", b""),
    }
    for name, data in cases.items():
        p.write_bytes(data)
        with pytest.raises(RuntimeError) as theirs:
            ref.read_mesh_ply(str(p))
        with pytest.raises(RuntimeError) as ours:
            sof.read_mesh_ply(str(p))
        assert str(ours.value) == str(theirs.value), name


# ---- camera JSON (io_camera.hpp:17-87; tests/test_io.cpp:109-140) ----------------------------

def test_cameras_save_byte_identical_and_round_trip(ref, tmp_path):
    c = ref.orbit_cameras(3, 4.0, 1.8)  # the reference test's CameraIO.RoundTrip cameras
    c.nearfar[0] = 0.5, 50.0
    ours, theirs = tmp_path / "a.json", tmp_path / "b.json"
    sof.save_cameras(c, str(ours))
    ref.save_cameras(c.R, c.t, c.intr, c.wh, c.nearfar, str(theirs))
    assert ours.read_bytes() == theirs.read_bytes()
    got = sof.load_cameras(str(theirs))
    want = ref.load_cameras(str(ours))
    for a, b in zip((got.R, got.t, got.intr, got.wh, got.nearfar), want):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(got.R, c.R.reshape(-1, 9))
    np.testing.assert_array_equal(got.nearfar, c.nearfar)


def test_cameras_defaults_and_errors(ref, tmp_path):
    p = tmp_path / "c.json"
    p.write_text('{"cameras": [{"width": 4, "height": 5, "fx": 1, "fy": 2, "cx": 2, "cy": 2,'
                 ' "rotation": [1,0,0,0,1,0,0,0,1], "translation": [0,0,1]}]}')
    got, want = sof.load_cameras(str(p)), ref.load_cameras(str(p))
    for a, b in zip((got.R, got.t, got.intr, got.wh, got.nearfar), want):
        np.testing.assert_array_equal(a, b)
    cases = {
        '{"cameras": [{"width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 2, "cy": 2,'
        ' "rotation": [1,0,0,0,1,0,0,0,1]}]}': "missing field 'translation'",
        '{"cameras": [{"width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 2, "cy": 2,'
        ' "rotation": [2,0,0,0,1,0,0,0,1], "translation": [0,0,0]}]}': "degenerate rotation",
        '{"cameras": [{"width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 2, "cy": 2,'
        ' "rotation": [1,0,0,0,1,0,0,0], "translation": [0,0,0]}]}': "rotation must have 9 entries",
        '{"cameras": [{"width": 0, "height": 4, "fx": 1, "fy": 1, "cx": 2, "cy": 2,'
        ' "rotation": [1,0,0,0,1,0,0,0,1], "translation": [0,0,0]}]}': "non-positive intrinsics",
        '{"views": []}': "missing field 'cameras'",
        '{"cameras": [': "camera schema error",
    }
    for text, msg in cases.items():
        p.write_text(text)
        for load in (sof.load_cameras, ref.load_cameras):
            with pytest.raises(RuntimeError, match=msg):
                load(str(p))
    with pytest.raises(RuntimeError, match="cannot open camera file"):
        sof.load_cameras(str(tmp_path / "absent.json"))


def _cpp_camera_io(tmp_path):
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "camera_io")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(root, "include"), "-I",
                        os.path.join(root, "oracle", "eigen_shim"), os.path.join(root, "tests", "cpp", "camera_io.cpp"),
                        "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return lambda a, b: subprocess.run([exe, a, b], capture_output=True, text=True)


def test_cpp_cameras_round_trip_byte_identical(ref, tmp_path):
    """C++ drop-in load_cameras + save_cameras reproduce the reference's file byte for byte."""
    run = _cpp_camera_io(tmp_path)
    c = ref.orbit_cameras(5, 4.0, 1.8)
    c.nearfar[0] = 0.5, 50.0
    c.intr[1] = 1e-05, 123456.789, 0.1, 3.0
    c.t[2] = -0.0, 1e20, 2.5e-7
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    ref.save_cameras(c.R, c.t, c.intr, c.wh, c.nearfar, str(a))
    r = run(str(a), str(b))
    assert r.returncode == 0, r.stdout
    assert b.read_bytes() == a.read_bytes()
    e, f = tmp_path / "e.json", tmp_path / "f.json"
    e.write_text('{"cameras": []}')
    ref.save_cameras(np.zeros((0, 9)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 2), np.int32),
                     np.zeros((0, 2)), str(f))
    assert run(str(e), str(b)).returncode == 0 and b.read_bytes() == f.read_bytes()


def test_cpp_cameras_errors(tmp_path):
    run = _cpp_camera_io(tmp_path)
    p = tmp_path / "c.json"
    base = '"width": 4, "height": 4, "fx": 1, "fy": 1, "cx": 2, "cy": 2'
    cases = {
        '{"cameras": [{' + base + ', "rotation": [1,0,0,0,1,0,0,0,1]}]}': "missing field 'translation'",
        '{"cameras": [{' + base + ', "rotation": [2,0,0,0,1,0,0,0,1], "translation": [0,0,0]}]}':
            "degenerate rotation",
        '{"cameras": [{' + base + ', "rotation": [1,0,0,0,1,0,0,0,1], "translation": [0,0]}]}':
            "translation must have 3 entries",
        '{"views": []}': "missing field 'cameras'",
        '{"cameras": [': "camera schema error",
    }
    for text, msg in cases.items():
        p.write_text(text)
        r = run(str(p), str(tmp_path / "o.json"))
        assert r.returncode == 3 and msg in r.stdout, (text, r.stdout)
    r = run(str(tmp_path / "absent.json"), str(tmp_path / "o.json"))
    assert r.returncode == 3 and "cannot open camera file" in r.stdout
