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
