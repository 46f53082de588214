"""Scene files on the device: parse_scene (io_scene.hpp:54-134) decoded
and activated by k_decode_scene, write_scene (io_scene.hpp:138-181) by k_encode_scene.
Bit-identical parameters, byte-identical files and the reference's error messages
(tests/test_io.cpp:41-107)."""
import struct

import numpy as np
import pytest

import paper_2506_19139_b200 as sof
from oracle.refpy import ALL, Scene

pytestmark = pytest.mark.gpu

REQ = ["x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3", "opacity", "f_dc_0",
       "f_dc_1", "f_dc_2"]


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def assert_scene_bits(a, b):
    for k in ("pos", "scale", "rot", "opacity", "dc"):
        np.testing.assert_array_equal(bits(getattr(a, k)), bits(getattr(b, k)), err_msg=k)


def ply(props, rows, count=None, extra_header="", fmt="binary_little_endian", eol="\n"):
    """A vertex PLY with (type, name) properties and rows of values."""
    codes = {"float": "f", "double": "d", "uchar": "B", "int": "i", "short": "h", "float32": "f", "float64": "d"}
    h = [f"format {fmt} 1.0", "comment made by test_io_gpu", extra_header.rstrip("\n"),
         f"element vertex {len(rows) if count is None else count}"]
    h += [f"property {t} {n}" for t, n in props] + ["end_header"]
    # the magic line must be exactly "ply"; later lines may end in CR LF (io_scene.hpp:70)
    head = "ply\n" + eol.join(x for x in h if x) + eol
    pay = b"".join(struct.pack("<" + "".join(codes[t] for t, _ in props), *r) for r in rows)
    return head.encode() + pay


def random_rows(rng, n, props):
    rows = []
    for _ in range(n):
        v = {"x": rng.normal(), "y": rng.normal(), "z": rng.normal(), "opacity": rng.normal() * 3}
        for k in range(3):
            v[f"scale_{k}"] = rng.uniform(-6, 0)
            v[f"f_dc_{k}"] = rng.normal()
        for k in range(4):
            v[f"rot_{k}"] = rng.normal()
        rows.append([v.get(nm, 7) for _, nm in props])
    return rows


def test_parse_scene_bitexact(ref, tmp_path):
    rng = np.random.default_rng(1)
    layouts = [
        [("float", n) for n in REQ],
        # shuffled, doubles, unknown properties of every size, a duplicated name
        [("uchar", "red"), ("double", "opacity"), ("float", "f_dc_2"), ("short", "junk")]
        + [("double" if i % 2 else "float", n) for i, n in enumerate(REQ) if n not in ("opacity", "f_dc_2")]
        + [("int", "label"), ("float", "x")],
    ]
    for li, props in enumerate(layouts):
        for eol in ("\n", "\r\n"):
            p = tmp_path / f"s{li}.ply"
            p.write_bytes(ply(props, random_rows(rng, 300, props), eol=eol))
            want = ref.parse_scene(str(p))
            got = sof.parse_scene(str(p), ctx=sof.Context(0))
            assert_scene_bits(got, want)


def test_write_scene_byte_identical_and_round_trip(ref, tmp_path):
    scene = ref.random_scene(61, 500, 1.0)
    scene.opacity[:3] = [0.0, 1.0, 1e-300]  # clamp paths of the logit
    scene.scale[3] = [0.0, 1e-12, 2.0]      # max(s, 1e-8)
    a, b = tmp_path / "a.ply", tmp_path / "b.ply"
    ctx = sof.Context(0)
    sof.write_scene(scene, str(a), ctx=ctx)
    ref.write_scene(scene, str(b))
    assert a.read_bytes() == b.read_bytes()
    got = sof.parse_scene(str(a), ctx=ctx)
    assert_scene_bits(got, ref.parse_scene(str(a)))
    assert np.allclose(got.pos, scene.pos, atol=1e-5)  # SceneIO.RoundTrip tolerances
    assert np.allclose(np.abs(np.einsum("ij,ij->i", got.rot, scene.rot / np.linalg.norm(scene.rot, axis=1,
                                                                                      keepdims=True))), 1, atol=1e-9)


@pytest.mark.parametrize("case", ["empty", "bigendian", "ascii", "missing", "truncated", "badmagic", "list",
                                  "badtype", "degenerate", "nonfinite", "incomplete", "token", "required_uchar",
                                  "crlf_magic"])
def test_parse_scene_errors(ref, tmp_path, case):
    props = [("float", n) for n in REQ]
    rows = random_rows(np.random.default_rng(2), 4, props)
    if case == "empty":
        data = ply(props, [], count=0)
    elif case == "bigendian":
        data = ply(props, rows, fmt="binary_big_endian")
    elif case == "ascii":
        data = ply(props, rows, fmt="ascii")
    elif case == "missing":
        data = ply(props[:3], [r[:3] for r in rows])
    elif case == "truncated":
        data = ply(props, rows)[:-10]
    elif case == "badmagic":
        data = b"not a ply file\n"
    elif case == "list":
        data = ply(props, rows).replace(b"property float x\n", b"property list uchar int x\n")
    elif case == "badtype":
        data = ply(props, rows).replace(b"property float x\n", b"property quad x\n")
    elif case == "degenerate":
        rows[2][6:10] = [0.0, 0.0, 0.0, 0.0]
        rows[3][0] = float("inf")
        data = ply(props, rows)
    elif case == "nonfinite":
        rows[1][3] = 1000.0  # exp overflows
        rows[2][6:10] = [0.0, 0.0, 0.0, 0.0]
        data = ply(props, rows)
    elif case == "incomplete":
        data = ply(props, rows).split(b"end_header")[0]
    elif case == "token":
        data = ply(props, rows).replace(b"comment made", b"bogus made")
    elif case == "crlf_magic":
        data = b"ply\r\n" + ply(props, rows)[4:]
    else:  # required_uchar
        p2 = [("uchar", "x")] + props[1:]
        data = ply(p2, [[1] + r[1:] for r in rows])
    p = tmp_path / f"{case}.ply"
    p.write_bytes(data)
    with pytest.raises(RuntimeError) as theirs:
        ref.parse_scene(str(p))
    with pytest.raises(RuntimeError) as ours:
        sof.parse_scene(str(p), ctx=sof.Context(0))
    assert str(theirs.value) in str(ours.value), (str(ours.value), str(theirs.value))


def test_loaded_scene_labels_bitexact(ref, tmp_path):
    """A scene loaded from a file drives the evaluator like sof_set_scene would."""
    scene = ref.random_scene(52, 300, 1.0)
    p = tmp_path / "s.ply"
    ref.write_scene(scene, str(p))
    parsed = ref.parse_scene(str(p))
    cams = ref.orbit_cameras(3, 4.0, 1.8, 48)
    ctx = sof.Context(0)
    ctx.load_scene_ply(str(p))
    ctx.set_views(cams)
    views = sof.ViewSet(ctx, ctx.scene, ctx.cams, 0.0)
    pts = np.random.default_rng(4).uniform(-1.2, 1.2, (2000, 3))
    ev = sof.FieldEvaluator(ctx.scene, views, sof.EvalStrategies.all())
    want = ref.context(parsed, cams).evaluator(ALL).label_grid(pts)
    np.testing.assert_array_equal(bits(ev.label_grid(pts)), bits(want))
