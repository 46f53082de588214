"""Float-map IO (io_maps.hpp:17-84) on the host: byte-identical to the reference
writer, and the reference's FloatMapIO tests (tests/test_io.cpp:205-235)."""
import numpy as np
import pytest

import paper_2506_19139_b200 as sof


def test_write_float_map_byte_identical(ref, tmp_path):
    rng = np.random.default_rng(4)
    for w, h, c in ((5, 3, 2), (17, 9, 3), (1, 1, 1)):
        data = rng.normal(size=w * h * c).astype(np.float32)
        data[::7] = np.nan
        ours, theirs = tmp_path / "a.sofmap", tmp_path / "b.sofmap"
        sof.write_float_map(sof.FloatMap(w, h, c, data), str(ours))
        assert ref.write_float_map(w, h, c, data, str(theirs)) == 0
        assert ours.read_bytes() == theirs.read_bytes()


def test_float_map_round_trip(tmp_path):
    """FloatMapIO.RoundTrip (test_io.cpp:205-219)."""
    data = np.arange(30, dtype=np.float32) * 0.25 - 2.0
    p = str(tmp_path / "map.sofmap")
    sof.write_float_map(sof.FloatMap(5, 3, 2, data), p)
    back = sof.read_float_map(p)
    assert (back.width, back.height, back.channels) == (5, 3, 2)
    np.testing.assert_array_equal(back.data, data)


def test_float_map_truncated_and_bad_header(tmp_path):
    """FloatMapIO.TruncatedRejected / BadHeaderRejected (test_io.cpp:221-235)."""
    p = tmp_path / "t.sofmap"
    sof.write_float_map(sof.FloatMap(4, 4, 1, np.ones(16, np.float32)), str(p))
    p.write_bytes(p.read_bytes()[:-3])
    with pytest.raises(RuntimeError, match="truncated"):
        sof.read_float_map(str(p))
    p.write_bytes(b"notamap 4 4 1\n")
    with pytest.raises(RuntimeError, match="malformed float map header"):
        sof.read_float_map(str(p))
    with pytest.raises(RuntimeError, match="size mismatch"):
        sof.write_float_map(sof.FloatMap(4, 4, 1, np.ones(15, np.float32)), str(p))


def test_map_conversions():
    depth = np.array([[1.5, np.nan], [2.0, 3.25]])
    opac = np.array([[0.5, 0.0], [0.25, 0.75]])
    m = sof.depth_to_map(depth, opac)
    assert (m.width, m.height, m.channels) == (2, 2, 2)
    np.testing.assert_array_equal(m.data.reshape(2, 2, 2)[..., 1], opac.astype(np.float32))
    n = sof.normals_to_map(np.ones((2, 3, 3)))
    assert (n.width, n.height, n.channels) == (3, 2, 3) and n.data.dtype == np.float32
