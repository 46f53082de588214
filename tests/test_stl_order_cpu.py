"""The libstdc++ ordering restatement (csrc/stl_order.cuh) behind the device
windowed_resort, checked on the host: compiled here with g++ into a throwaway library,
it must reproduce std::sort / std::make_heap+sort_heap element order (ties included) and
the reference's own windowed_resort (opacity_field.hpp:66-91, through oracle/_ref) on
tie-heavy inputs. The same header is what k_render.cu instantiates on the device."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

HARNESS = r'''
#include <algorithm>
#include <cstdint>
#include <vector>
#include "stl_order.cuh"
struct E { double t; int32_t idx; };
extern "C" void stlo_windowed(long n, const double* t, const int32_t* idx, long window, int32_t* out) {
  std::vector<E> in(n), o(n);
  for (long i = 0; i < n; ++i) in[i] = {t[i], idx[i]};
  stlo::windowed_resort(in.data(), o.data(), n, window, [](const E& a, const E& b) { return a.t < b.t; });
  for (long i = 0; i < n; ++i) out[i] = o[i].idx;
}
// 0 when stlo::sort and std::sort (and the heap sort pair) leave the same order
extern "C" int stlo_sort_check(long n, const double* t) {
  std::vector<E> a(n), b(n);
  for (long i = 0; i < n; ++i) a[i] = b[i] = {t[i], int32_t(i)};
  auto lt = [](const E& x, const E& y) { return x.t < y.t; };
  std::sort(a.begin(), a.end(), lt);
  stlo::sort(b.data(), n, lt);
  for (long i = 0; i < n; ++i) if (a[i].idx != b[i].idx) return 1;
  for (long i = 0; i < n; ++i) a[i] = b[i] = {t[i], int32_t(i)};
  std::make_heap(a.begin(), a.end(), lt);
  std::sort_heap(a.begin(), a.end(), lt);
  stlo::make_heap(b.data(), n, lt);
  stlo::sort_heap(b.data(), n, lt);
  for (long i = 0; i < n; ++i) if (a[i].idx != b[i].idx) return 2;
  return 0;
}
'''


@pytest.fixture(scope="module")
def stlo(tmp_path_factory):
    d = tmp_path_factory.mktemp("stlo")
    src = d / "h.cpp"
    src.write_text(HARNESS)
    so = str(d / "libstlo.so")
    r = subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I",
                        os.path.join(ROOT, "paper_2506_19139_b200", "csrc"), str(src), "-o", so],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    lib = ctypes.CDLL(so)
    lib.stlo_windowed.argtypes = [ctypes.c_long, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p]
    lib.stlo_sort_check.argtypes = [ctypes.c_long, ctypes.c_void_p]
    return lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@pytest.mark.parametrize("levels", [2, 5, 40, 0])
def test_sort_matches_libstdcxx(stlo, levels):
    rng = np.random.default_rng(levels)
    for n in list(range(0, 70)) + [100, 257, 1000, 4099]:
        t = rng.integers(0, levels, n).astype(np.float64) if levels else rng.random(n)
        assert stlo.stlo_sort_check(n, _p(t)) == 0, n


@pytest.mark.parametrize("levels", [2, 7, 0])
def test_windowed_matches_reference(ref, stlo, levels):
    rng = np.random.default_rng(100 + levels)
    for n in list(range(0, 40)) + [64, 200, 513]:
        t = rng.integers(1, levels + 1, n).astype(np.float64) if levels else rng.random(n) + 0.1
        idx = rng.permutation(n).astype(np.int32)
        for w in sorted({0, 1, 2, 3, 4, 5, 8, 16, max(n - 1, 0), n, n + 1}):
            want = ref.windowed_resort(t, idx, w)
            got = np.empty(n, np.int32)
            stlo.stlo_windowed(n, _p(t), _p(idx), w, _p(got))
            np.testing.assert_array_equal(got, want, err_msg=f"n={n} window={w}")
