// stl_order.cuh — the reference's element ORDER for windowed_resort (opacity_field.hpp:66-91),
// on the device, one thread per list.
//
// windowed_resort orders with std::sort (window 0 or >= n) and with a K-slot
// std::push_heap / std::pop_heap window; both compare t* only, so contributions with
// equal t* leave in whatever order the libstdc++ algorithms happen to produce. To be
// bit-identical on ties this header restates those algorithms step for step (introsort:
// 16-element threshold, depth limit 2 floor(log2 n), median-of-three pivot moved to the
// front, unguarded Hoare partition, heap-sort fallback, final guarded+unguarded insertion
// sort; heaps: __adjust_heap's hole descent and __push_heap's sift-up). The recursion of
// __introsort_loop is an explicit stack: its sub-ranges are disjoint, so the visiting order
// does not change the result. Element type and comparator are template parameters; the
// functions are __host__ __device__ so tests/test_stl_order_cpu.py can check them against
// the host's own std::sort / std::push_heap / std::pop_heap.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#ifndef __host__
#define __host__
#define __device__
#define __forceinline__ inline
#endif
#endif

namespace stlo {

template <typename T>
__host__ __device__ __forceinline__ void swap_at(T* a, int64_t i, int64_t j) {
  const T t = a[i];
  a[i] = a[j];
  a[j] = t;
}

// std::__push_heap
template <typename T, typename Less>
__host__ __device__ void push_heap_hole(T* a, int64_t hole, int64_t top, const T& value, Less comp) {
  int64_t parent = (hole - 1) / 2;
  while (hole > top && comp(a[parent], value)) {
    a[hole] = a[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  a[hole] = value;
}

// std::__adjust_heap
template <typename T, typename Less>
__host__ __device__ void adjust_heap(T* a, int64_t hole, int64_t len, const T& value, Less comp) {
  const int64_t top = hole;
  int64_t child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (comp(a[child], a[child - 1])) child--;
    a[hole] = a[child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    a[hole] = a[child - 1];
    hole = child - 1;
  }
  push_heap_hole(a, hole, top, value, comp);
}

// std::push_heap(a, a + len): the new element is a[len - 1]
template <typename T, typename Less>
__host__ __device__ __forceinline__ void push_heap(T* a, int64_t len, Less comp) {
  const T v = a[len - 1];
  push_heap_hole(a, len - 1, 0, v, comp);
}

// std::pop_heap(a, a + len): the top moves to a[len - 1]
template <typename T, typename Less>
__host__ __device__ __forceinline__ void pop_heap(T* a, int64_t len, Less comp) {
  if (len > 1) {
    const T v = a[len - 1];
    a[len - 1] = a[0];
    adjust_heap(a, 0, len - 1, v, comp);
  }
}

// std::__make_heap
template <typename T, typename Less>
__host__ __device__ void make_heap(T* a, int64_t len, Less comp) {
  if (len < 2) return;
  for (int64_t parent = (len - 2) / 2;; --parent) {
    const T v = a[parent];
    adjust_heap(a, parent, len, v, comp);
    if (parent == 0) return;
  }
}

// std::__sort_heap
template <typename T, typename Less>
__host__ __device__ void sort_heap(T* a, int64_t len, Less comp) {
  while (len > 1) {
    --len;
    const T v = a[len];
    a[len] = a[0];
    adjust_heap(a, 0, len, v, comp);
  }
}

// std::__move_median_to_first
template <typename T, typename Less>
__host__ __device__ __forceinline__ void median_to_first(T* a, int64_t r, int64_t x, int64_t y, int64_t z, Less comp) {
  if (comp(a[x], a[y])) {
    if (comp(a[y], a[z])) swap_at(a, r, y);
    else if (comp(a[x], a[z])) swap_at(a, r, z);
    else swap_at(a, r, x);
  } else if (comp(a[x], a[z])) {
    swap_at(a, r, x);
  } else if (comp(a[y], a[z])) {
    swap_at(a, r, z);
  } else {
    swap_at(a, r, y);
  }
}

// std::__unguarded_partition_pivot over [f, l): returns the cut
template <typename T, typename Less>
__host__ __device__ int64_t partition_pivot(T* a, int64_t f, int64_t l, Less comp) {
  const int64_t mid = f + (l - f) / 2;
  median_to_first(a, f, f + 1, mid, l - 1, comp);
  int64_t i = f + 1, j = l;
  while (true) {
    while (comp(a[i], a[f])) ++i;
    --j;
    while (comp(a[f], a[j])) --j;
    if (!(i < j)) return i;
    swap_at(a, i, j);
    ++i;
  }
}

// std::__unguarded_linear_insert
template <typename T, typename Less>
__host__ __device__ __forceinline__ void linear_insert(T* a, int64_t last, Less comp) {
  const T v = a[last];
  int64_t next = last - 1;
  while (comp(v, a[next])) {
    a[last] = a[next];
    last = next;
    --next;
  }
  a[last] = v;
}

// std::__insertion_sort over [f, l)
template <typename T, typename Less>
__host__ __device__ void insertion_sort(T* a, int64_t f, int64_t l, Less comp) {
  if (f == l) return;
  for (int64_t i = f + 1; i != l; ++i) {
    if (comp(a[i], a[f])) {
      const T v = a[i];
      for (int64_t k = i; k > f; --k) a[k] = a[k - 1];  // move_backward
      a[f] = v;
    } else {
      linear_insert(a, i, comp);
    }
  }
}

__host__ __device__ __forceinline__ int floor_log2(int64_t n) {
  int r = 0;
  while (n > 1) {
    n >>= 1;
    ++r;
  }
  return r;
}

constexpr int64_t kThreshold = 16;  // std::_S_threshold

// std::sort(a, a + n, comp)
template <typename T, typename Less>
__host__ __device__ void sort(T* a, int64_t n, Less comp) {
  if (n < 2) return;
  struct Range {
    int64_t f, l;
    int depth;
  };
  Range stack[66];  // depths strictly decrease up the stack: <= 2 log2(n) + 1 <= 65 frames
  int sp = 0;
  stack[sp++] = {0, n, 2 * floor_log2(n)};
  while (sp > 0) {
    Range r = stack[--sp];
    while (r.l - r.f > kThreshold) {
      if (r.depth == 0) {  // std::__partial_sort(f, l, l): make_heap + sort_heap
        make_heap(a + r.f, r.l - r.f, comp);
        sort_heap(a + r.f, r.l - r.f, comp);
        break;
      }
      --r.depth;
      const int64_t cut = partition_pivot(a, r.f, r.l, comp);
      stack[sp++] = {cut, r.l, r.depth};  // __introsort_loop(cut, last)
      r.l = cut;
    }
  }
  // std::__final_insertion_sort
  if (n > kThreshold) {
    insertion_sort(a, 0, kThreshold, comp);
    for (int64_t i = kThreshold; i != n; ++i) linear_insert(a, i, comp);
  } else {
    insertion_sort(a, 0, n, comp);
  }
}

// windowed_resort (opacity_field.hpp:66-91) with `less_t` = (l.t* < r.t*): in[0, n) in
// arrival order; the result goes to out[0, n). in[] is clobbered (the heap lives in its
// consumed prefix: after reading element i the window holds at most min(i + 1, K + 1)).
template <typename T, typename LessT>
__host__ __device__ void windowed_resort(T* in, T* out, int64_t n, int64_t window, LessT less_t) {
  if (window == 0 || window >= n) {
    sort(in, n, less_t);
    for (int64_t i = 0; i < n; ++i) out[i] = in[i];
    return;
  }
  auto greater = [&](const T& l, const T& r) { return less_t(r, l); };  // cmp: l.t* > r.t*
  int64_t h = 0, o = 0;
  for (int64_t i = 0; i < n; ++i) {
    const T v = in[i];
    in[h++] = v;  // heap.push_back + std::push_heap
    push_heap(in, h, greater);
    if (h > window) {  // std::pop_heap + out.push_back(heap.back()) + heap.pop_back()
      pop_heap(in, h, greater);
      out[o++] = in[--h];
    }
  }
  while (h > 0) {
    pop_heap(in, h, greater);
    out[o++] = in[--h];
  }
}

}  // namespace stlo
