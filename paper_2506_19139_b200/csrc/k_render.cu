// k_render.cu — the sorted opacity-field rasterizer (K5), FP64 parity path.
//
// Replaces render_depth_map (render.hpp:26-51) and render_pixel (opacity_field.hpp:
// 201-219) over collect_contributions (opacity_field.hpp:39-61). The reference
// tests EVERY Gaussian against every pixel ray and fully sorts the contributions
// by (t*, index). Here:
//   * a conservative per-tile binning: a Gaussian can only reach alpha >= 1/255 on
//     a ray whose closest-approach point p* lies in its E-ellipsoid (clamped scales),
//     whose screen box (dilated by one pixel) bounds every such pixel; lists are
//     ordered by L = |mu - o| - E s_max, a lower bound of t* for every contributing
//     ray (|p* - o| = t*, |p* - mu| <= E s_max);
//   * an exact streaming resort per pixel (a k-buffer in shared memory): before a
//     list entry with bound L is tested, every buffered contribution with t* < L is
//     final and is blended in (t*, index) order; a pixel whose buffer would
//     overflow is re-rendered by a per-pixel full-sort fallback;
//   * contribution tests, alpha, the blend, the median and the exact depth are the
//     reference's FP64 expressions (bit-identical); the opacity at depth
//     (opacity_along_ray, :104-108) is a product over all contributions taken in
//     list order (equal within a few ulps; the reference's order only matters for
//     the last bits of that product).
#include <cub/cub.cuh>

#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"

namespace sofk {

constexpr int kRTile = 16;     // render tile (pixels per side), one CTA per tile
#ifndef SOF_KBUF
#define SOF_KBUF 8
#endif
constexpr int kKBuf = SOF_KBUF;  // k-buffer capacity per pixel
constexpr int kRChunk = 32;    // records staged per step

// ray_through_pixel (camera.hpp:42-48): normalize(R^T ((px - cx)/fx, (py - cy)/fy, 1))
__device__ __forceinline__ void pixel_ray(const Cam& cam, int x, int y, double* d) {
  const double v0 = ((x + 0.5) - cam.cx) / cam.fx;
  const double v1 = ((y + 0.5) - cam.cy) / cam.fy;
  const double v2 = 1.0;
  for (int i = 0; i < 3; ++i) d[i] = cam.R[i] * v0 + cam.R[3 + i] * v1 + cam.R[6 + i] * v2;
  const double sq = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
  if (sq > 0.0) {
    const double nrm = sqrt(sq);
    for (int i = 0; i < 3; ++i) d[i] = d[i] / nrm;
  }
}

struct Contrib {
  double t, alpha;
  int idx;
  bool ok;
};

// collect_contributions' per-Gaussian test (opacity_field.hpp:43-53)
__device__ __forceinline__ Contrib contribution(const Rec& r, const double* d, int idx) {
  Contrib c;
  c.ok = false;
  c.idx = idx;
  if (r.op < kMinAlpha) return c;
  const double x = d[0], y = d[1], z = d[2];
  const double a = r.ic[0] * x * x + r.ic[3] * y * y + r.ic[5] * z * z +
                   2.0 * (r.ic[1] * x * y + r.ic[2] * x * z + r.ic[4] * y * z);
  const double b = 2.0 * (x * r.b[0] + y * r.b[1] + z * r.b[2]);
  const double alpha = r.op * sof_exp(-0.5 * (r.c - b * b / (4.0 * a)));  // peak_value
  if (alpha < kMinAlpha) return c;
  c.t = -b / (2.0 * a);
  if (c.t <= 0.0) return c;
  c.alpha = (kMaxAlpha < alpha) ? kMaxAlpha : alpha;
  c.ok = true;
  return c;
}

// alpha_at (opacity_field.hpp:95-101) of the contribution of record r at parameter t
__device__ __forceinline__ double alpha_at(const Rec& r, const double* d, double t_star, double t) {
  const double x = d[0], y = d[1], z = d[2];
  const double a = r.ic[0] * x * x + r.ic[3] * y * y + r.ic[5] * z * z +
                   2.0 * (r.ic[1] * x * y + r.ic[2] * x * z + r.ic[4] * y * z);
  const double b = 2.0 * (x * r.b[0] + y * r.b[1] + z * r.b[2]);
  const double te = (t < t_star) ? t : t_star;
  if (te <= 0.0) return 0.0;
  const double al = r.op * sof_exp(-0.5 * ((a * te + b) * te + r.c));
  if (al < kMinAlpha) return 0.0;
  return (kMaxAlpha < al) ? kMaxAlpha : al;
}

// Conservative render binning: E-box with clamped scales (inflated by 1e-6), one-pixel
// dilation, key L = |mu - o| - E' s'_max (a lower bound of t* of any contribution).
__global__ void k_render_rect(int64_t n, const GaussStatic* __restrict__ g, Cam cam, int ts,
                              int tiles_x, int tiles_y, int4* rect, uint32_t* cnt, uint64_t* key,
                              int32_t* idx, double* lkey) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i > n) return;
  if (i == n) {
    cnt[n] = 0;
    return;
  }
  const GaussStatic& G = g[i];
  uint32_t count = 0;
  double L = 0.0;
  if (G.E > 0.0) {
    const double E = G.E * (1.0 + 1e-6);
    double s[3], smax = 0.0;
    for (int k = 0; k < 3; ++k) {
      s[k] = (G.scale[k] < kMinScale) ? kMinScale : G.scale[k];
      smax = fmax(smax, s[k]);
    }
    double min_x = 1e300, max_x = -1e300, min_y = 1e300, max_y = -1e300;
    bool crosses = false;
    for (int mask = 0; mask < 8; ++mask) {
      const double l0 = E * s[0] * ((mask & 1) ? 1.0 : -1.0);
      const double l1 = E * s[1] * ((mask & 2) ? 1.0 : -1.0);
      const double l2 = E * s[2] * ((mask & 4) ? 1.0 : -1.0);
      const double p0 = G.pos[0] + (G.rot[0] * l0 + G.rot[1] * l1 + G.rot[2] * l2);
      const double p1 = G.pos[1] + (G.rot[3] * l0 + G.rot[4] * l1 + G.rot[5] * l2);
      const double p2 = G.pos[2] + (G.rot[6] * l0 + G.rot[7] * l1 + G.rot[8] * l2);
      const double vx = to_view_c(cam, 0, p0, p1, p2);
      const double vy = to_view_c(cam, 1, p0, p1, p2);
      const double vz = to_view_c(cam, 2, p0, p1, p2);
      if (vz <= 1e-9) {
        crosses = true;
        break;
      }
      const double px = cam.fx * vx / vz + cam.cx, py = cam.fy * vy / vz + cam.cy;
      min_x = fmin(min_x, px);
      max_x = fmax(max_x, px);
      min_y = fmin(min_y, py);
      max_y = fmax(max_y, py);
    }
    int tx0 = 0, tx1 = tiles_x - 1, ty0 = 0, ty1 = tiles_y - 1;
    bool on = true;
    if (!crosses) {
      min_x -= 1.0;
      min_y -= 1.0;
      max_x += 1.0;
      max_y += 1.0;
      on = !(max_x < 0.0 || min_x >= cam.w || max_y < 0.0 || min_y >= cam.h);
      const double lim = 1e9;
      tx0 = max(0, int(floor(fmax(min_x, -lim))) / ts);
      tx1 = min(tiles_x - 1, int(floor(fmin(max_x, lim))) / ts);
      ty0 = max(0, int(floor(fmax(min_y, -lim))) / ts);
      ty1 = min(tiles_y - 1, int(floor(fmin(max_y, lim))) / ts);
    }
    if (on && tx0 <= tx1 && ty0 <= ty1) {
      count = uint32_t(tx1 - tx0 + 1) * uint32_t(ty1 - ty0 + 1);
      rect[i] = make_int4(tx0, tx1, ty0, ty1);
    }
    const double e0 = G.pos[0] - cam.center[0], e1 = G.pos[1] - cam.center[1],
                 e2 = G.pos[2] - cam.center[2];
    L = sqrt(e0 * e0 + e1 * e1 + e2 * e2) - E * smax;
    L = L - 1e-9 * (1.0 + fabs(L));
  }
  cnt[i] = count;
  key[i] = double_key(L);
  idx[i] = int32_t(i);
  lkey[i] = L;
}

struct RenderOut {
  double* depth;
  double* opacity;
  double* rgb;
  double* tfinal;
};

// Spill area of the pixels whose k-buffer overflows: a pixel of tile t owns the slice
// [256 off[t] + lp len(t), +len(t)) of the pool (len(t) bounds its contributions),
// written in collect mode and sorted by (t*, index) inside k_render_finish.
struct Spill {
  uint64_t* keys;      // double_key(t*)
  int32_t* vals;       // Gaussian index
  double* alpha;       // contribution alpha
  int64_t* begin;      // [slot] slice begin
  int64_t* end;        // [slot] slice end (begin + count)
  int32_t* pixel;      // [slot] pixel id
  double* state;       // [slot][6] T, col[3], med_t, med_T
  int32_t* istate;     // [slot][2] med_idx, found
  int32_t* count;      // number of slots in use
};

__device__ __forceinline__ double exact_depth_at(const Rec& r, const double* d, double med_t,
                                                 double med_T, bool& fell_back) {
  // exact_depth (opacity_field.hpp:157-166)
  const double x = d[0], y = d[1], z = d[2];
  const double a = r.ic[0] * x * x + r.ic[3] * y * y + r.ic[5] * z * z +
                   2.0 * (r.ic[1] * x * y + r.ic[2] * x * z + r.ic[4] * y * z);
  const double b = 2.0 * (x * r.b[0] + y * r.b[1] + z * r.b[2]);
  const double lt = 2.0 * sof_log((med_T - 0.5) / (med_T * r.op));
  const double disc = b * b - 4.0 * a * (r.c + lt);
  fell_back = disc < 0.0;
  return fell_back ? med_t : med_t - sqrt(disc) / (2.0 * a);
}

// One CTA per 16x16 tile; thread = pixel. Pass 1: exact streaming resort (k-buffer)
// + blend + median (+ exact depth); pass 2: opacity at depth. A pixel whose k-buffer
// would overflow switches to collect mode and is finished by k_render_finish.
__global__ void __launch_bounds__(256) k_render(
    Cam cam, int tiles_x, const int64_t* __restrict__ loff, const int32_t* __restrict__ lent,
    const Rec* __restrict__ recs, const double* __restrict__ lkey, const double* __restrict__ dc,
    int exact_depth, RenderOut out, Spill spill, unsigned long long* stats, int tile_base) {
  extern __shared__ __align__(16) unsigned char smem[];
  Rec* srec = reinterpret_cast<Rec*>(smem);
  double* sL = reinterpret_cast<double*>(srec + kRChunk);
  int32_t* sidx = reinterpret_cast<int32_t*>(sL + kRChunk);
  double* bt = reinterpret_cast<double*>(sidx + kRChunk);  // [kKBuf][256]
  double* ba = bt + kKBuf * 256;
  int32_t* bi = reinterpret_cast<int32_t*>(ba + kKBuf * 256);
  const int tile = tile_base + int(blockIdx.x);
  const int tid = threadIdx.x;
  const int px = (tile % tiles_x) * kRTile + (tid % kRTile);
  const int py = (tile / tiles_x) * kRTile + (tid / kRTile);
  const bool valid = px < cam.w && py < cam.h;
  double d[3] = {0.0, 0.0, 1.0};
  if (valid) pixel_ray(cam, px, py, d);
  // pixel-centre coordinates for the screen-space conic cull (Rec::conic): the ray
  // direction through (px + 0.5, py + 0.5) is R^T K^-1 (u, v, 1) up to a positive scale
  const float cu = float(px) + 0.5f, cv = float(py) + 0.5f;
  const float cuu = cu * cu, cvv = cv * cv, cuv = cu * cv;
  const int64_t l0 = loff[tile], l1 = loff[tile + 1];
  const int64_t slice = 256 * (l0 - loff[tile_base]) + int64_t(tid) * (l1 - l0);
  double T = 1.0, col[3] = {0.0, 0.0, 0.0};
  int nbuf = 0;
  bool found = false, collect = false;
  int med_idx = -1;
  double med_t = 0.0, med_T = 1.0;
  int64_t nspill = 0;
  unsigned long long tested = 0, contributing = 0;

  auto blend = [&](double t, double alpha, int idx) {
    for (int k = 0; k < 3; ++k) col[k] = col[k] + dc[3 * idx + k] * alpha * T;
    const double next = T * (1.0 - alpha);
    if (!found && T > 0.5 && next < 0.5) {
      found = true;
      med_idx = idx;
      med_t = t;
      med_T = T;
    }
    T = next;
  };
  auto flush_below = [&](double bound) {
    while (nbuf > 0) {
      int m = 0;
      for (int k = 1; k < nbuf; ++k) {
        const double tk = bt[k * 256 + tid], tm = bt[m * 256 + tid];
        if (tk < tm || (tk == tm && bi[k * 256 + tid] < bi[m * 256 + tid])) m = k;
      }
      const double tm = bt[m * 256 + tid];
      if (!(tm < bound)) return;
      blend(tm, ba[m * 256 + tid], bi[m * 256 + tid]);
      --nbuf;
      bt[m * 256 + tid] = bt[nbuf * 256 + tid];
      ba[m * 256 + tid] = ba[nbuf * 256 + tid];
      bi[m * 256 + tid] = bi[nbuf * 256 + tid];
    }
  };
  auto spill_one = [&](double t, double alpha, int idx) {
    spill.keys[slice + nspill] = double_key(t);
    spill.vals[slice + nspill] = idx;
    spill.alpha[slice + nspill] = alpha;
    ++nspill;
  };

  for (int64_t base = l0; base < l1; base += kRChunk) {
    if (!__syncthreads_or(valid)) break;
    const int cnt = int(min(int64_t(kRChunk), l1 - base));
    for (int k = tid; k < cnt * kRecV2; k += blockDim.x) {
      const int r = k / kRecV2, q = k % kRecV2;
      const int32_t g = lent[base + r];
      reinterpret_cast<double2*>(&srec[r])[q] = __ldg(reinterpret_cast<const double2*>(recs + g) + q);
      if (q == 0) {
        sidx[r] = g;
        sL[r] = lkey[g];
      }
    }
    __syncthreads();
    if (valid) {
      for (int k = 0; k < cnt; ++k) {
        if (!collect) flush_below(sL[k]);
        ++tested;
        if (conic_culls(srec[k], cu, cv, cuu, cvv, cuv)) continue;  // cannot reach 1/255
        const Contrib c = contribution(srec[k], d, sidx[k]);
        if (!c.ok) continue;
        ++contributing;
        if (collect) {
          spill_one(c.t, c.alpha, c.idx);
        } else if (nbuf == kKBuf) {
          // the buffered entries are not final yet: hand them and the rest of the
          // list to the sort-based finish (blend state so far is kept)
          collect = true;
          for (int q = 0; q < nbuf; ++q) spill_one(bt[q * 256 + tid], ba[q * 256 + tid], bi[q * 256 + tid]);
          nbuf = 0;
          spill_one(c.t, c.alpha, c.idx);
        } else {
          bt[nbuf * 256 + tid] = c.t;
          ba[nbuf * 256 + tid] = c.alpha;
          bi[nbuf * 256 + tid] = c.idx;
          ++nbuf;
        }
      }
    }
  }
  if (valid && !collect) flush_below(INFINITY);
  double depth = NAN;
  bool fell_back = false;
  if (valid && !collect && found) {
    depth = med_t;
    if (exact_depth) depth = exact_depth_at(recs[med_idx], d, med_t, med_T, fell_back);
  }
  if (valid) {
    const int64_t p = int64_t(py) * cam.w + px;
    if (collect) {
      const int s = atomicAdd(spill.count, 1);
      spill.begin[s] = slice;
      spill.end[s] = slice + nspill;
      spill.pixel[s] = int32_t(p);
      double* st = spill.state + 6 * s;
      st[0] = T;
      st[1] = col[0];
      st[2] = col[1];
      st[3] = col[2];
      st[4] = med_t;
      st[5] = med_T;
      spill.istate[2 * s] = med_idx;
      spill.istate[2 * s + 1] = found;
    } else {
      out.depth[p] = depth;  // opacity at depth: k_render_opacity
      for (int k = 0; k < 3; ++k) out.rgb[3 * p + k] = col[k];
      out.tfinal[p] = T;
    }
  }
  unsigned long long s0 = tested, s1 = contributing, s3 = fell_back ? 1 : 0;
  for (int s = 16; s > 0; s >>= 1) {
    s0 += __shfl_down_sync(0xffffffffu, s0, s);
    s1 += __shfl_down_sync(0xffffffffu, s1, s);
    s3 += __shfl_down_sync(0xffffffffu, s3, s);
  }
  if ((tid & 31) == 0) {
    if (s0) atomicAdd(stats, s0);
    if (s1) atomicAdd(stats + 1, s1);
    if (s3) atomicAdd(stats + 3, s3);
  }
}

constexpr int kFChunk = 256;  // slice entries a warp sorts at once in shared memory
constexpr int kFWarps = 8;    // warps (spilled pixels) per finish CTA

__device__ __forceinline__ bool kv_less(uint64_t ka, int32_t va, uint64_t kb, int32_t vb) {
  return ka < kb || (ka == kb && va < vb);
}

// Warp-wide bitonic sort of m (a power of two, 32..kFChunk) (key, index) pairs (with
// their alpha) in shared memory, ascending.
__device__ __forceinline__ void warp_bitonic(uint64_t* k, int32_t* v, double* a, int m, int lane) {
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int i = lane; i < (m >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const uint64_t ka = k[lo], kb = k[hi];
        const int32_t va = v[lo], vb = v[hi];
        if (kv_less(kb, vb, ka, va) == up) {
          k[lo] = kb;
          k[hi] = ka;
          v[lo] = vb;
          v[hi] = va;
          const double aa = a[lo];
          a[lo] = a[hi];
          a[hi] = aa;
        }
      }
    }
  }
  __syncwarp();
}

// Resumes the blend of a collect-mode pixel (one warp per pixel) over its spill slice
// in the reference's (t*, index) order (opacity_field.hpp:56-59): the slice's
// (double_key(t*), index, alpha) entries are sorted in shared memory (slices longer
// than kFChunk: sorted chunks merged by rank into keys2/vals2/alpha2) and blended
// serially through shuffles; t* is recovered from its key.
#ifndef SOF_FIN_MINB
#define SOF_FIN_MINB 3
#endif
__global__ void __launch_bounds__(kFWarps * 32, SOF_FIN_MINB) k_render_finish(
    Cam cam, const Rec* __restrict__ recs, const double* __restrict__ dc, int exact_depth, Spill spill,
    uint64_t* __restrict__ gk2, int32_t* __restrict__ gv2, double* __restrict__ ga2, RenderOut out,
    unsigned long long* stats) {
  __shared__ uint64_t sk[kFWarps][kFChunk];
  __shared__ double sa[kFWarps][kFChunk];
  __shared__ int32_t sv[kFWarps][kFChunk];
  constexpr unsigned kAll = 0xffffffffu;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * kFWarps + w;
  if (s >= *spill.count) return;  // warp-uniform
  const int64_t p = spill.pixel[s];
  const int px = int(p % cam.w), py = int(p / cam.w);
  const double* st = spill.state + 6 * s;
  double T = st[0], col[3] = {st[1], st[2], st[3]}, med_t = st[4], med_T = st[5];
  int med_idx = spill.istate[2 * s];
  bool found = spill.istate[2 * s + 1];
  const int64_t b = spill.begin[s], n = spill.end[s] - b;
  uint64_t* K = sk[w];
  int32_t* V = sv[w];
  double* A = sa[w];
  for (int64_t c0 = 0; c0 < n; c0 += kFChunk) {
    const int cn = int(min(int64_t(kFChunk), n - c0));
    int m = 32;
    while (m < cn) m <<= 1;
    for (int i = lane; i < m; i += 32) {
      K[i] = i < cn ? spill.keys[b + c0 + i] : ~0ull;
      V[i] = i < cn ? spill.vals[b + c0 + i] : 0x7fffffff;
      A[i] = i < cn ? spill.alpha[b + c0 + i] : 0.0;
    }
    warp_bitonic(K, V, A, m, lane);
    if (n > kFChunk) {
      for (int i = lane; i < cn; i += 32) {
        spill.keys[b + c0 + i] = K[i];
        spill.vals[b + c0 + i] = V[i];
        spill.alpha[b + c0 + i] = A[i];
      }
      __syncwarp();
    }
  }
  const uint64_t* SK = K;
  const int32_t* SV = V;
  const double* SA = A;
  if (n > kFChunk) {
    // final position = position in own chunk + entries below it in every other chunk
    for (int64_t i = lane; i < n; i += 32) {
      const uint64_t ki = spill.keys[b + i];
      const int32_t vi = spill.vals[b + i];
      const int64_t own = i / kFChunk;
      int64_t rank = i - own * kFChunk;
      for (int64_t c0 = 0; c0 < n; c0 += kFChunk) {
        if (c0 == own * kFChunk) continue;
        int lo = 0, hi = int(min(int64_t(kFChunk), n - c0));
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (kv_less(spill.keys[b + c0 + mid], spill.vals[b + c0 + mid], ki, vi)) lo = mid + 1;
          else hi = mid;
        }
        rank += lo;
      }
      gk2[b + rank] = ki;
      gv2[b + rank] = vi;
      ga2[b + rank] = spill.alpha[b + i];
    }
    __syncwarp();
    SK = gk2 + b;
    SV = gv2 + b;
    SA = ga2 + b;
  }
  for (int64_t c0 = 0; c0 < n; c0 += 32) {
    const int64_t i = c0 + lane;
    double t = 0.0, al = 0.0, dq[3] = {0.0, 0.0, 0.0};
    int idx = 0;
    if (i < n) {
      idx = SV[i];
      t = key_double(SK[i]);
      al = SA[i];
      for (int k = 0; k < 3; ++k) dq[k] = dc[3 * idx + k];
    }
    const int cnt = int(min(int64_t(32), n - c0));
    for (int q = 0; q < cnt; ++q) {
      const double tq = __shfl_sync(kAll, t, q), aq = __shfl_sync(kAll, al, q);
      const int iq = __shfl_sync(kAll, idx, q);
      for (int k = 0; k < 3; ++k) col[k] = col[k] + __shfl_sync(kAll, dq[k], q) * aq * T;
      const double next = T * (1.0 - aq);
      if (!found && T > 0.5 && next < 0.5) {
        found = true;
        med_idx = iq;
        med_t = tq;
        med_T = T;
      }
      T = next;
    }
  }
  double d[3];
  pixel_ray(cam, px, py, d);
  double depth = NAN;
  if (found) {
    depth = med_t;
    if (exact_depth) {
      bool fb = false;
      depth = exact_depth_at(recs[med_idx], d, med_t, med_T, fb);
      if (fb && lane == 0) atomicAdd(stats + 3, 1ull);
    }
  }
  if (lane == 0) {
    out.depth[p] = depth;
    for (int k = 0; k < 3; ++k) out.rgb[3 * p + k] = col[k];
    out.tfinal[p] = T;
  }
}

// Pass 2 for every pixel once its depth is known (render_pixel's O_N(depth),
// opacity_field.hpp:201-219): one CTA per tile multiplies 1 - alpha_at(depth) over the
// tile's contributions in list order, records staged once per CTA in shared memory.
__global__ void __launch_bounds__(256) k_render_opacity(Cam cam, int tiles_x,
                                                        const int64_t* __restrict__ loff,
                                                        const int32_t* __restrict__ lent,
                                                        const Rec* __restrict__ recs, RenderOut out) {
  __shared__ __align__(16) Rec srec[kRChunk];
  __shared__ int32_t sidx[kRChunk];
  const int tile = int(blockIdx.x), tid = threadIdx.x;
  const int px = (tile % tiles_x) * kRTile + (tid % kRTile);
  const int py = (tile / tiles_x) * kRTile + (tid / kRTile);
  const bool valid = px < cam.w && py < cam.h;
  const int64_t p = int64_t(py) * cam.w + px;
  const double depth = valid ? out.depth[p] : NAN;
  const bool need = !isnan(depth);
  double d[3] = {0.0, 0.0, 1.0};
  if (need) pixel_ray(cam, px, py, d);
  const float cu = float(px) + 0.5f, cv = float(py) + 0.5f;
  const float cuu = cu * cu, cvv = cv * cv, cuv = cu * cv;
  double T2 = 1.0;
  for (int64_t base = loff[tile], l1 = loff[tile + 1]; base < l1; base += kRChunk) {
    if (!__syncthreads_or(need)) break;
    const int cnt = int(min(int64_t(kRChunk), l1 - base));
    for (int k = tid; k < cnt * kRecV2; k += blockDim.x) {
      const int r = k / kRecV2, q = k % kRecV2;
      const int32_t g = lent[base + r];
      reinterpret_cast<double2*>(&srec[r])[q] = __ldg(reinterpret_cast<const double2*>(recs + g) + q);
      if (q == 0) sidx[r] = g;
    }
    __syncthreads();
    if (need) {
      for (int k = 0; k < cnt; ++k) {
        if (conic_culls(srec[k], cu, cv, cuu, cvv, cuv)) continue;
        const Contrib c = contribution(srec[k], d, sidx[k]);
        if (!c.ok) continue;
        T2 *= 1.0 - alpha_at(srec[k], d, c.t, depth);
      }
    }
  }
  if (valid) out.opacity[p] = need ? 1.0 - T2 : 0.0;
}

// ---- normals (render.hpp:58-107) ---------------------------------------------------------------

// ray_through_pixel(cam, x + 0.5, y + 0.5).origin + depth * direction (render.hpp:64-67)
__device__ __forceinline__ void backproject(const Cam& cam, int x, int y, double depth, double* p) {
  double d[3];
  pixel_ray(cam, x, y, d);
  for (int i = 0; i < 3; ++i) p[i] = cam.center[i] + depth * d[i];
}

// normal_from_depth (render.hpp:60-88): forward differences of the back-projected depth
// map, cross product, camera-facing. One thread per pixel; the last row and column and
// pixels with a no-surface neighbour stay invalid with a zero normal.
__global__ void k_normal_from_depth(Cam cam, const double* __restrict__ depth, double* normal,
                                    uint8_t* valid) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= int64_t(cam.w) * cam.h) return;
  const int x = int(p % cam.w), y = int(p / cam.w);
  double n[3] = {0.0, 0.0, 0.0};
  uint8_t ok = 0;
  if (x + 1 < cam.w && y + 1 < cam.h) {
    const double d00 = depth[p], d10 = depth[p + 1], d01 = depth[p + cam.w];
    if (!isnan(d00) && !isnan(d10) && !isnan(d01)) {  // is_no_surface (core.hpp:26)
      double p0[3], p1[3], p2[3], dx[3], dy[3];
      backproject(cam, x, y, d00, p0);
      backproject(cam, x + 1, y, d10, p1);
      backproject(cam, x, y + 1, d01, p2);
      for (int i = 0; i < 3; ++i) {
        dx[i] = p1[i] - p0[i];
        dy[i] = p2[i] - p0[i];
      }
      double c[3] = {dx[1] * dy[2] - dx[2] * dy[1], dx[2] * dy[0] - dx[0] * dy[2],
                     dx[0] * dy[1] - dx[1] * dy[0]};
      const double len = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
      if (!(len < 1e-14)) {
        for (int i = 0; i < 3; ++i) c[i] = c[i] / len;
        double v[3] = {p0[0] - cam.center[0], p0[1] - cam.center[1], p0[2] - cam.center[2]};
        const double vz = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
        if (vz > 0.0) {
          const double vn = sqrt(vz);
          for (int i = 0; i < 3; ++i) v[i] = v[i] / vn;
        }
        if (c[0] * v[0] + c[1] * v[1] + c[2] * v[2] > 0.0)
          for (int i = 0; i < 3; ++i) c[i] = -c[i];
        for (int i = 0; i < 3; ++i) n[i] = c[i];
        ok = 1;
      }
    }
  }
  for (int i = 0; i < 3; ++i) normal[3 * p + i] = n[i];
  valid[p] = ok;
}

// gaussian_normal (render.hpp:93-107) for m (Gaussian, ray, t) queries: normalised
// inv_cov (x - mu) with inv_cov = R diag(1 / max(s, 1e-8)^2) R^T, the shortest-scale
// axis when it vanishes, flipped to face the camera.
__global__ void k_gaussian_normal(int64_t m, const int32_t* __restrict__ gidx,
                                  const double* __restrict__ pos, const double* __restrict__ scale,
                                  const double* __restrict__ rot, const double* __restrict__ ro,
                                  const double* __restrict__ rd, const double* __restrict__ tq,
                                  double* out) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= m) return;
  const int64_t g = gidx[k];
  double r[9];
  quat_to_rot(rot[4 * g], rot[4 * g + 1], rot[4 * g + 2], rot[4 * g + 3], r);
  double inv[3];
  for (int i = 0; i < 3; ++i) {
    const double sc = scale[3 * g + i];
    const double s = (sc < 1e-8) ? 1e-8 : sc;  // cwiseMax(kMinScale)
    inv[i] = 1.0 / (s * s);
  }
  double m1[9], ic[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m1[3 * i + j] = r[3 * i + j] * inv[j];  // r * diag
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      ic[3 * i + j] = m1[3 * i] * r[3 * j] + m1[3 * i + 1] * r[3 * j + 1] + m1[3 * i + 2] * r[3 * j + 2];
  const double t = tq[k];
  double diff[3];
  for (int i = 0; i < 3; ++i) diff[i] = (ro[3 * k + i] + t * rd[3 * k + i]) - pos[3 * g + i];
  double n[3];
  for (int i = 0; i < 3; ++i) n[i] = ic[3 * i] * diff[0] + ic[3 * i + 1] * diff[1] + ic[3 * i + 2] * diff[2];
  if (sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]) < 1e-12) {
    int axis = 0;  // minCoeff(&axis): first minimum of the raw scales
    double mn = scale[3 * g];
    for (int i = 1; i < 3; ++i)
      if (scale[3 * g + i] < mn) {
        mn = scale[3 * g + i];
        axis = i;
      }
    for (int i = 0; i < 3; ++i) n[i] = r[3 * i + axis];
  }
  const double z = n[0] * n[0] + n[1] * n[1] + n[2] * n[2];
  if (z > 0.0) {
    const double nn = sqrt(z);
    for (int i = 0; i < 3; ++i) n[i] = n[i] / nn;
  }
  if (n[0] * rd[3 * k] + n[1] * rd[3 * k + 1] + n[2] * rd[3 * k + 2] > 0.0)
    for (int i = 0; i < 3; ++i) n[i] = -n[i];
  for (int i = 0; i < 3; ++i) out[3 * k + i] = n[i];
}

}  // namespace sofk

using namespace sofk;

extern "C" int sof_render_view(sof_ctx* c, int view, int depth_mode, int tile_size, double* depth,
                               double* opacity, double* rgb, double* t_final, uint64_t* stats) {
  if (!c) return SOF_E_INVALID;
  try {
    SOF_CUDA(cudaSetDevice(c->device));
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    (void)tile_size;  // the reference render has no tiles; the render tile is fixed at 16
    const Cam& cam = c->cams[view];
    const int ts = kRTile;
    const int tiles_x = (cam.w + ts - 1) / ts, tiles_y = (cam.h + ts - 1) / ts;
    const int64_t T = int64_t(tiles_x) * tiles_y;
    const int64_t n = c->n, P = int64_t(cam.w) * cam.h;
    const Rec* rec = view_records(c, view);
    c->rect.ensure(std::max<int64_t>(n, 1));
    c->gcount.ensure(n + 1);
    c->zkey_in.ensure(std::max<int64_t>(n, 1));
    c->zkey_out.ensure(std::max<int64_t>(n, 1));
    c->gidx_in.ensure(std::max<int64_t>(n, 1));
    c->gidx_out.ensure(std::max<int64_t>(n, 1));
    c->goff.ensure(n + 1);
    c->r_lkey.ensure(std::max<int64_t>(n, 1));  // L keys (double) per Gaussian
    k_render_rect<<<grid_for(n + 1, 128), 128, 0, c->stream>>>(
        n, c->gstat.p, cam, ts, tiles_x, tiles_y, c->rect.p, c->gcount.p, c->zkey_in.p, c->gidx_in.p,
        c->r_lkey.p);
    SOF_LAUNCHED(c);
    if (n > 0) {
      bin_by_key(c, view, ts, tiles_x, tiles_y, c->rbind, false);
    } else {
      c->rbind.off.ensure(T + 1);
      SOF_CUDA(cudaMemsetAsync(c->rbind.off.p, 0, sizeof(int64_t) * (T + 1), c->stream));
      c->rbind.ent.ensure(1);
      c->rbind.entries = 0;
    }
    c->r_out.ensure(6 * P);
    RenderOut out{c->r_out.p, c->r_out.p + P, c->r_out.p + 2 * P, c->r_out.p + 5 * P};
    // Spill pool: a pixel of tile t may need len(t) slots, so a band of tiles [t0, t1)
    // needs 256 (off[t1] - off[t0]). Tiles are rendered in bands whose pool fits both
    // a 24 GB memory cap (and 32-bit slot counts).
    std::vector<int64_t> off(T + 1, 0);
    if (n > 0)
      SOF_CUDA(cudaMemcpyAsync(off.data(), c->rbind.off.p, sizeof(int64_t) * (T + 1),
                               cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t cap = std::min<int64_t>((int64_t(1) << 31) - 1, (int64_t(24) << 30) / 40);
    RenderScratch& rs = c->rs;
    c->r_stats.ensure(4);
    SOF_CUDA(cudaMemsetAsync(c->r_stats.p, 0, 4 * sizeof(unsigned long long), c->stream));
    const size_t smem = kRChunk * (sizeof(Rec) + sizeof(double) + sizeof(int32_t)) +
                        size_t(kKBuf) * 256 * (2 * sizeof(double) + sizeof(int32_t));
    if (!c->render_attr_set) {  // a per-device function attribute: set once per context
      SOF_CUDA(cudaFuncSetAttribute(k_render, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      c->render_attr_set = true;
    }
    int64_t nover_total = 0;
    for (int64_t t0 = 0; t0 < T;) {
      int64_t t1 = t0 + 1;  // always at least one tile
      while (t1 < T && 256 * (off[t1 + 1] - off[t0]) <= cap) ++t1;
      const int64_t pool = std::max<int64_t>(256 * (off[t1] - off[t0]), 1);
      if (pool > cap) throw InvalidArg("a single render tile's list exceeds the spill pool");
      const int64_t bpx = (t1 - t0) * 256;
      rs.keys.ensure(pool);
      rs.keys2.ensure(pool);
      rs.vals.ensure(pool);
      rs.vals2.ensure(pool);
      rs.alpha.ensure(pool);
      rs.alpha2.ensure(pool);
      rs.begin.ensure(bpx);
      rs.end.ensure(bpx);
      rs.pixel.ensure(bpx);
      rs.state.ensure(6 * bpx);
      rs.istate.ensure(2 * bpx);
      rs.count.ensure(1);
      SOF_CUDA(cudaMemsetAsync(rs.count.p, 0, sizeof(int32_t), c->stream));
      Spill spill{rs.keys.p, rs.vals.p, rs.alpha.p, rs.begin.p, rs.end.p, rs.pixel.p, rs.state.p, rs.istate.p, rs.count.p};
      k_render<<<unsigned(t1 - t0), 256, smem, c->stream>>>(
          cam, tiles_x, c->rbind.off.p, c->rbind.ent.p, rec, c->r_lkey.p, c->dc.p,
          depth_mode == SOF_DEPTH_EXACT, out, spill, c->r_stats.p, int(t0));
      SOF_LAUNCHED(c);
      const int32_t nover = read_scalar(c, rs.count.p);
      if (nover > 0) {
        k_render_finish<<<unsigned((nover + kFWarps - 1) / kFWarps), kFWarps * 32, 0, c->stream>>>(
            cam, rec, c->dc.p, depth_mode == SOF_DEPTH_EXACT, spill, rs.keys2.p, rs.vals2.p, rs.alpha2.p, out,
            c->r_stats.p);
        SOF_LAUNCHED(c);
      }
      nover_total += nover;
      t0 = t1;
    }
    if (T > 0) {
      k_render_opacity<<<unsigned(T), 256, 0, c->stream>>>(cam, tiles_x, c->rbind.off.p, c->rbind.ent.p, rec,
                                                            out);
      SOF_LAUNCHED(c);
    }
    c->r_view = view;
    const int64_t nover = nover_total;
    if (depth) SOF_CUDA(cudaMemcpyAsync(depth, out.depth, sizeof(double) * P, cudaMemcpyDeviceToHost, c->stream));
    if (opacity)
      SOF_CUDA(cudaMemcpyAsync(opacity, out.opacity, sizeof(double) * P, cudaMemcpyDeviceToHost, c->stream));
    if (rgb) SOF_CUDA(cudaMemcpyAsync(rgb, out.rgb, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, c->stream));
    if (t_final)
      SOF_CUDA(cudaMemcpyAsync(t_final, out.tfinal, sizeof(double) * P, cudaMemcpyDeviceToHost, c->stream));
    unsigned long long h[4];
    SOF_CUDA(cudaMemcpyAsync(h, c->r_stats.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
    if (stats) {
      stats[0] = h[0];
      stats[1] = h[1];
      stats[2] = uint64_t(nover);
      stats[3] = h[3];
    }
    return SOF_OK;
  } catch (const InvalidArg& e) {
    c->err = e.what();
    return SOF_E_INVALID;
  } catch (const StateError& e) {
    c->err = e.what();
    return SOF_E_STATE;
  } catch (const OomError& e) {
    c->err = e.what();
    return SOF_E_OOM;
  } catch (const std::exception& e) {
    c->err = e.what();
    return SOF_E_CUDA;
  }
}

extern "C" int sof_render_normals(sof_ctx* c, int view, double* normal, uint8_t* valid) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    if (c->r_view != view) throw StateError("no render of this view on the device: call sof_render_view first");
    const Cam& cam = c->cams[view];
    const int64_t P = int64_t(cam.w) * cam.h;
    c->r_normal.ensure(std::max<int64_t>(3 * P, 1));
    c->r_valid.ensure(std::max<int64_t>(P, 1));
    if (P > 0) {
      k_normal_from_depth<<<grid_for(P, 256), 256, 0, c->stream>>>(cam, c->r_out.p, c->r_normal.p, c->r_valid.p);
      SOF_LAUNCHED(c);
    }
    if (normal && P) SOF_CUDA(cudaMemcpyAsync(normal, c->r_normal.p, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, c->stream));
    if (valid && P) SOF_CUDA(cudaMemcpyAsync(valid, c->r_valid.p, P, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int sof_normal_from_depth(sof_ctx* c, int view, const double* depth, double* normal, uint8_t* valid) {
  if (!c || !depth) return SOF_E_INVALID;
  return guard(c, [&] {
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    const Cam& cam = c->cams[view];
    const int64_t P = int64_t(cam.w) * cam.h;
    c->r_depth_in.ensure(std::max<int64_t>(P, 1));
    c->r_normal.ensure(std::max<int64_t>(3 * P, 1));
    c->r_valid.ensure(std::max<int64_t>(P, 1));
    if (P > 0) {
      SOF_CUDA(cudaMemcpyAsync(c->r_depth_in.p, depth, sizeof(double) * P, cudaMemcpyHostToDevice, c->stream));
      k_normal_from_depth<<<grid_for(P, 256), 256, 0, c->stream>>>(cam, c->r_depth_in.p, c->r_normal.p,
                                                                   c->r_valid.p);
      SOF_LAUNCHED(c);
      if (normal) SOF_CUDA(cudaMemcpyAsync(normal, c->r_normal.p, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, c->stream));
      if (valid) SOF_CUDA(cudaMemcpyAsync(valid, c->r_valid.p, P, cudaMemcpyDeviceToHost, c->stream));
    }
    SOF_CUDA(cudaStreamSynchronize(c->stream));
  });
}

extern "C" int sof_gaussian_normals(sof_ctx* c, int64_t m, const int32_t* gidx, const double* origin,
                                    const double* dir, const double* t, double* out) {
  if (!c || m < 0 || (m > 0 && (!gidx || !origin || !dir || !t || !out))) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    if (m == 0) return;
    for (int64_t k = 0; k < m; ++k)
      if (gidx[k] < 0 || gidx[k] >= c->n) throw InvalidArg("gaussian index out of range");
    DBuf<char>& b = c->r_query;
    const size_t off_o = 0, off_d = 24 * m, off_t = 48 * m, off_i = 56 * m, off_out = 64 * m;
    b.ensure(int64_t(off_out + 24 * m));
    SOF_CUDA(cudaMemcpyAsync(b.p + off_o, origin, 24 * m, cudaMemcpyHostToDevice, c->stream));
    SOF_CUDA(cudaMemcpyAsync(b.p + off_d, dir, 24 * m, cudaMemcpyHostToDevice, c->stream));
    SOF_CUDA(cudaMemcpyAsync(b.p + off_t, t, 8 * m, cudaMemcpyHostToDevice, c->stream));
    SOF_CUDA(cudaMemcpyAsync(b.p + off_i, gidx, 4 * m, cudaMemcpyHostToDevice, c->stream));
    double* dout = reinterpret_cast<double*>(b.p + off_out);
    k_gaussian_normal<<<grid_for(m, 256), 256, 0, c->stream>>>(
        m, reinterpret_cast<const int32_t*>(b.p + off_i), c->pos.p, c->scale.p, c->rot.p,
        reinterpret_cast<const double*>(b.p + off_o), reinterpret_cast<const double*>(b.p + off_d),
        reinterpret_cast<const double*>(b.p + off_t), dout);
    SOF_LAUNCHED(c);
    SOF_CUDA(cudaMemcpyAsync(out, dout, 24 * m, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
  });
}
