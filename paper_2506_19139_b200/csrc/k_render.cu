// k_render.cu — the sorted opacity-field rasterizer (K5), FP64, bit-identical.
//
// Replaces render_depth_map (render.hpp:26-51) and render_pixel (opacity_field.hpp:
// 192-219) over collect_contributions (opacity_field.hpp:39-61). The reference tests
// EVERY Gaussian against every pixel ray, keeps the contributions with alpha >= 1/255 and
// t* > 0, sorts them by (t*, index) and blends front to back; the opacity at the depth is a
// product over all of them in that order. A pixel ray at a surface crossing has ~10^2
// contributions whose t* lie within a fraction of a Gaussian's extent, so any lower bound
// of t* that ignores the pixel leaves them all pending together: an exact streaming resort
// needs a window of that size per pixel. The design therefore sorts each pixel's
// contributions explicitly, in five steps per view:
//
//   R0 binning: each Gaussian's conservative screen rectangle (E-box with clamped scales,
//      one-pixel dilation; all tiles when the box crosses the camera plane, none when it
//      lies entirely behind it), then a counting sort by tile (histogram, scan, scatter:
//      no radix sort, the order inside a tile list is irrelevant because every pixel's
//      contributions are sorted later);
//   R1 k_rcount: per pixel, the number of list records that pass the screen-space conic
//      cull (FP32, Rec::conic) — an upper bound of its contributions; a scan turns the
//      bounds into per-pixel slices;
//   R2 k_rtest: one CTA per 16x16 tile streams the tile list through shared memory; each
//      warp computes its 32 pixels' conic masks for a 32-record chunk, compacts the
//      surviving (pixel, record) pairs into a queue and evaluates them on all 32 lanes
//      with the reference's FP64 expressions (no divergence on the FP64 work); every
//      contribution (t*, alpha, a, b, index) lands in its pixel's slice;
//   R3 k_rsort: one warp per pixel sorts the slice by (t*, index) in shared memory
//      (bitonic network; the key is t*'s bits with the low 10 bits replaced by the slot,
//      equal-prefix runs are re-ordered exactly); slices longer than 1024 go to a
//      CTA-wide sort in global memory (k_rsort_big);
//   R4 k_rblend: one thread per pixel walks its sorted slice: colour and transmittance
//      (render_pixel :204-210), the median (find_median :129-141), the exact depth
//      (:157-166) and the opacity at the depth (opacity_along_ray :104-108) — all in the
//      reference's order, so every output is bit-identical.
//
// Frames whose slices exceed the scratch budget are processed in bands of tiles.
#include <vector>

#include "../../include/sof_cuda.h"
#include "sof_internal.h"
#include "sof_tma.cuh"

namespace sofk {

constexpr int kRTile = 16;                // render tile (pixels per side), one CTA per tile
constexpr int kRPix = kRTile * kRTile;    // 256 pixels per tile
constexpr int kRChunk = 32;               // records staged per step
constexpr int kBigTiles = 64;             // Gaussians covering more tiles are binned by a CTA
constexpr int kSortCap = 1024;            // slice length sorted by one warp in shared memory
constexpr int kSortSlotBits = 10;         // log2(kSortCap)
constexpr int kSortWarps = 4;
constexpr int kEntryBytes = 4 * 8 + 4;  // et, ea, eA, eB, ei

// Pixel of local index l (0..255) in a tile: warp w = l / 32 covers an 8 x 4 block.
__device__ __forceinline__ void tile_pixel(int tile, int tiles_x, int l, int& x, int& y) {
  const int w = l >> 5, lane = l & 31;
  x = (tile % tiles_x) * kRTile + (w & 1) * 8 + (lane & 7);
  y = (tile / tiles_x) * kRTile + (w >> 1) * 4 + (lane >> 3);
}

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

// Per-(Gaussian, view) render record: the FP64 fields of PrecomputedGaussian that the
// contribution test reads (bit-identical to precompute.hpp:57-78, as Rec) and the
// screen-space cull in centre form. The rays that can reach alpha >= 1/255 project to
// the conic g(u, v) = d^T (b b^T - (c - L) S) d >= 0 (d the ray through pixel (u, v),
// L = 2 log(255 op); sof_device.cuh, gauss_view). For an ellipse it is stored about its
// float-rounded centre (uc, vc): g = q00 du^2 + q11 dv^2 + q01x2 du dv + g0, so the FP32
// evaluation has no cancellation, and a pixel is culled only if
//   g < -(2^-17 S + kmar),  S = |q00| du^2 + |q11| dv^2 + |q01x2 du dv| + |g0|,
// where 2^-17 S bounds the FP32 rounding (<= 10 ulp of S) and kmar bounds the FP64
// error of the conic, the dropped linear term at the rounded centre and the slack that
// keeps the reference's own FP64 alpha below 1/255 (L is raised by 1e-8 (1 + |L|) +
// 1e-12 |c|). Non-ellipses are never culled (g0 = +inf); dead records always are.
struct __align__(16) RRec {
  double ic[6];  // inv_cov upper triangle (as Rec)
  double b[3];   // b_vec
  double c;      // c_scalar
  double op;     // filtered opacity
  double pad;
  float thr;     // as Rec::thr: exponent < thr => alpha < 1/255
  float q00, q11, q01x2;
  float uc, vc;
  float g0;
  float kmar;
};
static_assert(sizeof(RRec) == 128, "render record layout");
constexpr int kRRecV2 = int(sizeof(RRec) / 16);

__device__ __forceinline__ float float_up(double x) { return __double2float_ru(x); }

__device__ void render_conic(const Rec& r, const Cam& cam, RRec& q) {
  q.q00 = q.q11 = q.q01x2 = 0.0f;
  q.uc = q.vc = 0.0f;
  q.kmar = 0.0f;
  if (r.op < kMinAlpha) {  // dead: collect_contributions skips it (:44)
    q.g0 = -1.0f;
    return;
  }
  q.g0 = INFINITY;  // never culled unless an ellipse is established below
  const double eps = 0x1p-53;
  const double L = 2.0 * log(255.0 * r.op);
  const double Lm = L + 1e-8 * (1.0 + fabs(L)) + 1e-12 * fabs(r.c);
  const double cl = r.c - Lm;
  const double S[9] = {r.ic[0], r.ic[1], r.ic[2], r.ic[1], r.ic[3], r.ic[4], r.ic[2], r.ic[4], r.ic[5]};
  double M[9], mabs = 0.0;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      M[3 * i + j] = r.b[i] * r.b[j] - cl * S[3 * i + j];
      mabs = fmax(mabs, fabs(r.b[i] * r.b[j]) + fabs(cl * S[3 * i + j]));
    }
  const double Ki[9] = {1.0 / cam.fx, 0.0, -cam.cx / cam.fx, 0.0, 1.0 / cam.fy, -cam.cy / cam.fy, 0.0, 0.0, 1.0};
  double A[9], MA[9], G[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      A[3 * i + j] = cam.R[i] * Ki[j] + cam.R[3 + i] * Ki[3 + j] + cam.R[6 + i] * Ki[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) MA[3 * i + j] = M[3 * i] * A[j] + M[3 * i + 1] * A[3 + j] + M[3 * i + 2] * A[6 + j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) G[3 * i + j] = A[i] * MA[j] + A[3 + i] * MA[3 + j] + A[6 + i] * MA[6 + j];
  const double g00 = G[0], g11 = G[4], g22 = G[8];
  const double g01 = 0.5 * (G[1] + G[3]), g02 = 0.5 * (G[2] + G[6]), g12 = 0.5 * (G[5] + G[7]);
  const double det = g00 * g11 - g01 * g01;
  if (!(g00 < 0.0 && g11 < 0.0 && det > 0.0)) return;  // not an ellipse
  const double ucd = (g01 * g12 - g11 * g02) / det, vcd = (g01 * g02 - g00 * g12) / det;
  if (!(fabs(ucd) < 1e7 && fabs(vcd) < 1e7)) return;
  const float ucf = float(ucd), vcf = float(vcd);
  const double U = ucf, V = vcf;
  // linear term left at the rounded centre (dropped) and its bound over the image
  const double l0 = g00 * U + g01 * V + g02, l1 = g01 * U + g11 * V + g12;
  const double lb = fabs(l0) + fabs(l1) +
                    4.0 * eps * (fabs(g00 * U) + 2.0 * fabs(g01 * V) + fabs(g02) + fabs(g01 * U) + fabs(g11 * V) + fabs(g12));
  const double g0 = U * (g00 * U + 2.0 * g01 * V + 2.0 * g02) + V * (g11 * V + 2.0 * g12) + g22;
  const double dg0 = 8.0 * eps *
                     (fabs(g00) * U * U + fabs(g11) * V * V + 2.0 * fabs(g01 * U * V) + 2.0 * fabs(g02 * U) +
                      2.0 * fabs(g12 * V) + fabs(g22));
  // FP64 error of G at any pixel of the image: <= 10 eps mabs |w|_1^2, w = R^T K^-1 (u, v, 1)
  const double wx = fmax(fabs(cam.cx), fabs(cam.w - cam.cx)) / cam.fx + 1.0 / cam.fx;
  const double wy = fmax(fabs(cam.cy), fabs(cam.h - cam.cy)) / cam.fy + 1.0 / cam.fy;
  const double kfp = 32.0 * eps * mabs * 3.0 * (1.0 + wx * wx + wy * wy);
  const double kmar = (2.0 * lb * (double(cam.w) + double(cam.h) + 4.0) + dg0 + kfp) * 1.01 + 1e-30;
  const float fq00 = float(g00), fq11 = float(g11), fq01 = float(2.0 * g01), fg0 = float(g0), fk = float_up(kmar);
  if (!(isfinite(fq00) && isfinite(fq11) && isfinite(fq01) && isfinite(fg0) && isfinite(fk))) return;
  q.q00 = fq00;
  q.q11 = fq11;
  q.q01x2 = fq01;
  q.uc = ucf;
  q.vc = vcf;
  q.g0 = fg0;
  q.kmar = fk;
}

// true when the ray through the pixel centre (u, v) provably stays below alpha = 1/255;
// lo = (thr, q00, q11, q01x2), hi = (uc, vc, g0, kmar): the record's last 32 bytes
__device__ __forceinline__ bool rcull(const float4& lo, const float4& hi, float u, float v) {
  const float du = u - hi.x, dv = v - hi.y;
  const float g = fmaf(lo.y * du, du, fmaf(lo.z * dv, dv, fmaf(lo.w * du, dv, hi.z)));
  const float s = fmaf(fabsf(lo.y) * du, du, fmaf(fabsf(lo.z) * dv, dv, fmaf(fabsf(lo.w * du), fabsf(dv), fabsf(hi.z))));
  return g < -fmaf(0x1p-17f, s, hi.w);
}

// K5.0 render records: gauss_view's FP64 fields (bit-identical) + the centre-form cull
__global__ void k_rrec(int64_t n, const GaussStatic* __restrict__ g, Cam cam, RRec* out) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  Rec r;
  gauss_view(g[i], cam, r);
  RRec q;
  for (int k = 0; k < 6; ++k) q.ic[k] = r.ic[k];
  for (int k = 0; k < 3; ++k) q.b[k] = r.b[k];
  q.c = r.c;
  q.op = r.op;
  q.pad = 0.0;
  q.thr = r.thr;
  render_conic(r, cam, q);
  out[i] = q;
}

template <typename Tab>
__device__ __forceinline__ double exp_any(double x, Tab tab) {
  return (x >= -700.0 && x <= 700.0) ? sof_exp_mid_cb(x, tab) : sof_exp(x);
}

// collect_contributions' per-Gaussian test (opacity_field.hpp:43-53) with the
// RayContribution fields it keeps: t*, the clamped peak alpha, and A, B of abc_cached.
template <typename Tab>
__device__ __forceinline__ bool contribution(const RRec& r, const double* d, Tab tab, double& t_star,
                                             double& alpha, double& a, double& b) {
  if (r.op < kMinAlpha) return false;  // :44
  const double x = d[0], y = d[1], z = d[2];
  a = r.ic[0] * x * x + r.ic[3] * y * y + r.ic[5] * z * z +
      2.0 * (r.ic[1] * x * y + r.ic[2] * x * z + r.ic[4] * y * z);  // abc_cached precompute.hpp:39-45
  b = 2.0 * (x * r.b[0] + y * r.b[1] + z * r.b[2]);
  // t* = -b / (2a) <= 0 (:51) exactly when b >= 0 for a > 0 (the division keeps the sign):
  // skipped before the divisions; NaN falls through to the reference expressions
  if (a > 0.0 && b >= 0.0) return false;
  const double arg = -0.5 * (r.c - b * b / (4.0 * a));  // peak_value gaussian.hpp:54-56
  if (arg < double(r.thr)) return false;                // alpha < 1/255 certain (Rec::thr)
  const double al = r.op * exp_any(arg, tab);
  if (al < kMinAlpha) return false;  // :48
  t_star = -b / (2.0 * a);           // peak_t gaussian.hpp:52
  if (t_star <= 0.0) return false;   // :51
  alpha = (kMaxAlpha < al) ? kMaxAlpha : al;  // std::min(alpha, kMaxAlpha) :52
  return true;
}

// ---- R0: render binning ------------------------------------------------------------------------

// Screen rectangle of every pixel whose ray can reach alpha >= 1/255 on Gaussian i. Such
// a ray's closest-approach point x* = o + t* d (t* > 0) lies in the E-ellipsoid of the
// clamped-scale covariance, hence in its E-box (E inflated by 1e-6): a box with every
// corner behind the camera plane cannot hold x* (its view z is t* d_z > 0), so no tiles.
// Otherwise, when the record's cull is an ellipse, the bounding box of the pixels it does
// not cull (g >= -(2^-17 S + kmar), see RRec), dilated by one pixel; else the projected
// E-box, dilated by one pixel, or every tile when the box crosses the camera plane.
__global__ void k_rrect(int64_t n, const GaussStatic* __restrict__ g, const RRec* __restrict__ rr, Cam cam,
                        int tiles_x, int tiles_y, int4* rect, uint32_t* cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const GaussStatic& G = g[i];
  uint32_t count = 0;
  if (G.E > 0.0) {
    const double E = G.E * (1.0 + 1e-6);
    double s[3];
    for (int k = 0; k < 3; ++k) s[k] = (G.scale[k] < kMinScale) ? kMinScale : G.scale[k];
    double min_x = 1e300, max_x = -1e300, min_y = 1e300, max_y = -1e300;
    bool crosses = false, behind = true;
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
      // behind iff every corner is clearly behind the plane (margin >> rounding)
      if (!(vz < -1e-9 * (fabs(vx) + fabs(vy) + fabs(vz) + 1.0))) behind = false;
      if (vz <= 1e-9) {
        crosses = true;
        continue;
      }
      const double px = cam.fx * vx / vz + cam.cx, py = cam.fy * vy / vz + cam.cy;
      min_x = fmin(min_x, px);
      max_x = fmax(max_x, px);
      min_y = fmin(min_y, py);
      max_y = fmax(max_y, py);
    }
    bool on = !behind, full = false;
    if (on) {
      // the ellipse of pixels the cull keeps: X = dp^T (-Q) dp <= R (see RRec)
      const RRec& q = rr[i];
      const double q00 = q.q00, q11 = q.q11, q01 = 0.5 * double(q.q01x2), g0 = q.g0;
      const double det = q00 * q11 - q01 * q01, tr = -(q00 + q11);
      bool ellipse = false;
      if (isfinite(g0) && q00 < 0.0 && q11 < 0.0 && det > 0.0) {
        const double kappa = (fabs(q00) + fabs(q11) + 2.0 * fabs(q01)) * tr / det;  // |Q| <= kappa (-Q)
        if (0x1p-16 * kappa < 0.5) {
          ellipse = true;
          const double R = (g0 + 0x1p-16 * fabs(g0) + double(q.kmar)) / (1.0 - 0x1p-16 * kappa) * (1.0 + 1e-9);
          if (R < 0.0) {
            on = false;
          } else {
            const double hu = sqrt(R * (-q11) / det) * (1.0 + 1e-9) + 1e-6;
            const double hv = sqrt(R * (-q00) / det) * (1.0 + 1e-9) + 1e-6;
            // pixel centres x + 0.5 within [uc - hu, uc + hu], one pixel of dilation
            min_x = double(q.uc) - hu - 1.5;
            max_x = double(q.uc) + hu + 0.5;
            min_y = double(q.vc) - hv - 1.5;
            max_y = double(q.vc) + hv + 0.5;
          }
        }
      }
      if (!ellipse) {
        if (crosses) {
          full = true;
        } else {
          min_x -= 1.0;
          min_y -= 1.0;
          max_x += 1.0;
          max_y += 1.0;
        }
      }
    }
    int tx0 = 0, tx1 = tiles_x - 1, ty0 = 0, ty1 = tiles_y - 1;
    if (on && !full) {
      on = !(max_x < 0.0 || min_x >= cam.w || max_y < 0.0 || min_y >= cam.h);
      const double lim = 1e9;
      tx0 = max(0, int(floor(fmax(min_x, -lim))) / kRTile);
      tx1 = min(tiles_x - 1, int(floor(fmin(max_x, lim))) / kRTile);
      ty0 = max(0, int(floor(fmax(min_y, -lim))) / kRTile);
      ty1 = min(tiles_y - 1, int(floor(fmin(max_y, lim))) / kRTile);
    }
    if (on && tx0 <= tx1 && ty0 <= ty1) {
      count = uint32_t(tx1 - tx0 + 1) * uint32_t(ty1 - ty0 + 1);
      rect[i] = make_int4(tx0, tx1, ty0, ty1);
    }
  }
  cnt[i] = count;
}

// Counting sort by tile. PASS 0: histogram; PASS 1: scatter through per-tile cursors.
// Gaussians with more than kBigTiles tiles are queued for the cooperative kernel.
template <int PASS>
__global__ void k_rbin(int64_t n, const int4* __restrict__ rect, const uint32_t* __restrict__ cnt, int tiles_x,
                       uint32_t* tile_cnt, const int64_t* __restrict__ tile_off, int32_t* ent, int32_t* big,
                       int32_t* big_cnt) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cnt[i];
  if (c == 0) return;
  if (c > uint32_t(kBigTiles)) {
    if (PASS == 0) big[atomicAdd(big_cnt, 1)] = int32_t(i);
    return;
  }
  const int4 r = rect[i];
  for (int ty = r.z; ty <= r.w; ++ty)
    for (int tx = r.x; tx <= r.y; ++tx) {
      const int t = ty * tiles_x + tx;
      const uint32_t slot = atomicAdd(&tile_cnt[t], 1u);
      if (PASS == 1) ent[tile_off[t] + slot] = int32_t(i);
    }
}

template <int PASS>
__global__ void k_rbin_big(const int4* __restrict__ rect, int tiles_x, uint32_t* tile_cnt,
                           const int64_t* __restrict__ tile_off, int32_t* ent, const int32_t* __restrict__ big,
                           const int32_t* __restrict__ big_cnt) {
  const int nb = *big_cnt;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int32_t g = big[b];
    const int4 r = rect[g];
    const int w = r.y - r.x + 1;
    const int count = w * (r.w - r.z + 1);
    for (int k = threadIdx.x; k < count; k += blockDim.x) {
      const int t = (r.z + k / w) * tiles_x + r.x + k % w;
      const uint32_t slot = atomicAdd(&tile_cnt[t], 1u);
      if (PASS == 1) ent[tile_off[t] + slot] = g;
    }
  }
}

// ---- R1: per-pixel bounds ------------------------------------------------------------------------

__global__ void __launch_bounds__(kRPix) k_rcount(Cam cam, int tiles_x, const int64_t* __restrict__ toff,
                                                  const int32_t* __restrict__ ent, const RRec* __restrict__ recs,
                                                  uint32_t* pcnt, unsigned long long* stats) {
  __shared__ float4 sc[kRChunk][2];
  const int tile = int(blockIdx.x), l = threadIdx.x;
  int x, y;
  tile_pixel(tile, tiles_x, l, x, y);
  const bool valid = x < cam.w && y < cam.h;
  const float cu = float(x) + 0.5f, cv = float(y) + 0.5f;
  const int64_t l0 = toff[tile], l1 = toff[tile + 1];
  uint32_t count = 0;
  for (int64_t base = l0; base < l1; base += kRChunk) {
    const int cnt = int(min(int64_t(kRChunk), l1 - base));
    if (l < 2 * cnt) {
      const int32_t g = ent[base + (l >> 1)];
      sc[l >> 1][l & 1] = __ldg(reinterpret_cast<const float4*>(recs + g) + 6 + (l & 1));
    }
    __syncthreads();
    if (valid)
      for (int k = 0; k < cnt; ++k) count += rcull(sc[k][0], sc[k][1], cu, cv) ? 0u : 1u;
    __syncthreads();
  }
  pcnt[int64_t(tile) * kRPix + l] = valid ? count : 0u;
  const int nvalid = __syncthreads_count(valid);
  if (l == 0 && nvalid) atomicAdd(stats, (unsigned long long)(l1 - l0) * nvalid);
}

// ---- R2: FP64 contribution tests -----------------------------------------------------------------

// The contributions of pixel q occupy [poff[q] - base, + ncon[q]) of each array (SoA);
// R3 sorts them in place by (t*, index).
struct REntries {
  double* t;      // t* (peak_t)
  double* alpha;  // clamped peak alpha
  double* a;      // A (abc_cached)
  double* b;      // B
  int32_t* idx;   // Gaussian index
};

__global__ void __launch_bounds__(kRPix) k_rtest(Cam cam, int tiles_x, int tile0, const int64_t* __restrict__ toff,
                                                 const int32_t* __restrict__ ent, const RRec* __restrict__ recs,
                                                 const int64_t* __restrict__ poff, int64_t base, REntries E,
                                                 uint32_t* ncon, unsigned long long* stats) {
  __shared__ __align__(16) RRec srec[kRChunk];
  __shared__ int32_t sidx[kRChunk];
  __shared__ double sray[3][kRPix];
  __shared__ int64_t sbase[kRPix];
  __shared__ int scur[kRPix];
  __shared__ uint16_t queue[kRPix / 32][32 * kRChunk];
  __shared__ __align__(16) double s_exp[128];
  const int tile = tile0 + int(blockIdx.x), l = threadIdx.x, w = l >> 5, lane = l & 31;
  int x, y;
  tile_pixel(tile, tiles_x, l, x, y);
  const bool valid = x < cam.w && y < cam.h;
  {
    double d[3] = {0.0, 0.0, 1.0};
    if (valid) pixel_ray(cam, x, y, d);
    for (int k = 0; k < 3; ++k) sray[k][l] = d[k];
  }
  const int64_t q = int64_t(tile) * kRPix + l;
  sbase[l] = poff[q] - base;
  scur[l] = 0;
  for (int k = l; k < 128; k += kRPix) s_exp[k] = kSofExpTabDev[k];
  const SofExpSmem tab{smem_u32(s_exp)};
  const float cu = float(x) + 0.5f, cv = float(y) + 0.5f;
  const int64_t l0 = toff[tile], l1 = toff[tile + 1];
  for (int64_t b0 = l0; b0 < l1; b0 += kRChunk) {
    const int cnt = int(min(int64_t(kRChunk), l1 - b0));
    for (int k = l; k < cnt * kRRecV2; k += kRPix) {
      const int r = k / kRRecV2, qq = k % kRRecV2;
      const int32_t g = ent[b0 + r];
      reinterpret_cast<double2*>(&srec[r])[qq] = __ldg(reinterpret_cast<const double2*>(recs + g) + qq);
      if (qq == 0) sidx[r] = g;
    }
    __syncthreads();
    // this lane's pixel: which of the chunk's records survive the cull
    uint32_t mask = 0;
    if (valid)
      for (int k = 0; k < cnt; ++k) {
        const float4* f = reinterpret_cast<const float4*>(&srec[k]) + 6;
        if (!rcull(f[0], f[1], cu, cv)) mask |= 1u << k;
      }
    // compact the warp's surviving (pixel, record) pairs into its queue
    const int np = __popc(mask);
    int at = np;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, at, s);
      if (lane >= s) at += u;
    }
    const int total = __shfl_sync(0xffffffffu, at, 31);
    at -= np;
    while (mask) {
      const int k = __ffs(mask) - 1;
      mask &= mask - 1;
      queue[w][at++] = uint16_t((lane << 5) | k);
    }
    __syncwarp();
    // FP64 tests on every lane
    for (int qi = lane; qi < total; qi += 32) {
      const int v = queue[w][qi];
      const int pl = (w << 5) | (v >> 5), k = v & 31;
      const double d[3] = {sray[0][pl], sray[1][pl], sray[2][pl]};
      double t_star, alpha, a, b;
      if (contribution(srec[k], d, tab, t_star, alpha, a, b)) {
        const int64_t o = sbase[pl] + atomicAdd(&scur[pl], 1);
        E.t[o] = t_star;
        E.alpha[o] = alpha;
        E.a[o] = a;
        E.b[o] = b;
        E.idx[o] = sidx[k];
      }
    }
    __syncthreads();
  }
  const uint32_t mine = uint32_t(scur[l]);
  ncon[q] = mine;
  unsigned long long s1 = mine;
  for (int s = 16; s > 0; s >>= 1) s1 += __shfl_down_sync(0xffffffffu, s1, s);
  if (lane == 0 && s1) atomicAdd(stats + 1, s1);
}

// ---- R3: per-pixel sort by (t*, index), in place ---------------------------------------------------

__device__ __forceinline__ bool entry_less(const double* __restrict__ t, const int32_t* __restrict__ idx, int64_t a,
                                           int64_t b) {
  const double ta = t[a], tb = t[b];
  return ta < tb || (ta == tb && idx[a] < idx[b]);
}

// Ascending sort of m (power of two, 32..kSortCap) keys in shared memory by one warp:
// the bitonic network in its "flip" form (every compare-exchange puts the smaller key at
// the lower position), so +inf padding stays at the end.
__device__ __forceinline__ void warp_sort_keys(uint64_t* k, int m, int lane) {
  for (int size = 2; size <= m; size <<= 1) {
    const int h = size >> 1;
    __syncwarp();
    for (int i = lane; i < (m >> 1); i += 32) {  // flip: i against its mirror in the block
      const int lo = (i / h) * size + (i % h), hi = (i / h) * size + size - 1 - (i % h);
      const uint64_t a = k[lo], b = k[hi];
      if (b < a) {
        k[lo] = b;
        k[hi] = a;
      }
    }
    for (int stride = size >> 2; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int i = lane; i < (m >> 1); i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const uint64_t a = k[lo], b = k[hi];
        if (b < a) {
          k[lo] = b;
          k[hi] = a;
        }
      }
    }
  }
  __syncwarp();
}

// Permutes one field of a slice in place: f[i] = f[perm[i]] for i < n (staged in K).
template <typename T>
__device__ __forceinline__ void apply_perm(T* f, const uint16_t* perm, uint64_t* K, int n, int lane) {
  for (int i = lane; i < n; i += 32) {
    T v = f[perm[i]];
    uint64_t u = 0;
    memcpy(&u, &v, sizeof(T));
    K[i] = u;
  }
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    T v;
    const uint64_t u = K[i];
    memcpy(&v, &u, sizeof(T));
    f[i] = v;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kSortWarps * 32) k_rsort(int64_t q0, int64_t nq, const int64_t* __restrict__ poff,
                                                          int64_t base, const uint32_t* __restrict__ ncon,
                                                          REntries E, int32_t* big, int32_t* big_cnt) {
  __shared__ uint64_t sk[kSortWarps][kSortCap];
  __shared__ uint16_t sp[kSortWarps][kSortCap];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* K = sk[w];
  uint16_t* perm = sp[w];
  for (int64_t qq = int64_t(blockIdx.x) * kSortWarps + w; qq < nq; qq += int64_t(gridDim.x) * kSortWarps) {
    const int64_t q = q0 + qq;
    const int n = int(ncon[q]);
    if (n <= 1) continue;
    if (n > kSortCap) {
      if (lane == 0) {
        big[atomicAdd(big_cnt, 1)] = int32_t(q);
        atomicAdd(big_cnt + 1, 1);  // frame total (stats)
      }
      continue;
    }
    const int64_t o = poff[q] - base;
    int m = 32;
    while (m < n) m <<= 1;
    double* T = E.t + o;
    int32_t* I = E.idx + o;
    // t* > 0: its bit pattern orders like the value; the low bits carry the slot
    constexpr uint64_t kLow = (uint64_t(1) << kSortSlotBits) - 1;
    for (int i = lane; i < m; i += 32)
      K[i] = (i < n) ? ((uint64_t(__double_as_longlong(T[i])) & ~kLow) | uint64_t(i)) : ~uint64_t(0);
    warp_sort_keys(K, m, lane);
    // keys equal above the slot bits are ordered exactly by (t*, index) — rare
    bool tie = false;
    for (int i = lane; i + 1 < n; i += 32) tie |= (K[i] >> kSortSlotBits) == (K[i + 1] >> kSortSlotBits);
    if (__any_sync(0xffffffffu, tie) && lane == 0) {
      for (int i = 1; i < n; ++i) {  // insertion sort: only equal-prefix runs move
        const uint64_t v = K[i];
        int j = i - 1;
        while (j >= 0 && entry_less(T, I, int64_t(v & kLow), int64_t(K[j] & kLow))) {
          K[j + 1] = K[j];
          --j;
        }
        K[j + 1] = v;
      }
    }
    __syncwarp();
    for (int i = lane; i < n; i += 32) perm[i] = uint16_t(K[i] & kLow);
    __syncwarp();
    apply_perm(T, perm, K, n, lane);
    apply_perm(E.alpha + o, perm, K, n, lane);
    apply_perm(E.a + o, perm, K, n, lane);
    apply_perm(E.b + o, perm, K, n, lane);
    apply_perm(I, perm, K, n, lane);
  }
}

// Slices longer than kSortCap (rare): one CTA per pixel runs the flip-bitonic network on
// the slice itself in global memory (exact (t*, index) comparisons, all five fields
// swapped); positions >= n act as +inf, so compare-exchanges touching them are no-ops.
__device__ __forceinline__ void swap_entries(REntries& E, int64_t a, int64_t b) {
  double t;
  t = E.t[a], E.t[a] = E.t[b], E.t[b] = t;
  t = E.alpha[a], E.alpha[a] = E.alpha[b], E.alpha[b] = t;
  t = E.a[a], E.a[a] = E.a[b], E.a[b] = t;
  t = E.b[a], E.b[a] = E.b[b], E.b[b] = t;
  const int32_t i = E.idx[a];
  E.idx[a] = E.idx[b];
  E.idx[b] = i;
}

__global__ void __launch_bounds__(512) k_rsort_big(const int64_t* __restrict__ poff, int64_t base,
                                                   const uint32_t* __restrict__ ncon, REntries E,
                                                   const int32_t* __restrict__ big, const int32_t* __restrict__ big_cnt) {
  const int nb = *big_cnt;
  for (int bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const int64_t q = big[bi];
    const int64_t n = ncon[q];
    const int64_t o = poff[q] - base;
    int64_t m = 1;
    while (m < n) m <<= 1;
    for (int64_t size = 2; size <= m; size <<= 1) {
      const int64_t h = size >> 1;
      for (int64_t i = threadIdx.x; i < (m >> 1); i += blockDim.x) {
        const int64_t lo = (i / h) * size + (i % h), hi = (i / h) * size + size - 1 - (i % h);
        if (hi < n && entry_less(E.t, E.idx, o + hi, o + lo)) swap_entries(E, o + lo, o + hi);
      }
      __syncthreads();
      for (int64_t stride = size >> 2; stride > 0; stride >>= 1) {
        for (int64_t i = threadIdx.x; i < (m >> 1); i += blockDim.x) {
          const int64_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
          if (hi < n && entry_less(E.t, E.idx, o + hi, o + lo)) swap_entries(E, o + lo, o + hi);
        }
        __syncthreads();
      }
    }
  }
}

// ---- R4: blend, depth, opacity at depth --------------------------------------------------------------

struct RenderOut {
  double* depth;
  double* opacity;
  double* rgb;
  double* tfinal;
};

// One thread per pixel over its sorted slice (sequential reads).
__global__ void __launch_bounds__(kRPix) k_rblend(Cam cam, int tiles_x, int tile0, const int64_t* __restrict__ poff,
                                                  int64_t base, const uint32_t* __restrict__ ncon, REntries E,
                                                  const RRec* __restrict__ recs, const double* __restrict__ dc,
                                                  int exact_depth, RenderOut out, unsigned long long* stats) {
  __shared__ __align__(16) double s_exp[128];
  for (int k = threadIdx.x; k < 128; k += blockDim.x) s_exp[k] = kSofExpTabDev[k];
  __syncthreads();
  const SofExpSmem tab{smem_u32(s_exp)};
  const int tile = tile0 + int(blockIdx.x), l = threadIdx.x;
  int x, y;
  tile_pixel(tile, tiles_x, l, x, y);
  if (!(x < cam.w && y < cam.h)) return;
  const int64_t q = int64_t(tile) * kRPix + l;
  const int n = int(ncon[q]);
  const int64_t o = poff[q] - base;
  const double* __restrict__ Tt = E.t + o;
  const double* __restrict__ Ta = E.alpha + o;
  const double* __restrict__ TA = E.a + o;
  const double* __restrict__ TB = E.b + o;
  const int32_t* __restrict__ Ti = E.idx + o;
  // render_pixel (opacity_field.hpp:201-210) + find_median (:129-141) in one pass
  double T = 1.0, col[3] = {0.0, 0.0, 0.0};
  int med = -1;
  double med_T = 1.0;
  for (int j = 0; j < n; ++j) {
    const double alpha = Ta[j];
    const int32_t g = Ti[j];
    for (int k = 0; k < 3; ++k) col[k] = col[k] + __ldg(dc + 3 * g + k) * alpha * T;
    const double next = T * (1.0 - alpha);
    if (med < 0 && T > 0.5 && next < 0.5) {
      med = j;
      med_T = T;
    }
    T = next;
  }
  double depth = NAN;
  if (med >= 0) {
    const double med_t = Tt[med];
    depth = med_t;      // median_depth (:143-147)
    if (exact_depth) {  // exact_depth (:157-166)
      const RRec& r = recs[Ti[med]];
      const double a = TA[med], b = TB[med];
      const double lt = 2.0 * sof_log((med_T - 0.5) / (med_T * r.op));
      const double disc = b * b - 4.0 * a * (r.c + lt);
      if (disc < 0.0) {
        atomicAdd(stats + 3, 1ull);
      } else {
        depth = med_t - sqrt(disc) / (2.0 * a);
      }
    }
  }
  // accumulated opacity = opacity_along_ray(contribs, depth) (:104-108, 216-217)
  double acc = 0.0;
  if (!isnan(depth)) {
    double T2 = 1.0;
    for (int j = 0; j < n; ++j) {
      const double ts = Tt[j];
      const double te = (depth < ts) ? depth : ts;  // alpha_at :95-101, std::min(t*, t)
      double al = 0.0;
      if (te > 0.0) {
        const RRec* r = recs + Ti[j];
        const double a = TA[j], b = TB[j];
        const double arg = -0.5 * ((a * te + b) * te + __ldg(&r->c));  // eval_1d gaussian.hpp:47-49
        if (!(arg < double(__ldg(&r->thr)))) {                         // else alpha < 1/255 certain
          al = __ldg(&r->op) * exp_any(arg, tab);
          if (al < kMinAlpha) al = 0.0;
          else if (kMaxAlpha < al) al = kMaxAlpha;
        }
      }
      T2 *= 1.0 - al;
    }
    acc = 1.0 - T2;
  }
  const int64_t p = int64_t(y) * cam.w + x;
  out.depth[p] = depth;
  out.opacity[p] = acc;
  for (int k = 0; k < 3; ++k) out.rgb[3 * p + k] = col[k];
  out.tfinal[p] = T;
}

// slice offset of every tile's first pixel (band planning)
__global__ void k_tile_slice_off(int64_t T, const int64_t* __restrict__ poff, int64_t* out) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t <= T) out[t] = poff[t * kRPix];
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

extern "C" int sof_set_render_pool(sof_ctx* c, int64_t bytes) {
  if (!c || bytes < 0) return SOF_E_INVALID;
  c->render_pool = bytes > 0 ? bytes : (int64_t(24) << 30);
  return SOF_OK;
}

extern "C" int sof_render_view(sof_ctx* c, int view, int depth_mode, int tile_size, double* depth,
                               double* opacity, double* rgb, double* t_final, uint64_t* stats) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    if (depth_mode != SOF_DEPTH_EXACT && depth_mode != SOF_DEPTH_MEDIAN) throw InvalidArg("unknown depth mode");
    (void)tile_size;  // the reference render has no tiles; the render tile is fixed at 16
    const Cam& cam = c->cams[view];
    const int tiles_x = (cam.w + kRTile - 1) / kRTile, tiles_y = (cam.h + kRTile - 1) / kRTile;
    const int64_t T = int64_t(tiles_x) * tiles_y;
    const int64_t n = c->n, P = int64_t(cam.w) * cam.h, Q = T * kRPix;
    if (T > INT32_MAX / kRPix) throw InvalidArg("image too large");
    RenderScratch& rs = c->rs;
    cudaStream_t st = c->stream;
    rs.big_cnt.ensure(4);  // [0] big Gaussians (binning), [1] big pixels (band), [2] big pixels (frame)
    SOF_CUDA(cudaMemsetAsync(rs.big_cnt.p, 0, 4 * sizeof(int32_t), st));
    c->r_stats.ensure(4);
    SOF_CUDA(cudaMemsetAsync(c->r_stats.p, 0, 4 * sizeof(unsigned long long), st));
    // R0: binning
    rs.tile_cnt.ensure(T);
    rs.tile_off.ensure(T + 1);
    SOF_CUDA(cudaMemsetAsync(rs.tile_cnt.p, 0, sizeof(uint32_t) * T, st));
    rs.rrec.ensure(std::max<int64_t>(n, 1) * sizeof(RRec));
    RRec* rec = reinterpret_cast<RRec*>(rs.rrec.p);
    if (n > 0) {
      rs.rect.ensure(n);
      rs.gcnt.ensure(n);
      rs.big.ensure(std::max<int64_t>(n, Q));
      k_rrec<<<grid_for(n, 128), 128, 0, st>>>(n, c->gstat.p, cam, rec);
      k_rrect<<<grid_for(n, 128), 128, 0, st>>>(n, c->gstat.p, rec, cam, tiles_x, tiles_y, rs.rect.p, rs.gcnt.p);
      c->launches += 1;
      k_rbin<0><<<grid_for(n, 256), 256, 0, st>>>(n, rs.rect.p, rs.gcnt.p, tiles_x, rs.tile_cnt.p, nullptr, nullptr,
                                                   rs.big.p, rs.big_cnt.p);
      k_rbin_big<0><<<2 * 148, 256, 0, st>>>(rs.rect.p, tiles_x, rs.tile_cnt.p, nullptr, nullptr, rs.big.p,
                                              rs.big_cnt.p);
      c->launches += 3;
      SOF_CUDA(cudaGetLastError());
    }
    scan_u32_i64(c, rs.tile_cnt.p, rs.tile_off.p, T);
    const int64_t M = read_scalar(c, rs.tile_off.p + T);
    rs.ent.ensure(std::max<int64_t>(M, 1));
    if (M > 0) {
      SOF_CUDA(cudaMemsetAsync(rs.tile_cnt.p, 0, sizeof(uint32_t) * T, st));
      k_rbin<1><<<grid_for(n, 256), 256, 0, st>>>(n, rs.rect.p, rs.gcnt.p, tiles_x, rs.tile_cnt.p, rs.tile_off.p,
                                                   rs.ent.p, rs.big.p, rs.big_cnt.p);
      k_rbin_big<1><<<2 * 148, 256, 0, st>>>(rs.rect.p, tiles_x, rs.tile_cnt.p, rs.tile_off.p, rs.ent.p, rs.big.p,
                                              rs.big_cnt.p);
      c->launches += 2;
      SOF_CUDA(cudaGetLastError());
    }
    // R1: per-pixel bounds and slices (tile-major pixel order)
    rs.pcnt.ensure(Q);
    rs.ncon.ensure(Q);
    rs.poff.ensure(Q + 1);
    k_rcount<<<unsigned(T), kRPix, 0, st>>>(cam, tiles_x, rs.tile_off.p, rs.ent.p, rec, rs.pcnt.p, c->r_stats.p);
    SOF_LAUNCHED(c);
    scan_u32_i64(c, rs.pcnt.p, rs.poff.p, Q);
    const int64_t total = read_scalar(c, rs.poff.p + Q);
    c->r_out.ensure(6 * P);
    RenderOut out{c->r_out.p, c->r_out.p + P, c->r_out.p + 2 * P, c->r_out.p + 5 * P};
    // bands of tiles whose slices fit the scratch budget
    const int64_t cap = std::max<int64_t>(c->render_pool / kEntryBytes, 1);
    std::vector<int64_t> toff;
    if (total > cap) {
      rs.band_off.ensure(T + 1);
      k_tile_slice_off<<<grid_for(T + 1, 256), 256, 0, st>>>(T, rs.poff.p, rs.band_off.p);
      SOF_LAUNCHED(c);
      toff.resize(T + 1);
      SOF_CUDA(cudaMemcpyAsync(toff.data(), rs.band_off.p, sizeof(int64_t) * (T + 1), cudaMemcpyDeviceToHost, st));
      SOF_CUDA(cudaStreamSynchronize(st));
    }
    int64_t nbands = 0;
    for (int64_t t0 = 0; t0 < T;) {
      int64_t t1 = T, e0 = 0, e1 = total;
      if (total > cap) {
        t1 = t0 + 1;  // at least one tile per band
        while (t1 < T && toff[t1 + 1] - toff[t0] <= cap) ++t1;
        e0 = toff[t0];
        e1 = toff[t1];
      }
      const int64_t ne = std::max<int64_t>(e1 - e0, 1);
      rs.et.ensure(ne);
      rs.ea.ensure(ne);
      rs.eA.ensure(ne);
      rs.eB.ensure(ne);
      rs.ei.ensure(ne);
      REntries E{rs.et.p, rs.ea.p, rs.eA.p, rs.eB.p, rs.ei.p};
      const unsigned nt = unsigned(t1 - t0);
      k_rtest<<<nt, kRPix, 0, st>>>(cam, tiles_x, int(t0), rs.tile_off.p, rs.ent.p, rec, rs.poff.p, e0, E,
                                    rs.ncon.p, c->r_stats.p);
      SOF_LAUNCHED(c);
      SOF_CUDA(cudaMemsetAsync(rs.big_cnt.p + 1, 0, sizeof(int32_t), st));
      const int64_t nq = int64_t(nt) * kRPix;
      const unsigned sort_grid = unsigned(std::min<int64_t>((nq + kSortWarps - 1) / kSortWarps, 148 * 32));
      k_rsort<<<sort_grid, kSortWarps * 32, 0, st>>>(t0 * kRPix, nq, rs.poff.p, e0, rs.ncon.p, E, rs.big.p,
                                                      rs.big_cnt.p + 1);
      k_rsort_big<<<148, 512, 0, st>>>(rs.poff.p, e0, rs.ncon.p, E, rs.big.p, rs.big_cnt.p + 1);
      k_rblend<<<nt, kRPix, 0, st>>>(cam, tiles_x, int(t0), rs.poff.p, e0, rs.ncon.p, E, rec, c->dc.p,
                                     depth_mode == SOF_DEPTH_EXACT, out, c->r_stats.p);
      c->launches += 3;
      SOF_CUDA(cudaGetLastError());
      ++nbands;
      t0 = t1;
    }
    c->r_view = view;
    c->r_bands = nbands;
    if (depth) SOF_CUDA(cudaMemcpyAsync(depth, out.depth, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
    if (opacity) SOF_CUDA(cudaMemcpyAsync(opacity, out.opacity, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
    if (rgb) SOF_CUDA(cudaMemcpyAsync(rgb, out.rgb, sizeof(double) * 3 * P, cudaMemcpyDeviceToHost, st));
    if (t_final) SOF_CUDA(cudaMemcpyAsync(t_final, out.tfinal, sizeof(double) * P, cudaMemcpyDeviceToHost, st));
    if (stats) {
      unsigned long long h[4];
      int32_t nbig = 0;
      SOF_CUDA(cudaMemcpyAsync(h, c->r_stats.p, sizeof h, cudaMemcpyDeviceToHost, st));
      SOF_CUDA(cudaMemcpyAsync(&nbig, rs.big_cnt.p + 2, sizeof nbig, cudaMemcpyDeviceToHost, st));
      SOF_CUDA(cudaStreamSynchronize(st));
      stats[0] = h[0];  // tested (pixel, list entry) pairs
      stats[1] = h[1];  // contributions
      stats[2] = uint64_t(nbig);  // pixels whose slice took the CTA-wide sort (> 1024 contributions)
      stats[3] = h[3];  // exact-depth fallbacks (negative discriminant)
    }
    SOF_CUDA(cudaStreamSynchronize(st));
  });
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
