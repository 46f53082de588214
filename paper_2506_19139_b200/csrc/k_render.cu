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
//   R0 binning: per Gaussian a render record (RRec: the FP64 fields of the test plus the
//      screen conic in centre form) and its conservative screen rectangle (the conic's
//      ellipse box, else the E-box with clamped scales, one-pixel dilation; all tiles when
//      the box crosses the camera plane, none when it lies entirely behind it), minus the
//      tiles whose every pixel centre the conic cull rejects (rtile_culled); then a
//      counting sort by tile (histogram, scan, scatter: the order inside a tile list is
//      irrelevant because every pixel's contributions are sorted later);
//   R1 k_rcount: per pixel, the number of list records that pass the FP32 conic cull —
//      an upper bound of its contributions; a scan turns the bounds into per-pixel slices;
//   R2 k_rtest: one CTA per 16x16 tile streams the tile list through shared memory (FP64
//      fields as columns); each warp computes its 32 pixels' cull masks for a 32-record
//      chunk, the CTA compacts the surviving (pixel, record) pairs into one queue and all
//      256 threads evaluate them with the reference's FP64 expressions; every contribution
//      lands in its pixel's slice as REnt {t*, list position, Gaussian index};
//   R3 k_rsort: one warp per pixel sorts its slice by (t*, index): a register bitonic
//      network on 32-bit keys (the top bits of bits(t*) - bits(min t*) above the slot),
//      runs of equal key then put in exact (t*, index) order, the entries permuted once
//      through shared memory; slices past 256 entries go to k_rsort_mid (512), then
//      k_rsort_big (one CTA, up to 4096 in shared memory, a global-memory network beyond);
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
#include "stl_order.cuh"

namespace sofk {

constexpr int kRTile = 16;                // render tile (pixels per side), one CTA per tile
constexpr int kRPix = kRTile * kRTile;    // 256 pixels per tile
constexpr int kRChunk = 32;               // records staged per step
constexpr int kBigTiles = 64;             // Gaussians covering more tiles are binned by a CTA
constexpr int kSortWarps = 8;
constexpr int kEntryBytes = 16;  // REnt

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

// The fields of one list record the blend reads (RRec's FP64 part + the DC colour),
// staged per tile in shared memory as 7 double2 rows.
struct BRec {
  double ic[6], b[3], c, op, dc[3];
  float thr;
};
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

// True when rcull culls every pixel of tile (tx, ty) for this record: the exact maximum of
// the centre-form conic over the tile's pixel centres (a concave quadratic: the centre if
// it lies inside the box, else the best point of the nearest edges) stays below
// -(3 2^-17 S_max + kmar), S_max the largest |term| sum over the box (at a corner). rcull's
// float evaluation at any pixel of the tile errs by at most 2^-17 S <= 2^-17 S_max, so it
// culls each of them: listing the record in that tile changes no test outcome.
__device__ __forceinline__ bool rtile_culled(const RRec& q, int tx, int ty) {
  const double q00 = q.q00, q11 = q.q11, q01 = 0.5 * double(q.q01x2), g0 = q.g0;
  if (!(isfinite(g0) && q00 < 0.0 && q11 < 0.0 && q00 * q11 - q01 * q01 > 0.0)) return false;
  const double u0 = tx * kRTile + 0.5 - double(q.uc), u1 = u0 + (kRTile - 1);
  const double v0 = ty * kRTile + 0.5 - double(q.vc), v1 = v0 + (kRTile - 1);
  auto g = [&](double du, double dv) { return (q00 * du * du + q11 * dv * dv) + 2.0 * q01 * du * dv + g0; };
  auto clampd = [](double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); };
  double m;
  if (u0 <= 0.0 && 0.0 <= u1 && v0 <= 0.0 && 0.0 <= v1) {
    m = g0;  // the apex lies in the box
  } else {
    // along each edge the concave 1D quadratic peaks at its clamped vertex
    m = -INFINITY;
    const double us[2] = {u0, u1}, vs[2] = {v0, v1};
    for (int k = 0; k < 2; ++k) {
      const double dv = clampd(-q01 * us[k] / q11, v0, v1);
      m = fmax(m, g(us[k], dv));
      const double du = clampd(-q01 * vs[k] / q00, u0, u1);
      m = fmax(m, g(du, vs[k]));
    }
  }
  const double au = fmax(fabs(u0), fabs(u1)), av = fmax(fabs(v0), fabs(v1));
  const double smax = (fabs(q00) * au * au + fabs(q11) * av * av + fabs(double(q.q01x2)) * au * av + fabs(g0)) *
                      (1.0 + 1e-5);
  return m < -(3.0 * 0x1p-17 * smax + double(q.kmar));
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
template <typename Tab, typename R>
__device__ __forceinline__ bool contribution(const R& r, const double* d, Tab tab, double& t_star,
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
                        int tiles_x, int tiles_y, int4* rect, uint32_t* cnt, uint64_t* tmask) {
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
      if (count <= uint32_t(kBigTiles)) {  // the rectangle's tiles the cull leaves, row-major bits
        const RRec q = rr[i];
        uint64_t m = 0;
        int k = 0;
        for (int ty = ty0; ty <= ty1; ++ty)
          for (int tx = tx0; tx <= tx1; ++tx, ++k)
            if (!rtile_culled(q, tx, ty)) m |= uint64_t(1) << k;
        tmask[i] = m;
        if (m == 0) count = 0;
      }
    }
  }
  cnt[i] = count;
}

// Counting sort by tile. PASS 0: histogram; PASS 1: scatter through per-tile cursors.
// Gaussians with more than kBigTiles tiles are queued for the cooperative kernel.
// Tiles of the rectangle whose pixels the record's cull rejects entirely (rtile_culled) are
// skipped in both passes: per-Gaussian tile masks from k_rrect for rectangles of up to
// kBigTiles tiles, the test itself in the cooperative kernel for the larger ones.
template <int PASS>
__global__ void k_rbin(int64_t n, const int4* __restrict__ rect, const uint32_t* __restrict__ cnt, int tiles_x,
                       uint32_t* tile_cnt, const int64_t* __restrict__ tile_off, int32_t* ent, int32_t* big,
                       int32_t* big_cnt, const uint64_t* __restrict__ tmask) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const uint32_t c = cnt[i];
  if (c == 0) return;
  if (c > uint32_t(kBigTiles)) {
    if (PASS == 0) big[atomicAdd(big_cnt, 1)] = int32_t(i);
    return;
  }
  const int4 r = rect[i];
  const uint64_t m = tmask[i];
  int k = 0;
  for (int ty = r.z; ty <= r.w; ++ty)
    for (int tx = r.x; tx <= r.y; ++tx, ++k) {
      if (!((m >> k) & 1)) continue;  // rtile_culled (k_rrect)
      const int t = ty * tiles_x + tx;
      const uint32_t slot = atomicAdd(&tile_cnt[t], 1u);
      if (PASS == 1) ent[tile_off[t] + slot] = int32_t(i);
    }
}

template <int PASS>
__global__ void k_rbin_big(const int4* __restrict__ rect, int tiles_x, uint32_t* tile_cnt,
                           const int64_t* __restrict__ tile_off, int32_t* ent, const int32_t* __restrict__ big,
                           const int32_t* __restrict__ big_cnt, const RRec* __restrict__ recs) {
  const int nb = *big_cnt;
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int32_t g = big[b];
    const int4 r = rect[g];
    const RRec q = recs[g];
    const int w = r.y - r.x + 1;
    const int count = w * (r.w - r.z + 1);
    for (int k = threadIdx.x; k < count; k += blockDim.x) {
      const int tx = r.x + k % w, ty = r.z + k / w;
      if (rtile_culled(q, tx, ty)) continue;
      const int t = ty * tiles_x + tx;
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

// One contribution of a pixel ray (RayContribution, opacity_field.hpp:13-19, reduced to
// what the sort and the blend cannot recompute cheaply): t* and the Gaussian index are
// the sort key (:56-59); pos is the record's position in the tile list. A, B and alpha
// are recomputed from the record in R4 with the same expressions (same bits). The
// contributions of pixel q occupy [poff[q] - base, + ncon[q]); R3 sorts them in place.
struct __align__(16) REnt {
  double t;
  int32_t pos;
  int32_t idx;
};
static_assert(sizeof(REnt) == 16, "entry layout");

#ifndef SOF_RTEST_MINB
#define SOF_RTEST_MINB 4  // 64 registers, 4 CTAs per SM (70 registers, 3 CTAs: 3.45 vs 3.31 ms per C2 view)
#endif
__global__ void __launch_bounds__(kRPix, SOF_RTEST_MINB) k_rtest(Cam cam, int tiles_x, int tile0, const int64_t* __restrict__ toff,
                                                 const int32_t* __restrict__ ent, const RRec* __restrict__ recs,
                                                 const int64_t* __restrict__ poff, int64_t base, REnt* E,
                                                 uint32_t* ncon, unsigned long long* stats) {
  // the chunk's records: conic floats as rows (every lane reads the same record: a
  // broadcast), FP64 fields as columns (lanes of the FP64 phase read different records:
  // consecutive words, no bank conflicts; 128-byte rows would put every record's field in
  // the same bank)
  __shared__ __align__(16) float4 sc[kRChunk][2];
  __shared__ double sd[11][kRChunk];
  __shared__ int32_t sidx[kRChunk];
  __shared__ double sray[3][kRPix];
  __shared__ int64_t sbase[kRPix];
  __shared__ int scur[kRPix];
  __shared__ uint16_t queue[kRPix * kRChunk];
  __shared__ int swarp[kRPix / 32];
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
      const double2 v = __ldg(reinterpret_cast<const double2*>(recs + g) + qq);
      if (qq < 5) {
        sd[2 * qq][r] = v.x;
        sd[2 * qq + 1][r] = v.y;
      } else if (qq == 5) {
        sd[10][r] = v.x;  // op
        sidx[r] = g;
      } else {
        sc[r][qq - 6] = *reinterpret_cast<const float4*>(&v);
      }
    }
    __syncthreads();
    // this lane's pixel: which of the chunk's records survive the cull
    uint32_t mask = 0;
    if (valid)
      for (int k = 0; k < cnt; ++k)
        if (!rcull(sc[k][0], sc[k][1], cu, cv)) mask |= 1u << k;
    // compact the CTA's surviving (pixel, record) pairs into one queue: warp prefix sums,
    // then the warps' offsets, so the FP64 work is spread over all 256 threads
    const int np = __popc(mask);
    int at = np;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, at, s);
      if (lane >= s) at += u;
    }
    if (lane == 31) swarp[w] = at;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int k = 0; k < kRPix / 32; ++k) {
      const int c = swarp[k];
      before += (k < w) ? c : 0;
      total += c;
    }
    at += before - np;
    while (mask) {
      const int k = __ffs(mask) - 1;
      mask &= mask - 1;
      queue[at++] = uint16_t((l << 5) | k);
    }
    __syncthreads();
    // FP64 tests on every thread
    for (int qi = l; qi < total; qi += kRPix) {
      const int v = queue[qi];
      const int pl = v >> 5, k = v & 31;
      const double d[3] = {sray[0][pl], sray[1][pl], sray[2][pl]};
      BRec r;
      for (int f = 0; f < 6; ++f) r.ic[f] = sd[f][k];
      for (int f = 0; f < 3; ++f) r.b[f] = sd[6 + f][k];
      r.c = sd[9][k];
      r.op = sd[10][k];
      r.thr = sc[k][0].x;
      double t_star, alpha, a, b;
      if (contribution(r, d, tab, t_star, alpha, a, b)) {
        const int64_t o = sbase[pl] + atomicAdd(&scur[pl], 1);
        REnt e;
        e.t = t_star;
        e.pos = int32_t(b0 - l0) + k;
        e.idx = sidx[k];
        E[o] = e;
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
//
// A pixel's contributions are sorted by keys held in registers: t* > 0, so its bit pattern
// orders like the value, and q = (bits(t*) - lo) >> sh is non-decreasing in t*. The key is
// q above the entry's slot (32 bits: log2(capacity) slot bits, q the rest, sh chosen from
// the slice's span so that it always fits); the order it gives is exact except inside
// runs of equal q (t* within 2^(sh-52) relative, or equal), which one thread per run then
// re-orders by the exact (t*, index) comparison. The bitonic network runs on NT threads x
// E keys in the blocked layout (position i = E tid + e): partners within a warp exchange
// through shuffles, partners in another warp through shared memory, partners in the same
// thread in registers. Only 4 bytes move per key and stage (sorting the 16-byte entries
// themselves was shared-memory-bandwidth bound); the entries are permuted once at the end.
// Measured against the round-1 64-bit keys (exact bit distance << 9, SOF_SORT64 builds
// it): k_rsort 5.1 -> 3.6 ms per C2 view.

__device__ __forceinline__ bool rent_less(const REnt& a, const REnt& b) {
  return a.t < b.t || (a.t == b.t && a.idx < b.idx);
}

__device__ __forceinline__ REnt rent_pad() {
  REnt e;
  e.t = INFINITY;
  e.pos = 0;
  e.idx = INT_MAX;
  return e;
}

// 16-byte moves of an entry (one LDS/STS/LDG/STG.128 each)
__device__ __forceinline__ REnt ld_rent(const REnt* p) {
  const int4 v = *reinterpret_cast<const int4*>(p);
  REnt e;
  e.t = __hiloint2double(v.y, v.x);
  e.pos = v.z;
  e.idx = v.w;
  return e;
}
__device__ __forceinline__ void st_rent(REnt* p, const REnt& e) {
  *reinterpret_cast<int4*>(p) = make_int4(__double2loint(e.t), __double2hiint(e.t), e.pos, e.idx);
}

// Warp-private barrier: a named barrier (bar.sync id, 32) per warp, so the per-pixel loop
// needs no proof of warp convergence (__syncwarp there compiles to the slow collective
// form). NT == 32: warp w's barrier; otherwise the CTA barrier.
template <int NT>
__device__ __forceinline__ void sorter_sync(int w) {
  if (NT == 32) asm volatile("bar.sync %0, 32;" ::"r"(w + 1) : "memory");
  else __syncthreads();
}

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(v), m);
  const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(v >> 32), m);
  return (uint64_t(hi) << 32) | lo;
}

__device__ __forceinline__ uint32_t shfl_xor_key(uint32_t v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
__device__ __forceinline__ uint64_t shfl_xor_key(uint64_t v, int m) { return shfl_xor_u64(v, m); }

// in-thread stage: elements e and e + ES (ES < E, compile time), position i = E tid + e
template <int E, int ES, typename K>
__device__ __forceinline__ void keys_inthread(K (&k)[E], int size, int tid) {
  if constexpr (ES < E) {
#pragma unroll
    for (int e = 0; e < E; ++e)
      if ((e & ES) == 0) {
        const bool asc = ((E * tid + e) & size) == 0;
        const K a = k[e], b = k[e + ES];
        const K lo = min(a, b), hi = max(a, b);  // keys are distinct (equal only as padding)
        k[e] = asc ? lo : hi;
        k[e + ES] = asc ? hi : lo;
      }
  }
}
// compare-exchange of element e with element e of thread tid ^ (stride / E) (stride >= E)
template <int NT, int E, typename K>
__device__ __forceinline__ void bitonic_cross(K (&k)[E], int size, int stride, int tid, int w, K* xb) {
  const int ts = stride / E;  // partner thread distance
  const bool lower = (tid & ts) == 0;
  if (ts < 32) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const K p = shfl_xor_key(k[e], ts);
      const bool take_min = lower == (((E * tid + e) & size) == 0);
      k[e] = take_min ? min(p, k[e]) : max(p, k[e]);  // distinct keys (equal only as padding)
    }
  } else {  // partner thread in another warp: exchange through shared memory
#pragma unroll
    for (int e = 0; e < E; ++e) xb[E * tid + e] = k[e];
    sorter_sync<NT>(w);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const K p = xb[E * (tid ^ ts) + e];
      const bool take_min = lower == (((E * tid + e) & size) == 0);
      k[e] = take_min ? min(p, k[e]) : max(p, k[e]);
    }
    sorter_sync<NT>(w);
  }
}

template <int NT, int E, typename K>
__device__ __forceinline__ void bitonic_stage(K (&k)[E], int size, int stride, int tid, int w, K* xb) {
  if (stride < E) {
    if (stride == 1) keys_inthread<E, 1>(k, size, tid);
    else if (stride == 2) keys_inthread<E, 2>(k, size, tid);
    else if (stride == 4) keys_inthread<E, 4>(k, size, tid);
    else if (stride == 8) keys_inthread<E, 8>(k, size, tid);
  } else {
    bitonic_cross<NT, E>(k, size, stride, tid, w, xb);
  }
}

// Ascending bitonic sort of NT x E keys in the blocked layout (position i = E tid + e):
// strides below E are compare-exchanges inside a thread, larger ones pair element e of
// threads tid and tid ^ (stride / E) — through shuffles inside a warp, through shared
// memory (xb: NT x E keys) across warps. Small strides, the most frequent in the network,
// thus cost no data movement. Networks up to SOF_SORT_UNROLL keys are unrolled completely
// (stage parameters and direction bits become constants).
#ifndef SOF_SORT_UNROLL
#define SOF_SORT_UNROLL 64
#endif
template <int NT, int E, typename K>
__device__ __forceinline__ void sort_keys(K (&k)[E], int tid, int w, K* xb) {
  constexpr int M = NT * E;
  if constexpr (M <= SOF_SORT_UNROLL) {
#pragma unroll
    for (int lg = 1; (1 << lg) <= M; ++lg)
#pragma unroll
      for (int stride = (1 << lg) >> 1; stride > 0; stride >>= 1) bitonic_stage<NT, E>(k, 1 << lg, stride, tid, w, xb);
  } else {
    // sizes up to E: inside the thread, unrolled
#pragma unroll
    for (int lg = 1; (1 << lg) <= E; ++lg)
#pragma unroll
      for (int stride = (1 << lg) >> 1; stride > 0; stride >>= 1) bitonic_stage<NT, E>(k, 1 << lg, stride, tid, w, xb);
    // larger sizes: the partner-thread strides in a loop, then the in-thread tail unrolled
#pragma unroll 1
    for (int size = 2 * E; size <= M; size <<= 1) {
#pragma unroll 1
      for (int stride = size >> 1; stride >= E; stride >>= 1) bitonic_cross<NT, E>(k, size, stride, tid, w, xb);
#pragma unroll
      for (int stride = E >> 1; stride > 0; stride >>= 1) bitonic_stage<NT, E>(k, size, stride, tid, w, xb);
    }
  }
}

// log2 of a power of two, at compile time
constexpr int ilog2c(int m) { return m <= 1 ? 0 : 1 + ilog2c(m >> 1); }

// Sorts S[0, n) (n <= NT E) in place by (t*, index). buf: NT E x 16 B of shared memory.
// The sort key is the entry's slot below a monotone image of t*: t* > 0, so its bit
// pattern orders like the value, and q = (bits - min bits) >> sh is non-decreasing in t*.
// K = uint32_t (SORT32, the default): slot bits = log2(NT E), q takes the rest and sh is
// whatever makes the slice's span fit — never fails; entries with equal q (t* within
// 2^(sh-52) relative of each other, or equal) are put in exact (t*, index) order
// afterwards, each run of equal q by its own thread. K = uint64_t: sh = 0 (q is the exact
// bit distance, equal q only for equal t*); returns false (nothing changed) when the t*
// span does not fit the key.
template <int NT, int E, typename K>
__device__ __forceinline__ bool sort_slice_keys(REnt* __restrict__ S, int n, int tid, int w, void* buf,
                                                uint64_t* red) {
  constexpr int M = NT * E;
  static_assert(M <= 4096, "slot bits");
  constexpr bool k32 = sizeof(K) == 4;
  constexpr int SB = k32 ? ilog2c(M) : ((M <= 512) ? 9 : 12);  // slot bits
  static_assert(!k32 || (1 << SB) == M, "power-of-two slice capacity");
  constexpr int QB = 8 * int(sizeof(K)) - SB;  // bits of q
  constexpr K kLow = (K(1) << SB) - 1;
  uint64_t tb[E];
  uint64_t lo = ~uint64_t(0), hi = 0;
  int sh = 0;
  if constexpr (k32) {
    // the span only sets the shift: reduce the high words (one REDUX each) and take
    // lo = (min high word) << 32, which only coarsens q by at most one bit
    uint32_t lw = ~0u, hw = 0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = E * tid + e;
      tb[e] = (i < n) ? uint64_t(__double_as_longlong(S[i].t)) : 0;
      if (i < n) {
        lw = min(lw, uint32_t(tb[e] >> 32));
        hw = max(hw, uint32_t(tb[e] >> 32));
      }
    }
    lw = __reduce_min_sync(0xffffffffu, lw);
    hw = __reduce_max_sync(0xffffffffu, hw);
    if (NT > 32) {  // across the warps of the CTA
      if ((tid & 31) == 0) {
        red[2 * (tid >> 5)] = lw;
        red[2 * (tid >> 5) + 1] = hw;
      }
      __syncthreads();
      for (int k = 0; k < NT / 32; ++k) {
        lw = min(lw, uint32_t(red[2 * k]));
        hw = max(hw, uint32_t(red[2 * k + 1]));
      }
      __syncthreads();
    }
    lo = uint64_t(lw) << 32;
    const uint64_t span = ((uint64_t(hw) << 32) | 0xffffffffu) - lo;
    const int need = 64 - __clzll((long long)span);  // bits of the span
    sh = need > QB ? need - QB : 0;
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = E * tid + e;
      tb[e] = (i < n) ? uint64_t(__double_as_longlong(S[i].t)) : 0;
      if (i < n) {
        lo = min(lo, tb[e]);
        hi = max(hi, tb[e]);
      }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      lo = min(lo, shfl_xor_u64(lo, s));
      hi = max(hi, shfl_xor_u64(hi, s));
    }
    if (NT > 32) {  // across the warps of the CTA
      if ((tid & 31) == 0) {
        red[2 * (tid >> 5)] = lo;
        red[2 * (tid >> 5) + 1] = hi;
      }
      __syncthreads();
      for (int k = 0; k < NT / 32; ++k) {
        lo = min(lo, red[2 * k]);
        hi = max(hi, red[2 * k + 1]);
      }
      __syncthreads();
    }
    if (hi - lo >= (uint64_t(1) << QB)) return false;
  }
  K k[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = E * tid + e;
    k[e] = (i < n) ? ((K((tb[e] - lo) >> sh) << SB) | K(i)) : ~K(0);
  }
  K* xb = static_cast<K*>(buf);
  sort_keys<NT, E>(k, tid, w, xb);
  // runs of equal q at neighbouring positions: exact (t*, index) order inside each run.
  // The runs are found first (every key read before any is moved; run ends kept in
  // registers), then each is insertion-sorted by the thread holding its first position.
#pragma unroll
  for (int e = 0; e < E; ++e) xb[E * tid + e] = k[e];
  sorter_sync<NT>(w);
  bool tie = false;
  int rend[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = E * tid + e;
    rend[e] = -1;
    if (i + 1 < n && (xb[i] >> SB) == (xb[i + 1] >> SB) && (i == 0 || (xb[i - 1] >> SB) != (xb[i] >> SB))) {
      const K q = xb[i] >> SB;
      int end = i + 2;
      while (end < n && (xb[end] >> SB) == q) ++end;
      rend[e] = end;
      tie = true;
    }
  }
  const bool any_tie = (NT == 32) ? __any_sync(0xffffffffu, tie) : __syncthreads_or(tie);
  if (any_tie) {
    sorter_sync<NT>(w);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = E * tid + e;
      for (int a = i + 1; a < rend[e]; ++a) {  // rend < 0: not a run start
        const K v = xb[a];
        const REnt ev = ld_rent(S + (v & kLow));
        int j = a - 1;
        while (j >= i && rent_less(ev, ld_rent(S + (xb[j] & kLow)))) {
          xb[j + 1] = xb[j];
          --j;
        }
        xb[j + 1] = v;
      }
    }
    sorter_sync<NT>(w);
#pragma unroll
    for (int e = 0; e < E; ++e) k[e] = xb[E * tid + e];
  }
  sorter_sync<NT>(w);
  // permute the entries through shared memory
  REnt* stage = static_cast<REnt*>(buf);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = E * tid + e;
    if (i < n) st_rent(stage + i, ld_rent(S + (k[e] & kLow)));
  }
  sorter_sync<NT>(w);
  for (int i = tid; i < n; i += NT) st_rent(S + i, ld_rent(stage + i));  // coalesced
  sorter_sync<NT>(w);
  return true;
}

#ifndef SOF_SORT64
using SortKey = uint32_t;
#else
using SortKey = uint64_t;
#endif

__device__ __forceinline__ void swap_rent(REnt* S, int64_t a, int64_t b) {
  const REnt t = ld_rent(S + a);
  st_rent(S + a, ld_rent(S + b));
  st_rent(S + b, t);
}

// Exact fallback for one CTA (any n): the flip-bitonic network directly on the entries in
// global memory (positions >= n act as +inf: compare-exchanges touching them are no-ops).
__device__ void sort_slice_global(REnt* S, int64_t n) {
  int64_t m = 1;
  while (m < n) m <<= 1;
  for (int64_t size = 2; size <= m; size <<= 1) {
    const int64_t h = size >> 1;
    for (int64_t i = threadIdx.x; i < (m >> 1); i += blockDim.x) {
      const int64_t lo = (i / h) * size + (i % h), hi = (i / h) * size + size - 1 - (i % h);
      if (hi < n && rent_less(ld_rent(S + hi), ld_rent(S + lo))) swap_rent(S, lo, hi);
    }
    __syncthreads();
    for (int64_t stride = size >> 2; stride > 0; stride >>= 1) {
      for (int64_t i = threadIdx.x; i < (m >> 1); i += blockDim.x) {
        const int64_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        if (hi < n && rent_less(ld_rent(S + hi), ld_rent(S + lo))) swap_rent(S, lo, hi);
      }
      __syncthreads();
    }
  }
}

constexpr int kWarpSortCap = 256;   // one warp: 8 keys per lane, 4 KB of shared memory
constexpr int kCtaSortCap = 4096;   // one CTA of 256: 16 keys per thread, 64 KB

// One warp per pixel (grid-stride over the band's pixels), 8 warps per CTA.
#ifndef SOF_RSORT_MINB
#define SOF_RSORT_MINB 4
#endif
__global__ void __launch_bounds__(kSortWarps * 32, SOF_RSORT_MINB) k_rsort(int64_t q0, int64_t nq, const int64_t* __restrict__ poff,
                                                             int64_t base, const uint32_t* __restrict__ ncon, REnt* E,
                                                             int32_t* big, int32_t* big_cnt) {
  __shared__ __align__(16) REnt sbuf[kSortWarps][kWarpSortCap];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t step = int64_t(gridDim.x) * kSortWarps;
  int64_t qq = int64_t(blockIdx.x) * kSortWarps + w;
  int n = (qq < nq) ? int(ncon[q0 + qq]) : 0;
  int64_t o = (qq < nq) ? poff[q0 + qq] : 0;
  for (; qq < nq; qq += step) {
    const int64_t q = q0 + qq;
    const int cn = n;
    REnt* S = E + (o - base);
    if (qq + step < nq) {  // the next pixel's count and offset, in flight during this sort
      n = int(ncon[q + step]);
      o = poff[q + step];
    }
    if (cn <= 1) continue;
    bool done = false;
    if (cn <= 32) done = sort_slice_keys<32, 1, SortKey>(S, cn, lane, w, sbuf[w], nullptr);
    else if (cn <= 64) done = sort_slice_keys<32, 2, SortKey>(S, cn, lane, w, sbuf[w], nullptr);
    else if (cn <= 128) done = sort_slice_keys<32, 4, SortKey>(S, cn, lane, w, sbuf[w], nullptr);
    else if (cn <= 256) done = sort_slice_keys<32, 8, SortKey>(S, cn, lane, w, sbuf[w], nullptr);
    if (!done && lane == 0) {  // longer slices (or, SOF_SORT64 only, a t* span past the 55-bit key)
      big[atomicAdd(big_cnt, 1)] = int32_t(q);
      atomicAdd(big_cnt + 1, 1);  // frame total (stats)
    }
  }
}

// The queued slices up to 512 entries (SOF_SORT64: or with a t* span past the warp sort's key): one
// warp per pixel with 8 KB of shared memory; longer ones go to the CTA sort.
__global__ void __launch_bounds__(kSortWarps * 32) k_rsort_mid(const int64_t* __restrict__ poff, int64_t base,
                                                               const uint32_t* __restrict__ ncon, REnt* E,
                                                               const int32_t* __restrict__ big,
                                                               const int32_t* __restrict__ big_cnt, int32_t* huge,
                                                               int32_t* huge_cnt) {
  extern __shared__ __align__(16) unsigned char sdyn[];  // kSortWarps x 512 x 16 B
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = *big_cnt;
  for (int bi = blockIdx.x * kSortWarps + w; bi < nb; bi += gridDim.x * kSortWarps) {
    const int64_t q = big[bi];
    const int n = int(ncon[q]);
    REnt* S = E + (poff[q] - base);
    const bool done = (n <= 512) && sort_slice_keys<32, 16, SortKey>(S, n, lane, w, sdyn + w * 512 * 16, nullptr);
    if (!done && lane == 0) huge[atomicAdd(huge_cnt, 1)] = int32_t(q);
  }
}

// Slices past 512 entries (rare): one CTA of 256 per pixel.
__global__ void __launch_bounds__(256) k_rsort_big(const int64_t* __restrict__ poff, int64_t base,
                                                   const uint32_t* __restrict__ ncon, REnt* E,
                                                   const int32_t* __restrict__ big, const int32_t* __restrict__ big_cnt) {
  extern __shared__ __align__(16) unsigned char sdyn[];  // kCtaSortCap x 16 B
  __shared__ uint64_t red[16];
  const int nb = *big_cnt;
  for (int bi = blockIdx.x; bi < nb; bi += gridDim.x) {
    const int64_t q = big[bi];
    const int64_t n = ncon[q];
    REnt* S = E + (poff[q] - base);
    bool done = false;
    const int t = threadIdx.x;
    if (n <= 1024) done = sort_slice_keys<256, 4, SortKey>(S, int(n), t, 0, sdyn, red);
    else if (n <= 4096) done = sort_slice_keys<256, 16, SortKey>(S, int(n), t, 0, sdyn, red);
    if (!done) sort_slice_global(S, n);
    __syncthreads();
  }
}

// ---- R4: blend, depth, opacity at depth --------------------------------------------------------------

struct RenderOut {
  double* depth;
  double* opacity;
  double* rgb;
  double* tfinal;
};


#ifndef SOF_BLEND_CAP
#define SOF_BLEND_CAP 640
#endif
#ifndef SOF_BLEND_MINB
#define SOF_BLEND_MINB 1
#endif
#ifndef SOF_BLEND_BATCH
#define SOF_BLEND_BATCH 4
#endif
constexpr int kBlendBatch = SOF_BLEND_BATCH;  // entries loaded per group (one memory latency each)
constexpr int kBlendCap = SOF_BLEND_CAP;  // records staged per tile (74 KB); later list positions read global memory
constexpr int kBlendSmem = kBlendCap * (14 * 8 + 4);

__device__ __forceinline__ BRec brec_global(const RRec* __restrict__ recs, const double* __restrict__ dc, int g) {
  const double2* r = reinterpret_cast<const double2*>(recs + g);
  BRec o;
  double2 v = __ldg(r + 0);
  o.ic[0] = v.x, o.ic[1] = v.y;
  v = __ldg(r + 1);
  o.ic[2] = v.x, o.ic[3] = v.y;
  v = __ldg(r + 2);
  o.ic[4] = v.x, o.ic[5] = v.y;
  v = __ldg(r + 3);
  o.b[0] = v.x, o.b[1] = v.y;
  v = __ldg(r + 4);
  o.b[2] = v.x, o.c = v.y;
  v = __ldg(r + 5);
  o.op = v.x;
  o.thr = __ldg(&recs[g].thr);
  for (int k = 0; k < 3; ++k) o.dc[k] = __ldg(dc + 3 * g + k);
  return o;
}

// staged columns of field pairs: sd[f * kBlendCap + pos] as double2, f = (ic0, ic1),
// (ic2, ic3), (ic4, ic5), (b0, b1), (b2, c), (op, dc0), (dc1, dc2): one 16-byte shared
// load per pair (lanes read different records: the per-lane reads of a column are
// consecutive-stride words, and half the load instructions of single-field columns)
constexpr int kBlendF = 14;
__device__ __forceinline__ BRec brec_smem(const double2* sd, const float* thr, int pos) {
  BRec o;
  double2 v = sd[0 * kBlendCap + pos];
  o.ic[0] = v.x, o.ic[1] = v.y;
  v = sd[1 * kBlendCap + pos];
  o.ic[2] = v.x, o.ic[3] = v.y;
  v = sd[2 * kBlendCap + pos];
  o.ic[4] = v.x, o.ic[5] = v.y;
  v = sd[3 * kBlendCap + pos];
  o.b[0] = v.x, o.b[1] = v.y;
  v = sd[4 * kBlendCap + pos];
  o.b[2] = v.x, o.c = v.y;
  v = sd[5 * kBlendCap + pos];
  o.op = v.x, o.dc[0] = v.y;
  v = sd[6 * kBlendCap + pos];
  o.dc[1] = v.x, o.dc[2] = v.y;
  o.thr = thr[pos];
  return o;
}

// A, B of abc_cached (precompute.hpp:39-45) for the record and the pixel ray
__device__ __forceinline__ void rec_ab(const BRec& r, const double* d, double& a, double& b) {
  const double x = d[0], y = d[1], z = d[2];
  a = r.ic[0] * x * x + r.ic[3] * y * y + r.ic[5] * z * z + 2.0 * (r.ic[1] * x * y + r.ic[2] * x * z + r.ic[4] * y * z);
  b = 2.0 * (x * r.b[0] + y * r.b[1] + z * r.b[2]);
}

// alpha_at(rc, depth) (opacity_field.hpp:95-101) for a contribution whose A, B are known
template <typename Tab>
__device__ __forceinline__ double alpha_at_depth(const BRec& r, double a, double b, double ts, double depth, Tab tab) {
  const double te = (depth < ts) ? depth : ts;  // std::min(t*, t)
  if (!(te > 0.0)) return 0.0;
  const double arg = -0.5 * ((a * te + b) * te + r.c);  // eval_1d gaussian.hpp:47-49
  if (arg < double(r.thr)) return 0.0;                   // alpha < 1/255 certain
  const double al = r.op * exp_any(arg, tab);
  if (al < kMinAlpha) return 0.0;
  return (kMaxAlpha < al) ? kMaxAlpha : al;
}

// One thread per pixel over its sorted slice; the tile list's records (up to kBlendCap)
// staged in shared memory and addressed by the entry's list position. The contribution's
// A, B and alpha are recomputed with the exact expressions R2 used. Phase A blends
// (render_pixel :204-210) up to the median (find_median :129-141); phase B fixes the
// depth (exact_depth :157-166) and takes the opacity product of opacity_along_ray
// (:104-108) over the prefix up to the median; phase C blends the rest and extends the
// product in the same pass. Lanes leave phase A at different entries, but every phase is
// one loop per lane, so the warp never serialises one lane's prefix after another's.
__global__ void __launch_bounds__(kRPix, SOF_BLEND_MINB) k_rblend(Cam cam, int tiles_x, int tile0, const int64_t* __restrict__ toff,
                                                  const int32_t* __restrict__ ent, const int64_t* __restrict__ poff,
                                                  int64_t base, const uint32_t* __restrict__ ncon,
                                                  const REnt* __restrict__ E, const RRec* __restrict__ recs,
                                                  const double* __restrict__ dc, int exact_depth, RenderOut out,
                                                  unsigned long long* stats) {
  extern __shared__ __align__(16) unsigned char sdyn[];
  double2* scol = reinterpret_cast<double2*>(sdyn);                         // [kBlendF / 2][kBlendCap]
  float* sthr = reinterpret_cast<float*>(scol + (kBlendF / 2) * kBlendCap);  // [kBlendCap]
  __shared__ __align__(16) double s_exp[128];
  const int tile = tile0 + int(blockIdx.x), l = threadIdx.x;
  for (int k = l; k < 128; k += blockDim.x) s_exp[k] = kSofExpTabDev[k];
  const int64_t l0 = toff[tile];
  const int len = int(min(int64_t(kBlendCap), toff[tile + 1] - l0));
  for (int k = l; k < len * 8; k += kRPix) {
    const int r = k >> 3, qq = k & 7;
    const int32_t g = ent[l0 + r];
    if (qq < 5) {
      const double2 v = __ldg(reinterpret_cast<const double2*>(recs + g) + qq);
      scol[qq * kBlendCap + r] = v;
    } else if (qq == 5) {
      scol[5 * kBlendCap + r].x = __ldg(&recs[g].op);
      sthr[r] = __ldg(&recs[g].thr);
    } else if (qq == 6) {
      scol[5 * kBlendCap + r].y = __ldg(dc + 3 * g);
      scol[6 * kBlendCap + r].x = __ldg(dc + 3 * g + 1);
    } else {
      scol[6 * kBlendCap + r].y = __ldg(dc + 3 * g + 2);
    }
  }
  __syncthreads();
  const SofExpSmem tab{smem_u32(s_exp)};
  int x, y;
  tile_pixel(tile, tiles_x, l, x, y);
  if (!(x < cam.w && y < cam.h)) return;
  const int64_t q = int64_t(tile) * kRPix + l;
  const int n = int(ncon[q]);
  const REnt* __restrict__ S = E + (poff[q] - base);
  double d[3];
  pixel_ray(cam, x, y, d);
  auto rec = [&](const REnt& e) { return (e.pos < kBlendCap) ? brec_smem(scol, sthr, e.pos) : brec_global(recs, dc, e.idx); };
  double T = 1.0, col[3] = {0.0, 0.0, 0.0};
  auto blend = [&](const BRec& r, double& a, double& b) {
    rec_ab(r, d, a, b);
    const double arg = -0.5 * (r.c - b * b / (4.0 * a));  // peak_value gaussian.hpp:54-56
    const double al = r.op * exp_any(arg, tab);
    const double alpha = (kMaxAlpha < al) ? kMaxAlpha : al;
    for (int k = 0; k < 3; ++k) col[k] = col[k] + r.dc[k] * alpha * T;
    return alpha;
  };
  // phase A (entries fetched four at a time: one memory latency per group)
  int j = 0, med = -1;
  double med_T = 1.0, ma = 0.0, mb = 0.0, mc = 0.0, mop = 0.0;
  while (j < n && med < 0) {
    REnt g[kBlendBatch];
#pragma unroll
    for (int u = 0; u < kBlendBatch; ++u) g[u] = (j + u < n) ? ld_rent(S + j + u) : rent_pad();
#pragma unroll
    for (int u = 0; u < kBlendBatch; ++u) {
      if (med < 0 && j < n) {
        const BRec r = rec(g[u]);
        double a, b;
        const double alpha = blend(r, a, b);
        const double next = T * (1.0 - alpha);
        if (T > 0.5 && next < 0.5) {
          med = j;
          med_T = T;
          ma = a;
          mb = b;
          mc = r.c;
          mop = r.op;
        }
        T = next;
        ++j;
      }
    }
  }
  // phase B
  double depth = NAN, T2 = 1.0;
  if (med >= 0) {
    const double mt = S[med].t;
    depth = mt;         // median_depth (:143-147)
    if (exact_depth) {  // exact_depth (:157-166)
      const double lt = 2.0 * sof_log((med_T - 0.5) / (med_T * mop));
      const double disc = mb * mb - 4.0 * ma * (mc + lt);
      if (disc < 0.0) {
        atomicAdd(stats + 3, 1ull);
      } else {
        depth = mt - sqrt(disc) / (2.0 * ma);
      }
    }
    for (int i = 0; i <= med; i += kBlendBatch) {
      REnt g[kBlendBatch];
#pragma unroll
      for (int u = 0; u < kBlendBatch; ++u) g[u] = (i + u <= med) ? ld_rent(S + i + u) : rent_pad();
#pragma unroll
      for (int u = 0; u < kBlendBatch; ++u)
        if (i + u <= med) {
          const BRec r = rec(g[u]);
          double a, b;
          rec_ab(r, d, a, b);
          T2 *= 1.0 - alpha_at_depth(r, a, b, g[u].t, depth, tab);
        }
    }
  }
  // phase C
  while (j < n) {
    REnt g[kBlendBatch];
#pragma unroll
    for (int u = 0; u < kBlendBatch; ++u) g[u] = (j + u < n) ? ld_rent(S + j + u) : rent_pad();
#pragma unroll
    for (int u = 0; u < kBlendBatch; ++u) {
      if (j < n) {
        const BRec r = rec(g[u]);
        double a, b;
        const double alpha = blend(r, a, b);
        if (med >= 0) T2 *= 1.0 - alpha_at_depth(r, a, b, g[u].t, depth, tab);
        T = T * (1.0 - alpha);
        ++j;
      }
    }
  }
  const int64_t p = int64_t(y) * cam.w + x;
  out.depth[p] = depth;
  out.opacity[p] = (med >= 0 && !isnan(depth)) ? 1.0 - T2 : 0.0;  // accumulated opacity (:216-217)
  for (int k = 0; k < 3; ++k) out.rgb[3 * p + k] = col[k];
  out.tfinal[p] = T;
}

// slice offset of every tile's first pixel (band planning)
__global__ void k_tile_slice_off(int64_t T, const int64_t* __restrict__ poff, int64_t* out) {
  const int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (t <= T) out[t] = poff[t * kRPix];
}

// per-pixel contribution counts of the last render, image order (diagnostics / tests)
__global__ void k_rcounts_image(Cam cam, int tiles_x, int64_t Q, const uint32_t* __restrict__ ncon, uint32_t* out) {
  const int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (q >= Q) return;
  int x, y;
  tile_pixel(int(q / kRPix), tiles_x, int(q % kRPix), x, y);
  if (x < cam.w && y < cam.h) out[int64_t(y) * cam.w + x] = ncon[q];
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


// ---- the K-window resort mode and the per-ray API ---------------------------------------------

// view-space centre depth cam.to_view(mu).z() (camera.hpp:19, Eigen sums left to right):
// the arrival order of the window mode
__global__ void k_center_depth(int64_t n, const GaussStatic* __restrict__ g, Cam cam, double* zc) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const double* x = g[i].pos;
  zc[i] = ((cam.R[6] * x[0] + cam.R[7] * x[1]) + cam.R[8] * x[2]) + cam.t[2];
}

// One thread per pixel: the slice (any order after R2) goes into arrival order -- centre
// depth, ties by index, a strict total order -- then through windowed_resort's K-slot
// window (stl_order.cuh) into A. Serial per pixel: this mode trades the exact sort's
// warp-parallel network for the reference's streaming window semantics.
__global__ void __launch_bounds__(128) k_rwindow(int64_t q0, int64_t nq, const int64_t* __restrict__ poff,
                                                 int64_t base, const uint32_t* __restrict__ ncon, REnt* E, REnt* A,
                                                 const double* __restrict__ zc, int64_t window) {
  const int64_t qq = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (qq >= nq) return;
  const int64_t q = q0 + qq;
  const int64_t n = ncon[q];
  REnt* S = E + (poff[q] - base);
  REnt* O = A + (poff[q] - base);
  stlo::sort(S, n, [zc](const REnt& a, const REnt& b) {
    const double za = __ldg(zc + a.idx), zb = __ldg(zc + b.idx);
    return za < zb || (za == zb && a.idx < b.idx);
  });
  stlo::windowed_resort(S, O, n, window, [](const REnt& a, const REnt& b) { return a.t < b.t; });
}

// collect_contributions over ALL Gaussians for each ray (grid.y strides the rays): PASS 0
// counts per ray, PASS 1 scatters REnt{t*, 0, index} into the ray's slice (any order;
// the exact sort follows).
template <int PASS>
__global__ void __launch_bounds__(256) k_ct_scan(int64_t n, const Rec* __restrict__ rec, int64_t nr,
                                                 const double* __restrict__ dirs, uint32_t* cnt,
                                                 const int64_t* __restrict__ off, REnt* E) {
  const int lane = threadIdx.x & 31;
  const double* tab = kSofExpTabDev;
  for (int64_t r = blockIdx.y; r < nr; r += gridDim.y) {
    const double d[3] = {dirs[3 * r], dirs[3 * r + 1], dirs[3 * r + 2]};
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    for (int64_t g0 = int64_t(blockIdx.x) * blockDim.x; g0 < n; g0 += stride) {
      const int64_t g = g0 + threadIdx.x;
      double t = 0.0, alpha, a, b;
      const bool hit = g < n && contribution(rec[g], d, tab, t, alpha, a, b);
      const unsigned m = __ballot_sync(0xffffffffu, hit);
      if (!m) continue;
      const int leader = __ffs(m) - 1;
      uint32_t slot = 0;
      if (lane == leader) slot = atomicAdd(cnt + r, uint32_t(__popc(m)));
      slot = __shfl_sync(0xffffffffu, slot, leader) + __popc(m & ((1u << lane) - 1u));
      if (PASS == 1 && hit) {
        REnt e;
        e.t = t;
        e.pos = 0;
        e.idx = int32_t(g);
        st_rent(E + off[r] + slot, e);
      }
    }
  }
}

// RayContribution fields of every sorted entry (the expressions of the scan, recomputed)
__global__ void k_ct_values(int64_t C, int64_t nr, const int64_t* __restrict__ off, const REnt* __restrict__ E,
                            const Rec* __restrict__ rec, const double* __restrict__ dirs, int32_t* idx, double* val) {
  const int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (k >= C) return;
  int64_t lo = 0, hi = nr;  // the ray: last r with off[r] <= k
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (off[mid] <= k) lo = mid;
    else hi = mid;
  }
  const REnt e = ld_rent(E + k);
  const double d[3] = {dirs[3 * lo], dirs[3 * lo + 1], dirs[3 * lo + 2]};
  double t = 0.0, alpha = 0.0, a = 0.0, b = 0.0;
  contribution(rec[e.idx], d, kSofExpTabDev, t, alpha, a, b);
  idx[k] = e.idx;
  double* v = val + 6 * k;
  v[0] = t;
  v[1] = alpha;
  v[2] = a;
  v[3] = b;
  v[4] = rec[e.idx].c;
  v[5] = rec[e.idx].op;
}

// windowed_resort of independent lists, one thread per list
__global__ void k_wresort(int64_t nl, const int64_t* __restrict__ off, const double* __restrict__ t, int64_t window,
                          REnt* S, REnt* O, int64_t* order) {
  const int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (l >= nl) return;
  const int64_t b = off[l], n = off[l + 1] - b;
  for (int64_t k = 0; k < n; ++k) {
    REnt e;
    e.t = t[b + k];
    e.pos = int32_t(k);
    e.idx = 0;
    S[b + k] = e;
  }
  stlo::windowed_resort(S + b, O + b, n, window, [](const REnt& x, const REnt& y) { return x.t < y.t; });
  for (int64_t k = 0; k < n; ++k) order[b + k] = b + O[b + k].pos;
}

// render_pixel (opacity_field.hpp:201-219) of given lists, one thread per list
__global__ void k_rpixel(int64_t nl, const int64_t* __restrict__ off, const int32_t* __restrict__ idx,
                         const double* __restrict__ val, const double* __restrict__ dc, int exact, double* color,
                         double* depth_out, double* acc, double* tfinal) {
  const int64_t l = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (l >= nl) return;
  const int64_t b = off[l], e = off[l + 1];
  double T = 1.0, col[3] = {0.0, 0.0, 0.0}, med_T = 1.0;
  int64_t med = -1;
  for (int64_t k = b; k < e; ++k) {
    const double alpha = val[6 * k + 1];
    const int64_t g = idx[k];
    for (int c = 0; c < 3; ++c) col[c] = col[c] + dc[3 * g + c] * alpha * T;  // :207
    const double next = T * (1.0 - alpha);
    if (med < 0 && T > 0.5 && next < 0.5) {  // find_median :132-141
      med = k;
      med_T = T;
    }
    T = next;
  }
  double depth = NAN;
  if (med >= 0) {
    const double* m = val + 6 * med;
    depth = m[0];  // median_depth :143-147
    if (exact) {   // exact_depth :157-166
      const double lt = 2.0 * sof_log((med_T - 0.5) / (med_T * m[5]));
      const double disc = m[3] * m[3] - 4.0 * m[2] * (m[4] + lt);
      if (!(disc < 0.0)) depth = m[0] - sqrt(disc) / (2.0 * m[2]);
    }
  }
  double o = 0.0;
  if (!isnan(depth)) {  // opacity_along_ray(contribs, depth) :104-108
    double T2 = 1.0;
    for (int64_t k = b; k < e; ++k) {
      const double* v = val + 6 * k;
      const double te = (depth < v[0]) ? depth : v[0];
      double al = 0.0;
      if (!(te <= 0.0)) {
        al = v[5] * exp_any(-0.5 * ((v[2] * te + v[3]) * te + v[4]), kSofExpTabDev);  // alpha_at :95-101
        if (al < kMinAlpha) al = 0.0;
        else if (kMaxAlpha < al) al = kMaxAlpha;
      }
      T2 *= 1.0 - al;
    }
    o = 1.0 - T2;
  }
  if (color)
    for (int c = 0; c < 3; ++c) color[3 * l + c] = col[c];
  if (depth_out) depth_out[l] = depth;
  if (acc) acc[l] = o;
  if (tfinal) tfinal[l] = T;
}

}  // namespace sofk

using namespace sofk;

namespace {
void render_attrs(sof_ctx* c) {
  if (c->rs.attr_set) return;  // the sorts' and the blend's dynamic shared memory (per device)
  SOF_CUDA(cudaFuncSetAttribute(k_rsort_big, cudaFuncAttributeMaxDynamicSharedMemorySize, kCtaSortCap * 16));
  SOF_CUDA(cudaFuncSetAttribute(k_rsort_mid, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortWarps * 512 * 16));
  SOF_CUDA(cudaFuncSetAttribute(k_rblend, cudaFuncAttributeMaxDynamicSharedMemorySize, kBlendSmem));
  c->rs.attr_set = true;
}

// the exact (t*, index) sort of nq slices [poff[q0 + i] - base, +ncon) of E (R3)
void sort_slices(sof_ctx* c, int64_t q0, int64_t nq, const int64_t* poff, int64_t base, const uint32_t* ncon, REnt* E) {
  RenderScratch& rs = c->rs;
  cudaStream_t st = c->stream;
  rs.big.ensure(std::max<int64_t>(int64_t(rs.big.n), 2 * nq));
  rs.big_cnt.ensure(4);
  SOF_CUDA(cudaMemsetAsync(rs.big_cnt.p + 1, 0, sizeof(int32_t), st));
  SOF_CUDA(cudaMemsetAsync(rs.big_cnt.p + 3, 0, sizeof(int32_t), st));
  const unsigned sort_grid = unsigned(std::max<int64_t>(1, std::min<int64_t>((nq + kSortWarps - 1) / kSortWarps, 148 * 8)));
  int32_t* qmid = rs.big.p;  // rs.big[0, n) served the binning; reused for the sort queues
  int32_t* qhuge = rs.big.p + nq;
  k_rsort<<<sort_grid, kSortWarps * 32, 0, st>>>(q0, nq, poff, base, ncon, E, qmid, rs.big_cnt.p + 1);
#ifndef SOF_MID_CTAS
#define SOF_MID_CTAS 3
#endif
  k_rsort_mid<<<148 * SOF_MID_CTAS, kSortWarps * 32, kSortWarps * 512 * 16, st>>>(poff, base, ncon, E, qmid, rs.big_cnt.p + 1,
                                                                      qhuge, rs.big_cnt.p + 3);
  k_rsort_big<<<148, 256, kCtaSortCap * 16, st>>>(poff, base, ncon, E, qhuge, rs.big_cnt.p + 3);
  c->launches += 3;
  SOF_CUDA(cudaGetLastError());
}
}  // namespace

extern "C" int sof_set_render_window(sof_ctx* c, int64_t window) {
  if (!c || window < 0) return SOF_E_INVALID;
  c->r_window = window;
  return SOF_OK;
}

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
    render_attrs(c);
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
    rs.big.ensure(std::max<int64_t>(n, 2 * Q));
    if (n > 0) {
      rs.rect.ensure(n);
      rs.gcnt.ensure(n);
      k_rrec<<<grid_for(n, 128), 128, 0, st>>>(n, c->gstat.p, cam, rec);
      rs.tmask.ensure(n);
      k_rrect<<<grid_for(n, 128), 128, 0, st>>>(n, c->gstat.p, rec, cam, tiles_x, tiles_y, rs.rect.p, rs.gcnt.p,
                                                rs.tmask.p);
      c->launches += 1;
      k_rbin<0><<<grid_for(n, 256), 256, 0, st>>>(n, rs.rect.p, rs.gcnt.p, tiles_x, rs.tile_cnt.p, nullptr, nullptr,
                                                   rs.big.p, rs.big_cnt.p, rs.tmask.p);
      k_rbin_big<0><<<2 * 148, 256, 0, st>>>(rs.rect.p, tiles_x, rs.tile_cnt.p, nullptr, nullptr, rs.big.p,
                                              rs.big_cnt.p, rec);
      c->launches += 3;
      SOF_CUDA(cudaGetLastError());
    }
    scan_u32_i64(c, rs.tile_cnt.p, rs.tile_off.p, T);
    const int64_t M = read_scalar(c, rs.tile_off.p + T);
    rs.ent.ensure(std::max<int64_t>(M, 1));
    if (M > 0) {
      SOF_CUDA(cudaMemsetAsync(rs.tile_cnt.p, 0, sizeof(uint32_t) * T, st));
      k_rbin<1><<<grid_for(n, 256), 256, 0, st>>>(n, rs.rect.p, rs.gcnt.p, tiles_x, rs.tile_cnt.p, rs.tile_off.p,
                                                   rs.ent.p, rs.big.p, rs.big_cnt.p, rs.tmask.p);
      k_rbin_big<1><<<2 * 148, 256, 0, st>>>(rs.rect.p, tiles_x, rs.tile_cnt.p, rs.tile_off.p, rs.ent.p, rs.big.p,
                                              rs.big_cnt.p, rec);
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
    // bands of tiles whose slices fit the scratch budget (two slice buffers in window mode)
    const int64_t window = c->r_window;
    const int64_t cap = std::max<int64_t>(c->render_pool / (window > 0 ? 2 * kEntryBytes : kEntryBytes), 1);
    if (window > 0 && n > 0) {
      rs.zc.ensure(n);
      k_center_depth<<<grid_for(n, 256), 256, 0, st>>>(n, c->gstat.p, cam, rs.zc.p);
      SOF_LAUNCHED(c);
    }
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
      rs.ent16.ensure(ne * sizeof(REnt));
      REnt* E = reinterpret_cast<REnt*>(rs.ent16.p);
      const unsigned nt = unsigned(t1 - t0);
      k_rtest<<<nt, kRPix, 0, st>>>(cam, tiles_x, int(t0), rs.tile_off.p, rs.ent.p, rec, rs.poff.p, e0, E,
                                    rs.ncon.p, c->r_stats.p);
      SOF_LAUNCHED(c);
      const int64_t nq = int64_t(nt) * kRPix;
      const REnt* B = E;
      if (window > 0) {
        rs.ent16b.ensure(ne * sizeof(REnt));
        REnt* A = reinterpret_cast<REnt*>(rs.ent16b.p);
        k_rwindow<<<grid_for(nq, 128), 128, 0, st>>>(t0 * kRPix, nq, rs.poff.p, e0, rs.ncon.p, E, A, rs.zc.p, window);
        SOF_LAUNCHED(c);
        B = A;
      } else {
        sort_slices(c, t0 * kRPix, nq, rs.poff.p, e0, rs.ncon.p, E);  // k_rsort counts big_cnt[2] per frame
      }
      k_rblend<<<nt, kRPix, kBlendSmem, st>>>(cam, tiles_x, int(t0), rs.tile_off.p, rs.ent.p, rs.poff.p, e0,
                                               rs.ncon.p, B, rec, c->dc.p, depth_mode == SOF_DEPTH_EXACT, out,
                                               c->r_stats.p);
      SOF_LAUNCHED(c);
      SOF_CUDA(cudaGetLastError());
      ++nbands;
      t0 = t1;
    }
    c->r_view = view;
    c->r_bands = nbands;
    c->r_Q = Q;
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
      stats[2] = uint64_t(nbig);  // pixels whose slice took the CTA-wide sort (> kWarpSortCap contributions)
      stats[3] = h[3];  // exact-depth fallbacks (negative discriminant)
    }
    SOF_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int sof_render_views(sof_ctx* c, int first_view, int n_views, int depth_mode, double* rgb, double* depth,
                                double* opacity, double* t_final) {
  if (!c || n_views < 0) return SOF_E_INVALID;
  if (first_view < 0 || int64_t(first_view) + n_views > int64_t(c->cams.size())) {
    c->err = "view range out of range";
    return SOF_E_INVALID;
  }
  int64_t at = 0;  // pixel offset of the view in the concatenated outputs
  for (int v = first_view; v < first_view + n_views; ++v) {
    const int st = sof_render_view(c, v, depth_mode, kRTile, depth ? depth + at : nullptr,
                                   opacity ? opacity + at : nullptr, rgb ? rgb + 3 * at : nullptr,
                                   t_final ? t_final + at : nullptr, nullptr);
    if (st != SOF_OK) return st;
    at += int64_t(c->cams[v].w) * c->cams[v].h;
  }
  return SOF_OK;
}

extern "C" int sof_render_counts(sof_ctx* c, int view, uint32_t* counts) {
  if (!c || !counts) return SOF_E_INVALID;
  return guard(c, [&] {
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    if (c->r_view != view) throw StateError("no render of this view on the device: call sof_render_view first");
    const Cam& cam = c->cams[view];
    const int tiles_x = (cam.w + kRTile - 1) / kRTile;
    const int64_t P = int64_t(cam.w) * cam.h;
    DBuf<uint32_t>& o = c->rs.pcnt;  // the bounds are no longer needed after the render
    o.ensure(std::max<int64_t>(P, 1));
    k_rcounts_image<<<grid_for(c->r_Q, 256), 256, 0, c->stream>>>(cam, tiles_x, c->r_Q, c->rs.ncon.p, o.p);
    SOF_LAUNCHED(c);
    SOF_CUDA(cudaMemcpyAsync(counts, o.p, sizeof(uint32_t) * P, cudaMemcpyDeviceToHost, c->stream));
    SOF_CUDA(cudaStreamSynchronize(c->stream));
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

namespace {
// carve a per-call scratch of `bytes` (16-byte aligned pieces) out of c->r_query
struct Carve {
  char* base;
  size_t at = 0;
  template <typename T>
  T* take(int64_t count) {
    T* p = reinterpret_cast<T*>(base + at);
    at += (size_t(std::max<int64_t>(count, 1)) * sizeof(T) + 15) & ~size_t(15);
    return p;
  }
};
size_t carve_size(std::initializer_list<size_t> bytes) {
  size_t s = 0;
  for (size_t b : bytes) s += (std::max<size_t>(b, 1) + 15) & ~size_t(15);
  return s;
}
}  // namespace

extern "C" int sof_collect_contributions(sof_ctx* c, int view, int64_t nr, const double* dirs, int64_t* offsets_out) {
  if (!c || nr < 0 || (nr > 0 && (!dirs || !offsets_out))) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!c->has_scene) throw StateError("no scene: call sof_set_scene first");
    if (view < 0 || view >= int(c->cams.size())) throw InvalidArg("view index out of range");
    for (int64_t k = 0; k < 3 * nr; ++k)
      if (!std::isfinite(dirs[k])) throw InvalidArg("non-finite ray direction");
    render_attrs(c);
    c->n_contrib = -1;
    cudaStream_t st = c->stream;
    const Rec* rec = view_records(c, view);
    const int64_t n = c->n;
    DBuf<char>& b = c->r_query;
    b.ensure(int64_t(carve_size({size_t(24 * nr), size_t(4 * nr), size_t(8 * (nr + 1))})));
    Carve cv{b.p};
    double* d_dirs = cv.take<double>(3 * nr);
    uint32_t* cnt = cv.take<uint32_t>(nr);
    int64_t* off = cv.take<int64_t>(nr + 1);
    SOF_CUDA(cudaMemcpyAsync(d_dirs, dirs, 24 * nr, cudaMemcpyHostToDevice, st));
    SOF_CUDA(cudaMemsetAsync(cnt, 0, 4 * std::max<int64_t>(nr, 1), st));
    const dim3 grid(unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8))),
                    unsigned(std::max<int64_t>(1, std::min<int64_t>(nr, 65535))));
    if (nr > 0 && n > 0) {
      k_ct_scan<0><<<grid, 256, 0, st>>>(n, rec, nr, d_dirs, cnt, nullptr, nullptr);
      SOF_LAUNCHED(c);
    }
    scan_u32_i64(c, cnt, off, nr);
    const int64_t C = read_scalar(c, off + nr);
    c->rs.ent16.ensure(std::max<int64_t>(C, 1) * sizeof(REnt));
    REnt* E = reinterpret_cast<REnt*>(c->rs.ent16.p);
    if (C > 0) {
      SOF_CUDA(cudaMemsetAsync(cnt, 0, 4 * nr, st));
      k_ct_scan<1><<<grid, 256, 0, st>>>(n, rec, nr, d_dirs, cnt, off, E);
      SOF_LAUNCHED(c);
      sort_slices(c, 0, nr, off, 0, cnt, E);
    }
    c->ct_idx.ensure(std::max<int64_t>(C, 1));
    c->ct_val.ensure(6 * std::max<int64_t>(C, 1));
    if (C > 0) {
      k_ct_values<<<grid_for(C, 256), 256, 0, st>>>(C, nr, off, E, rec, d_dirs, c->ct_idx.p, c->ct_val.p);
      SOF_LAUNCHED(c);
    }
    SOF_CUDA(cudaMemcpyAsync(offsets_out, off, 8 * (nr + 1), cudaMemcpyDeviceToHost, st));
    SOF_CUDA(cudaStreamSynchronize(st));
    c->n_contrib = C;
  });
}

extern "C" int sof_windowed_resort(sof_ctx* c, int64_t nl, const int64_t* offsets, const double* t_star,
                                   int64_t window, int64_t* order_out) {
  if (!c || nl < 0 || window < 0 || (nl > 0 && !offsets)) return SOF_E_INVALID;
  return guard(c, [&] {
    if (nl == 0) return;
    if (offsets[0] != 0) throw InvalidArg("offsets[0] must be 0");
    for (int64_t l = 0; l < nl; ++l) {
      if (offsets[l + 1] < offsets[l]) throw InvalidArg("offsets must be non-decreasing");
      if (offsets[l + 1] - offsets[l] > INT32_MAX) throw InvalidArg("list longer than 2^31 - 1");
    }
    const int64_t C = offsets[nl];
    if (C > 0 && (!t_star || !order_out)) throw InvalidArg("null t_star / order");
    cudaStream_t st = c->stream;
    DBuf<char>& b = c->r_query;
    b.ensure(int64_t(carve_size({size_t(8 * (nl + 1)), size_t(8 * C), size_t(8 * C), size_t(16 * C), size_t(16 * C)})));
    Carve cv{b.p};
    int64_t* off = cv.take<int64_t>(nl + 1);
    double* t = cv.take<double>(C);
    int64_t* order = cv.take<int64_t>(C);
    REnt* S = cv.take<REnt>(C);
    REnt* O = cv.take<REnt>(C);
    SOF_CUDA(cudaMemcpyAsync(off, offsets, 8 * (nl + 1), cudaMemcpyHostToDevice, st));
    if (C > 0) SOF_CUDA(cudaMemcpyAsync(t, t_star, 8 * C, cudaMemcpyHostToDevice, st));
    k_wresort<<<grid_for(nl, 128), 128, 0, st>>>(nl, off, t, window, S, O, order);
    SOF_LAUNCHED(c);
    if (C > 0) SOF_CUDA(cudaMemcpyAsync(order_out, order, 8 * C, cudaMemcpyDeviceToHost, st));
    SOF_CUDA(cudaStreamSynchronize(st));
  });
}

extern "C" int sof_render_pixel(sof_ctx* c, int64_t nl, const int64_t* offsets, const int32_t* index,
                                const double* values, int64_t n_gauss, const double* dc, int depth_mode, double* color,
                                double* depth, double* acc_opacity, double* t_final) {
  if (!c || nl < 0 || n_gauss < 0 || (nl > 0 && !offsets)) return SOF_E_INVALID;
  return guard(c, [&] {
    if (!dc && !c->has_scene) throw StateError("no scene: call sof_set_scene first or pass the colours");
    const int64_t ng = dc ? n_gauss : c->n;
    if (depth_mode != SOF_DEPTH_EXACT && depth_mode != SOF_DEPTH_MEDIAN) throw InvalidArg("unknown depth mode");
    if (nl == 0) return;
    if (offsets[0] != 0) throw InvalidArg("offsets[0] must be 0");
    for (int64_t l = 0; l < nl; ++l)
      if (offsets[l + 1] < offsets[l]) throw InvalidArg("offsets must be non-decreasing");
    const int64_t C = offsets[nl];
    if (C > 0 && (!index || !values)) throw InvalidArg("null index / values");
    for (int64_t k = 0; k < C; ++k)
      if (index[k] < 0 || index[k] >= ng) throw InvalidArg("gaussian index out of range");
    cudaStream_t st = c->stream;
    DBuf<char>& b = c->r_query;
    b.ensure(int64_t(carve_size({size_t(8 * (nl + 1)), size_t(4 * C), size_t(48 * C), size_t(48 * nl),
                                 size_t(dc ? 24 * ng : 0)})));
    Carve cv{b.p};
    int64_t* off = cv.take<int64_t>(nl + 1);
    int32_t* idx = cv.take<int32_t>(C);
    double* val = cv.take<double>(6 * C);
    double* out = cv.take<double>(6 * nl);
    const double* colours = c->dc.p;
    if (dc) {
      double* d = cv.take<double>(3 * ng);
      if (ng > 0) SOF_CUDA(cudaMemcpyAsync(d, dc, 24 * ng, cudaMemcpyHostToDevice, st));
      colours = d;
    }
    SOF_CUDA(cudaMemcpyAsync(off, offsets, 8 * (nl + 1), cudaMemcpyHostToDevice, st));
    if (C > 0) {
      SOF_CUDA(cudaMemcpyAsync(idx, index, 4 * C, cudaMemcpyHostToDevice, st));
      SOF_CUDA(cudaMemcpyAsync(val, values, 48 * C, cudaMemcpyHostToDevice, st));
    }
    k_rpixel<<<grid_for(nl, 128), 128, 0, st>>>(nl, off, idx, val, colours, depth_mode == SOF_DEPTH_EXACT, out,
                                                 out + 3 * nl, out + 4 * nl, out + 5 * nl);
    SOF_LAUNCHED(c);
    if (color) SOF_CUDA(cudaMemcpyAsync(color, out, 24 * nl, cudaMemcpyDeviceToHost, st));
    if (depth) SOF_CUDA(cudaMemcpyAsync(depth, out + 3 * nl, 8 * nl, cudaMemcpyDeviceToHost, st));
    if (acc_opacity) SOF_CUDA(cudaMemcpyAsync(acc_opacity, out + 4 * nl, 8 * nl, cudaMemcpyDeviceToHost, st));
    if (t_final) SOF_CUDA(cudaMemcpyAsync(t_final, out + 5 * nl, 8 * nl, cudaMemcpyDeviceToHost, st));
    SOF_CUDA(cudaStreamSynchronize(st));
  });
}
