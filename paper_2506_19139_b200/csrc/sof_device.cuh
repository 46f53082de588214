// sof_device.cuh — device-side restatement of the reference's per-(Gaussian, view)
// and per-(point, Gaussian) arithmetic in FP64, operation for operation.
//
// Every expression follows the reference's C++ evaluation order (left-assoc,
// no contraction; this translation unit is compiled with --fmad=false) and the
// Eigen-API semantics pinned in oracle/eigen_shim/Eigen/Dense, so the results
// are bit-identical to the reference compiled against that shim. Each function
// cites the reference line it restates.
#pragma once

#include <cstdint>

#include "sof_math.h"

#ifndef SOF_EXP_CBANK
#define SOF_EXP_CBANK 1
#endif

namespace sofk {

constexpr double kMinAlpha = 1.0 / 255.0;  // core.hpp:18
constexpr double kMaxAlpha = 0.999;        // core.hpp:22
constexpr double kMinScale = 1e-8;         // gaussian.hpp:20
constexpr int kBlockPoints = 256;          // kBlockSize tiles.hpp:15

// Camera (camera.hpp:10-21) with the derived centre and tile grid.
struct Cam {
  double R[9];  // row-major world-to-view
  double t[3];
  double fx, fy, cx, cy;
  int w, h;
  double center[3];  // -R^T t (camera.hpp:20), computed on the host in reference order
};

// Per-(Gaussian, view) record used by the opacity evaluation:
// PrecomputedGaussian minus tight_bound (precompute.hpp:21-28), plus the exponent
// threshold below which alpha < 1/255 is certain. 112 B, 16-B aligned.
struct __align__(16) Rec {
  double ic[6];  // inv_cov upper triangle xx xy xz yy yz zz
  double b[3];   // b_vec
  double c;      // c_scalar
  double op;     // filtered opacity
  double zmin;   // min_z
  // log(1/(255 op)) - 1e-9 (1 + |.|), rounded toward -inf to float:
  // exponent < thr => alpha < 1/255
  float thr;
  // screen-space conic of the rays that can reach alpha >= 1/255: for the point's
  // pixel (u, v), g = G00 u^2 + G11 v^2 + G22 + 2 (G01 uv + G02 u + G12 v) equals
  // a(d) (L - m2_min(d)) for the (unnormalised) ray direction d through (u, v), with
  // L = 2 log(255 op); g < -gmargin proves m2 > L on the whole ray, i.e. alpha < 1/255
  // at every te (field_eval.hpp:100-101), so the pair is skipped without FP64 work.
  float conic[6];  // G00, G11, G22, 2 G01, 2 G02, 2 G12
  float gmargin;   // 256 ulp x the largest |term| over the image
};
static_assert(sizeof(Rec) == 128, "record layout");
constexpr int kRecV2 = int(sizeof(Rec) / 16);  // double2 per record

// FP32 filter record (64 B): a rounded copy of Rec plus error-bound constants.
// It only decides which pairs are PROVABLY skipped by the reference's tests
// (te <= 0 at field_eval.hpp:99, alpha < 1/255 at :101); every other pair is
// evaluated exactly from the FP64 Rec, so results stay bit-identical.
//   skip if b >= kb                      (then b_fp64 >= 0, i.e. t* <= 0 and te <= 0)
//   skip if g - (ka te^2 + kb |te| + kc) > gthr, g = (a te + b) te + c
//                                        (then the FP64 exponent is below log(1/(255 o)))
// ka, kb, kc bound the float error of a, b, g with a 64-ulp margin.
struct __align__(16) RecF {
  float ic[6];   // xx, yy, zz, 2xy, 2xz, 2yz coefficients (off-diagonals doubled)
  float b2[3];   // 2 * b_vec
  float c;
  float gthr;    // 2 log(255 o) + margin (-inf when o == 0)
  float zmin;    // nearest float of min_z
  float ka;      // 64 eps * ||Sigma^-1||_F  (bound on |a_f - a|)
  float kb;      // 64 eps * 2 ||b_vec||_1    (bound on |b_f - b|)
  float kc;      // 64 eps * |c| + 1e-5
  uint32_t flags;  // bit 0: dead (filtered opacity < 1/255, exact FP64 compare)
};
static_assert(sizeof(RecF) == 64, "float record layout");

constexpr float kEpsMargin = 64.0f * 5.9604645e-8f;  // 64 ulp of 1.0f

__device__ __forceinline__ RecF make_recf(const Rec& r) {
  RecF f;
  f.ic[0] = float(r.ic[0]);
  f.ic[1] = float(r.ic[3]);
  f.ic[2] = float(r.ic[5]);
  f.ic[3] = float(2.0 * r.ic[1]);
  f.ic[4] = float(2.0 * r.ic[2]);
  f.ic[5] = float(2.0 * r.ic[4]);
  for (int k = 0; k < 3; ++k) f.b2[k] = float(2.0 * r.b[k]);
  f.c = float(r.c);
  const double fro = sqrt(r.ic[0] * r.ic[0] + r.ic[3] * r.ic[3] + r.ic[5] * r.ic[5] +
                          2.0 * (r.ic[1] * r.ic[1] + r.ic[2] * r.ic[2] + r.ic[4] * r.ic[4]));
  const double b1 = 2.0 * (fabs(r.b[0]) + fabs(r.b[1]) + fabs(r.b[2]));
  f.ka = float(double(kEpsMargin) * fro * 1.0001 + 1e-30);
  f.kb = float(double(kEpsMargin) * b1 * 1.0001 + 1e-30);
  f.kc = float(double(kEpsMargin) * fabs(r.c) * 1.0001 + 1e-5);
  if (r.op > 0.0) {
    const double L = 2.0 * log(255.0 * r.op);
    f.gthr = float(L + 1e-6 * (1.0 + fabs(L)));
  } else {
    f.gthr = -INFINITY;
  }
  f.zmin = __double2float_rn(r.zmin);
  f.flags = (r.op < kMinAlpha) ? 1u : 0u;
  return f;
}

// Largest float <= x (round toward -inf), host and device.
__host__ __device__ inline float float_down(double x) {
#if defined(__CUDA_ARCH__)
  return __double2float_rd(x);
#else
  float f = (float)x;
  if ((double)f > x) f = nextafterf(f, -INFINITY);
  return f;
#endif
}

// View-independent per-Gaussian data (the parts of precompute.hpp:65-75 that do
// not depend on the camera, hoisted out of the per-view loop).
#ifndef SOF_GS_ALIGN
#define SOF_GS_ALIGN 16
#endif
// 16-byte aligned (one pad word): the per-view pass loads it with 16-byte loads, half the
// load instructions of 8-byte ones (that pass was LSU-throttled)
struct __align__(SOF_GS_ALIGN) GaussStatic {
  double pos[3];
  double scale[3];
  double rot[9];   // toRotationMatrix(q)            (gaussian.hpp:24)
  double cov[9];   // covariance(g) = R S^2 R^T      (gaussian.hpp:23-26)
  double icf[9];   // full inv_cov (NOT symmetrised: b_vec uses all 9, precompute.hpp:66-72)
  double op;       // filtered_opacity               (gaussian.hpp:67-73)
  double E;        // tight_bound, 0 when dead       (gaussian.hpp:60-64)
#if SOF_GS_ALIGN == 16
  double pad = 0.0;
#endif
};

// ---- L0: Eigen-shim semantics ---------------------------------------------------------

// Quaternion::toRotationMatrix (Eigen formula), q = (w, x, y, z).
__host__ __device__ inline void quat_to_rot(double w, double x, double y, double z, double* r) {
  const double tx = 2.0 * x, ty = 2.0 * y, tz = 2.0 * z;
  const double twx = tx * w, twy = ty * w, twz = tz * w;
  const double txx = tx * x, txy = ty * x, txz = tz * x;
  const double tyy = ty * y, tyz = tz * y, tzz = tz * z;
  r[0] = 1.0 - (tyy + tzz);
  r[1] = txy - twz;
  r[2] = txz + twy;
  r[3] = txy + twz;
  r[4] = 1.0 - (txx + tzz);
  r[5] = tyz - twx;
  r[6] = txz - twy;
  r[7] = tyz + twx;
  r[8] = 1.0 - (txx + tyy);
}

// 3x3 determinant, Eigen's bruteforce_det3 expansion.
__host__ __device__ inline double det3(const double* m) {
  const double h0 = m[0] * (m[4] * m[8] - m[5] * m[7]);
  const double h1 = m[1] * (m[3] * m[8] - m[5] * m[6]);
  const double h2 = m[2] * (m[3] * m[7] - m[4] * m[6]);
  return h0 - h1 + h2;
}

// r * diag(d) * r^T, each entry ((M(i,0) r(j,0) + M(i,1) r(j,1)) + M(i,2) r(j,2)).
__host__ __device__ inline void r_diag_rt(const double* r, const double* d, double* out) {
  double m[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) m[3 * i + j] = r[3 * i + j] * d[j];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      out[3 * i + j] = m[3 * i] * r[3 * j] + m[3 * i + 1] * r[3 * j + 1] + m[3 * i + 2] * r[3 * j + 2];
}

// Camera::to_view (camera.hpp:19): R x + t, one component.
__host__ __device__ inline double to_view_c(const Cam& c, int i, double x0, double x1, double x2) {
  return c.R[3 * i] * x0 + c.R[3 * i + 1] * x1 + c.R[3 * i + 2] * x2 + c.t[i];
}

// ---- L1: per-(Gaussian, view) preprocessing ----------------------------------------------

// View-independent half of precompute() (precompute.hpp:65-70) + filtered_opacity
// (gaussian.hpp:67-73) + tight_bound (gaussian.hpp:60-64).
__host__ __device__ inline void gauss_static(const double* pos, const double* scale,
                                             const double* q, double opacity,
                                             double filter_scale, GaussStatic& g) {
  for (int k = 0; k < 3; ++k) {
    g.pos[k] = pos[k];
    g.scale[k] = scale[k];
  }
  quat_to_rot(q[0], q[1], q[2], q[3], g.rot);
  // covariance(g): r * scale.cwiseProduct(scale).asDiagonal() * r^T  (unclamped scale)
  const double s2[3] = {scale[0] * scale[0], scale[1] * scale[1], scale[2] * scale[2]};
  r_diag_rt(g.rot, s2, g.cov);
  // inv_cov: r * (s.cwiseProduct(s)).cwiseInverse().asDiagonal() * r^T with s = max(scale, 1e-8)
  double s[3], inv[3];
  for (int k = 0; k < 3; ++k) {
    s[k] = (scale[k] < kMinScale) ? kMinScale : scale[k];
    inv[k] = 1.0 / (s[k] * s[k]);
  }
  r_diag_rt(g.rot, inv, g.icf);
  // filtered_opacity
  if (filter_scale <= 0.0) {
    g.op = opacity;
  } else {
    const double det = det3(g.cov);
    double cf[9];
    for (int k = 0; k < 9; ++k) cf[k] = g.cov[k] + filter_scale * ((k % 4 == 0) ? 1.0 : 0.0);
    const double det_f = det3(cf);
    g.op = opacity * sqrt(det / det_f);
  }
  // tight_bound(filtered opacity).value_or(0.0)
  if (g.op < kMinAlpha) {
    g.E = 0.0;
  } else {
    const double v = 2.0 * sof_log(255.0 * g.op);
    g.E = sqrt((v < 0.0) ? 0.0 : v);
  }
}

// View-dependent half of precompute() (precompute.hpp:71-76), diagonal z-extent mode.
__host__ __device__ inline void gauss_view(const GaussStatic& g, const Cam& cam, Rec& r) {
  // pc.inv_cov = upper triangle xx xy xz yy yz zz (precompute.hpp:69-70)
  r.ic[0] = g.icf[0];
  r.ic[1] = g.icf[1];
  r.ic[2] = g.icf[2];
  r.ic[3] = g.icf[4];
  r.ic[4] = g.icf[5];
  r.ic[5] = g.icf[8];
  const double d0 = cam.center[0] - g.pos[0];
  const double d1 = cam.center[1] - g.pos[1];
  const double d2 = cam.center[2] - g.pos[2];
  // b_vec = inv_cov * delta with the full (unsymmetrised) matrix (precompute.hpp:71-72)
  r.b[0] = g.icf[0] * d0 + g.icf[1] * d1 + g.icf[2] * d2;
  r.b[1] = g.icf[3] * d0 + g.icf[4] * d1 + g.icf[5] * d2;
  r.b[2] = g.icf[6] * d0 + g.icf[7] * d1 + g.icf[8] * d2;
  r.c = d0 * r.b[0] + d1 * r.b[1] + d2 * r.b[2];
  r.op = g.op;
  // z_extent_sigma kDiagonal (precompute.hpp:49-55): sqrt((W Sigma W^T)(2,2))
  double wc[3];
  for (int j = 0; j < 3; ++j)
    wc[j] = cam.R[6] * g.cov[j] + cam.R[7] * g.cov[3 + j] + cam.R[8] * g.cov[6 + j];
  const double czz = wc[0] * cam.R[6] + wc[1] * cam.R[7] + wc[2] * cam.R[8];
  const double zc = to_view_c(cam, 2, g.pos[0], g.pos[1], g.pos[2]);
  r.zmin = zc - g.E * sqrt(czz);
  // alpha = op exp(arg) < 1/255 whenever arg < log(1/(255 op)); the 1e-9 relative
  // margin dwarfs the ulp-level error of exp and of the product, so skipping the exp
  // below thr never changes a decision (field_eval.hpp:100-101, opacity_field.hpp:98-99)
  if (r.op > 0.0) {
    const double L = -log(255.0 * r.op);
    r.thr = float_down(L - 1e-9 * (1.0 + fabs(L)));
  } else {
    r.thr = INFINITY;
  }
  // Screen-space conic (see Rec). Rays through pixel p = (u, v, 1) have direction
  // d = R^T K^-1 p; with S the symmetric inverse covariance (upper triangle as used by
  // abc_cached) and L = 2 log(255 op): a(d) (L - m2_min(d)) = d^T (b b^T - (c - L) S) d.
  if (!(r.op >= kMinAlpha * (1.0 - 1e-9))) {
    // alpha = op G <= op (1 + 1e-15) < 1/255 for every ray: always skipped
    for (int k = 0; k < 6; ++k) r.conic[k] = 0.0f;
    r.conic[2] = -1.0f;
    r.gmargin = 0.0f;
  } else {
    const double L = 2.0 * log(255.0 * r.op);
    const double S[9] = {r.ic[0], r.ic[1], r.ic[2], r.ic[1], r.ic[3], r.ic[4], r.ic[2], r.ic[4], r.ic[5]};
    double M[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) M[3 * i + j] = r.b[i] * r.b[j] - (r.c - L) * S[3 * i + j];
    const double Ki[9] = {1.0 / cam.fx, 0.0, -cam.cx / cam.fx, 0.0, 1.0 / cam.fy, -cam.cy / cam.fy, 0.0, 0.0, 1.0};
    double A[9];  // R^T K^-1
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        A[3 * i + j] = cam.R[i] * Ki[j] + cam.R[3 + i] * Ki[3 + j] + cam.R[6 + i] * Ki[6 + j];
    double MA[9], G[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        MA[3 * i + j] = M[3 * i] * A[j] + M[3 * i + 1] * A[3 + j] + M[3 * i + 2] * A[6 + j];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        G[3 * i + j] = A[i] * MA[j] + A[3 + i] * MA[3 + j] + A[6 + i] * MA[6 + j];
    const double g00 = G[0], g11 = G[4], g22 = G[8];
    const double g01 = 0.5 * (G[1] + G[3]), g02 = 0.5 * (G[2] + G[6]), g12 = 0.5 * (G[5] + G[7]);
    r.conic[0] = float(g00);
    r.conic[1] = float(g11);
    r.conic[2] = float(g22);
    r.conic[3] = float(2.0 * g01);
    r.conic[4] = float(2.0 * g02);
    r.conic[5] = float(2.0 * g12);
    const double W = cam.w + 1.0, H = cam.h + 1.0;
    const double smax = fabs(g00) * W * W + fabs(g11) * H * H + fabs(g22) + 2.0 * fabs(g01) * W * H +
                        2.0 * fabs(g02) * W + 2.0 * fabs(g12) * H;
    // 256 ulp of 1.0f: covers the float rounding of the coefficients, of u, v and of
    // the 6-term evaluation, and the FP64 error of G, with a wide margin
    r.gmargin = float(smax * (256.0 * 5.9604645e-8) * 1.01 + 1e-30);
    if (!(r.gmargin < 3.0e38f)) {  // overflow / NaN: never cull
      for (int k = 0; k < 6; ++k) r.conic[k] = 0.0f;
      r.gmargin = 3.0e38f;
    }
  }
}

// x86-64 cvttsd2si semantics for int(x) (out of range / NaN -> INT_MIN), the
// reference binary's behaviour for int(std::floor(.)) at tiles.hpp:127-130.
__host__ __device__ inline int x86_int(double x) {
  return (x >= -2147483648.0 && x < 2147483648.0) ? (int)x : (int)0x80000000;
}

// glibc x86-64 std::llround: exact for |x| < 2^63; beyond that (and NaN) the result is
// (long long) x, i.e. cvttsd2si's 0x8000000000000000 for either sign (the reference
// binary's key at mesh.hpp:57-62 and seed_points.hpp:61-64).
__host__ __device__ inline long long x86_llround(double x) {
  return (x > -9223372036854775808.0 && x < 9223372036854775808.0) ? llround(x)
                                                                   : (long long)0x8000000000000000ull;
}

// Tile rectangle of one Gaussian's E-scaled OBB (build_tile_binding tiles.hpp:104-133).
// Returns false when the Gaussian is skipped (E <= 0 or fully off screen).
// *crosses_out (optional): the box crosses the camera plane (the all-tiles binding).
__host__ __device__ inline bool tile_rect(const GaussStatic& g, const Cam& cam, int tile_size,
                                          int tiles_x, int tiles_y, int& tx0, int& tx1, int& ty0,
                                          int& ty1, bool* crosses_out = nullptr) {
  const double r = g.E;
  if (r <= 0.0) return false;
  double min_x = 1e300, max_x = -1e300, min_y = 1e300, max_y = -1e300;
  bool crosses = false;
  for (int mask = 0; mask < 8; ++mask) {
    const double l0 = r * g.scale[0] * (double)((mask & 1) ? 1 : -1);
    const double l1 = r * g.scale[1] * (double)((mask & 2) ? 1 : -1);
    const double l2 = r * g.scale[2] * (double)((mask & 4) ? 1 : -1);
    // g.position + rot * local
    const double p0 = g.pos[0] + (g.rot[0] * l0 + g.rot[1] * l1 + g.rot[2] * l2);
    const double p1 = g.pos[1] + (g.rot[3] * l0 + g.rot[4] * l1 + g.rot[5] * l2);
    const double p2 = g.pos[2] + (g.rot[6] * l0 + g.rot[7] * l1 + g.rot[8] * l2);
    const double vx = to_view_c(cam, 0, p0, p1, p2);
    const double vy = to_view_c(cam, 1, p0, p1, p2);
    const double vz = to_view_c(cam, 2, p0, p1, p2);
    if (vz <= 1e-9) {
      crosses = true;
      break;
    }
    const double px = cam.fx * vx / vz + cam.cx;
    const double py = cam.fy * vy / vz + cam.cy;
    min_x = (px < min_x) ? px : min_x;  // std::min(min_x, px)
    max_x = (max_x < px) ? px : max_x;  // std::max(max_x, px)
    min_y = (py < min_y) ? py : min_y;
    max_y = (max_y < py) ? py : max_y;
  }
  tx0 = 0;
  tx1 = tiles_x - 1;
  ty0 = 0;
  ty1 = tiles_y - 1;
  if (crosses_out) *crosses_out = crosses;
  if (!crosses) {
    int a = x86_int(floor(min_x)) / tile_size;
    tx0 = (0 < a) ? a : 0;
    a = x86_int(floor(max_x)) / tile_size;
    tx1 = (a < tiles_x - 1) ? a : tiles_x - 1;
    a = x86_int(floor(min_y)) / tile_size;
    ty0 = (0 < a) ? a : 0;
    a = x86_int(floor(max_y)) / tile_size;
    ty1 = (a < tiles_y - 1) ? a : tiles_y - 1;
    if (max_x < 0.0 || min_x >= (double)cam.w || max_y < 0.0 || min_y >= (double)cam.h)
      return false;
  }
  return tx0 <= tx1 && ty0 <= ty1;
}

// A live Gaussian lying behind the camera in Mahalanobis terms: its centre at view depth
// zc < 0 and zc^2 >= s_z^2 (E^2 (1 + 1e-4) + 1e-4), s_z^2 the clamped-scale covariance's
// variance along the view axis (so every point at view z >= 0 has squared Mahalanobis
// distance q >= zc^2 / s_z^2 from it). Consequences, all exact:
//  * the reference binds it to every tile (a box centred behind the plane has a corner at
//    z <= 1e-9, tiles.hpp:116-126) with min_z < zc < 0, ahead of every other entry with
//    min_z > 0 and of any min-z break (field_eval.hpp:90-93);
//  * along a point ray (view z >= 0 for te >= 0) alpha = op exp(-q / 2) stays below
//    (1 / 255) exp(-5e-5): the pair is counted (:94) and contributes nothing (:99-101);
//    c <= 1e10 keeps the FP64 evaluation error of q far below that margin.
// The fast evaluation loop therefore leaves these out of the tile lists and counts them
// (Binding::nb).
__host__ __device__ inline bool gauss_behind(const GaussStatic& g, const Cam& cam, double c_scalar) {
  if (!(g.E > 0.0) || !(c_scalar <= 1e10)) return false;
  const double zc = to_view_c(cam, 2, g.pos[0], g.pos[1], g.pos[2]);
  if (!(zc < 0.0)) return false;
  double czz = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double w = cam.R[6] * g.rot[k] + cam.R[7] * g.rot[3 + k] + cam.R[8] * g.rot[6 + k];  // (W R)_zk
    const double sk = (g.scale[k] < kMinScale) ? kMinScale : g.scale[k];
    czz += w * w * sk * sk;
  }
  return zc * zc >= czz * (g.E * g.E * (1.0 + 1e-4) + 1e-4) * (1.0 + 1e-12);
}

// ---- L2: per-point ray setup (field_eval.hpp:62-79) -------------------------------------

struct PointRay {
  double d[3];   // unit direction camera -> x
  double t;      // |x - o|
  double zp;     // view-space z of x
  double px, py; // pixel coordinates of x (camera.hpp:26)
  int tile;      // tile index (valid when observed)
  bool observed;
};

__host__ __device__ inline PointRay point_ray(const Cam& cam, double x0, double x1, double x2,
                                              int tile_size, int tiles_x) {
  PointRay pr;
  pr.observed = false;
  pr.tile = -1;
  // Camera::observes via project (camera.hpp:23-33)
  const double vx = to_view_c(cam, 0, x0, x1, x2);
  const double vy = to_view_c(cam, 1, x0, x1, x2);
  const double vz = to_view_c(cam, 2, x0, x1, x2);
  pr.zp = vz;
  if (vz <= 0.0) return pr;
  const double px = cam.fx * vx / vz + cam.cx;
  const double py = cam.fy * vy / vz + cam.cy;
  pr.px = px;
  pr.py = py;
  if (!(px >= 0.0 && px < (double)cam.w && py >= 0.0 && py < (double)cam.h)) return pr;
  // ray_through_point (camera.hpp:52-59)
  const double e0 = x0 - cam.center[0], e1 = x1 - cam.center[1], e2 = x2 - cam.center[2];
  pr.t = sqrt(e0 * e0 + e1 * e1 + e2 * e2);
  if (pr.t < 1e-12) return pr;  // field_eval.hpp:67-70
  pr.d[0] = e0 / pr.t;
  pr.d[1] = e1 / pr.t;
  pr.d[2] = e2 / pr.t;
  pr.tile = (int)py / tile_size * tiles_x + (int)px / tile_size;  // field_eval.hpp:79
  pr.observed = true;
  return pr;
}

// point_ray's observed flag and tile only (the scheduler's per-view pass): the same
// projection and tests, with `t < 1e-12` (field_eval.hpp:67-70) decided on the squared
// distance outside a relative guard band of 1e-10 around 1e-24 — sqrt and rounding are
// monotone, so outside the band the comparison cannot differ — and by the exact sqrt
// inside it.
struct PointTile {
  double px, py;
  int tile;  // -1 when not observed
};
template <int TS = 0>  // TS = 16: the default tile size as a compile-time constant
__device__ __forceinline__ PointTile point_tile(const Cam& cam, double x0, double x1, double x2, int tile_size,
                                                int tiles_x) {
  PointTile pt;
  pt.tile = -1;
  pt.px = pt.py = 0.0;
  const double vx = to_view_c(cam, 0, x0, x1, x2);
  const double vy = to_view_c(cam, 1, x0, x1, x2);
  const double vz = to_view_c(cam, 2, x0, x1, x2);
  if (vz <= 0.0) return pt;
  const double px = cam.fx * vx / vz + cam.cx;
  const double py = cam.fy * vy / vz + cam.cy;
  pt.px = px;
  pt.py = py;
  if (!(px >= 0.0 && px < (double)cam.w && py >= 0.0 && py < (double)cam.h)) return pt;
  const double e0 = x0 - cam.center[0], e1 = x1 - cam.center[1], e2 = x2 - cam.center[2];
  const double s2 = e0 * e0 + e1 * e1 + e2 * e2;
  const bool near = (s2 < 1e-24 * (1.0 - 1e-10)) ? true : (s2 > 1e-24 * (1.0 + 1e-10)) ? false : (sqrt(s2) < 1e-12);
  if (near) return pt;
  pt.tile = (TS == 16) ? ((int)py >> 4) * tiles_x + ((int)px >> 4)  // px, py >= 0: shifts = divisions
                       : (int)py / tile_size * tiles_x + (int)px / tile_size;
  return pt;
}

// ---- L2: one (point, Gaussian) pair of view_opacity (field_eval.hpp:95-103) ---------------
// Returns the clamped alpha, or 0 when the pair is skipped (te <= 0 or alpha < 1/255).
template <typename Tab = const double*>
__device__ __forceinline__ double pair_alpha(const Rec& r, const double* d, double t,
                                             Tab exp_tab = kSofExpTabDev) {
  const double x = d[0], y = d[1], z = d[2];
  // abc_cached (precompute.hpp:39-45)
  const double a = r.ic[0] * x * x + r.ic[3] * y * y + r.ic[5] * z * z +
                   2.0 * (r.ic[1] * x * y + r.ic[2] * x * z + r.ic[4] * y * z);
  const double b = 2.0 * (x * r.b[0] + y * r.b[1] + z * r.b[2]);
  const double two_a = 2.0 * a;
  double te;
  if (a > 0.0 && __fma_rn(two_a, t, b) < 0.0) {
    // 2 a t + b < 0 exactly (the sign of a correctly rounded fma is exact), so
    // t* = -b / (2a) > t and min(fl(t*), t) = t: the IEEE division is not needed
    te = t;
  } else {
    const double t_star = -b / two_a;           // peak_t gaussian.hpp:52
    te = (t < t_star) ? t : t_star;             // std::min(t_star, t)
    if (te <= 0.0) return 0.0;
  }
  const double arg = -0.5 * ((a * te + b) * te + r.c);  // eval_1d gaussian.hpp:47-49
  if (arg < double(r.thr)) return 0.0;                  // alpha < 1/255 certain
#if SOF_EXP_CBANK
  const double e = (arg >= -700.0 && arg <= 700.0) ? sof_exp_mid_cb(arg, exp_tab) : sof_exp(arg);
#else
  const double e = (arg >= -700.0 && arg <= 700.0) ? sof_exp_mid(arg, exp_tab) : sof_exp(arg);  // generic table
#endif
  const double alpha = r.op * e;
  if (alpha < kMinAlpha) return 0.0;
  return (kMaxAlpha < alpha) ? kMaxAlpha : alpha;  // std::min(alpha, kMaxAlpha)
}

// Screen-space cull (Rec::conic): true when the ray through pixel (u, v) provably
// stays below alpha = 1/255. uu = u*u, vv = v*v, uv = u*v in float.
__device__ __forceinline__ bool conic_culls(const Rec& r, float u, float v, float uu, float vv,
                                            float uv) {
  const float g = fmaf(r.conic[0], uu, fmaf(r.conic[1], vv, fmaf(r.conic[3], uv,
                  fmaf(r.conic[4], u, fmaf(r.conic[5], v, r.conic[2])))));
  return g < -r.gmargin;
}

// Upper bound of the screen conic (Rec::conic, evaluated in FP64 from its float
// coefficients) over the pixel box [u0, u1] x [v0, v1]: a quadratic's maximum over a box
// lies at a corner, at the vertex of an edge (concave along it), or at the interior
// vertex (concave). Locating a vertex with rounding error lowers the value found only to
// second order, far inside the 1e-6 gmargin slack of conic_box_culled.
__host__ __device__ inline double conic_max_box(const Rec& r, double u0, double u1, double v0, double v1) {
  const double A = r.conic[0], B = r.conic[1], F = r.conic[2], C = r.conic[3], D = r.conic[4], E = r.conic[5];
  auto g = [&](double u, double v) { return ((A * u * u + B * v * v) + C * u * v) + ((D * u + E * v) + F); };
  double m = g(u0, v0);
  auto take = [&](double x) { m = (m < x || x != x) ? x : m; };  // NaN propagates: never culled
  take(g(u1, v0));
  take(g(u0, v1));
  take(g(u1, v1));
  if (B < 0.0) {
    const double us[2] = {u0, u1};
    for (int i = 0; i < 2; ++i) {
      const double u = us[i], v = -(C * u + E) / (2.0 * B);
      if (v > v0 && v < v1) take(g(u, v));
    }
  }
  if (A < 0.0) {
    const double vs[2] = {v0, v1};
    for (int i = 0; i < 2; ++i) {
      const double v = vs[i], u = -(C * v + D) / (2.0 * A);
      if (u > u0 && u < u1) take(g(u, v));
    }
  }
  const double det = 4.0 * A * B - C * C;
  if (A < 0.0 && det > 0.0) {
    const double u = (C * E - 2.0 * B * D) / det, v = (C * D - 2.0 * A * E) / det;
    if (u > u0 && u < u1 && v > v0 && v < v1) take(g(u, v));
  }
  return m;
}

// True when no ray through the pixel box reaches alpha >= 1/255 on this Gaussian: the
// point-level conic_culls would skip every point that projects into the box.
__host__ __device__ inline bool conic_box_culled(const Rec& r, double u0, double u1, double v0, double v1) {
  return conic_max_box(r, u0, u1, v0, v1) < -double(r.gmargin) * (1.0 + 1e-6);
}

// The all-tiles binding of a live Gaussian whose box crosses the camera plane
// (tiles.hpp:116-126), restricted to the tiles whose points it may reach: the whole
// screen, then the tile's row, then the tile must survive conic_box_culled. The other
// (tile, Gaussian) pairs of the reference's lists are counted, never evaluated
// (Binding::nb / xpos).
__host__ __device__ inline bool cross_screen_live(const Rec& r, int ts, int tiles_x, int tiles_y) {
  return !conic_box_culled(r, 0.0, double(tiles_x) * ts, 0.0, double(tiles_y) * ts);
}
__host__ __device__ inline bool cross_row_live(const Rec& r, int ts, int tiles_x, int ty) {
  return !conic_box_culled(r, 0.0, double(tiles_x) * ts, double(ty) * ts, double(ty + 1) * ts);
}
__host__ __device__ inline bool cross_tile_live(const Rec& r, int ts, int tx, int ty) {
  return !conic_box_culled(r, double(tx) * ts, double(tx + 1) * ts, double(ty) * ts, double(ty + 1) * ts);
}
__host__ __device__ inline uint32_t cross_tile_count(const Rec& r, int ts, int tiles_x, int tiles_y) {
  if (!cross_screen_live(r, ts, tiles_x, tiles_y)) return 0;
  uint32_t k = 0;
  for (int ty = 0; ty < tiles_y; ++ty) {
    if (!cross_row_live(r, ts, tiles_x, ty)) continue;
    for (int tx = 0; tx < tiles_x; ++tx) k += cross_tile_live(r, ts, tx, ty);
  }
  return k;
}

// Orderable 64-bit key of a double (ascending), with -0 folded onto +0 so that
// equal values compare equal as in `min_z != min_z` (tiles.hpp:141).
__host__ __device__ inline uint64_t double_key(double v) {
  if (v == 0.0) v = 0.0;
  const uint64_t u = sof_double_to_bits(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// inverse of double_key
__host__ __device__ inline double key_double(uint64_t k) {
  return sof_bits_to_double((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k);
}

}  // namespace sofk
