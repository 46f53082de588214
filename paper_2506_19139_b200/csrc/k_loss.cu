// k_loss.cu — SOF training losses with their analytic gradients, batched on the device
// (reference proj/include/sof/losses.hpp).
//
// The reference evaluates each loss for ONE ray (a vector of samples) or one image. Here
// a batch of rays arrives as CSR arrays (ray r owns samples [off[r], off[r + 1])) and one
// thread runs the reference's loops for its ray in the reference's operation order
// (--fmad=false, sof_exp for std::exp), so per-ray losses and per-sample gradients are
// bit-identical. Image losses (normal smoothness, L1 colour) compute per-pixel terms in
// parallel; their scalar sums run in the reference's scan order in one thread so the
// scalars are bit-identical too. Host buffers in, host buffers out (like the reference's
// std::vector API).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "sof_internal.h"

namespace sofk {

// ndc_map / ndc_derivative (losses.hpp:29-37); t > 0 is guaranteed by the callers
__device__ __forceinline__ double ndc_map_d(double t, double n, double f) { return f * (t - n) / (t * (f - n)); }
__device__ __forceinline__ double ndc_deriv_d(double t, double n, double f) { return f * n / ((f - n) * t * t); }

// distortion_loss (losses.hpp:54-107), one thread per ray. w, d, trans: per-sample scratch.
__global__ void k_distortion(int64_t nrays, const int64_t* __restrict__ off, const double* __restrict__ alpha,
                             const double* __restrict__ ts, double nearp, double farp, bool attach_w,
                             double* w, double* d, double* trans, double* loss, double* d_alpha, double* d_t) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= nrays) return;
  const int64_t b = off[r], e = off[r + 1];
  double transmittance = 1.0;
  for (int64_t i = b; i < e; ++i) {
    d_t[i] = 0.0;
    if (attach_w) d_alpha[i] = 0.0;
    if (ts[i] <= 0.0) {  // peak behind the camera (:70-76)
      w[i] = 0.0;
      d[i] = 0.0;
      trans[i] = transmittance;
      continue;
    }
    trans[i] = transmittance;
    w[i] = alpha[i] * transmittance;
    d[i] = ndc_map_d(ts[i], nearp, farp);
    transmittance *= 1.0 - alpha[i];
  }
  double l = 0.0, pa = 0.0, pd = 0.0, pdd = 0.0;
  for (int64_t i = b; i < e; ++i) {  // forward over prefix accumulators (:84-90)
    l += 2.0 * w[i] * (d[i] * d[i] * pa + pdd - 2.0 * d[i] * pd);
    pa += w[i];
    pd += w[i] * d[i];
    pdd += w[i] * d[i] * d[i];
  }
  loss[r] = l;
  const double full_a = pa, full_d = pd, full_dd = pdd;
  pa = pd = pdd = 0.0;
  for (int64_t k = b; k < e; ++k) {  // backward, front to back (:93-106)
    if (ts[k] <= 0.0) continue;
    const double gw = 2.0 * (d[k] * d[k] * full_a + full_dd - 2.0 * d[k] * full_d);
    d_t[k] = 4.0 * w[k] * (d[k] * full_a - full_d) * ndc_deriv_d(ts[k], nearp, farp);
    pa += w[k];
    pd += w[k] * d[k];
    pdd += w[k] * d[k] * d[k];
    if (attach_w) {
      const double suffix = 2.0 * (full_a * (full_dd - pdd) + full_dd * (full_a - pa) -
                                   2.0 * full_d * (full_d - pd));
      const double denom = 1.0 - alpha[k];
      d_alpha[k] = trans[k] * gw - (denom > 0.0 ? suffix / denom : 0.0);
    }
  }
}

// extent_loss (losses.hpp:152-179), one thread per ray; skipped counts per ray
__global__ void k_extent(int64_t nrays, const int64_t* __restrict__ off, const double* __restrict__ sw,
                         const double* __restrict__ sa, const double* __restrict__ sb, const double* __restrict__ sc,
                         const double* __restrict__ sbound, double nearp, double farp, double* loss, int32_t* skipped,
                         double* d_a, double* d_b, double* d_c, double* d_w) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= nrays) return;
  const double scale = farp * nearp / (farp - nearp);
  double l = 0.0;
  int skip = 0;
  for (int64_t i = off[r]; i < off[r + 1]; ++i) {
    d_a[i] = d_b[i] = d_c[i] = d_w[i] = 0.0;
    const double a = sa[i], bb = sb[i], w = sw[i];
    const double b2 = bb * bb;
    const double shifted_c = sc[i] - sbound[i] * sbound[i];
    const double disc = b2 - 4.0 * a * shifted_c;
    if (disc <= 0.0 || fabs(bb) < 1e-12) {
      ++skip;
      continue;
    }
    const double root = sqrt(disc);
    const double g = 2.0 * a * root / b2;
    l += scale * w * g;
    d_w[i] = scale * g;
    d_a[i] = scale * w * (2.0 * root / b2 - 4.0 * a * shifted_c / (b2 * root));
    d_b[i] = scale * w * (2.0 * a / (b2 * bb)) * (b2 / root - 2.0 * root);
    d_c[i] = scale * w * (-4.0 * a * a / (b2 * root));
  }
  loss[r] = l;
  skipped[r] = skip;
}

// depth_normal_loss (losses.hpp:119-133), one thread per ray; nrm / pix: xyz triples
__global__ void k_depth_normal(int64_t nrays, const int64_t* __restrict__ off, const double* __restrict__ w,
                               const double* __restrict__ nrm, const double* __restrict__ pix, double* loss,
                               double* d_w, double* d_n) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= nrays) return;
  const double px = pix[3 * r], py = pix[3 * r + 1], pz = pix[3 * r + 2];
  double l = 0.0;
  for (int64_t i = off[r]; i < off[r + 1]; ++i) {
    const double mis = 1.0 - (nrm[3 * i] * px + nrm[3 * i + 1] * py + nrm[3 * i + 2] * pz);
    l += w[i] * mis;
    d_w[i] = mis;
    d_n[3 * i] = -w[i] * px;
    d_n[3 * i + 1] = -w[i] * py;
    d_n[3 * i + 2] = -w[i] * pz;
  }
  loss[r] = l;
}

// alpha_at (opacity_field.hpp:95-101); contribution record: t*, alpha, a, b, c, opacity
__device__ __forceinline__ double alpha_at_d(const double* rc, double t) {
  const double te = (t < rc[0]) ? t : rc[0];  // std::min(t_star, t)
  if (te <= 0.0) return 0.0;
  const double a = rc[5] * sof_exp(-0.5 * ((rc[2] * te + rc[3]) * te + rc[4]));  // eval_1d gaussian.hpp:47-49
  if (a < kMinAlpha) return 0.0;
  return (kMaxAlpha < a) ? kMaxAlpha : a;
}

// opacity_supervision_loss (losses.hpp:195-229), one thread per ray; contribs: 6 doubles
// per sample (t*, alpha, a, b, c, opacity) in the ray's sorted order
__global__ void k_opacity_supervision(int64_t nrays, const int64_t* __restrict__ off, const double* __restrict__ rc,
                                      const double* __restrict__ depth, double* loss, double* field,
                                      uint8_t* defined, double* d_alpha) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= nrays) return;
  const int64_t b = off[r], e = off[r + 1];
  for (int64_t i = b; i < e; ++i) d_alpha[i] = 0.0;
  loss[r] = 0.0;
  field[r] = 0.0;
  defined[r] = 0;
  // find_median (opacity_field.hpp:132-142)
  int64_t k = -1;
  double tr = 1.0;
  for (int64_t i = b; i < e; ++i) {
    const double next = tr * (1.0 - rc[6 * i + 1]);
    if (tr > 0.5 && next < 0.5) {
      k = i;
      break;
    }
    tr = next;
  }
  const double dep = depth[r];
  if (k < 0 || dep != dep) return;  // no median or no surface (is_no_surface)
  double suffix = 0.0, tau = 1.0;
  for (int64_t i = k; i < e; ++i) {
    const double a = alpha_at_d(rc + 6 * i, dep);
    suffix += a * tau;
    tau *= 1.0 - a;
  }
  double prefix = 0.0, transmittance = 1.0;
  for (int64_t i = b; i < k; ++i) {
    const double a = alpha_at_d(rc + 6 * i, dep);
    prefix += a * transmittance;
    transmittance *= 1.0 - a;
  }
  const double fv = prefix + transmittance * suffix;
  const double residual = fv - 0.5;
  loss[r] = residual * residual;
  field[r] = fv;
  defined[r] = 1;
  const double survive = (1.0 - fv);
  for (int64_t i = b; i < e; ++i) {
    const double a = alpha_at_d(rc + 6 * i, dep);
    d_alpha[i] = 2.0 * residual * survive / (1.0 - a);
  }
}

// normal_smoothness_loss (losses.hpp:247-293), per pixel (x, y) with x + 1 < W, y + 1 < H:
// the term |grad N| exp(-|grad I|) and the two gradient pieces dgx, dgy; used[p] = 0
// (skipped), 1 (counted), 2 (counted, and |grad N| > 1e-14 so it adds gradients).
__device__ __forceinline__ double lum_d(const double* c) { return 0.299 * c[0] + 0.587 * c[1] + 0.114 * c[2]; }

__global__ void k_smooth_terms(int W, int H, const double* __restrict__ nrm, const uint8_t* __restrict__ valid,
                               const double* __restrict__ img, int per_channel, double* term, uint8_t* used,
                               double* dgx, double* dgy) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= int64_t(W) * H) return;
  const int x = int(p % W), y = int(p / W);
  term[p] = 0.0;
  used[p] = 0;
  for (int c = 0; c < 3; ++c) dgx[3 * p + c] = dgy[3 * p + c] = 0.0;
  if (x + 1 >= W || y + 1 >= H) return;
  const int64_t px = p + 1, py = p + W;
  if (!valid[p] || !valid[px] || !valid[py]) return;
  double gx[3], gy[3];
  for (int c = 0; c < 3; ++c) {
    gx[c] = nrm[3 * px + c] - nrm[3 * p + c];
    gy[c] = nrm[3 * py + c] - nrm[3 * p + c];
  }
  const double sgx = gx[0] * gx[0] + gx[1] * gx[1] + gx[2] * gx[2];
  const double sgy = gy[0] * gy[0] + gy[1] * gy[1] + gy[2] * gy[2];
  const double norm_n = sqrt(sgx + sgy);
  double grad_i;
  if (!per_channel) {
    const double ix = lum_d(img + 3 * px) - lum_d(img + 3 * p);
    const double iy = lum_d(img + 3 * py) - lum_d(img + 3 * p);
    grad_i = sqrt(ix * ix + iy * iy);
  } else {
    double ix[3], iy[3];
    for (int c = 0; c < 3; ++c) {
      ix[c] = img[3 * px + c] - img[3 * p + c];
      iy[c] = img[3 * py + c] - img[3 * p + c];
    }
    grad_i = sqrt((ix[0] * ix[0] + ix[1] * ix[1] + ix[2] * ix[2]) + (iy[0] * iy[0] + iy[1] * iy[1] + iy[2] * iy[2]));
  }
  const double weight = sof_exp(-grad_i);
  term[p] = norm_n * weight;
  used[p] = (norm_n > 1e-14) ? 2 : 1;  // 2: the pixel also contributes gradients
  if (norm_n > 1e-14)
    for (int c = 0; c < 3; ++c) {
      dgx[3 * p + c] = weight * gx[c] / norm_n;
      dgy[3 * p + c] = weight * gy[c] / norm_n;
    }
}

// d_normal of pixel (x, y) in the reference's accumulation order: += dgy from (x, y-1)
// (previous row), += dgx from (x-1, y), -= (dgx + dgy) of (x, y); then / used.
__global__ void k_smooth_grad(int W, int H, const uint8_t* __restrict__ used, const double* __restrict__ term,
                              const double* __restrict__ dgx, const double* __restrict__ dgy,
                              const int64_t* __restrict__ n_used, double* d_normal) {
  const int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (p >= int64_t(W) * H) return;
  const int x = int(p % W), y = int(p / W);
  const int64_t nu = *n_used;
  auto active = [&](int64_t q) { return used[q] == 2; };
  for (int c = 0; c < 3; ++c) {
    double v = 0.0;
    if (y > 0 && active(p - W)) v += dgy[3 * (p - W) + c];
    if (x > 0 && active(p - 1)) v += dgx[3 * (p - 1) + c];
    if (active(p)) v -= dgx[3 * p + c] + dgy[3 * p + c];
    d_normal[3 * p + c] = (nu > 0) ? v / double(nu) : v;
  }
}

// The scalar sums in the reference's scan order (one thread: bit-identical sums).
__global__ void k_smooth_sum(int64_t np, const double* __restrict__ term, const uint8_t* __restrict__ used,
                             double* out_sum, int64_t* n_used) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  int64_t u = 0;
  for (int64_t p = 0; p < np; ++p)
    if (used[p]) {
      s += term[p];
      ++u;
    }
  *out_sum = s;
  *n_used = u;
}

// l1_rgb_loss (losses.hpp:305-312): per pixel |dr| + |dg| + |db|, summed in pixel order
__global__ void k_l1_sum(int64_t np, const double* __restrict__ a, const double* __restrict__ b, double* out) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  for (int64_t p = 0; p < np; ++p)
    s += (fabs(a[3 * p] - b[3 * p]) + fabs(a[3 * p + 1] - b[3 * p + 1])) + fabs(a[3 * p + 2] - b[3 * p + 2]);
  *out = s;
}

}  // namespace sofk

using namespace sofk;

namespace {

template <typename T>
T* dev_copy(sof_ctx* c, DBuf<char>& buf, size_t& at, const T* host, int64_t count) {
  T* p = reinterpret_cast<T*>(buf.p + at);
  if (count > 0 && host)
    SOF_CUDA(cudaMemcpyAsync(p, host, sizeof(T) * size_t(count), cudaMemcpyHostToDevice, c->stream));
  at += (sizeof(T) * size_t(count) + 255) & ~size_t(255);
  return p;
}

template <typename T>
T* dev_alloc(DBuf<char>& buf, size_t& at, int64_t count) {
  T* p = reinterpret_cast<T*>(buf.p + at);
  at += (sizeof(T) * size_t(count) + 255) & ~size_t(255);
  return p;
}

template <typename T>
void host_copy(sof_ctx* c, T* host, const T* dev, int64_t count) {
  if (host && count > 0)
    SOF_CUDA(cudaMemcpyAsync(host, dev, sizeof(T) * size_t(count), cudaMemcpyDeviceToHost, c->stream));
}

size_t pad(size_t b) { return (b + 255) & ~size_t(255); }

void sync(sof_ctx* c) { SOF_CUDA(cudaStreamSynchronize(c->stream)); }

void need(bool ok, const char* what) {
  if (!ok) throw InvalidArg(what);
}

void check_off(int64_t nrays, const int64_t* off) {
  if (nrays < 0 || (nrays > 0 && !off)) throw InvalidArg("invalid ray offsets");
  if (nrays > 0 && off[0] != 0) throw InvalidArg("ray offsets must start at 0");
  for (int64_t r = 0; r < nrays; ++r)
    if (off[r + 1] < off[r]) throw InvalidArg("ray offsets must be non-decreasing");
}

}  // namespace

extern "C" {

int sof_distortion_loss(sof_ctx* c, int64_t nrays, const int64_t* off, const double* alpha, const double* t,
                        double near_plane, double far_plane, int attach_w, double* loss, double* d_alpha,
                        double* d_t) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    check_off(nrays, off);
    // no near/far check: the reference's distortion_loss has none (ndc_map divides by
    // far - near, so equal planes give the same inf / NaN there)
    const int64_t S = nrays ? off[nrays] : 0;
    need(S == 0 || (alpha && t), "null sample arrays");
    c->loss_buf.ensure(pad(8 * (nrays + 1)) + pad(8 * size_t(S)) * 7 + pad(8 * nrays) + 4096);
    size_t at = 0;
    int64_t* doff = dev_copy(c, c->loss_buf, at, off, nrays + 1);
    double* da = dev_copy(c, c->loss_buf, at, alpha, S);
    double* dt = dev_copy(c, c->loss_buf, at, t, S);
    double* w = dev_alloc<double>(c->loss_buf, at, S);
    double* d = dev_alloc<double>(c->loss_buf, at, S);
    double* tr = dev_alloc<double>(c->loss_buf, at, S);
    double* gl = dev_alloc<double>(c->loss_buf, at, nrays);
    double* ga = dev_alloc<double>(c->loss_buf, at, S);
    double* gt = dev_alloc<double>(c->loss_buf, at, S);
    if (nrays > 0) {
      k_distortion<<<grid_for(nrays, 128), 128, 0, c->stream>>>(nrays, doff, da, dt, near_plane, far_plane,
                                                                 attach_w != 0, w, d, tr, gl, ga, gt);
      SOF_LAUNCHED(c);
    }
    host_copy(c, loss, gl, nrays);
    if (attach_w) host_copy(c, d_alpha, ga, S);
    host_copy(c, d_t, gt, S);
    sync(c);
  });
}

int sof_extent_loss(sof_ctx* c, int64_t nrays, const int64_t* off, const double* w, const double* a,
                    const double* b, const double* cc, const double* bound, double near_plane, double far_plane,
                    double* loss, int32_t* skipped, double* d_a, double* d_b, double* d_c, double* d_w) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    check_off(nrays, off);
    const int64_t S = nrays ? off[nrays] : 0;
    need(S == 0 || (w && a && b && cc && bound), "null sample arrays");
    c->loss_buf.ensure(pad(8 * (nrays + 1)) + pad(8 * size_t(S)) * 9 + pad(8 * nrays) + pad(4 * nrays) + 4096);
    size_t at = 0;
    int64_t* doff = dev_copy(c, c->loss_buf, at, off, nrays + 1);
    double* dw = dev_copy(c, c->loss_buf, at, w, S);
    double* dA = dev_copy(c, c->loss_buf, at, a, S);
    double* dB = dev_copy(c, c->loss_buf, at, b, S);
    double* dC = dev_copy(c, c->loss_buf, at, cc, S);
    double* dE = dev_copy(c, c->loss_buf, at, bound, S);
    double* gl = dev_alloc<double>(c->loss_buf, at, nrays);
    int32_t* gs = dev_alloc<int32_t>(c->loss_buf, at, nrays);
    double* ga = dev_alloc<double>(c->loss_buf, at, S);
    double* gb = dev_alloc<double>(c->loss_buf, at, S);
    double* gc = dev_alloc<double>(c->loss_buf, at, S);
    double* gw = dev_alloc<double>(c->loss_buf, at, S);
    if (nrays > 0) {
      k_extent<<<grid_for(nrays, 128), 128, 0, c->stream>>>(nrays, doff, dw, dA, dB, dC, dE, near_plane, far_plane,
                                                             gl, gs, ga, gb, gc, gw);
      SOF_LAUNCHED(c);
    }
    host_copy(c, loss, gl, nrays);
    host_copy(c, skipped, gs, nrays);
    host_copy(c, d_a, ga, S);
    host_copy(c, d_b, gb, S);
    host_copy(c, d_c, gc, S);
    host_copy(c, d_w, gw, S);
    sync(c);
  });
}

int sof_depth_normal_loss(sof_ctx* c, int64_t nrays, const int64_t* off, const double* w, const double* normals,
                          const double* pixel_normals, double* loss, double* d_w, double* d_n) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    check_off(nrays, off);
    const int64_t S = nrays ? off[nrays] : 0;
    need(S == 0 || (w && normals), "null sample arrays");
    need(nrays == 0 || pixel_normals, "null pixel normals");
    c->loss_buf.ensure(pad(8 * (nrays + 1)) + pad(8 * size_t(S)) * 8 + pad(24 * nrays) + pad(8 * nrays) + 4096);
    size_t at = 0;
    int64_t* doff = dev_copy(c, c->loss_buf, at, off, nrays + 1);
    double* dw = dev_copy(c, c->loss_buf, at, w, S);
    double* dn = dev_copy(c, c->loss_buf, at, normals, 3 * S);
    double* dp = dev_copy(c, c->loss_buf, at, pixel_normals, 3 * nrays);
    double* gl = dev_alloc<double>(c->loss_buf, at, nrays);
    double* gw = dev_alloc<double>(c->loss_buf, at, S);
    double* gn = dev_alloc<double>(c->loss_buf, at, 3 * S);
    if (nrays > 0) {
      k_depth_normal<<<grid_for(nrays, 128), 128, 0, c->stream>>>(nrays, doff, dw, dn, dp, gl, gw, gn);
      SOF_LAUNCHED(c);
    }
    host_copy(c, loss, gl, nrays);
    host_copy(c, d_w, gw, S);
    host_copy(c, d_n, gn, 3 * S);
    sync(c);
  });
}

int sof_opacity_supervision_loss(sof_ctx* c, int64_t nrays, const int64_t* off, const double* contribs,
                                 const double* depth, double* loss, double* field_value, uint8_t* defined,
                                 double* d_alpha) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    check_off(nrays, off);
    const int64_t S = nrays ? off[nrays] : 0;
    need(S == 0 || contribs, "null contributions");
    need(nrays == 0 || depth, "null depths");
    c->loss_buf.ensure(pad(8 * (nrays + 1)) + pad(48 * size_t(S)) + pad(8 * size_t(S)) + pad(8 * nrays) * 3 +
                       pad(nrays) + 4096);
    size_t at = 0;
    int64_t* doff = dev_copy(c, c->loss_buf, at, off, nrays + 1);
    double* drc = dev_copy(c, c->loss_buf, at, contribs, 6 * S);
    double* ddep = dev_copy(c, c->loss_buf, at, depth, nrays);
    double* gl = dev_alloc<double>(c->loss_buf, at, nrays);
    double* gf = dev_alloc<double>(c->loss_buf, at, nrays);
    uint8_t* gd = dev_alloc<uint8_t>(c->loss_buf, at, nrays);
    double* ga = dev_alloc<double>(c->loss_buf, at, S);
    if (nrays > 0) {
      k_opacity_supervision<<<grid_for(nrays, 128), 128, 0, c->stream>>>(nrays, doff, drc, ddep, gl, gf, gd, ga);
      SOF_LAUNCHED(c);
    }
    host_copy(c, loss, gl, nrays);
    host_copy(c, field_value, gf, nrays);
    host_copy(c, defined, gd, nrays);
    host_copy(c, d_alpha, ga, S);
    sync(c);
  });
}

int sof_normal_smoothness_loss(sof_ctx* c, int width, int height, const double* normals, const uint8_t* valid,
                               const double* image, int per_channel, double* loss, int64_t* pixels_used,
                               double* d_normal) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (width < 0 || height < 0) throw InvalidArg("invalid image size");
    const int64_t P = int64_t(width) * height;
    need(P == 0 || (normals && valid && image), "null maps");
    c->loss_buf.ensure(pad(24 * size_t(P)) * 5 + pad(8 * size_t(P)) + pad(size_t(P)) * 2 + 4096);
    size_t at = 0;
    double* dn = dev_copy(c, c->loss_buf, at, normals, 3 * P);
    uint8_t* dv = dev_copy(c, c->loss_buf, at, valid, P);
    double* di = dev_copy(c, c->loss_buf, at, image, 3 * P);
    double* term = dev_alloc<double>(c->loss_buf, at, P);
    uint8_t* used = dev_alloc<uint8_t>(c->loss_buf, at, P);
    double* gx = dev_alloc<double>(c->loss_buf, at, 3 * P);
    double* gy = dev_alloc<double>(c->loss_buf, at, 3 * P);
    double* gn = dev_alloc<double>(c->loss_buf, at, 3 * P);
    double* sum = dev_alloc<double>(c->loss_buf, at, 1);
    int64_t* nu = dev_alloc<int64_t>(c->loss_buf, at, 1);
    double s = 0.0;
    int64_t u = 0;
    if (P > 0) {
      k_smooth_terms<<<grid_for(P, 256), 256, 0, c->stream>>>(width, height, dn, dv, di, per_channel, term, used, gx,
                                                               gy);
      SOF_LAUNCHED(c);
      k_smooth_sum<<<1, 32, 0, c->stream>>>(P, term, used, sum, nu);
      SOF_LAUNCHED(c);
      k_smooth_grad<<<grid_for(P, 256), 256, 0, c->stream>>>(width, height, used, term, gx, gy, nu, gn);
      SOF_LAUNCHED(c);
      SOF_CUDA(cudaMemcpyAsync(&s, sum, sizeof s, cudaMemcpyDeviceToHost, c->stream));
      SOF_CUDA(cudaMemcpyAsync(&u, nu, sizeof u, cudaMemcpyDeviceToHost, c->stream));
      host_copy(c, d_normal, gn, 3 * P);
    }
    sync(c);
    if (loss) *loss = (u > 0) ? s / double(u) : 0.0;
    if (pixels_used) *pixels_used = u;
  });
}

int sof_l1_rgb_loss(sof_ctx* c, int64_t pixels, const double* rendered, const double* reference, double* loss) {
  if (!c) return SOF_E_INVALID;
  return guard(c, [&] {
    if (pixels < 0 || (pixels > 0 && (!rendered || !reference))) throw InvalidArg("invalid images");
    c->loss_buf.ensure(pad(24 * size_t(pixels)) * 2 + 4096);
    size_t at = 0;
    double* da = dev_copy(c, c->loss_buf, at, rendered, 3 * pixels);
    double* db = dev_copy(c, c->loss_buf, at, reference, 3 * pixels);
    double* sum = dev_alloc<double>(c->loss_buf, at, 1);
    double s = 0.0;
    if (pixels > 0) {
      k_l1_sum<<<1, 32, 0, c->stream>>>(pixels, da, db, sum);
      SOF_LAUNCHED(c);
      SOF_CUDA(cudaMemcpyAsync(&s, sum, sizeof s, cudaMemcpyDeviceToHost, c->stream));
    }
    sync(c);
    if (loss) *loss = pixels ? s / (3.0 * double(pixels)) : 0.0;
  });
}

}  // extern "C"
