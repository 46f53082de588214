// sof_math.h — the framework's double-precision exp/log, one implementation for
// host and device.
//
// The reference calls std::exp in eval_1d / peak_value (gaussian.hpp:47-56,
// reached from field_eval.hpp:100 and opacity_field.hpp:47,98) and std::log in
// tight_bound (gaussian.hpp:60-64) and exact_depth (opacity_field.hpp:161-162).
// Neither glibc's exp/log nor CUDA's are correctly rounded, and they disagree in
// the last bit on some arguments, which would make the sorted-opacity decisions
// (alpha < 1/255, 1 - survive > 0.5, the median transmittance crossing) differ
// between a CPU run and a GPU run on rare inputs. This header fixes ONE
// algorithm for both sides:
//   * every + - * / is IEEE round-to-nearest and sqrt/fma are correctly rounded
//     on x86-64 and on sm_100a, so identical operation sequences give identical
//     bits;
//   * on the device every operation is written with __dadd_rn/__dmul_rn/__fma_rn
//     so nvcc's FMA contraction can never change the sequence; host builds use
//     -ffp-contract=off.
// Accuracy: < 1 ulp for both (tests/test_oracle_cpu.py compares against glibc
// on 10^6 arguments and reports the agreement rate).
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define SOF_HD __host__ __device__ __forceinline__
#else
#define SOF_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define SOF_ADD(a, b) __dadd_rn((a), (b))
#define SOF_SUB(a, b) __dsub_rn((a), (b))
#define SOF_MUL(a, b) __dmul_rn((a), (b))
#define SOF_DIV(a, b) __ddiv_rn((a), (b))
#define SOF_FMA(a, b, c) __fma_rn((a), (b), (c))
#define SOF_RINT(a) rint(a)
#else
#define SOF_ADD(a, b) ((a) + (b))
#define SOF_SUB(a, b) ((a) - (b))
#define SOF_MUL(a, b) ((a) * (b))
#define SOF_DIV(a, b) ((a) / (b))
#define SOF_FMA(a, b, c) fma((a), (b), (c))
#define SOF_RINT(a) rint(a)
#endif

SOF_HD double sof_bits_to_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double d;
  memcpy(&d, &u, 8);
  return d;
#endif
}

SOF_HD uint64_t sof_double_to_bits(double d) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(d);
#else
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
#endif
}

/// 2^n for -1022 <= n <= 1023 (exact).
SOF_HD double sof_pow2i(int n) { return sof_bits_to_double((uint64_t)(n + 1023) << 52); }

// 2^(j/64) = hi + lo for j = 0..63 (hi = RN(2^(j/64)), lo = RN(2^(j/64) - hi)),
// computed with 80-digit decimal arithmetic.
#define SOF_EXP_TAB_INIT { \
    0x1.0000000000000p+0, 0x0.0p+0, \
    0x1.02c9a3e778061p+0, -0x1.19083535b085dp-56, \
    0x1.059b0d3158574p+0, 0x1.d73e2a475b465p-55, \
    0x1.0874518759bc8p+0, 0x1.186be4bb284ffp-57, \
    0x1.0b5586cf9890fp+0, 0x1.8a62e4adc610bp-54, \
    0x1.0e3ec32d3d1a2p+0, 0x1.03a1727c57b53p-59, \
    0x1.11301d0125b51p+0, -0x1.6c51039449b3ap-54, \
    0x1.1429aaea92de0p+0, -0x1.32fbf9af1369ep-54, \
    0x1.172b83c7d517bp+0, -0x1.19041b9d78a76p-55, \
    0x1.1a35beb6fcb75p+0, 0x1.e5b4c7b4968e4p-55, \
    0x1.1d4873168b9aap+0, 0x1.e016e00a2643cp-54, \
    0x1.2063b88628cd6p+0, 0x1.dc775814a8495p-55, \
    0x1.2387a6e756238p+0, 0x1.9b07eb6c70573p-54, \
    0x1.26b4565e27cddp+0, 0x1.2bd339940e9d9p-55, \
    0x1.29e9df51fdee1p+0, 0x1.612e8afad1255p-55, \
    0x1.2d285a6e4030bp+0, 0x1.0024754db41d5p-54, \
    0x1.306fe0a31b715p+0, 0x1.6f46ad23182e4p-55, \
    0x1.33c08b26416ffp+0, 0x1.32721843659a6p-54, \
    0x1.371a7373aa9cbp+0, -0x1.63aeabf42eae2p-54, \
    0x1.3a7db34e59ff7p+0, -0x1.5e436d661f5e3p-56, \
    0x1.3dea64c123422p+0, 0x1.ada0911f09ebcp-55, \
    0x1.4160a21f72e2ap+0, -0x1.ef3691c309278p-58, \
    0x1.44e086061892dp+0, 0x1.89b7a04ef80d0p-59, \
    0x1.486a2b5c13cd0p+0, 0x1.3c1a3b69062f0p-56, \
    0x1.4bfdad5362a27p+0, 0x1.d4397afec42e2p-56, \
    0x1.4f9b2769d2ca7p+0, -0x1.4b309d25957e3p-54, \
    0x1.5342b569d4f82p+0, -0x1.07abe1db13cadp-55, \
    0x1.56f4736b527dap+0, 0x1.9bb2c011d93adp-54, \
    0x1.5ab07dd485429p+0, 0x1.6324c054647adp-54, \
    0x1.5e76f15ad2148p+0, 0x1.ba6f93080e65ep-54, \
    0x1.6247eb03a5585p+0, -0x1.383c17e40b497p-54, \
    0x1.6623882552225p+0, -0x1.bb60987591c34p-54, \
    0x1.6a09e667f3bcdp+0, -0x1.bdd3413b26456p-54, \
    0x1.6dfb23c651a2fp+0, -0x1.bbe3a683c88abp-57, \
    0x1.71f75e8ec5f74p+0, -0x1.16e4786887a99p-55, \
    0x1.75feb564267c9p+0, -0x1.0245957316dd3p-54, \
    0x1.7a11473eb0187p+0, -0x1.41577ee04992fp-55, \
    0x1.7e2f336cf4e62p+0, 0x1.05d02ba15797ep-56, \
    0x1.82589994cce13p+0, -0x1.d4c1dd41532d8p-54, \
    0x1.868d99b4492edp+0, -0x1.fc6f89bd4f6bap-54, \
    0x1.8ace5422aa0dbp+0, 0x1.6e9f156864b27p-54, \
    0x1.8f1ae99157736p+0, 0x1.5cc13a2e3976cp-55, \
    0x1.93737b0cdc5e5p+0, -0x1.75fc781b57ebcp-57, \
    0x1.97d829fde4e50p+0, -0x1.d185b7c1b85d1p-54, \
    0x1.9c49182a3f090p+0, 0x1.c7c46b071f2bep-56, \
    0x1.a0c667b5de565p+0, -0x1.359495d1cd533p-54, \
    0x1.a5503b23e255dp+0, -0x1.d2f6edb8d41e1p-54, \
    0x1.a9e6b5579fdbfp+0, 0x1.0fac90ef7fd31p-54, \
    0x1.ae89f995ad3adp+0, 0x1.7a1cd345dcc81p-54, \
    0x1.b33a2b84f15fbp+0, -0x1.2805e3084d708p-57, \
    0x1.b7f76f2fb5e47p+0, -0x1.5584f7e54ac3bp-56, \
    0x1.bcc1e904bc1d2p+0, 0x1.23dd07a2d9e84p-55, \
    0x1.c199bdd85529cp+0, 0x1.11065895048ddp-55, \
    0x1.c67f12e57d14bp+0, 0x1.2884dff483cadp-54, \
    0x1.cb720dcef9069p+0, 0x1.503cbd1e949dbp-56, \
    0x1.d072d4a07897cp+0, -0x1.cbc3743797a9cp-54, \
    0x1.d5818dcfba487p+0, 0x1.2ed02d75b3707p-55, \
    0x1.da9e603db3285p+0, 0x1.c2300696db532p-54, \
    0x1.dfc97337b9b5fp+0, -0x1.1a5cd4f184b5cp-54, \
    0x1.e502ee78b3ff6p+0, 0x1.39e8980a9cc8fp-55, \
    0x1.ea4afa2a490dap+0, -0x1.e9c23179c2893p-54, \
    0x1.efa1bee615a27p+0, 0x1.dc7f486a4b6b0p-54, \
    0x1.f50765b6e4540p+0, 0x1.9d3e12dd8a18bp-54, \
    0x1.fa7c1819e90d8p+0, 0x1.74853f3a5931ep-55 }
static const double kSofExpTab[128] = SOF_EXP_TAB_INIT;
#if defined(__CUDACC__)
static __device__ __align__(16) const double kSofExpTabDev[128] = SOF_EXP_TAB_INIT;
#endif

SOF_HD double sof_exp_tab(int i) {
#if defined(__CUDA_ARCH__)
  return __ldg(&kSofExpTabDev[i]);
#else
  return kSofExpTab[i];
#endif
}

/// e^x for finite x in [-745.14, 709.79]: k = rint(x 64/ln2) = 64 m + j,
/// r = x - k ln2/64 (two fma steps; ln2/64 split into a 36-bit head, exact times k,
/// and a tail), e^r - 1 = r + r^2 (1/2 + r (1/6 + r (1/24 + r/120))) (|r| <=
/// ln2/128: truncation 3.5e-17), 2^(j/64) (1 + p) = hi + (hi p + lo) with one final
/// rounding, then an exact scale by 2^m (a single rounding for subnormal results).
SOF_HD double sof_exp_core(double x) {
  const double kInv64Ln2 = 0x1.71547652b82fep+6;  // 64 / ln2
  const double kLn2Hi = 0x1.62e42fefa0000p-7;     // ln2 / 64, 36 significant bits
  const double kLn2Lo = 0x1.cf79abc9e3b3ap-46;
  const double kd = SOF_RINT(SOF_MUL(x, kInv64Ln2));
  const int k = (int)kd;
  double r = SOF_FMA(-kd, kLn2Hi, x);
  r = SOF_FMA(-kd, kLn2Lo, r);
  double q = SOF_FMA(r, 1.0 / 720.0, 1.0 / 120.0);
  q = SOF_FMA(q, r, 1.0 / 24.0);
  q = SOF_FMA(q, r, 1.0 / 6.0);
  q = SOF_FMA(q, r, 0.5);
  const double p = SOF_FMA(SOF_MUL(r, r), q, r);
  const int j = k & 63, m = k >> 6;  // arithmetic shift: floor(k / 64)
  const double th = sof_exp_tab(2 * j), tl = sof_exp_tab(2 * j + 1);
  const double y = SOF_ADD(th, SOF_FMA(th, p, tl));
  if (m > 1023) return SOF_MUL(SOF_MUL(y, 2.0), sof_pow2i(m - 1));
  if (m < -1020) return SOF_MUL(SOF_MUL(y, sof_pow2i(m + 1000)), sof_pow2i(-1000));
  return SOF_MUL(y, sof_pow2i(m));
}

/// e^x (< 1 ulp; see the header comment).
SOF_HD double sof_exp(double x) {
  if (x != x) return SOF_ADD(x, x);
  if (x > 709.782712893383973096) return sof_bits_to_double(0x7ff0000000000000ull);
  if (x < -745.1332191019412076235) return 0.0;
  return sof_exp_core(x);
}

#ifdef __CUDACC__
/// sof_exp for -700 <= x <= 700: the same operations without the range tests and the
/// extreme scalings, which cannot occur there (|m| <= 1010): bit-identical results.
/// tab: kSofExpTabDev or a copy of it in shared memory.
__device__ __forceinline__ double sof_exp_mid(double x, const double* tab = kSofExpTabDev) {
  const double kd = rint(__dmul_rn(x, 0x1.71547652b82fep+6));
  const int k = (int)kd;
  double r = __fma_rn(-kd, 0x1.62e42fefa0000p-7, x);
  r = __fma_rn(-kd, 0x1.cf79abc9e3b3ap-46, r);
  double q = __fma_rn(r, 1.0 / 720.0, 1.0 / 120.0);
  q = __fma_rn(q, r, 1.0 / 24.0);
  q = __fma_rn(q, r, 1.0 / 6.0);
  q = __fma_rn(q, r, 0.5);
  const double p = __fma_rn(__dmul_rn(r, r), q, r);
  const int j = k & 63;
  const double2 t = reinterpret_cast<const double2*>(tab)[j];  // (hi, lo)
  const double y = __dadd_rn(t.x, __fma_rn(t.x, p, t.y));
  return __dmul_rn(y, sof_pow2i(k >> 6));
}

/// sof_exp_mid with its coefficients in the constant bank: every DFMA / DMUL takes its
/// constant as a c[bank][offset] operand instead of materialising a 64-bit immediate
/// through uniform-register moves (fewer issue slots per evaluation). Same operations,
/// same bits.
static __constant__ double kSofExpC[8] = {0x1.71547652b82fep+6, 0x1.62e42fefa0000p-7, 0x1.cf79abc9e3b3ap-46,
                                          1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0, 0.5};
/// the (hi, lo) table entry j: from a generic pointer, or from a shared-memory copy
/// addressed by its 32-bit shared-window address (no generic->shared conversion per use)
struct SofExpSmem {
  uint32_t addr;
};
__device__ __forceinline__ double2 sof_exp_entry(const double* tab, int j) {
  return reinterpret_cast<const double2*>(tab)[j];
}
__device__ __forceinline__ double2 sof_exp_entry(SofExpSmem tab, int j) {
  double2 t;
  asm("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(t.x), "=d"(t.y) : "r"(tab.addr + 16u * uint32_t(j)));
  return t;
}
template <typename Tab>
__device__ __forceinline__ double sof_exp_mid_cb(double x, Tab tab) {
  const double kd = rint(__dmul_rn(x, kSofExpC[0]));
  const int k = (int)kd;
  double r = __fma_rn(-kd, kSofExpC[1], x);
  r = __fma_rn(-kd, kSofExpC[2], r);
  double q = __fma_rn(r, kSofExpC[3], kSofExpC[4]);
  q = __fma_rn(q, r, kSofExpC[5]);
  q = __fma_rn(q, r, kSofExpC[6]);
  q = __fma_rn(q, r, kSofExpC[7]);
  const double p = __fma_rn(__dmul_rn(r, r), q, r);
  const double2 t = sof_exp_entry(tab, k & 63);  // (hi, lo)
  const double y = __dadd_rn(t.x, __fma_rn(t.x, p, t.y));
  return __dmul_rn(y, sof_pow2i(k >> 6));
}
#endif

/// natural log: x = 2^k m with m in [sqrt(2)/2, sqrt(2)), f = m - 1,
/// s = f / (2 + f), log(1+f) = f - hfsq + s (hfsq + R(s^2)) with the classic
/// minimax coefficients for R (fdlibm's Lg1..Lg7), k ln2 split hi/lo.
SOF_HD double sof_log(double x) {
  if (x != x) return SOF_ADD(x, x);
  if (x < 0.0) return sof_bits_to_double(0x7ff8000000000000ull);
  if (x == 0.0) return sof_bits_to_double(0xfff0000000000000ull);
  if (x > 1.7976931348623157e308) return x;  // +inf
  int k = 0;
  uint64_t u = sof_double_to_bits(x);
  if ((u >> 52) == 0) {  // subnormal: scale by 2^54 (exact)
    x = SOF_MUL(x, 18014398509481984.0);
    u = sof_double_to_bits(x);
    k = -54;
  }
  k += (int)(u >> 52) - 1023;
  u = (u & 0x000fffffffffffffull) | 0x3ff0000000000000ull;  // m in [1, 2)
  if (u > 0x3ff6a09e667f3bcdull) {                           // m > sqrt(2): halve (exact)
    u -= 0x0010000000000000ull;
    k += 1;
  }
  const double m = sof_bits_to_double(u);
  const double f = SOF_SUB(m, 1.0);
  const double kLg1 = 6.666666666666735130e-01, kLg2 = 3.999999999940941908e-01,
               kLg3 = 2.857142874366239149e-01, kLg4 = 2.222219843214978396e-01,
               kLg5 = 1.818357216161805012e-01, kLg6 = 1.531383769920937332e-01,
               kLg7 = 1.479819860511658591e-01;
  const double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
  const double s = SOF_DIV(f, SOF_ADD(2.0, f));
  const double z = SOF_MUL(s, s);
  double R = kLg7;
  R = SOF_FMA(R, z, kLg6);
  R = SOF_FMA(R, z, kLg5);
  R = SOF_FMA(R, z, kLg4);
  R = SOF_FMA(R, z, kLg3);
  R = SOF_FMA(R, z, kLg2);
  R = SOF_FMA(R, z, kLg1);
  R = SOF_MUL(R, z);
  const double hfsq = SOF_MUL(SOF_MUL(0.5, f), f);
  const double dk = (double)k;
  // log = k ln2_hi + (f - (hfsq - (s (hfsq + R) + k ln2_lo)))
  const double t = SOF_FMA(s, SOF_ADD(hfsq, R), SOF_MUL(dk, kLn2Lo));
  return SOF_ADD(SOF_MUL(dk, kLn2Hi), SOF_SUB(f, SOF_SUB(hfsq, t)));
}
