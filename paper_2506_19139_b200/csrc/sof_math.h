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

/// e^x: Cody-Waite reduction x = n ln2 + r (|r| <= ln2/2, two fma steps),
/// e^r = 1 + (r + r^2 q(r)) with a degree-11 Taylor tail in Horner form, then
/// an exact (or single-rounding, for subnormal results) scale by 2^n.
SOF_HD double sof_exp(double x) {
  if (x != x) return SOF_ADD(x, x);
  if (x > 709.782712893383973096) return sof_bits_to_double(0x7ff0000000000000ull);
  if (x < -745.1332191019412076235) return 0.0;
  const double kInvLn2 = 1.44269504088896338700e+00;
  const double kLn2Hi = 6.93147180369123816490e-01;  // 32 significant bits
  const double kLn2Lo = 1.90821492927058770002e-10;
  const double n = SOF_RINT(SOF_MUL(x, kInvLn2));
  double r = SOF_FMA(-n, kLn2Hi, x);
  r = SOF_FMA(-n, kLn2Lo, r);
  // q(r) = sum_{k>=2} r^(k-2) / k!   (k = 2..13)
  double q = 1.0 / 6227020800.0;            // 1/13!
  q = SOF_FMA(q, r, 1.0 / 479001600.0);     // 1/12!
  q = SOF_FMA(q, r, 1.0 / 39916800.0);      // 1/11!
  q = SOF_FMA(q, r, 1.0 / 3628800.0);       // 1/10!
  q = SOF_FMA(q, r, 1.0 / 362880.0);        // 1/9!
  q = SOF_FMA(q, r, 1.0 / 40320.0);         // 1/8!
  q = SOF_FMA(q, r, 1.0 / 5040.0);          // 1/7!
  q = SOF_FMA(q, r, 1.0 / 720.0);           // 1/6!
  q = SOF_FMA(q, r, 1.0 / 120.0);           // 1/5!
  q = SOF_FMA(q, r, 1.0 / 24.0);            // 1/4!
  q = SOF_FMA(q, r, 1.0 / 6.0);             // 1/3!
  q = SOF_FMA(q, r, 0.5);                   // 1/2!
  const double p = SOF_FMA(SOF_MUL(r, r), q, r);  // e^r - 1
  const double y = SOF_ADD(1.0, p);
  int ni = (int)n;
  if (ni > 1023) return SOF_MUL(SOF_MUL(y, 2.0), sof_pow2i(ni - 1));
  if (ni < -1020) return SOF_MUL(SOF_MUL(y, sof_pow2i(ni + 1000)), sof_pow2i(-1000));
  return SOF_MUL(y, sof_pow2i(ni));
}

#ifdef __CUDACC__
// sof_exp's constants in constant memory: the DFMAs of sof_exp_mid take them as
// c-bank operands instead of materialising each one with two uniform moves.
static __constant__ double kSofExpC[15] = {
    1.44269504088896338700e+00, 6.93147180369123816490e-01, 1.90821492927058770002e-10,
    1.0 / 6227020800.0, 1.0 / 479001600.0, 1.0 / 39916800.0, 1.0 / 3628800.0, 1.0 / 362880.0,
    1.0 / 40320.0,      1.0 / 5040.0,      1.0 / 720.0,      1.0 / 120.0,     1.0 / 24.0,
    1.0 / 6.0,          0.5};

/// sof_exp for -700 <= x <= 700 (finite): the same operation sequence without the
/// special cases, which cannot occur in this range (|n| <= 1010), so the result is
/// bit-identical to sof_exp(x).
__device__ __forceinline__ double sof_exp_mid(double x) {
  const double n = rint(__dmul_rn(x, kSofExpC[0]));
  double r = __fma_rn(-n, kSofExpC[1], x);
  r = __fma_rn(-n, kSofExpC[2], r);
  double q = kSofExpC[3];
#pragma unroll
  for (int k = 4; k < 15; ++k) q = __fma_rn(q, r, kSofExpC[k]);
  const double p = __fma_rn(__dmul_rn(r, r), q, r);
  const double y = __dadd_rn(1.0, p);
  return __dmul_rn(y, sof_pow2i((int)n));
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
