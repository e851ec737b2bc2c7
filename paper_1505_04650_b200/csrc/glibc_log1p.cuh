// log1p(x) bit-identical to the C library the reference's numpy calls.
//
// numpy's Generator.standard_normal finishes a ziggurat tail draw with
// npy_log1p(-u), which is the C library's log1p. On x86-64 glibc (2.39 here)
// an ifunc selects the FMA build of the fdlibm algorithm
// (sysdeps/ieee754/dbl-64/s_log1p.c) when the CPU has FMA + AVX2; that build
// is not correctly rounded, and its result depends on exactly which products
// the compiler fused. This is a restatement of that published algorithm with
// every operation spelled out -- the fused ones as fma(), the others as
// separately rounded IEEE operations (never contracted) -- in the order the
// FMA build evaluates them, so device and host agree bit for bit
// (tests/test_gpu_parity.py compares against the host's log1p).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

namespace cnmf {
namespace l1p {

#ifdef __CUDA_ARCH__
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double fmad(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ uint64_t bits(double x) { return (uint64_t)__double_as_longlong(x); }
__device__ __forceinline__ double from_bits(uint64_t b) { return __longlong_as_double((long long)b); }
#else
// host build: the translation unit must not contract (it is only used by tests/tools)
inline double mul(double a, double b) { volatile double r = a * b; return r; }
inline double add(double a, double b) { volatile double r = a + b; return r; }
inline double sub(double a, double b) { volatile double r = a - b; return r; }
inline double div(double a, double b) { volatile double r = a / b; return r; }
inline double fmad(double a, double b, double c) { return std::fma(a, b, c); }
inline uint64_t bits(double x) { uint64_t b; std::memcpy(&b, &x, 8); return b; }
inline double from_bits(uint64_t b) { double x; std::memcpy(&x, &b, 8); return x; }
#endif

constexpr double kLn2Hi = 6.93147180369123816490e-01;  // 3fe62e42 fee00000
constexpr double kLn2Lo = 1.90821492927058770002e-10;  // 3dea39ef 35793c76
constexpr double kLp1 = 6.666666666666735130e-01;      // 3FE55555 55555593
constexpr double kLp2 = 3.999999999940941908e-01;      // 3FD99999 9997FA04
constexpr double kLp3 = 2.857142874366239149e-01;      // 3FD24924 94229359
constexpr double kLp4 = 2.222219843214978396e-01;      // 3FCC71C5 1D8E78AF
constexpr double kLp5 = 1.818357216161805012e-01;      // 3FC74664 96CB03DE
constexpr double kLp6 = 1.531383769920937332e-01;      // 3FC39A09 D078C69F
constexpr double kLp7 = 1.479819860511658591e-01;      // 3FC2F112 DF3E5244

#ifdef __CUDA_ARCH__
__device__
#endif
inline double with_high(double x, uint32_t hi) {
  return from_bits(((uint64_t)hi << 32) | (bits(x) & 0xffffffffull));
}

}  // namespace l1p

#ifdef __CUDA_ARCH__
__device__
#endif
inline double glibc_log1p(double x) {
  using namespace l1p;
  const int32_t hx = (int32_t)(bits(x) >> 32);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {                 // x < 0.41422
    if (ax >= 0x3ff00000) {              // x <= -1.0
      if (x == -1.0) return -INFINITY;
      return NAN;
    }
    if (ax < 0x3e200000) {               // |x| < 2^-29
      if (ax < 0x3c900000) return x;     // |x| < 2^-54
      return fmad(-mul(x, x), 0.5, x);   // x - (x*x)*0.5, one fused step
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {  // -0.2929 < x < 0.41422
      k = 0;
      f = x;
      hu = 1;
    }
  } else if (hx >= 0x7ff00000) {
    return add(x, x);
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = add(1.0, x);
      hu = (int32_t)(bits(u) >> 32);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? sub(1.0, sub(u, x)) : sub(x, sub(u, 1.0));  // correction term
      c = div(c, u);
    } else {
      u = x;
      hu = (int32_t)(bits(u) >> 32);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_high(u, (uint32_t)hu | 0x3ff00000u);  // normalise u
    } else {
      k += 1;
      u = with_high(u, (uint32_t)hu | 0x3fe00000u);  // normalise u / 2
      hu = (0x00100000 - hu) >> 2;
    }
    f = sub(u, 1.0);
  }
  const double hfsq = mul(mul(0.5, f), f);
  if (hu == 0) {  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = (double)k;
      return fmad(kd, kLn2Hi, fmad(kd, kLn2Lo, c));
    }
    const double R = mul(fmad(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return sub(f, R);
    const double kd = (double)k;
    return fmad(kd, kLn2Hi, -sub(sub(R, fmad(kd, kLn2Lo, c)), f));
  }
  const double s = div(f, add(f, 2.0));
  const double z = mul(s, s);
  const double r3 = fmad(z, kLp3, kLp2);
  const double r5 = fmad(z, kLp5, kLp4);
  const double r7 = fmad(z, kLp7, kLp6);
  const double z2 = mul(z, z);
  const double z4 = mul(z2, z2);
  const double z6 = mul(z2, z4);
  double R = fmad(z, kLp1, mul(z2, r3));
  R = fmad(z4, r5, R);
  R = fmad(z6, r7, R);
  const double t = mul(add(R, hfsq), s);
  if (k == 0) return sub(f, sub(hfsq, t));
  const double kd = (double)k;
  return fmad(kd, kLn2Hi, -sub(sub(hfsq, add(fmad(kd, kLn2Lo, c), t)), f));
}

}  // namespace cnmf
