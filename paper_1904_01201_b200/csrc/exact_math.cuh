// exact_math.cuh -- IEEE-exact scalar helpers shared by host and device.
//
// The reference (navsim, pure Python + numba) computes every hot-path scalar
// in binary64 with round-to-nearest and NO fused multiply-add: numba compiles
// its kernels without fastmath (pkg/src/navsim/_kernels.py:1-5), and the
// Python glue uses plain float ops.  nvcc contracts a*b+c into DFMA by
// default, so every expression whose rounding must match the reference is
// written here with explicit _rn operations, which nvcc never contracts.
//
// Transcendentals: the reference calls glibc cos/sin/hypot through Python's
// math module / numpy (src/sensors.py:100-101, src/sim.py:98-99, :112).
// CUDA's libdevice versions are accurate to 1-2 ulp, not correctly rounded,
// so we evaluate cos/sin/hypot in double-double arithmetic and round once:
// the result is the correctly rounded value, which is what glibc returns for
// all but a vanishing fraction of inputs (checked in tests/test_exact_math.py).
#pragma once

#include <math.h>
#include <stdint.h>

#if defined(__CUDACC__)
#define NV_HD __host__ __device__ __forceinline__
#else
#define NV_HD static inline
#endif

namespace nvx {

// ---------------------------------------------------------------- basic ops
#if defined(__CUDA_ARCH__)
NV_HD double add(double a, double b) { return __dadd_rn(a, b); }
NV_HD double sub(double a, double b) { return __dsub_rn(a, b); }
NV_HD double mul(double a, double b) { return __dmul_rn(a, b); }
NV_HD double div(double a, double b) { return __ddiv_rn(a, b); }
NV_HD double sqrt_rn(double a) { return __dsqrt_rn(a); }
NV_HD double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
// host: compiled with -ffp-contract=off, so plain operators are exact IEEE ops
NV_HD double add(double a, double b) { return a + b; }
NV_HD double sub(double a, double b) { return a - b; }
NV_HD double mul(double a, double b) { return a * b; }
NV_HD double div(double a, double b) { return a / b; }
NV_HD double sqrt_rn(double a) { return sqrt(a); }
NV_HD double fma_rn(double a, double b, double c) { return fma(a, b, c); }
#endif

// ----------------------------------------------------------- double-double
struct dd {
  double hi, lo;
};

NV_HD dd two_sum(double a, double b) {
  double s = add(a, b);
  double bb = sub(s, a);
  double e = add(sub(a, sub(s, bb)), sub(b, bb));
  return {s, e};
}
NV_HD dd fast_two_sum(double a, double b) {  // |a| >= |b|
  double s = add(a, b);
  double e = sub(b, sub(s, a));
  return {s, e};
}
NV_HD dd two_prod(double a, double b) {
  double p = mul(a, b);
  double e = fma_rn(a, b, -p);
  return {p, e};
}
NV_HD dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  dd t = two_sum(a.lo, b.lo);
  s.lo = add(s.lo, t.hi);
  s = fast_two_sum(s.hi, s.lo);
  s.lo = add(s.lo, t.lo);
  return fast_two_sum(s.hi, s.lo);
}
NV_HD dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo = add(p.lo, add(mul(a.hi, b.lo), mul(a.lo, b.hi)));
  return fast_two_sum(p.hi, p.lo);
}

// 1/n! as double-double, n = 0..27 (generated with fractions.Fraction)
NV_HD dd invfact(int n) {
  // switch keeps the table in registers/immediates on device (no local memory)
  switch (n) {
#define NVX_CASE(k, h, l) case k: return {h, l};
    NVX_CASE(0, 0x1.0000000000000p+0, 0.0)
    NVX_CASE(1, 0x1.0000000000000p+0, 0.0)
    NVX_CASE(2, 0x1.0000000000000p-1, 0.0)
    NVX_CASE(3, 0x1.5555555555555p-3, 0x1.5555555555555p-57)
    NVX_CASE(4, 0x1.5555555555555p-5, 0x1.5555555555555p-59)
    NVX_CASE(5, 0x1.1111111111111p-7, 0x1.1111111111111p-63)
    NVX_CASE(6, 0x1.6c16c16c16c17p-10, -0x1.f49f49f49f49fp-65)
    NVX_CASE(7, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-73)
    NVX_CASE(8, 0x1.a01a01a01a01ap-16, 0x1.a01a01a01a01ap-76)
    NVX_CASE(9, 0x1.71de3a556c734p-19, -0x1.c154f8ddc6c00p-73)
    NVX_CASE(10, 0x1.27e4fb7789f5cp-22, 0x1.cbbc05b4fa99ap-76)
    NVX_CASE(11, 0x1.ae64567f544e4p-26, -0x1.c062e06d1f209p-80)
    NVX_CASE(12, 0x1.1eed8eff8d898p-29, -0x1.2aec959e14c06p-83)
    NVX_CASE(13, 0x1.6124613a86d09p-33, 0x1.f28e0cc748ebep-87)
    NVX_CASE(14, 0x1.93974a8c07c9dp-37, 0x1.05d6f8a2efd1fp-92)
    NVX_CASE(15, 0x1.ae7f3e733b81fp-41, 0x1.1d8656b0ee8cbp-97)
    NVX_CASE(16, 0x1.ae7f3e733b81fp-45, 0x1.1d8656b0ee8cbp-101)
    NVX_CASE(17, 0x1.952c77030ad4ap-49, 0x1.ac981465ddc6cp-103)
    NVX_CASE(18, 0x1.6827863b97d97p-53, 0x1.eec01221a8b0bp-107)
    NVX_CASE(19, 0x1.2f49b46814157p-57, 0x1.2650f61dbdcb4p-112)
    NVX_CASE(20, 0x1.e542ba4020225p-62, 0x1.ea72b4afe3c2fp-120)
    NVX_CASE(21, 0x1.71b8ef6dcf572p-66, -0x1.d043ae40c4647p-120)
    NVX_CASE(22, 0x1.0ce396db7f853p-70, -0x1.aebcdbd20331cp-124)
    NVX_CASE(23, 0x1.761b41316381ap-75, -0x1.3423c7d91404fp-130)
    NVX_CASE(24, 0x1.f2cf01972f578p-80, -0x1.9ada5fcc1ab14p-135)
    NVX_CASE(25, 0x1.3f3ccdd165fa9p-84, -0x1.58ddadf344487p-139)
    NVX_CASE(26, 0x1.88e85fc6a4e5ap-89, -0x1.71c37ebd16540p-143)
    NVX_CASE(27, 0x1.d1ab1c2dccea3p-94, 0x1.054d0c78aea14p-149)
#undef NVX_CASE
    default: return {0.0, 0.0};
  }
}

// sin(r), cos(r) for |r| <= pi/4 (+margin), r given as double-double.
NV_HD void dd_sincos_kernel(dd r, dd* s, dd* c) {
  dd r2 = dd_mul(r, r);
  // sin(r)/r = sum_k (-1)^k r^2k/(2k+1)!, cos(r) = sum_k (-1)^k r^2k/(2k)!,
  // k = 0..13: truncation error < 2^-110 relative for |r| <= pi/4.
  dd ps = {0.0, 0.0};
  dd pc = {0.0, 0.0};
#pragma unroll
  for (int k = 13; k >= 0; --k) {
    dd cs = invfact(2 * k + 1);
    dd cc = invfact(2 * k);
    if (k & 1) { cs.hi = -cs.hi; cs.lo = -cs.lo; cc.hi = -cc.hi; cc.lo = -cc.lo; }
    ps = dd_add(dd_mul(ps, r2), cs);
    pc = dd_add(dd_mul(pc, r2), cc);
  }
  *s = dd_mul(ps, r);
  *c = pc;
}

// Correctly rounded (up to a ~2^-100 relative DD error) sin and cos of x.
// Valid for |x| < 2^19; larger arguments never occur on the hot path
// (headings are wrapped to (-pi, pi] by wrap_angle, src/geometry.py:19-24).
NV_HD void sincos_cr(double x, double* sn, double* cs) {
  const double p1 = 0x1.921fb54400000p+0;   // pi/2, first 33 bits
  const double p2 = 0x1.0b4611a626331p-34;  // next 53 bits
  const double p3 = 0x1.1701b839a2520p-88;  // next 53 bits
  const double two_over_pi = 0x1.45f306dc9c883p-1;
  double kd = rint(mul(x, two_over_pi));
  // a = x - k*p1 is exact: k*p1 has <= 53 bits for |k| < 2^20 and the
  // subtraction cancels (Sterbenz) whenever k != 0.
  double a = sub(x, mul(kd, p1));
  dd b = two_prod(kd, p2);
  dd r = two_sum(a, -b.hi);
  r.lo = sub(sub(r.lo, b.lo), mul(kd, p3));
  r = fast_two_sum(r.hi, r.lo);
  dd s, c;
  dd_sincos_kernel(r, &s, &c);
  long long k = (long long)kd;
  int q = (int)(k & 3);
  double sv = add(s.hi, s.lo), cv = add(c.hi, c.lo);
  switch (q) {
    case 0: *sn = sv;  *cs = cv;  break;
    case 1: *sn = cv;  *cs = -sv; break;
    case 2: *sn = -sv; *cs = -cv; break;
    default: *sn = -cv; *cs = sv; break;
  }
}

// Correctly rounded hypot for moderate magnitudes (no scaling needed for the
// agent-step values, |x|,|y| <= forward_step).  np.hypot -> glibc hypot.
NV_HD double hypot_cr(double x, double y) {
  dd xx = two_prod(x, x);
  dd yy = two_prod(y, y);
  dd s = dd_add(xx, yy);
  if (s.hi == 0.0) return 0.0;
  double r = sqrt_rn(s.hi);
  // residual s - r^2 in double-double, then one Newton correction
  double e = fma_rn(-r, r, s.hi);
  double rem = add(e, s.lo);
  return add(r, div(rem, mul(2.0, r)));
}

// wrap_angle (src/geometry.py:19-24): fmod is exact in IEEE arithmetic.
NV_HD double wrap_angle(double theta) {
  const double PI = 3.141592653589793;
  const double TWO_PI = 6.283185307179586;
  double out = fmod(add(theta, PI), TWO_PI);
  if (out <= 0.0) out = add(out, TWO_PI);
  return sub(out, PI);
}

}  // namespace nvx
