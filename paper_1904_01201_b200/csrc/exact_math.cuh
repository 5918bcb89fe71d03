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

// sin(j/64), cos(j/64) for j = 0..51 as double-doubles {sin.hi, sin.lo,
// cos.hi, cos.lo} (generated with mpmath at 300 bits): the table of the
// argument reduction r = j/64 + t, |t| <= 1/128, of sincos_cr.
#define NVX_SINCOS_TABLE \
  {0x0.0p+0, 0x0.0p+0, 0x1.0000000000000p+0, 0x0.0p+0}, \
  {0x1.fffaaaaeeeed5p-7, -0x1.2ab639a9f0776p-63, 0x1.fff000155549fp-1, 0x1.28a28a03a5ef3p-55}, \
  {0x1.ffeaaaeeee86fp-6, -0x1.cd406fb224ae2p-60, 0x1.ffc00155527d3p-1, -0x1.3b54492d89b5bp-55}, \
  {0x1.7fdc01032fba9p-5, -0x1.599bdf46e997ap-59, 0x1.ff7006bfdf99fp-1, -0x1.8b3b560648d5fp-56}, \
  {0x1.ffaaaeeed4edbp-5, -0x1.2d16d32684b69p-59, 0x1.ff0015549f4d3p-1, 0x1.328387b99426fp-55}, \
  {0x1.3facb12d1755bp-4, -0x1.921915299468bp-58, 0x1.fe7034129ef6fp-1, -0x1.cbf4337c96f97p-57}, \
  {0x1.7f701032550e4p-4, 0x1.afc2d1800501ap-60, 0x1.fdc06bf7e6b9bp-1, 0x1.31902b535f8dbp-55}, \
  {0x1.bf1b78568391dp-4, 0x1.e91841dea4cc8p-58, 0x1.fcf0c800e99b1p-1, 0x1.ea3d786d186acp-57}, \
  {0x1.feaaeee86ee36p-4, -0x1.afcb2bcc6f03bp-59, 0x1.fc015527d5bd3p-1, 0x1.b68f35094efb8p-55}, \
  {0x1.1f0d3d7afceafp-3, -0x1.6ef95099769a5p-57, 0x1.faf22263c4bd3p-1, -0x1.52ace133a2769p-58}, \
  {0x1.3eb312c5d66cbp-3, 0x1.47d666b66cb91p-57, 0x1.f9c340a7cc428p-1, 0x1.c5b6b063b7462p-55}, \
  {0x1.5e44fcfa126f3p-3, -0x1.6f443063f89b6p-57, 0x1.f874c2e1eecf6p-1, -0x1.c6514e1332b16p-55}, \
  {0x1.7dc102fbaf2b5p-3, 0x1.5ab50e23c97c3p-59, 0x1.f706bdf9ece1cp-1, -0x1.698c80c36dcb4p-55}, \
  {0x1.9d252d0cec312p-3, 0x1.9c43d80b1137dp-58, 0x1.f57948cff6797p-1, 0x1.e3a0d3e03b1d4p-57}, \
  {0x1.bc6f84edc6199p-3, 0x1.9c1a56a7b0cabp-57, 0x1.f3cc7c3b3d16ep-1, -0x1.21a3ad28a3494p-57}, \
  {0x1.db9e15fb5a5d0p-3, -0x1.32e20d6cc6fc2p-57, 0x1.f20073086649fp-1, 0x1.b940416c1984bp-56}, \
  {0x1.faaeed4f31577p-3, -0x1.15d88508e32b8p-57, 0x1.f01549f7deea1p-1, 0x1.d3c1e99e5cafdp-55}, \
  {0x1.0cd00cef36436p-2, -0x1.9fb0a0c93e2b4p-56, 0x1.ee0b1fbc0f11cp-1, -0x1.bfd2380bbc3b1p-59}, \
  {0x1.1c37d64c6b876p-2, 0x1.46076fe0dcff4p-56, 0x1.ebe214f76efa8p-1, -0x1.02f9f12ba543ep-55}, \
  {0x1.2b8ddc43eb49fp-2, 0x1.1553899f2d807p-57, 0x1.e99a4c3a7cd83p-1, -0x1.2264b1bc53ce8p-55}, \
  {0x1.3ad129769d3d8p-2, 0x1.03d550487839ap-63, 0x1.e733ea0193d40p-1, -0x1.6428b3546ce13p-55}, \
  {0x1.4a00c9b0f3d20p-2, 0x1.823ba6bb08eadp-56, 0x1.e4af14b2a449cp-1, -0x1.68ca02e8a6833p-55}, \
  {0x1.591bc9fa2f597p-2, 0x1.7c74bac3fe0cbp-57, 0x1.e20bf49acd6c1p-1, -0x1.660aec7ef636bp-58}, \
  {0x1.682138a38d7f7p-2, -0x1.d889202444aadp-56, 0x1.df4ab3ebd875ep-1, -0x1.e2d8a7e6736c4p-55}, \
  {0x1.7710255764214p-2, -0x1.6ead7314bb6cep-57, 0x1.dc6b7eb995912p-1, 0x1.4b364776dcd35p-58}, \
  {0x1.85e7a12826949p-2, 0x1.8a40e9b5face0p-56, 0x1.d96e82f71a9dcp-1, 0x1.ff61bd5d2039dp-55}, \
  {0x1.94a6be9f546c5p-2, -0x1.69ce13e683f58p-56, 0x1.d653f073e4040p-1, -0x1.76236434bec37p-55}, \
  {0x1.a34c91cc50ccap-2, -0x1.a310e3b50cecdp-58, 0x1.d31bf8d8d7c06p-1, 0x1.e60dd3089cbddp-56}, \
  {0x1.b1d8305321617p-2, -0x1.ae242cb99f519p-56, 0x1.cfc6cfa52ad9fp-1, 0x1.8b5b5508f2a0dp-55}, \
  {0x1.c048b17b140a3p-2, 0x1.19fe6757e9fa7p-57, 0x1.cc54aa2b2972ep-1, 0x1.4ee162ba83a98p-57}, \
  {0x1.ce9d2e3d4a51fp-2, -0x1.2fc8a12dae298p-57, 0x1.c8c5bf8ce1a84p-1, 0x1.ab3d1a1590123p-56}, \
  {0x1.dcd4c15329c9ap-2, 0x1.0d4c6e171fd9ap-56, 0x1.c51a48b8b175ep-1, -0x1.1bbb43b9aa880p-57}, \
  {0x1.eaee8744b05f0p-2, -0x1.789b43c9b027dp-58, 0x1.c1528065b7d50p-1, -0x1.892111312e828p-55}, \
  {0x1.f8e99e76abc97p-2, 0x1.9d950af2d00a3p-58, 0x1.bd6ea310294f5p-1, 0x1.31bbcc88c109dp-56}, \
  {0x1.0362939c69955p-1, -0x1.2d8cd78397b01p-55, 0x1.b96eeef58840ep-1, 0x1.45a3cc78fade0p-58}, \
  {0x1.0a4021e9e1001p-1, -0x1.6f643a13914f6p-55, 0x1.b553a410c104ep-1, 0x1.8ff7947027a15p-58}, \
  {0x1.110d0c4b69c3bp-1, 0x1.d918998809981p-55, 0x1.b11d04162a4c6p-1, 0x1.1dd561efbc0c2p-56}, \
  {0x1.17c8e5f2eedb0p-1, 0x1.35e57102e2488p-57, 0x1.accb526f69de5p-1, 0x1.8fb6a8dd6b6ccp-55}, \
  {0x1.1e7343236574cp-1, 0x1.22a3fa4f41d5ap-56, 0x1.a85ed4373e02dp-1, 0x1.9be06385ec792p-57}, \
  {0x1.250bb93788bbbp-1, 0x1.ea3d02457bccep-56, 0x1.a3d7d0352bdcfp-1, -0x1.68dbaeca19669p-55}, \
  {0x1.2b91dea88421ep-1, -0x1.fa371db216ab0p-55, 0x1.9f368ed912f85p-1, -0x1.1d200c5791606p-55}, \
  {0x1.32054b148bc4fp-1, 0x1.f6b42095a135bp-55, 0x1.9a7b5a36a6514p-1, 0x1.722cfcc9fa7a9p-55}, \
  {0x1.386597456282bp-1, -0x1.10fada93b07a8p-56, 0x1.95a67e00cb1fdp-1, -0x1.0befda21f862dp-55}, \
  {0x1.3eb25d36cd53ap-1, -0x1.be570e1570fc0p-58, 0x1.90b84784ddaf7p-1, -0x1.0feb10ab93b87p-56}, \
  {0x1.44eb381cf386bp-1, -0x1.3ed6c1e6a5505p-55, 0x1.8bb105a5dc900p-1, 0x1.863e03e9474c1p-55}, \
  {0x1.4b0fc46aab761p-1, 0x1.0da05738cc59cp-61, 0x1.869108d77a6c6p-1, 0x1.338ffe2bfe9ddp-56}, \
  {0x1.511f9fd7b351cp-1, -0x1.5c0e861c48831p-55, 0x1.8158a31916d5dp-1, -0x1.de8b90b8228dep-57}, \
  {0x1.571a6966d59b3p-1, 0x1.c843b4d0fb197p-58, 0x1.7c0827f09e54fp-1, -0x1.c73d6d72aee68p-57}, \
  {0x1.5cffc16bf8f0dp-1, 0x1.96cb370eb578ap-55, 0x1.769fec655211fp-1, -0x1.827d5cf8c68c5p-57}, \
  {0x1.62cf49921ac79p-1, -0x1.edd9855b6241ap-55, 0x1.712046fa77678p-1, 0x1.425b0a5029c81p-55}, \
  {0x1.6888a4e134b2fp-1, -0x1.6b7d37644d5e6p-55, 0x1.6b898fa9efb5dp-1, 0x1.15ac786ccf4b2p-56}, \
  {0x1.6e2b77c40bde1p-1, -0x1.0e729857fad53p-56, 0x1.65dc1fdeb8cbap-1, -0x1.97c1b47337c77p-58}

#if defined(__CUDACC__)
__device__ __constant__ double nvx_sc_tab_dev[52][4] = {NVX_SINCOS_TABLE};
#endif
static const double nvx_sc_tab_host[52][4] = {NVX_SINCOS_TABLE};

NV_HD const double *sc_tab(int j) {
#if defined(__CUDA_ARCH__)
  return nvx_sc_tab_dev[j];
#else
  return nvx_sc_tab_host[j];
#endif
}

// sin(t), cos(t) for |t| <= 1/128 (+ rounding), t as double-double: the
// series' leading terms in double-double, the tail (relative weight <= 2^-35)
// in double; total relative error < 2^-87, so the final rounding to double
// is the correctly rounded one except with probability ~2^-34 per call.
NV_HD void dd_sincos_small(dd t, dd *s, dd *c) {
  const dd t2 = dd_mul(t, t);
  const double u = t2.hi;
  // sin(t) = t (1 + t2 (-1/6 + t2 (1/120 + t2 (-1/5040 + t2 (1/9! - t2/11!)))))
  const double ts = mul(u, add(-0x1.a01a01a01a01ap-13, mul(u, sub(0x1.71de3a556c734p-19,
                                                                 mul(u, 0x1.ae64567f544e4p-26)))));
  dd ps = dd_add(dd{0x1.1111111111111p-7, 0x1.1111111111111p-63}, dd{ts, 0.0});
  ps = dd_add(dd{-0x1.5555555555555p-3, -0x1.5555555555555p-57}, dd_mul(t2, ps));
  ps = dd_add(dd{1.0, 0.0}, dd_mul(t2, ps));
  *s = dd_mul(t, ps);
  // cos(t) = 1 + t2 (-1/2 + t2 (1/24 + t2 (-1/720 + t2 (1/8! - t2/10!))))
  const double tc = mul(u, add(-0x1.6c16c16c16c17p-10, mul(u, sub(0x1.a01a01a01a01ap-16,
                                                                 mul(u, 0x1.27e4fb7789f5cp-22)))));
  dd pc = dd_add(dd{0x1.5555555555555p-5, 0x1.5555555555555p-59}, dd{tc, 0.0});
  pc = dd_add(dd{-0.5, 0.0}, dd_mul(t2, pc));
  *c = dd_add(dd{1.0, 0.0}, dd_mul(t2, pc));
}

// Correctly rounded (up to the ~2^-87 relative error above) sin and cos of
// x.  x = k pi/2 + r (Cody-Waite, 3-part pi/2), r = j/64 + t with the
// double-double table of sin/cos(j/64), then the addition formulas.
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
  // r = j/64 + t: r.hi - j/64 is exact (|r.hi - j/64| <= 1/128, Sterbenz)
  const double jd = rint(mul(r.hi, 64.0));
  const int j = (int)jd;
  const dd t = two_sum(sub(r.hi, mul(jd, 0x1p-6)), r.lo);
  dd st, ct;
  dd_sincos_small(t, &st, &ct);
  dd s, c;
  if (j == 0) {
    s = st;
    c = ct;
  } else {
    const double *e = sc_tab(j < 0 ? -j : j);
    const double sg = j < 0 ? -1.0 : 1.0;  // sin(-a) = -sin(a), cos(-a) = cos(a)
    const dd sa = {sg * e[0], sg * e[1]}, ca = {e[2], e[3]};
    s = dd_add(dd_mul(sa, ct), dd_mul(ca, st));
    const dd m = dd_mul(sa, st);
    c = dd_add(dd_mul(ca, ct), dd{-m.hi, -m.lo});
  }
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
