// kernels.cuh -- sm_100a kernels of the navsim hot path.
//
//   k_agent_step   Simulator.step kinematics (sim.py:83-130), one warp / env:
//                  swept-disc casts (disc_cast, _kernels.py:393-465) over the
//                  grid candidates with a warp-lexicographic (t, idx) min.
//   k_column_cast  raycast_grid (_kernels.py:51-120), one thread / (env,
//                  column), exact FP64 DDA + segment test, then the column
//                  epilogue: exact FP64 row classification against the tc/tf
//                  tables (fill_frame's per-pixel compares, _kernels.py:141-170,
//                  restated as two binary searches per column) -> ColRec.
//   k_fill_tma     fill_frame's per-pixel resolve (_kernels.py:171-207) as a
//                  streaming writer: each warp renders whole rows into a
//                  private double-buffered shared-memory stage and its lane 0
//                  writes them out with cp.async.bulk (TMA bulk) stores,
//                  evict-first in L2; work is pulled from a global counter.
//   k_fill_generic the same resolve, one thread per pixel, any W/H.
//
// Exactness: every FP64 operation that decides coverage, semantics, depth or
// pose uses the nvx:: _rn helpers (no FMA contraction), replicating the
// reference's operation order.  Shading is FP32 (RGB tolerance 1/255).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include "device.cuh"
#include "exact_math.cuh"

namespace nvk {

using namespace nvd;
using nvx::add;
using nvx::div;
using nvx::mul;
using nvx::sub;

#define NV_INF CUDART_INF

// ---------------------------------------------------------------- helpers

// SegmentIndex._cell_of (geometry.py:146-149): trunc toward zero, clamp.
__device__ __forceinline__ int cell_coord(double v, double o, int n) {
  double d = sub(v, o);  // (v - o) / CELL with CELL = 1.0: division by 1 is exact
  if (!(d >= 1.0)) return 0;
  if (d >= (double)(n - 1)) return n - 1;
  return (int)d;
}

// One segment test of raycast_grid / raycast_all (_kernels.py:91-103), split
// into a division-free prefilter and the exact IEEE path.  The prefilter only
// rejects a segment when the reference's own checks would `continue` on it:
//   t < 0     <=> sign(tn) != sign(den), tn != 0 (tn = +-0 gives t = +-0,
//               which passes `t < 0.0`);
//   r < 0     likewise with rn;
//   r > 1     if |rn| > |den| (1 + 1e-12): RN(rn/den) > 1;
//   t > best  if |tn| > |den| best (1 + 1e-12): RN(tn/den) > best.
// (Exact for coordinates whose products do not underflow, i.e. any scene
// with |coordinates| and segment lengths in [2^-400, 2^400].)  The exact path
// is the reference's arithmetic and update rule, a lexicographic (t, idx)
// minimum, so the order in which candidates are tested is irrelevant.
#define NV_R1 1.0000000000010

__device__ __forceinline__ bool seg_pre(double px, double py, double dx, double dy,
                                        double ax, double ay, double ex, double ey,
                                        double best_t, double &den, double &tn, double &rn) {
  den = sub(mul(dx, ey), mul(dy, ex));
  double sx = sub(ax, px), sy = sub(ay, py);
  tn = sub(mul(sx, ey), mul(sy, ex));
  rn = sub(mul(sx, dy), mul(sy, dx));
  const bool neg = den < 0.0;
  const double aden = fabs(den);
  bool ok = den != 0.0;
  ok &= !(tn != 0.0 && ((tn < 0.0) != neg));
  ok &= !(rn != 0.0 && ((rn < 0.0) != neg));
  ok &= !(fabs(rn) > aden * NV_R1);
  ok &= !(fabs(tn) > aden * best_t * NV_R1);
  return ok;
}

__device__ __forceinline__ void seg_exact(double den, double tn, double rn, int i,
                                          double &best_t, int &best_i) {
  double t = div(tn, den);
  if (t < 0.0 || t > best_t) return;
  double r = div(rn, den);
  if (0.0 <= r && r <= 1.0) {
    if (t < best_t || i < best_i) {
      best_t = t;
      best_i = i;
    }
  }
}

__device__ __forceinline__ void seg_test(double px, double py, double dx, double dy,
                                         double ax, double ay, double ex, double ey,
                                         int i, double &best_t, int &best_i) {
  double den, tn, rn;
  if (seg_pre(px, py, dx, dy, ax, ay, ex, ey, best_t, den, tn, rn))
    seg_exact(den, tn, rn, i, best_t, best_i);
}

// Tests the bucket run [q0, q1) of one cell, NB entries per round with all
// loads issued up front (memory-level parallelism); indices past the end are
// clamped to q1-1 -- re-testing a segment cannot change a lexicographic min.
template <int NB>
__device__ __forceinline__ void test_cell(const SceneView &sc, int q0, int q1, double px,
                                          double py, double dx, double dy, double &best_t,
                                          int &best_i) {
  for (int q = q0; q < q1; q += NB) {
    double2 a[NB], e[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const int qq = min(q + k, q1 - 1);
      const double2 *p2 = reinterpret_cast<const double2 *>(sc.ent + qq);
      a[k] = __ldg(p2);
      e[k] = __ldg(p2 + 1);
    }
    double den[NB], tn[NB], rn[NB];
    bool ok[NB];
    bool any = false;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      ok[k] = seg_pre(px, py, dx, dy, a[k].x, a[k].y, e[k].x, e[k].y, best_t, den[k], tn[k],
                      rn[k]);
      any |= ok[k];
    }
    if (any) {
#pragma unroll
      for (int k = 0; k < NB; ++k)
        if (ok[k]) seg_exact(den[k], tn[k], rn[k], __ldg(sc.items + min(q + k, q1 - 1)), best_t,
                             best_i);
    }
  }
}

// FP32 prefilter for one cell of the DDA (side test).  The ray's line
// crosses segment [a, b] iff a and b are not strictly on the same side:
// with s_a = d x (a - p) and s_b = d x (b - p), the reference's
// r = rn/den = s_a / (s_a - s_b), so both s_a, s_b > 0 (or both < 0) means
// r < 0 or r > 1 (or den == 0) and the reference skips the segment.
// Entries are stored in f32 relative to the cell anchor (X0c, Y0c) =
// (x0 + cx, y0 + cy); the ray origin is rebased to the same anchor in f64
// and rounded once.  E = 2^-18 |d|_1 (A + |p_rel|_1) bounds the f32 error of
// s_a, s_b (conversions, products, sums; ~8x over the worst case) and the
// reference's own f64 rounding, so a segment is skipped only when it is
// certain that the reference skips it.  Survivors -- the segments the ray's
// line actually crosses, plus a hairline margin -- take the exact FP64 test,
// so the result is bit-identical to the unfiltered DDA.
#define NV_K32 0x1p-18f

struct CellF {
  float cp, E;  // d x p_rel, error bound
};

__device__ __forceinline__ CellF cell_f32(const SceneView &sc, int cx, int cy, int c, double px,
                                          double py, float dxf, float dyf, float sd) {
  const double X0 = add(sc.x0, (double)cx), Y0 = add(sc.y0, (double)cy);
  const float pxr = (float)sub(px, X0), pyr = (float)sub(py, Y0);
  CellF f;
  f.cp = fmaf(dxf, pyr, -(dyf * pxr));
  f.E = NV_K32 * sd * (__ldg(sc.cellb + c) + fabsf(pxr) + fabsf(pyr) + 1e-30f);
  return f;
}

// Tests the bucket run [q0, q1) of one cell: NB f32 side tests per round
// (loads issued up front), then the exact FP64 test for the survivors.
template <int NB>
__device__ __forceinline__ void test_cell_f32(const SceneView &sc, int q0, int q1,
                                              const CellF &cf, double px, double py, double dx,
                                              double dy, float dxf, float dyf, double &best_t,
                                              int &best_i) {
  for (int q = q0; q < q1; q += NB) {
    float4 e[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) e[k] = __ldg(sc.entf + min(q + k, q1 - 1));
    unsigned keep = 0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const float sa = fmaf(dxf, e[k].y, -(dyf * e[k].x)) - cf.cp;
      const float sb = fmaf(dxf, e[k].w, -(dyf * e[k].z)) - cf.cp;
      const bool skip = fminf(sa, sb) > cf.E || fmaxf(sa, sb) < -cf.E;
      keep |= (skip ? 0u : 1u) << k;
    }
    while (keep) {
      const int k = __ffs(keep) - 1;
      keep &= keep - 1;
      const int qq = min(q + k, q1 - 1);
      const double2 *p2 = reinterpret_cast<const double2 *>(sc.ent + qq);
      const double2 a2 = __ldg(p2), e2 = __ldg(p2 + 1);
      double den, tn, rn;
      if (seg_pre(px, py, dx, dy, a2.x, a2.y, e2.x, e2.y, best_t, den, tn, rn))
        seg_exact(den, tn, rn, __ldg(sc.items + qq), best_t, best_i);
    }
  }
}

// raycast_grid (_kernels.py:51-120), one ray, exact replica of the DDA.
// The walk is software-pipelined: the next cell's record {q0, q1, bound} is
// loaded (one 16-byte load) before the current cell's entries are tested, so
// the cell-to-cell latency overlaps the tests; the visit order and the
// early-out are the reference's.
#ifndef NV_CAST_NB
#define NV_CAST_NB 8
#endif
#ifndef NV_CAST_CHUNKS
#define NV_CAST_CHUNKS 1
#endif
#ifndef NV_CAST_PF_NEXT
#define NV_CAST_PF_NEXT 0  // L1 prefetch of the next cell's runs (no gain measured)
#endif
#ifndef NV_CAST_NCB
#define NV_CAST_NCB 4  // run boxes loaded per round
#endif
__device__ __forceinline__ void ray_grid(const SceneView &sc, double px, double py,
                                         double dx, double dy, double t_max,
                                         double &out_t, int &out_i) {
  const double cell = 1.0;
  double best_t = NV_INF;
  int best_i = -1;
  if (isnan(px) || isnan(py) || isnan(dx) || isnan(dy)) {  // reference would spin
    out_t = best_t;
    out_i = best_i;
    return;
  }
  // (p - x0) / cell with cell = 1.0 is exact without the division
  long long cx = (long long)floor(sub(px, sc.x0));
  long long cy = (long long)floor(sub(py, sc.y0));
  const int stepx = dx > 0.0 ? 1 : -1;
  const int stepy = dy > 0.0 ? 1 : -1;
  double tnx, tdx, tny, tdy;
  if (dx != 0.0) {
    double nbx = add(sc.x0, mul((double)(cx + (dx > 0.0 ? 1 : 0)), cell));
    tnx = div(sub(nbx, px), dx);
    tdx = fabs(div(cell, dx));
  } else {
    tnx = NV_INF;
    tdx = NV_INF;
  }
  if (dy != 0.0) {
    double nby = add(sc.y0, mul((double)(cy + (dy > 0.0 ? 1 : 0)), cell));
    tny = div(sub(nby, py), dy);
    tdy = fabs(div(cell, dy));
  } else {
    tny = NV_INF;
    tdy = NV_INF;
  }
  const long long gnx = sc.gnx, gny = sc.gny;
  const float dxf = (float)dx, dyf = (float)dy;
  const float sd = (fabsf(dxf) + fabsf(dyf)) * (1.0f + 0x1p-20f);
  const bool pos_dx = dxf >= 0.0f, pos_dy = dyf >= 0.0f;
  (void)pos_dx; (void)pos_dy;
  auto inb = [&](long long x, long long y) { return 0 <= x && x < gnx && 0 <= y && y < gny; };
  int4 rec = make_int4(0, 0, 0, 0);
  if (inb(cx, cy)) rec = __ldg(sc.cells + (cy * gnx + cx));
  for (int guard = 0; guard < (1 << 24); ++guard) {
    const double t_exit = tnx < tny ? tnx : tny;
    // the cell after this one (the reference advances to it unless it stops)
    long long ncx = cx, ncy = cy;
    double ntnx = tnx, ntny = tny;
    if (tnx < tny) {
      ncx += stepx;
      ntnx = add(tnx, tdx);
    } else {
      ncy += stepy;
      ntny = add(tny, tdy);
    }
    int4 nrec = make_int4(0, 0, 0, 0);
    if (!(t_exit > t_max) && inb(ncx, ncy)) nrec = __ldg(sc.cells + (ncy * gnx + ncx));
    if (rec.y > rec.x) {
      const double X0 = add(sc.x0, (double)cx), Y0 = add(sc.y0, (double)cy);
      const float pxr = (float)sub(px, X0), pyr = (float)sub(py, Y0);
      CellF cf;
      cf.cp = fmaf(dxf, pyr, -(dyf * pxr));
      cf.E = NV_K32 * sd * (__int_as_float(rec.z) + fabsf(pxr) + fabsf(pyr) + 1e-30f);
#if NV_CAST_CHUNKS
      // s(x, y) = d x ((x, y) - p) is linear, so over a run's box it is
      // bounded by two corners; a run whose box lies beyond +-E on one side
      // holds no entry the per-entry side test would keep.
      // The boxes of up to NV_CAST_NCB runs are loaded together (one memory
      // round trip per cell in the common case); a passing run's f64 entries
      // are prefetched into L1 before its f32 side tests, so the exact tests
      // of its survivors hit L1.
      const int nch = (rec.y - rec.x + NV_CHUNK - 1) / NV_CHUNK;
      for (int c0 = 0; c0 < nch; c0 += NV_CAST_NCB) {
        float4 bb[NV_CAST_NCB];
#pragma unroll
        for (int k = 0; k < NV_CAST_NCB; ++k) bb[k] = __ldg(sc.chunks + rec.w + min(c0 + k, nch - 1));
        unsigned pass = 0;
#pragma unroll
        for (int k = 0; k < NV_CAST_NCB; ++k) {
          const float4 b = bb[k];
          const float smin = fmaf(dxf, pos_dx ? b.y : b.w, -(dyf * (pos_dy ? b.z : b.x))) - cf.cp;
          const float smax = fmaf(dxf, pos_dx ? b.w : b.y, -(dyf * (pos_dy ? b.x : b.z))) - cf.cp;
          const bool ok = c0 + k < nch && !(smin > cf.E || smax < -cf.E);
          pass |= (ok ? 1u : 0u) << k;
        }
        for (unsigned m = pass; m; m &= m - 1) {  // prefetch first, then test
          const int q = rec.x + (c0 + __ffs(m) - 1) * NV_CHUNK;
          const char *p = reinterpret_cast<const char *>(sc.ent + q);
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(p + 128));
        }
        while (pass) {
          const int q = rec.x + (c0 + __ffs(pass) - 1) * NV_CHUNK;
          pass &= pass - 1;
          test_cell_f32<NV_CAST_NB>(sc, q, min(q + NV_CHUNK, rec.y), cf, px, py, dx, dy, dxf,
                                    dyf, best_t, best_i);
        }
      }
#else
      test_cell_f32<NV_CAST_NB>(sc, rec.x, rec.y, cf, px, py, dx, dy, dxf, dyf, best_t, best_i);
#endif
    }
    if (best_t <= t_exit || t_exit > t_max) break;
#if NV_CAST_PF_NEXT
    if (nrec.y > nrec.x) {  // the next cell's run boxes and first entries -> L1
      asm volatile("prefetch.global.L1 [%0];" ::"l"(sc.chunks + nrec.w));
      asm volatile("prefetch.global.L1 [%0];" ::"l"(sc.entf + nrec.x));
    }
#endif
    cx = ncx;
    cy = ncy;
    tnx = ntnx;
    tny = ntny;
    rec = nrec;
    if (cx < 0 || cx >= gnx || cy < 0 || cy >= gny) {
      bool out_x = (cx < 0 && dx <= 0.0) || (cx >= gnx && dx >= 0.0);
      bool out_y = (cy < 0 && dy <= 0.0) || (cy >= gny && dy >= 0.0);
      if (out_x || out_y) break;
    }
  }
  out_t = best_t;
  out_i = best_i;
}

// raycast_all (_kernels.py:16-48)
__device__ __forceinline__ void ray_brute(const SceneView &sc, double px, double py,
                                          double dx, double dy, double &out_t,
                                          int &out_i) {
  double best_t = NV_INF;
  int best_i = -1;
  for (int64_t i = 0; i < sc.n; ++i)
    seg_test(px, py, dx, dy, __ldg(sc.ax + i), __ldg(sc.ay + i), __ldg(sc.ex + i),
             __ldg(sc.ey + i), (int)i, best_t, best_i);
  out_t = best_t;
  out_i = best_i;
}

// Per-segment first-contact time of disc_cast (_kernels.py:405-459): the
// minimum over the face / band / endpoint candidates of one segment, taken in
// the reference's order with its strict `<`.  The reference's result is then
// the lexicographic (t, idx) minimum over segments (its scan is ascending in
// idx with strict `<`), which lets the warp scan candidates in any order.
__device__ __forceinline__ double disc_seg_t(double px, double py, double ux, double uy,
                                             double radius, double u2, double axi,
                                             double ayi, double bxi, double byi) {
  double best = NV_INF;
  double exi = sub(bxi, axi), eyi = sub(byi, ayi);
  double seg_len = nvx::sqrt_rn(add(mul(exi, exi), mul(eyi, eyi)));
  if (seg_len <= 0.0) return best;
  double tx = div(exi, seg_len), ty = div(eyi, seg_len);
  double nx = -ty, ny = tx;
  double relx = sub(px, axi), rely = sub(py, ayi);
  double d0 = add(mul(relx, nx), mul(rely, ny));
  double vn = add(mul(ux, nx), mul(uy, ny));
  if (fabs(d0) >= radius) {
    double side = d0 > 0.0 ? 1.0 : -1.0;
    if (mul(vn, side) < 0.0) {
      double t = div(sub(mul(side, radius), d0), vn);
      if (0.0 <= t && t <= 1.0) {
        double proj = add(mul(add(relx, mul(t, ux)), tx), mul(add(rely, mul(t, uy)), ty));
        if (0.0 <= proj && proj <= seg_len) {
          if (t < best) best = t;
        }
      }
    }
  } else {
    double proj = add(mul(relx, tx), mul(rely, ty));
    if (0.0 <= proj && proj <= seg_len && mul(vn, d0) < 0.0) {
      if (0.0 < best) best = 0.0;
    }
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    double cxp = e == 0 ? axi : bxi;
    double cyp = e == 0 ? ayi : byi;
    double wx = sub(px, cxp), wy = sub(py, cyp);
    double b = add(mul(wx, ux), mul(wy, uy));
    double c = sub(add(mul(wx, wx), mul(wy, wy)), mul(radius, radius));
    if (c < 0.0) {
      if (b < 0.0 && 0.0 < best) best = 0.0;
      continue;
    }
    if (u2 == 0.0) continue;
    double disc = sub(mul(b, b), mul(u2, c));
    if (disc < 0.0) continue;
    double t = div(sub(-b, nvx::sqrt_rn(disc)), u2);
    if (0.0 <= t && t <= 1.0 && t < best) best = t;
  }
  return best;
}

// disc_seg_t with the segment's seg_len and unit tangent taken from its
// DiscEntry (the identical values the reference recomputes per candidate).
__device__ __forceinline__ double disc_seg_t_pre(double px, double py, double ux, double uy,
                                                 double radius, double u2, const DiscEntry &d) {
  double best = NV_INF;
  const double seg_len = d.len;
  if (seg_len <= 0.0) return best;
  const double tx = d.tx, ty = d.ty;
  const double nx = -ty, ny = tx;
  const double relx = sub(px, d.ax), rely = sub(py, d.ay);
  const double d0 = add(mul(relx, nx), mul(rely, ny));
  const double vn = add(mul(ux, nx), mul(uy, ny));
  if (fabs(d0) >= radius) {
    const double side = d0 > 0.0 ? 1.0 : -1.0;
    if (mul(vn, side) < 0.0) {
      const double t = div(sub(mul(side, radius), d0), vn);
      if (0.0 <= t && t <= 1.0) {
        const double proj = add(mul(add(relx, mul(t, ux)), tx), mul(add(rely, mul(t, uy)), ty));
        if (0.0 <= proj && proj <= seg_len) {
          if (t < best) best = t;
        }
      }
    }
  } else {
    const double proj = add(mul(relx, tx), mul(rely, ty));
    if (0.0 <= proj && proj <= seg_len && mul(vn, d0) < 0.0) {
      if (0.0 < best) best = 0.0;
    }
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const double cxp = e == 0 ? d.ax : d.bx;
    const double cyp = e == 0 ? d.ay : d.by;
    const double wx = sub(px, cxp), wy = sub(py, cyp);
    const double b = add(mul(wx, ux), mul(wy, uy));
    const double c = sub(add(mul(wx, wx), mul(wy, wy)), mul(radius, radius));
    if (c < 0.0) {
      if (b < 0.0 && 0.0 < best) best = 0.0;
      continue;
    }
    if (u2 == 0.0) continue;
    const double disc = sub(mul(b, b), mul(u2, c));
    if (disc < 0.0) continue;
    const double t = div(sub(-b, nvx::sqrt_rn(disc)), u2);
    if (0.0 <= t && t <= 1.0 && t < best) best = t;
  }
  return best;
}

#ifndef NV_DISC_K
#define NV_DISC_K 4  // candidates per lane per round of the flat disc-cast pass
#endif
__device__ __forceinline__ void lex_min(double &t, int &i, double t2, int i2) {
  if (t2 < t || (t2 == t && i2 < i)) {
    t = t2;
    i = i2;
  }
}

__device__ __forceinline__ void warp_lex_min(double &t, int &i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double t2 = __shfl_xor_sync(0xffffffffu, t, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    lex_min(t, i, t2, i2);
  }
}

// SegmentIndex.cast_disc (geometry.py:183-192): candidates from the padded
// swept AABB (query_aabb), first contact, tangent of the contacted segment.
__device__ void warp_cast_disc(const SceneView &sc, double px, double py, double ux,
                               double uy, double radius, double &t_out, int &i_out,
                               double &tan_x, double &tan_y) {
  const int lane = threadIdx.x & 31;
  double pad = add(radius, 1e-6);
  double xa = add(px, ux), ya = add(py, uy);
  double lox = xa < px ? xa : px, loy = ya < py ? ya : py;  // Python min(a, b)
  double hix = xa > px ? xa : px, hiy = ya > py ? ya : py;  // Python max(a, b)
  int cx0 = cell_coord(sub(lox, pad), sc.x0, sc.gnx);
  int cy0 = cell_coord(sub(loy, pad), sc.y0, sc.gny);
  int cx1 = cell_coord(add(hix, pad), sc.x0, sc.gnx);
  int cy1 = cell_coord(add(hiy, pad), sc.y0, sc.gny);
  double u2 = add(mul(ux, ux), mul(uy, uy));
  double bt = NV_INF;
  int bi = 0x7fffffff;
  double btx = 0.0, bty = 0.0;  // tangent of this lane's best
  // f32 prefilter on the cell-relative endpoints: any contact (face, band or
  // endpoint case of disc_cast) needs a point of the segment within `radius`
  // of a point of the sweep, so the segment's box must meet the sweep's box
  // grown by radius; the 1e-3 m slack dwarfs every f32/f64 rounding at these
  // magnitudes.  Skipped segments are ones disc_cast finds no valid t for.
  const float grow = (float)radius + 1e-3f;
  const int ncx = cx1 - cx0 + 1, ncell = ncx * (cy1 - cy0 + 1);
  if (ncell <= 32) {
    // all query cells at once: lane k owns cell k's run; a warp prefix sum
    // flattens the runs so every lane tests independent candidates
    int cnt = 0, q0 = 0, cxk = 0, cyk = 0;
    if (lane < ncell) {
      cyk = cy0 + lane / ncx;
      cxk = cx0 + lane % ncx;
      const int c = cyk * sc.gnx + cxk;
      q0 = __ldg(sc.starts + c);
      cnt = __ldg(sc.starts + c + 1) - q0;
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    // All candidates (up to NV_DISC_K per lane) are located and their f32
    // endpoint records loaded in one memory round trip; the survivors of the
    // box test are compacted through shared memory to one lane each, which
    // loads its disc record (second round trip) and runs disc_cast's math.
    constexpr int K = NV_DISC_K;
    __shared__ int s_q[8][32 * K];
    int *sq = s_q[(threadIdx.x >> 5) & 7];
    for (int base = 0; base < total; base += 32 * K) {
      int qq[K];
      bool sv[K];
#pragma unroll
      for (int h = 0; h < K; ++h) {
        const int g = min(base + h * 32 + lane, total - 1);
        int o = 0;
#pragma unroll
        for (int b = 16; b > 0; b >>= 1) {
          const int v = __shfl_sync(0xffffffffu, incl, o + b - 1);
          if (v <= g) o += b;
        }
        const int oq0 = __shfl_sync(0xffffffffu, q0, o);
        const int oincl = __shfl_sync(0xffffffffu, incl, o);
        const int ocnt = __shfl_sync(0xffffffffu, cnt, o);
        const int ocx = __shfl_sync(0xffffffffu, cxk, o);
        const int ocy = __shfl_sync(0xffffffffu, cyk, o);
        qq[h] = oq0 + (g - (oincl - ocnt));
        const double X0 = add(sc.x0, (double)ocx), Y0 = add(sc.y0, (double)ocy);
        const float bx0 = (float)sub(lox, X0) - grow, bx1 = (float)sub(hix, X0) + grow;
        const float by0 = (float)sub(loy, Y0) - grow, by1 = (float)sub(hiy, Y0) + grow;
        const float4 f = __ldg(sc.entf + qq[h]);
        sv[h] = base + h * 32 + lane < total && !(fmaxf(f.x, f.z) < bx0 || fminf(f.x, f.z) > bx1 ||
                                                   fmaxf(f.y, f.w) < by0 || fminf(f.y, f.w) > by1);
      }
      int nsurv = 0;
#pragma unroll
      for (int h = 0; h < K; ++h) {
        const unsigned m = __ballot_sync(0xffffffffu, sv[h]);
        if (sv[h]) sq[nsurv + __popc(m & ((1u << lane) - 1u))] = qq[h];
        nsurv += __popc(m);
      }
      __syncwarp();
      for (int r = lane; r < nsurv; r += 32) {
        const DiscEntry d = sc.dent[sq[r]];
        const double t = disc_seg_t_pre(px, py, ux, uy, radius, u2, d);
        if (t < bt || (t == bt && d.idx < bi)) {
          bt = t;
          bi = d.idx;
          btx = d.tx;
          bty = d.ty;
        }
      }
      __syncwarp();
    }
  } else {
    for (int cy = cy0; cy <= cy1; ++cy)
      for (int cx = cx0; cx <= cx1; ++cx) {
        int c = cy * sc.gnx + cx;
        int q0 = __ldg(sc.starts + c), q1 = __ldg(sc.starts + c + 1);
        if (q0 == q1) continue;
        const double X0 = add(sc.x0, (double)cx), Y0 = add(sc.y0, (double)cy);
        const float sx0 = (float)sub(lox, X0) - grow, sx1 = (float)sub(hix, X0) + grow;
        const float sy0 = (float)sub(loy, Y0) - grow, sy1 = (float)sub(hiy, Y0) + grow;
        for (int q = q0 + lane; q < q1; q += 32) {
          const float4 f = __ldg(sc.entf + q);
          if (fmaxf(f.x, f.z) < sx0 || fminf(f.x, f.z) > sx1 || fmaxf(f.y, f.w) < sy0 ||
              fminf(f.y, f.w) > sy1)
            continue;
          const DiscEntry d = sc.dent[q];
          const double t = disc_seg_t_pre(px, py, ux, uy, radius, u2, d);
          if (t < bt || (t == bt && d.idx < bi)) {
            bt = t;
            bi = d.idx;
            btx = d.tx;
            bty = d.ty;
          }
        }
      }
  }
  const double lt = bt;
  const int li = bi;
  warp_lex_min(bt, bi);
  if (!(bt < NV_INF) || bi == 0x7fffffff) {  // t is inf whenever nothing hit
    t_out = NV_INF;
    i_out = -1;
    tan_x = 0.0;
    tan_y = 0.0;
    return;
  }
  // the winner's unit tangent (ex / seg_len, ey / seg_len, precomputed) from
  // the lane that found it -- no memory round trip
  const unsigned own = __ballot_sync(0xffffffffu, lt == bt && li == bi);
  const int src = __ffs(own) - 1;
  t_out = bt;
  i_out = bi;
  tan_x = __shfl_sync(0xffffffffu, btx, src);
  tan_y = __shfl_sync(0xffffffffu, bty, src);
}

// min_seg_distance (_kernels.py:468-493), one segment.
__device__ __forceinline__ double seg_dist(double px, double py, double axi, double ayi,
                                           double bxi, double byi) {
  double exi = sub(bxi, axi), eyi = sub(byi, ayi);
  double l2 = add(mul(exi, exi), mul(eyi, eyi));
  double wx = sub(px, axi), wy = sub(py, ayi);
  double cx, cy;
  if (l2 > 0.0) {
    double t = div(add(mul(wx, exi), mul(wy, eyi)), l2);
    if (t < 0.0)
      t = 0.0;
    else if (t > 1.0)
      t = 1.0;
    cx = sub(wx, mul(t, exi));
    cy = sub(wy, mul(t, eyi));
  } else {
    cx = wx;
    cy = wy;
  }
  return nvx::sqrt_rn(add(mul(cx, cx), mul(cy, cy)));
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// SegmentIndex.clearance (geometry.py:194-206): local query, then global.
__device__ double warp_clearance(const SceneView &sc, double px, double py, double sr) {
  const int lane = threadIdx.x & 31;
  int cx0 = cell_coord(sub(px, sr), sc.x0, sc.gnx);
  int cy0 = cell_coord(sub(py, sr), sc.y0, sc.gny);
  int cx1 = cell_coord(add(px, sr), sc.x0, sc.gnx);
  int cy1 = cell_coord(add(py, sr), sc.y0, sc.gny);
  double best = NV_INF;
  int any = 0;
  for (int cy = cy0; cy <= cy1; ++cy)
    for (int cx = cx0; cx <= cx1; ++cx) {
      int c = cy * sc.gnx + cx;
      int q0 = __ldg(sc.starts + c), q1 = __ldg(sc.starts + c + 1);
      any |= (q1 > q0);
      for (int q = q0 + lane; q < q1; q += 32) {
        int i = __ldg(sc.items + q);
        double d = seg_dist(px, py, __ldg(sc.ax + i), __ldg(sc.ay + i), __ldg(sc.bx + i),
                            __ldg(sc.by + i));
        if (d < best) best = d;
      }
    }
  best = warp_min(best);
  if (any && best <= sr) return best;
  if (sc.n == 0) return NV_INF;
  best = NV_INF;
  for (int64_t i = lane; i < sc.n; i += 32) {
    double d = seg_dist(px, py, __ldg(sc.ax + i), __ldg(sc.ay + i), __ldg(sc.bx + i),
                        __ldg(sc.by + i));
    if (d < best) best = d;
  }
  return warp_min(best);
}

// ------------------------------------------------------------ agent step

struct AgentCfg {
  double radius, step, turn_rad;
};

#define NV_CONTACT_EPSILON 1e-4  // sim.py:24

// apply_forward (sim.py:90-130) for one env, executed by a whole warp.
__device__ void warp_forward(const SceneView &sc, const AgentCfg &cfg, double &x,
                             double &y, double ch, double sh, double &moved,
                             int &collided) {
  double ux = mul(cfg.step, ch), uy = mul(cfg.step, sh);
  double t1, tx, ty;
  int i1;
  warp_cast_disc(sc, x, y, ux, uy, cfg.radius, t1, i1, tx, ty);
  if (!(t1 < 1.0)) {
    x = add(x, ux);
    y = add(y, uy);
    moved = cfg.step;
    collided = 0;
    return;
  }
  double d1 = sub(mul(t1, cfg.step), NV_CONTACT_EPSILON);
  if (!(d1 > 0.0)) d1 = 0.0;  // Python max(0.0, d1)
  double unx = div(ux, cfg.step), uny = div(uy, cfg.step);
  double p1x = add(x, mul(unx, d1)), p1y = add(y, mul(uny, d1));
  double omt = sub(1.0, t1);
  double remx = mul(ux, omt), remy = mul(uy, omt);
  double dot = nvx::fma_rn(remy, ty, mul(remx, tx));  // np.dot -> OpenBLAS ddot
  double slx = mul(dot, tx), sly = mul(dot, ty);
  double slide_len = nvx::hypot_cr(slx, sly);
  double d2 = 0.0;
  if (slide_len > NV_CONTACT_EPSILON) {
    double t2, t2x, t2y;
    int i2;
    warp_cast_disc(sc, p1x, p1y, slx, sly, cfg.radius, t2, i2, t2x, t2y);
    if (!(t2 < 1.0)) {
      d2 = slide_len;
    } else {
      d2 = sub(mul(t2, slide_len), NV_CONTACT_EPSILON);
      if (!(d2 > 0.0)) d2 = 0.0;
    }
    p1x = add(p1x, mul(div(slx, slide_len), d2));
    p1y = add(p1y, mul(div(sly, slide_len), d2));
  }
  x = p1x;
  y = p1y;
  moved = add(d1, d2);
  collided = 1;
}

// Simulator.step (sim.py:202-219) for env e, executed by one warp.
// Post-step agent values, identical in every lane (for fused consumers).
struct AgentPost {
  double x, y, path;
  long long coll;
  int status;
};

__device__ __forceinline__ void warp_agent_step(const EnvView &ev, const SceneView &sc,
                                                const AgentCfg &cfg, int e, int a,
                                                uint8_t *collided_out, double *disp_out,
                                                int32_t *status_out, AgentPost *post = nullptr) {
  const int lane = threadIdx.x & 31;
  int status = 0, collided = 0;
  double moved = 0.0;
  // all of the env's state is loaded up front (one memory round trip)
  const uint8_t was_reset = ev.reset[e];
  double x = ev.x[e], y = ev.y[e], h0 = ev.h[e], ch = ev.ch[e], sh = ev.sh[e];
  const double path = ev.path[e];
  const long long coll0 = ev.coll[e];
  if (!was_reset) {
    status = 2;  // NV_ENV_NOT_RESET
  } else if (ev.frozen && ev.frozen[e]) {
    status = 4;  // NV_ENV_DONE: the task episode is over (task.py:196-197)
  } else if (a == 0) {
    warp_forward(sc, cfg, x, y, ch, sh, moved, collided);
    if (lane == 0) {
      ev.x[e] = x;
      ev.y[e] = y;
      ev.path[e] = add(path, moved);
      ev.coll[e] = coll0 + collided;
    }
  } else if (a == 1 || a == 2) {
    // apply_turn (sim.py:83-87): wrap(h + sign * radians(turn)); +-x is exact
    double h = nvx::wrap_angle(add(h0, a == 1 ? cfg.turn_rad : -cfg.turn_rad));
    if (lane == 0) {
      double s, c;
      nvx::sincos_cr(h, &s, &c);
      ev.h[e] = h;
      ev.sh[e] = s;
      ev.ch[e] = c;
    }
  } else if (a != 3) {
    status = 3;  // NV_ENV_BAD_ACTION
  }
  if (lane == 0) {
    if (collided_out) collided_out[e] = (uint8_t)collided;
    if (disp_out) disp_out[e] = moved;
    if (status_out) status_out[e] = status;
  }
  if (post) {
    post->x = x;
    post->y = y;
    post->path = status == 0 && a == 0 ? add(path, moved) : path;
    post->coll = coll0 + collided;
    post->status = status;
  }
}

// Simulator.step for all envs: one warp per env.  With `ready` (programmatic
// dependent launch of the cast), the dependent grid is released at once and
// each env's pose is published through ready[e] (release) as soon as its warp
// is done, so the casts of finished envs overlap the long agent chains.
__global__ void __launch_bounds__(128) k_agent_step(EnvView ev, SceneView sc, AgentCfg cfg,
                                                    const int8_t *__restrict__ actions,
                                                    uint8_t *collided_out,
                                                    double *disp_out, int32_t *status_out,
                                                    unsigned *ready) {
  if (ready) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int e = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (e >= ev.n) return;
  warp_agent_step(ev, sc, cfg, e, actions[e], collided_out, disp_out, status_out);
  if (ready && (threadIdx.x & 31) == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + e), "r"(1u) : "memory");
  }
}

// Cast side of the agent->cast overlap: thread 0 of a CTA waits for every env
// the CTA covers (acquire), then the CTA's last arrival per env resets the
// env's flag for the next step.  (CTAs of the cast grid cover rays
// [b*B, (b+1)*B) of the env-major ray order.)
__device__ __forceinline__ void wait_envs_ready(unsigned *ready, unsigned *arrive, int W,
                                                long long n_rays) {
  const long long r0 = (long long)blockIdx.x * blockDim.x;
  const long long r1 = min(n_rays, r0 + blockDim.x) - 1;
  const int e0 = (int)(r0 / W), e1 = (int)(r1 / W);
  if (threadIdx.x == 0) {
    for (int e = e0; e <= e1; ++e) {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + e) : "memory");
        if (!v) __nanosleep(64);
      } while (!v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int e = e0; e <= e1; ++e) {
      // CTAs that cover env e: blocks [first, last] of its ray range
      const long long f = (long long)e * W / blockDim.x, l = ((long long)(e + 1) * W - 1) / blockDim.x;
      if (atomicAdd(arrive + e, 1u) == (unsigned)(l - f)) {
        arrive[e] = 0;
        ready[e] = 0;
      }
    }
  }
}

// Simulator.set_agent_state (sim.py:172-184), one warp per env.  Inputs are
// device copies of the host arrays.
__global__ void __launch_bounds__(128) k_set_poses(EnvView ev, SceneView sc, double radius,
                                                   const double *__restrict__ xy,
                                                   const double *__restrict__ hd,
                                                   const uint8_t *__restrict__ mask,
                                                   int32_t *status, double *clear_out) {
  const int e = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (e >= ev.n) return;
  if (mask && !mask[e]) {
    if (lane == 0) status[e] = 0;
    return;
  }
  double px = xy[2 * e], py = xy[2 * e + 1];
  double clr = warp_clearance(sc, px, py, 2.0);
  if (lane != 0) return;
  clear_out[e] = clr;
  if (clr < radius) {
    status[e] = 1;  // NV_ENV_TOO_CLOSE, state untouched
    return;
  }
  double h = nvx::wrap_angle(hd[e]);
  double s, c;
  nvx::sincos_cr(h, &s, &c);
  ev.x[e] = px;
  ev.y[e] = py;
  ev.h[e] = h;
  ev.ch[e] = c;
  ev.sh[e] = s;
  ev.path[e] = 0.0;
  ev.coll[e] = 0;
  ev.ox[e] = px;
  ev.oy[e] = py;
  ev.oh[e] = h;
  // EpisodeFrame.to_frame uses cos(-h0), sin(-h0) (sensors.py:166)
  double fs, fc;
  nvx::sincos_cr(-h, &fs, &fc);
  ev.fc[e] = fc;
  ev.fs[e] = fs;
  ev.reset[e] = 1;
  status[e] = 0;
}

// --------------------------------------------------------- column casts

// Column epilogue: exact classification of the column into ceiling rows
// [0, lo), middle rows [lo, hi) (wall, or void when s >= max_range) and floor
// rows [hi, H), equal to fill_frame's per-pixel FP64 compares
// (_kernels.py:149-170) because tc is non-decreasing over the v > 0 rows and
// tf non-increasing over the v < 0 rows (IEEE division is monotone).
__device__ __forceinline__ void column_epilogue(const SceneView &sc, const CamView &cam,
                                                double s, int k, double dx, double dy,
                                                ColRec &out) {
  // lo = #{i < n_top : tc[i] <= s} and hi = first i >= b0 with tf[i] <= s.
  // In exact arithmetic tc_i <= s iff i <= hc - ktop / s and tf_i <= s iff
  // i >= hc + kbot / s; an f32 estimate of each boundary is settled by the
  // reference's own FP64 comparisons against the exact tc / tf tables (both
  // monotone), so the result is exact whatever the estimate's error.
  const float fs = (float)s;
  int lo = (int)fminf(fmaxf(floorf(cam.hc - cam.ktop / fs) + 1.0f, 0.0f), (float)cam.n_top);
  while (lo > 0 && !(__ldg(cam.tc + lo - 1) <= s)) --lo;
  while (lo < cam.n_top && __ldg(cam.tc + lo) <= s) ++lo;
  int hi = (int)fminf(fmaxf(ceilf(cam.hc + cam.kbot / fs), (float)cam.b0), (float)cam.H);
  while (hi > cam.b0 && __ldg(cam.tf + hi - 1) <= s) --hi;
  while (hi < cam.H && !(__ldg(cam.tf + hi) <= s)) ++hi;
  const bool lit = s < cam.max_range && k >= 0;
  out.lohi = (uint32_t)lo | ((uint32_t)hi << 16);
  float fdx = (float)dx, fdy = (float)dy;
  out.d2 = fdx * fdx + fdy * fdy;
  if (lit) {
    out.depth_w = (float)s;
    double dt = fabs(add(mul(dx, __ldg(sc.nx + k)), mul(dy, __ldg(sc.ny + k))));
    out.num08_w = 0.8f * (float)dt;
    float4 c = __ldg(sc.alb255 + k);
    out.col_w[0] = c.x;
    out.col_w[1] = c.y;
    out.col_w[2] = c.z;
    out.sem_w = __ldg(sc.sem + k);
  } else {
    out.depth_w = (float)cam.max_range;
    out.num08_w = 0.0f;
    out.col_w[0] = out.col_w[1] = out.col_w[2] = 0.0f;
    out.sem_w = 0;
  }
}

__device__ __forceinline__ void put_rec(const RecOut &ro, long long e, int j, const ColRec &r) {
  const size_t p = (size_t)e * ro.W + rec_pos(j, ro.cpl);
  const float4 *h = reinterpret_cast<const float4 *>(&r);
  ro.a[p] = h[0];
  ro.b[p] = h[1];
}

// _column_directions (sensors.py:96-102) + raycast_grid + epilogue for one
// (env, column); column 0 also writes gps_compass (sensors.py:175-180).
// COH: agent state was written earlier in the same launch (megakernel), so it
// is read through L2 (ld.global.cg) rather than the non-coherent path.
template <bool COH>
__device__ __forceinline__ void cast_column(const EnvView &ev, const SceneView &sc,
                                            const CamView &cam, int e, int j, const RecOut &ro,
                                            double t_max, double *gps, double *compass) {
  double px, py, c, s;
  if (COH) {
    px = __ldcg(ev.x + e); py = __ldcg(ev.y + e); c = __ldcg(ev.ch + e); s = __ldcg(ev.sh + e);
  } else {
    px = ev.x[e]; py = ev.y[e]; c = ev.ch[e]; s = ev.sh[e];
  }
  const double u = __ldg(cam.u + j);
  const double dx = add(c, mul(u, s));
  const double dy = add(s, mul(u, -c));
  double t;
  int k;
  ray_grid(sc, px, py, dx, dy, t_max, t, k);
  ColRec r;
  column_epilogue(sc, cam, t, k, dx, dy, r);
  put_rec(ro, e, j, r);
  if (j == 0 && (gps || compass)) {
    double ddx = sub(px, ev.ox[e]), ddy = sub(py, ev.oy[e]);
    double fc = ev.fc[e], fs = ev.fs[e];
    if (gps) {
      gps[2 * e] = sub(mul(fc, ddx), mul(fs, ddy));
      gps[2 * e + 1] = add(mul(fs, ddx), mul(fc, ddy));
    }
    if (compass) {
      const double h = COH ? __ldcg(ev.h + e) : ev.h[e];
      compass[e] = nvx::wrap_angle(sub(h, ev.oh[e]));
    }
  }
}

// raycast_grid for one ray by a whole warp (small batches: latency, not
// throughput).  Every lane walks the same DDA (uniform control flow, the
// reference's visit order and early-out); a cell's entries are spread over
// the lanes (f32 side test, then the exact FP64 test), and the warp keeps the
// lexicographic (t, idx) minimum.  Returns the result in every lane.
__device__ __forceinline__ void ray_grid_warp(const SceneView &sc, double px, double py,
                                              double dx, double dy, double t_max, double &out_t,
                                              int &out_i) {
  const int lane = threadIdx.x & 31;
  const double cell = 1.0;
  double best_t = NV_INF;
  int best_i = -1;
  if (isnan(px) || isnan(py) || isnan(dx) || isnan(dy)) {
    out_t = best_t;
    out_i = best_i;
    return;
  }
  long long cx = (long long)floor(sub(px, sc.x0));
  long long cy = (long long)floor(sub(py, sc.y0));
  const int stepx = dx > 0.0 ? 1 : -1;
  const int stepy = dy > 0.0 ? 1 : -1;
  double tnx, tdx, tny, tdy;
  if (dx != 0.0) {
    double nbx = add(sc.x0, mul((double)(cx + (dx > 0.0 ? 1 : 0)), cell));
    tnx = div(sub(nbx, px), dx);
    tdx = fabs(div(cell, dx));
  } else {
    tnx = NV_INF;
    tdx = NV_INF;
  }
  if (dy != 0.0) {
    double nby = add(sc.y0, mul((double)(cy + (dy > 0.0 ? 1 : 0)), cell));
    tny = div(sub(nby, py), dy);
    tdy = fabs(div(cell, dy));
  } else {
    tny = NV_INF;
    tdy = NV_INF;
  }
  const long long gnx = sc.gnx, gny = sc.gny;
  const float dxf = (float)dx, dyf = (float)dy;
  const float sd = (fabsf(dxf) + fabsf(dyf)) * (1.0f + 0x1p-20f);
  for (int guard = 0; guard < (1 << 24); ++guard) {
    if (0 <= cx && cx < gnx && 0 <= cy && cy < gny) {
      const int4 rec = __ldg(sc.cells + (cy * gnx + cx));
      if (rec.y > rec.x) {
        const double X0 = add(sc.x0, (double)cx), Y0 = add(sc.y0, (double)cy);
        const float pxr = (float)sub(px, X0), pyr = (float)sub(py, Y0);
        const float cp = fmaf(dxf, pyr, -(dyf * pxr));
        const float E = NV_K32 * sd * (__int_as_float(rec.z) + fabsf(pxr) + fabsf(pyr) + 1e-30f);
        for (int q = rec.x + lane; q < rec.y; q += 32) {
          const float4 e = __ldg(sc.entf + q);
          const float sa = fmaf(dxf, e.y, -(dyf * e.x)) - cp;
          const float sb = fmaf(dxf, e.w, -(dyf * e.z)) - cp;
          if (fminf(sa, sb) > E || fmaxf(sa, sb) < -E) continue;
          const double2 *p2 = reinterpret_cast<const double2 *>(sc.ent + q);
          const double2 a2 = __ldg(p2), e2 = __ldg(p2 + 1);
          double den, tn, rn;
          if (seg_pre(px, py, dx, dy, a2.x, a2.y, e2.x, e2.y, best_t, den, tn, rn))
            seg_exact(den, tn, rn, __ldg(sc.items + q), best_t, best_i);
        }
        // the lexicographic minimum is order-free: combine the lanes
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double t2 = __shfl_xor_sync(0xffffffffu, best_t, o);
          const int i2 = __shfl_xor_sync(0xffffffffu, best_i, o);
          if (t2 < best_t || (t2 == best_t && (unsigned)i2 < (unsigned)best_i)) {
            best_t = t2;
            best_i = i2;
          }
        }
      }
    }
    const double t_exit = tnx < tny ? tnx : tny;
    if (best_t <= t_exit || t_exit > t_max) break;
    if (tnx < tny) {
      cx += stepx;
      tnx = add(tnx, tdx);
    } else {
      cy += stepy;
      tny = add(tny, tdy);
    }
    if (cx < 0 || cx >= gnx || cy < 0 || cy >= gny) {
      bool out_x = (cx < 0 && dx <= 0.0) || (cx >= gnx && dx >= 0.0);
      bool out_y = (cy < 0 && dy <= 0.0) || (cy >= gny && dy >= 0.0);
      if (out_x || out_y) break;
    }
  }
  out_t = best_t;
  out_i = best_i;
}

// One warp per (env, column): the latency-bound small-batch cast.
__device__ __forceinline__ void k_column_cast_warp_body(const EnvView &ev, const SceneView &sc,
                                                        const CamView &cam, const RecOut &ro,
                                                        double t_max, double *gps,
                                                        double *compass, int e, int j) {
  const int lane = threadIdx.x & 31;
  const double px = ev.x[e], py = ev.y[e], c = ev.ch[e], s = ev.sh[e];
  const double u = __ldg(cam.u + j);
  const double dx = add(c, mul(u, s));
  const double dy = add(s, mul(u, -c));
  double t;
  int k;
  ray_grid_warp(sc, px, py, dx, dy, t_max, t, k);
  if (lane != 0) return;
  ColRec r;
  column_epilogue(sc, cam, t, k, dx, dy, r);
  put_rec(ro, e, j, r);
  if (j == 0 && (gps || compass)) {
    double ddx = sub(px, ev.ox[e]), ddy = sub(py, ev.oy[e]);
    double fc = ev.fc[e], fs = ev.fs[e];
    if (gps) {
      gps[2 * e] = sub(mul(fc, ddx), mul(fs, ddy));
      gps[2 * e + 1] = add(mul(fs, ddx), mul(fc, ddy));
    }
    if (compass) compass[e] = nvx::wrap_angle(sub(ev.h[e], ev.oh[e]));
  }
}

__global__ void __launch_bounds__(128) k_column_cast_warp(EnvView ev, SceneView sc, CamView cam,
                                                          RecOut ro, double t_max, double *gps,
                                                          double *compass) {
  const long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long total = (long long)ev.n * cam.W;
  if (g >= total) return;
  const int e = (int)(g / cam.W);
  const int j = (int)(g - (long long)e * cam.W);
  k_column_cast_warp_body(ev, sc, cam, ro, t_max, gps, compass, e, j);
}

// One thread per (env, column).  With `ready`: launched as a programmatic
// dependent of k_agent_step; waits per env instead of for the whole step.
__global__ void __launch_bounds__(128) k_column_cast(EnvView ev, SceneView sc, CamView cam,
                                                     RecOut ro, double t_max,
                                                     double *gps, double *compass,
                                                     unsigned *ready, unsigned *arrive) {
  const long long total = (long long)ev.n * cam.W;
  if (ready) wait_envs_ready(ready, arrive, cam.W, total);
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= total) return;
  const int e = (int)(g / cam.W);
  const int j = (int)(g - (long long)e * cam.W);
  if (ready)
    cast_column<true>(ev, sc, cam, e, j, ro, t_max, gps, compass);
  else
    cast_column<false>(ev, sc, cam, e, j, ro, t_max, gps, compass);
}

// Simulator.step + the column casts of one env per CTA: warp 0 runs the
// agent step (the same warp_agent_step as k_agent_step), then every thread
// casts columns of the env at its new pose.  CTAs progress independently, so
// the agent step's long FP64 latency chains of some envs overlap the casts of
// others (no grid-wide step -> cast barrier).
__global__ void __launch_bounds__(256) k_step_cast(EnvView ev, SceneView sc, AgentCfg cfg,
                                                   const int8_t *__restrict__ actions,
                                                   uint8_t *collided_out, double *disp_out,
                                                   int32_t *status_out, CamView cam, RecOut ro,
                                                   double t_max, double *gps, double *compass) {
  const int e = blockIdx.x;
  if (threadIdx.x < 32) {
    warp_agent_step(ev, sc, cfg, e, actions[e], collided_out, disp_out, status_out);
    __threadfence();
  }
  __syncthreads();
  for (int j = threadIdx.x; j < cam.W; j += blockDim.x)
    cast_column<true>(ev, sc, cam, e, j, ro, t_max, gps, compass);
}

// Persistent variant: every warp pulls (env, 32-column group) work items from
// a self-resetting global counter until none are left, so all warp slots stay
// busy to the end of the launch (no tail of half-empty CTAs); consecutive
// items are neighbouring column groups of one env (shared cells in L1).
#ifndef NV_CAST_MINB
#define NV_CAST_MINB 1
#endif
__global__ void __launch_bounds__(128, NV_CAST_MINB) k_column_cast_q(EnvView ev, SceneView sc,
                                                                     CamView cam, RecOut ro,
                                                                     double t_max, double *gps,
                                                                     double *compass,
                                                                     unsigned int *ctr) {
  const int lane = threadIdx.x & 31;
  const int gpe = (cam.W + 31) >> 5;  // column groups per env
  const long long total = (long long)ev.n * gpe;
  for (;;) {
    long long item = 0;
    if (lane == 0) item = atomicAdd(ctr, 1u);
    item = __shfl_sync(0xffffffffu, item, 0);
    if (item >= total) break;
    const int e = (int)(item / gpe);
    const int j = (int)(item - (long long)e * gpe) * 32 + lane;
    if (j < cam.W) cast_column<false>(ev, sc, cam, e, j, ro, t_max, gps, compass);
  }
  if (lane == 0) {  // the last warp out resets the counters for the next launch
    __threadfence();
    const unsigned total_warps = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(ctr + 1, 1u) == total_warps - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

// ---------------------------------------------------- binned column cast
//
// k_cast_binned: one CTA per env computes all W column hits by tile-binned
// segment setup instead of W independent DDA walks:
//   1. the cells overlapping the view frustum up to max_range (the triangle
//      p, p + R d_0, p + R d_{W-1}; hits at z-depth t <= max_range lie inside)
//      are distributed over the warps;
//   2. each lane projects one entry of a cell to a conservative column span
//      (the columns whose ray can cross the segment: the side tests of its
//      endpoints are linear in the column coordinate u, roots u = x/z; +-1
//      column of slack);
//   3. warp prefix sums over the span lengths compact the (entry, column)
//      pairs, 32 pairs per round, so every lane does useful exact work;
//   4. each pair runs the reference's exact FP64 segment test
//      (_kernels.py:33-45); hits fold into a per-column shared-memory
//      atomicMin on t and, in a second pass, the lowest index among the
//      minimal-t hits: the lexicographic (t, idx) minimum of raycast_all.
// The reference states and tests raycast_grid == raycast_all exactly
// (_kernels.py:55-58, tests/test_acceptance.py:290-305); hits beyond
// max_range render void whether found or not.  A CTA whose
// hit list overflows falls back to the per-column DDA.
#define NV_HIT_CAP 2048
#define NV_KEY_INF 0x7ff0000000000000ull

__device__ __forceinline__ unsigned long long t_key(double t) {
  return t == 0.0 ? 0ull : (unsigned long long)__double_as_longlong(t);  // t >= 0 or -0
}

// Exact segment test of one ray (no best-t pruning): true and t on a hit.
__device__ __forceinline__ bool seg_hit(double px, double py, double dx, double dy, double ax,
                                        double ay, double ex, double ey, double bound,
                                        double &t) {
  double den, tn, rn;
  if (!seg_pre(px, py, dx, dy, ax, ay, ex, ey, bound, den, tn, rn)) return false;
  t = div(tn, den);
  if (t < 0.0) return false;
  const double r = div(rn, den);
  return 0.0 <= r && r <= 1.0;
}

#define NV_BIN_MAXCELLS 1024   // frustum-AABB cells handled with depth banding
#define NV_BAND_M 2.0f          // depth band width (m)
#define NV_COLTILE 8            // columns per occlusion tile

struct BinShared {
  double *dirx, *diry;
  unsigned long long *tkey;
  int *ibest;
  int2 *hits;
  int *nhits;
  int4 *cellinfo;   // per candidate cell: (cell id | band << 24, jc0, jc1, zmin bits)
  int *clist;       // accepted cells of the current band
  int *nlist;
  int *next;        // dynamic cell counter of the current band
  float *tilemax;   // per column tile: max current best t (inf if any column open)
};

// Process the entries of one cell: spans -> warp-compacted (entry, column)
// pairs -> exact tests -> per-column atomicMin.  Returns true on overflow.
__device__ __forceinline__ bool bin_cell(const SceneView &sc, const BinShared &S, int cc, float rx,
                                         float ry, float cf, float sf, float cw, float half,
                                         int W, double px, double py) {
  const int lane = threadIdx.x & 31;
  bool overflow = false;
  const int q0 = __ldg(sc.starts + cc), q1 = __ldg(sc.starts + cc + 1);
  for (int qb = q0; qb < q1; qb += 32) {
    const int q = qb + lane;
    int jlo = 0, cnt = 0;
    if (q < q1) {
      const float4 f = __ldg(sc.entf + q);  // endpoints rel. to the cell anchor
      const float ax = f.x + rx, ay = f.y + ry, bx = f.z + rx, by = f.w + ry;
      const float zA = ax * cf + ay * sf, xA = ax * sf - ay * cf;
      const float zB = bx * cf + by * sf, xB = bx * sf - by * cf;
      const float ZN = 1e-3f;
      float lo = -1e30f, hi = 1e30f;
      bool skip = false;
      if (zA >= ZN && zB >= ZN) {
        const float ua = xA / zA, ub = xB / zB;
        lo = fminf(ua, ub);
        hi = fmaxf(ua, ub);
      } else if (zA <= -ZN && zB <= -ZN) {
        skip = true;  // entirely behind the camera: only t < 0 crossings
      } else if ((zA >= ZN && zB <= -ZN) || (zB >= ZN && zA <= -ZN)) {
        const float zF = zA >= ZN ? zA : zB, xF = zA >= ZN ? xA : xB;
        const float zK = zA >= ZN ? zB : zA, xK = zA >= ZN ? xB : xA;
        const float x0 = xF + (xK - xF) * (zF / (zF - zK));  // x where z = 0
        const float uF = xF / zF;
        if (x0 > ZN) lo = uF;
        else if (x0 < -ZN) hi = uF;
      }  // else: an endpoint near the camera plane -> full width
      if (!skip) {
        const float jl = fmaxf(lo * cw + half, -4.f), jh = fminf(hi * cw + half, (float)W + 4.f);
        jlo = max((int)floorf(jl) - 1, 0);
        const int jhi = min((int)ceilf(jh) + 1, W - 1);
        cnt = max(jhi - jlo + 1, 0);
        // per-entry occlusion: every hit on this segment has t >= zmin (t is
        // z-depth); if each column of its span already holds a strictly
        // nearer hit, no pair of this entry can be a lexicographic minimum
        if (cnt > 0 && cnt <= 24) {
          const float zmin = fminf(zA, zB) * (1.0f - 1e-5f) - 1e-4f;
          bool open = false;
          for (int j = jlo; j <= jhi && !open; ++j) {
            const unsigned long long key = S.tkey[j];
            open = key == NV_KEY_INF ||
                   (float)__longlong_as_double((long long)key) * (1.0f + 1e-6f) >= zmin;
          }
          if (!open) cnt = 0;
        }
      }
    }
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int base = 0; base < total; base += 32) {
      const int g = min(base + lane, total - 1);
      int o = 0;
#pragma unroll
      for (int b = 16; b > 0; b >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, o + b - 1);
        if (v <= g) o += b;
      }
      const int oq = __shfl_sync(0xffffffffu, q, o);
      const int ojlo = __shfl_sync(0xffffffffu, jlo, o);
      const int oincl = __shfl_sync(0xffffffffu, incl, o);
      const int ocnt = __shfl_sync(0xffffffffu, cnt, o);
      if (base + lane < total) {
        const int j = ojlo + (g - (oincl - ocnt));
        const double2 *p2 = reinterpret_cast<const double2 *>(sc.ent + oq);
        const double2 a2 = __ldg(p2), e2 = __ldg(p2 + 1);
        const unsigned long long cur = S.tkey[j];
        const double bound = cur == NV_KEY_INF ? NV_INF : __longlong_as_double((long long)cur);
        double t;
        if (seg_hit(px, py, S.dirx[j], S.diry[j], a2.x, a2.y, e2.x, e2.y, bound, t)) {
          atomicMin(S.tkey + j, t_key(t));
          const int slot = atomicAdd(S.nhits, 1);
          if (slot < NV_HIT_CAP) S.hits[slot] = make_int2(oq, j);
          else overflow = true;
        }
      }
    }
  }
  return overflow;
}

__global__ void __launch_bounds__(128) k_cast_binned(EnvView ev, SceneView sc, CamView cam,
                                                     double focal, RecOut ro,
                                                     double *gps, double *compass) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int W = cam.W;
  const int ntiles = (W + NV_COLTILE - 1) / NV_COLTILE;
  BinShared S;
  S.dirx = reinterpret_cast<double *>(smem);
  S.diry = S.dirx + W;
  S.tkey = reinterpret_cast<unsigned long long *>(S.diry + W);
  S.cellinfo = reinterpret_cast<int4 *>(S.tkey + W);
  S.ibest = reinterpret_cast<int *>(S.cellinfo + NV_BIN_MAXCELLS);
  S.clist = S.ibest + ((W + 3) & ~3);
  S.tilemax = reinterpret_cast<float *>(S.clist + NV_BIN_MAXCELLS);
  S.hits = reinterpret_cast<int2 *>(S.tilemax + ((ntiles + 3) & ~3));
  S.nhits = reinterpret_cast<int *>(S.hits + NV_HIT_CAP);
  S.nlist = S.nhits + 1;
  S.next = S.nhits + 2;
  const int e = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const double px = ev.x[e], py = ev.y[e], c = ev.ch[e], s = ev.sh[e];
  for (int j = tid; j < W; j += blockDim.x) {
    const double u = __ldg(cam.u + j);
    S.dirx[j] = add(c, mul(u, s));
    S.diry[j] = add(s, mul(u, -c));
    S.tkey[j] = NV_KEY_INF;
    S.ibest[j] = 0x7fffffff;
  }
  for (int t = tid; t < ntiles; t += blockDim.x) S.tilemax[t] = 3.0e38f;
  if (tid == 0) {
    *S.nhits = 0;
    *S.nlist = 0;
    *S.next = 0;
  }

  // view frustum triangle (f32, relative to p) and its cell range
  const float cf = (float)c, sf = (float)s;
  const float R = (float)cam.max_range * 1.0001f + 0.01f;
  const float u0 = (float)__ldg(cam.u), u1 = (float)__ldg(cam.u + W - 1);
  const float v1x = R * (cf + u0 * sf), v1y = R * (sf - u0 * cf);
  const float v2x = R * (cf + u1 * sf), v2y = R * (sf - u1 * cf);
  const double bx0 = px + fminf(0.f, fminf(v1x, v2x)), bx1 = px + fmaxf(0.f, fmaxf(v1x, v2x));
  const double by0 = py + fminf(0.f, fminf(v1y, v2y)), by1 = py + fmaxf(0.f, fmaxf(v1y, v2y));
  const int cx0 = cell_coord(bx0, sc.x0, sc.gnx), cx1 = cell_coord(bx1, sc.x0, sc.gnx);
  const int cy0 = cell_coord(by0, sc.y0, sc.gny), cy1 = cell_coord(by1, sc.y0, sc.gny);
  const int ncx = cx1 - cx0 + 1, ncells = ncx * (cy1 - cy0 + 1);
  float en[3][3];  // triangle edges as inward half-planes n.x + k >= 0 (slack 0.01 m)
  {
    const float vx[3] = {0.f, v1x, v2x}, vy[3] = {0.f, v1y, v2y};
    const float orient = (v1x * v2y - v1y * v2x) >= 0.f ? 1.f : -1.f;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int k2 = (k + 1) % 3;
      float nx = -(vy[k2] - vy[k]) * orient, ny = (vx[k2] - vx[k]) * orient;
      const float inv = rsqrtf(nx * nx + ny * ny + 1e-30f);
      nx *= inv;
      ny *= inv;
      en[k][0] = nx;
      en[k][1] = ny;
      en[k][2] = -(nx * vx[k] + ny * vy[k]) + 0.01f;
    }
  }
  const float cw = (float)focal, half = 0.5f * (float)W - 0.5f;
  const bool banded = ncells <= NV_BIN_MAXCELLS;
  int nbands = 1;
  if (banded) {
    // per candidate cell: depth band of its nearest corner, and the column
    // range its rays can cross (projection of its corners, +-1 column)
    for (int k = tid; k < ncells; k += blockDim.x) {
      const int cy = cy0 + k / ncx, cx = cx0 + k % ncx;
      const float rx = (float)sub(add(sc.x0, (double)cx), px);
      const float ry = (float)sub(add(sc.y0, (double)cy), py);
      bool outside = false;
#pragma unroll
      for (int h = 0; h < 3; ++h) {
        const float bmax = fmaxf(en[h][0] * rx, en[h][0] * (rx + 1.f)) +
                           fmaxf(en[h][1] * ry, en[h][1] * (ry + 1.f)) + en[h][2];
        outside |= bmax < 0.f;
      }
      const int cc = cy * sc.gnx + cx;
      const bool empty = __ldg(sc.starts + cc) == __ldg(sc.starts + cc + 1);
      float zmin = 3.0e38f, ulo = 3.0e38f, uhi = -3.0e38f;
      bool near = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float qx = rx + (float)(q & 1), qy = ry + (float)(q >> 1);
        const float z = qx * cf + qy * sf, x = qx * sf - qy * cf;
        zmin = fminf(zmin, z);
        if (z < 0.05f) near = true;
        else {
          ulo = fminf(ulo, x / z);
          uhi = fmaxf(uhi, x / z);
        }
      }
      int jc0 = 0, jc1 = W - 1;
      if (!near) {
        jc0 = max((int)floorf(fmaxf(ulo * cw + half, -4.f)) - 1, 0);
        jc1 = min((int)ceilf(fminf(uhi * cw + half, (float)W + 4.f)) + 1, W - 1);
      }
      const int band = (outside || empty || jc1 < jc0)
                           ? 255
                           : min((int)(fmaxf(zmin, 0.f) * (1.0f / NV_BAND_M)), 254);
      S.cellinfo[k] = make_int4(cc | (band << 24) /* cc < 2^24 */, jc0, jc1,
                                __float_as_int(fmaxf(zmin, 0.f) * (1.0f - 1e-5f) - 1e-4f));
    }
    nbands = (int)(cam.max_range / NV_BAND_M) + 2;
  }
  __syncthreads();

  bool overflow = false;
  if (!banded) {  // very wide frusta: one pass over every candidate cell
    for (int k = warp; k < ncells; k += nwarps) {
      const int cy = cy0 + k / ncx, cx = cx0 + k % ncx;
      const float rx = (float)sub(add(sc.x0, (double)cx), px);
      const float ry = (float)sub(add(sc.y0, (double)cy), py);
      overflow |= bin_cell(sc, S, cy * sc.gnx + cx, rx, ry, cf, sf, cw, half, W, px, py);
    }
  } else {
    for (int band = 0; band < nbands; ++band) {
      // accept this band's cells unless every column they can reach already
      // holds a hit strictly nearer than the cell's nearest point
      for (int k = tid; k < ncells; k += blockDim.x) {
        const int4 ci = S.cellinfo[k];
        const int cb = (ci.x >> 24) & 0xff;
        if (cb != band && !(band == nbands - 1 && cb > band && cb != 255)) continue;
        float tmax = 0.f;
        for (int t = ci.y / NV_COLTILE; t <= ci.z / NV_COLTILE; ++t) tmax = fmaxf(tmax, S.tilemax[t]);
        if (tmax < __int_as_float(ci.w)) continue;  // occluded
        S.clist[atomicAdd(S.nlist, 1)] = k;
      }
      __syncthreads();
      const int nl = *S.nlist;
      for (;;) {  // warps pull cells dynamically (cells differ wildly in entries)
        int l = 0;
        if ((tid & 31) == 0) l = atomicAdd(S.next, 1);
        l = __shfl_sync(0xffffffffu, l, 0);
        if (l >= nl) break;
        const int k = S.clist[l];
        const int cy = cy0 + k / ncx, cx = cx0 + k % ncx;
        const float rx = (float)sub(add(sc.x0, (double)cx), px);
        const float ry = (float)sub(add(sc.y0, (double)cy), py);
        overflow |= bin_cell(sc, S, cy * sc.gnx + cx, rx, ry, cf, sf, cw, half, W, px, py);
      }
      __syncthreads();
      // refresh the occlusion tiles: max over each tile of the best t so far
      for (int t = tid; t < ntiles; t += blockDim.x) {
        float v = 0.f;
        for (int j = t * NV_COLTILE; j < min(W, (t + 1) * NV_COLTILE); ++j) {
          const unsigned long long key = S.tkey[j];
          v = fmaxf(v, key == NV_KEY_INF ? 3.0e38f
                                         : (float)__longlong_as_double((long long)key) * (1.0f + 1e-6f));
        }
        S.tilemax[t] = v;
      }
      if (tid == 0) {
        *S.nlist = 0;
        *S.next = 0;
      }
      __syncthreads();
    }
  }
  overflow = __syncthreads_or(overflow);
  if (overflow) {  // hit list overflow: per-column DDA (always correct)
    for (int j = tid; j < W; j += blockDim.x) {
      double t;
      int k;
      ray_grid(sc, px, py, S.dirx[j], S.diry[j], cam.max_range, t, k);
      ColRec r;
      column_epilogue(sc, cam, t, k, S.dirx[j], S.diry[j], r);
      put_rec(ro, e, j, r);
    }
  } else {
    // pass 2: lowest index among each column's minimal-t hits
    const int nh = *S.nhits;
    for (int h = tid; h < nh; h += blockDim.x) {
      const int2 hq = S.hits[h];
      const double2 *p2 = reinterpret_cast<const double2 *>(sc.ent + hq.x);
      const double2 a2 = __ldg(p2), e2 = __ldg(p2 + 1);
      double t;
      if (seg_hit(px, py, S.dirx[hq.y], S.diry[hq.y], a2.x, a2.y, e2.x, e2.y, NV_INF, t) &&
          t_key(t) == S.tkey[hq.y])
        atomicMin(S.ibest + hq.y, __ldg(sc.items + hq.x));
    }
    __syncthreads();
    for (int j = tid; j < W; j += blockDim.x) {
      const unsigned long long key = S.tkey[j];
      const double t = key == NV_KEY_INF ? NV_INF : __longlong_as_double((long long)key);
      const int k = key == NV_KEY_INF ? -1 : S.ibest[j];
      ColRec r;
      column_epilogue(sc, cam, t, k, S.dirx[j], S.diry[j], r);
      put_rec(ro, e, j, r);
    }
  }
  if (tid == 0 && (gps || compass)) {
    double ddx = sub(px, ev.ox[e]), ddy = sub(py, ev.oy[e]);
    double fc = ev.fc[e], fs = ev.fs[e];
    if (gps) {
      gps[2 * e] = sub(mul(fc, ddx), mul(fs, ddy));
      gps[2 * e + 1] = add(mul(fs, ddx), mul(fc, ddy));
    }
    if (compass) compass[e] = nvx::wrap_angle(sub(ev.h[e], ev.oh[e]));
  }
}

// gps_compass (sensors.py:175-180) for all envs (no visual sensors case).
__global__ void k_gps_compass(EnvView ev, double *gps, double *compass) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ev.n) return;
  double ddx = sub(ev.x[e], ev.ox[e]), ddy = sub(ev.y[e], ev.oy[e]);
  double fc = ev.fc[e], fs = ev.fs[e];
  if (gps) {
    gps[2 * e] = sub(mul(fc, ddx), mul(fs, ddy));
    gps[2 * e + 1] = add(mul(fs, ddx), mul(fc, ddy));
  }
  if (compass) compass[e] = nvx::wrap_angle(sub(ev.h[e], ev.oh[e]));
}

// Column records from caller-supplied hits (fill_frame operator entry).
__global__ void k_cols_from_hits(SceneView sc, CamView cam, long long total,
                                 const double *__restrict__ t_col,
                                 const int64_t *__restrict__ i_col,
                                 const double *__restrict__ dirx,
                                 const double *__restrict__ diry, RecOut ro) {
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (g >= total) return;
  ColRec r;
  column_epilogue(sc, cam, t_col[g], (int)i_col[g], dirx[g], diry[g], r);
  put_rec(ro, g / ro.W, (int)(g % ro.W), r);
}

// Operator entry: raycast_grid / raycast_all over arbitrary rays.
__global__ void k_raycast(SceneView sc, const double *ox, const double *oy,
                          const double *dirx, const double *diry, long long m, double t_max,
                          int brute, double *t_out, int64_t *i_out) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= m) return;
  double t;
  int i;
  if (brute)
    ray_brute(sc, ox[k], oy[k], dirx[k], diry[k], t, i);
  else
    ray_grid(sc, ox[k], oy[k], dirx[k], diry[k], t_max, t, i);
  t_out[k] = t;
  i_out[k] = i;
}

__global__ void __launch_bounds__(128) k_cast_disc(SceneView sc, const double *px,
                                                   const double *py, const double *ux,
                                                   const double *uy, const double *rad,
                                                   long long m, double *t_out,
                                                   int64_t *seg_out, double *tan_out) {
  const long long q = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (q >= m) return;
  double t, tx, ty;
  int i;
  warp_cast_disc(sc, px[q], py[q], ux[q], uy[q], rad[q], t, i, tx, ty);
  if ((threadIdx.x & 31) == 0) {
    t_out[q] = t;
    seg_out[q] = i;
    tan_out[2 * q] = tx;
    tan_out[2 * q + 1] = ty;
  }
}

__global__ void __launch_bounds__(128) k_clearance(SceneView sc, const double *px,
                                                   const double *py, long long m, double sr,
                                                   double *out) {
  const long long q = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  if (q >= m) return;
  double d = warp_clearance(sc, px[q], py[q], sr);
  if ((threadIdx.x & 31) == 0) out[q] = d;
}

// ------------------------------------------------------------ frame fill

// ---- fill: packed-f16 shading --------------------------------------------
//
// Per pixel (fill_frame, _kernels.py:171-207): the pixel is a plane pixel
// (ceiling rows [0, lo), floor rows [hi, H)) or a middle-band pixel (wall, or
// void when s >= max_range); lo/hi were classified exactly in FP64 by the
// column epilogue.  Depth (f32) and semantic (u16) are selected exactly.  RGB
// is shaded in f16 pairs, two pixels per instruction:
//   t   = 0.2 + (0.8 cos-numerator) * inv      inv = 1/|(d, v)| from the f16 table
//                                              invh (env-independent; rows mirrored)
//   c8  = round(col255 * t)                    via HFMA2(col255, t, 1024): the
//                                              low byte of the f16 result
// Worst-case error vs the reference's f64 rgb: 0.5 (rounding) + 0.0625 (f16
// col255) + 255 * 1e-3 (t) < 0.85 of one 8-bit step (tolerance: 1 step).
//
// Lane mapping (all fast writers): a warp covers a row segment of 32*CPL
// columns; lane l owns CPL/GW groups of GW = min(CPL, 4) adjacent columns,
// group g at segment offset g*32*GW + l*GW.  A warp's group-g stores are then
// contiguous across lanes (12-byte RGB, 16-byte depth, 8-byte semantic
// strides: bank-conflict-free shared-memory rows), and its column records are
// 32 consecutive 16-byte halves (device.cuh rec_pos).

#define NV_H2_POINT2 0x32663266u   // (0.2, 0.2) in f16
#define NV_H2_1024 0x64006400u     // (1024, 1024): low byte of 1024+x = round(x)

struct FillArgs {
  const float4 *ra, *rb;  // column-record planes (device.cuh), index env * W + rec_pos
  int cpl;                // record order
  const RowRec *rows;
  int N, W, H;
  uint8_t *rgb;
  float *depth;
  uint16_t *sem;
  int rows_per_unit;   // rows of one work unit
  int units_per_seg;   // ceil(H / rows_per_unit)
  int segs_per_row;    // W / (32 * CPL)
  long long n_units;   // N * segs_per_row * units_per_seg
  unsigned int *ctr;   // [0] next unit, [1] finished warps (self-resetting)
  const uint16_t *invh;  // ceil(H/2) x W f16 shading table 1/|(d_j, v_i)|, rows
                         // mirrored (v_{H-1-i} = -v_i); env-independent
  // inverse-depth noise (sensors.apply_inverse_depth_noise, sensors.py:183-205)
  float noise_sigma;     // 0 = off
  float max_range;
  unsigned long long noise_seed, noise_frame;
  long long env_offset;  // global id of env 0 (sharding-invariant streams)
};

// ---- inverse-depth noise ---------------------------------------------------
// z' = max_range / (max_range / d + eps), eps ~ N(0, sigma), clamped to
// [0.05, max_range]; saturated pixels (d >= max_range) pass through
// (sensors.py:195-205).  eps comes from a counter-based generator: one
// splitmix64 draw per horizontal pixel pair, keyed by (seed, frame, global
// env, row, pair), turned into two normals by Box-Muller -- so every fill
// path produces the same noisy frame.  numpy's Generator.normal stream
// cannot be reproduced on the device; parity is distributional (the
// reference's own moment test, tests/test_sensors.py:179-184).
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float2 noise_pair(const FillArgs &a, int env, int row, int col) {
  const unsigned long long key =
      ((((a.noise_frame << 20) ^ (unsigned long long)(env + a.env_offset)) * (unsigned long long)a.H +
        (unsigned long long)row) * (unsigned long long)a.W + (unsigned long long)col) >> 1;
  const unsigned long long z = splitmix64(a.noise_seed ^ splitmix64(key));
  const float u1 = (float)((z >> 40) + 1ull) * 0x1p-24f;           // (0, 1]
  const float u2 = (float)((z >> 16) & 0xFFFFFFull) * 0x1p-24f;     // [0, 1)
  const float r = sqrtf(-2.0f * __logf(u1));
  float sn, cs;
  __sincosf(6.283185307f * u2, &sn, &cs);
  return make_float2(r * cs * a.noise_sigma, r * sn * a.noise_sigma);
}

__device__ __forceinline__ float noisy_depth(float d, float eps, float max_range) {
  if (!(d < max_range)) return d;
  const float inv = max_range / d + eps;
  const float z = inv != 0.0f ? max_range / inv : __int_as_float(0x7f800000);
  return fminf(fmaxf(z, 0.05f), max_range);
}

template <int CPL>
struct Lanes {
  static constexpr int GW = CPL < 4 ? CPL : 4;  // columns per group
  static constexpr int G = CPL / GW;            // groups per lane
  static constexpr int SEGW = 32 * CPL;         // columns per warp segment
};

__device__ __forceinline__ uint32_t h2_fma(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t h2_pack(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// (a & m) | (b & ~m): per-half select with a 0xFFFF-granular mask
__device__ __forceinline__ uint32_t sel_mask(uint32_t a, uint32_t b, uint32_t m) {
  return (a & m) | (b & ~m);
}

__device__ __forceinline__ unsigned smem_addr(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void bulk_store(void *gdst, const void *ssrc, unsigned bytes,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n" ::"l"(
          gdst),
      "r"(smem_addr(ssrc)), "r"(bytes), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy completing on an mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void bulk_load(void *sdst, const void *gsrc, unsigned bytes,
                                          uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// A lane's CPL columns (CPL/2 pixel pairs, column k = g*GW + c) in registers.
template <int CPL>
struct ColRegs {
  float dw[CPL];                 // wall depth (or max_range)
  uint32_t lo[CPL], hi[CPL];     // plane rows: i < lo or i >= hi
  uint32_t nw[CPL / 2], rw[CPL / 2], gw[CPL / 2], bw[CPL / 2];  // f16 pairs
  uint32_t sw[CPL / 2];          // semantic pairs
};

template <int CPL>
__device__ __forceinline__ void unpack_cols(const float4 (&A)[CPL], const float4 (&B)[CPL],
                                            ColRegs<CPL> &cr) {
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    cr.dw[k] = A[k].x;
    const uint32_t l = __float_as_uint(A[k].w);
    cr.lo[k] = l & 0xffffu;
    cr.hi[k] = l >> 16;
  }
#pragma unroll
  for (int m = 0; m < CPL / 2; ++m) {
    cr.nw[m] = h2_pack(A[2 * m].y, A[2 * m + 1].y);
    cr.rw[m] = h2_pack(B[2 * m].x, B[2 * m + 1].x);
    cr.gw[m] = h2_pack(B[2 * m].y, B[2 * m + 1].y);
    cr.bw[m] = h2_pack(B[2 * m].z, B[2 * m + 1].z);
    cr.sw[m] = (__float_as_uint(B[2 * m].w) & 0xffffu) | (__float_as_uint(B[2 * m + 1].w) << 16);
  }
}

// Global planes; base = env * W + seg * SEGW (records in rec_pos order).
// COH: written earlier in the same launch (read through L2).
template <int CPL, bool COH>
__device__ __forceinline__ void load_cols(const FillArgs &a, size_t base, int lane,
                                          ColRegs<CPL> &cr) {
  float4 A[CPL], B[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    const size_t p = base + (size_t)k * 32 + lane;
    if (COH) {
      A[k] = __ldcg(a.ra + p);
      B[k] = __ldcg(a.rb + p);
    } else {
      A[k] = __ldg(a.ra + p);
      B[k] = __ldg(a.rb + p);
    }
  }
  unpack_cols<CPL>(A, B, cr);
}

// Shared-memory planes of one env: sA/sB + seg * SEGW.
template <int CPL>
__device__ __forceinline__ void load_cols_smem(const float4 *sA, const float4 *sB, int lane,
                                               ColRegs<CPL> &cr) {
  float4 A[CPL], B[CPL];
#pragma unroll
  for (int k = 0; k < CPL; ++k) {
    A[k] = sA[k * 32 + lane];
    B[k] = sB[k * 32 + lane];
  }
  unpack_cols<CPL>(A, B, cr);
}

// Shade one pixel pair (columns 2k, 2k+1 of the lane) of row i.
struct PairOut {
  uint32_t r, g, b, s;  // f16 pairs (low byte of each half = value), sem pair
  float d0, d1;
};

__device__ __forceinline__ PairOut shade_pair(uint32_t i, const RowRec &R, uint32_t lo0,
                                              uint32_t hi0, uint32_t lo1, uint32_t hi1, float dw0,
                                              float dw1, uint32_t nw, uint32_t rw, uint32_t gw,
                                              uint32_t bw, uint32_t sw, uint32_t inv2) {
  const bool in0 = i >= lo0 && i < hi0;  // middle band (wall / void)
  const bool in1 = i >= lo1 && i < hi1;
  const uint32_t m = (in0 ? 0x0000ffffu : 0u) | (in1 ? 0xffff0000u : 0u);
  PairOut o;
  o.d0 = in0 ? dw0 : R.depth_p;
  o.d1 = in1 ? dw1 : R.depth_p;
  o.s = sel_mask(sw, R.sem2, m);
  const uint32_t num = sel_mask(nw, R.num2, m);
  const uint32_t t = h2_fma(num, inv2, NV_H2_POINT2);
  o.r = h2_fma(sel_mask(rw, R.r2, m), t, NV_H2_1024);
  o.g = h2_fma(sel_mask(gw, R.g2, m), t, NV_H2_1024);
  o.b = h2_fma(sel_mask(bw, R.b2, m), t, NV_H2_1024);
  return o;
}

// Two pixel pairs (4 pixels) -> 12 interleaved RGB bytes (3 words).
__device__ __forceinline__ void pack_rgb4(const PairOut &p, const PairOut &q, uint32_t &w0,
                                          uint32_t &w1, uint32_t &w2) {
  const uint32_t rg0 = __byte_perm(p.r, p.g, 0x6240);  // r0 g0 r1 g1
  const uint32_t rg1 = __byte_perm(q.r, q.g, 0x6240);  // r2 g2 r3 g3
  w0 = __byte_perm(rg0, p.b, 0x2410);                  // r0 g0 b0 r1
  const uint32_t t = __byte_perm(rg0, p.b, 0x3263);    // g1 b1 . .
  w1 = __byte_perm(t, rg1, 0x5410);                    // g1 b1 r2 g2
  w2 = __byte_perm(rg1, q.b, 0x6324);                  // b2 r3 g3 b3
}

__device__ __forceinline__ RowRec unpack_row(const RowRec *rows_s, uint32_t i) {
  const uint4 *rq = reinterpret_cast<const uint4 *>(rows_s + i);
  const uint4 q0 = rq[0], q1 = rq[1];
  RowRec R;
  R.depth_p = __uint_as_float(q0.x);
  R.sem2 = q0.y;
  R.num2 = q0.z;
  R.r2 = q0.w;
  R.g2 = q1.x;
  R.b2 = q1.y;
  return R;
}

// Shading-table row of image row i: the table holds rows [0, ceil(H/2)) and
// row H-1-i equals row i (v_{H-1-i} = -v_i exactly).
__device__ __forceinline__ uint32_t inv_row(uint32_t i, int H) {
  return i < (uint32_t)(H >> 1) ? i : (uint32_t)(H - 1) - i;
}

// The lane's shading-table pairs from table row `ip` (+ segment offset).
template <int CPL, bool GLOBAL>
__device__ __forceinline__ void load_inv(const uint16_t *ip, int lane, uint32_t (&iv)[CPL / 2]) {
  using Ln = Lanes<CPL>;
#pragma unroll
  for (int g = 0; g < Ln::G; ++g) {
    const uint16_t *q = ip + g * 32 * Ln::GW + lane * Ln::GW;
    if constexpr (Ln::GW == 4) {
      const uint2 v = GLOBAL ? __ldg(reinterpret_cast<const uint2 *>(q))
                             : *reinterpret_cast<const uint2 *>(q);
      iv[2 * g] = v.x;
      iv[2 * g + 1] = v.y;
    } else {
      iv[g] = GLOBAL ? __ldg(reinterpret_cast<const uint32_t *>(q))
                     : *reinterpret_cast<const uint32_t *>(q);
    }
  }
}

template <int CPL>
__device__ __forceinline__ void shade_row(uint32_t i, const RowRec &R, const ColRegs<CPL> &cr,
                                          const uint32_t (&iv)[CPL / 2],
                                          PairOut (&po)[CPL / 2]) {
#pragma unroll
  for (int c = 0; c < CPL / 2; ++c)
    po[c] = shade_pair(i, R, cr.lo[2 * c], cr.hi[2 * c], cr.lo[2 * c + 1], cr.hi[2 * c + 1],
                       cr.dw[2 * c], cr.dw[2 * c + 1], cr.nw[c], cr.rw[c], cr.gw[c], cr.bw[c],
                       cr.sw[c], iv[c]);
}

// Writes the lane's shaded pixels of one row segment into a buffer laid out
// like the frame (shared-memory stage / slot): px0 = pixel index of the
// segment's first column in the buffer.
template <int CPL>
__device__ __forceinline__ void put_row(const PairOut (&po)[CPL / 2], uint8_t *rgb, float *dep,
                                        uint16_t *sem, int px0, int lane) {
  using Ln = Lanes<CPL>;
#pragma unroll
  for (int g = 0; g < Ln::G; ++g) {
    const int px = px0 + g * 32 * Ln::GW + lane * Ln::GW;
    if constexpr (Ln::GW == 4) {
      const PairOut &p = po[2 * g], &q = po[2 * g + 1];
      if (rgb) {
        uint32_t w0, w1, w2;
        pack_rgb4(p, q, w0, w1, w2);
        uint32_t *d = reinterpret_cast<uint32_t *>(rgb + (size_t)px * 3);
        d[0] = w0;
        d[1] = w1;
        d[2] = w2;
      }
      if (dep) *reinterpret_cast<float4 *>(dep + px) = make_float4(p.d0, p.d1, q.d0, q.d1);
      if (sem) *reinterpret_cast<uint2 *>(sem + px) = make_uint2(p.s, q.s);
    } else {
      const PairOut &p = po[g];
      if (rgb) {
        uint16_t *d16 = reinterpret_cast<uint16_t *>(rgb + (size_t)px * 3);
        d16[0] = (uint16_t)__byte_perm(p.r, p.g, 0x0040);  // r0 g0
        d16[1] = (uint16_t)__byte_perm(p.b, p.r, 0x0060);  // b0 r1
        d16[2] = (uint16_t)__byte_perm(p.g, p.b, 0x0062);  // g1 b1
      }
      if (dep) *reinterpret_cast<float2 *>(dep + px) = make_float2(p.d0, p.d1);
      if (sem) *reinterpret_cast<uint32_t *>(sem + px) = p.s;
    }
  }
}

// Copies the camera's row table (H x 32 B) into shared memory; every warp of
// the CTA reads its rows from there (uniform LDS, no L1/L2 misses under the
// write stream).  Returns the first byte after the table (16-aligned).
__device__ __forceinline__ uint8_t *stage_rows(const FillArgs &a, uint8_t *smem) {
  const uint4 *src = reinterpret_cast<const uint4 *>(a.rows);
  uint4 *dst = reinterpret_cast<uint4 *>(smem);
  for (int k = threadIdx.x; k < a.H * 2; k += blockDim.x) dst[k] = __ldg(src + k);
  __syncthreads();
  return smem + (size_t)a.H * sizeof(RowRec);
}

// Per-warp state of the streaming writer: a private ring of NS smem stages.
template <int CPL, int RW>
struct FillWarp {
  static constexpr int NS = 2;
  static constexpr int SEGW = 32 * CPL;
  uint8_t *wbase;
  const RowRec *rows_s;  // shared-memory row table
  int off_d, off_s, stage_bytes;
  bool want_rgb, want_d, want_s;
  uint64_t pol;
  int k;  // stages issued so far
  // smem layout: [row table H x 32 B][per-warp stage rings]
  __device__ __forceinline__ void init(const FillArgs &a, uint8_t *smem, int wib) {
    rows_s = reinterpret_cast<const RowRec *>(smem);
    smem = stage_rows(a, smem);
    want_rgb = a.rgb != nullptr;
    want_d = a.depth != nullptr;
    want_s = a.sem != nullptr;
    off_d = want_rgb ? RW * SEGW * 3 : 0;
    off_s = off_d + (want_d ? RW * SEGW * 4 : 0);
    stage_bytes = off_s + (want_s ? RW * SEGW * 2 : 0);
    wbase = smem + (size_t)wib * NS * stage_bytes;
    pol = policy_evict_first();
    k = 0;
  }
};

// Render one unit = (env, column segment of 32*CPL columns, rows
// [gidx*rpu, ...)) of fill_frame: the lane's CPL columns' parameters sit in
// registers; RW rows at a time are rendered into a smem stage laid out exactly
// like global memory, which lane 0 writes out with cp.async.bulk (one copy
// per channel per stage when a warp covers full rows), evict-first in L2.
// COH: the column records were written earlier in the same launch.
template <int CPL, int RW, bool COH>
__device__ __forceinline__ void fill_unit(const FillArgs &a, FillWarp<CPL, RW> &fw, int env,
                                          int seg, int gidx) {
  constexpr int NS = FillWarp<CPL, RW>::NS;
  constexpr int SEGW = FillWarp<CPL, RW>::SEGW;
  const int lane = threadIdx.x & 31;
  const int W = a.W, H = a.H;
  ColRegs<CPL> cr;
  load_cols<CPL, COH>(a, (size_t)env * W + (size_t)seg * SEGW, lane, cr);
  const int r_begin = gidx * a.rows_per_unit;
  const int r_end = min(H, r_begin + a.rows_per_unit);
  for (int r0 = r_begin; r0 < r_end; r0 += RW) {
    const int nr = min(RW, r_end - r0);
    uint8_t *buf = fw.wbase + (fw.k & (NS - 1)) * fw.stage_bytes;
    if (fw.k >= NS) {
      if (lane == 0) bulk_wait_read<NS - 1>();
      __syncwarp();
    }
    for (int rr = 0; rr < nr; ++rr) {
      const uint32_t i = (uint32_t)(r0 + rr);
      const RowRec R = unpack_row(fw.rows_s, i);
      uint32_t iv[CPL / 2];
      load_inv<CPL, true>(a.invh + (size_t)inv_row(i, H) * W + seg * SEGW, lane, iv);
      PairOut po[CPL / 2];
      shade_row<CPL>(i, R, cr, iv, po);
      put_row<CPL>(po, fw.want_rgb ? buf : nullptr,
                   fw.want_d ? reinterpret_cast<float *>(buf + fw.off_d) : nullptr,
                   fw.want_s ? reinterpret_cast<uint16_t *>(buf + fw.off_s) : nullptr,
                   rr * SEGW, lane);
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) {
      if (a.segs_per_row == 1) {
        const size_t pix0 = ((size_t)env * H + r0) * W;
        if (fw.want_rgb) bulk_store(a.rgb + pix0 * 3, buf, (unsigned)(nr * W * 3), fw.pol);
        if (fw.want_d) bulk_store(a.depth + pix0, buf + fw.off_d, (unsigned)(nr * W * 4), fw.pol);
        if (fw.want_s) bulk_store(a.sem + pix0, buf + fw.off_s, (unsigned)(nr * W * 2), fw.pol);
      } else {
        for (int rr = 0; rr < nr; ++rr) {
          const size_t pix0 = ((size_t)env * H + r0 + rr) * W + (size_t)seg * SEGW;
          if (fw.want_rgb)
            bulk_store(a.rgb + pix0 * 3, buf + rr * SEGW * 3, (unsigned)(SEGW * 3), fw.pol);
          if (fw.want_d)
            bulk_store(a.depth + pix0, buf + fw.off_d + rr * SEGW * 4, (unsigned)(SEGW * 4),
                       fw.pol);
          if (fw.want_s)
            bulk_store(a.sem + pix0, buf + fw.off_s + rr * SEGW * 2, (unsigned)(SEGW * 2), fw.pol);
        }
      }
      bulk_commit();
    }
    ++fw.k;
  }
}

// Drains this warp's bulk stores and, for the last warp of the grid, resets
// the self-resetting work counter for the next launch.
__device__ __forceinline__ void finish_grid(unsigned int *ctr) {
  if ((threadIdx.x & 31) == 0) {
    bulk_wait_all();
    const unsigned total_warps = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(ctr + 1, 1u) == total_warps - 1) {
      ctr[0] = 0;
      ctr[1] = 0;
      __threadfence();
    }
  }
}

// k_fill_tma: streaming frame writer over all units of a frame batch; units
// are pulled from a self-resetting global counter (one prefetched ahead).
template <int CPL, int RW>
__global__ void __launch_bounds__(128) k_fill_tma(FillArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  FillWarp<CPL, RW> fw;
  fw.init(a, smem, threadIdx.x >> 5);
  long long u = 0;
  if (lane == 0) u = atomicAdd(a.ctr, 1u);
  u = __shfl_sync(0xffffffffu, u, 0);
  while (u < a.n_units) {
    long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.ctr, 1u);
    // row-block-major order: warps across the GPU render the same rows of
    // different envs at the same time (shared row records / table rows)
    const long long n_es = (long long)a.N * a.segs_per_row;
    const int gidx = (int)(u / n_es);
    const long long es = u - (long long)gidx * n_es;
    const int env = (int)(es / a.segs_per_row);
    const int seg = (int)(es - (long long)env * a.segs_per_row);
    fill_unit<CPL, RW, false>(a, fw, env, seg, gidx);
    u = __shfl_sync(0xffffffffu, nxt, 0);
  }
  finish_grid(a.ctr);
}

// ---- direct-store variant: no smem staging ---------------------------------
// Each lane stores its pixels of a row straight from registers with
// evict-first 128/64/32-bit stores; a warp's group-g stores are contiguous.
__device__ __forceinline__ void st_v4f(float *p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_v2u(void *p, uint32_t a, uint32_t b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.b32 [%0], {%1,%2}, %3;" ::"l"(p), "r"(a), "r"(b),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void st_u(void *p, uint32_t a, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(a), "l"(pol)
               : "memory");
}

template <int CPL, bool COH>
__device__ __forceinline__ void fill_unit_direct(const FillArgs &a, const RowRec *rows_s,
                                                 uint64_t pol, int env, int seg, int gidx) {
  using Ln = Lanes<CPL>;
  const int lane = threadIdx.x & 31;
  const int W = a.W, H = a.H;
  ColRegs<CPL> cr;
  load_cols<CPL, COH>(a, (size_t)env * W + (size_t)seg * Ln::SEGW, lane, cr);
  const int r_begin = gidx * a.rows_per_unit;
  const int r_end = min(H, r_begin + a.rows_per_unit);
  for (int r = r_begin; r < r_end; ++r) {
    const uint32_t i = (uint32_t)r;
    const RowRec R = unpack_row(rows_s, i);
    uint32_t iv[CPL / 2];
    load_inv<CPL, true>(a.invh + (size_t)inv_row(i, H) * W + seg * Ln::SEGW, lane, iv);
    PairOut po[CPL / 2];
    shade_row<CPL>(i, R, cr, iv, po);
    const size_t row0 = ((size_t)env * H + r) * W + (size_t)seg * Ln::SEGW;
#pragma unroll
    for (int g = 0; g < Ln::G; ++g) {
      const size_t px = row0 + g * 32 * Ln::GW + lane * Ln::GW;
      if constexpr (Ln::GW == 4) {
        const PairOut &p = po[2 * g], &q = po[2 * g + 1];
        if (a.rgb) {
          uint32_t w0, w1, w2;
          pack_rgb4(p, q, w0, w1, w2);
          uint8_t *d = a.rgb + px * 3;
          st_u(d, w0, pol);
          st_u(d + 4, w1, pol);
          st_u(d + 8, w2, pol);
        }
        if (a.depth) st_v4f(a.depth + px, make_float4(p.d0, p.d1, q.d0, q.d1), pol);
        if (a.sem) st_v2u(a.sem + px, p.s, q.s, pol);
      } else {
        const PairOut &p = po[g];
        if (a.rgb) {
          uint16_t *d16 = reinterpret_cast<uint16_t *>(a.rgb + px * 3);
          d16[0] = (uint16_t)__byte_perm(p.r, p.g, 0x0040);
          d16[1] = (uint16_t)__byte_perm(p.b, p.r, 0x0060);
          d16[2] = (uint16_t)__byte_perm(p.g, p.b, 0x0062);
        }
        if (a.depth) *reinterpret_cast<float2 *>(a.depth + px) = make_float2(p.d0, p.d1);
        if (a.sem) *reinterpret_cast<uint32_t *>(a.sem + px) = p.s;
      }
    }
  }
}

template <int CPL>
__global__ void __launch_bounds__(128) k_fill_direct(FillArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  stage_rows(a, smem);
  const RowRec *rows_s = reinterpret_cast<const RowRec *>(smem);
  const int lane = threadIdx.x & 31;
  const uint64_t pol = policy_evict_first();
  long long u = 0;
  if (lane == 0) u = atomicAdd(a.ctr, 1u);
  u = __shfl_sync(0xffffffffu, u, 0);
  while (u < a.n_units) {
    long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(a.ctr, 1u);
    const long long n_es = (long long)a.N * a.segs_per_row;
    const int gidx = (int)(u / n_es);
    const long long es = u - (long long)gidx * n_es;
    const int env = (int)(es / a.segs_per_row);
    const int seg = (int)(es - (long long)env * a.segs_per_row);
    fill_unit_direct<CPL, false>(a, rows_s, pol, env, seg, gidx);
    u = __shfl_sync(0xffffffffu, nxt, 0);
  }
  finish_grid(a.ctr);
}

// ---- warp-specialised frame writer ------------------------------------------
//
// k_fill_ws: persistent, one CTA per SM = NW producer warps + 1 store warp; a
// work item is one env's frame.  Producers render rows into a ring of NSLOT
// shared-memory slots (a slot = R consecutive frame rows, all channels, laid
// out exactly like the frame, so ONE bulk copy per channel writes it out);
// the store warp's elected lane waits on the slot's `full` mbarrier, issues
// the cp.async.bulk stores (evict-first), and releases the previous slot
// through its `empty` mbarrier once the bulk engine has read it.  The same
// lane prefetches the next item's column-record planes into a double buffer
// with bulk copies.  Producers never touch L2: row records, the shading table
// and column records are all shared-memory reads.
#ifndef NV_WS_DEBUG
#define NV_WS_DEBUG 0  // 1: producers skip rendering, 2: no bulk stores (bound studies)
#endif
struct FillWsLayout {  // byte offsets into dynamic shared memory + ring geometry
  int rows, inv, cols, bars, slots;
  int slot_bytes, nslot, slot_rows;
  int depth_direct;  // 1: producers store depth straight from registers (STG),
                     // the slots carry RGB / semantic only
};

template <int CPL, bool TAB, int RPW, bool NOISE>
__global__ void __launch_bounds__(544, 1) k_fill_ws(FillArgs a, FillWsLayout L) {
  extern __shared__ __align__(128) uint8_t smem[];
  using Ln = Lanes<CPL>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x >> 5) - 1;  // producer warps
  const int W = a.W, H = a.H, S = a.segs_per_row, R = L.slot_rows, NSLOT = L.nslot;
  const RowRec *rows_s = reinterpret_cast<const RowRec *>(smem + L.rows);
  const uint16_t *inv_s = reinterpret_cast<const uint16_t *>(smem + L.inv);
  float4 *cols_s = reinterpret_cast<float4 *>(smem + L.cols);  // [buf][A | B][W]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bars);
  uint64_t *empty = full + NSLOT;
  uint64_t *colfull = empty + NSLOT;
  uint64_t *colempty = colfull + 2;
  uint8_t *slots = smem + L.slots;
  const unsigned plane_bytes = (unsigned)W * 16u;
  const bool want_rgb = a.rgb != nullptr, want_d = a.depth != nullptr, want_s = a.sem != nullptr;
  const bool slot_d = want_d && !L.depth_direct;
  const int off_d = want_rgb ? R * W * 3 : 0;
  const int off_s = off_d + (slot_d ? R * W * 4 : 0);
  const int slots_per_item = H / R;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NSLOT; ++k) {
      mbar_init(full + k, (unsigned)nw);
      mbar_init(empty + k, 1);
    }
    for (int k = 0; k < 2; ++k) {
      mbar_init(colfull + k, 1);
      mbar_init(colempty + k, (unsigned)nw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(a.rows);
    uint4 *dst = reinterpret_cast<uint4 *>(smem + L.rows);
    for (int k = threadIdx.x; k < H * 2; k += blockDim.x) dst[k] = __ldg(src + k);
    if (TAB) {
      const uint4 *s2 = reinterpret_cast<const uint4 *>(a.invh);
      uint4 *d2 = reinterpret_cast<uint4 *>(smem + L.inv);
      const int n16 = ((H + 1) / 2) * W * 2 / 16;
      for (int k = threadIdx.x; k < n16; k += blockDim.x) d2[k] = __ldg(s2 + k);
    }
  }
  __syncthreads();
  if (warp == nw) {
    // ------------------------------------------------------------ store warp
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    auto load_item = [&](int buf, int env) {
      uint64_t *b = colfull + buf;
      mbar_expect_tx(b, 2 * plane_bytes);
      bulk_load(cols_s + (size_t)buf * 2 * W, a.ra + (size_t)env * W, plane_bytes, b);
      bulk_load(cols_s + (size_t)buf * 2 * W + W, a.rb + (size_t)env * W, plane_bytes, b);
    };
    int e = blockIdx.x;
    if (e < a.N) load_item(0, e);
    unsigned k = 0, slot = 0, use = 0, prev = 0;
    for (int it = 0; e < a.N; ++it, e += gridDim.x) {
      const int en = e + gridDim.x;
      if (en < a.N) {
        const int j = it + 1;
        if (j >= 2) mbar_wait(colempty + (j & 1), (unsigned)(((j >> 1) - 1) & 1));
        load_item(j & 1, en);
      }
      for (int sl = 0; sl < slots_per_item; ++sl, ++k) {
        mbar_wait(full + slot, use & 1u);
        const uint8_t *buf = slots + (size_t)slot * L.slot_bytes;
        const size_t pix0 = ((size_t)e * H + (size_t)sl * R) * W;
#if NV_WS_DEBUG != 2
        if (want_rgb) bulk_store(a.rgb + pix0 * 3, buf, (unsigned)(R * W * 3), pol);
        if (slot_d) bulk_store(a.depth + pix0, buf + off_d, (unsigned)(R * W * 4), pol);
        if (want_s) bulk_store(a.sem + pix0, buf + off_s, (unsigned)(R * W * 2), pol);
#else
        (void)buf; (void)pix0; (void)pol;
#endif
        bulk_commit();
        if (k >= 1) {
          bulk_wait_read<1>();
          mbar_arrive(empty + prev);
        }
        prev = slot;
        if (++slot == (unsigned)NSLOT) {
          slot = 0;
          ++use;
        }
      }
    }
    bulk_wait_all();
    return;
  }
  // -------------------------------------------------------------- producers
  const uint64_t dpol = policy_evict_first();
  const int seg = warp % S;
  const int rsub = warp / S;   // first row of this warp within a slot
  const int rstride = nw / S;  // row stride between the warp's RPW rows
  unsigned slot = 0, use = 0;
  int e = blockIdx.x;
  for (int it = 0; e < a.N; ++it, e += gridDim.x) {
    mbar_wait(colfull + (it & 1), (unsigned)((it >> 1) & 1));
    ColRegs<CPL> cr;
    const float4 *cA = cols_s + (size_t)(it & 1) * 2 * W + seg * Ln::SEGW;
    load_cols_smem<CPL>(cA, cA + W, lane, cr);
    __syncwarp();
    if (lane == 0) mbar_arrive(colempty + (it & 1));
    for (int sl = 0; sl < slots_per_item; ++sl) {
      if (use >= 1) mbar_wait(empty + slot, (use - 1) & 1u);
      uint8_t *buf = slots + (size_t)slot * L.slot_bytes;
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int rs = rsub + rr * rstride;  // row within the slot
        const uint32_t i = (uint32_t)(sl * R + rs);
#if NV_WS_DEBUG == 1
        (void)buf; (void)i;
        continue;
#endif
        const RowRec Rr = unpack_row(rows_s, i);
        uint32_t iv[CPL / 2];
        if constexpr (TAB)
          load_inv<CPL, false>(inv_s + (size_t)inv_row(i, H) * W + seg * Ln::SEGW, lane, iv);
        else
          load_inv<CPL, true>(a.invh + (size_t)inv_row(i, H) * W + seg * Ln::SEGW, lane, iv);
        PairOut po[CPL / 2];
        shade_row<CPL>(i, Rr, cr, iv, po);
        if constexpr (NOISE) {
#pragma unroll
          for (int c = 0; c < CPL / 2; ++c) {
            const int col = seg * Ln::SEGW + (c / (Ln::GW / 2)) * 32 * Ln::GW + lane * Ln::GW +
                            2 * (c % (Ln::GW / 2));
            const float2 n = noise_pair(a, e, (int)i, col);
            po[c].d0 = noisy_depth(po[c].d0, n.x, a.max_range);
            po[c].d1 = noisy_depth(po[c].d1, n.y, a.max_range);
          }
        }
        put_row<CPL>(po, want_rgb ? buf : nullptr,
                     slot_d ? reinterpret_cast<float *>(buf + off_d) : nullptr,
                     want_s ? reinterpret_cast<uint16_t *>(buf + off_s) : nullptr,
                     rs * W + seg * Ln::SEGW, lane);
        if (want_d && !slot_d) {  // depth straight to HBM: 16 B per lane, coalesced
          float *drow = a.depth + ((size_t)e * H + i) * W + seg * Ln::SEGW;
#pragma unroll
          for (int g = 0; g < Ln::G; ++g) {
            float *dp = drow + g * 32 * Ln::GW + lane * Ln::GW;
            if constexpr (Ln::GW == 4) {
              const PairOut &p = po[2 * g], &q = po[2 * g + 1];
              asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(dp),
                           "f"(p.d0), "f"(p.d1), "f"(q.d0), "f"(q.d1), "l"(dpol)
                           : "memory");
            } else {
              *reinterpret_cast<float2 *>(dp) = make_float2(po[g].d0, po[g].d1);
            }
          }
        }
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(full + slot);
      if (++slot == (unsigned)NSLOT) {
        slot = 0;
        ++use;
      }
    }
  }
}

// ----------------------------------------------------------- megakernel
//
// k_step_render: one launch per simulator step.  Persistent warps pull tasks
// from a host-built queue in which every dependency precedes its dependents:
//   STEP(e)      Simulator.step kinematics of env e            (one warp)
//   CAST(e, c)   32 columns of env e: DDA + epilogue -> ColRec  (one warp)
//   FILL(e, u)   one fill unit of env e                         (one warp)
// The queue interleaves STEP(e + LS + LC), CAST(e + LC, *), FILL(e, *) so the
// latency-bound casts run ahead of, and overlap with, the HBM-bound fill.
// Per-env counters (step done, casts done, fills done) carry the
// dependencies (release/acquire through L2); the last fill of an env resets
// them for the next launch, the last warp resets the queue counter.
// Every dequeued task's dependencies were dequeued earlier by running warps,
// so waiting can never deadlock.
enum : int { NV_TASK_STEP = 0, NV_TASK_CAST = 1, NV_TASK_FILL = 2 };

struct MegaArgs {
  EnvView ev;
  SceneView sc;
  CamView cam;
  AgentCfg cfg;
  FillArgs f;
  RecOut ro;  // the same planes as f.ra / f.rb, writable
  const int8_t *actions;
  uint8_t *collided;
  double *disp;
  int32_t *status;
  double *gps, *compass;
  double t_max;
  const int2 *tasks;  // (type << 24 | sub, env)
  int n_tasks;
  int n_cast;         // cast tasks per env
  int n_fill;         // fill tasks per env
  unsigned int *envsync;  // 3 per env: step done, casts done, fills done
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_at_least(const unsigned *p, unsigned target) {
  if ((threadIdx.x & 31) == 0) {
    unsigned ns = 32;
    while (ld_acquire(p) < target) {
      __nanosleep(ns);
      ns = min(ns * 2, 256u);
    }
  }
  __syncwarp();
}

template <int CPL, int RW>
__global__ void __launch_bounds__(128) k_step_render(MegaArgs m) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  FillWarp<CPL, RW> fw;
  fw.init(m.f, smem, threadIdx.x >> 5);
  long long slot = 0;
  if (lane == 0) slot = atomicAdd(m.f.ctr, 1u);
  slot = __shfl_sync(0xffffffffu, slot, 0);
  while (slot < m.n_tasks) {
    long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(m.f.ctr, 1u);
    const int2 t = __ldg(m.tasks + slot);
    const int type = t.x >> 24, sub = t.x & 0xffffff, e = t.y;
    unsigned *sync = m.envsync + 3 * (size_t)e;
    if (type == NV_TASK_STEP) {
      warp_agent_step(m.ev, m.sc, m.cfg, e, m.actions[e], m.collided, m.disp, m.status);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicExch(sync, 1u);
      }
    } else if (type == NV_TASK_CAST) {
      wait_at_least(sync, 1u);
      const int j = sub * 32 + lane;
      if (j < m.cam.W) cast_column<true>(m.ev, m.sc, m.cam, e, j, m.ro, m.t_max, m.gps, m.compass);
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAdd(sync + 1, 1u);
      }
    } else {
      wait_at_least(sync + 1, (unsigned)m.n_cast);
      const int seg = sub / m.f.units_per_seg;
      const int gidx = sub - seg * m.f.units_per_seg;
      fill_unit<CPL, RW, true>(m.f, fw, e, seg, gidx);
      if (lane == 0 && atomicAdd(sync + 2, 1u) == (unsigned)m.n_fill - 1) {
        sync[0] = 0;  // every task of env e is done: reset for the next launch
        sync[1] = 0;
        sync[2] = 0;
      }
    }
    slot = __shfl_sync(0xffffffffu, nxt, 0);
  }
  finish_grid(m.f.ctr);
}

// Inverse-depth noise as a separate pass over a written depth batch (the
// writers other than k_fill_ws); same per-pixel values as the fused path.
__global__ void k_depth_noise(FillArgs a, float *depth) {
  const long long p2 = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // pixel pair
  const int half = (a.W + 1) / 2;
  const long long total = (long long)a.N * a.H * half;
  if (p2 >= total) return;
  const int cp = (int)(p2 % half);
  const long long er = p2 / half;
  const int row = (int)(er % a.H), env = (int)(er / a.H);
  const float2 n = noise_pair(a, env, row, 2 * cp);
  float *d = depth + ((size_t)env * a.H + row) * a.W + 2 * cp;
  d[0] = noisy_depth(d[0], n.x, a.max_range);
  if (2 * cp + 1 < a.W) d[1] = noisy_depth(d[1], n.y, a.max_range);
}

// One thread per pixel, any W/H; the same f16 arithmetic as the fast writers
// (one half of each pair), so every path produces identical frames.
__global__ void k_fill_generic(FillArgs a) {
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long total = (long long)a.N * a.H * a.W;
  if (p >= total) return;
  const int j = (int)(p % a.W);
  const long long ei = p / a.W;
  const uint32_t i = (uint32_t)(ei % a.H);
  const int e = (int)(ei / a.H);
  const size_t q = (size_t)e * a.W + rec_pos(j, a.cpl);
  const float4 A = a.ra[q], B = a.rb[q];
  const RowRec R = a.rows[i];
  const uint32_t l = __float_as_uint(A.w);
  const uint32_t lo = l & 0xffffu, hi = l >> 16;
  const uint32_t inv = a.invh[(size_t)inv_row(i, a.H) * a.W + j];
  PairOut o = shade_pair(i, R, lo, hi, lo, hi, A.x, A.x, h2_pack(A.y, 0.f), h2_pack(B.x, 0.f),
                         h2_pack(B.y, 0.f), h2_pack(B.z, 0.f), __float_as_uint(B.w) & 0xffffu,
                         inv);
  if (a.depth) a.depth[p] = o.d0;
  if (a.sem) a.sem[p] = (uint16_t)o.s;
  if (a.rgb) {
    a.rgb[3 * p] = (uint8_t)o.r;
    a.rgb[3 * p + 1] = (uint8_t)o.g;
    a.rgb[3 * p + 2] = (uint8_t)o.b;
  }
}

}  // namespace nvk
