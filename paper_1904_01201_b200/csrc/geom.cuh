// geom.cuh -- shared FP64 geometry of the navsim hot path: the exact segment
// test, raycast_grid's DDA, disc_cast and
// min_seg_distance (see kernels.cuh for the kernel overview).
//
// Exactness: every FP64 operation that decides coverage, semantics, depth or
// pose uses the nvx:: _rn helpers (no FMA contraction), replicating the
// reference's operation order.
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

// End of a grid launched as a programmatic dependent: the grid must not
// complete before its predecessor (so stream order holds for whatever
// follows).  One CTA waiting is enough for that -- a grid completes when its
// last CTA exits -- so only the last CTA in launch order waits and every
// other CTA frees its SM slot at once instead of idling until the previous
// frame writer ends (NV_GDW_ALL: every CTA waits, the round-2 baseline).
#ifndef NV_GDW_ALL
#define NV_GDW_ALL 0
#endif
__device__ __forceinline__ void grid_completes_after_predecessor() {
  if (NV_GDW_ALL || blockIdx.x == gridDim.x - 1) asm volatile("griddepcontrol.wait;" ::: "memory");
}

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

// The reference's exact path for a prefilter survivor.  `0 <= RN(rn/den) <= 1`
// is decided without the division: seg_pre already rejected sign(rn) !=
// sign(den) (so RN(rn/den) >= 0) and |rn| > |den| (1 + 1e-12), and for
// |den| <= |rn| <= 2 |den| the difference |rn| - |den| is exact (Sterbenz):
// RN(q) <= 1 iff q <= 1 + 2^-53 (the midpoint rounds to even, 1.0) iff
// |rn| - |den| <= |den| 2^-53 (an exact power-of-two scaling).
#ifndef NV_R_DIVFREE
#define NV_R_DIVFREE 1
#endif
__device__ __forceinline__ void seg_exact(double den, double tn, double rn, int i,
                                          double &best_t, int &best_i) {
  double t = div(tn, den);
  if (t < 0.0 || t > best_t) return;
#if NV_R_DIVFREE
  const double ar = fabs(rn), ad = fabs(den);
  const bool r_ok = ar <= ad || sub(ar, ad) <= ad * 0x1p-53;
#else
  const double r = div(rn, den);
  const bool r_ok = 0.0 <= r && r <= 1.0;
#endif
  if (r_ok) {
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

// FP32 prefilter for one cell of the DDA (side test).  The ray's line
// crosses segment [a, b] iff a and b are not strictly on the same side:
// with s_a = d x (a - p) and s_b = d x (b - p), the reference's
// r = rn/den = s_a / (s_a - s_b), so both s_a, s_b > 0 (or both < 0) means
// r < 0 or r > 1 (or den == 0) and the reference skips the segment.
// Entries are stored in f32 relative to the cell anchor (X0c, Y0c) =
// (x0 + cx, y0 + cy) as midpoint m and half-vector h (a = m - h, b = m + h,
// each within 2^-23 A of the stored f32 endpoints); the ray origin is rebased
// to the same anchor in f64 and rounded once.  Then s_a, s_b = s_m -+ s_h with
// s_m = d x (m - p), s_h = d x h, and both lie strictly on one side iff
// |s_m| > |s_h|: the entry is skipped when |s_m| > |s_h| + E.
// E = 2^-18 |d|_1 (A + |p_rel|_1) bounds the f32 error of these sums
// (conversions, products, sums, the midpoint form; > 4x over the worst case)
// and the reference's own f64 rounding, so a segment is skipped only when it
// is certain that the reference skips it.  Survivors -- the segments the
// ray's line actually crosses, plus a hairline margin -- take the exact FP64
// test, so the result is bit-identical to the unfiltered DDA.
#define NV_K32 0x1p-18f

struct CellF {
  float cp, E;  // d x p_rel, error bound
  float adx, ady;  // |d| components (box half-extent term)
};

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
    for (int k = 0; k < NB; ++k) e[k] = __ldg(sc.entm + (unsigned)min(q + k, q1 - 1));
    unsigned keep = 0;
#pragma unroll
    for (int k = 0; k < NB; ++k) {
      const float sm = fmaf(dxf, e[k].y, -(dyf * e[k].x)) - cf.cp;
      const float sh = fmaf(dxf, e[k].w, -(dyf * e[k].z));
      const bool skip = fabsf(sm) > fabsf(sh) + cf.E;
      keep |= (skip ? 0u : 1u) << k;
    }
    while (keep) {
      const int k = __ffs(keep) - 1;
      keep &= keep - 1;
      const unsigned qq = (unsigned)min(q + k, q1 - 1);
      const double2 *p2 = reinterpret_cast<const double2 *>(sc.ent + qq);
      const double2 a2 = __ldg(p2), e2 = __ldg(p2 + 1);
      double den, tn, rn;
      if (seg_pre(px, py, dx, dy, a2.x, a2.y, e2.x, e2.y, best_t, den, tn, rn))
        seg_exact(den, tn, rn, __ldg(sc.items + qq), best_t, best_i);
    }
  }
}

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
// The tests of one DDA cell (record `rec`) for a ray: run boxes, f32 side
// tests, exact FP64 tests of the survivors; updates (best_t, best_i).
template <typename IT>
__device__ __forceinline__ void cell_tests(const SceneView &sc, IT cx, IT cy,
                                           const int4 &rec, double px, double py, double dx,
                                           double dy, float dxf, float dyf, float sd,
                                           bool pos_dx, bool pos_dy, double &best_t,
                                           int &best_i) {
  if (rec.y > rec.x) {
    const double X0 = add(sc.x0, (double)cx), Y0 = add(sc.y0, (double)cy);
    const float pxr = (float)sub(px, X0), pyr = (float)sub(py, Y0);
    CellF cf;
    cf.cp = fmaf(dxf, pyr, -(dyf * pxr));
    cf.E = NV_K32 * sd * (__int_as_float(rec.z) + fabsf(pxr) + fabsf(pyr) + 1e-30f);
    cf.adx = fabsf(dxf);
    cf.ady = fabsf(dyf);
#if NV_CAST_CHUNKS
    // s(x, y) = d x ((x, y) - p) is linear, so over a run's box (centre c,
    // half-extents h) it spans s(c) +- (|dx| h_y + |dy| h_x); a run whose box
    // lies beyond +-E on one side holds no entry the per-entry side test
    // would keep.  The boxes of up to NV_CAST_NCB runs are loaded together
    // (one memory round trip per cell in the common case); a passing run's
    // f64 entries are prefetched into L1 before its f32 side tests, so the
    // exact tests of its survivors hit L1.
    const int nch = (rec.y - rec.x + NV_CHUNK - 1) / NV_CHUNK;
    for (int c0 = 0; c0 < nch; c0 += NV_CAST_NCB) {
      float4 bb[NV_CAST_NCB];
#pragma unroll
      for (int k = 0; k < NV_CAST_NCB; ++k)
        bb[k] = __ldg(sc.chunks + (unsigned)(rec.w + min(c0 + k, nch - 1)));
      unsigned pass = 0;
#pragma unroll
      for (int k = 0; k < NV_CAST_NCB; ++k) {
        const float4 b = bb[k];
        const float sc_ = fmaf(dxf, b.y, -(dyf * b.x)) - cf.cp;
        const float hr = fmaf(cf.adx, b.w, cf.ady * b.z);
        const bool ok = c0 + k < nch && !(fabsf(sc_) > hr + cf.E);
        pass |= (ok ? 1u : 0u) << k;
      }
      for (unsigned m = pass; m; m &= m - 1) {  // prefetch first, then test
        const unsigned q = (unsigned)(rec.x + (c0 + __ffs(m) - 1) * NV_CHUNK);
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
}

// raycast_grid (_kernels.py:51-120), one ray, exact replica of the DDA.
// The walk is software-pipelined: the next cell's record {q0, q1, bound} is
// loaded (one 16-byte load) before the current cell's entries are tested, so
// the cell-to-cell latency overlaps the tests; the visit order and the
// early-out are the reference's.  IT: the cell-coordinate type (32-bit: the
// start cell lies within +-2^30 cells of the grid origin, see ray_grid).
template <typename IT>
__device__ __forceinline__ void ray_grid_walk(const SceneView &sc, double px, double py,
                                              double dx, double dy, double t_max, IT cx, IT cy,
                                              double &out_t, int &out_i) {
  const double cell = 1.0;
  double best_t = NV_INF;
  int best_i = -1;
  const int stepx = dx > 0.0 ? 1 : -1;
  const int stepy = dy > 0.0 ? 1 : -1;
  double tnx, tdx, tny, tdy;
  // |cell / d| = |RN(1 / d)|: the correctly rounded reciprocal is the same value
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
  const IT gnx = sc.gnx, gny = sc.gny;
  const float dxf = (float)dx, dyf = (float)dy;
  const float sd = (fabsf(dxf) + fabsf(dyf)) * (1.0f + 0x1p-20f);
  const bool pos_dx = dxf >= 0.0f, pos_dy = dyf >= 0.0f;
  auto inb = [&](IT x, IT y) { return 0 <= x && x < gnx && 0 <= y && y < gny; };
  auto cell_rec = [&](IT x, IT y) {
    return __ldg(sc.cells + (unsigned)((int)y * sc.gnx + (int)x));  // in the grid: < 2^31
  };
  int4 rec = make_int4(0, 0, 0, 0);
  if (inb(cx, cy)) rec = cell_rec(cx, cy);
  for (int guard = 0; guard < (1 << 24); ++guard) {
    const double t_exit = tnx < tny ? tnx : tny;
    // the cell after this one (the reference advances to it unless it stops)
    IT ncx = cx, ncy = cy;
    double ntnx = tnx, ntny = tny;
    if (tnx < tny) {
      ncx += stepx;
      ntnx = add(tnx, tdx);
    } else {
      ncy += stepy;
      ntny = add(tny, tdy);
    }
    int4 nrec = make_int4(0, 0, 0, 0);
    if (!(t_exit > t_max) && inb(ncx, ncy)) nrec = cell_rec(ncx, ncy);
    cell_tests<IT>(sc, cx, cy, rec, px, py, dx, dy, dxf, dyf, sd, pos_dx, pos_dy, best_t, best_i);
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

__device__ __forceinline__ void ray_grid(const SceneView &sc, double px, double py,
                                         double dx, double dy, double t_max,
                                         double &out_t, int &out_i) {
  if (isnan(px) || isnan(py) || isnan(dx) || isnan(dy)) {  // reference would spin
    out_t = NV_INF;
    out_i = -1;
    return;
  }
  // (p - x0) / cell with cell = 1.0 is exact without the division
  const double fx = floor(sub(px, sc.x0)), fy = floor(sub(py, sc.y0));
  if (!(fabs(fx) < 0x1p30 && fabs(fy) < 0x1p30)) {
    // >= 2^30 cells from the grid origin: the walk's 2^24-step guard ends it
    // long before it could reach a grid cell (grids are < 2^31 cells in all)
    out_t = NV_INF;
    out_i = -1;
    return;
  }
  ray_grid_walk<int>(sc, px, py, dx, dy, t_max, (int)fx, (int)fy, out_t, out_i);
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
// the reference's order with its strict `<`; the segment's seg_len and unit
// tangent come from its DiscEntry (the identical values the reference
// recomputes per candidate).  The reference's result is then the
// lexicographic (t, idx) minimum over segments (its scan is ascending in idx
// with strict `<`), which lets the warp scan candidates in any order.
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

}  // namespace nvk
