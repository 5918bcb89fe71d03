// cast.cuh -- column casts (raycast_grid + row classification -> column records), the
// binned cast and the operator-level raycast / disc / clearance kernels.
#pragma once

#include "agent.cuh"

namespace nvk {

using nvx::add;
using nvx::div;
using nvx::mul;
using nvx::sub;

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

// One warp per (env, column): the latency-bound small-batch cast.  COH: the
// agent state was written by a still-running grid (programmatic dependent
// launch), so it is read through L2 (ld.global.cg).
template <bool COH = false>
__device__ __forceinline__ void k_column_cast_warp_body(const EnvView &ev, const SceneView &sc,
                                                        const CamView &cam, const RecOut &ro,
                                                        double t_max, double *gps,
                                                        double *compass, int e, int j) {
  const int lane = threadIdx.x & 31;
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
    if (compass) compass[e] = nvx::wrap_angle(sub(COH ? __ldcg(ev.h + e) : ev.h[e], ev.oh[e]));
  }
}

// With `ready`: a programmatic dependent of k_agent_step, waiting per env.
#ifndef NV_CASTW_MINB
#define NV_CASTW_MINB 8  // min resident CTAs/SM for the warp-per-ray cast (register cap <= 64; C2 31.1 -> 28.9 us/step)
#endif
__global__ void __launch_bounds__(128, NV_CASTW_MINB) k_column_cast_warp(EnvView ev, SceneView sc, CamView cam,
                                                          RecOut ro, double t_max, double *gps,
                                                          double *compass, unsigned *ready,
                                                          unsigned *arrive, const unsigned *order,
                                                          unsigned *cost) {
  // `order` / `cost`: longest-first block order, as in k_column_cast
  const long long blk = order ? (long long)__ldg(order + blockIdx.x) : (long long)blockIdx.x;
  long long t0 = 0;
  if (order && threadIdx.x == 0) t0 = clock64();
  const long long total = (long long)ev.n * cam.W;
  if (ready) wait_envs_ready(ready, arrive, cam.W, total, (int)(blockDim.x >> 5), blk);
  const long long g = (blk * (long long)blockDim.x + threadIdx.x) >> 5;
  if (g < total) {
    const int e = (int)(g / cam.W);
    const int j = (int)(g - (long long)e * cam.W);
    if (ready)
      k_column_cast_warp_body<true>(ev, sc, cam, ro, t_max, gps, compass, e, j);
    else
      k_column_cast_warp_body<false>(ev, sc, cam, ro, t_max, gps, compass, e, j);
  }
  if (order) {
    __syncthreads();
    if (threadIdx.x == 0) cost[blk] = (unsigned)min(clock64() - t0, 0xffffffffLL);
  }
}

// ---- ray-pool cast: lanes refill from a per-warp pool of rays --------------
//
// k_column_cast_pool: each warp owns a pool of consecutive rays (env-major,
// column-minor) and walks them as one DDA cell per loop iteration per lane;
// a lane whose ray finished writes its column record and takes the next ray
// of the pool in the same iteration, so lanes do not idle behind the warp's
// longest ray (the per-ray DDA leaves half the lanes idle on average).  The
// visit order and early-out of every ray are raycast_grid's.
struct RayState {
  double px, py, dx, dy, tnx, tny, tdx, tdy, best_t;
  long long cx, cy;
  int stepx, stepy, best_i, e, j;
  int4 rec;
  float dxf, dyf, sd;
};

// _column_directions + the DDA prologue of raycast_grid; false when the ray
// is already finished (NaN input: the reference would spin, the DDA returns
// the empty hit).
__device__ __forceinline__ bool ray_begin(const EnvView &ev, const SceneView &sc,
                                          const CamView &cam, int e, int j, RayState &r) {
  r.e = e;
  r.j = j;
  r.px = ev.x[e];
  r.py = ev.y[e];
  const double c = ev.ch[e], s = ev.sh[e];
  const double u = __ldg(cam.u + j);
  r.dx = add(c, mul(u, s));
  r.dy = add(s, mul(u, -c));
  r.best_t = NV_INF;
  r.best_i = -1;
  if (isnan(r.px) || isnan(r.py) || isnan(r.dx) || isnan(r.dy)) return false;
  const double cell = 1.0;
  r.cx = (long long)floor(sub(r.px, sc.x0));
  r.cy = (long long)floor(sub(r.py, sc.y0));
  r.stepx = r.dx > 0.0 ? 1 : -1;
  r.stepy = r.dy > 0.0 ? 1 : -1;
  if (r.dx != 0.0) {
    const double nbx = add(sc.x0, mul((double)(r.cx + (r.dx > 0.0 ? 1 : 0)), cell));
    r.tnx = div(sub(nbx, r.px), r.dx);
    r.tdx = fabs(div(cell, r.dx));
  } else {
    r.tnx = NV_INF;
    r.tdx = NV_INF;
  }
  if (r.dy != 0.0) {
    const double nby = add(sc.y0, mul((double)(r.cy + (r.dy > 0.0 ? 1 : 0)), cell));
    r.tny = div(sub(nby, r.py), r.dy);
    r.tdy = fabs(div(cell, r.dy));
  } else {
    r.tny = NV_INF;
    r.tdy = NV_INF;
  }
  r.dxf = (float)r.dx;
  r.dyf = (float)r.dy;
  r.sd = (fabsf(r.dxf) + fabsf(r.dyf)) * (1.0f + 0x1p-20f);
  r.rec = make_int4(0, 0, 0, 0);
  if (0 <= r.cx && r.cx < sc.gnx && 0 <= r.cy && r.cy < sc.gny)
    r.rec = __ldg(sc.cells + (r.cy * sc.gnx + r.cx));
  return true;
}

// One iteration of raycast_grid's loop (one cell); true when the ray is done.
__device__ __forceinline__ bool ray_cell(const SceneView &sc, RayState &r, double t_max) {
  const long long gnx = sc.gnx, gny = sc.gny;
  const double t_exit = r.tnx < r.tny ? r.tnx : r.tny;
  long long ncx = r.cx, ncy = r.cy;
  double ntnx = r.tnx, ntny = r.tny;
  if (r.tnx < r.tny) {
    ncx += r.stepx;
    ntnx = add(r.tnx, r.tdx);
  } else {
    ncy += r.stepy;
    ntny = add(r.tny, r.tdy);
  }
  int4 nrec = make_int4(0, 0, 0, 0);
  if (!(t_exit > t_max) && 0 <= ncx && ncx < gnx && 0 <= ncy && ncy < gny)
    nrec = __ldg(sc.cells + (ncy * gnx + ncx));
  cell_tests(sc, r.cx, r.cy, r.rec, r.px, r.py, r.dx, r.dy, r.dxf, r.dyf, r.sd, r.dxf >= 0.0f,
             r.dyf >= 0.0f, r.best_t, r.best_i);
  if (r.best_t <= t_exit || t_exit > t_max) return true;
  r.cx = ncx;
  r.cy = ncy;
  r.tnx = ntnx;
  r.tny = ntny;
  r.rec = nrec;
  if (r.cx < 0 || r.cx >= gnx || r.cy < 0 || r.cy >= gny) {
    const bool out_x = (r.cx < 0 && r.dx <= 0.0) || (r.cx >= gnx && r.dx >= 0.0);
    const bool out_y = (r.cy < 0 && r.dy <= 0.0) || (r.cy >= gny && r.dy >= 0.0);
    if (out_x || out_y) return true;
  }
  return false;
}

__device__ __forceinline__ void ray_finish(const EnvView &ev, const SceneView &sc,
                                           const CamView &cam, const RecOut &ro,
                                           const RayState &r, double *gps, double *compass) {
  ColRec rc;
  column_epilogue(sc, cam, r.best_t, r.best_i, r.dx, r.dy, rc);
  put_rec(ro, r.e, r.j, rc);
  if (r.j == 0 && (gps || compass)) {
    const int e = r.e;
    const double ddx = sub(r.px, ev.ox[e]), ddy = sub(r.py, ev.oy[e]);
    const double fc = ev.fc[e], fs = ev.fs[e];
    if (gps) {
      gps[2 * e] = sub(mul(fc, ddx), mul(fs, ddy));
      gps[2 * e + 1] = add(mul(fs, ddx), mul(fc, ddy));
    }
    if (compass) compass[e] = nvx::wrap_angle(sub(ev.h[e], ev.oh[e]));
  }
}

__global__ void __launch_bounds__(128) k_column_cast_pool(EnvView ev, SceneView sc, CamView cam,
                                                          RecOut ro, double t_max, double *gps,
                                                          double *compass, int pool) {
  const int lane = threadIdx.x & 31;
  const long long n_rays = (long long)ev.n * cam.W;
  const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long lo = wid * pool;
  if (lo >= n_rays) return;
  const long long hi = min(n_rays, lo + pool);
  long long next = lo;  // warp-uniform
  RayState r;
  bool active = false;
  for (;;) {
    // refill idle lanes from the pool (lane order keeps rays adjacent)
    const unsigned idle = __ballot_sync(0xffffffffu, !active);
    const long long avail = hi - next;
    if (!active) {
      const int rank = __popc(idle & ((1u << lane) - 1u));
      if (rank < avail) {
        const long long g = next + rank;
        const int e = (int)(g / cam.W);
        const int j = (int)(g - (long long)e * cam.W);
        active = ray_begin(ev, sc, cam, e, j, r);
        if (!active) ray_finish(ev, sc, cam, ro, r, gps, compass);  // NaN pose: empty hit
      }
    }
    next += min((long long)__popc(idle), avail);
    if (!__any_sync(0xffffffffu, active)) {
      if (next >= hi) break;
      continue;
    }
    if (active && ray_cell(sc, r, t_max)) {
      ray_finish(ev, sc, cam, ro, r, gps, compass);
      active = false;
    }
  }
}

// One thread per (env, column).  With `ready`: launched as a programmatic
// dependent of k_agent_step; waits per env instead of for the whole step.
#ifndef NV_CAST_KMINB
#define NV_CAST_KMINB 7  // min resident CTAs/SM for the thread-per-ray cast (register cap: <= 72; A/B with the longest-first order: 5 / 6 / 7 / 8 -> 117.4 / 115.9 / 115.0 / 117.3 us per C3 step)
#endif
__global__ void __launch_bounds__(128, NV_CAST_KMINB) k_column_cast(EnvView ev, SceneView sc, CamView cam,
                                                     RecOut ro, double t_max,
                                                     double *gps, double *compass,
                                                     unsigned *ready, unsigned *arrive,
                                                     const unsigned *order, unsigned *cost) {
  // With `order`: CTA b casts ray block order[b] (blocks the previous step
  // found slowest first -- longest-processing-time order, so the grid's last
  // wave is made of short blocks) and records its block's duration in
  // cost[] for the next step's ordering.  The rays, their results and the
  // visit order inside each ray are unchanged.
  const long long blk = order ? (long long)__ldg(order + blockIdx.x) : (long long)blockIdx.x;
  long long t0 = 0;
  if (order && threadIdx.x == 0) t0 = clock64();
  const long long total = (long long)ev.n * cam.W;
  if (ready) wait_envs_ready(ready, arrive, cam.W, total, 0, blk);
  const long long g = blk * (long long)blockDim.x + threadIdx.x;
  if (g < total) {
    // 32-bit division whenever the ray count fits (always, in practice)
    const int e = total <= 0xffffffffLL ? (int)((unsigned)g / (unsigned)cam.W) : (int)(g / cam.W);
    const int j = (int)(g - (long long)e * cam.W);
    if (ready)
      cast_column<true>(ev, sc, cam, e, j, ro, t_max, gps, compass);
    else
      cast_column<false>(ev, sc, cam, e, j, ro, t_max, gps, compass);
  }
  if (order) {
    __syncthreads();
    if (threadIdx.x == 0) cost[blk] = (unsigned)min(clock64() - t0, 0xffffffffLL);
  }
}

__global__ void k_lpt_init(unsigned *order, unsigned *cost, unsigned n) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    order[i] = i;
    cost[i] = 0;
  }
}

// Longest-first order of the cast's ray blocks from their last durations:
// a one-CTA counting sort over 256 log-spaced buckets (descending), run on
// a side stream beside the frame writer.
__global__ void __launch_bounds__(1024) k_cast_order(const unsigned *cost, unsigned *order,
                                                     int nblk) {
  __shared__ unsigned hist[256], base[256], mx;
  const int t = threadIdx.x;
  if (t == 0) mx = 0;
  for (int k = t; k < 256; k += blockDim.x) hist[k] = 0;
  __syncthreads();
  for (int b = t; b < nblk; b += blockDim.x) atomicMax(&mx, cost[b]);
  __syncthreads();
  const int top = 32 - __clz(mx | 1u);          // bits of the largest cost
  const int shift = top > 8 ? top - 8 : 0;
  auto bucket = [&](unsigned c) { return 255 - (int)min(255u, c >> shift); };  // slow first
  for (int b = t; b < nblk; b += blockDim.x) atomicAdd(&hist[bucket(cost[b])], 1u);
  __syncthreads();
  // exclusive prefix over the 256 buckets: 8 warps scan 32 each, then offsets
  __shared__ unsigned wsum[8];
  if (t < 256) {
    const int lane = t & 31, w = t >> 5;
    unsigned v = hist[t];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) wsum[w] = v;
    base[t] = v - hist[t];
  }
  __syncthreads();
  if (t < 256) {
    unsigned off = 0;
    for (int w = 0; w < (t >> 5); ++w) off += wsum[w];
    base[t] += off;
  }
  __syncthreads();
  for (int b = t; b < nblk; b += blockDim.x) order[atomicAdd(&base[bucket(cost[b])], 1u)] = (unsigned)b;
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


}  // namespace nvk
