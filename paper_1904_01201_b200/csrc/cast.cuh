// cast.cuh -- column casts (raycast_grid + row classification -> column records) and
// the operator-level raycast / disc / clearance kernels.
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
// COH: the agent state was written by a still-running grid (programmatic
// dependent launch), so it is read through L2 (ld.global.cg) rather than the
// non-coherent path.
// (env e's pose px, py, cos c, sin s, heading h: h only read for column 0)
__device__ __forceinline__ void cast_column_at(const EnvView &ev, const SceneView &sc,
                                               const CamView &cam, int e, int j, const RecOut &ro,
                                               double t_max, double *gps, double *compass,
                                               double px, double py, double c, double s,
                                               double heading) {
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
    if (compass) compass[e] = nvx::wrap_angle(sub(heading, ev.oh[e]));
  }
}

template <bool COH>
__device__ __forceinline__ void cast_column(const EnvView &ev, const SceneView &sc,
                                            const CamView &cam, int e, int j, const RecOut &ro,
                                            double t_max, double *gps, double *compass) {
  double px, py, c, s, h = 0.0;
  if (COH) {
    px = __ldcg(ev.x + e); py = __ldcg(ev.y + e); c = __ldcg(ev.ch + e); s = __ldcg(ev.sh + e);
    if (j == 0) h = __ldcg(ev.h + e);
  } else {
    px = ev.x[e]; py = ev.y[e]; c = ev.ch[e]; s = ev.sh[e];
    if (j == 0) h = ev.h[e];
  }
  cast_column_at(ev, sc, cam, e, j, ro, t_max, gps, compass, px, py, c, s, h);
}

__device__ __forceinline__ double ld_relaxed_f64(const double *p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool is_pose_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == NV_POSE_SENTINEL;
}
// Release-mode cast side with pose records: reload the env's record from L2
// until no field is the sentinel (each field is written once per step, after
// the reset, so five non-sentinel fields are all this step's); a wait longer
// than 200 ms raises `fault` and casts whatever was read.
__device__ __forceinline__ void load_pose_record(const double *rec, unsigned *fault, double &px,
                                                 double &py, double &c, double &s, double &h) {
  unsigned long long t0 = 0;
  for (;;) {
    px = ld_relaxed_f64(rec);
    py = ld_relaxed_f64(rec + 1);
    c = ld_relaxed_f64(rec + 2);
    s = ld_relaxed_f64(rec + 3);
    h = ld_relaxed_f64(rec + 4);
    if (!(is_pose_sentinel(px) | is_pose_sentinel(py) | is_pose_sentinel(c) | is_pose_sentinel(s) |
          is_pose_sentinel(h)))
      return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (!t0) {
      t0 = t;
    } else if (t - t0 > 200000000ull || *reinterpret_cast<volatile unsigned *>(fault)) {
      atomicExch(fault, 1u);
      return;
    }
    __nanosleep(64);
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
          const float4 e = __ldg(sc.entm + q);  // side test as in test_cell_f32
          const float sm = fmaf(dxf, e.y, -(dyf * e.x)) - cp;
          const float sh = fmaf(dxf, e.w, -(dyf * e.z));
          if (fabsf(sm) > fabsf(sh) + E) continue;
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

// Per-env release to the frame writer: after a block's records are written
// (the caller's __syncthreads), thread 0 adds the block's column count of
// each env it covers to done[env] with a release reduction (the barrier
// orders the block's record stores before it; release, not a sequentially
// consistent fence, is what the writer's acquire pairs with).  Blocks cover rays
// [blk * rpb, (blk + 1) * rpb) of the env-major ray order.
__device__ __forceinline__ void release_envs(unsigned *done, long long blk, int rpb, int W,
                                             long long n_rays) {
  const long long r0 = blk * rpb, r1 = min(n_rays, r0 + rpb) - 1;
  if (r0 > r1) return;
#ifndef NV_REL_MODE
#define NV_REL_MODE 1  // 1 red.release.gpu (MEMBAR.ALL), 0 fence.sc + atomicAdd (MEMBAR.SC: C3 +0.9 us/step), 2 no fence (timing-only study)
#endif
  if (NV_REL_MODE == 0) __threadfence();
  for (long long e = r0 / W; e <= r1 / W; ++e) {
    const long long lo = max(r0, e * W), hi = min(r1, (e + 1) * W - 1);
    if (NV_REL_MODE == 1)
      asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(done + e),
                   "r"((unsigned)(hi - lo + 1)) : "memory");
    else
      atomicAdd(done + e, (unsigned)(hi - lo + 1));
  }
}

#ifndef NV_STUDY_NOWAIT
#define NV_STUDY_NOWAIT 0  // timing-only studies: 1 the cast does not wait for the agent step, 2 one acquire without spinning
#endif
// Release-mode side of the agent -> cast overlap: lane 0 of each warp
// acquires the ready flags of the envs of the warp's rays [r0, r1] and the
// warp proceeds (no CTA barrier, no atomics: the flags of this record half
// are reset by the frame writer once it has consumed the env, see
// wait_env_cast).  A wait longer than 200 ms raises `fault` and stops waiting,
// so a broken launch can never hang the GPU.
__device__ __forceinline__ void warp_wait_envs_ready(const unsigned *ready, unsigned *fault,
                                                     unsigned r0, unsigned r1, unsigned W) {
  if ((threadIdx.x & 31) == 0) {
    for (unsigned e = r0 / W; e <= r1 / W; ++e) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + e) : "memory");
      if (v || NV_STUDY_NOWAIT == 2) continue;  // (2: timing-only, one acquire, no spin)
      unsigned long long t0, t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      do {
        __nanosleep(64);
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + e) : "memory");
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (!v && (t - t0 > 200000000ull || *reinterpret_cast<volatile unsigned *>(fault))) {
          atomicExch(fault, 1u);
          v = 1;
        }
      } while (!v);
    }
  }
  __syncwarp();
}

// With `ready`: a programmatic dependent of k_agent_step, waiting per env.
// `trigger`: a frame writer follows as this grid's programmatic dependent (it
// may launch once every cast CTA runs); without one the grid does not trigger,
// so a following agent step (a programmatic dependent of whatever precedes it)
// cannot start while the casts still read the env state.
#ifndef NV_CASTW_MINB
#define NV_CASTW_MINB 8  // min resident CTAs/SM for the warp-per-ray cast (register cap <= 64; C2 31.1 -> 28.9 us/step)
#endif
__global__ void __launch_bounds__(128, NV_CASTW_MINB) k_column_cast_warp(EnvView ev, SceneView sc, CamView cam,
                                                          RecOut ro, double t_max, double *gps,
                                                          double *compass, unsigned *ready,
                                                          unsigned *arrive, unsigned *rfault,
                                                          const unsigned *order, unsigned *cost,
                                                          unsigned *done, bool trigger,
                                                          const double *posrec) {
  (void)rfault;  // the warp cast always resets its ready flags itself (arrive)
  (void)posrec;  // and never runs in release mode
  // `order` / `cost`: longest-first block order, as in k_column_cast
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // see k_column_cast
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
  if (order || done) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (order) cost[blk] = (unsigned)min(clock64() - t0, 0xffffffffLL);
      if (done) release_envs(done, blk, (int)(blockDim.x >> 5), cam.W, total);
    }
  }
  grid_completes_after_predecessor();  // completes after the agent step
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
                                                     unsigned *rfault, const unsigned *order,
                                                     unsigned *cost, unsigned *done,
                                                     bool trigger, const double *posrec) {
  // With `order`: CTA b casts ray block order[b] (blocks the previous step
  // found slowest first -- longest-processing-time order, so the grid's last
  // wave is made of short blocks) and records its block's duration in
  // cost[] for the next step's ordering.  The rays, their results and the
  // visit order inside each ray are unchanged.
  // the frame writer (a programmatic dependent) may launch once every cast
  // CTA is running: its set-up then overlaps the cast's tail
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long blk = order ? (long long)__ldg(order + blockIdx.x) : (long long)blockIdx.x;
  long long t0 = 0;
  if (order && threadIdx.x == 0) t0 = clock64();
  const long long total = (long long)ev.n * cam.W;
  const long long g = blk * (long long)blockDim.x + threadIdx.x;
  if (ready && NV_STUDY_NOWAIT != 1) {
    if (arrive) {
      wait_envs_ready(ready, arrive, cam.W, total, 0, blk);
    } else {  // release mode: per warp, flags reset by the writer
      const long long w0 = blk * (long long)blockDim.x + (threadIdx.x & ~31u);
      if (w0 < total)
        warp_wait_envs_ready(ready, rfault, (unsigned)w0, (unsigned)min(total - 1, w0 + 31),
                             (unsigned)cam.W);
    }
  }
  if (g < total) {
    // 32-bit division whenever the ray count fits (always, in practice)
    const int e = total <= 0xffffffffLL ? (int)((unsigned)g / (unsigned)cam.W) : (int)(g / cam.W);
    const int j = (int)(g - (long long)e * cam.W);
    if (posrec) {
      double px, py, c, s, h;
      if (NV_STUDY_NOWAIT == 1) {  // timing-only: the current state, no wait
        px = __ldcg(ev.x + e); py = __ldcg(ev.y + e); c = __ldcg(ev.ch + e); s = __ldcg(ev.sh + e);
        h = __ldcg(ev.h + e);
      } else {
        load_pose_record(posrec + (size_t)e * NV_POSE_STRIDE, rfault, px, py, c, s, h);
      }
      cast_column_at(ev, sc, cam, e, j, ro, t_max, gps, compass, px, py, c, s, h);
    } else if (ready)
      cast_column<true>(ev, sc, cam, e, j, ro, t_max, gps, compass);
    else
      cast_column<false>(ev, sc, cam, e, j, ro, t_max, gps, compass);
  }
  if (order || done) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (order) cost[blk] = (unsigned)min(clock64() - t0, 0xffffffffLL);
      if (done) release_envs(done, blk, (int)blockDim.x, cam.W, total);
    }
  }
  grid_completes_after_predecessor();  // completes after the agent step
}

// every field of n pose records -> the sentinel (NV_POSE_SENTINEL)
__global__ void k_pose_init(unsigned long long *rec, long long n_words) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n_words) rec[i] = NV_POSE_SENTINEL;
}

__global__ void k_lpt_init(unsigned *order, unsigned *cost, unsigned n) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    order[i] = i;
    cost[i] = 0;
  }
}

// Longest-first order of the cast's ray blocks from their last durations:
// a counting sort over 256 log-spaced buckets (descending), run on a side
// stream beside the frame writer.  The next step's agent step depends on it,
// so it must fit an SM next to a writer CTA and end well inside the writer:
// NV_ORDER_WARPS warps of <= 32 registers (one warp per SM sub-partition
// fits beside the writer's 18 warps x 96 registers).  Equal-bucket blocks
// come out in any order (the order only schedules; results do not depend
// on it).
#ifndef NV_ORDER_WARPS
#define NV_ORDER_WARPS 4
#endif
__global__ void __launch_bounds__(32 * NV_ORDER_WARPS, 64 / NV_ORDER_WARPS)
    k_cast_order(const unsigned *cost, unsigned *order, int nblk) {
  __shared__ unsigned hist[256];
  __shared__ unsigned wmax[NV_ORDER_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int T = 32 * NV_ORDER_WARPS;
  unsigned mx = 0;
  for (int k = tid; k < 256; k += T) hist[k] = 0;
  for (int b = tid; b < nblk; b += T) mx = max(mx, cost[b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) wmax[warp] = mx;
  __syncthreads();
  mx = 0;
#pragma unroll
  for (int w = 0; w < NV_ORDER_WARPS; ++w) mx = max(mx, wmax[w]);
  const int top = 32 - __clz(mx | 1u);          // bits of the largest cost
  const int shift = top > 8 ? top - 8 : 0;
  auto bucket = [&](unsigned c) { return 255 - (int)min(255u, c >> shift); };  // slow first
  for (int b = tid; b < nblk; b += T) atomicAdd(&hist[bucket(cost[b])], 1u);
  __syncthreads();
  if (warp == 0) {
    // exclusive prefix over the 256 buckets: 8 consecutive buckets per lane
    unsigned v[8], run = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = run;
      run += hist[lane * 8 + k];
    }
    unsigned incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const unsigned base = incl - run;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) hist[lane * 8 + k] = base + v[k];
  }
  __syncthreads();
  for (int b = tid; b < nblk; b += T) order[atomicAdd(&hist[bucket(cost[b])], 1u)] = (unsigned)b;
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
