// agent.cuh -- Simulator.step kinematics (sim.py:83-219): warp-per-env agent step and reset.
#pragma once

#include "geom.cuh"

namespace nvk {

using nvx::add;
using nvx::div;
using nvx::mul;
using nvx::sub;

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
  double h, c, s;  // heading and its cos / sin after the step (valid in lane 0)
};

// Per-env pose records of the release-mode agent -> cast handshake
// (NV_POSE_REC): {x, y, cos h, sin h, h, path, collisions, status} per env
// and record half, 64-byte stride.  The frame writer resets a consumed env's record to the sentinel,
// a signalling-NaN pattern no arithmetic produces; the agent step's lane 0
// writes the new pose (plain 8-byte stores), and a cast lane reloads the
// record from L2 until no field is the sentinel -- one memory round trip
// instead of a flag acquire followed by the pose loads.
#define NV_POSE_SENTINEL 0x7FF0DEAD00000001ull
#define NV_POSE_STRIDE 8
__device__ __forceinline__ double pose_field(double v) {
  // a user-set pose with the sentinel's exact bits becomes a quiet NaN (the
  // cast's result for any NaN pose is the same: no hit)
  return (unsigned long long)__double_as_longlong(v) == NV_POSE_SENTINEL ? __longlong_as_double(0x7FF8000000000000ll) : v;
}

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
  double hn = h0, cn = ch, sn = sh;
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
      hn = h;
      sn = s;
      cn = c;
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
    post->h = hn;
    post->c = cn;
    post->s = sn;
  }
}

// Simulator.step for all envs: one warp per env.  With `ready` (programmatic
// dependent launch of the cast), the dependent grid is released at once and
// each env's pose is published through ready[e] (release) as soon as its warp
// is done, so the casts of finished envs overlap the long agent chains.
#ifndef NV_AGENT_FENCE
#define NV_AGENT_FENCE 0
#endif
#ifndef NV_AGENT_MAXREG
#define NV_AGENT_MAXREG 0  // > 0: register cap of the agent step (room beside a writer CTA)
#endif
#if NV_AGENT_MAXREG > 0
#define NV_AGENT_BOUNDS __maxnreg__(NV_AGENT_MAXREG)
#else
#define NV_AGENT_BOUNDS __launch_bounds__(128)
#endif
__global__ void NV_AGENT_BOUNDS k_agent_step(EnvView ev, SceneView sc, AgentCfg cfg,
                                                    const int8_t *__restrict__ actions,
                                                    uint8_t *collided_out,
                                                    double *disp_out, int32_t *status_out,
                                                    unsigned *ready, double *posrec,
                                                    int wait_first) {
  // wait_first: the preceding frame writer's grid does not fill the GPU, so
  // residency no longer keeps this step (and the casts it releases) behind
  // the previous ones (see "The path" in DESIGN.md): start the step's work,
  // and let the casts launch, only once that writer -- and with it every
  // earlier grid of the chain -- has completed.  The launch itself still
  // overlaps it.
  if (wait_first) asm volatile("griddepcontrol.wait;" ::: "memory");
  // ready: per-env flags, posrec: per-env pose records (see NV_POSE_SENTINEL)
  if (ready || posrec) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int e = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  if (e < ev.n) {
    AgentPost post;
    warp_agent_step(ev, sc, cfg, e, actions[e], collided_out, disp_out, status_out,
                    posrec ? &post : nullptr);
    if (posrec && (threadIdx.x & 31) == 0) {
      double *r = posrec + (size_t)e * NV_POSE_STRIDE;
      r[0] = pose_field(post.x);
      r[1] = pose_field(post.y);
      r[2] = pose_field(post.c);
      r[3] = pose_field(post.s);
      r[4] = pose_field(post.h);
      // the task cast's inputs too: path length, collision count, step status
      // (never the sentinel's bits: a path is a finite length or a plain NaN,
      // counts and statuses are small)
      r[5] = pose_field(post.path);
      r[6] = __longlong_as_double(post.coll);
      r[7] = (double)post.status;
    }
    if (ready && (threadIdx.x & 31) == 0) {
      // lane 0 made every store of the env's step: its release store orders
      // them before the flag (NV_AGENT_FENCE: an extra sequentially consistent
      // fence, the round-2 study baseline)
      if (NV_AGENT_FENCE) __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + e), "r"(1u) : "memory");
    }
  }
  // launched as a programmatic dependent of the previous frame writer: this
  // grid completes only after it, so stream order still holds for what follows
  grid_completes_after_predecessor();
}

// Cast side of the agent->cast overlap: thread 0 of a CTA waits for every env
// the CTA covers (acquire), then the CTA's last arrival per env resets the
// env's flag for the next step.  (CTAs of the cast grid cover rays
// [b*B, (b+1)*B) of the env-major ray order.)
__device__ __forceinline__ void wait_envs_ready(unsigned *ready, unsigned *arrive, int W,
                                                long long n_rays, int rays_per_block = 0,
                                                long long block = -1) {
  const unsigned rpb = rays_per_block > 0 ? (unsigned)rays_per_block : blockDim.x;
  const unsigned blk = block >= 0 ? (unsigned)block : blockIdx.x;
  // 32-bit arithmetic: the ray count of a batch fits (n_envs * W < 2^32)
  const unsigned r0 = blk * rpb;
  const unsigned r1 = (unsigned)min(n_rays, (long long)r0 + rpb) - 1u;
  const unsigned w = (unsigned)W;
  const int e0 = (int)(r0 / w), e1 = (int)(r1 / w);
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
      const unsigned f = (unsigned)e * w / rpb, l = ((unsigned)(e + 1) * w - 1u) / rpb;
      if (atomicAdd(arrive + e, 1u) == l - f) {
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


}  // namespace nvk
