// mega.cuh -- the persistent step+render megakernel (opt-in nv_set_fused).
#pragma once

#include "fill.cuh"

namespace nvk {

using nvx::add;
using nvx::div;
using nvx::mul;
using nvx::sub;

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


}  // namespace nvk
