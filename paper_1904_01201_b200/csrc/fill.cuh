// fill.cuh -- frame writers (fill_frame, _kernels.py:128-207): packed-f16 shading, the
// warp-specialised TMA writer, depth noise, the generic per-pixel kernel.
#pragma once

#include "cast.cuh"

namespace nvk {

using nvx::add;
using nvx::div;
using nvx::mul;
using nvx::sub;

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
  int segs_per_row;    // W / (32 * CPL)
  const uint16_t *invh;  // ceil(H/2) x W f16 shading table 1/|(d_j, v_i)|, rows
                         // mirrored (v_{H-1-i} = -v_i); env-independent
  // inverse-depth noise (sensors.apply_inverse_depth_noise, sensors.py:183-205)
  float noise_sigma;     // 0 = off
  float max_range;
  unsigned long long noise_seed, noise_frame;
  long long env_offset;  // global id of env 0 (sharding-invariant streams)
  // per-env release from the column cast (the writer is its programmatic
  // dependent): finished-column counts, band consumers, timeout flag;
  // nullptr = the records are complete when the writer's loads start
  unsigned *done, *consumed, *fault;
  // agent -> cast ready flags of this record half (release mode of
  // nv_step_render): reset by the env's last consumer, like done
  unsigned *ready;
  // or the pose records of this record half (NV_POSE_REC): reset to the
  // sentinel by the env's last consumer
  double *posrec;
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
  // key (frame, global env, row, pair): a pair never straddles two rows, even
  // for odd W
  const unsigned long long key =
      (((a.noise_frame << 20) ^ (unsigned long long)(env + a.env_offset)) * (unsigned long long)a.H +
       (unsigned long long)row) * (unsigned long long)((a.W + 1) >> 1) + (unsigned long long)(col >> 1);
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
#ifndef NV_FRAME_POLICY
#define NV_FRAME_POLICY 0  // L2 policy of frame stores: 0 evict_first, 1 evict_normal, 2 evict_last
#endif
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
#if NV_FRAME_POLICY == 1
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
#elif NV_FRAME_POLICY == 2
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
#endif
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
#ifndef NV_WS_CBUF
#define NV_WS_CBUF 2  // record-plane buffers (prefetch distance CBUF - 1 items)
#endif
#ifndef NV_WS_DEBUG
#define NV_WS_DEBUG 0  // 1: producers skip rendering, 2: no bulk stores (bound studies)
#endif
struct FillWsLayout {  // byte offsets into dynamic shared memory + ring geometry
  int rows, inv, cols, bars, slots;
  int slot_bytes, nslot, slot_rows;
  int nw;            // producer warps (the CTA is nw + 1 warps)
  int bands;         // work items per env frame (row bands of H / bands rows):
                     // balances CTAs when envs per CTA is small
};

#ifndef NV_FILL_MAXREG
#define NV_FILL_MAXREG 0  // > 0: register cap of the ws writer (room for co-resident cast CTAs)
#endif
#if NV_FILL_MAXREG > 0
#define NV_FILL_BOUNDS __maxnreg__(NV_FILL_MAXREG)
#else
#define NV_FILL_BOUNDS __launch_bounds__(REL ? 576 : 544, 1)
#endif
#ifndef NV_STUDY_WAITSTAT
#define NV_STUDY_WAITSTAT 0  // study build: the REL writer's loader accumulates its wait per item rank
#endif
#if NV_STUDY_WAITSTAT
__device__ unsigned long long g_waitstat[16];
#endif
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool env_cast_done(const unsigned *done, int env, int W) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + env) : "memory");
  return v >= (unsigned)W;
}
// Store-warp side of the per-env release: wait (acquire) until env's column
// records are all written, order the later bulk (async-proxy) reads after it,
// and let the env's last consumer reset its count (the counts of the other
// record half serve the next step).  A wait longer than 200 ms raises the
// fault flag and stops waiting, so a broken launch can never hang the GPU.
__device__ __forceinline__ void wait_env_cast(unsigned *done, unsigned *consumed,
                                              unsigned *fault, unsigned *ready, double *posrec,
                                              int env, int W, int bands) {
  if (!env_cast_done(done, env, W)) {
    const unsigned long long t0 = global_ns();
    while (!env_cast_done(done, env, W)) {
      if (*reinterpret_cast<volatile unsigned *>(fault)) break;
      if (global_ns() - t0 > 200000000ull) {
        atomicExch(fault, 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (bands == 1 || atomicAdd(consumed + env, 1u) == (unsigned)(bands - 1)) {
    if (bands > 1) consumed[env] = 0;
    done[env] = 0;
    if (ready) ready[env] = 0;  // every cast CTA of the env is past its wait
    if (posrec) {
      unsigned long long *r =
          reinterpret_cast<unsigned long long *>(posrec + (size_t)env * NV_POSE_STRIDE);
#pragma unroll
      for (int k = 0; k < NV_POSE_STRIDE; ++k) r[k] = NV_POSE_SENTINEL;
    }
  }
}

// REL: per-env release from the cast (FillArgs.done); a separate
// instantiation so the ordinary writer keeps its own code.
template <int CPL, bool TAB, int RPW, bool NOISE, bool BANDED, bool REL>
__global__ void NV_FILL_BOUNDS k_fill_ws(FillArgs a, FillWsLayout L) {
  // the next step's agent step (a programmatic dependent) may start on SMs
  // this grid leaves: it touches none of the writer's inputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) uint8_t smem[];
  using Ln = Lanes<CPL>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = L.nw;  // producer warps (then the store warp, then with REL the loader warp)
  const int W = a.W, H = a.H, S = a.segs_per_row, R = L.slot_rows, NSLOT = L.nslot;
  const RowRec *rows_s = reinterpret_cast<const RowRec *>(smem + L.rows);
  const uint16_t *inv_s = reinterpret_cast<const uint16_t *>(smem + L.inv);
  float4 *cols_s = reinterpret_cast<float4 *>(smem + L.cols);  // [buf][A | B][W]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + L.bars);
  uint64_t *empty = full + NSLOT;
  uint64_t *colfull = empty + NSLOT;
  uint64_t *colempty = colfull + NV_WS_CBUF;
  uint8_t *slots = smem + L.slots;
  const unsigned plane_bytes = (unsigned)W * 16u;
  const bool want_rgb = a.rgb != nullptr, want_d = a.depth != nullptr, want_s = a.sem != nullptr;
  const int off_d = want_rgb ? R * W * 3 : 0;
  const int off_s = off_d + (want_d ? R * W * 4 : 0);
  const int bands = BANDED ? L.bands : 1, band_rows = BANDED ? H / bands : H;
  const int slots_per_item = band_rows / R;
  const int n_items = a.N * bands;
  if (threadIdx.x == 0) {
    for (int k = 0; k < NSLOT; ++k) {
      mbar_init(full + k, (unsigned)nw);
      mbar_init(empty + k, 1);
    }
    for (int k = 0; k < NV_WS_CBUF; ++k) {
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
  auto load_item = [&](int buf, int env) {
    uint64_t *b = colfull + buf;
    mbar_expect_tx(b, 2 * plane_bytes);
    bulk_load(cols_s + (size_t)buf * 2 * W, a.ra + (size_t)env * W, plane_bytes, b);
    bulk_load(cols_s + (size_t)buf * 2 * W + W, a.rb + (size_t)env * W, plane_bytes, b);
  };
  if constexpr (REL) {
    if (warp == nw + 1) {
      // --------------------------------------------------------- loader warp
      // per-env release: wait (acquire) for each item's env to be cast, then
      // bulk-load its record planes into the next free buffer; the store
      // warp never waits on the cast
      if (lane != 0) return;
      int it = 0;
      for (int q = blockIdx.x; q < n_items; q += gridDim.x, ++it) {
#if NV_STUDY_WAITSTAT
        const unsigned long long w0 = global_ns();
#endif
        wait_env_cast(a.done, a.consumed, a.fault, a.ready, a.posrec, q / bands, W, bands);
#if NV_STUDY_WAITSTAT
        // study build: ns the loader waited per item rank, and the items
        atomicAdd(g_waitstat + min(it, 7), global_ns() - w0);
        atomicAdd(g_waitstat + 8 + min(it, 7), 1ull);
#endif
        if (it >= NV_WS_CBUF)
          mbar_wait(colempty + (it % NV_WS_CBUF), (unsigned)(((it / NV_WS_CBUF) - 1) & 1));
        load_item(it % NV_WS_CBUF, q / bands);
      }
      return;
    }
    if (warp == nw) {
      // ---------------------------------------------------------- store warp
      if (lane != 0) return;
      const uint64_t pol = policy_evict_first();
      unsigned slot = 0, use = 0;
      for (int q = blockIdx.x; q < n_items; q += gridDim.x) {
        const int e = q / bands, row0 = (q - e * bands) * band_rows;
        for (int sl = 0; sl < slots_per_item; ++sl) {
          mbar_wait(full + slot, use & 1u);
          const uint8_t *buf = slots + (size_t)slot * L.slot_bytes;
          const size_t pix0 = ((size_t)e * H + (size_t)row0 + (size_t)sl * R) * W;
          if (want_rgb) bulk_store(a.rgb + pix0 * 3, buf, (unsigned)(R * W * 3), pol);
          if (want_d) bulk_store(a.depth + pix0, buf + off_d, (unsigned)(R * W * 4), pol);
          if (want_s) bulk_store(a.sem + pix0, buf + off_s, (unsigned)(R * W * 2), pol);
          bulk_commit();
          bulk_wait_read<0>();
          mbar_arrive(empty + slot);
          if (++slot == (unsigned)NSLOT) {
            slot = 0;
            ++use;
          }
        }
      }
      bulk_wait_all();
      // completes after the cast grid (stream order for what follows)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      return;
    }
  }
  if (!REL && warp == nw) {
    // ------------------------------------------------------------ store warp
    if (lane != 0) return;
    const uint64_t pol = policy_evict_first();
    int q = blockIdx.x;  // work item = (env, row band)
    // launched as a programmatic dependent of the column cast: the CTA's
    // set-up above overlapped the cast's tail; the records are complete and
    // visible once the cast grid is (a no-op for an ordinary launch)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // record planes run NV_WS_CBUF - 1 items ahead of the item being stored
#pragma unroll
    for (int j = 0; j < NV_WS_CBUF - 1; ++j)
      if (q + j * (int)gridDim.x < n_items) load_item(j, (q + j * (int)gridDim.x) / bands);
    unsigned slot = 0, use = 0;
    for (int it = 0; q < n_items; ++it, q += gridDim.x) {
      const int qn = q + (NV_WS_CBUF - 1) * (int)gridDim.x;
      if (qn < n_items) {
        const int j = it + NV_WS_CBUF - 1;  // item to post; buffer j % CBUF last held item j - CBUF
        if (j >= NV_WS_CBUF)
          mbar_wait(colempty + (j % NV_WS_CBUF), (unsigned)(((j / NV_WS_CBUF) - 1) & 1));
        load_item(j % NV_WS_CBUF, qn / bands);
      }
      const int e = q / bands, row0 = (q - e * bands) * band_rows;
      for (int sl = 0; sl < slots_per_item; ++sl) {
        mbar_wait(full + slot, use & 1u);
        const uint8_t *buf = slots + (size_t)slot * L.slot_bytes;
        const size_t pix0 = ((size_t)e * H + (size_t)row0 + (size_t)sl * R) * W;
#if NV_WS_DEBUG != 2
        if (want_rgb) bulk_store(a.rgb + pix0 * 3, buf, (unsigned)(R * W * 3), pol);
        if (want_d) bulk_store(a.depth + pix0, buf + off_d, (unsigned)(R * W * 4), pol);
        if (want_s) bulk_store(a.sem + pix0, buf + off_s, (unsigned)(R * W * 2), pol);
#else
        (void)buf; (void)pix0; (void)pol;
#endif
        bulk_commit();
        // wait for this slot's smem reads and hand it back at once
        bulk_wait_read<0>();
        mbar_arrive(empty + slot);
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
  const int seg = warp % S;
  const int rsub = warp / S;   // first row of this warp within a slot
  const int rstride = nw / S;  // row stride between the warp's RPW rows
  unsigned slot = 0, use = 0;
  int q = blockIdx.x;
  for (int it = 0; q < n_items; ++it, q += gridDim.x) {
    const int e = q / bands, row0 = (q - e * bands) * band_rows;
    mbar_wait(colfull + (it % NV_WS_CBUF), (unsigned)((it / NV_WS_CBUF) & 1));
    ColRegs<CPL> cr;
    const float4 *cA = cols_s + (size_t)(it % NV_WS_CBUF) * 2 * W + seg * Ln::SEGW;
    load_cols_smem<CPL>(cA, cA + W, lane, cr);
    __syncwarp();
    if (lane == 0) mbar_arrive(colempty + (it % NV_WS_CBUF));
    for (int sl = 0; sl < slots_per_item; ++sl) {
      if (use >= 1) mbar_wait(empty + slot, (use - 1) & 1u);
      uint8_t *buf = slots + (size_t)slot * L.slot_bytes;
#pragma unroll
      for (int rr = 0; rr < RPW; ++rr) {
        const int rs = rsub + rr * rstride;  // row within the slot
        const uint32_t i = (uint32_t)(row0 + sl * R + rs);
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
                     want_d ? reinterpret_cast<float *>(buf + off_d) : nullptr,
                     want_s ? reinterpret_cast<uint16_t *>(buf + off_s) : nullptr,
                     rs * W + seg * Ln::SEGW, lane);
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

// Inverse-depth noise as a separate pass over a written depth batch (after
// k_fill_generic, and nv_depth_noise_apply); same per-pixel values as the
// fused path of k_fill_ws.
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
