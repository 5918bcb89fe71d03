// device.cuh -- data layout shared by the kernels and the host side.
//
// HBM layout (one scene replica + one env shard per GPU):
//   * segment SoA, f64: ax, ay, bx, by, ex, ey, nx, ny (n each) -- the
//     reference's SegmentIndex / RenderGeometry arrays (geometry.py:111-117,
//     sensors.py:84-93), read by the disc casts and the column epilogue;
//   * uniform-grid CSR (geometry.py:128-141) with the bucket items EXPANDED
//     into 32-byte CellEntry records {ax, ay, ex, ey} (+ the parallel int32
//     items array, read only for prefilter survivors): the DDA reads one
//     contiguous run per cell instead of gathering through bucket_items;
//   * per-env agent state SoA (x, y, heading, path, collisions, cos/sin of
//     heading, episode frame);
//   * per camera: u_j (W f64), tc/tf row tables (H f64) for the exact FP64
//     row/column classification, and RowRec (H x 32 B) for shading;
//   * per camera, per step: ColRec (N x W x 32 B), the column hits + the
//     column's shading parameters, written by the cast kernel and read by the
//     fill kernel (8 MB at 1024 envs x 256 columns: L2-resident);
//   * frames: caller-owned u8 [N,H,W,3], f32 [N,H,W], u16 [N,H,W].
#pragma once

#include <stdint.h>

#ifndef NV_CHUNK
#define NV_CHUNK 8  // entries per prefilter box (cast)
#endif

namespace nvd {

struct __align__(16) CellEntry {
  double ax, ay;  // segment start
  double ex, ey;  // b - a (SegmentIndex.ex/ey, geometry.py:116-117)
};                // the segment index (tie-break key) is items[q]

// Per grid entry, for the swept-disc casts (disc_cast, _kernels.py:393-465):
// the segment's endpoints and the per-segment quantities the reference
// recomputes for every candidate -- seg_len = sqrt(ex^2 + ey^2) and the unit
// tangent (ex / seg_len, ey / seg_len) -- precomputed on the host with the
// same IEEE operations (no contraction), so the values are identical.
struct __align__(16) DiscEntry {
  double ax, ay, bx, by;
  double tx, ty, len;
  int32_t idx, pad;
};

struct SceneView {
  const double *ax, *ay, *bx, *by, *ex, *ey, *nx, *ny;
  const uint16_t *sem;
  const float4 *alb255;  // albedo * 255 (rgb, pad)
  const int32_t *starts; // nc + 1
  const CellEntry *ent;  // starts[nc] entries
  const int32_t *items;  // same order, index only (disc casts)
  const float4 *entf;    // same order, f32 endpoints (a - X0c, b - X0c), X0c = x0 + cx
  const float4 *entm;    // same order, f32 midpoint and half-vector (m - X0c, (b - a) / 2)
  const int4 *cells;     // per cell: {starts[c], starts[c+1], bits(bound), first chunk}
  const float4 *chunks;  // per run of NV_CHUNK entries: f32 box as centre and half-extents
                         // (xc, yc, hx, hy), cell-relative, containing every endpoint
  const DiscEntry *dent; // per entry (same order as items): disc-cast record
  const double *stx, *sty;  // per segment: unit tangent (ex, ey) / seg_len (0 if degenerate)
  double x0, y0;
  int gnx, gny;
  int64_t n;
};

struct EnvView {
  double *x, *y, *h, *path;
  int64_t *coll;
  double *ch, *sh;             // cos/sin of heading (correctly rounded)
  double *ox, *oy, *oh;        // episode frame (sensors.py:155-172)
  double *fc, *fs;             // cos(-oh), sin(-oh)
  uint8_t *reset;
  const uint8_t *frozen;       // task layer: finished episodes (nullptr = none)
  int n;
};

// Per-row shading record (fill kernel), 32 B.  Plane (floor / ceiling)
// parameters of the row, void-substituted when the plane depth >= max_range;
// colour/shading values are f16 pairs splatted over both halves so the fill
// kernel can blend them with per-pixel wall values two pixels at a time.
struct __align__(16) RowRec {
  float depth_p;  // plane depth (tc / tf), or max_range when void
  uint32_t sem2;  // plane semantic, splatted (s | s << 16)
  uint32_t num2;  // half2 splat of 0.8 * |v| (0 when void)
  uint32_t r2, g2, b2;  // half2 splats of the plane colour * 255 (0 when void)
  uint32_t pad[2];
};

// Per-column record (cast -> fill), 32 B.
struct __align__(16) ColRec {
  float depth_w;   // wall depth (f32(s)) or max_range when void
  float num08_w;   // 0.8 * |d . n_k| (0 when void)
  float d2;        // dx*dx + dy*dy
  uint32_t lohi;   // lo (ceiling rows [0, lo)) | hi << 16 (floor rows [hi, H))
  float col_w[3];  // albedo_k * 255 (0 when void)
  uint32_t sem_w;  // seg_sem[k] (0 when void)
};

// Column records live in two planes of 16-byte halves per camera,
//   A = {depth_w, num08_w, d2, lohi},  B = {col_w[0..2], sem_w},
// at index env * W + rec_pos(j): within each 32*CPL-column segment the record
// of column seg*32*CPL + g*32*GW + l*GW + c (lane l, group g, column c of the
// group, GW = min(CPL, 4)) sits at seg*32*CPL + (g*GW + c)*32 + l, so the 32
// lanes of a fill warp read 32 consecutive halves (conflict-free shared-memory
// rows, coalesced global loads).  cpl = 0: identity order.
#if defined(__CUDACC__)
#define NV_HDI __host__ __device__ __forceinline__
#else
#define NV_HDI static inline
#endif
NV_HDI int rec_pos(int j, int cpl) {
  if (cpl <= 0) return j;
  // cpl is a power of two (2, 4, 8): shifts and masks instead of divisions
#if defined(__CUDA_ARCH__)
  const int lc = __ffs(cpl) - 1;
#else
  const int lc = __builtin_ctz((unsigned)cpl);
#endif
  const int lg = lc < 2 ? lc : 2;  // log2 of the group width min(cpl, 4)
  const int seg = j >> (5 + lc), r = j & ((32 << lc) - 1);
  const int g = r >> (5 + lg), r2 = r & ((32 << lg) - 1);
  const int l = r2 >> lg, c = r2 & ((1 << lg) - 1);
  return (seg << (5 + lc)) + (((g << lg) + c) << 5) + l;
}

struct RecOut {  // column-record planes written by the casts
  float4 *a, *b;
  int W, cpl;
};

struct CamView {
  int W, H;
  int n_top;  // rows with v > 0
  int b0;     // first row with v < 0
  double max_range;
  const double *u;   // W: ((j + 0.5) - W*0.5) / focal
  const double *tc;  // H: (wall_h - cam_h) / v for v > 0 rows
  const double *tf;  // H: -cam_h / v for v < 0 rows
  const RowRec *rows;
  int cpl;  // record order of rec_pos (0 = identity)
  float hc, ktop, kbot;  // H/2 - 1/2, focal (wall_h - cam_h), focal cam_h (row estimates)
};

}  // namespace nvd
