// nav.cuh -- sm_100a kernels of the navigation / task row (SURVEY.md §8f
// rows 1-2): occupancy rasterisation, geodesic distance fields, geodesic
// queries, goal snapping and the batched PointGoal task step.
//
//   k_nav_clearance  geometry.navigable_mask's per-cell wall distance
//                    (point_segment_distances, geometry.py:76-97): one thread
//                    per cell center, exact FP64 point-segment distances over
//                    the uniform segment grid, rings of 1 m cells grown until
//                    no unvisited segment can be closer.
//   k_nav_flood      the "outside" components (4-connected open cells that
//                    touch the border, geometry.py:236-241) as a tiled flood:
//                    each CTA floods its 32x32 tile in shared memory to local
//                    convergence; the host repeats until nothing changes.
//   k_nav_dilate / k_nav_mask   binary_dilation (geometry.py:243-246) and
//                    mask = (dist >= radius) & inside.
//   k_nav_relax      distance fields: Dijkstra's fixed point (dijkstra_grid,
//                    _kernels.py:210-282) by tiled Bellman-Ford relaxation.
//                    Dijkstra's output satisfies d[v] = min_u fl(d[u] + w) and
//                    is the least such fixed point (FP addition is monotone),
//                    so ANY relaxation order that reaches a fixed point from
//                    (0 at the goal, inf elsewhere) returns identical bits.
//                    Tiles whose neighbourhood did not change are skipped.
//   k_nav_geodesic   nav.geodesic_distance (nav.py:135-166) per query.
//   k_nav_snap       nav._snap_to_navigable (nav.py:103-119) per query.
//   k_task_step      Environment.step's task arithmetic (task.py:193-243):
//                    distance_to_goal with the 1-ray line-of-sight shortcut
//                    (task.py:160-177, raycast_grid), success, SPL, reward,
//                    termination, EpisodeOutcome records.
#pragma once

#include <cooperative_groups.h>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace nvk {

struct NavView {
  const uint8_t *mask;  // ny x nx (row i = y), navigable
  int nx, ny;
  double ox, oy, res;
};

// geometry.point_segment_distances for one (point, segment): squared
// distance, the reference's operation order (einsum over 2-vectors = x0*y0 +
// x1*y1 without FMA, np.maximum(l2, 1e-300), np.clip(t, 0, 1)).
__device__ __forceinline__ double pt_seg_d2(double px, double py, double ax, double ay,
                                           double ex, double ey) {
  double l2 = add(mul(ex, ex), mul(ey, ey));
  if (!(l2 >= 1e-300)) l2 = 1e-300;
  const double wx = sub(px, ax), wy = sub(py, ay);
  double t = div(add(mul(wx, ex), mul(wy, ey)), l2);
  t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
  const double dx = sub(wx, mul(t, ex)), dy = sub(wy, mul(t, ey));
  return add(mul(dx, dx), mul(dy, dy));
}

// Per cell center (ox + res*j, oy + res*i): distance to the nearest segment.
// A segment passing within R of p has a point inside the (2R+1)^2 block of
// 1 m cells around p's cell, so once every cell of rings 0..R is scanned and
// the best distance is <= R, no unscanned segment can be closer.
__global__ void __launch_bounds__(128) k_nav_clearance(SceneView sc, int nx, int ny, double ox,
                                                       double oy, double res, double *dist) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)nx * ny) return;
  const int i = (int)(c / nx), j = (int)(c - (long long)i * nx);
  const double px = add(ox, mul(res, (double)j)), py = add(oy, mul(res, (double)i));
  double best = NV_INF;
  if (sc.n > 0) {
    const int cx = cell_coord(px, sc.x0, sc.gnx), cy = cell_coord(py, sc.y0, sc.gny);
    const int rmax = max(max(cx, sc.gnx - 1 - cx), max(cy, sc.gny - 1 - cy));
    for (int r = 0; r <= rmax; ++r) {
      for (int yy = cy - r; yy <= cy + r; ++yy) {
        if (yy < 0 || yy >= sc.gny) continue;
        const bool edge_row = (yy == cy - r) || (yy == cy + r);
        for (int xx = cx - r; xx <= cx + r; xx += edge_row ? 1 : 2 * r) {
          if (xx >= 0 && xx < sc.gnx) {
            const int cc = yy * sc.gnx + xx;
            const int q0 = __ldg(sc.starts + cc), q1 = __ldg(sc.starts + cc + 1);
            for (int q = q0; q < q1; ++q) {
              const int s = __ldg(sc.items + q);
              const double d2 = pt_seg_d2(px, py, __ldg(sc.ax + s), __ldg(sc.ay + s),
                                          __ldg(sc.ex + s), __ldg(sc.ey + s));
              if (d2 < best) best = d2;
            }
          }
          if (r == 0) break;
        }
      }
      if (best <= (double)r * (double)r) break;
    }
  }
  dist[c] = nvx::sqrt_rn(best);
}

// open = dist >= barrier; outside seeds = open cells on the array border.
__global__ void k_nav_open(const double *dist, int nx, int ny, double barrier, uint8_t *open,
                           uint8_t *outside) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)nx * ny) return;
  const int i = (int)(c / nx), j = (int)(c - (long long)i * nx);
  const uint8_t o = dist[c] >= barrier;
  open[c] = o;
  outside[c] = o && (i == 0 || i == ny - 1 || j == 0 || j == nx - 1);
}

#define NV_NT 32  // nav tile edge (cells)

// One 32x32 tile (+1 halo) of the outside flood, to local convergence.
__global__ void __launch_bounds__(256) k_nav_flood(const uint8_t *open, uint8_t *outside, int nx,
                                                   int ny, int *changed) {
  __shared__ uint8_t so[NV_NT + 2][NV_NT + 2], sf[NV_NT + 2][NV_NT + 2];
  const int bx = blockIdx.x * NV_NT, by = blockIdx.y * NV_NT;
  for (int k = threadIdx.x; k < (NV_NT + 2) * (NV_NT + 2); k += blockDim.x) {
    const int ti = k / (NV_NT + 2), tj = k - ti * (NV_NT + 2);
    const int i = by + ti - 1, j = bx + tj - 1;
    const bool in = i >= 0 && i < ny && j >= 0 && j < nx;
    so[ti][tj] = in ? open[(size_t)i * nx + j] : 0;
    sf[ti][tj] = in ? outside[(size_t)i * nx + j] : 0;
  }
  __syncthreads();
  bool any = false;
  for (int it = 0; it < 4 * NV_NT * NV_NT; ++it) {
    bool ch = false;
    for (int k = threadIdx.x; k < NV_NT * NV_NT; k += blockDim.x) {
      const int ti = k / NV_NT + 1, tj = k % NV_NT + 1;
      if (so[ti][tj] && !sf[ti][tj] &&
          (sf[ti - 1][tj] | sf[ti + 1][tj] | sf[ti][tj - 1] | sf[ti][tj + 1])) {
        sf[ti][tj] = 1;
        ch = true;
      }
    }
    any |= ch;
    if (!__syncthreads_or(ch)) break;
  }
  if (__syncthreads_or(any)) {
    for (int k = threadIdx.x; k < NV_NT * NV_NT; k += blockDim.x) {
      const int ti = k / NV_NT + 1, tj = k % NV_NT + 1;
      const int i = by + ti - 1, j = bx + tj - 1;
      if (i < ny && j < nx) outside[(size_t)i * nx + j] = sf[ti][tj];
    }
    if (threadIdx.x == 0) atomicExch(changed, 1);
  }
}

// inside = open & !outside
__global__ void k_nav_inside(const uint8_t *open, const uint8_t *outside, long long n,
                             uint8_t *inside) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c < n) inside[c] = open[c] && !outside[c];
}

// One iteration of ndimage.binary_dilation with the 4-cross, border value 0.
__global__ void k_nav_dilate(const uint8_t *in, int nx, int ny, uint8_t *out) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= (long long)nx * ny) return;
  const int i = (int)(c / nx), j = (int)(c - (long long)i * nx);
  out[c] = in[c] || (i > 0 && in[c - nx]) || (i < ny - 1 && in[c + nx]) || (j > 0 && in[c - 1]) ||
           (j < nx - 1 && in[c + 1]);
}

__global__ void k_nav_mask(const double *dist, const uint8_t *inside, long long n, double radius,
                           uint8_t *mask) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c < n) mask[c] = dist[c] >= radius && inside[c];
}

// ---------------------------------------------------------- distance fields

__global__ void k_nav_field_init(double *fields, const int2 *goal_ij, int nx, int ny, int k) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n = (long long)nx * ny;
  if (c >= n * k) return;
  const int f = (int)(c / n);
  const long long cc = c - (long long)f * n;
  const int2 g = goal_ij[f];
  fields[c] = cc == (long long)g.x * nx + g.y ? 0.0 : NV_INF;
}

// One tile of one field (blockIdx.z): relax to local convergence in shared
// memory.  act_in[f][tile] says whether the tile or a neighbour changed in
// the previous pass; changed tiles raise act_out (for the next pass) and the
// global flag.  Update rule = dijkstra_grid's relaxation (_kernels.py:254-270):
// axial +res, diagonal +res*sqrt(2) only when both axial cells are navigable;
// only navigable cells carry distances.
// One tile of one field relaxed to local convergence in shared memory (all
// threads of the CTA).  Tile (and halo) distances are read through L2
// (ld.cg): in the cooperative kernel other CTAs write them during the launch.
__device__ __forceinline__ void relax_tile(double *D, const NavView &nv, double diag, int tx,
                                           int ty, int ntx, int nty, const uint8_t *act_in,
                                           uint8_t *act_out, int *changed) {
  __shared__ double sd[NV_NT + 2][NV_NT + 2];
  __shared__ uint8_t sm[NV_NT + 2][NV_NT + 2];
  if (!__ldcg(act_in + (size_t)ty * ntx + tx)) return;
  const int nx = nv.nx, ny = nv.ny;
  const int bx = tx * NV_NT, by = ty * NV_NT;
  for (int k = threadIdx.x; k < (NV_NT + 2) * (NV_NT + 2); k += blockDim.x) {
    const int ti = k / (NV_NT + 2), tj = k - ti * (NV_NT + 2);
    const int i = by + ti - 1, j = bx + tj - 1;
    const bool in = i >= 0 && i < ny && j >= 0 && j < nx;
    sm[ti][tj] = in ? nv.mask[(size_t)i * nx + j] : 0;
    sd[ti][tj] = in ? __ldcg(D + (size_t)i * nx + j) : NV_INF;
  }
  __syncthreads();
  const double res = nv.res;
  bool any = false;
  for (int it = 0; it < 8 * NV_NT * NV_NT; ++it) {
    bool ch = false;
    for (int k = threadIdx.x; k < NV_NT * NV_NT; k += blockDim.x) {
      const int ti = k / NV_NT + 1, tj = k % NV_NT + 1;
      if (!sm[ti][tj]) continue;
      double best = sd[ti][tj];
#pragma unroll
      for (int di = -1; di <= 1; ++di)
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj) {
          if (di == 0 && dj == 0) continue;
          const int ui = ti + di, uj = tj + dj;  // neighbour u relaxes this cell
          if (!sm[ui][uj]) continue;
          double nd;
          if (di != 0 && dj != 0) {
            // the diagonal u -> v needs both axial cells between them
            if (!(sm[ti][uj] && sm[ui][tj])) continue;
            nd = add(sd[ui][uj], diag);
          } else {
            nd = add(sd[ui][uj], res);
          }
          if (nd < best) best = nd;
        }
      if (best < sd[ti][tj]) {
        sd[ti][tj] = best;
        ch = true;
      }
    }
    any |= ch;
    if (!__syncthreads_or(ch)) break;
  }
  if (__syncthreads_or(any)) {
    for (int k = threadIdx.x; k < NV_NT * NV_NT; k += blockDim.x) {
      const int ti = k / NV_NT + 1, tj = k % NV_NT + 1;
      const int i = by + ti - 1, j = bx + tj - 1;
      if (i < ny && j < nx) D[(size_t)i * nx + j] = sd[ti][tj];
    }
    if (threadIdx.x < 9) {  // this tile and its 8 neighbours run next pass
      const int ay = ty + threadIdx.x / 3 - 1, ax = tx + threadIdx.x % 3 - 1;
      if (ay >= 0 && ay < nty && ax >= 0 && ax < ntx) act_out[(size_t)ay * ntx + ax] = 1;
    }
    if (threadIdx.x == 0) atomicExch(changed, 1);
  }
  __syncthreads();  // shared tile buffers are reused by the next tile of this CTA
}

// One pass over all tiles of all fields (host-driven variant).
__global__ void __launch_bounds__(256) k_nav_relax(double *fields, NavView nv, double diag,
                                                   const uint8_t *act_in, uint8_t *act_out,
                                                   int *changed) {
  const int tx = blockIdx.x, ty = blockIdx.y, f = blockIdx.z;
  const int ntx = gridDim.x, nty = gridDim.y;
  const size_t tb = (size_t)f * ntx * nty;
  relax_tile(fields + (size_t)f * nv.nx * nv.ny, nv, diag, tx, ty, ntx, nty, act_in + tb,
             act_out + tb, changed);
}

// All passes in one cooperative launch: CTAs stride over the (field, tile)
// list, a grid-wide barrier separates passes, and the run ends when a pass
// changed nothing.  flags[0..1]: change flags of even / odd passes.
__global__ void __launch_bounds__(256) k_nav_relax_coop(double *fields, NavView nv, double diag,
                                                        uint8_t *act_a, uint8_t *act_b, int ntx,
                                                        int nty, int k, int *flags) {
  cg::grid_group grid = cg::this_grid();
  const long long per_field = (long long)ntx * nty;
  const long long ntiles = per_field * k;
  for (int pass = 0;; ++pass) {
    uint8_t *ain = (pass & 1) ? act_b : act_a;
    uint8_t *aout = (pass & 1) ? act_a : act_b;
    int *changed = flags + (pass & 1);
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int f = (int)(t / per_field);
      const long long r = t - (long long)f * per_field;
      const int ty = (int)(r / ntx), tx = (int)(r - (long long)ty * ntx);
      relax_tile(fields + (size_t)f * nv.nx * nv.ny, nv, diag, tx, ty, ntx, nty,
                 ain + (size_t)f * per_field, aout + (size_t)f * per_field, changed);
    }
    grid.sync();
    if (!__ldcg(changed)) break;
    // this pass's input flags become the next pass's output: clear them
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < ntiles;
         t += (long long)gridDim.x * blockDim.x)
      ain[t] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) flags[(pass + 1) & 1] = 0;
    grid.sync();
  }
}

// ---------------------------------------------------------- queries

// nav.geodesic_distance (nav.py:135-166).  NaN marks the reference's
// NavError (point outside the grid bounds).
__device__ __forceinline__ double geodesic_at(const double *D, const NavView &nv, double px,
                                              double py) {
  const int w = nv.nx, h = nv.ny;
  const double fx = div(sub(px, nv.ox), nv.res), fy = div(sub(py, nv.oy), nv.res);
  if (!(-0.5 <= fx && fx <= (double)w - 0.5 && -0.5 <= fy && fy <= (double)h - 0.5))
    return __longlong_as_double(0x7ff8000000000000ll);
  int j0 = 0, i0 = 0;
  if (w > 1) j0 = min(max((int)floor(fx), 0), w - 2);
  if (h > 1) i0 = min(max((int)floor(fy), 0), h - 2);
  double tx = sub(fx, (double)j0), ty = sub(fy, (double)i0);
  tx = fmin(fmax(tx, 0.0), 1.0);
  ty = fmin(fmax(ty, 0.0), 1.0);
  const double u = sub(1.0, tx), v = sub(1.0, ty);
  const double wts[4] = {mul(u, v), mul(tx, v), mul(u, ty), mul(tx, ty)};
  double val[4];
  int fin = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = i0 + (k >> 1), j = j0 + (k & 1);
    val[k] = (i >= 0 && i < h && j >= 0 && j < w) ? D[(size_t)i * w + j] : NV_INF;
    if (isfinite(val[k])) fin |= 1 << k;
  }
  if (!fin) return NV_INF;
  if (fin != 15) {
    int best = -1;
    double bd = NV_INF;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (!(fin >> k & 1)) continue;
      const double a = sub((double)(k >> 1), ty), b = sub((double)(k & 1), tx);
      const double cd = add(mul(a, a), mul(b, b));
      if (cd < bd) {
        bd = cd;
        best = k;
      }
    }
    const double vb = val[best];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (!(fin >> k & 1)) val[k] = vb;
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s = add(s, mul(val[k], wts[k]));
  return s;
}

__global__ void k_nav_geodesic(const double *fields, const int32_t *fid, const double *pts,
                               long long m, NavView nv, double *out) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= m) return;
  const double *D = fields + (size_t)fid[q] * nv.nx * nv.ny;
  out[q] = geodesic_at(D, nv, pts[2 * q], pts[2 * q + 1]);
}

// nav._snap_to_navigable (nav.py:103-119): nearest navigable center within
// radius (math.hypot -> correctly rounded), first minimum in row-major scan.
__global__ void k_nav_snap(const double *pts, long long m, NavView nv, double radius,
                           int32_t *cells) {
  const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (q >= m) return;
  const double px = pts[2 * q], py = pts[2 * q + 1];
  const int j0 = (int)floor(add(div(sub(px, nv.ox), nv.res), 0.5));
  const int i0 = (int)floor(add(div(sub(py, nv.oy), nv.res), 0.5));
  const int rc = (int)ceil(div(radius, nv.res)) + 1;
  double bd = NV_INF;
  int bi = -1, bj = -1;
  for (int i = max(0, i0 - rc); i < min(nv.ny, i0 + rc + 1); ++i)
    for (int j = max(0, j0 - rc); j < min(nv.nx, j0 + rc + 1); ++j) {
      if (!nv.mask[(size_t)i * nv.nx + j]) continue;
      const double cx = add(nv.ox, mul(nv.res, (double)j)), cy = add(nv.oy, mul(nv.res, (double)i));
      const double d = nvx::hypot_cr(sub(cx, px), sub(cy, py));
      if (d < bd) {
        bd = d;
        bi = i;
        bj = j;
      }
    }
  if (bi < 0 || bd > radius) bi = bj = -1;
  cells[2 * q] = bi;
  cells[2 * q + 1] = bj;
}

// ---------------------------------------------------------- task step

// Per-env task state (Environment, task.py:123-160) and config.
struct TaskView {
  const double *goal;    // n x 2
  const double *gdsp;    // n (episode shortest path, task.py:33-38)
  const int32_t *fid;    // n: field of the env's goal
  const double *fields;  // k x ny x nx
  double *d_last;        // n
  int32_t *steps;        // n
  uint8_t *done;         // n
  int max_steps;
  double success_radius, success_reward, step_penalty;
};

// EpisodeOutcome (task.py:58-66) as the 40-byte all-gather record.
struct __align__(8) OutcomeRec {
  uint8_t success, terminated_by;  // 1 stop, 2 step_limit (0: running)
  uint8_t pad[2];
  int32_t steps;
  int32_t collisions;
  int32_t pad2;
  double path_taken, shortest_path, spl;
};

// Environment._distance_to_goal (task.py:160-177).
__device__ __forceinline__ double distance_to_goal(const SceneView &sc, const NavView &nv,
                                                   const TaskView &tv, int e, double px,
                                                   double py) {
  const double gx = tv.goal[2 * e], gy = tv.goal[2 * e + 1];
  const double dx = sub(gx, px), dy = sub(gy, py);
  const double euclid = nvx::hypot_cr(dx, dy);  // np.hypot -> correctly rounded hypot
  if (euclid <= 1.0) {
    if (euclid < 1e-12) return 0.0;
    double t;
    int k;
    ray_grid(sc, px, py, dx, dy, 1e9, t, k);  // SegmentIndex.raycast default t_max
    if (!(t <= 1.0)) return euclid;
  }
  return geodesic_at(tv.fields + (size_t)tv.fid[e] * nv.nx * nv.ny, nv, px, py);
}

// Environment.step's task arithmetic (task.py:198-243) for a stepped env e
// whose new distance is d_cur: step counter, termination (stop / budget),
// success, reward, EpisodeOutcome.  One thread.
__device__ __forceinline__ void task_finish(const TaskView &tv, int e, int a, double d_cur,
                                            double path, long long coll, double *reward,
                                            double *dist, uint8_t *done_out, OutcomeRec *out) {
  const int steps = tv.steps[e] + 1;
  tv.steps[e] = steps;
  const double d_prev = tv.d_last[e];
  tv.d_last[e] = d_cur;
  int term = 0;
  bool success = false;
  if (a == 3) {
    term = 1;
    success = d_cur <= tv.success_radius;  // task.success_test
  } else if (steps >= tv.max_steps) {
    term = 2;
  }
  const double base = add(sub(d_prev, d_cur), tv.step_penalty);  // task.reward
  if (reward) reward[e] = term && success ? add(base, tv.success_reward) : base;
  if (dist) dist[e] = d_cur;
  if (term) {
    tv.done[e] = 1;
    if (out) {
      OutcomeRec o;
      o.success = success;
      o.terminated_by = (uint8_t)term;
      o.pad[0] = o.pad[1] = 0;
      o.steps = steps;
      o.collisions = (int32_t)coll;
      o.pad2 = 0;
      o.path_taken = path;
      o.shortest_path = tv.gdsp[e];
      const double sh = o.shortest_path, tk = o.path_taken;  // task.spl
      o.spl = success ? div(sh, tk > sh ? tk : sh) : 0.0;
      out[e] = o;
    }
  }
  if (done_out) done_out[e] = tv.done[e];
}

// An env the step did not advance (not reset, episode over, bad action:
// status != 0) earns nothing this step: reward 0, distance unchanged (the
// reference raises instead of stepping it, task.py:196-197), so a caller
// summing rewards over batch steps never counts a terminal reward twice.
__device__ __forceinline__ void task_skip(const TaskView &tv, int e, double *reward, double *dist,
                                          uint8_t *done_out) {
  if (reward) reward[e] = 0.0;
  if (dist) dist[e] = tv.d_last[e];
  if (done_out) done_out[e] = tv.done[e];
}

// Environment.step's task arithmetic (task.py:193-243) after the agent step.
__global__ void k_task_step(EnvView ev, SceneView sc, NavView nv, TaskView tv,
                            const int8_t *__restrict__ actions, const int32_t *step_status,
                            double *reward, double *dist, uint8_t *done_out, OutcomeRec *out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ev.n) return;
  if (step_status && step_status[e] != 0) {  // not stepped (not reset / done / bad)
    task_skip(tv, e, reward, dist, done_out);
    return;
  }
  const double d_cur = distance_to_goal(sc, nv, tv, e, ev.x[e], ev.y[e]);
  task_finish(tv, e, actions[e], d_cur, ev.path[e], ev.coll[e], reward, dist, done_out, out);
}

// Environment._distance_to_goal by a whole warp (the line-of-sight ray uses
// the warp DDA); the result is identical in every lane.
__device__ __forceinline__ double distance_to_goal_warp(const SceneView &sc, const NavView &nv,
                                                        const TaskView &tv, int e, double px,
                                                        double py) {
  const double gx = tv.goal[2 * e], gy = tv.goal[2 * e + 1];
  const double dx = sub(gx, px), dy = sub(gy, py);
  const double euclid = nvx::hypot_cr(dx, dy);
  if (euclid <= 1.0) {
    if (euclid < 1e-12) return 0.0;
    double t;
    int k;
    ray_grid_warp(sc, px, py, dx, dy, 1e9, t, k);
    if (!(t <= 1.0)) return euclid;
  }
  return geodesic_at(tv.fields + (size_t)tv.fid[e] * nv.nx * nv.ny, nv, px, py);
}

// The task arithmetic riding on the column cast (nv_task_step_render with the
// DDA casts): the thread (or warp) of column 0 of each env, which is short
// next to the env's longest ray, computes the env's distance to the goal and
// the step's task outputs after the agent step of the previous launch.
struct TaskOut {
  NavView nv;
  TaskView tv;
  const int8_t *actions;
  const int32_t *status;
  double *reward, *dist;
  uint8_t *done;
  OutcomeRec *out;
};

// done: per-env release to the frame writer (its programmatic dependent), as
// in k_column_cast.
// With `ready`: a programmatic dependent of the agent step, waiting per env
// like k_column_cast (release mode when `arrive` is null); the agent step's
// outputs are then read through L2.
template <bool COH>
__device__ __forceinline__ void task_column(const EnvView &ev, const SceneView &sc,
                                            const CamView &cam, const RecOut &ro, double t_max,
                                            double *gps, double *compass, const TaskOut &to, int e,
                                            int j) {
  if (j == 0) {  // before the ray: the env's task step
    const int32_t status = COH ? __ldcg(to.status + e) : to.status[e];
    if (status != 0) {
      task_skip(to.tv, e, to.reward, to.dist, to.done);
    } else {
      const double px = COH ? __ldcg(ev.x + e) : ev.x[e], py = COH ? __ldcg(ev.y + e) : ev.y[e];
      const double d_cur = distance_to_goal(sc, to.nv, to.tv, e, px, py);
      task_finish(to.tv, e, to.actions[e], d_cur, COH ? __ldcg(ev.path + e) : ev.path[e],
                  COH ? __ldcg(ev.coll + e) : ev.coll[e], to.reward, to.dist, to.done, to.out);
    }
  }
  cast_column<COH>(ev, sc, cam, e, j, ro, t_max, gps, compass);
}

// The task step from a pose record (release mode, NV_POSE_REC): every input
// the agent step produced comes from the record.
__device__ __forceinline__ void task_column_rec(const EnvView &ev, const SceneView &sc,
                                                const CamView &cam, const RecOut &ro,
                                                double t_max, double *gps, double *compass,
                                                const TaskOut &to, int e, int j,
                                                const double *rec, unsigned *fault) {
  double px, py, c, s, h, path, collb, stat;
  unsigned long long t0 = 0;
  for (;;) {
    px = ld_relaxed_f64(rec);
    py = ld_relaxed_f64(rec + 1);
    c = ld_relaxed_f64(rec + 2);
    s = ld_relaxed_f64(rec + 3);
    h = ld_relaxed_f64(rec + 4);
    path = ld_relaxed_f64(rec + 5);
    collb = ld_relaxed_f64(rec + 6);
    stat = ld_relaxed_f64(rec + 7);
    if (!(is_pose_sentinel(px) | is_pose_sentinel(py) | is_pose_sentinel(c) | is_pose_sentinel(s) |
          is_pose_sentinel(h) | is_pose_sentinel(path) | is_pose_sentinel(collb) |
          is_pose_sentinel(stat)))
      break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (!t0) {
      t0 = t;
    } else if (t - t0 > 200000000ull || *reinterpret_cast<volatile unsigned *>(fault)) {
      atomicExch(fault, 1u);
      break;
    }
    __nanosleep(64);
  }
  if (j == 0) {  // before the ray: the env's task step
    if ((int)stat != 0) {
      task_skip(to.tv, e, to.reward, to.dist, to.done);
    } else {
      const double d_cur = distance_to_goal(sc, to.nv, to.tv, e, px, py);
      task_finish(to.tv, e, to.actions[e], d_cur, path, __double_as_longlong(collb), to.reward,
                  to.dist, to.done, to.out);
    }
  }
  cast_column_at(ev, sc, cam, e, j, ro, t_max, gps, compass, px, py, c, s, h);
}

__global__ void __launch_bounds__(128) k_column_cast_task(EnvView ev, SceneView sc, CamView cam,
                                                          RecOut ro, double t_max, double *gps,
                                                          double *compass, TaskOut to,
                                                          unsigned *done, unsigned *ready,
                                                          unsigned *arrive, unsigned *rfault,
                                                          const double *posrec) {
  // triggers only when the writer follows as its programmatic dependent
  // (release), see k_column_cast
  if (done) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long total = (long long)ev.n * cam.W;
  if (ready) {
    if (arrive) {
      wait_envs_ready(ready, arrive, cam.W, total);
    } else {
      const long long w0 = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31u);
      if (w0 < total)
        warp_wait_envs_ready(ready, rfault, (unsigned)w0, (unsigned)min(total - 1, w0 + 31),
                             (unsigned)cam.W);
    }
  }
  if (g < total) {
    const int e = (int)(g / cam.W);
    const int j = (int)(g - (long long)e * cam.W);
    if (posrec)
      task_column_rec(ev, sc, cam, ro, t_max, gps, compass, to, e, j,
                      posrec + (size_t)e * NV_POSE_STRIDE, rfault);
    else if (ready)
      task_column<true>(ev, sc, cam, ro, t_max, gps, compass, to, e, j);
    else
      task_column<false>(ev, sc, cam, ro, t_max, gps, compass, to, e, j);
  }
  if (done) {
    __syncthreads();
    if (threadIdx.x == 0) release_envs(done, blockIdx.x, (int)blockDim.x, cam.W, total);
  }
  grid_completes_after_predecessor();
}

__global__ void __launch_bounds__(128) k_column_cast_warp_task(EnvView ev, SceneView sc,
                                                               CamView cam, RecOut ro,
                                                               double t_max, double *gps,
                                                               double *compass, TaskOut to) {
  const long long g = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long total = (long long)ev.n * cam.W;
  if (g >= total) return;
  const int e = (int)(g / cam.W);
  const int j = (int)(g - (long long)e * cam.W);
  if (j == 0) {
    const int lane = threadIdx.x & 31;
    if (to.status[e] != 0) {
      if (lane == 0) task_skip(to.tv, e, to.reward, to.dist, to.done);
    } else {
      const double d_cur = distance_to_goal_warp(sc, to.nv, to.tv, e, ev.x[e], ev.y[e]);
      if (lane == 0)
        task_finish(to.tv, e, to.actions[e], d_cur, ev.path[e], ev.coll[e], to.reward,
                    to.dist, to.done, to.out);
    }
  }
  k_column_cast_warp_body(ev, sc, cam, ro, t_max, gps, compass, e, j);
}

// Environment.reset's initial distance (task.py:188) for masked envs.
__global__ void k_task_reset(EnvView ev, SceneView sc, NavView nv, TaskView tv,
                             const uint8_t *mask) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ev.n || (mask && !mask[e])) return;
  tv.steps[e] = 0;
  tv.done[e] = 0;
  tv.d_last[e] = distance_to_goal(sc, nv, tv, e, ev.x[e], ev.y[e]);
}

}  // namespace nvk
