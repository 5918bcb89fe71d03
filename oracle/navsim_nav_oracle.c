/* navsim_nav_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's navigation / task row (SURVEY.md §8f
 * rows 1-2): occupancy rasterisation, geodesic distance fields, bilinear
 * geodesic queries, goal snapping and the PointGoal task arithmetic.  Used
 * by tests/ as the parity checker of the CUDA nav/task kernels and pinned
 * against fixtures produced by the unmodified reference
 * (tests/golden/make_golden_task.py).  The product package never links it.
 *
 * Reference: /root/reference/pkg/src/navsim
 *   geometry.point_segment_distances   geometry.py:76-97
 *   geometry.navigable_mask            geometry.py:209-250
 *   _kernels.dijkstra_grid             _kernels.py:210-282
 *   nav._snap_to_navigable             nav.py:103-119
 *   nav.geodesic_distance              nav.py:135-166
 *   task.success_test / spl / reward   task.py:73-101
 *   Environment._distance_to_goal      task.py:160-177
 *
 * Arithmetic: binary64, round to nearest, no contraction (-ffp-contract=off);
 * numpy's einsum over 2-vectors evaluates x0*y0 + x1*y1 without FMA (checked
 * in the build container), which is what the code below does.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* geometry.point_segment_distances (geometry.py:86-96) for one point. */
double or_point_seg_dist(const double *segs, int64_t n, double px, double py) {
  double best = INFINITY;
  for (int64_t k = 0; k < n; ++k) {
    const double ax = segs[4 * k], ay = segs[4 * k + 1];
    const double ex = segs[4 * k + 2] - ax, ey = segs[4 * k + 3] - ay;
    double l2 = ex * ex + ey * ey;
    if (!(l2 >= 1e-300)) l2 = 1e-300;  /* np.maximum(l2, 1e-300) */
    const double wx = px - ax, wy = py - ay;
    double t = (wx * ex + wy * ey) / l2;
    if (t < 0.0) t = 0.0;               /* np.clip(., 0, 1) */
    if (t > 1.0) t = 1.0;
    const double dx = wx - t * ex, dy = wy - t * ey;
    const double d2 = dx * dx + dy * dy;
    if (d2 < best) best = d2;           /* sqrt is monotone: min then sqrt */
  }
  return sqrt(best);
}

/* Grid geometry of navigable_mask (geometry.py:227-233). */
void or_nav_dims(double xmin, double ymin, double xmax, double ymax, double res,
                 int64_t *nx, int64_t *ny, double *ox, double *oy) {
  const double pad = 2 * res;
  *nx = (int64_t)ceil((xmax - xmin + 2 * pad) / res);
  *ny = (int64_t)ceil((ymax - ymin + 2 * pad) / res);
  *ox = xmin - pad + res / 2.0;
  *oy = ymin - pad + res / 2.0;
}

/* In-place 4-connected flood of `out` from seeds over cells with open[] set. */
static void flood4(const uint8_t *open, uint8_t *out, int64_t h, int64_t w) {
  int64_t *stack = (int64_t *)malloc(sizeof(int64_t) * (size_t)(h * w + 1));
  int64_t sp = 0;
  for (int64_t c = 0; c < h * w; ++c)
    if (out[c]) stack[sp++] = c;
  while (sp > 0) {
    const int64_t c = stack[--sp];
    const int64_t i = c / w, j = c - i * w;
    const int64_t nb[4][2] = {{i - 1, j}, {i + 1, j}, {i, j - 1}, {i, j + 1}};
    for (int k = 0; k < 4; ++k) {
      const int64_t a = nb[k][0], b = nb[k][1];
      if (a < 0 || a >= h || b < 0 || b >= w) continue;
      const int64_t q = a * w + b;
      if (open[q] && !out[q]) {
        out[q] = 1;
        stack[sp++] = q;
      }
    }
  }
  free(stack);
}

/* geometry.navigable_mask (geometry.py:209-250).  mask / dist are ny*nx,
 * row i = y.  The reference labels the 4-connected components of the open
 * cells and calls every component touching the array border "outside"; the
 * union of those components is exactly the 4-flood of the open border cells. */
void or_navigable_mask(const double *segs, int64_t n, double xmin, double ymin, double xmax,
                       double ymax, double res, double agent_radius, uint8_t *mask,
                       double *dist) {
  int64_t nx, ny;
  double ox, oy;
  or_nav_dims(xmin, ymin, xmax, ymax, res, &nx, &ny, &ox, &oy);
  for (int64_t i = 0; i < ny; ++i) {
    const double y = oy + res * (double)i;
    for (int64_t j = 0; j < nx; ++j) {
      const double x = ox + res * (double)j;
      dist[i * nx + j] = n > 0 ? or_point_seg_dist(segs, n, x, y) : INFINITY;
    }
  }
  const double barrier = agent_radius > res ? agent_radius : res;
  const int64_t nc = nx * ny;
  uint8_t *open = (uint8_t *)calloc((size_t)nc, 1), *outside = (uint8_t *)calloc((size_t)nc, 1);
  for (int64_t c = 0; c < nc; ++c) open[c] = dist[c] >= barrier;
  for (int64_t i = 0; i < ny; ++i)
    for (int64_t j = 0; j < nx; ++j)
      if ((i == 0 || i == ny - 1 || j == 0 || j == nx - 1) && open[i * nx + j])
        outside[i * nx + j] = 1;
  flood4(open, outside, ny, nx);
  uint8_t *inside = (uint8_t *)calloc((size_t)nc, 1);
  for (int64_t c = 0; c < nc; ++c) inside[c] = open[c] && !outside[c];
  if (agent_radius < barrier) {
    /* ndimage.binary_dilation(structure=4-cross, iterations=k), border 0 */
    const int iters = (int)(ceil(barrier / res)) > 1 ? (int)ceil(barrier / res) : 1;
    uint8_t *tmp = (uint8_t *)calloc((size_t)nc, 1);
    for (int it = 0; it < iters; ++it) {
      for (int64_t i = 0; i < ny; ++i)
        for (int64_t j = 0; j < nx; ++j) {
          const int64_t c = i * nx + j;
          tmp[c] = inside[c] || (i > 0 && inside[c - nx]) || (i < ny - 1 && inside[c + nx]) ||
                   (j > 0 && inside[c - 1]) || (j < nx - 1 && inside[c + 1]);
        }
      memcpy(inside, tmp, (size_t)nc);
    }
    free(tmp);
  }
  for (int64_t c = 0; c < nc; ++c) mask[c] = dist[c] >= agent_radius && inside[c];
  free(open);
  free(outside);
  free(inside);
}

/* _kernels.dijkstra_grid (_kernels.py:210-282): binary-heap Dijkstra, the
 * reference's own heap discipline (sift with strict <, push up with <=). */
void or_dijkstra(const uint8_t *nav, int64_t h, int64_t w, int64_t si, int64_t sj, double res,
                 double *dist) {
  const int64_t n = h * w;
  for (int64_t c = 0; c < n; ++c) dist[c] = INFINITY;
  const int64_t cap = 4 * n + 16;
  double *hd = (double *)malloc(sizeof(double) * (size_t)cap);
  int64_t *hn = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
  const double diag = res * sqrt(2.0);
  const int64_t start = si * w + sj;
  dist[start] = 0.0;
  hd[0] = 0.0;
  hn[0] = start;
  int64_t size = 1;
  while (size > 0) {
    const double d0 = hd[0];
    const int64_t node = hn[0];
    size -= 1;
    hd[0] = hd[size];
    hn[0] = hn[size];
    int64_t k = 0;
    for (;;) {
      const int64_t l = 2 * k + 1, r = l + 1;
      int64_t s = k;
      if (l < size && hd[l] < hd[s]) s = l;
      if (r < size && hd[r] < hd[s]) s = r;
      if (s == k) break;
      double td = hd[k]; hd[k] = hd[s]; hd[s] = td;
      int64_t tn = hn[k]; hn[k] = hn[s]; hn[s] = tn;
      k = s;
    }
    if (d0 > dist[node]) continue;
    const int64_t ci = node / w, cj = node - ci * w;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj) {
        if (di == 0 && dj == 0) continue;
        const int64_t ni = ci + di, nj = cj + dj;
        if (ni < 0 || ni >= h || nj < 0 || nj >= w) continue;
        if (!nav[ni * w + nj]) continue;
        double nd;
        if (di != 0 && dj != 0) {
          if (!(nav[ci * w + nj] && nav[ni * w + cj])) continue;
          nd = d0 + diag;
        } else {
          nd = d0 + res;
        }
        const int64_t code = ni * w + nj;
        if (nd < dist[code]) {
          dist[code] = nd;
          hd[size] = nd;
          hn[size] = code;
          k = size;
          size += 1;
          while (k > 0) {
            const int64_t p = (k - 1) / 2;
            if (hd[p] <= hd[k]) break;
            double td = hd[k]; hd[k] = hd[p]; hd[p] = td;
            int64_t tn = hn[k]; hn[k] = hn[p]; hn[p] = tn;
            k = p;
          }
        }
      }
  }
  free(hd);
  free(hn);
}

/* OccupancyGrid.cell_of (nav.py:41-44) */
static void cell_of(double ox, double oy, double res, double px, double py, int64_t *i,
                    int64_t *j) {
  *j = (int64_t)floor((px - ox) / res + 0.5);
  *i = (int64_t)floor((py - oy) / res + 0.5);
}

/* nav._snap_to_navigable (nav.py:103-119); returns 1 and the cell, or 0. */
int or_snap(const uint8_t *nav, int64_t h, int64_t w, double ox, double oy, double res,
            double px, double py, double radius, int64_t *ci, int64_t *cj) {
  int64_t i0, j0;
  cell_of(ox, oy, res, px, py, &i0, &j0);
  const int64_t rc = (int64_t)ceil(radius / res) + 1;
  int found = 0;
  double best_d = INFINITY;
  const int64_t ilo = i0 - rc > 0 ? i0 - rc : 0, ihi = i0 + rc + 1 < h ? i0 + rc + 1 : h;
  const int64_t jlo = j0 - rc > 0 ? j0 - rc : 0, jhi = j0 + rc + 1 < w ? j0 + rc + 1 : w;
  for (int64_t i = ilo; i < ihi; ++i)
    for (int64_t j = jlo; j < jhi; ++j) {
      if (!nav[i * w + j]) continue;
      /* center_of: origin + res * [j, i] (numpy: elementwise product then sum) */
      const double cx = ox + res * (double)j, cy = oy + res * (double)i;
      const double d = hypot(cx - px, cy - py);
      if (d < best_d) {
        best_d = d;
        *ci = i;
        *cj = j;
        found = 1;
      }
    }
  if (!found || best_d > radius) return 0;
  return 1;
}

/* nav.geodesic_distance (nav.py:135-166).  *err = 1 when p is outside the
 * grid bounds (the reference raises NavError). */
double or_geodesic(const double *dist, int64_t h, int64_t w, double ox, double oy, double res,
                   double px, double py, int *err) {
  *err = 0;
  const double fx = (px - ox) / res, fy = (py - oy) / res;
  if (!(-0.5 <= fx && fx <= (double)w - 0.5 && -0.5 <= fy && fy <= (double)h - 0.5)) {
    *err = 1;
    return NAN;
  }
  int64_t j0 = 0, i0 = 0;
  if (w > 1) {
    j0 = (int64_t)floor(fx);
    if (j0 < 0) j0 = 0;
    if (j0 > w - 2) j0 = w - 2;
  }
  if (h > 1) {
    i0 = (int64_t)floor(fy);
    if (i0 < 0) i0 = 0;
    if (i0 > h - 2) i0 = h - 2;
  }
  double tx = fx - (double)j0, ty = fy - (double)i0;
  tx = tx < 0.0 ? 0.0 : (tx > 1.0 ? 1.0 : tx);   /* min(max(., 0), 1) */
  ty = ty < 0.0 ? 0.0 : (ty > 1.0 ? 1.0 : ty);
  const int di[4] = {0, 0, 1, 1}, dj[4] = {0, 1, 0, 1};
  const double wts[4] = {(1.0 - tx) * (1.0 - ty), tx * (1.0 - ty), (1.0 - tx) * ty, tx * ty};
  double v[4];
  int nfin = 0, fin[4];
  for (int k = 0; k < 4; ++k) {
    const int64_t i = i0 + di[k], j = j0 + dj[k];
    v[k] = (i >= 0 && i < h && j >= 0 && j < w) ? dist[i * w + j] : INFINITY;
    if (isfinite(v[k])) fin[nfin++] = k;
  }
  if (nfin == 0) return INFINITY;
  if (nfin < 4) {
    /* nearest finite corner by (di - ty)^2 + (dj - tx)^2, first minimum */
    int best = fin[0];
    double bd = INFINITY;
    for (int q = 0; q < nfin; ++q) {
      const int k = fin[q];
      const double a = (double)di[k] - ty, b = (double)dj[k] - tx;
      const double cd = a * a + b * b;   /* Python ** 2 of a float: x * x */
      if (cd < bd) {
        bd = cd;
        best = k;
      }
    }
    for (int k = 0; k < 4; ++k)
      if (!isfinite(v[k])) v[k] = v[best];
  }
  double s = 0.0;                        /* Python sum(): 0 + v0 w0 + ... */
  for (int k = 0; k < 4; ++k) s = s + v[k] * wts[k];
  return s;
}

/* task.spl (task.py:80-88); returns -1 on the reference's TaskError cases. */
double or_spl(int success, double shortest, double taken) {
  if (shortest <= 0.0 || taken < 0.0) return -1.0;
  if (!success) return 0.0;
  return shortest / (taken > shortest ? taken : shortest);
}

/* task.reward (task.py:91-97) */
double or_reward(double d_prev, double d_cur, int reached, double success_reward,
                 double step_penalty) {
  const double base = d_prev - d_cur + step_penalty;
  return reached ? base + success_reward : base;
}
