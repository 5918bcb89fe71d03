/* navsim_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C restatement of the reference's hot path (navsim, pure Python +
 * numba, /root/reference/pkg/src/navsim).  Every function cites the
 * reference lines it follows.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library; the
 * product path (paper_1904_01201_b200) never does.
 *
 * Arithmetic contract: binary64, round-to-nearest, NO contraction (built with
 * -ffp-contract=off) -- the numba kernels are compiled without fastmath and
 * contain no FMA (src/_kernels.py:1-5).  cos/sin/tan/hypot/fmod come from the
 * same glibc libm that Python's math module and numpy call, so this file is
 * bit-identical to the reference (pinned by tests/test_oracle_golden.py).
 * The one host-dependent op, np.dot on 2-vectors (src/sim.py:111), resolves to
 * OpenBLAS ddot, which on this image equals fma(a1, b1, a0*b0) exactly (0 of
 * 100k mismatches); we mirror that.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define SEM_VOID 0       /* src/_kernels.py:123 */
#define SEM_FLOOR 65534  /* src/_kernels.py:124 */
#define SEM_CEILING 65535 /* src/_kernels.py:125 */
#define CONTACT_EPSILON 1e-4 /* src/sim.py:24 */
#define CELL 1.0         /* src/geometry.py:107 */

/* ------------------------------------------------------------------ grid */

/* SegmentIndex.__init__ bounds, src/geometry.py:118-127 */
void or_grid_dims(const double *segs, int64_t n, double *x0, double *y0,
                  int64_t *nx, int64_t *ny) {
  double gx0, gy0, x1, y1;
  if (n > 0) {
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      const double *s = segs + 4 * i;
      /* min(ax.min(), bx.min()) */
      if (s[0] < mnx) mnx = s[0];
      if (s[2] < mnx) mnx = s[2];
      if (s[1] < mny) mny = s[1];
      if (s[3] < mny) mny = s[3];
      if (s[0] > mxx) mxx = s[0];
      if (s[2] > mxx) mxx = s[2];
      if (s[1] > mxy) mxy = s[1];
      if (s[3] > mxy) mxy = s[3];
    }
    gx0 = mnx - 0.5;
    gy0 = mny - 0.5;
    x1 = mxx + 0.5;
    y1 = mxy + 0.5;
  } else {
    gx0 = gy0 = -0.5;
    x1 = y1 = 0.5;
  }
  int64_t cx = (int64_t)ceil((x1 - gx0) / CELL);
  int64_t cy = (int64_t)ceil((y1 - gy0) / CELL);
  *x0 = gx0;
  *y0 = gy0;
  *nx = cx > 1 ? cx : 1;
  *ny = cy > 1 ? cy : 1;
}

/* SegmentIndex._cell_of, src/geometry.py:146-149: int() truncates toward
 * zero, then clamps; done in the double domain to stay defined for any x. */
static int64_t cell_coord(double v, double o, int64_t n) {
  double d = (v - o) / CELL;
  if (!(d >= 1.0)) return 0; /* trunc(d) <= 0 -> clamp to 0 (also NaN) */
  if (d >= (double)(n - 1)) return n - 1;
  return (int64_t)d;
}

/* CSR bucket build, src/geometry.py:128-141.  Call with items == NULL to get
 * the item count; starts has nx*ny+1 entries. */
int64_t or_grid_build(const double *segs, int64_t n, double x0, double y0,
                      int64_t nx, int64_t ny, int64_t *starts, int64_t *items) {
  int64_t nc = nx * ny;
  int64_t *cnt = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    for (int64_t i = 0; i < n; ++i) {
      const double *s = segs + 4 * i;
      double mnx = s[0] < s[2] ? s[0] : s[2], mny = s[1] < s[3] ? s[1] : s[3];
      double mxx = s[0] > s[2] ? s[0] : s[2], mxy = s[1] > s[3] ? s[1] : s[3];
      int64_t cx0 = cell_coord(mnx, x0, nx), cy0 = cell_coord(mny, y0, ny);
      int64_t cx1 = cell_coord(mxx, x0, nx), cy1 = cell_coord(mxy, y0, ny);
      for (int64_t cy = cy0; cy <= cy1; ++cy)
        for (int64_t cx = cx0; cx <= cx1; ++cx) {
          int64_t c = cy * nx + cx;
          if (pass == 0)
            cnt[c + 1]++;
          else if (items)
            items[cnt[c]++] = i;
        }
    }
    if (pass == 0) {
      for (int64_t c = 0; c < nc; ++c) cnt[c + 1] += cnt[c];
      if (starts) memcpy(starts, cnt, sizeof(int64_t) * (size_t)(nc + 1));
      if (!items) break;
    }
  }
  int64_t total = starts ? starts[nc] : 0;
  if (!starts) { /* count-only query */
    total = cnt[nc];
  }
  free(cnt);
  return total;
}

static int cmp_i64(const void *a, const void *b) {
  const int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}

/* SegmentIndex.query_aabb, src/geometry.py:151-163: sorted unique ids.
 * mark is scratch of n bytes (zeroed on entry and on exit). Returns count. */
int64_t or_query_aabb(double xmin, double ymin, double xmax, double ymax,
                      double x0, double y0, int64_t nx, int64_t ny,
                      const int64_t *starts, const int64_t *items, int64_t n,
                      uint8_t *mark, int64_t *out) {
  int64_t cx0 = cell_coord(xmin, x0, nx), cy0 = cell_coord(ymin, y0, ny);
  int64_t cx1 = cell_coord(xmax, x0, nx), cy1 = cell_coord(ymax, y0, ny);
  /* np.unique(np.concatenate(buckets)): the marked ids in ascending order,
     gathered from the buckets and sorted (O(k log k) like np.unique, not a
     scan over all n segments) */
  int64_t m = 0;
  (void)n;
  for (int64_t cy = cy0; cy <= cy1; ++cy)
    for (int64_t cx = cx0; cx <= cx1; ++cx) {
      int64_t k = cy * nx + cx;
      for (int64_t q = starts[k]; q < starts[k + 1]; ++q)
        if (!mark[items[q]]) {
          mark[items[q]] = 1;
          out[m++] = items[q];
        }
    }
  qsort(out, (size_t)m, sizeof(int64_t), cmp_i64);
  for (int64_t i = 0; i < m; ++i) mark[out[i]] = 0;
  return m;
}

/* ------------------------------------------------------------- raycasts */

/* raycast_all, src/_kernels.py:16-48 */
void or_raycast_all(double px, double py, const double *dirx, const double *diry,
                    int64_t m, const double *ax, const double *ay,
                    const double *ex, const double *ey, int64_t n,
                    double *t_out, int64_t *i_out) {
  for (int64_t k = 0; k < m; ++k) {
    double dx = dirx[k], dy = diry[k];
    double best_t = INFINITY;
    int64_t best_i = -1;
    for (int64_t i = 0; i < n; ++i) {
      double den = dx * ey[i] - dy * ex[i];
      if (den == 0.0) continue;
      double sx = ax[i] - px, sy = ay[i] - py;
      double t = (sx * ey[i] - sy * ex[i]) / den;
      if (t < 0.0 || t > best_t) continue;
      double r = (sx * dy - sy * dx) / den;
      if (0.0 <= r && r <= 1.0) {
        if (t < best_t || i < best_i) {
          best_t = t;
          best_i = i;
        }
      }
    }
    t_out[k] = best_t;
    i_out[k] = best_i;
  }
}

/* raycast_grid, src/_kernels.py:51-120 (one ray) */
static void ray_grid1(double px, double py, double dx, double dy, double gx0,
                      double gy0, double cell, int64_t gnx, int64_t gny,
                      const int64_t *bs, const int64_t *bi, const double *ax,
                      const double *ay, const double *ex, const double *ey,
                      double t_max, double *t_res, int64_t *i_res) {
  int64_t cx = (int64_t)floor((px - gx0) / cell);
  int64_t cy = (int64_t)floor((py - gy0) / cell);
  int64_t stepx = dx > 0.0 ? 1 : -1;
  int64_t stepy = dy > 0.0 ? 1 : -1;
  double tnx, tdx, tny, tdy;
  if (dx != 0.0) {
    double nbx = gx0 + (double)(cx + (dx > 0.0 ? 1 : 0)) * cell;
    tnx = (nbx - px) / dx;
    tdx = fabs(cell / dx);
  } else {
    tnx = INFINITY;
    tdx = INFINITY;
  }
  if (dy != 0.0) {
    double nby = gy0 + (double)(cy + (dy > 0.0 ? 1 : 0)) * cell;
    tny = (nby - py) / dy;
    tdy = fabs(cell / dy);
  } else {
    tny = INFINITY;
    tdy = INFINITY;
  }
  double best_t = INFINITY;
  int64_t best_i = -1;
  for (;;) {
    if (0 <= cx && cx < gnx && 0 <= cy && cy < gny) {
      int64_t c = cy * gnx + cx;
      for (int64_t q = bs[c]; q < bs[c + 1]; ++q) {
        int64_t i = bi[q];
        double den = dx * ey[i] - dy * ex[i];
        if (den == 0.0) continue;
        double sx = ax[i] - px, sy = ay[i] - py;
        double t = (sx * ey[i] - sy * ex[i]) / den;
        if (t < 0.0 || t > best_t) continue;
        double r = (sx * dy - sy * dx) / den;
        if (0.0 <= r && r <= 1.0) {
          if (t < best_t || i < best_i) {
            best_t = t;
            best_i = i;
          }
        }
      }
    }
    double t_exit = tnx < tny ? tnx : tny;
    if (best_t <= t_exit || t_exit > t_max) break;
    if (tnx < tny) {
      cx += stepx;
      tnx += tdx;
    } else {
      cy += stepy;
      tny += tdy;
    }
    if (cx < 0 || cx >= gnx || cy < 0 || cy >= gny) {
      int out_x = (cx < 0 && dx <= 0.0) || (cx >= gnx && dx >= 0.0);
      int out_y = (cy < 0 && dy <= 0.0) || (cy >= gny && dy >= 0.0);
      if (out_x || out_y) break;
    }
  }
  *t_res = best_t;
  *i_res = best_i;
}

void or_raycast_grid(double px, double py, const double *dirx, const double *diry,
                     int64_t m, double gx0, double gy0, double cell, int64_t gnx,
                     int64_t gny, const int64_t *bs, const int64_t *bi,
                     const double *ax, const double *ay, const double *ex,
                     const double *ey, double t_max, double *t_out,
                     int64_t *i_out) {
  for (int64_t k = 0; k < m; ++k)
    ray_grid1(px, py, dirx[k], diry[k], gx0, gy0, cell, gnx, gny, bs, bi, ax, ay,
              ex, ey, t_max, &t_out[k], &i_out[k]);
}

/* ----------------------------------------------------------- frame fill */

/* fill_frame, src/_kernels.py:128-207.  depth (H,W) f64, rgb (H,W,3) f64,
 * sem (H,W) u16; unwanted channels may be NULL. */
void or_fill_frame(const double *t_col, const int64_t *i_col, int64_t height,
                   int64_t width, double focal, double cam_h, double wall_h,
                   double max_range, const double *seg_albedo,
                   const uint16_t *seg_sem, const double *seg_nx,
                   const double *seg_ny, const double *dirx, const double *diry,
                   const double *floor_color, const double *ceil_color,
                   double *depth, double *rgb, uint16_t *sem) {
  for (int64_t i = 0; i < height; ++i) {
    double v = ((double)height * 0.5 - ((double)i + 0.5)) / focal;
    for (int64_t j = 0; j < width; ++j) {
      double s = t_col[j];
      double dx = dirx[j], dy = diry[j];
      double inv_len = 1.0 / sqrt(dx * dx + dy * dy + v * v);
      double t = INFINITY;
      int kind = 0;
      if (v < 0.0) {
        double tf = -cam_h / v;
        if (tf <= s) {
          t = tf;
          kind = 2;
        } else if (s != INFINITY) {
          t = s;
          kind = 1;
        }
      } else if (v > 0.0) {
        double tc = (wall_h - cam_h) / v;
        if (tc <= s) {
          t = tc;
          kind = 3;
        } else if (s != INFINITY) {
          t = s;
          kind = 1;
        }
      } else {
        if (s != INFINITY) {
          t = s;
          kind = 1;
        }
      }
      if (t >= max_range) kind = 0;
      int64_t p = i * width + j;
      if (kind == 0) {
        if (depth) depth[p] = max_range;
        if (sem) sem[p] = SEM_VOID;
        if (rgb) rgb[3 * p] = rgb[3 * p + 1] = rgb[3 * p + 2] = 0.0;
      } else if (kind == 1) {
        int64_t k = i_col[j];
        if (depth) depth[p] = t;
        if (sem) sem[p] = seg_sem[k];
        if (rgb) {
          double cos_a = fabs(dx * seg_nx[k] + dy * seg_ny[k]) * inv_len;
          double shade = 0.2 + 0.8 * cos_a;
          rgb[3 * p] = seg_albedo[3 * k] * shade;
          rgb[3 * p + 1] = seg_albedo[3 * k + 1] * shade;
          rgb[3 * p + 2] = seg_albedo[3 * k + 2] * shade;
        }
      } else {
        if (depth) depth[p] = t;
        if (sem) sem[p] = kind == 2 ? SEM_FLOOR : SEM_CEILING;
        if (rgb) {
          double cos_a = fabs(v) * inv_len;
          double shade = 0.2 + 0.8 * cos_a;
          const double *c = kind == 2 ? floor_color : ceil_color;
          rgb[3 * p] = c[0] * shade;
          rgb[3 * p + 1] = c[1] * shade;
          rgb[3 * p + 2] = c[2] * shade;
        }
      }
    }
  }
}

/* _column_directions, src/sensors.py:96-102 */
void or_column_directions(double heading, int64_t width, double focal,
                          double *dirx, double *diry) {
  double fx = cos(heading), fy = sin(heading);
  double rx = sin(heading), ry = -cos(heading);
  for (int64_t j = 0; j < width; ++j) {
    double u = (((double)j + 0.5) - (double)width * 0.5) / focal;
    dirx[j] = fx + u * rx;
    diry[j] = fy + u * ry;
  }
}

/* segment_normals, src/geometry.py:66-73 */
void or_segment_normals(const double *segs, int64_t n, double *nx, double *ny) {
  for (int64_t i = 0; i < n; ++i) {
    const double *s = segs + 4 * i;
    double ex = s[2] - s[0], ey = s[3] - s[1];
    double ln = hypot(ex, ey);
    if (!(ln > 0.0)) ln = 1.0;
    nx[i] = -ey / ln;
    ny[i] = ex / ln;
  }
}

/* ---------------------------------------------------------- disc casts */

/* disc_cast, src/_kernels.py:393-465 */
void or_disc_cast(double px, double py, double ux, double uy, double radius,
                  const int64_t *cand, int64_t ncand, const double *ax,
                  const double *ay, const double *bx, const double *by,
                  double *t_res, int64_t *i_res, double *tan_x, double *tan_y) {
  double best_t = INFINITY;
  int64_t best_i = -1;
  double u2 = ux * ux + uy * uy;
  for (int64_t q = 0; q < ncand; ++q) {
    int64_t i = cand[q];
    double exi = bx[i] - ax[i], eyi = by[i] - ay[i];
    double seg_len = sqrt(exi * exi + eyi * eyi);
    if (seg_len <= 0.0) continue;
    double tx = exi / seg_len, ty = eyi / seg_len;
    double nx = -ty, ny = tx;
    double relx = px - ax[i], rely = py - ay[i];
    double d0 = relx * nx + rely * ny;
    double vn = ux * nx + uy * ny;
    if (fabs(d0) >= radius) {
      double side = d0 > 0.0 ? 1.0 : -1.0;
      if (vn * side < 0.0) {
        double t = (side * radius - d0) / vn;
        if (0.0 <= t && t <= 1.0) {
          double proj = (relx + t * ux) * tx + (rely + t * uy) * ty;
          if (0.0 <= proj && proj <= seg_len) {
            if (t < best_t) {
              best_t = t;
              best_i = i;
            }
          }
        }
      }
    } else {
      double proj = relx * tx + rely * ty;
      if (0.0 <= proj && proj <= seg_len && vn * d0 < 0.0) {
        if (0.0 < best_t) {
          best_t = 0.0;
          best_i = i;
        }
      }
    }
    for (int e = 0; e < 2; ++e) {
      double cxp = e == 0 ? ax[i] : bx[i];
      double cyp = e == 0 ? ay[i] : by[i];
      double wx = px - cxp, wy = py - cyp;
      double b = wx * ux + wy * uy;
      double c = wx * wx + wy * wy - radius * radius;
      if (c < 0.0) {
        if (b < 0.0 && 0.0 < best_t) {
          best_t = 0.0;
          best_i = i;
        }
        continue;
      }
      if (u2 == 0.0) continue;
      double disc = b * b - u2 * c;
      if (disc < 0.0) continue;
      double t = (-b - sqrt(disc)) / u2;
      if (0.0 <= t && t <= 1.0 && t < best_t) {
        best_t = t;
        best_i = i;
      }
    }
  }
  if (best_i < 0) {
    *t_res = INFINITY;
    *i_res = -1;
    *tan_x = 0.0;
    *tan_y = 0.0;
    return;
  }
  double exi = bx[best_i] - ax[best_i], eyi = by[best_i] - ay[best_i];
  double seg_len = sqrt(exi * exi + eyi * eyi);
  *t_res = best_t;
  *i_res = best_i;
  *tan_x = exi / seg_len;
  *tan_y = eyi / seg_len;
}

/* min_seg_distance, src/_kernels.py:468-493 */
double or_min_seg_distance(double px, double py, const int64_t *cand,
                           int64_t ncand, const double *ax, const double *ay,
                           const double *bx, const double *by) {
  double best = INFINITY;
  for (int64_t q = 0; q < ncand; ++q) {
    int64_t i = cand ? cand[q] : q;
    double exi = bx[i] - ax[i], eyi = by[i] - ay[i];
    double l2 = exi * exi + eyi * eyi;
    double wx = px - ax[i], wy = py - ay[i];
    double cx, cy;
    if (l2 > 0.0) {
      double t = (wx * exi + wy * eyi) / l2;
      if (t < 0.0)
        t = 0.0;
      else if (t > 1.0)
        t = 1.0;
      cx = wx - t * exi;
      cy = wy - t * eyi;
    } else {
      cx = wx;
      cy = wy;
    }
    double d = sqrt(cx * cx + cy * cy);
    if (d < best) best = d;
  }
  return best;
}

/* ------------------------------------------------ scene bundle (context) */

typedef struct {
  int64_t n;
  double *ax, *ay, *bx, *by, *ex, *ey, *nx, *ny, *albedo; /* albedo n*3 */
  uint16_t *sem;
  double x0, y0;
  int64_t gnx, gny;
  int64_t *starts, *items;
  double wall_h, floor_color[3], ceil_color[3];
  /* per-worker scratch of or_batch_step_render, kept across calls (a
     per-call malloc/free of the candidate arrays means mmap/munmap and TLB
     shootdowns in every worker: the baseline would not scale with threads) */
  int npool;
  int64_t pool_w;
  uint8_t **p_mark;
  int64_t **p_cand, **p_isc;
  double **p_scratch;
} or_scene;

/* RenderGeometry.__init__, src/sensors.py:81-93 */
void *or_scene_create(const double *segs, const uint16_t *sem,
                      const double *albedo, int64_t n, double wall_h,
                      const double *floor3, const double *ceil3) {
  or_scene *s = (or_scene *)calloc(1, sizeof(or_scene));
  s->n = n;
  size_t nn = (size_t)(n > 0 ? n : 1);
  s->ax = malloc(nn * 8); s->ay = malloc(nn * 8); s->bx = malloc(nn * 8);
  s->by = malloc(nn * 8); s->ex = malloc(nn * 8); s->ey = malloc(nn * 8);
  s->nx = malloc(nn * 8); s->ny = malloc(nn * 8);
  s->albedo = malloc(nn * 24);
  s->sem = malloc(nn * 2);
  for (int64_t i = 0; i < n; ++i) {
    s->ax[i] = segs[4 * i]; s->ay[i] = segs[4 * i + 1];
    s->bx[i] = segs[4 * i + 2]; s->by[i] = segs[4 * i + 3];
    s->ex[i] = s->bx[i] - s->ax[i]; s->ey[i] = s->by[i] - s->ay[i];
    s->sem[i] = sem[i];
    s->albedo[3 * i] = albedo[3 * i];
    s->albedo[3 * i + 1] = albedo[3 * i + 1];
    s->albedo[3 * i + 2] = albedo[3 * i + 2];
  }
  or_segment_normals(segs, n, s->nx, s->ny);
  or_grid_dims(segs, n, &s->x0, &s->y0, &s->gnx, &s->gny);
  s->starts = malloc(sizeof(int64_t) * (size_t)(s->gnx * s->gny + 1));
  int64_t tot = or_grid_build(segs, n, s->x0, s->y0, s->gnx, s->gny, s->starts, NULL);
  s->items = malloc(sizeof(int64_t) * (size_t)(tot > 0 ? tot : 1));
  or_grid_build(segs, n, s->x0, s->y0, s->gnx, s->gny, s->starts, s->items);
  s->wall_h = wall_h;
  for (int c = 0; c < 3; ++c) {
    s->floor_color[c] = floor3[c];
    s->ceil_color[c] = ceil3[c];
  }
  return s;
}

void or_scene_destroy(void *p) {
  or_scene *s = (or_scene *)p;
  if (!s) return;
  free(s->ax); free(s->ay); free(s->bx); free(s->by); free(s->ex); free(s->ey);
  free(s->nx); free(s->ny); free(s->albedo); free(s->sem);
  free(s->starts); free(s->items);
  for (int k = 0; k < s->npool; ++k) {
    free(s->p_mark[k]); free(s->p_cand[k]); free(s->p_isc[k]); free(s->p_scratch[k]);
  }
  free(s->p_mark); free(s->p_cand); free(s->p_isc); free(s->p_scratch);
  free(s);
}

void or_scene_grid(void *p, double *x0, double *y0, int64_t *nx, int64_t *ny,
                   int64_t *nitems) {
  or_scene *s = (or_scene *)p;
  *x0 = s->x0; *y0 = s->y0; *nx = s->gnx; *ny = s->gny;
  *nitems = s->starts[s->gnx * s->gny];
}

void or_scene_grid_copy(void *p, int64_t *starts, int64_t *items) {
  or_scene *s = (or_scene *)p;
  int64_t nc = s->gnx * s->gny;
  memcpy(starts, s->starts, sizeof(int64_t) * (size_t)(nc + 1));
  memcpy(items, s->items, sizeof(int64_t) * (size_t)s->starts[nc]);
}

/* SegmentIndex.cast_disc, src/geometry.py:183-192 */
static void scene_cast_disc(const or_scene *s, double px, double py, double ux,
                            double uy, double radius, uint8_t *mark,
                            int64_t *cand, double *t, int64_t *i, double *tx,
                            double *ty) {
  double pad = radius + 1e-6;
  double xa = px + ux, ya = py + uy;
  int64_t m = or_query_aabb((px < xa ? px : xa) - pad, (py < ya ? py : ya) - pad,
                            (px > xa ? px : xa) + pad, (py > ya ? py : ya) + pad,
                            s->x0, s->y0, s->gnx, s->gny, s->starts, s->items,
                            s->n, mark, cand);
  or_disc_cast(px, py, ux, uy, radius, cand, m, s->ax, s->ay, s->bx, s->by, t, i,
               tx, ty);
}

void or_cast_disc(void *p, double px, double py, double ux, double uy,
                  double radius, double *t, int64_t *i, double *tx, double *ty) {
  or_scene *s = (or_scene *)p;
  size_t nn = (size_t)(s->n > 0 ? s->n : 1);
  uint8_t *mark = calloc(nn, 1);
  int64_t *cand = malloc(nn * 8);
  scene_cast_disc(s, px, py, ux, uy, radius, mark, cand, t, i, tx, ty);
  free(mark);
  free(cand);
}

/* SegmentIndex.clearance, src/geometry.py:194-206 */
static double scene_clearance(const or_scene *s, double px, double py,
                              double search_radius, uint8_t *mark,
                              int64_t *cand) {
  int64_t m = or_query_aabb(px - search_radius, py - search_radius,
                            px + search_radius, py + search_radius, s->x0, s->y0,
                            s->gnx, s->gny, s->starts, s->items, s->n, mark, cand);
  if (m > 0) {
    double d = or_min_seg_distance(px, py, cand, m, s->ax, s->ay, s->bx, s->by);
    if (d <= search_radius) return d;
  }
  if (s->n == 0) return INFINITY;
  return or_min_seg_distance(px, py, NULL, s->n, s->ax, s->ay, s->bx, s->by);
}

double or_clearance(void *p, double px, double py, double search_radius) {
  or_scene *s = (or_scene *)p;
  size_t nn = (size_t)(s->n > 0 ? s->n : 1);
  uint8_t *mark = calloc(nn, 1);
  int64_t *cand = malloc(nn * 8);
  double d = scene_clearance(s, px, py, search_radius, mark, cand);
  free(mark);
  free(cand);
  return d;
}

void or_scene_raycast(void *p, double px, double py, const double *dirx,
                      const double *diry, int64_t m, double t_max, int brute,
                      double *t_out, int64_t *i_out) {
  or_scene *s = (or_scene *)p;
  if (brute)
    or_raycast_all(px, py, dirx, diry, m, s->ax, s->ay, s->ex, s->ey, s->n, t_out,
                   i_out);
  else
    or_raycast_grid(px, py, dirx, diry, m, s->x0, s->y0, CELL, s->gnx, s->gny,
                    s->starts, s->items, s->ax, s->ay, s->ex, s->ey, t_max, t_out,
                    i_out);
}

/* ------------------------------------------------------------ kinematics */

/* wrap_angle, src/geometry.py:19-24 */
double or_wrap_angle(double theta) {
  double out = fmod(theta + M_PI, 2.0 * M_PI);
  if (out <= 0.0) out += 2.0 * M_PI;
  return out - M_PI;
}

typedef struct {
  double x, y, heading, path_len;
  int64_t collisions;
} or_agent;

/* apply_forward, src/sim.py:90-130.  Returns collided; *moved = displacement */
static int scene_forward(const or_scene *s, or_agent *a, double radius,
                         double step, uint8_t *mark, int64_t *cand,
                         double *moved_out) {
  double ux = step * cos(a->heading), uy = step * sin(a->heading);
  double px = a->x, py = a->y;
  double t1, tx, ty;
  int64_t i1;
  scene_cast_disc(s, px, py, ux, uy, radius, mark, cand, &t1, &i1, &tx, &ty);
  double nx_, ny_, moved;
  int collided;
  if (!(t1 < 1.0)) {
    nx_ = px + ux;
    ny_ = py + uy;
    moved = step;
    collided = 0;
  } else {
    double d1 = t1 * step - CONTACT_EPSILON;
    if (!(d1 > 0.0)) d1 = 0.0; /* max(0.0, x) returns 0.0 unless x > 0 */
    double unx = ux / step, uny = uy / step;
    double p1x = px + unx * d1, p1y = py + uny * d1;
    double remx = ux * (1.0 - t1), remy = uy * (1.0 - t1);
    double dot = fma(remy, ty, remx * tx); /* np.dot (OpenBLAS ddot) */
    double slx = dot * tx, sly = dot * ty;
    double slide_len = hypot(slx, sly);
    double d2 = 0.0;
    if (slide_len > CONTACT_EPSILON) {
      double t2, t2x, t2y;
      int64_t i2;
      scene_cast_disc(s, p1x, p1y, slx, sly, radius, mark, cand, &t2, &i2, &t2x,
                      &t2y);
      if (!(t2 < 1.0)) {
        d2 = slide_len;
      } else {
        d2 = t2 * slide_len - CONTACT_EPSILON;
        if (!(d2 > 0.0)) d2 = 0.0;
      }
      p1x = p1x + (slx / slide_len) * d2;
      p1y = p1y + (sly / slide_len) * d2;
    }
    nx_ = p1x;
    ny_ = p1y;
    moved = d1 + d2;
    collided = 1;
  }
  a->x = nx_;
  a->y = ny_;
  a->path_len = a->path_len + moved;
  a->collisions += collided;
  *moved_out = moved;
  return collided;
}

/* Simulator.step action dispatch, src/sim.py:202-219.
 * action: 0 MOVE_FORWARD, 1 TURN_LEFT, 2 TURN_RIGHT, 3 STOP (Action order,
 * src/sim.py:31-35).  turn_rad = math.radians(turn_angle) from the host. */
int or_step(void *p, double *x, double *y, double *heading, double *path_len,
            int64_t *collisions, int action, double radius, double step,
            double turn_rad, double *moved) {
  or_scene *s = (or_scene *)p;
  or_agent a = {*x, *y, *heading, *path_len, *collisions};
  int collided = 0;
  *moved = 0.0;
  if (action == 0) {
    size_t nn = (size_t)(s->n > 0 ? s->n : 1);
    uint8_t *mark = calloc(nn, 1);
    int64_t *cand = malloc(nn * 8);
    collided = scene_forward(s, &a, radius, step, mark, cand, moved);
    free(mark);
    free(cand);
  } else if (action == 1) {
    a.heading = or_wrap_angle(a.heading + turn_rad);
  } else if (action == 2) {
    a.heading = or_wrap_angle(a.heading + (-turn_rad));
  }
  *x = a.x; *y = a.y; *heading = a.heading; *path_len = a.path_len;
  *collisions = a.collisions;
  return collided;
}

/* sensors.render for one camera group, src/sensors.py:105-152 (indexed path,
 * t_max = 1e9 default of SegmentIndex.raycast, src/geometry.py:165) */
static void scene_render(const or_scene *s, double px, double py, double heading,
                         double sensor_h, int64_t W, int64_t H, double focal,
                         double max_range, double t_max, int brute,
                         double *scratch /* 4*W doubles */, int64_t *iscratch,
                         double *depth, double *rgb, uint16_t *sem) {
  double *dirx = scratch, *diry = scratch + W, *tcol = scratch + 2 * W;
  or_column_directions(heading, W, focal, dirx, diry);
  if (brute)
    or_raycast_all(px, py, dirx, diry, W, s->ax, s->ay, s->ex, s->ey, s->n, tcol,
                   iscratch);
  else
    or_raycast_grid(px, py, dirx, diry, W, s->x0, s->y0, CELL, s->gnx, s->gny,
                    s->starts, s->items, s->ax, s->ay, s->ex, s->ey, t_max, tcol,
                    iscratch);
  or_fill_frame(tcol, iscratch, H, W, focal, sensor_h, s->wall_h, max_range,
                s->albedo, s->sem, s->nx, s->ny, dirx, diry, s->floor_color,
                s->ceil_color, depth, rgb, sem);
}

void or_render(void *p, double px, double py, double heading, double sensor_h,
               int64_t W, int64_t H, double focal, double max_range, double t_max,
               int brute, double *depth, double *rgb, uint16_t *sem) {
  or_scene *s = (or_scene *)p;
  double *scratch = malloc(sizeof(double) * 4 * (size_t)W);
  int64_t *isc = malloc(sizeof(int64_t) * (size_t)W);
  scene_render(s, px, py, heading, sensor_h, W, H, focal, max_range, t_max, brute,
               scratch, isc, depth, rgb, sem);
  free(scratch);
  free(isc);
}

/* EpisodeFrame.to_frame + gps_compass, src/sensors.py:163-180 */
void or_gps_compass(double x, double y, double heading, double ox, double oy,
                    double oh, double *gps2, double *compass) {
  double dx = x - ox, dy = y - oy;
  double c = cos(-oh), s = sin(-oh);
  gps2[0] = c * dx - s * dy;
  gps2[1] = s * dx + c * dy;
  *compass = or_wrap_angle(heading - oh);
}

/* Batched CPU baseline: N independent Simulator.step calls (src/sim.py:202)
 * followed by observations() (src/sim.py:192), envs pulled from a shared
 * counter by nthreads pthreads -- the same per-env work the reference's forked
 * bench workers do (src/bench.py:122-144).  Frames are written into per-env
 * f64/u16 buffers like fill_frame's outputs (src/sensors.py:136-138). */
typedef struct {
  or_scene *s;
  int64_t N;
  double *x, *y, *heading, *path_len;
  int64_t *collisions;
  const int8_t *actions;
  double radius, step, turn_rad, sensor_h, focal, max_range;
  int64_t W, H;
  double *depth, *rgb;
  uint16_t *sem;
  int64_t next; /* atomic work counter */
  int per_thread; /* frames: one per worker thread (reused), not one per env */
} or_batch_job;

typedef struct {
  or_batch_job *j;
  int64_t tid;
} or_batch_arg;

static void *batch_worker(void *arg) {
  or_batch_job *j = ((or_batch_arg *)arg)->j;
  const int64_t tid = ((or_batch_arg *)arg)->tid;
  or_scene *s = j->s;
  uint8_t *mark = s->p_mark[tid];
  int64_t *cand = s->p_cand[tid];
  double *scratch = s->p_scratch[tid];
  int64_t *isc = s->p_isc[tid];
  size_t px = (size_t)(j->W * j->H);
  for (;;) {
    int64_t e = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (e >= j->N) break;
    or_agent a = {j->x[e], j->y[e], j->heading[e], j->path_len[e],
                  j->collisions[e]};
    int act = j->actions[e];
    double moved;
    if (act == 0)
      scene_forward(s, &a, j->radius, j->step, mark, cand, &moved);
    else if (act == 1)
      a.heading = or_wrap_angle(a.heading + j->turn_rad);
    else if (act == 2)
      a.heading = or_wrap_angle(a.heading + (-j->turn_rad));
    j->x[e] = a.x; j->y[e] = a.y; j->heading[e] = a.heading;
    j->path_len[e] = a.path_len; j->collisions[e] = a.collisions;
    const size_t f = (size_t)(j->per_thread ? tid : e);  /* frame slot */
    scene_render(s, a.x, a.y, a.heading, j->sensor_h, j->W, j->H, j->focal,
                 j->max_range, 1e9, 0, scratch, isc,
                 j->depth ? j->depth + px * f : NULL,
                 j->rgb ? j->rgb + 3 * px * f : NULL,
                 j->sem ? j->sem + px * f : NULL);
  }
  return NULL;
}

/* per-thread scratch for nthreads workers and width W (grown, never shrunk) */
static void scratch_pool(or_scene *s, int nthreads, int64_t W) {
  size_t nn = (size_t)(s->n > 0 ? s->n : 1);
  if (nthreads <= s->npool && W <= s->pool_w) return;
  for (int k = 0; k < s->npool; ++k) {
    free(s->p_mark[k]); free(s->p_cand[k]); free(s->p_isc[k]); free(s->p_scratch[k]);
  }
  free(s->p_mark); free(s->p_cand); free(s->p_isc); free(s->p_scratch);
  int np = nthreads > s->npool ? nthreads : s->npool;
  int64_t w = W > s->pool_w ? W : s->pool_w;
  s->p_mark = malloc(sizeof(uint8_t *) * (size_t)np);
  s->p_cand = malloc(sizeof(int64_t *) * (size_t)np);
  s->p_isc = malloc(sizeof(int64_t *) * (size_t)np);
  s->p_scratch = malloc(sizeof(double *) * (size_t)np);
  for (int k = 0; k < np; ++k) {
    s->p_mark[k] = calloc(nn, 1);  /* scene_forward leaves it all zero again */
    s->p_cand[k] = malloc(nn * 8);
    s->p_isc[k] = malloc(sizeof(int64_t) * (size_t)w);
    s->p_scratch[k] = malloc(sizeof(double) * 4 * (size_t)w);
  }
  s->npool = np;
  s->pool_w = w;
}

void or_batch_step_render(void *p, int64_t N, double *x, double *y,
                          double *heading, double *path_len, int64_t *collisions,
                          const int8_t *actions, double radius, double step,
                          double turn_rad, double sensor_h, int64_t W, int64_t H,
                          double focal, double max_range, double *depth,
                          double *rgb, uint16_t *sem, int nthreads, int per_thread) {
  /* per_thread != 0: depth/rgb/sem hold one frame per worker thread, reused
     for every env the thread steps -- the memory behaviour of the
     reference's bench workers (one env per process, bench.py:128-137, whose
     fresh per-call frame arrays reuse the same freed block) */
  or_batch_job j = {(or_scene *)p, N, x, y, heading, path_len, collisions,
                    actions, radius, step, turn_rad, sensor_h, focal, max_range,
                    W, H, depth, rgb, sem, 0, per_thread};
  if (nthreads < 1) nthreads = 1;
  scratch_pool((or_scene *)p, nthreads, W);
  pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
  or_batch_arg *args = malloc(sizeof(or_batch_arg) * (size_t)nthreads);
  for (int k = 0; k < nthreads; ++k) {
    args[k].j = &j;
    args[k].tid = k;
  }
  for (int k = 1; k < nthreads; ++k) pthread_create(&th[k], NULL, batch_worker, &args[k]);
  batch_worker(&args[0]);
  for (int k = 1; k < nthreads; ++k) pthread_join(th[k], NULL);
  free(th);
  free(args);
}

/* ---------------------------------------------- CPU baseline harness (bench)
 * The reference harness's cell (bench.py:128-177): `nthreads` workers, each
 * stepping ONE env (its own start pose, its own column of the action table)
 * with Simulator.step + observations for `seconds`, rendering into its own
 * reused frame, released together by a barrier; aggregate frames/s =
 * sum(frames) / (max end - min start) (bench.py:170-174).  Threads stand in
 * for the harness's forked processes (no shared mutable state). */
#include <time.h>

typedef struct {
  or_scene *s;
  int64_t N, n_steps;
  const double *x0, *y0, *h0;
  const int8_t *actions; /* n_steps x N */
  double radius, step, turn_rad, sensor_h, focal, max_range, seconds;
  int64_t W, H;
  int want_rgb, want_depth, want_sem;
  pthread_barrier_t bar;
} or_cell_job;

typedef struct {
  or_cell_job *j;
  int64_t wid;
  double t0, t1;
  int64_t frames;
} or_cell_arg;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void *cell_worker(void *arg) {
  or_cell_arg *w = (or_cell_arg *)arg;
  or_cell_job *j = w->j;
  or_scene *s = j->s;
  size_t nn = (size_t)(s->n > 0 ? s->n : 1);
  size_t px = (size_t)(j->W * j->H);
  uint8_t *mark = calloc(nn, 1);
  int64_t *cand = malloc(nn * 8);
  double *scratch = malloc(sizeof(double) * 4 * (size_t)j->W);
  int64_t *isc = malloc(sizeof(int64_t) * (size_t)j->W);
  double *depth = j->want_depth ? malloc(sizeof(double) * px) : NULL;
  double *rgb = j->want_rgb ? malloc(sizeof(double) * 3 * px) : NULL;
  uint16_t *sem = j->want_sem ? malloc(sizeof(uint16_t) * px) : NULL;
  const int64_t e = w->wid % j->N;
  or_agent a = {j->x0[e], j->y0[e], or_wrap_angle(j->h0[e]), 0.0, 0};
  pthread_barrier_wait(&j->bar);
  w->t0 = now_s();
  int64_t k = 0;
  for (;; ++k) {
    const int act = j->actions[(k % j->n_steps) * j->N + e];
    double moved;
    if (act == 0)
      scene_forward(s, &a, j->radius, j->step, mark, cand, &moved);
    else if (act == 1)
      a.heading = or_wrap_angle(a.heading + j->turn_rad);
    else if (act == 2)
      a.heading = or_wrap_angle(a.heading + (-j->turn_rad));
    scene_render(s, a.x, a.y, a.heading, j->sensor_h, j->W, j->H, j->focal, j->max_range, 1e9,
                 0, scratch, isc, depth, rgb, sem);
    if ((k & 7) == 7 && now_s() - w->t0 >= j->seconds) break;
  }
  w->t1 = now_s();
  w->frames = k + 1;
  free(mark); free(cand); free(scratch); free(isc); free(depth); free(rgb); free(sem);
  return NULL;
}

double or_bench_cell(void *p, int64_t N, const double *x0, const double *y0, const double *h0,
                     const int8_t *actions, int64_t n_steps, double radius, double step,
                     double turn_rad, double sensor_h, int64_t W, int64_t H, double focal,
                     double max_range, int want_rgb, int want_depth, int want_sem,
                     int nthreads, double seconds, int64_t *frames_out) {
  if (nthreads < 1) nthreads = 1;
  or_cell_job j = {(or_scene *)p, N, n_steps, x0, y0, h0, actions, radius, step, turn_rad,
                   sensor_h, focal, max_range, seconds, W, H, want_rgb, want_depth, want_sem};
  pthread_barrier_init(&j.bar, NULL, (unsigned)nthreads);
  pthread_t *th = malloc(sizeof(pthread_t) * (size_t)nthreads);
  or_cell_arg *args = calloc((size_t)nthreads, sizeof(or_cell_arg));
  for (int k = 0; k < nthreads; ++k) {
    args[k].j = &j;
    args[k].wid = k;
  }
  for (int k = 1; k < nthreads; ++k) pthread_create(&th[k], NULL, cell_worker, &args[k]);
  cell_worker(&args[0]);
  for (int k = 1; k < nthreads; ++k) pthread_join(th[k], NULL);
  double t0 = args[0].t0, t1 = args[0].t1;
  int64_t frames = 0;
  for (int k = 0; k < nthreads; ++k) {
    if (args[k].t0 < t0) t0 = args[k].t0;
    if (args[k].t1 > t1) t1 = args[k].t1;
    frames += args[k].frames;
  }
  pthread_barrier_destroy(&j.bar);
  free(th);
  free(args);
  if (frames_out) *frames_out = frames;
  return (double)frames / (t1 - t0);
}
