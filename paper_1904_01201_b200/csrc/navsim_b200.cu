// navsim_b200.cu -- host side of the C ABI (include/navsim_b200.h).
//
// Scene upload builds the reference's uniform grid on the host exactly like
// SegmentIndex.__init__ (geometry.py:109-141), expands bucket items into
// contiguous CellEntry runs, and uploads everything once.  Per-step calls
// only enqueue kernels on the caller's stream (no host synchronisation).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/navsim_b200.h"
#include "device.cuh"
#include "exact_math.cuh"
#include "kernels.cuh"
#include "nav.cuh"
#include "codec.cuh"

using namespace nvd;

// Compile-time study switches (A/B builds with -D...).  The shipped library
// is built with these defaults; its behaviour does not depend on the
// environment.  A/B numbers: profiles/r01_fill_ab_history.json, DESIGN.md.
#ifndef NV_CAST_WARP_RAYS
#define NV_CAST_WARP_RAYS 16384  // batches with at most this many rays cast one warp per ray
#endif
#ifndef NV_CAST_BLOCK
#define NV_CAST_BLOCK 64  // threads per CTA of the thread-per-ray cast (C3: 64 95.3 / 128 95.7 / 32 96.0 us per step with the 4-warp block-order kernel)
#endif
#ifndef NV_CAST_LPT
#define NV_CAST_LPT 1  // longest-first order of the cast's blocks (C3 -2 us/step)
#endif
#ifndef NV_WS_NW
#define NV_WS_NW 16  // producer warps of the ws writer (4 / 8 / 16)
#endif
#ifndef NV_FILL_PDL
#define NV_FILL_PDL 1  // the ws writer is a programmatic dependent of the column cast
#endif
#ifndef NV_FILL_RELEASE
#define NV_FILL_RELEASE 1  // the writer takes each env as soon as its casts are done
#endif
#ifndef NV_AGENT_BLOCK
#define NV_AGENT_BLOCK 32  // threads per CTA of the agent step (a warp per env; one-warp CTAs fit beside a writer CTA)
#endif
#ifndef NV_STEP_CHAIN
#define NV_STEP_CHAIN 1  // the agent step is a programmatic dependent of the previous frame writer
#endif
#ifndef NV_WS_SLOTS
#define NV_WS_SLOTS 0  // ring slots of the ws writer (0: as many as fit, <= 4)
#endif
#ifndef NV_WS_TAB
#define NV_WS_TAB 0  // 1: stage the shading table in shared memory
#endif
#ifndef NV_WS_BANDS
#define NV_WS_BANDS 0  // row bands per env frame (0: cost model)
#endif
#ifndef NV_WS_RPW
#define NV_WS_RPW 0  // rows per producer warp per slot (0: auto)
#endif
#ifndef NV_E2E_MAPPED
#define NV_E2E_MAPPED 1  // host-buffer step: kernels read actions / write results in mapped pinned memory
#endif
#ifndef NV_READY_BY_HALF
#define NV_READY_BY_HALF 1  // release mode: per-warp ready waits, flags per record half reset by the writer
#endif
#ifndef NV_POSE_REC
#define NV_POSE_REC 1  // release-mode handshake through per-env pose records (else ready flags)
#endif
#ifndef NV_TASK_PDL
#define NV_TASK_PDL 1  // task-layer step: the task cast as the agent step's programmatic dependent
#endif
#ifndef NV_E2E_ACT_COPY
#define NV_E2E_ACT_COPY 0  // mapped host step: copy the actions in (a graph copy node) instead of reading them over PCIe
#endif
#ifndef NV_E2E_PINGPONG
#define NV_E2E_PINGPONG 1  // host-buffer steps alternate two graphs / streams / frame sets
#endif
#ifndef NV_NAV_HOSTLOOP
#define NV_NAV_HOSTLOOP 0  // 1: distance-field relaxation as host-driven launches
#endif

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(NV_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                             \
  } while (0)

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  int alloc(size_t b) {
    if (b <= bytes && p) return NV_OK;
    release();
    if (b == 0) b = 16;
    if (cudaMalloc(&p, b) != cudaSuccess) {
      cudaGetLastError();
      return fail(NV_ERR_OOM, "cudaMalloc(%zu) failed", b);
    }
    bytes = b;
    return NV_OK;
  }
  template <class T>
  T *as() const { return reinterpret_cast<T *>(p); }
};

#define TRY(x)               \
  do {                       \
    int r_ = (x);            \
    if (r_ != NV_OK) return r_; \
  } while (0)

template <class T>
int upload(DevBuf &b, const std::vector<T> &v) {
  TRY(b.alloc(sizeof(T) * std::max<size_t>(v.size(), 1)));
  if (!v.empty()) CK(cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
  return NV_OK;
}

struct Camera {
  bool on = false;
  int W = 0, H = 0;
  double focal = 0, max_range = 0;
  int n_top = 0, b0 = 0;
  float ktop = 0.f, kbot = 0.f;
  double tables_cam_h = NAN;
  DevBuf u, tc, tf, rows, invh;
  DevBuf rec;      // ColRec, two halves of N x W (A then B planes each): consecutive
                   // renders alternate (rec_flip), so a step's casts never write
                   // the records the previous step's writer may still read
  int rec_half = 0;
  // per-env release counts (cast -> writer), one set per record half:
  // [half][done N | consumed N], then the fault flag; zero between steps
  DevBuf rel, rel_e2e;
  int64_t rel_n = -1, rel_n_e2e = -1;
  DevBuf lpt_order, lpt_cost;  // thread-per-ray cast: block order (slowest first) + durations
  int64_t lpt_n = -1;           // blocks the order is valid for
  // The host-buffer step's own record buffer and block order (its frame
  // writer may still run after nv_step_render_host returns, concurrently with
  // device steps on other streams) and its device frames (nv_host_frames).
  DevBuf rec_e2e, lpt_order_e2e, lpt_cost_e2e;
  int64_t lpt_n_e2e = -1;
  // two frame sets: consecutive host steps alternate (NV_E2E_PINGPONG), so a
  // step's writer never writes the frames the previous step's writer may
  // still be writing
  DevBuf e_rgb[2], e_depth[2], e_sem[2];
};

}  // namespace

struct nv_ctx {
  int device = 0;
  int sm_count = 148;
  int max_smem_optin = 0;
  // scene
  bool has_scene = false;
  int64_t n = 0;
  double wall_h = 2.5;
  double floor3[3] = {0.35, 0.33, 0.30}, ceil3[3] = {0.85, 0.85, 0.85};
  double gx0 = -0.5, gy0 = -0.5;
  int gnx = 1, gny = 1;
  int64_t nitems = 0;
  DevBuf ax, ay, bx, by, ex, ey, nx, ny, sem, alb, starts, ent, items, entf, entm, cells, chunks;
  DevBuf dent, stx, sty;
  // agent
  double radius = 0.1, step = 0.25, turn_rad = 0.17453292519943295, sensor_h = 1.5;
  // envs
  // navigation grid (nv_nav_build) and PointGoal task state (nv_task_*)
  bool has_nav = false;
  int nav_nx = 0, nav_ny = 0;
  double nav_ox = 0, nav_oy = 0, nav_res = 0, nav_radius = 0;
  DevBuf nav_mask, nav_dist, nav_tmp0, nav_tmp1, nav_flag;
  double sbounds[4] = {0, 0, 0, 0};  // Scene.bounds of the uploaded segments
  bool task_on = false;
  int t_max_steps = 500;
  double t_success_radius = 0.2, t_success_reward = 10.0, t_step_penalty = -0.01;
  DevBuf t_goal, t_gdsp, t_fid, t_dlast, t_steps, t_done, t_status;
  const double *t_fields = nullptr;
  int64_t t_nfields = 0;
  double noise_sigma = 0.0;  // inverse-depth noise (nv_depth_noise)
  unsigned long long noise_seed = 0, noise_frame = 0;
  long long noise_env_offset = 0;
  int64_t n_envs = 0;
  DevBuf x, y, h, path, coll, ch, sh, ox, oy, oh, fc, fs, reset;
  Camera cams[8];
  // host-buffer (e2e) path scratch
  DevBuf e_act, e_pack;  // e_pack: gps 16N | compass 8N | disp 8N | coll N
  // host-buffer path as one CUDA graph: H2D actions -> step+render -> one D2H
  // of the packed step results, replayed while (cam, channels, N) stay fixed
  // Two host-step graphs on two streams, used alternately (NV_E2E_PINGPONG):
  // graph p renders into record half / frame set p, so step t+1's agent step
  // and casts (stream 1-p) need only step t's casts, not its frame writer --
  // they take the SMs the writer frees, as in one long graph
  cudaStream_t e_stream[2] = {nullptr, nullptr};
  cudaEvent_t e_ev = nullptr;
  cudaEvent_t e_cast_ev[2] = {nullptr, nullptr};  // recorded in graph p after the casts
  int e_par = 0;   // graph of the next host step
  int e_last = 0;  // frame set of the last host step (nv_host_frames)
  cudaEvent_t mid_ev = nullptr;     // nv_step_render records it after the casts (capture only)
  bool e_pending = false;           // a host step's frame writer may still be running
  cudaStream_t o_stream = nullptr;  // side stream of the ordering kernel (beside the writer)
  cudaEvent_t o_ev0 = nullptr, o_ev1 = nullptr;
  // capture only: a branch of its own for the host event after the casts (the
  // ordering kernel's branch would hold it back by that kernel's duration),
  // and the event recorded after the ordering kernel (the next host step's
  // casts read its order)
  cudaStream_t m_stream = nullptr;
  cudaEvent_t m_ev0 = nullptr, m_ev1 = nullptr;
  cudaEvent_t order_ev = nullptr;
  cudaEvent_t e_order_ev[2] = {nullptr, nullptr};
  bool o_fork = false;              // an ordering kernel was forked in this step
  cudaGraphExec_t e_graph[2] = {nullptr, nullptr};
  std::vector<uint64_t> e_key;  // everything the captured graph depends on (HostStepKey)
  void *e_out_host[4] = {nullptr, nullptr, nullptr, nullptr};  // last caller buffers
  void *e_out_dev[4] = {nullptr, nullptr, nullptr, nullptr};   // their device aliases
  int64_t gen = 0;  // bumped by every call that changes kernel arguments (graph key)
  void *e_hin = nullptr, *e_hout = nullptr;  // pinned staging (actions in, packed results out)
  size_t e_hin_bytes = 0, e_hout_bytes = 0;
  int64_t launches = 0;
  int cast_mode = NV_CAST_AUTO;  // nv_set_cast_mode (include/navsim_b200.h)
  bool e2e_mapped = NV_E2E_MAPPED != 0;  // host-buffer graph path: zero-copy actions / results
  bool pdl = true;           // agent step -> cast programmatic dependent launch (nv_set_overlap)
  bool pdl_armed = false, pdl_init = false;
  // flags of the armed agent -> cast handshake: ready (per env), arrive
  // (nullptr in release mode: the writer resets the flags), fault
  unsigned *pdl_cur_ready = nullptr, *pdl_cur_arrive = nullptr;
  unsigned *fill_ready = nullptr;  // ready flags the next release writer resets
  // pose records of the release-mode handshake (NV_POSE_REC): [half][env][8]
  DevBuf pose_rec;
  bool pose_init = false;
  // the host-buffer step's own handshake buffers (its writer may still run
  // beside device steps on other streams; swapped in around its captures)
  DevBuf pdl_ready_e2e, pdl_arrive_e2e, pose_rec_e2e;
  bool pdl_init_e2e = false, pose_init_e2e = false;
  double *pdl_cur_posrec = nullptr, *fill_posrec = nullptr;
  // the last ws writer launched: its stream and whether its grid filled the
  // GPU (one CTA on every SM) -- only then may the next agent step work
  // beside it (do_step)
  cudaStream_t ws_tail_stream = nullptr;
  bool ws_tail_full = false;
  bool fill_pdl = false;  // the next ws writer launch follows its column cast (launch_ws_kernel)
  DevBuf pdl_ready, pdl_arrive;
  // dynamic shared memory opted in per kernel on this context's device
  std::unordered_map<const void *, size_t> smem_cfg;
  int fill_mode = NV_FILL_AUTO;  // nv_set_fill_mode
  // optional per-kernel CUDA-event timing (bench roofline evidence)
  bool prof_on = false;
  std::vector<cudaEvent_t> prof_ev;   // pool, pairs
  std::vector<int> prof_kind;         // kind per pair in use
  size_t prof_used = 0;               // pairs in use
  double prof_ms[4] = {0, 0, 0, 0};
  int64_t prof_n[4] = {0, 0, 0, 0};
  ~nv_ctx() {
    for (auto e : prof_ev) cudaEventDestroy(e);
    for (int p = 0; p < 2; ++p) {
      if (e_graph[p]) cudaGraphExecDestroy(e_graph[p]);
      if (e_cast_ev[p]) cudaEventDestroy(e_cast_ev[p]);
      if (e_stream[p]) cudaStreamDestroy(e_stream[p]);
    }
    if (e_ev) cudaEventDestroy(e_ev);
    if (o_ev0) cudaEventDestroy(o_ev0);
    if (o_ev1) cudaEventDestroy(o_ev1);
    if (o_stream) cudaStreamDestroy(o_stream);
    if (m_ev0) cudaEventDestroy(m_ev0);
    if (m_ev1) cudaEventDestroy(m_ev1);
    if (m_stream) cudaStreamDestroy(m_stream);
    for (int p = 0; p < 2; ++p)
      if (e_order_ev[p]) cudaEventDestroy(e_order_ev[p]);
    if (e_hin) cudaFreeHost(e_hin);
    if (e_hout) cudaFreeHost(e_hout);
  }
  // launch config
  SceneView scene_view() const {
    SceneView v;
    v.ax = ax.as<double>(); v.ay = ay.as<double>(); v.bx = bx.as<double>();
    v.by = by.as<double>(); v.ex = ex.as<double>(); v.ey = ey.as<double>();
    v.nx = nx.as<double>(); v.ny = ny.as<double>();
    v.sem = sem.as<uint16_t>(); v.alb255 = alb.as<float4>();
    v.starts = starts.as<int32_t>(); v.ent = ent.as<CellEntry>(); v.items = items.as<int32_t>();
    v.entf = entf.as<float4>(); v.entm = entm.as<float4>(); v.cells = cells.as<int4>();
    v.chunks = chunks.as<float4>();
    v.dent = dent.as<DiscEntry>(); v.stx = stx.as<double>(); v.sty = sty.as<double>();
    v.x0 = gx0; v.y0 = gy0; v.gnx = gnx; v.gny = gny; v.n = n;
    return v;
  }
  EnvView env_view() const {
    EnvView v;
    v.x = x.as<double>(); v.y = y.as<double>(); v.h = h.as<double>(); v.path = path.as<double>();
    v.coll = coll.as<int64_t>(); v.ch = ch.as<double>(); v.sh = sh.as<double>();
    v.ox = ox.as<double>(); v.oy = oy.as<double>(); v.oh = oh.as<double>();
    v.fc = fc.as<double>(); v.fs = fs.as<double>(); v.reset = reset.as<uint8_t>();
    v.frozen = task_on ? t_done.as<uint8_t>() : nullptr;
    v.n = (int)n_envs;
    return v;
  }
};

namespace {

// --------------------------------------------------------------- grid build
// Exact restatement of SegmentIndex.__init__ (geometry.py:109-141).
int64_t cell_coord_h(double v, double o, int64_t n) {
  double d = (v - o) / 1.0;
  if (!(d >= 1.0)) return 0;
  if (d >= (double)(n - 1)) return n - 1;
  return (int64_t)d;
}

struct HostGrid {
  double x0, y0;
  int64_t nx, ny;
  std::vector<int64_t> starts, items;
};

HostGrid build_grid(const double *segs, int64_t n) {
  HostGrid g;
  double x1, y1;
  if (n > 0) {
    double mnx = INFINITY, mny = INFINITY, mxx = -INFINITY, mxy = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      const double *s = segs + 4 * i;
      mnx = std::min(mnx, std::min(s[0], s[2]));
      mny = std::min(mny, std::min(s[1], s[3]));
      mxx = std::max(mxx, std::max(s[0], s[2]));
      mxy = std::max(mxy, std::max(s[1], s[3]));
    }
    g.x0 = mnx - 0.5; g.y0 = mny - 0.5; x1 = mxx + 0.5; y1 = mxy + 0.5;
  } else {
    g.x0 = g.y0 = -0.5; x1 = y1 = 0.5;
  }
  g.nx = std::max<int64_t>(1, (int64_t)std::ceil((x1 - g.x0) / 1.0));
  g.ny = std::max<int64_t>(1, (int64_t)std::ceil((y1 - g.y0) / 1.0));
  const int64_t nc = g.nx * g.ny;
  std::vector<int64_t> cnt(nc + 1, 0);
  auto range = [&](int64_t i, int64_t &cx0, int64_t &cy0, int64_t &cx1, int64_t &cy1) {
    const double *s = segs + 4 * i;
    cx0 = cell_coord_h(std::min(s[0], s[2]), g.x0, g.nx);
    cy0 = cell_coord_h(std::min(s[1], s[3]), g.y0, g.ny);
    cx1 = cell_coord_h(std::max(s[0], s[2]), g.x0, g.nx);
    cy1 = cell_coord_h(std::max(s[1], s[3]), g.y0, g.ny);
  };
  for (int64_t i = 0; i < n; ++i) {
    int64_t a, b, c, d;
    range(i, a, b, c, d);
    for (int64_t cy = b; cy <= d; ++cy)
      for (int64_t cx = a; cx <= c; ++cx) cnt[cy * g.nx + cx + 1]++;
  }
  for (int64_t c = 0; c < nc; ++c) cnt[c + 1] += cnt[c];
  g.starts = cnt;
  g.items.assign(cnt[nc], 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t a, b, c, d;
    range(i, a, b, c, d);
    for (int64_t cy = b; cy <= d; ++cy)
      for (int64_t cx = a; cx <= c; ++cx) g.items[cnt[cy * g.nx + cx]++] = i;
  }
  return g;
}

int ensure_scene(nv_ctx *c) {
  if (!c->has_scene) return fail(NV_ERR_STATE, "no scene uploaded (nv_scene_upload)");
  return NV_OK;
}
int ensure_envs(nv_ctx *c) {
  TRY(ensure_scene(c));
  if (c->n_envs <= 0) return fail(NV_ERR_STATE, "no envs allocated (nv_envs_alloc)");
  return NV_OK;
}

uint16_t f2h(float x) { return __half_as_ushort(__float2half_rn(x)); }
uint32_t h2splat(float x) {
  uint32_t h = f2h(x);
  return h | (h << 16);
}

// Row tables for a camera (fill_frame's per-row quantities, _kernels.py:141,
// 150, 158): v, tc, tf in exact f64 (host IEEE, no contraction); the f16
// shading table invh[i][j] = 1/sqrt(|d_j|^2 + v_i^2), |d_j|^2 = 1 + u_j^2
// (column directions have unit forward component, sensors.py:96-102), is the
// same for every env and heading; rows i >= ceil(H/2) mirror row H-1-i.
int build_camera_tables(nv_ctx *c, Camera &cam, double cam_h) {
  c->gen++;
  const int W = cam.W, H = cam.H;
  std::vector<double> u(W), tc(H, 0.0), tf(H, 0.0), vv(H);
  for (int j = 0; j < W; ++j) u[j] = (((double)j + 0.5) - (double)W * 0.5) / cam.focal;
  std::vector<RowRec> rows(H);
  int n_top = 0, b0 = H;
  for (int i = 0; i < H; ++i) {
    double v = ((double)H * 0.5 - ((double)i + 0.5)) / cam.focal;
    vv[i] = v;
    RowRec r;
    std::memset(&r, 0, sizeof r);
    bool lit = false;
    double t = 0.0;
    const double *col = nullptr;
    uint32_t sem = 0;
    if (v > 0.0) {
      n_top = i + 1;
      tc[i] = (c->wall_h - cam_h) / v;
      t = tc[i];
      lit = t < cam.max_range;
      col = c->ceil3;
      sem = 65535;
    } else if (v < 0.0) {
      if (b0 == H) b0 = i;
      tf[i] = -cam_h / v;
      t = tf[i];
      lit = t < cam.max_range;
      col = c->floor3;
      sem = 65534;
    }
    if (lit) {
      r.depth_p = (float)t;
      r.sem2 = sem | (sem << 16);
      r.num2 = h2splat(0.8f * (float)std::fabs(v));
      r.r2 = h2splat((float)(col[0] * 255.0));
      r.g2 = h2splat((float)(col[1] * 255.0));
      r.b2 = h2splat((float)(col[2] * 255.0));
    } else {
      r.depth_p = (float)cam.max_range;
    }
    rows[i] = r;
  }
  const int Hh = (H + 1) / 2;
  std::vector<uint16_t> invh((size_t)Hh * W);
  for (int i = 0; i < Hh; ++i)
    for (int j = 0; j < W; ++j)
      invh[(size_t)i * W + j] = f2h((float)(1.0 / std::sqrt(1.0 + u[j] * u[j] + vv[i] * vv[i])));
  TRY(upload(cam.invh, invh));
  cam.n_top = n_top;
  cam.b0 = b0;
  cam.ktop = (float)(cam.focal * (c->wall_h - cam_h));
  cam.kbot = (float)(cam.focal * cam_h);
  TRY(upload(cam.u, u));
  TRY(upload(cam.tc, tc));
  TRY(upload(cam.tf, tf));
  TRY(upload(cam.rows, rows));
  cam.tables_cam_h = cam_h;
  return NV_OK;
}

// Record order used by the fast fill writers for a frame width (rec_pos).
#ifndef NV_CPL256
#define NV_CPL256 8  // columns per lane of the ws writer for W a multiple of 256 (8 or 4)
#endif
int fast_cpl(int W) { return W % 256 == 0 ? NV_CPL256 : (W == 128 ? 4 : (W == 64 ? 2 : 0)); }

// A render's casts write the other half of the record buffer than the last one.
void rec_flip(Camera &cam) { cam.rec_half ^= 1; }

// Release counters of the camera for n envs (zeroed when (re)allocated).
int rel_buffers(DevBuf &b, int64_t &have, int64_t n) {
  if (have == n) return NV_OK;
  const size_t bytes = sizeof(unsigned) * (size_t)(4 * n + 1);
  TRY(b.alloc(bytes));
  CK(cudaMemset(b.p, 0, bytes));
  have = n;
  return NV_OK;
}
unsigned *rel_done(Camera &k, int64_t N) { return k.rel.as<unsigned>() + (size_t)k.rec_half * 2 * N; }
unsigned *rel_fault(Camera &k, int64_t N) { return k.rel.as<unsigned>() + 4 * (size_t)N; }

// Column-record planes of N envs in the current half of the camera's record
// buffer (A then B).
RecOut rec_out(Camera &cam, int64_t N) {
  RecOut r;
  r.a = cam.rec.as<float4>() + (size_t)cam.rec_half * (cam.rec.bytes / 2 / sizeof(float4));
  r.b = r.a + (size_t)N * cam.W;
  r.W = cam.W;
  r.cpl = fast_cpl(cam.W);
  return r;
}

CamView cam_view(const Camera &cam) {
  CamView v;
  v.cpl = fast_cpl(cam.W);
  v.hc = (float)(cam.H * 0.5 - 0.5);
  v.ktop = cam.ktop;
  v.kbot = cam.kbot;
  v.W = cam.W; v.H = cam.H; v.n_top = cam.n_top; v.b0 = cam.b0; v.max_range = cam.max_range;
  v.u = cam.u.as<double>(); v.tc = cam.tc.as<double>(); v.tf = cam.tf.as<double>();
  v.rows = cam.rows.as<RowRec>();
  return v;
}

// Event pair around one launch of kind k (0 step, 1 cast, 2 fill, 3 other).
struct Prof {
  nv_ctx *c;
  cudaStream_t st;
  int pair = -1;
  Prof(nv_ctx *c_, cudaStream_t s_, int kind) : c(c_), st(s_) {
    if (!c->prof_on) return;
    if (2 * (c->prof_used + 1) > c->prof_ev.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      c->prof_ev.push_back(a);
      c->prof_ev.push_back(b);
      c->prof_kind.push_back(kind);
    }
    pair = (int)c->prof_used++;
    c->prof_kind[pair] = kind;
    cudaEventRecord(c->prof_ev[2 * pair], st);
  }
  ~Prof() {
    if (pair >= 0) cudaEventRecord(c->prof_ev[2 * pair + 1], st);
  }
};

int check_launch(nv_ctx *c) {
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NV_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
  return NV_OK;
}

// Opts kernel `fn` into `smem` bytes of dynamic shared memory on the context's
// device (once per size increase).
int set_smem(nv_ctx *c, const void *fn, size_t smem) {
  size_t &have = c->smem_cfg[fn];
  if (smem > have) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    have = smem;
  }
  return NV_OK;
}

unsigned blocks_for(long long work, int per_block) {
  return (unsigned)std::max<long long>(1, (work + per_block - 1) / per_block);
}

// Warp-specialised writer: NV_WS_NW producer warps + 1 store warp.
// Preference order: RPW (rows per producer warp per slot) = 1 then 2, the
// shading table read through L1 (staging it in shared memory measured slower
// at C1/C2/C3: C3 fill 76.9 vs 75.7 us; NV_WS_TAB=1 builds the staged
// variant), with as many ring slots as fit (<= 4; A/B at C3: 3 / 4 / 5 / 6
// slots -> 75.5 / 75.2 / 76.6 / 76.4 us).
template <int CPL, bool TAB, int RPW>
int launch_ws_kernel(nv_ctx *c, nvk::FillArgs &a, const nvk::FillWsLayout &L, size_t smem,
                     cudaStream_t st) {
  const bool noise = a.noise_sigma > 0.0f && a.depth;
  auto pick = [&](auto rel) {
    constexpr bool R = decltype(rel)::value;
    return L.bands > 1 ? (noise ? nvk::k_fill_ws<CPL, TAB, RPW, true, true, R>
                                : nvk::k_fill_ws<CPL, TAB, RPW, false, true, R>)
                       : (noise ? nvk::k_fill_ws<CPL, TAB, RPW, true, false, R>
                                : nvk::k_fill_ws<CPL, TAB, RPW, false, false, R>);
  };
  auto kern = a.done ? pick(std::true_type{}) : pick(std::false_type{});
  TRY(set_smem(c, (const void *)kern, smem));
  const unsigned grid =
      (unsigned)std::max<int64_t>(1, std::min<int64_t>(a.N * (int64_t)L.bands, c->sm_count));
  c->ws_tail_full = grid == (unsigned)c->sm_count;
  c->ws_tail_stream = st;
  Prof pf(c, st, 2);
  if (c->fill_pdl) {  // a programmatic dependent of the column cast just launched
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3((L.nw + (a.done ? 2 : 1)) * 32);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, kern, a, L));
  } else {
    kern<<<grid, (L.nw + (a.done ? 2 : 1)) * 32, smem, st>>>(a, L);
  }
  return check_launch(c);
}

template <int CPL>
int launch_fill_ws(nv_ctx *c, nvk::FillArgs &a, cudaStream_t st) {
  const int segw = 32 * CPL;
  const int S = a.W / segw;
  constexpr int nw = NV_WS_NW;
  const int bpp = (a.rgb ? 3 : 0) + (a.depth ? 4 : 0) + (a.sem ? 2 : 0);
  auto up = [](size_t x) { return (x + 127) & ~(size_t)127; };
  if (nw % S) return fail(NV_ERR_ARG, "frame layout unsupported by ws fill");
  const size_t rows_b = up((size_t)a.H * sizeof(RowRec));
  const size_t inv_b = up((size_t)((a.H + 1) / 2) * a.W * 2);
  const size_t cols_b = up((size_t)NV_WS_CBUF * a.W * sizeof(ColRec));
  const size_t bars_b = 128;
  struct Opt { bool tab; int rpw, nmin, nmax; };
  static const Opt opts[] = {{true, 1, 2, 4}, {true, 2, 2, 4}, {false, 1, 2, 4}, {false, 2, 2, 4}};
  nvk::FillWsLayout L;
  bool tab = false;
  int rpw = 0;
  size_t smem = 0;
  for (const Opt &o : opts) {
    if (NV_WS_RPW && o.rpw != NV_WS_RPW) continue;
    if (!NV_WS_TAB && o.tab) continue;
    const int R = o.rpw * nw / S;
    if (a.H % R) continue;
    const size_t slot = up((size_t)R * a.W * bpp);
    for (int ns = NV_WS_SLOTS ? NV_WS_SLOTS : o.nmax; ns >= o.nmin && !rpw; --ns) {
      const size_t tot = rows_b + (o.tab ? inv_b : 0) + cols_b + bars_b + (size_t)ns * slot;
      if ((int)tot <= c->max_smem_optin) {
        tab = o.tab; rpw = o.rpw; smem = tot;
        L.nslot = ns; L.slot_rows = R; L.slot_bytes = (int)slot;
      }
    }
    if (rpw) break;
  }
  if (!rpw) return fail(NV_ERR_ARG, "frame layout too large for the ws fill writer");
  L.rows = 0;
  L.inv = (int)rows_b;
  L.cols = L.inv + (tab ? (int)inv_b : 0);
  L.bars = L.cols + (int)cols_b;
  L.slots = L.bars + (int)bars_b;
  L.nw = nw;
  {  // row bands per env: minimise the busiest CTA's time, ceil(N b / grid) items
     // of (1/b frame + a fixed per-item cost).  Per-item cost measured at C3
     // (2 bands: +8 us over 1024 extra items on 148 CTAs) ~ 1.1 us, i.e. the
     // time one SM streams ~50 KB at its ~45 GB/s store rate.
    const double frame_bytes = (double)a.W * a.H * bpp;
    const double ovh = 49500.0 / std::max(1.0, frame_bytes);
    int best = 1;
    double best_t = 1e30;
    for (int b = 1; b <= 64; b *= 2) {
      if ((a.H / L.slot_rows) % b) break;
      const int64_t items = a.N * (int64_t)b;
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(items, c->sm_count));
      const double t = (double)((items + grid - 1) / grid) * (1.0 / b + ovh);
      if (t < best_t * (1.0 - 1e-9)) {
        best_t = t;
        best = b;
      }
    }
    constexpr int force_bands = NV_WS_BANDS > 0 ? NV_WS_BANDS : 1;
    L.bands = NV_WS_BANDS > 0 && (a.H / L.slot_rows) % force_bands == 0 ? force_bands : best;
  }
  a.segs_per_row = S;
  if constexpr (NV_WS_TAB != 0) {  // study builds only (staged shading table)
    if (tab && rpw == 2) return launch_ws_kernel<CPL, true, 2>(c, a, L, smem, st);
    if (tab) return launch_ws_kernel<CPL, true, 1>(c, a, L, smem, st);
  }
  if (rpw == 2) return launch_ws_kernel<CPL, false, 2>(c, a, L, smem, st);
  return launch_ws_kernel<CPL, false, 1>(c, a, L, smem, st);
}

// Whether the warp-specialised writer takes this frame layout: W in {64, 128,
// 256k <= 4096}, whole slots of rows, 16-byte aligned outputs (bulk copies).
bool ws_layout_ok(const Camera &cam, const void *rgb, const void *depth, const void *sem) {
  auto al16 = [](const void *p) { return ((uintptr_t)p & 15) == 0; };
  if (!(al16(rgb) && al16(depth) && al16(sem))) return false;
  if (cam.W % 256 == 0) return cam.W <= 4096 && cam.H % (16 / std::min(16, cam.W / 256)) == 0;
  return (cam.W == 128 || cam.W == 64) && cam.H % 16 == 0;
}

int launch_fill(nv_ctx *c, Camera &cam, int64_t N, uint8_t *rgb, float *depth, uint16_t *sem,
                cudaStream_t st, bool release = false) {
  if (!rgb && !depth && !sem) return NV_OK;
  nvk::FillArgs a;
  a.done = release ? rel_done(cam, N) : nullptr;
  a.consumed = release ? rel_done(cam, N) + N : nullptr;
  a.fault = release ? rel_fault(cam, N) : nullptr;
  a.ready = release ? c->fill_ready : nullptr;
  a.posrec = release ? c->fill_posrec : nullptr;
  const RecOut ro = rec_out(cam, N);
  a.ra = ro.a;
  a.rb = ro.b;
  a.cpl = ro.cpl;
  a.rows = cam.rows.as<RowRec>();
  a.invh = cam.invh.as<uint16_t>();
  a.N = (int)N; a.W = cam.W; a.H = cam.H;
  a.rgb = rgb; a.depth = depth; a.sem = sem;
  a.segs_per_row = 1;
  const bool noise = c->noise_sigma > 0.0 && depth;
  a.noise_sigma = noise ? (float)c->noise_sigma : 0.0f;
  a.max_range = (float)cam.max_range;
  a.noise_seed = c->noise_seed;
  a.noise_frame = noise ? c->noise_frame++ : 0;
  a.env_offset = c->noise_env_offset;
  // auto: the warp-specialised writer whenever the frame layout allows it
  // (row bands spread small batches over the SMs), else the per-pixel
  // kernel; both produce identical frames.  The ws writer applies the depth
  // noise itself, the per-pixel kernel gets a pass.
  if (c->fill_mode != NV_FILL_GENERIC && ws_layout_ok(cam, rgb, depth, sem)) {
    if (cam.W % 256 == 0) return launch_fill_ws<NV_CPL256>(c, a, st);
    if (cam.W == 128) return launch_fill_ws<4>(c, a, st);
    return launch_fill_ws<2>(c, a, st);
  }
  {
    const long long total = N * (long long)cam.W * cam.H;
    Prof pf(c, st, 2);
    nvk::k_fill_generic<<<blocks_for(total, 256), 256, 0, st>>>(a);
    TRY(check_launch(c));
  }
  if (noise) {
    const long long pairs = N * (long long)cam.H * ((cam.W + 1) / 2);
    nvk::k_depth_noise<<<blocks_for(pairs, 256), 256, 0, st>>>(a, depth);
    TRY(check_launch(c));
  }
  return NV_OK;
}

int cam_check(nv_ctx *c, int cam) {
  if (cam < 0 || cam >= 8 || !c->cams[cam].on)
    return fail(NV_ERR_STATE, "camera %d not configured (nv_camera_config)", cam);
  Camera &k = c->cams[cam];
  if (c->sensor_h > c->wall_h) return fail(NV_ERR_ARG, "sensor height must stay below wall height");
  if (c->n_envs * (int64_t)k.W >= (1LL << 31))  // ray indices are 32-bit in the casts
    return fail(NV_ERR_ARG, "n_envs * W = %lld rays per camera exceeds 2^31",
                (long long)(c->n_envs * (int64_t)k.W));
  if (k.tables_cam_h != c->sensor_h) TRY(build_camera_tables(c, k, c->sensor_h));
  TRY(k.rec.alloc(2 * sizeof(ColRec) * (size_t)std::max<int64_t>(1, c->n_envs) * k.W));
  TRY(rel_buffers(k.rel, k.rel_n, std::max<int64_t>(1, c->n_envs)));
  return NV_OK;
}

// small batches (rays fit in about one wave of warps): one warp per ray
bool use_warp_cast(const nv_ctx *c, long long rays) {
  return c->cast_mode == NV_CAST_WARP || (c->cast_mode == NV_CAST_AUTO && rays <= NV_CAST_WARP_RAYS);
}

// CTAs of the column cast for `rays` rays (warp or thread per ray)
unsigned cast_blocks(const nv_ctx *c, long long rays) {
  return use_warp_cast(c, rays) ? blocks_for(rays * 32, 128) : blocks_for(rays, NV_CAST_BLOCK);
}

// block order (identity) and durations (zero) for `nblk` cast blocks
int lpt_buffers(nv_ctx *c, DevBuf &order, DevBuf &cost, int64_t &n, unsigned nblk,
                cudaStream_t st) {
  if (n == (int64_t)nblk) return NV_OK;
  TRY(order.alloc(sizeof(unsigned) * nblk));
  TRY(cost.alloc(sizeof(unsigned) * nblk));
  nvk::k_lpt_init<<<blocks_for(nblk, 256), 256, 0, st>>>(order.as<unsigned>(),
                                                          cost.as<unsigned>(), nblk);
  TRY(check_launch(c));
  n = nblk;
  return NV_OK;
}

// Longest-first ordering only pays when the cast runs several waves of
// blocks (C2: 30.1 -> 28.3 us/step); a one-wave cast (C1: 64 blocks) only
// gains the ordering kernel's latency (14.9 -> 17.1 us/step).
bool lpt_pays(const nv_ctx *c, unsigned nblk) { return nblk >= 4u * (unsigned)c->sm_count; }

// the next step's block order, on a side stream beside the frame writer
// (joined into `st` by lpt_join after the writer is launched)
// Side stream beside the frame writer, forked from `st` after the casts
// (joined by lpt_join after the writer is launched).  In a captured graph the
// fork is a dependency edge only, so the writer stays a programmatic
// dependent of the casts.
int side_fork(nv_ctx *c, cudaStream_t st) {
  if (!c->o_stream) {
    CK(cudaStreamCreateWithFlags(&c->o_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->o_ev0, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->o_ev1, cudaEventDisableTiming));
  }
  if (c->o_fork) return NV_OK;
  CK(cudaEventRecord(c->o_ev0, st));
  CK(cudaStreamWaitEvent(c->o_stream, c->o_ev0, 0));
  c->o_fork = true;
  return NV_OK;
}

int lpt_fork(nv_ctx *c, cudaStream_t st, unsigned *order, unsigned *cost, unsigned nblk) {
  TRY(side_fork(c, st));
  nvk::k_cast_order<<<1, 32 * NV_ORDER_WARPS, 0, c->o_stream>>>(cost, order, (int)nblk);
  return check_launch(c);
}

// release: publish per-env finished-column counts for a writer launched as
// this cast's programmatic dependent (k_fill_ws with FillArgs.done)
unsigned *pdl_fault(nv_ctx *c);

// trigger: a frame writer follows as the cast's programmatic dependent
int do_cast(nv_ctx *c, int cam, double *gps, double *compass, cudaStream_t st,
            bool release = false, bool trigger = false) {
  Camera &k = c->cams[cam];
  // t_max = max_range: capping the walk is output-identical for rendered
  // frames (tests/test_gpu_parity.py checks it against the
  // reference's uncapped t_max = 1e9 render).
  const long long total = c->n_envs * (long long)k.W;
  const bool warp = use_warp_cast(c, total);
  const unsigned nblk = cast_blocks(c, total);
  rec_flip(k);
  const unsigned threads = warp ? 128u : (unsigned)NV_CAST_BLOCK;
  unsigned *order = nullptr, *cost = nullptr;
  if (NV_CAST_LPT && lpt_pays(c, nblk)) {
    TRY(lpt_buffers(c, k.lpt_order, k.lpt_cost, k.lpt_n, nblk, st));
    order = k.lpt_order.as<unsigned>();
    cost = k.lpt_cost.as<unsigned>();
  }
  {
    Prof pf(c, st, 1);
    auto kern = warp ? nvk::k_column_cast_warp : nvk::k_column_cast;
    unsigned *ready = nullptr, *arrive = nullptr, *rfault = nullptr;
    const double *posrec = nullptr;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(nblk);
    lc.blockDim = dim3(threads);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    if (c->pdl_armed) {  // programmatic dependent of the agent step just launched
      c->pdl_armed = false;
      ready = c->pdl_cur_ready;
      arrive = c->pdl_cur_arrive;
      posrec = c->pdl_cur_posrec;
      rfault = pdl_fault(c);
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
    }
    CK(cudaLaunchKernelEx(&lc, kern, c->env_view(), c->scene_view(), cam_view(k),
                          rec_out(k, c->n_envs), k.max_range, gps, compass, ready, arrive, rfault,
                          (const unsigned *)order, cost,
                          release ? rel_done(k, c->n_envs) : (unsigned *)nullptr, trigger,
                          posrec));
    TRY(check_launch(c));
  }
  return order ? lpt_fork(c, st, order, cost, nblk) : NV_OK;
}

// join of the ordering kernel forked by do_cast
int lpt_join(nv_ctx *c, cudaStream_t st) {
  if (!c->o_fork) return NV_OK;
  c->o_fork = false;
  if (c->order_ev) CK(cudaEventRecordWithFlags(c->order_ev, c->o_stream, cudaEventRecordExternal));
  CK(cudaEventRecord(c->o_ev1, c->o_stream));
  CK(cudaStreamWaitEvent(st, c->o_ev1, 0));
  return NV_OK;
}

// per-env ready / arrive flags of the agent -> cast overlap (zero between steps)
// ready: [release half 0 | release half 1 | arrive mode] x N, then the fault
// flag of the release-mode waits.  The release-mode flags of a record half are
// reset by the writer that consumes them, the arrive-mode ones by the casts;
// separate sets, so mixing the modes between steps never loses a flag.
int pdl_buffers(nv_ctx *c) {
  const size_t n = (size_t)std::max<int64_t>(1, c->n_envs);
  const size_t b = sizeof(unsigned) * (3 * n + 1);
  if (c->pdl_ready.bytes < b || !c->pdl_init) {
    TRY(c->pdl_ready.alloc(b));
    TRY(c->pdl_arrive.alloc(sizeof(unsigned) * n));
    CK(cudaMemset(c->pdl_ready.p, 0, b));
    CK(cudaMemset(c->pdl_arrive.p, 0, sizeof(unsigned) * n));
    c->pdl_init = true;
  }
  const size_t words = 2 * n * NV_POSE_STRIDE;
  if (NV_POSE_REC && (c->pose_rec.bytes < words * 8 || !c->pose_init)) {
    TRY(c->pose_rec.alloc(words * 8));
    nvk::k_pose_init<<<blocks_for((int64_t)words, 256), 256>>>(
        c->pose_rec.as<unsigned long long>(), (long long)words);
    TRY(check_launch(c));
    CK(cudaDeviceSynchronize());
    c->pose_init = true;
  }
  return NV_OK;
}
// the ready flags of a step: release mode -> the set of the record half the
// coming casts write, else the arrive-mode set
unsigned *pdl_ready_set(nv_ctx *c, int release_half) {
  const size_t n = (size_t)std::max<int64_t>(1, c->n_envs);
  return c->pdl_ready.as<unsigned>() + (release_half >= 0 ? (size_t)release_half : 2) * n;
}
unsigned *pdl_fault(nv_ctx *c) {
  return c->pdl_ready.as<unsigned>() + 3 * (size_t)std::max<int64_t>(1, c->n_envs);
}

// arm_pdl: the cast that follows is this agent step's programmatic dependent;
// release_half >= 0: release mode (the casts write that record half, its
// frame writer resets the ready flags), -1: the casts reset them (arrive)
// pose_rec: release mode with pose records instead of ready flags (the
// casts load the half's records, its writer resets them)
int do_step(nv_ctx *c, const int8_t *actions, uint8_t *collided, double *disp, int32_t *status,
            cudaStream_t st, bool arm_pdl = false, int release_half = -1, bool pose_rec = false) {
  nvk::AgentCfg cfg{c->radius, c->step, c->turn_rad};
  long long threads = c->n_envs * 32;
  unsigned *ready = nullptr;
  double *posrec = nullptr;
  c->pdl_cur_posrec = nullptr;
  if (arm_pdl) {
    TRY(pdl_buffers(c));
    if (pose_rec && release_half >= 0) {
      posrec = c->pose_rec.as<double>() +
               (size_t)release_half * std::max<int64_t>(1, c->n_envs) * NV_POSE_STRIDE;
      c->pdl_cur_posrec = posrec;
      c->pdl_cur_ready = nullptr;
      c->pdl_cur_arrive = nullptr;
    } else {
      ready = pdl_ready_set(c, release_half);
      c->pdl_cur_ready = ready;
      c->pdl_cur_arrive = release_half >= 0 ? nullptr : c->pdl_arrive.as<unsigned>();
    }
  }
  Prof pf(c, st, 0);
  {
    // a programmatic dependent of whatever kernel precedes it: the previous
    // step's frame writer releases it early (its records live in the other
    // half), any other kernel simply completes first
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(blocks_for(threads, NV_AGENT_BLOCK));
    lc.blockDim = dim3(NV_AGENT_BLOCK);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = NV_STEP_CHAIN && c->pdl && !c->prof_on ? 1 : 0;
    // (the agent step is a programmatic dependent of whatever precedes it;
    // beside a full-grid writer it may work at once, else it waits for it --
    // also while a host step's writer may still hold SMs, which voids the
    // residency argument)
    const int wait_first = !(c->ws_tail_full && c->ws_tail_stream == st) || c->e_pending;
    CK(cudaLaunchKernelEx(&lc, nvk::k_agent_step, c->env_view(), c->scene_view(), cfg, actions,
                          collided, disp, status, ready, posrec, wait_first));
  }
  TRY(check_launch(c));
  c->pdl_armed = arm_pdl;
  return NV_OK;
}

// A host-buffer step returns once its step results are on the host; its frame
// writer may still run on the internal stream.  Entry points that reallocate
// or expose the buffers it uses wait for it first.
int e2e_fence(nv_ctx *c) {
  if (c->e_pending) {
    c->e_pending = false;
    for (int p = 0; p < 2; ++p)
      if (c->e_stream[p]) CK(cudaStreamSynchronize(c->e_stream[p]));
  }
  return NV_OK;
}

}  // namespace

// ====================================================================== ABI

extern "C" {

const char *nv_last_error(void) { return g_err.c_str(); }
int nv_version(void) { return 1; }

int nv_create(int device, nv_ctx **out) {
  if (!out) return fail(NV_ERR_ARG, "out is NULL");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(NV_ERR_ARG, "device %d out of range (%d)", device, ndev);
  CK(cudaSetDevice(device));
  nv_ctx *c = new nv_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&c->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  *out = c;
  return NV_OK;
}

int nv_destroy(nv_ctx *ctx) {
  if (!ctx) return NV_OK;
  cudaSetDevice(ctx->device);
  e2e_fence(ctx);
  delete ctx;
  return NV_OK;
}

int nv_scene_upload(nv_ctx *c, const double *segs, const uint16_t *sem, const double *albedo,
                    int64_t n, double wall_height, const double *floor3, const double *ceil3) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(e2e_fence(c));
  c->gen++;
  if (n < 0 || (n > 0 && (!segs || !sem || !albedo)))
    return fail(NV_ERR_ARG, "bad scene arrays");
  if (n >= (1LL << 31)) return fail(NV_ERR_ARG, "too many segments (%lld)", (long long)n);
  CK(cudaSetDevice(c->device));
  HostGrid g = build_grid(segs, n);
  if (n > 0) {  // Scene.bounds (scene.py:69-76)
    double b0 = INFINITY, b1 = INFINITY, b2 = -INFINITY, b3 = -INFINITY;
    for (int64_t i = 0; i < n; ++i) {
      b0 = std::min(b0, std::min(segs[4 * i], segs[4 * i + 2]));
      b1 = std::min(b1, std::min(segs[4 * i + 1], segs[4 * i + 3]));
      b2 = std::max(b2, std::max(segs[4 * i], segs[4 * i + 2]));
      b3 = std::max(b3, std::max(segs[4 * i + 1], segs[4 * i + 3]));
    }
    c->sbounds[0] = b0; c->sbounds[1] = b1; c->sbounds[2] = b2; c->sbounds[3] = b3;
  }
  c->has_nav = false;
  if (g.nx * g.ny >= (1LL << 31) || (int64_t)g.items.size() >= (1LL << 31))
    return fail(NV_ERR_ARG, "scene grid too large");
  std::vector<double> ax(n), ay(n), bx(n), by(n), ex(n), ey(n), nx(n), ny(n);
  std::vector<uint16_t> sm(n);
  std::vector<float4> alb(n);
  for (int64_t i = 0; i < n; ++i) {
    ax[i] = segs[4 * i]; ay[i] = segs[4 * i + 1]; bx[i] = segs[4 * i + 2]; by[i] = segs[4 * i + 3];
    ex[i] = bx[i] - ax[i]; ey[i] = by[i] - ay[i];
    // segment_normals (geometry.py:66-73): glibc hypot, like np.hypot
    double ln = std::hypot(ex[i], ey[i]);
    if (!(ln > 0.0)) ln = 1.0;
    nx[i] = -ey[i] / ln;
    ny[i] = ex[i] / ln;
    sm[i] = sem[i];
    alb[i] = make_float4((float)(albedo[3 * i] * 255.0), (float)(albedo[3 * i + 1] * 255.0),
                         (float)(albedo[3 * i + 2] * 255.0), 0.0f);
  }
  std::vector<int32_t> starts(g.starts.size()), items(g.items.size());
  std::vector<CellEntry> ent(g.items.size());
  std::vector<float4> entf(g.items.size()), entm(g.items.size());
  std::vector<float> cellb((size_t)(g.nx * g.ny), 0.f);
  for (size_t k = 0; k < g.starts.size(); ++k) starts[k] = (int32_t)g.starts[k];
  for (int64_t cy = 0; cy < g.ny; ++cy)
    for (int64_t cx = 0; cx < g.nx; ++cx) {
      const int64_t c = cy * g.nx + cx;
      // cell anchor, the same IEEE sums the device forms (kernels.cuh cell_bounds)
      const double X0 = g.x0 + (double)cx, Y0 = g.y0 + (double)cy;
      float amax = 0.f;
      for (int64_t q = g.starts[c]; q < g.starts[c + 1]; ++q) {
        int64_t i = g.items[q];
        items[q] = (int32_t)i;
        CellEntry e;
        e.ax = ax[i]; e.ay = ay[i]; e.ex = ex[i]; e.ey = ey[i];
        ent[q] = e;
        // endpoints a and a + e (the segment the reference's arithmetic tests)
        float4 f = make_float4((float)(ax[i] - X0), (float)(ay[i] - Y0),
                               (float)(ax[i] + ex[i] - X0), (float)(ay[i] + ey[i] - Y0));
        entf[q] = f;
        // midpoint / half-vector form of the same f32 endpoints (the cast's side test)
        const float4 m = make_float4((float)(0.5 * ((double)f.x + (double)f.z)),
                                     (float)(0.5 * ((double)f.y + (double)f.w)),
                                     (float)(0.5 * ((double)f.z - (double)f.x)),
                                     (float)(0.5 * ((double)f.w - (double)f.y)));
        entm[q] = m;
        amax = std::max(amax, std::max(std::fabs(f.x) + std::fabs(f.y), std::fabs(f.z) + std::fabs(f.w)));
        amax = std::max(amax, std::fabs(m.x) + std::fabs(m.z) + std::fabs(m.y) + std::fabs(m.w));
      }
      // 2^-20 relative slack covers the f32 rounding of the stored values
      cellb[c] = amax * (1.0f + 0x1p-20f);
    }
  TRY(upload(c->ax, ax)); TRY(upload(c->ay, ay)); TRY(upload(c->bx, bx)); TRY(upload(c->by, by));
  TRY(upload(c->ex, ex)); TRY(upload(c->ey, ey)); TRY(upload(c->nx, nx)); TRY(upload(c->ny, ny));
  TRY(upload(c->sem, sm)); TRY(upload(c->alb, alb));
  TRY(upload(c->starts, starts)); TRY(upload(c->items, items)); TRY(upload(c->ent, ent));
  TRY(upload(c->entf, entf));
  TRY(upload(c->entm, entm));
  // Per cell: runs of NV_CHUNK entries (bucket order) with the f32 bounding box
  // of their cell-relative endpoints, stored as centre + half-extents rounded
  // outwards (the stored box contains every endpoint); the cast rejects a
  // whole run when the ray's line passes the box on one side (geom.cuh
  // cell_tests).  The cell bound grows to cover the box, so one error bound
  // E serves both.
  std::vector<int4> cells((size_t)(g.nx * g.ny));
  std::vector<float4> chunks;
  for (size_t k = 0; k < cells.size(); ++k) {
    float b = cellb[k];
    const int32_t q0 = starts[k], q1 = starts[k + 1];
    const int32_t ch0 = (int32_t)chunks.size();
    for (int32_t q = q0; q < q1; q += NV_CHUNK) {
      float4 bx = make_float4(INFINITY, INFINITY, -INFINITY, -INFINITY);
      for (int32_t r = q; r < std::min(q1, q + NV_CHUNK); ++r) {
        const float4 f = entf[r];
        bx.x = std::min(bx.x, std::min(f.x, f.z));
        bx.y = std::min(bx.y, std::min(f.y, f.w));
        bx.z = std::max(bx.z, std::max(f.x, f.z));
        bx.w = std::max(bx.w, std::max(f.y, f.w));
      }
      // centre (rounded) and half-extent (rounded up) so [c - h, c + h] covers [lo, hi]
      auto centre_half = [](float lo, float hi, float &cc, float &hh) {
        cc = (float)(0.5 * ((double)lo + (double)hi));
        const double h = std::max((double)hi - (double)cc, (double)cc - (double)lo);
        hh = (float)h;
        if ((double)hh < h) hh = std::nextafter(hh, INFINITY);
      };
      float4 cm;
      centre_half(bx.x, bx.z, cm.x, cm.z);
      centre_half(bx.y, bx.w, cm.y, cm.w);
      chunks.push_back(cm);
      const float cb = std::max(std::max(std::fabs(bx.x), std::fabs(bx.z)), std::fabs(cm.x) + cm.z) +
                       std::max(std::max(std::fabs(bx.y), std::fabs(bx.w)), std::fabs(cm.y) + cm.w);
      b = std::max(b, cb * (1.0f + 0x1p-20f));
    }
    int bi;
    std::memcpy(&bi, &b, 4);
    cells[k] = make_int4(q0, q1, bi, ch0);
  }
  if (chunks.empty()) chunks.push_back(make_float4(0.f, 0.f, 0.f, 0.f));
  // disc-cast records: disc_cast's per-candidate seg_len / tangent
  // (_kernels.py:407-413), host IEEE ops without contraction = device ops
  std::vector<double> stx(n), sty(n), slen(n);
  for (int64_t i = 0; i < n; ++i) {
    const double exi = bx[i] - ax[i], eyi = by[i] - ay[i];
    slen[i] = std::sqrt(exi * exi + eyi * eyi);
    stx[i] = slen[i] > 0.0 ? exi / slen[i] : 0.0;
    sty[i] = slen[i] > 0.0 ? eyi / slen[i] : 0.0;
  }
  std::vector<DiscEntry> dent(items.size());
  for (size_t q = 0; q < items.size(); ++q) {
    const int32_t i = items[q];
    DiscEntry d;
    d.ax = ax[i]; d.ay = ay[i]; d.bx = bx[i]; d.by = by[i];
    d.tx = stx[i]; d.ty = sty[i]; d.len = slen[i];
    d.idx = i; d.pad = 0;
    dent[q] = d;
  }
  if (dent.empty()) dent.push_back(DiscEntry{});
  if (stx.empty()) { stx.push_back(0.0); sty.push_back(0.0); }
  TRY(upload(c->dent, dent)); TRY(upload(c->stx, stx)); TRY(upload(c->sty, sty));
  TRY(upload(c->cells, cells));
  TRY(upload(c->chunks, chunks));
  c->n = n;
  c->wall_h = wall_height;
  for (int k = 0; k < 3; ++k) {
    c->floor3[k] = floor3 ? floor3[k] : c->floor3[k];
    c->ceil3[k] = ceil3 ? ceil3[k] : c->ceil3[k];
  }
  c->gx0 = g.x0; c->gy0 = g.y0; c->gnx = (int)g.nx; c->gny = (int)g.ny;
  c->nitems = (int64_t)g.items.size();
  c->has_scene = true;
  for (auto &k : c->cams) k.tables_cam_h = NAN;  // colours / wall height changed
  return NV_OK;
}

int nv_scene_grid_info(nv_ctx *c, double *x0, double *y0, int64_t *nx, int64_t *ny,
                       int64_t *nitems) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_scene(c));
  if (x0) *x0 = c->gx0;
  if (y0) *y0 = c->gy0;
  if (nx) *nx = c->gnx;
  if (ny) *ny = c->gny;
  if (nitems) *nitems = c->nitems;
  return NV_OK;
}

int nv_agent_config(nv_ctx *c, double radius, double forward_step, double turn_rad,
                    double sensor_height) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  c->gen++;
  if (!(radius >= 0.0) || !(forward_step > 0.0) || !(turn_rad > 0.0) || !(sensor_height > 0.0))
    return fail(NV_ERR_ARG, "invalid agent config");
  if (c->has_scene && sensor_height > c->wall_h)
    return fail(NV_ERR_ARG, "sensor height %g exceeds wall height %g", sensor_height, c->wall_h);
  c->radius = radius;
  c->step = forward_step;
  c->turn_rad = turn_rad;
  c->sensor_h = sensor_height;
  return NV_OK;
}

int nv_envs_alloc(nv_ctx *c, int64_t n_envs) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(e2e_fence(c));
  c->gen++;
  if (n_envs <= 0 || n_envs >= (1LL << 30)) return fail(NV_ERR_ARG, "bad n_envs %lld", (long long)n_envs);
  CK(cudaSetDevice(c->device));
  size_t d = sizeof(double) * (size_t)n_envs;
  for (DevBuf *b : {&c->x, &c->y, &c->h, &c->path, &c->ch, &c->sh, &c->ox, &c->oy, &c->oh, &c->fc,
                    &c->fs}) {
    b->release();
    TRY(b->alloc(d));
    CK(cudaMemset(b->p, 0, d));
  }
  c->coll.release();
  TRY(c->coll.alloc(sizeof(int64_t) * (size_t)n_envs));
  CK(cudaMemset(c->coll.p, 0, sizeof(int64_t) * (size_t)n_envs));
  c->reset.release();
  TRY(c->reset.alloc((size_t)n_envs));
  CK(cudaMemset(c->reset.p, 0, (size_t)n_envs));
  // The un-reset pose is the reference Simulator's initial AgentState
  // (origin, heading 0; sim.py:159): cos(heading) = 1 so observations()
  // before set_agent_state renders like the reference (sim.py:192-200).
  {
    const std::vector<double> ones((size_t)n_envs, 1.0);
    CK(cudaMemcpy(c->ch.p, ones.data(), d, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->fc.p, ones.data(), d, cudaMemcpyHostToDevice));
  }
  // PointGoal episodes belong to the old env batch: drop them (a stale done
  // flag would freeze the new envs; a smaller buffer would be read past its
  // end) -- nv_task_reset starts new ones
  c->task_on = false;
  for (DevBuf *b : {&c->t_goal, &c->t_gdsp, &c->t_fid, &c->t_dlast, &c->t_steps, &c->t_done,
                    &c->t_status})
    b->release();
  c->t_fields = nullptr;
  c->t_nfields = 0;
  // the agent -> cast ready flags are sized per env
  c->pdl_init = false;
  c->pose_init = false;
  c->pdl_init_e2e = false;
  c->pose_init_e2e = false;
  c->n_envs = n_envs;
  // (now, outside any stream capture a first step might be recorded in)
  return pdl_buffers(c);
}

int nv_camera_config(nv_ctx *c, int cam, int width, int height, double focal, double max_range) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(e2e_fence(c));
  c->gen++;
  if (cam < 0 || cam >= 8) return fail(NV_ERR_ARG, "camera index %d out of range [0, 8)", cam);
  if (width < 1 || height < 1 || width > 16384 || height > 16384)
    return fail(NV_ERR_ARG, "sensor resolution must be at least 1x1 (got %dx%d)", width, height);
  if (!(focal > 0.0) || !std::isfinite(focal)) return fail(NV_ERR_ARG, "bad focal %g", focal);
  if (!(max_range > 0.0)) return fail(NV_ERR_ARG, "max_range must be positive");
  TRY(ensure_scene(c));
  CK(cudaSetDevice(c->device));
  Camera &k = c->cams[cam];
  k.W = width;
  k.H = height;
  k.focal = focal;
  k.max_range = max_range;
  TRY(build_camera_tables(c, k, c->sensor_h));
  k.on = true;
  return NV_OK;
}

int nv_set_poses(nv_ctx *c, const double *xy, const double *heading, const uint8_t *mask,
                 int32_t *status_out, double *clearance_out) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  if (!xy || !heading) return fail(NV_ERR_ARG, "xy/heading are NULL");
  CK(cudaSetDevice(c->device));
  const size_t N = (size_t)c->n_envs;
  DevBuf dxy, dh, dm, dst, dcl;
  TRY(dxy.alloc(16 * N)); TRY(dh.alloc(8 * N)); TRY(dst.alloc(4 * N)); TRY(dcl.alloc(8 * N));
  CK(cudaMemcpy(dxy.p, xy, 16 * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dh.p, heading, 8 * N, cudaMemcpyHostToDevice));
  if (mask) {
    TRY(dm.alloc(N));
    CK(cudaMemcpy(dm.p, mask, N, cudaMemcpyHostToDevice));
  }
  nvk::k_set_poses<<<blocks_for((long long)N * 32, 128), 128>>>(
      c->env_view(), c->scene_view(), c->radius, dxy.as<double>(), dh.as<double>(),
      mask ? dm.as<uint8_t>() : nullptr, dst.as<int32_t>(), dcl.as<double>());
  TRY(check_launch(c));
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> st(N);
  std::vector<double> cl(N);
  CK(cudaMemcpy(st.data(), dst.p, 4 * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cl.data(), dcl.p, 8 * N, cudaMemcpyDeviceToHost));
  if (status_out) std::memcpy(status_out, st.data(), 4 * N);
  if (clearance_out) std::memcpy(clearance_out, cl.data(), 8 * N);
  for (size_t e = 0; e < N; ++e)
    if (st[e] == NV_ENV_TOO_CLOSE)
      return fail(NV_ERR_ARG, "env %zu: position (%.3f, %.3f) is %.3f m from the nearest wall; agent radius is %g",
                  e, xy[2 * e], xy[2 * e + 1], cl[e], c->radius);
  return NV_OK;
}

int nv_step(nv_ctx *c, const int8_t *actions, uint8_t *collided, double *displacement,
            int32_t *status, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  if (!actions) return fail(NV_ERR_ARG, "actions is NULL");
  return do_step(c, actions, collided, displacement, status, (cudaStream_t)stream);
}

int nv_render(nv_ctx *c, int cam, uint8_t *rgb, float *depth, uint16_t *sem, double *gps,
              double *compass, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  TRY(cam_check(c, cam));
  cudaStream_t st = (cudaStream_t)stream;
  TRY(do_cast(c, cam, gps, compass, st, false, rgb || depth || sem));
  const int rc = launch_fill(c, c->cams[cam], c->n_envs, rgb, depth, sem, st);
  TRY(lpt_join(c, st));
  return rc;
}

int nv_step_render(nv_ctx *c, const int8_t *actions, int cam, uint8_t *rgb, float *depth,
                   uint16_t *sem, double *gps, double *compass, uint8_t *collided,
                   double *displacement, int32_t *status, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  TRY(cam_check(c, cam));
  if (!actions) return fail(NV_ERR_ARG, "actions is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  Camera &k = c->cams[cam];
  // agent step -> cast overlap (programmatic dependent launch), unless
  // profiling events are on (an event between the two launches would break
  // the programmatic edge)
  const bool pdl = c->pdl && !c->prof_on;
  // cast -> writer programmatic launch (set-up beside the cast's tail); with
  // the ws writer, per-env release
  c->fill_pdl = NV_FILL_PDL && c->pdl && !c->prof_on;
  // (thread-per-ray batches: with the warp-per-ray cast of small batches the
  // per-env waits cost more than they overlap, C2 25.7 -> 27.3 us)
  const bool release = c->fill_pdl && NV_FILL_RELEASE && (rgb || depth || sem) &&
                       c->fill_mode != NV_FILL_GENERIC && ws_layout_ok(k, rgb, depth, sem) &&
                       !use_warp_cast(c, c->n_envs * (long long)k.W);
  // release mode: the agent -> cast ready flags of the record half the casts
  // are about to write (do_cast flips to it), reset by that half's writer
  const int rhalf = release && NV_READY_BY_HALF ? (k.rec_half ^ 1) : -1;
  TRY(do_step(c, actions, collided, displacement, status, st, pdl, rhalf, NV_POSE_REC != 0));
  c->fill_ready = pdl && rhalf >= 0 ? c->pdl_cur_ready : nullptr;
  c->fill_posrec = pdl && rhalf >= 0 ? c->pdl_cur_posrec : nullptr;
  TRY(do_cast(c, cam, gps, compass, st, release, rgb || depth || sem));
  c->pdl_armed = false;
  if (c->mid_ev) {  // on a branch of its own: no node between the casts and the writer
    if (!c->m_stream) {
      CK(cudaStreamCreateWithFlags(&c->m_stream, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->m_ev0, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->m_ev1, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(c->m_ev0, st));
    CK(cudaStreamWaitEvent(c->m_stream, c->m_ev0, 0));
    CK(cudaEventRecordWithFlags(c->mid_ev, c->m_stream, cudaEventRecordExternal));
  }
  const int rc = launch_fill(c, k, c->n_envs, rgb, depth, sem, st, release);
  c->fill_pdl = false;
  c->fill_ready = nullptr;
  c->fill_posrec = nullptr;
  TRY(lpt_join(c, st));
  if (c->mid_ev) {
    CK(cudaEventRecord(c->m_ev1, c->m_stream));
    CK(cudaStreamWaitEvent(st, c->m_ev1, 0));
  }
  return rc;
}

int nv_set_cast_mode(nv_ctx *c, int mode) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  if (mode != NV_CAST_AUTO && mode != NV_CAST_THREAD && mode != NV_CAST_WARP)
    return fail(NV_ERR_ARG, "cast mode must be NV_CAST_AUTO (0), NV_CAST_THREAD (1) or "
                            "NV_CAST_WARP (2)");
  c->gen++;
  c->cast_mode = mode;
  return NV_OK;
}

int nv_set_fill_mode(nv_ctx *c, int mode) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  if (mode != NV_FILL_AUTO && mode != NV_FILL_GENERIC)
    return fail(NV_ERR_ARG, "fill mode must be NV_FILL_AUTO (0) or NV_FILL_GENERIC (1)");
  c->gen++;
  c->fill_mode = mode;
  return NV_OK;
}

int nv_set_overlap(nv_ctx *c, int on) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  c->gen++;
  c->pdl = on != 0;
  return NV_OK;
}

int nv_step_render_host(nv_ctx *c, const int8_t *actions_host, int cam, uint32_t channels,
                        uint8_t *rgb_host, float *depth_host, uint16_t *sem_host,
                        double *gps_host, double *compass_host, uint8_t *collided_host,
                        double *displacement_host, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  if (!actions_host) return fail(NV_ERR_ARG, "actions is NULL");
  const bool frames_out = rgb_host || depth_host || sem_host;
  // the cameras this step renders, in order; the first one carries the step
  // (nv_step_render) and gps/compass, the others are nv_render calls
  int cams[8], ncam = 0;
  uint32_t chans[8];
  if (cam == NV_ALL_CAMERAS) {
    if (frames_out) return fail(NV_ERR_ARG, "host frame pointers need a single camera");
    for (int k = 0; k < 8; ++k) {
      const uint32_t b = (channels >> (3 * k)) & 7u;
      if (!b) continue;
      if (!c->cams[k].on) return fail(NV_ERR_STATE, "camera %d not configured (nv_camera_config)", k);
      cams[ncam] = k;
      chans[ncam++] = b;
    }
    if (!ncam) return fail(NV_ERR_ARG, "no camera channels requested");
  } else {
    cams[0] = cam;
    chans[0] = (channels & 7u) | (rgb_host ? NV_CH_RGB : 0u) | (depth_host ? NV_CH_DEPTH : 0u) |
               (sem_host ? NV_CH_SEM : 0u);
    ncam = 1;
  }
  for (int q = 0; q < ncam; ++q) TRY(cam_check(c, cams[q]));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t N = (size_t)c->n_envs;
  // graph path: no host frames, no profiling, no noise (its frame counter
  // advances per call) -- the common per-step case
  const bool graph_ok = !frames_out && !c->prof_on && !(c->noise_sigma > 0.0);
  // (one camera: with several, the next step's agent step would have to wait
  // for every camera's casts, not just the first one's)
  const int nsets = graph_ok && NV_E2E_PINGPONG && ncam == 1 ? 2 : 1;
  for (int q = 0; q < ncam; ++q) {
    Camera &k = c->cams[cams[q]];
    const size_t px = N * k.W * k.H;
    for (int f = 0; f < nsets; ++f) {
      if (chans[q] & NV_CH_RGB) TRY(k.e_rgb[f].alloc(px * 3));
      if (chans[q] & NV_CH_DEPTH) TRY(k.e_depth[f].alloc(px * 4));
      if (chans[q] & NV_CH_SEM) TRY(k.e_sem[f].alloc(px * 2));
    }
  }
  auto frame_ptrs = [&](int q, int f, uint8_t *&r, float *&d, uint16_t *&s) {
    Camera &k = c->cams[cams[q]];
    r = (chans[q] & NV_CH_RGB) ? k.e_rgb[f].as<uint8_t>() : nullptr;
    d = (chans[q] & NV_CH_DEPTH) ? k.e_depth[f].as<float>() : nullptr;
    s = (chans[q] & NV_CH_SEM) ? k.e_sem[f].as<uint16_t>() : nullptr;
  };
  TRY(c->e_act.alloc(N));
  const size_t pack = 33 * N;
  TRY(c->e_pack.alloc(pack));
  uint8_t *pk = c->e_pack.as<uint8_t>();
  double *d_gps = reinterpret_cast<double *>(pk), *d_comp = d_gps + 2 * N, *d_disp = d_comp + N;
  uint8_t *d_coll = pk + 32 * N;
  if (graph_ok) {
    if (!c->e_stream[0]) {
      // blocking streams: ordered after the legacy default stream's work
      // implicitly, so callers on stream 0 need no event handshake
      for (int p = 0; p < 2; ++p) {
        CK(cudaStreamCreate(&c->e_stream[p]));
        CK(cudaEventCreateWithFlags(&c->e_cast_ev[p], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->e_order_ev[p], cudaEventDisableTiming));
      }
      CK(cudaEventCreateWithFlags(&c->e_ev, cudaEventDisableTiming));
    }
    // pinned, mapped staging: with e2e_mapped the kernels read the actions
    // from and write the packed step results to host memory directly (no
    // copy nodes in the graph)
    if (c->e_hin_bytes < N) {
      TRY(e2e_fence(c));
      if (c->e_hin) cudaFreeHost(c->e_hin);
      CK(cudaHostAlloc(&c->e_hin, N, cudaHostAllocMapped));
      c->e_hin_bytes = N;
    }
    if (c->e_hout_bytes < pack) {
      TRY(e2e_fence(c));
      if (c->e_hout) cudaFreeHost(c->e_hout);
      CK(cudaHostAlloc(&c->e_hout, pack, cudaHostAllocMapped));
      c->e_hout_bytes = pack;
    }
    // step results straight into the caller's buffers when all four are
    // pinned (mapped) host memory: no staging copy after the step
    void *const outs[4] = {gps_host, compass_host, displacement_host, collided_host};
    bool direct = c->e2e_mapped;
    for (int q = 0; q < 4 && direct; ++q) {
      if (!outs[q]) {
        direct = false;
        break;
      }
      if (outs[q] != c->e_out_host[q]) {  // look up (and remember) the device alias
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, outs[q]) != cudaSuccess ||
            at.type != cudaMemoryTypeHost || !at.devicePointer) {
          cudaGetLastError();
          direct = false;
          c->e_out_host[q] = nullptr;
          break;
        }
        c->e_out_host[q] = outs[q];
        c->e_out_dev[q] = at.devicePointer;
      }
    }
    // everything the graph's kernels touch exists before the key is taken
    // (a reallocated buffer changes the key: the graph is never replayed
    // into freed memory)
    for (int q = 0; q < ncam; ++q) {
      Camera &k = c->cams[cams[q]];
      TRY(k.rec_e2e.alloc(k.rec.bytes));
      const unsigned nblk = cast_blocks(c, c->n_envs * (long long)k.W);
      if (NV_CAST_LPT && lpt_pays(c, nblk) && k.lpt_n_e2e != (int64_t)nblk) {
        TRY(e2e_fence(c));
        TRY(lpt_buffers(c, k.lpt_order_e2e, k.lpt_cost_e2e, k.lpt_n_e2e, nblk, nullptr));
        CK(cudaDeviceSynchronize());
      }
    }
    // the handshake buffers of the device path and of the host steps
    auto swap_pdl = [&]() {
      std::swap(c->pdl_ready.p, c->pdl_ready_e2e.p);
      std::swap(c->pdl_ready.bytes, c->pdl_ready_e2e.bytes);
      std::swap(c->pdl_arrive.p, c->pdl_arrive_e2e.p);
      std::swap(c->pdl_arrive.bytes, c->pdl_arrive_e2e.bytes);
      std::swap(c->pose_rec.p, c->pose_rec_e2e.p);
      std::swap(c->pose_rec.bytes, c->pose_rec_e2e.bytes);
      std::swap(c->pdl_init, c->pdl_init_e2e);
      std::swap(c->pose_init, c->pose_init_e2e);
    };
    if (c->pdl) {
      swap_pdl();
      const int prc = pdl_buffers(c);
      swap_pdl();
      TRY(prc);
    }
    for (int q = 0; q < ncam; ++q) {
      Camera &k = c->cams[cams[q]];
      TRY(rel_buffers(k.rel_e2e, k.rel_n_e2e, c->n_envs));
    }
    std::vector<uint64_t> key = {(uint64_t)c->n_envs, (uint64_t)c->gen, (uint64_t)ncam,
                                 (uint64_t)c->e2e_mapped, (uint64_t)direct,
                                 (uint64_t)(uintptr_t)c->e_hin, (uint64_t)(uintptr_t)c->e_hout,
                                 (uint64_t)(uintptr_t)c->e_act.p, (uint64_t)(uintptr_t)c->e_pack.p,
                                 (uint64_t)(uintptr_t)c->pdl_ready_e2e.p,
                                 (uint64_t)(uintptr_t)c->pose_rec_e2e.p};
    if (direct)
      for (int q = 0; q < 4; ++q) key.push_back((uint64_t)(uintptr_t)c->e_out_dev[q]);
    for (int q = 0; q < ncam; ++q) {
      const Camera &k = c->cams[cams[q]];
      for (uint64_t v : {(uint64_t)cams[q], (uint64_t)chans[q], (uint64_t)(uintptr_t)k.rec_e2e.p,
                         (uint64_t)(uintptr_t)k.rel_e2e.p,
                         (uint64_t)(uintptr_t)k.lpt_order_e2e.p, (uint64_t)(uintptr_t)k.lpt_cost_e2e.p})
        key.push_back(v);
      for (int f = 0; f < nsets; ++f) {
        uint8_t *r; float *d; uint16_t *sm;
        frame_ptrs(q, f, r, d, sm);
        for (uint64_t v : {(uint64_t)(uintptr_t)r, (uint64_t)(uintptr_t)d, (uint64_t)(uintptr_t)sm})
          key.push_back(v);
      }
    }
    const bool same = c->e_graph[0] && key == c->e_key;
    if (!same) {
      TRY(e2e_fence(c));  // the old graphs' writers may still be running
      for (int p = 0; p < 2; ++p) {
        if (c->e_graph[p]) cudaGraphExecDestroy(c->e_graph[p]);
        c->e_graph[p] = nullptr;
      }
      c->e_par = 0;
      c->e_key.clear();
      const int8_t *acts = c->e_act.as<int8_t>();
      double *o_gps = d_gps, *o_comp = d_comp, *o_disp = d_disp;
      uint8_t *o_coll = d_coll;
      if (c->e2e_mapped) {
        void *din = nullptr, *dout = nullptr;
        CK(cudaHostGetDevicePointer(&din, c->e_hin, 0));
        CK(cudaHostGetDevicePointer(&dout, c->e_hout, 0));
        if (!NV_E2E_ACT_COPY) acts = static_cast<const int8_t *>(din);
        o_gps = static_cast<double *>(dout);
        o_comp = o_gps + 2 * N;
        o_disp = o_comp + N;
        o_coll = static_cast<uint8_t *>(dout) + 32 * N;
        if (direct) {
          o_gps = static_cast<double *>(c->e_out_dev[0]);
          o_comp = static_cast<double *>(c->e_out_dev[1]);
          o_disp = static_cast<double *>(c->e_out_dev[2]);
          o_coll = static_cast<uint8_t *>(c->e_out_dev[3]);
        }
      }
      // the graph's casts and writers use the host step's own record buffers
      // and block orders; an event after the first camera's casts tells the
      // host the step results are in
      auto swap_e2e = [&]() {
        for (int q = 0; q < ncam; ++q) {
          Camera &k = c->cams[cams[q]];
          std::swap(k.rec.p, k.rec_e2e.p);
          std::swap(k.rec.bytes, k.rec_e2e.bytes);
          std::swap(k.rel.p, k.rel_e2e.p);
          std::swap(k.rel.bytes, k.rel_e2e.bytes);
          std::swap(k.rel_n, k.rel_n_e2e);
          std::swap(k.lpt_order.p, k.lpt_order_e2e.p);
          std::swap(k.lpt_order.bytes, k.lpt_order_e2e.bytes);
          std::swap(k.lpt_cost.p, k.lpt_cost_e2e.p);
          std::swap(k.lpt_cost.bytes, k.lpt_cost_e2e.bytes);
          std::swap(k.lpt_n, k.lpt_n_e2e);
        }
        swap_pdl();
      };
      // graph p: record half and release counters of the p-th render after
      // the capture began (do_cast alternates them), frame set p
      for (int p = 0; p < nsets; ++p) {
        cudaStream_t es = c->e_stream[p];
        CK(cudaStreamBeginCapture(es, cudaStreamCaptureModeThreadLocal));
        if (!c->e2e_mapped || NV_E2E_ACT_COPY)
          cudaMemcpyAsync(c->e_act.p, c->e_hin, N, cudaMemcpyHostToDevice, es);
        swap_e2e();
        c->mid_ev = c->e2e_mapped ? c->e_cast_ev[p] : nullptr;
        c->order_ev = nsets == 2 ? c->e_order_ev[p] : nullptr;
        uint8_t *r; float *d; uint16_t *sm;
        frame_ptrs(0, p, r, d, sm);
        int rc = nv_step_render(c, acts, cams[0], r, d, sm, o_gps, o_comp, o_coll, o_disp, nullptr, es);
        c->mid_ev = nullptr;
        c->order_ev = nullptr;
        for (int q = 1; q < ncam && rc == NV_OK; ++q) {
          frame_ptrs(q, p, r, d, sm);
          rc = nv_render(c, cams[q], r, d, sm, nullptr, nullptr, es);
        }
        swap_e2e();
        if (!c->e2e_mapped) cudaMemcpyAsync(c->e_hout, pk, pack, cudaMemcpyDeviceToHost, es);
        cudaGraph_t g = nullptr;
        cudaError_t ce = cudaStreamEndCapture(es, &g);
        if (rc != NV_OK) {
          if (g) cudaGraphDestroy(g);
          return rc;
        }
        if (ce != cudaSuccess) return fail(NV_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(ce));
        ce = cudaGraphInstantiate(&c->e_graph[p], g, 0);
        cudaGraphDestroy(g);
        if (ce != cudaSuccess) return fail(NV_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(ce));
      }
      c->e_key = key;
    }
    // the previous host step's casts are complete (the host waited for them)
    // and its writer uses the other record half and frame set: this step's
    // agent step and casts may run beside that writer
    const int p = nsets == 2 ? c->e_par : 0;
    cudaStream_t es = c->e_stream[p];
    std::memcpy(c->e_hin, actions_host, N);
    if (st) {  // after the caller's prior work on its own stream
      CK(cudaEventRecord(c->e_ev, st));
      CK(cudaStreamWaitEvent(es, c->e_ev, 0));
    }
    // the previous step's casts are complete (the host waited for them); its
    // ordering kernel, which writes the block order this step's casts read,
    // may still run
    if (nsets == 2) CK(cudaStreamWaitEvent(es, c->e_order_ev[p ^ 1], 0));
    CK(cudaGraphLaunch(c->e_graph[p], es));
    c->launches += 3 * ncam;
    c->e_last = p;
    c->e_par = p ^ (nsets - 1);
    if (c->e2e_mapped) {
      // the step results are in host memory once the casts are done; the
      // frame writer finishes behind the caller (the next-but-one host step
      // is ordered after it on its stream; nv_host_frames and reallocating
      // calls wait for it)
      CK(cudaEventSynchronize(c->e_cast_ev[p]));
      c->e_pending = true;
    } else {
      CK(cudaStreamSynchronize(es));
    }
    if (direct) return NV_OK;  // the kernels wrote the caller's buffers
    const uint8_t *h = static_cast<const uint8_t *>(c->e_hout);
    if (gps_host) std::memcpy(gps_host, h, 16 * N);
    if (compass_host) std::memcpy(compass_host, h + 16 * N, 8 * N);
    if (displacement_host) std::memcpy(displacement_host, h + 24 * N, 8 * N);
    if (collided_host) std::memcpy(collided_host, h + 32 * N, N);
    return NV_OK;
  }
  TRY(e2e_fence(c));
  c->e_last = 0;
  CK(cudaMemcpyAsync(c->e_act.p, actions_host, N, cudaMemcpyHostToDevice, st));
  {
    uint8_t *r; float *d; uint16_t *sm;
    frame_ptrs(0, 0, r, d, sm);
    TRY(nv_step_render(c, c->e_act.as<int8_t>(), cams[0], r, d, sm, d_gps, d_comp, d_coll, d_disp,
                       nullptr, stream));
    for (int q = 1; q < ncam; ++q) {
      frame_ptrs(q, 0, r, d, sm);
      TRY(nv_render(c, cams[q], r, d, sm, nullptr, nullptr, stream));
    }
  }
  {
    const Camera &k = c->cams[cams[0]];
    const size_t px = N * k.W * k.H;
    if (rgb_host) CK(cudaMemcpyAsync(rgb_host, k.e_rgb[0].p, px * 3, cudaMemcpyDeviceToHost, st));
    if (depth_host) CK(cudaMemcpyAsync(depth_host, k.e_depth[0].p, px * 4, cudaMemcpyDeviceToHost, st));
    if (sem_host) CK(cudaMemcpyAsync(sem_host, k.e_sem[0].p, px * 2, cudaMemcpyDeviceToHost, st));
  }
  if (gps_host || compass_host || collided_host || displacement_host) {
    std::vector<uint8_t> h(pack);
    CK(cudaMemcpyAsync(h.data(), pk, pack, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (gps_host) std::memcpy(gps_host, h.data(), 16 * N);
    if (compass_host) std::memcpy(compass_host, h.data() + 16 * N, 8 * N);
    if (displacement_host) std::memcpy(displacement_host, h.data() + 24 * N, 8 * N);
    if (collided_host) std::memcpy(collided_host, h.data() + 32 * N, N);
  }
  CK(cudaStreamSynchronize(st));
  return NV_OK;
}

int nv_host_frames(nv_ctx *c, int cam, uint8_t **rgb, float **depth, uint16_t **sem) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  if (cam < 0 || cam >= 8) return fail(NV_ERR_ARG, "camera index %d out of range [0, 8)", cam);
  TRY(e2e_fence(c));  // the frames are complete when this returns
  const Camera &k = c->cams[cam];
  if (rgb) *rgb = k.e_rgb[c->e_last].as<uint8_t>();
  if (depth) *depth = k.e_depth[c->e_last].as<float>();
  if (sem) *sem = k.e_sem[c->e_last].as<uint16_t>();
  return NV_OK;
}

int nv_gps_compass(nv_ctx *c, double *gps, double *compass, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  nvk::k_gps_compass<<<blocks_for(c->n_envs, 128), 128, 0, (cudaStream_t)stream>>>(
      c->env_view(), gps, compass);
  return check_launch(c);
}

int nv_get_state(nv_ctx *c, double *xy, double *heading, double *path_len, int64_t *collisions,
                 void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t N = (size_t)c->n_envs;
  if (xy) {
    CK(cudaMemcpy2DAsync(xy, 16, c->x.p, 8, 8, N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpy2DAsync(xy + 1, 16, c->y.p, 8, 8, N, cudaMemcpyDeviceToDevice, st));
  }
  if (heading) CK(cudaMemcpyAsync(heading, c->h.p, 8 * N, cudaMemcpyDeviceToDevice, st));
  if (path_len) CK(cudaMemcpyAsync(path_len, c->path.p, 8 * N, cudaMemcpyDeviceToDevice, st));
  if (collisions) CK(cudaMemcpyAsync(collisions, c->coll.p, 8 * N, cudaMemcpyDeviceToDevice, st));
  return NV_OK;
}

int nv_get_frame(nv_ctx *c, double *origin_xy, double *heading, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_envs(c));
  cudaStream_t st = (cudaStream_t)stream;
  const size_t N = (size_t)c->n_envs;
  if (origin_xy) {
    CK(cudaMemcpy2DAsync(origin_xy, 16, c->ox.p, 8, 8, N, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpy2DAsync(origin_xy + 1, 16, c->oy.p, 8, 8, N, cudaMemcpyDeviceToDevice, st));
  }
  if (heading) CK(cudaMemcpyAsync(heading, c->oh.p, 8 * N, cudaMemcpyDeviceToDevice, st));
  return NV_OK;
}

int nv_raycast(nv_ctx *c, const double *ox, const double *oy, const double *dirx,
               const double *diry, int64_t m, double t_max, int brute, double *t_out,
               int64_t *idx_out, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_scene(c));
  if (m < 0) return fail(NV_ERR_ARG, "m < 0");
  if (m == 0) return NV_OK;
  nvk::k_raycast<<<blocks_for(m, 128), 128, 0, (cudaStream_t)stream>>>(
      c->scene_view(), ox, oy, dirx, diry, m, t_max, brute, t_out, idx_out);
  return check_launch(c);
}

int nv_fill_frames(nv_ctx *c, int cam, int64_t n, const double *t_col, const int64_t *i_col,
                   const double *dirx, const double *diry, double sensor_height, uint8_t *rgb,
                   float *depth, uint16_t *sem, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_scene(c));
  if (cam < 0 || cam >= 8 || !c->cams[cam].on) return fail(NV_ERR_STATE, "camera %d not configured", cam);
  if (n <= 0) return NV_OK;
  if (sensor_height > c->wall_h) return fail(NV_ERR_ARG, "sensor height must stay below wall height");
  Camera &k = c->cams[cam];
  cudaStream_t st = (cudaStream_t)stream;
  if (k.tables_cam_h != sensor_height) {
    CK(cudaStreamSynchronize(st));
    TRY(build_camera_tables(c, k, sensor_height));
  }
  TRY(k.rec.alloc(2 * sizeof(ColRec) * (size_t)n * k.W));
  rec_flip(k);
  long long total = n * (long long)k.W;
  nvk::k_cols_from_hits<<<blocks_for(total, 256), 256, 0, st>>>(
      c->scene_view(), cam_view(k), total, t_col, i_col, dirx, diry, rec_out(k, n));
  TRY(check_launch(c));
  return launch_fill(c, k, n, rgb, depth, sem, st);
}

int nv_cast_disc(nv_ctx *c, const double *px, const double *py, const double *ux,
                 const double *uy, const double *radius, int64_t m, double *t_out,
                 int64_t *seg_out, double *tan_out, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_scene(c));
  if (m <= 0) return NV_OK;
  nvk::k_cast_disc<<<blocks_for(m * 32, 128), 128, 0, (cudaStream_t)stream>>>(
      c->scene_view(), px, py, ux, uy, radius, m, t_out, seg_out, tan_out);
  return check_launch(c);
}

int nv_clearance(nv_ctx *c, const double *px, const double *py, int64_t m, double search_radius,
                 double *out, void *stream) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  TRY(ensure_scene(c));
  if (m <= 0) return NV_OK;
  nvk::k_clearance<<<blocks_for(m * 32, 128), 128, 0, (cudaStream_t)stream>>>(
      c->scene_view(), px, py, m, search_radius, out);
  return check_launch(c);
}

void nv_host_sincos(double x, double *s, double *c) { nvx::sincos_cr(x, s, c); }
double nv_host_hypot(double x, double y) { return nvx::hypot_cr(x, y); }

int64_t nv_launch_count(nv_ctx *c) { return c ? c->launches : 0; }

int nv_faults(nv_ctx *c, uint32_t *mask) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  if (!mask) return fail(NV_ERR_ARG, "mask is NULL");
  TRY(e2e_fence(c));
  CK(cudaDeviceSynchronize());
  uint32_t m = 0;
  auto take = [&](unsigned *word, uint32_t bit) -> int {
    unsigned v = 0;
    CK(cudaMemcpy(&v, word, sizeof v, cudaMemcpyDeviceToHost));
    if (v) {
      m |= bit;
      CK(cudaMemset(word, 0, sizeof v));
    }
    return NV_OK;
  };
  for (Camera &k : c->cams) {
    if (k.rel.p && k.rel_n > 0) TRY(take(k.rel.as<unsigned>() + 4 * (size_t)k.rel_n, NV_FAULT_WRITER_WAIT));
    if (k.rel_e2e.p && k.rel_n_e2e > 0)
      TRY(take(k.rel_e2e.as<unsigned>() + 4 * (size_t)k.rel_n_e2e, NV_FAULT_WRITER_WAIT));
  }
  if (c->pdl_ready.p && c->pdl_init) TRY(take(pdl_fault(c), NV_FAULT_CAST_WAIT));
  if (c->pdl_ready_e2e.p && c->pdl_init_e2e) {
    const size_t n = (size_t)std::max<int64_t>(1, c->n_envs);
    TRY(take(c->pdl_ready_e2e.as<unsigned>() + 3 * n, NV_FAULT_CAST_WAIT));
  }
  *mask = m;
  return NV_OK;
}

int nv_profile(nv_ctx *c, int enable) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  c->prof_on = enable != 0;
  c->prof_used = 0;
  for (int k = 0; k < 4; ++k) {
    c->prof_ms[k] = 0.0;
    c->prof_n[k] = 0;
  }
  return NV_OK;
}

int nv_profile_read(nv_ctx *c, double *ms, int64_t *counts) {
  if (!c) return fail(NV_ERR_ARG, "ctx is NULL");
  for (size_t p = 0; p < c->prof_used; ++p) {
    CK(cudaEventSynchronize(c->prof_ev[2 * p + 1]));
    float m = 0.0f;
    CK(cudaEventElapsedTime(&m, c->prof_ev[2 * p], c->prof_ev[2 * p + 1]));
    int k = c->prof_kind[p];
    c->prof_ms[k] += m;
    c->prof_n[k] += 1;
  }
  c->prof_used = 0;
  for (int k = 0; k < 4; ++k) {
    if (ms) ms[k] = c->prof_ms[k];
    if (counts) counts[k] = c->prof_n[k];
  }
  return NV_OK;
}

}  // extern "C"

#include "nav_task_abi.inc"
#include "codec_abi.inc"
