/* navsim_b200.h -- C ABI of the B200-native navsim hot path.
 *
 * Drop-in boundary for the reference's two-level hot-path interface
 * (/root/reference/pkg/src/navsim):
 *   - the numba "operator" layer  (_kernels.raycast_grid :51, raycast_all :16,
 *     fill_frame :128, disc_cast :393, min_seg_distance :468), and
 *   - the Python Simulator / render API built on it (sim.py:133-219,
 *     sensors.py:105-152, geometry.py:100-206).
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - Every call returns 0 on success or a negative NV_ERR_* code; the message
 *     of the last failure on the calling host thread is nv_last_error().
 *   - A context is owned by ONE host thread at a time, mirroring the
 *     reference's exclusive-owner rule for a Simulator (sim.py:134-137).
 *   - "dev" pointers are CUDA device pointers (e.g. torch tensor data_ptr());
 *     "host" pointers are ordinary host memory.  Hot per-step calls take
 *     device pointers and a cudaStream_t (passed as void*; NULL = legacy
 *     default stream) and never synchronise the host.
 *   - Actions use the reference enum order (sim.py:31-35):
 *     0 MOVE_FORWARD, 1 TURN_LEFT, 2 TURN_RIGHT, 3 STOP.
 *   - Frames: rgb u8 [N,H,W,3] (reference: f64 in [0,1], tolerance 1/255),
 *     depth f32 [N,H,W] metres (reference f64, tolerance 1e-5 rel),
 *     semantic u16 [N,H,W] (exact).  Any frame pointer may be NULL to skip
 *     that channel (fill_frame's want_* flags, _kernels.py:131).
 */
#ifndef NAVSIM_B200_H
#define NAVSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NV_OK 0
#define NV_ERR_ARG -1        /* invalid argument (SensorError/SimError class)  */
#define NV_ERR_CUDA -2       /* CUDA runtime failure                           */
#define NV_ERR_STATE -3      /* call order: no scene / envs / camera / reset   */
#define NV_ERR_OOM -4        /* device allocation failed                       */

#define NV_ACTION_MOVE_FORWARD 0
#define NV_ACTION_TURN_LEFT 1
#define NV_ACTION_TURN_RIGHT 2
#define NV_ACTION_STOP 3

/* per-env status written by nv_set_poses / nv_step */
#define NV_ENV_OK 0
#define NV_ENV_TOO_CLOSE 1   /* clearance < radius (sim.py:176-180)            */
#define NV_ENV_NOT_RESET 2   /* step before reset (sim.py:203-204)             */
#define NV_ENV_BAD_ACTION 3  /* unknown action (sim.py:215-216)                */

typedef struct nv_ctx nv_ctx;

const char *nv_last_error(void);
int nv_version(void);

/* Context on CUDA device `device` (one per process per GPU). */
int nv_create(int device, nv_ctx **out);
int nv_destroy(nv_ctx *ctx);

/* Scene upload -- replaces RenderGeometry.__init__ (sensors.py:81-93) +
 * SegmentIndex.__init__ (geometry.py:109-141) + segment_normals
 * (geometry.py:66-73).  segs: n x (ax, ay, bx, by) f64 world coordinates
 * (scene.flatten_arrays output, scene.py:349-378); sem: n u16; albedo: n x 3
 * f64; floor3/ceil3: 3 f64.  All HOST pointers.  The 1 m uniform grid is built
 * on the host exactly like SegmentIndex and uploaded once. */
int nv_scene_upload(nv_ctx *ctx, const double *segs, const uint16_t *sem,
                    const double *albedo, int64_t n, double wall_height,
                    const double *floor3, const double *ceil3);
/* Grid introspection (parity tests): x0, y0, nx, ny, item count. */
int nv_scene_grid_info(nv_ctx *ctx, double *x0, double *y0, int64_t *nx,
                       int64_t *ny, int64_t *nitems);

/* Agent kinematics -- AgentConfig (sim.py:49-61).  turn_rad is
 * math.radians(turn_angle) computed by the caller. */
int nv_agent_config(nv_ctx *ctx, double radius, double forward_step,
                    double turn_rad, double sensor_height);

/* Allocate device state for n_envs environments (all un-reset: origin,
 * heading 0, the reference Simulator's initial AgentState, sim.py:159).  May
 * be called again; it drops the PointGoal episodes of the previous batch
 * (nv_task_reset starts new ones). */
int nv_envs_alloc(nv_ctx *ctx, int64_t n_envs);

/* Camera (sensor group sharing one traversal, sensors.py:121-123).
 * cam in [0, 8).  focal = SensorConfig.focal (sensors.py:55-57) computed by
 * the caller.  Fails (NV_ERR_ARG) if sensor_height > wall_height
 * (sensors.py:119-120). */
int nv_camera_config(nv_ctx *ctx, int cam, int width, int height, double focal,
                     double max_range);

/* Reset -- Simulator.set_agent_state (sim.py:172-184), batched.
 * HOST arrays of n_envs: xy (n x 2), heading, mask (NULL = all; 0 = leave env
 * untouched).  status_out (HOST, n_envs i32, may be NULL) receives NV_ENV_*;
 * clearance_out (HOST, may be NULL) the clearance used for the check.
 * Synchronous.  Returns NV_ERR_ARG if any masked env failed its check. */
int nv_set_poses(nv_ctx *ctx, const double *xy, const double *heading,
                 const uint8_t *mask, int32_t *status_out,
                 double *clearance_out);

/* Step -- Simulator.step's kinematics (sim.py:202-219: apply_forward :90,
 * apply_turn :83), batched over all envs.  actions: DEVICE i8[n_envs].
 * Outputs (DEVICE, each may be NULL): collided u8[n], displacement f64[n],
 * status i32[n] (NV_ENV_*).  Envs never reset report NV_ENV_NOT_RESET and are
 * not moved. */
int nv_step(nv_ctx *ctx, const int8_t *actions, uint8_t *collided,
            double *displacement, int32_t *status, void *stream);

/* Observations -- sensors.render (sensors.py:105-152) for camera `cam` at the
 * current poses of all envs, plus gps_compass (sensors.py:175-180).  DEVICE
 * outputs, each may be NULL: rgb u8[n,H,W,3], depth f32[n,H,W],
 * sem u16[n,H,W], gps f64[n,2], compass f64[n]. */
int nv_render(nv_ctx *ctx, int cam, uint8_t *rgb, float *depth, uint16_t *sem,
              double *gps, double *compass, void *stream);

/* Step + render: one call per simulator step for all envs -- nv_step then
 * nv_render for camera `cam`, enqueued as three launches on `stream`: the
 * agent step (k_agent_step, a warp per env in one-warp CTAs; a programmatic
 * dependent of the previous step's frame writer, which it never reads from --
 * consecutive renders alternate between two column-record buffers -- so it
 * runs beside the writer and on the SMs its tail frees, and completes after
 * it), the column
 * cast (a programmatic dependent of the agent step that starts each env's
 * rays as soon as its new pose is published, see nv_set_overlap) and the
 * frame writer (the
 * warp-specialised TMA writer k_fill_ws when the frame layout allows it:
 * W in {64, 128, 256k <= 4096}, whole 16-row slots, 16-byte aligned outputs;
 * else the per-pixel k_fill_generic). */
int nv_step_render(nv_ctx *ctx, const int8_t *actions, int cam, uint8_t *rgb,
                   float *depth, uint16_t *sem, double *gps, double *compass,
                   uint8_t *collided, double *displacement, int32_t *status,
                   void *stream);

/* Programmatic-dependent-launch chaining in nv_step_render (and in
 * nv_task_step_render), on by default: each env's casts start as soon as its
 * agent warp has published the new pose (a per-env pose record the casts
 * reload until it is complete, or an acquired ready flag); the frame writer
 * takes each env as soon as its casts have published their column records
 * (thread-per-ray batches); the next step's agent step runs beside the
 * previous writer when that writer's grid fills the GPU (after it
 * otherwise, and while a host step's writer may still run).  The ordering
 * across steps assumes the context has the whole GPU: with MPS SM limits or
 * other contexts running concurrently, turn it off.  0 turns all of it off
 * (serialised launches; identical results). */
int nv_set_overlap(nv_ctx *ctx, int on);
/* Column cast (raycast_grid's DDA over the grid, bit-exact in every mode):
 * NV_CAST_AUTO (default) = one thread per ray, or one warp per ray (lanes
 * split each cell's entries) when the batch has at most 16384 rays
 * (latency-bound sizes); NV_CAST_THREAD / NV_CAST_WARP force one of the two
 * (parity tests compare them). */
#define NV_CAST_AUTO 0
#define NV_CAST_THREAD 1
#define NV_CAST_WARP 2
int nv_set_cast_mode(nv_ctx *ctx, int mode);
/* Frame writer: NV_FILL_AUTO (default) = the warp-specialised TMA writer
 * (16 producer warps render rows into a ring of smem slots, one store warp
 * writes each slot with one bulk copy per channel; one CTA per SM, small
 * batches split each frame into row bands) whenever the frame layout allows
 * it, else the per-pixel kernel; NV_FILL_GENERIC forces the per-pixel kernel.
 * Both produce identical frames. */
#define NV_FILL_AUTO 0
#define NV_FILL_GENERIC 1
int nv_set_fill_mode(nv_ctx *ctx, int mode);

/* End-to-end call over HOST buffers (the reference-facing path: host actions
 * in, host results out).  Copies actions (host, n i8) in, runs
 * nv_step_render into device frames owned by the context (channels: bitmask
 * of NV_CH_*; a non-NULL host frame pointer implies its channel) -- for
 * camera `cam`, or with cam = NV_ALL_CAMERAS for every camera k whose
 * channel bits (channels >> 3k) & 7 are non-zero (the first such camera
 * carries the step and gps/compass, the others are rendered after it; host
 * frame pointers need a single camera) -- copies the
 * per-env step results (collided u8, displacement f64, gps f64x2, compass
 * f64) back to host buffers (any may be NULL) and, where the host frame
 * pointers are non-NULL, the frames too.  Host buffers should be pinned.
 * Returns when the step results are in the host buffers.  Without host frame
 * pointers the step runs as one replayed graph on an internal blocking stream
 * and returns as soon as its casts are done (the results are complete then);
 * the frame writer finishes behind the caller on the step's own record
 * buffer and counters (device steps on any stream may follow at once),
 * before nv_host_frames / nv_camera_config / nv_envs_alloc / nv_scene_upload
 * / nv_destroy return.  With one camera, consecutive host steps alternate
 * between two graphs, streams, record halves and frame sets: the next host
 * step's agent step and casts run beside this step's writer (they depend only
 * on this step's casts), the next-but-one is ordered after it.
 * With host frame pointers the call synchronises before returning. */
#define NV_CH_RGB 1u
#define NV_CH_DEPTH 2u
#define NV_CH_SEM 4u
#define NV_ALL_CAMERAS (-1)
int nv_step_render_host(nv_ctx *ctx, const int8_t *actions_host, int cam,
                        uint32_t channels, uint8_t *rgb_host, float *depth_host,
                        uint16_t *sem_host, double *gps_host,
                        double *compass_host, uint8_t *collided_host,
                        double *displacement_host, void *stream);
/* Device frame buffers of camera `cam` written by the last
 * nv_step_render_host (complete when this returns; for a GPU consumer of the
 * host-driven path; NULL for channels never rendered).  The pointers
 * alternate between two frame sets from one host step to the next: the
 * frames stay valid until the next-but-one host step starts. */
int nv_host_frames(nv_ctx *ctx, int cam, uint8_t **rgb, float **depth, uint16_t **sem);

/* gps_compass (sensors.py:175-180) alone, for suites without visual sensors.
 * DEVICE outputs gps f64[n,2], compass f64[n] (either may be NULL). */
int nv_gps_compass(nv_ctx *ctx, double *gps, double *compass, void *stream);

/* Agent state in/out (DEVICE arrays of n_envs; any may be NULL):
 * position xy f64[n,2], heading f64[n], path length f64[n],
 * collision count i64[n] -- AgentState (sim.py:65-73). */
int nv_get_state(nv_ctx *ctx, double *xy, double *heading, double *path_len,
                 int64_t *collisions, void *stream);
/* Episode frame origin/heading (EpisodeFrame, sensors.py:155-172). */
int nv_get_frame(nv_ctx *ctx, double *origin_xy, double *heading, void *stream);

/* ---- operator-level entry points (numba kernels, _kernels.py) ---------- */

/* raycast_grid (_kernels.py:51-120; SegmentIndex.raycast geometry.py:165) or,
 * with brute != 0, raycast_all (_kernels.py:16-48).  m rays, ray k starts at
 * (ox[k], oy[k]) with direction (dirx[k], diry[k]).  DEVICE arrays.
 * Outputs t f64[m] (inf on miss), idx i64[m] (-1 on miss). */
int nv_raycast(nv_ctx *ctx, const double *ox, const double *oy,
               const double *dirx, const double *diry, int64_t m, double t_max,
               int brute, double *t_out, int64_t *idx_out, void *stream);

/* fill_frame (_kernels.py:128-207) for n frames of camera `cam` from given
 * per-column hits: t_col f64[n,W], i_col i64[n,W], dirx/diry f64[n,W].
 * sensor_height = cam_h.  DEVICE arrays; outputs as in nv_render. */
int nv_fill_frames(nv_ctx *ctx, int cam, int64_t n, const double *t_col,
                   const int64_t *i_col, const double *dirx, const double *diry,
                   double sensor_height, uint8_t *rgb, float *depth,
                   uint16_t *sem, void *stream);

/* SegmentIndex.cast_disc (geometry.py:183-192) -> disc_cast
 * (_kernels.py:393-465) for m queries.  DEVICE arrays: px, py, ux, uy,
 * radius (f64[m] each).  Outputs t f64[m], seg i64[m], tan f64[m,2]. */
int nv_cast_disc(nv_ctx *ctx, const double *px, const double *py,
                 const double *ux, const double *uy, const double *radius,
                 int64_t m, double *t_out, int64_t *seg_out, double *tan_out,
                 void *stream);

/* SegmentIndex.clearance (geometry.py:194-206) -> min_seg_distance
 * (_kernels.py:468-493) for m points.  DEVICE arrays. */
int nv_clearance(nv_ctx *ctx, const double *px, const double *py, int64_t m,
                 double search_radius, double *out, void *stream);

/* Correctly rounded sin/cos/hypot used on the device agent path, exposed
 * (host implementation) for tests. */
void nv_host_sincos(double x, double *s, double *c);
double nv_host_hypot(double x, double y);

/* Number of kernel launches issued by this context so far (bench evidence). */
int64_t nv_launch_count(nv_ctx *ctx);

/* Handshake faults since the last call (synchronises the device, then
 * clears them): bit NV_FAULT_WRITER_WAIT -- a frame writer waited longer than
 * 200 ms for an env's column records, NV_FAULT_CAST_WAIT -- a column cast
 * waited longer than 200 ms for an env's agent step.  Either means a broken
 * launch sequence (the waits give up rather than hang the GPU; the frames of
 * that step are not valid).  0 in every correct run. */
#define NV_FAULT_WRITER_WAIT 1u
#define NV_FAULT_CAST_WAIT 2u
int nv_faults(nv_ctx *ctx, uint32_t *mask);

/* Per-kernel CUDA-event timing of the hot-path launches (bench roofline
 * evidence).  nv_profile(ctx, 1) clears and enables; nv_profile_read waits
 * for the recorded events and returns accumulated milliseconds and launch
 * counts for [agent_step, column_cast, frame_fill, step_render (fused)]. */
int nv_profile(nv_ctx *ctx, int enable);
int nv_profile_read(nv_ctx *ctx, double *ms4, int64_t *counts4);

/* ---- navigation grid + geodesic distance fields ------ */

#define NV_ENV_DONE 4        /* task episode finished: env frozen (task.py:196-197) */

/* Occupancy grid -- replaces nav.rasterize_navigable (nav.py:65-78) /
 * geometry.navigable_mask (geometry.py:209-250) over HOST bounds
 * (xmin, ymin, xmax, ymax), NULL = the uploaded scene's Scene.bounds
 * (scene.py:69-76).  Builds on the device the per-cell wall clearance
 * (point_segment_distances, geometry.py:76-97) and the navigable mask of
 * the uploaded segments; returns the grid size and the world position of
 * cell (0, 0)'s center.  Synchronous. */
int nv_nav_build(nv_ctx *ctx, const double *bounds, double resolution, double agent_radius,
                 int64_t *nx, int64_t *ny, double *origin2);
/* Copies the mask (u8 ny x nx) and clearance (f64 ny x nx) to HOST buffers
 * sized for an nx x ny grid; NV_ERR_STATE if the context's current grid has
 * another size (it was rebuilt since the caller's nv_nav_build). */
int nv_nav_copy(nv_ctx *ctx, int64_t nx, int64_t ny, uint8_t *mask, double *clearance);
/* nav._snap_to_navigable (nav.py:103-119) for m HOST points (m x 2); HOST
 * cells out (m x 2 i32: i, j, or -1, -1 when nothing is within radius). */
int nv_nav_snap(nv_ctx *ctx, const double *pts, int64_t m, double radius, int32_t *cells);
/* Distance fields -- nav.distance_field / _kernels.dijkstra_grid
 * (nav.py:122-132, _kernels.py:210-282) for k goal cells (HOST k x 2 i32),
 * into DEVICE fields f64[k, ny, nx] (+inf unreachable).  Bit-identical to the
 * reference's Dijkstra (its output is the least fixed point of the
 * relaxation, which the device reaches by tiled Bellman-Ford).  Synchronous
 * on `stream`. */
int nv_nav_fields(nv_ctx *ctx, const int32_t *goal_cells, int64_t k, double *fields,
                  void *stream);
/* nav.geodesic_distance (nav.py:135-166) at m DEVICE points (m x 2) in the
 * fields fid[q] (DEVICE i32); DEVICE out f64[m], NaN = outside the grid
 * (the reference's NavError). */
int nv_nav_geodesic(nv_ctx *ctx, const double *fields, const int32_t *fid, const double *pts,
                    int64_t m, double *out, void *stream);

/* ---- batched PointGoal task (task.py:123-243) ---------- */

/* MAX_EPISODE_STEPS, SUCCESS_RADIUS (task.py:24-25), RewardParams (task.py:52-55). */
int nv_task_config(nv_ctx *ctx, int max_steps, double success_radius, double success_reward,
                   double step_penalty);
/* Environment.reset's task part for the masked envs (HOST arrays of n_envs;
 * mask NULL = all): goal xy (n x 2), episode gdsp, field index into the
 * DEVICE fields (f64[n_fields, ny, nx], caller-owned, must outlive the
 * episodes).  Call after nv_set_poses.  Writes the initial geodesic distance
 * d0 (HOST f64[n], may be NULL).  Synchronous. */
int nv_task_reset(nv_ctx *ctx, const double *goal, const double *gdsp, const int32_t *fid,
                  const double *fields, int64_t n_fields, const uint8_t *mask, double *d0);
/* Environment.step's task arithmetic after nv_step / nv_step_render with the
 * same actions (DEVICE i8[n]) and that call's step status (DEVICE i32[n]):
 * Environment._distance_to_goal (1-ray line of sight, else the field),
 * success, SPL, reward, termination.  DEVICE outputs (each may be NULL):
 * reward f64[n], dist f64[n] (envs the step did not advance -- status != 0 --
 * get reward 0 and their unchanged distance), done u8[n], outcome: 40-byte
 * EpisodeOutcome
 * records written when an env terminates {u8 success, u8 terminated_by
 * (1 stop, 2 step_limit), u8[2], i32 steps, i32 collisions, i32, f64
 * path_taken, f64 shortest_path, f64 spl}.  Finished envs are frozen: later
 * steps report NV_ENV_DONE until the next nv_task_reset. */
int nv_task_step(nv_ctx *ctx, const int8_t *actions, const int32_t *status, double *reward,
                 double *dist, uint8_t *done, void *outcome, void *stream);
/* nv_step_render + nv_task_step in one call: the agent step, then the
 * column cast with the task arithmetic of each env (distance to goal with
 * Environment._distance_to_goal's line-of-sight ray, reward, termination,
 * outcome) riding on its column-0 thread (or warp), then the frame fill.
 * Outputs as in nv_step_render and nv_task_step (the step status is
 * optional here). */
int nv_task_step_render(nv_ctx *ctx, const int8_t *actions, int cam, uint8_t *rgb,
                        float *depth, uint16_t *sem, double *gps, double *compass,
                        uint8_t *collided, double *displacement, int32_t *status,
                        double *reward, double *dist, uint8_t *done, void *outcome,
                        void *stream);
/* Task state (any pointer may be NULL; host or device memory): steps i32[n],
 * done u8[n], last distance f64[n]. */
int nv_task_state(nv_ctx *ctx, int32_t *steps, uint8_t *done, double *d_last, void *stream);

/* ---- inverse-depth noise ------------------------------ */

/* sensors.apply_inverse_depth_noise (sensors.py:183-205) applied to every
 * depth frame the context renders from now on: z' = max_range / (max_range /
 * d + eps), eps ~ N(0, sigma), clamped to [0.05, max_range], saturated pixels
 * untouched; sigma = 0 turns it off (sigma < 0: NV_ERR_ARG, the reference's
 * SensorError).  eps comes from a counter-based generator keyed by (seed,
 * frame counter -- reset here --, env_offset + env, row, pixel pair): the
 * warp-specialised writer fuses it into the frame fill, the other writers run
 * it as a pass; every path gives the same frame.  numpy's normal stream is
 * not reproducible on the device: parity is the reference's moment test. */
int nv_depth_noise(nv_ctx *ctx, double sigma, uint64_t seed, int64_t env_offset);

/* sensors.apply_inverse_depth_noise (sensors.py:183-205) on caller frames: n
 * device f32 depth frames [n, height, width] in place, the same generator
 * and formula as above with stream key (seed, frame, env_offset + k, row,
 * pixel pair); stateless (no context).  sigma = 0: untouched; sigma < 0 or
 * max_range <= 0: NV_ERR_ARG. */
int nv_depth_noise_apply(float *depth, int64_t n, int height, int width, double sigma,
                         double max_range, uint64_t seed, uint64_t frame, int64_t env_offset,
                         void *stream);

/* ---- frame codecs ------------------------------------ */

/* sensors.depth_to_png / rgb_to_png / semantic_to_png (sensors.py:211-246),
 * batched on the device: kind 0 = depth (16-bit gray, round(d / max_range *
 * 65535) clipped), 1 = RGB (8-bit, round(rgb * 255) clipped; u8 input passes
 * through), 2 = semantic (16-bit gray).  frames: DEVICE [n, H, W(, 3)] of f32
 * depth / u8 rgb / u16 semantic, or the reference's f64 arrays with src_f64.
 * out: DEVICE n x stride bytes, each a complete PNG of nv_png_size(kind, W, H)
 * bytes (zlib stored blocks: any PNG decoder returns exactly the quantised
 * samples; Adler-32 and CRC-32 computed on the device).  Asynchronous. */
int64_t nv_png_size(int kind, int width, int height);
int nv_png_encode(int kind, int src_f64, const void *frames, int64_t n, int width, int height,
                  double max_range, uint8_t *out, int64_t stride, void *stream);
/* Host restatement of the device's chunked CRC-32 combination (tests). */
uint32_t nv_host_crc32_chunked(const uint8_t *p, int64_t len, int chunks);

#ifdef __cplusplus
}
#endif
#endif /* NAVSIM_B200_H */
