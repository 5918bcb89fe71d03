// kernels.cuh -- sm_100a kernels of the navsim hot path (umbrella header).
//
//   geom.cuh   the exact FP64 geometry shared by every kernel: the segment test
//              of raycast_grid / raycast_all (_kernels.py:16-120) with its
//              exactness-preserving f32 prefilters, the DDA, disc_cast
//              (_kernels.py:393-465) and min_seg_distance (_kernels.py:468-493).
//   agent.cuh  Simulator.step kinematics (sim.py:83-219): k_agent_step, one warp
//              per env (swept-disc casts with a warp (t, idx) minimum, slide),
//              and k_set_poses (set_agent_state's clearance check).
//   cast.cuh   the column casts: _column_directions + raycast_grid + the exact
//              row classification of fill_frame -> column records
//              (k_column_cast thread per ray, k_column_cast_warp warp per ray
//              for small batches) and the operator-level kernels (raycast,
//              disc casts, clearance, fill from given hits).
//   fill.cuh   fill_frame's per-pixel resolve (_kernels.py:128-207) as HBM
//              writers: k_fill_ws (warp-specialised: producer warps -> smem slots
//              -> one TMA store warp), k_fill_generic (any size), inverse-depth
//              noise.
//
// Exactness: every FP64 operation that decides coverage, semantics, depth or
// pose uses the nvx:: _rn helpers (no FMA contraction), replicating the
// reference's operation order.  Shading is packed f16 (RGB tolerance 1/255).
#pragma once

#include "fill.cuh"  // geom -> agent -> cast -> fill
