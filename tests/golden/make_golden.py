"""Generate the golden fixtures from the UNMODIFIED reference (navsim).

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every array below is produced by the reference's own public functions:
``sensors.render`` / ``_column_directions`` (src/sensors.py:96-152),
``SegmentIndex.raycast / raycast_brute / cast_disc / clearance``
(src/geometry.py:165-206) and ``Simulator.step`` (src/sim.py:202-219).
f64 frames are stored as sha256 digests (bit-exact pinning of the oracle) plus
f32 copies (tolerance checks of the CUDA path); semantics are stored exactly.
"""
from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from navsim import nav  # noqa: E402  (reference)
from navsim import sensors as rs  # noqa: E402
from navsim import sim as rsim  # noqa: E402
from navsim.geometry import SegmentIndex  # noqa: E402
from navsim.scene import (Scene, WallSegment, build_scene_graph,  # noqa: E402
                          flatten_arrays, generate_scene)

from paper_1904_01201_b200 import synth  # noqa: E402  (scene data only)

FRAME_SIZES = ((64, 48), (40, 33))   # (width, height): even and odd H, W % 16 != 0
CAST_W = 256


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scene_from_arrays(segs, sem, alb, wall_h=2.5, floor=(0.35, 0.33, 0.30),
                      ceil=(0.85, 0.85, 0.85), sid="golden"):
    walls = [WallSegment(a=(s[0], s[1]), b=(s[2], s[3]), semantic_id=int(i),
                         albedo=tuple(float(c) for c in a)) for s, i, a in zip(segs, sem, alb)]
    return Scene(id=sid, walls=walls, floor_color=tuple(floor), ceiling_color=tuple(ceil),
                 wall_height=wall_h)


def render_geom(scene):
    segs, sem, alb = flatten_arrays(build_scene_graph(scene))
    return rs.RenderGeometry(segs, sem, alb, scene.wall_height, scene.floor_color,
                             scene.ceiling_color)


def make(name, scene, poses, rng, kin_starts, sensor_h=1.5, extra_frames=()):
    geom = render_geom(scene)
    idx = geom.index
    out = dict(
        segments=geom.segments, semantic_ids=geom.semantic_ids, albedo=geom.albedo,
        wall_height=np.float64(scene.wall_height), floor_color=geom.floor_color,
        ceiling_color=geom.ceiling_color, sensor_height=np.float64(sensor_h),
        poses=np.asarray(poses, dtype=np.float64),
        grid_x0=np.float64(idx.x0), grid_y0=np.float64(idx.y0),
        grid_nx=np.int64(idx.nx), grid_ny=np.int64(idx.ny),
        grid_starts=idx.bucket_starts, grid_items=idx.bucket_items,
    )
    # --- column casts at W=256 on the reference's own column directions
    cfg = rs.SensorConfig("depth", width=CAST_W, height=CAST_W)
    dirs, tg, ig, tb, ib = [], [], [], [], []
    for (x, y, h) in poses:
        dx, dy = rs._column_directions(h, cfg)
        rays = np.stack([dx, dy], axis=1)
        t1, i1 = idx.raycast((x, y), rays)
        t2, i2 = idx.raycast_brute((x, y), rays)
        dirs.append(rays)
        tg.append(t1); ig.append(i1); tb.append(t2); ib.append(i2)
    out.update(cast_focal=np.float64(cfg.focal), cast_dirs=np.asarray(dirs),
               cast_t_grid=np.asarray(tg), cast_i_grid=np.asarray(ig),
               cast_t_brute=np.asarray(tb), cast_i_brute=np.asarray(ib))
    # --- frames (rgb + depth + semantic) at small sizes
    for (w, h) in tuple(FRAME_SIZES) + tuple(extra_frames):
        suite = (rs.SensorConfig("rgb", width=w, height=h),
                 rs.SensorConfig("depth", width=w, height=h),
                 rs.SensorConfig("semantic", width=w, height=h))
        rgb, dep, sem = [], [], []
        for (x, y, hd) in poses:
            o = rs.render(geom, (x, y), hd, sensor_h, suite)
            rgb.append(o.rgb); dep.append(o.depth); sem.append(o.semantic)
        key = f"frame_{w}x{h}"
        out[key + "_focal"] = np.float64(suite[0].focal)
        out[key + "_rgb_f32"] = np.asarray(rgb, dtype=np.float32)
        out[key + "_depth_f32"] = np.asarray(dep, dtype=np.float32)
        out[key + "_sem"] = np.asarray(sem)
        out[key + "_rgb_sha"] = np.array([sha(a) for a in rgb])
        out[key + "_depth_sha"] = np.array([sha(a) for a in dep])
    # --- kinematics episodes through Simulator.step (blind simulator)
    graph = build_scene_graph(scene)
    actions_all, states_all, coll_all, moved_all = [], [], [], []
    acts = (rsim.Action.MOVE_FORWARD, rsim.Action.TURN_LEFT, rsim.Action.TURN_RIGHT,
            rsim.Action.STOP)
    for (x, y, h) in kin_starts:
        sim = rsim.Simulator(graph)
        sim.set_agent_state((x, y), h)
        a_codes = rng.choice(4, size=300, p=[0.6, 0.18, 0.18, 0.04]).astype(np.int8)
        st, co, mv = [], [], []
        for a in a_codes:
            res, _ = sim.step(acts[int(a)])
            s = sim.state
            st.append((s.position[0], s.position[1], s.heading, s.cumulative_path_length,
                       float(s.collision_count)))
            co.append(res.collided); mv.append(res.displacement)
        actions_all.append(a_codes); states_all.append(st)
        coll_all.append(co); moved_all.append(mv)
    out.update(kin_starts=np.asarray(kin_starts, dtype=np.float64),
               kin_actions=np.asarray(actions_all), kin_states=np.asarray(states_all),
               kin_collided=np.asarray(coll_all), kin_moved=np.asarray(moved_all))
    # --- disc casts and clearance at random queries near the poses
    q = []
    for (x, y, h) in poses:
        for _ in range(24):
            px = x + rng.uniform(-1.5, 1.5)
            py = y + rng.uniform(-1.5, 1.5)
            ang = rng.uniform(-math.pi, math.pi)
            ln = rng.choice([0.25, 0.1, 0.6, 1.7])
            q.append((px, py, ln * math.cos(ang), ln * math.sin(ang),
                      rng.choice([0.1, 0.0, 0.25])))
    q = np.asarray(q)
    dres = []
    for (px, py, ux, uy, r) in q:
        t, i, tan = idx.cast_disc((px, py), (ux, uy), r)
        dres.append((t, float(i), tan[0], tan[1]))
    clr = np.array([idx.clearance((px, py)) for (px, py, _, _, _) in q])
    out.update(disc_queries=q, disc_results=np.asarray(dres), clearance=clr)
    path = os.path.join(HERE, f"golden_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {len(geom.segments)} segs, {len(poses)} poses -> "
          f"{os.path.getsize(path) / 1e3:.0f} kB")


def main():
    rng = np.random.default_rng(20261017)
    square = [((0.0, 0.0), (10.0, 0.0), 1, (0.6, 0.5, 0.4)),
              ((10.0, 0.0), (10.0, 10.0), 2, (0.5, 0.6, 0.4)),
              ((10.0, 10.0), (0.0, 10.0), 3, (0.4, 0.5, 0.6)),
              ((0.0, 10.0), (0.0, 0.0), 4, (0.6, 0.4, 0.5))]

    def mk(walls, sid):
        return Scene(id=sid, walls=[WallSegment(a=a, b=b, semantic_id=s, albedo=c)
                                    for a, b, s, c in walls],
                     floor_color=(0.3, 0.3, 0.3), ceiling_color=(0.9, 0.9, 0.9))

    ref_poses = [(7.0, 5.0, 0.0), (2.0, 3.0, 0.7), (5.0, 5.0, 0.0), (1.0, 9.0, -2.0),
                 (2.5, 4.0, 0.9), (5.0, 5.0, 0.3), (5.0, 5.0, math.pi / 4),
                 (5.0, 5.0, math.pi / 2), (9.5, 0.5, math.pi * 0.75)]
    make("square", mk(square, "square-10"), ref_poses, rng,
         [(5.0, 5.0, 0.4), (1.0, 1.0, 0.0)], extra_frames=((128, 128),))
    make("open_square", mk([w for w in square if w[2] != 2], "open"), ref_poses[:5], rng,
         [(5.0, 5.0, 0.0)])

    room = synth.single_room(250)
    room_poses = [tuple(p) for p in synth.sample_poses(room, 6, seed=3)] + [
        (5.0, 5.0, 0.0), (5.0, 5.0, math.pi / 4), (0.2, 0.2, math.pi / 4)]
    make("room1000", scene_from_arrays(room.segments, room.semantic_ids, room.albedo,
                                       floor=room.floor_color, ceil=room.ceiling_color),
         room_poses, rng, [tuple(p) for p in synth.sample_poses(room, 2, seed=4)])

    gen = generate_scene(101)
    grid = nav.rasterize_navigable(gen.segment_array(), gen.bounds())
    gposes = []
    for _ in range(8):
        p = nav.sample_navigable(grid, rng)
        gposes.append((float(p[0]), float(p[1]), float(rng.uniform(-math.pi, math.pi))))
    make("gen101", gen, gposes, rng, gposes[:2])

    r7 = np.random.default_rng(7)
    segs = r7.uniform(-8, 8, size=(120, 4))
    sem = np.arange(1, 121)
    alb = r7.uniform(0.2, 0.9, size=(120, 3))
    rposes = [(float(x), float(y), float(h)) for x, y, h in
              zip(r7.uniform(-7, 7, 8), r7.uniform(-7, 7, 8), r7.uniform(-math.pi, math.pi, 8))]
    make("rand120", scene_from_arrays(segs, sem, alb), rposes, rng, [])

    apt = synth.config_scene("C2")
    aposes = [tuple(p) for p in synth.sample_poses(apt, 8, seed=11)]
    make("apt10k", scene_from_arrays(apt.segments, apt.semantic_ids, apt.albedo), aposes,
         rng, aposes[:2])


if __name__ == "__main__":
    main()
