"""Generate the nav/task golden fixtures from the UNMODIFIED reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_task.py

Produced by the reference's public functions: ``nav.rasterize_navigable``
(geometry.navigable_mask, src/geometry.py:209-250), ``nav.distance_field``
(_kernels.dijkstra_grid, src/_kernels.py:210-282), ``nav.geodesic_distance``
(src/nav.py:135-166), ``nav._snap_to_navigable`` (src/nav.py:103-119) and
``task.Environment.reset/step`` (src/task.py:123-256).  f64 grids are pinned
by sha256 plus exact samples; episodes record every step's distance, reward,
done flag and the final EpisodeOutcome.
"""
from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from navsim import nav  # noqa: E402  (reference)
from navsim import task  # noqa: E402
from navsim.scene import Scene, WallSegment, generate_scene  # noqa: E402
from navsim.sensors import SensorConfig  # noqa: E402
from navsim.sim import Action, AgentConfig  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mk(walls, sid):
    return Scene(id=sid, walls=[WallSegment(a=a, b=b, semantic_id=s, albedo=(0.5, 0.5, 0.5))
                                for a, b, s in walls],
                 floor_color=(0.3, 0.3, 0.3), ceiling_color=(0.9, 0.9, 0.9))


def rect(x0, y0, x1, y1, s=1):
    return [((x0, y0), (x1, y0), s), ((x1, y0), (x1, y1), s + 1), ((x1, y1), (x0, y1), s + 2),
            ((x0, y1), (x0, y0), s + 3)]


def grids(name, scene, rng, goals, radii=(0.1,), n_geo=400):
    out = {}
    segs = scene.segment_array()
    bnds = scene.bounds()
    out["segments"] = segs
    out["bounds"] = np.array(bnds)
    for r in radii:
        g = nav.rasterize_navigable(segs, bnds, 0.05, r)
        key = f"r{int(round(r * 1000))}"
        out[f"{key}_origin"] = g.origin
        out[f"{key}_navigable"] = g.navigable.astype(np.uint8)
        out[f"{key}_clearance_sha"] = np.array(sha(g.clearance))
        pick = rng.integers(0, g.clearance.size, size=2000)
        out[f"{key}_clearance_idx"] = pick
        out[f"{key}_clearance_val"] = g.clearance.ravel()[pick]
        if r != 0.1:
            continue
        # snapping at random points (None -> (-1, -1))
        pts = np.stack([rng.uniform(bnds[0] - 0.3, bnds[2] + 0.3, 300),
                        rng.uniform(bnds[1] - 0.3, bnds[3] + 0.3, 300)], axis=1)
        sn = [nav._snap_to_navigable(g, p) for p in pts]
        out["snap_pts"] = pts
        out["snap_cells"] = np.array([c if c is not None else (-1, -1) for c in sn])
        fsha, fcell, fgoal, qpts, qval, fsamp_i, fsamp_v = [], [], [], [], [], [], []
        for goal in goals:
            f = nav.distance_field(g, goal)
            fsha.append(sha(f.dist))
            fcell.append(f.goal_cell)
            fgoal.append(goal)
            nav_cells = np.argwhere(g.navigable)
            sel = nav_cells[rng.integers(0, len(nav_cells), size=n_geo)]
            pts = g.origin + 0.05 * sel[:, ::-1] + rng.uniform(-0.06, 0.06, size=sel.shape)
            vals = []
            for p in pts:
                try:
                    vals.append(nav.geodesic_distance(f, p))
                except nav.NavError:
                    vals.append(np.nan)
            qpts.append(pts)
            qval.append(vals)
            pick = rng.integers(0, f.dist.size, size=2000)
            fsamp_i.append(pick)
            fsamp_v.append(f.dist.ravel()[pick])
        out.update(field_sha=np.array(fsha), field_cell=np.array(fcell),
                   field_goal=np.array(fgoal), geo_pts=np.array(qpts), geo_val=np.array(qval),
                   field_idx=np.array(fsamp_i), field_val=np.array(fsamp_v))
    return out


def episodes(scene, rng, specs):
    """specs: (start, heading, goal, action list or 'greedy')."""
    agent = AgentConfig()
    env = task.Environment(scene, agent, sensor_configs=(SensorConfig("depth", width=16,
                                                                        height=16),))
    recs = []
    for k, (start, heading, goal, acts) in enumerate(specs):
        f = nav.distance_field(env.grid, goal)
        gd = nav.geodesic_distance(f, start)
        eu = math.hypot(goal[0] - start[0], goal[1] - start[1])
        ep = task.Episode(episode_id=f"e{k}", scene_id=scene.id, start_position=tuple(start),
                          start_heading=float(heading), goal_position=tuple(goal),
                          gdsp=float(gd), euclidean=float(eu), ratio=float(gd / eu))
        env.reset(ep)
        rows, codes = [], []
        d0 = env._d_last
        s0 = env.sim.state
        i = 0
        while not env.done:
            if acts == "greedy":
                a = nav.greedy_gradient_action(env.field, env.sim.state, 0.15, agent,
                                               env.sim.geometry.index)
            else:
                a = acts[i] if i < len(acts) else Action.STOP
            i += 1
            _, done, info = env.step(a)
            codes.append(a.value if hasattr(a, "value") and isinstance(a.value, int) else
                         [Action.MOVE_FORWARD, Action.TURN_LEFT, Action.TURN_RIGHT,
                          Action.STOP].index(a))
            st = env.sim.state
            rows.append((info["d"], info["reward"], float(done), float(info["collided"]),
                         info["displacement"], st.position[0], st.position[1], st.heading))
        o = env.outcome
        recs.append(dict(start=np.array([s0.position[0], s0.position[1], s0.heading]),
                         start_raw=np.array([start[0], start[1], heading]),
                         goal=np.array(goal), gdsp=gd, d0=d0, actions=np.array(codes, np.int8),
                         rows=np.array(rows),
                         outcome=np.array([float(o.success), o.shortest_path, o.path_taken,
                                           o.spl, float(o.steps), float(o.collisions),
                                           1.0 if o.terminated_by == "stop" else 2.0])))
    return recs


def main():
    rng = np.random.default_rng(20261017)
    scenes = {
        "square": (mk(rect(0, 0, 10, 10), "square-10"), [(2.0, 5.0), (5.0, 5.0), (9.0, 9.0)]),
        "udetour": (mk(rect(0, 0, 8, 8) + [((3.0, 2.0), (3.0, 6.0), 5), ((3.0, 6.0), (5.0, 6.0), 5),
                                           ((5.0, 6.0), (5.0, 2.0), 5)], "u"),
                    [(4.0, 7.2), (4.0, 3.0)]),
        "split": (mk(rect(0, 0, 10, 10) + [((5.0, 0.0), (5.0, 10.0), 9)], "split"),
                  [(2.0, 2.0)]),
        "pocket": (mk(rect(0, 0, 10, 10) + rect(4, 4, 6, 6, 10), "pocket"), [(1.0, 1.0)]),
        "gen101": (generate_scene(101), None),
    }
    for name, (scene, goals) in scenes.items():
        if goals is None:
            g = nav.rasterize_navigable(scene.segment_array(), scene.bounds())
            goals = [tuple(nav.sample_navigable(g, rng)) for _ in range(3)]
        out = grids(name, scene, rng, goals, radii=(0.1, 0.02) if name == "udetour" else (0.1,))
        if name in ("square", "gen101"):
            g = nav.rasterize_navigable(scene.segment_array(), scene.bounds())
            specs = []
            for k in range(4):
                while True:
                    s = nav.sample_navigable(g, rng)
                    gl = nav.sample_navigable(g, rng)
                    if 1.5 <= math.hypot(*(np.array(gl) - s)) <= 7.0:
                        break
                h = float(rng.uniform(-math.pi, math.pi))
                if k == 0:
                    acts = "greedy"
                elif k == 1:  # runs into the 500-step budget
                    acts = [[Action.MOVE_FORWARD, Action.TURN_LEFT, Action.TURN_RIGHT][int(c)]
                            for c in rng.choice(3, size=600, p=[0.6, 0.2, 0.2])]
                else:
                    acts = [[Action.MOVE_FORWARD, Action.TURN_LEFT, Action.TURN_RIGHT][int(c)]
                            for c in rng.choice(3, size=int(rng.integers(5, 60)),
                                                p=[0.6, 0.2, 0.2])]
                specs.append((tuple(s), h, tuple(gl), acts))
            for k, rec in enumerate(episodes(scene, rng, specs)):
                for kk, v in rec.items():
                    out[f"ep{k}_{kk}"] = v
            out["n_episodes"] = np.int64(len(specs))
        path = os.path.join(HERE, f"golden_task_{name}.npz")
        np.savez_compressed(path, **out)
        print(f"{name}: -> {os.path.getsize(path) / 1e3:.0f} kB")


if __name__ == "__main__":
    main()
