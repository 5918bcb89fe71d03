"""Deterministic synthetic scenes and start poses for the benchmark configs.

BASELINE.json names its workloads by triangle count: one wall segment is one
vertical quad = 2 triangles; floor and ceiling are analytic planes (0 tris),
so "~N tris" means ~N/2 segments.

* ``single_room``  -- C1: the reference's 10x10 m test room
  (pkg/tests/conftest.py:8-20) with each wall split into collinear pieces,
  every piece its own semantic id, so shared endpoints exercise the (t, idx)
  tie rule of raycast_grid (src/_kernels.py:12-13, 101).
* ``apartment``    -- C2/C3/C5: a jittered grid of rooms with one door per
  shared wall and per-room clutter (pillars, stubs, L-baffles -- the same
  object vocabulary as the reference generator, src/scene.py:507-554), walls
  subdivided to hit the segment target.  Semantic id = object id
  (``(id % 65000) + 1``), albedo per object, wall height 2.5
  (src/scene.py:22-23, 56-57).

This is host tooling (numpy); it does not run the reference generator, whose
load-time validation is O(cells x segments) and infeasible at 100k+ segments
(SURVEY.md §8d).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

FLOOR_COLOR = (0.35, 0.33, 0.30)     # src/scene.py:56
CEILING_COLOR = (0.85, 0.85, 0.85)   # src/scene.py:57
WALL_HEIGHT = 2.5                    # src/scene.py:23


@dataclass
class SynthScene:
    name: str
    segments: np.ndarray        # (n, 4) f64 world (ax, ay, bx, by)
    semantic_ids: np.ndarray    # (n,) u16, in [1, 65000]
    albedo: np.ndarray          # (n, 3) f64
    rooms: np.ndarray           # (r, 4) interior rectangles for pose sampling
    wall_height: float = WALL_HEIGHT
    floor_color: tuple = FLOOR_COLOR
    ceiling_color: tuple = CEILING_COLOR

    @property
    def n_segments(self) -> int:
        return len(self.segments)

    @property
    def n_triangles(self) -> int:
        return 2 * len(self.segments)


def _subdivide(segs, obj, pieces_per_meter):
    """Split each (a, b) into collinear pieces sharing exact endpoints."""
    out, oid = [], []
    for (ax, ay, bx, by), o in zip(segs, obj):
        ln = math.hypot(bx - ax, by - ay)
        k = max(1, int(round(ln * pieces_per_meter)))
        f = np.arange(k + 1) / k
        xs = ax + (bx - ax) * f
        ys = ay + (by - ay) * f
        xs[-1], ys[-1] = bx, by
        out.append(np.stack([xs[:-1], ys[:-1], xs[1:], ys[1:]], axis=1))
        oid.append(np.full(k, o, dtype=np.int64))
    return np.concatenate(out), np.concatenate(oid)


def single_room(pieces_per_wall: int = 250, size: float = 10.0) -> SynthScene:
    """C1: 4 walls x pieces_per_wall collinear pieces (1000 segs ~ 2k tris)."""
    corners = [(0.0, 0.0), (size, 0.0), (size, size), (0.0, size)]
    albedo_wall = [(0.6, 0.5, 0.4), (0.5, 0.6, 0.4), (0.4, 0.5, 0.6), (0.6, 0.4, 0.5)]
    segs, alb = [], []
    for w in range(4):
        (ax, ay), (bx, by) = corners[w], corners[(w + 1) % 4]
        f = np.arange(pieces_per_wall + 1) / pieces_per_wall
        xs, ys = ax + (bx - ax) * f, ay + (by - ay) * f
        xs[-1], ys[-1] = bx, by
        segs.append(np.stack([xs[:-1], ys[:-1], xs[1:], ys[1:]], axis=1))
        shade = 1.0 - 0.3 * (np.arange(pieces_per_wall) % 7) / 7.0
        alb.append(np.asarray(albedo_wall[w])[None, :] * shade[:, None])
    segs = np.concatenate(segs)
    sem = (np.arange(len(segs)) % 65000 + 1).astype(np.uint16)
    rooms = np.array([[0.0, 0.0, size, size]])
    return SynthScene("single_room", segs, sem, np.concatenate(alb), rooms,
                      floor_color=(0.3, 0.3, 0.3), ceiling_color=(0.9, 0.9, 0.9))


def apartment(seed: int, rooms_x: int, rooms_y: int, target_segments: int,
              room_size=(3.5, 6.5), door=1.0, name: str | None = None) -> SynthScene:
    """Grid-of-rooms apartment with doors and clutter, ~target_segments."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, rooms_x, rooms_y]))
    mean = 0.5 * (room_size[0] + room_size[1])
    # jittered grid lines
    def lines(n):
        w = rng.uniform(room_size[0], room_size[1], n)
        return np.concatenate([[0.0], np.cumsum(w)])
    xs, ys = lines(rooms_x), lines(rooms_y)
    raw, obj, colors = [], [], []

    def add(segs, color):
        if not segs:
            return
        o = len(colors)
        colors.append(color)
        for s in segs:
            raw.append(s)
            obj.append(o)

    W, H = xs[-1], ys[-1]
    bcol = tuple(rng.uniform(0.45, 0.75, 3).round(3))
    add([(0.0, 0.0, W, 0.0)], bcol)
    add([(W, 0.0, W, H)], bcol)
    add([(W, H, 0.0, H)], bcol)
    add([(0.0, H, 0.0, 0.0)], bcol)
    # interior walls between adjacent rooms, one door per room-room boundary
    for i in range(1, rooms_x):
        x = xs[i]
        for j in range(rooms_y):
            lo, hi = ys[j], ys[j + 1]
            off = lo + rng.uniform(0.3, hi - lo - door - 0.3)
            col = tuple(rng.uniform(0.35, 0.8, 3).round(3))
            add([(x, lo, x, off), (x, off + door, x, hi)], col)
    for j in range(1, rooms_y):
        y = ys[j]
        for i in range(rooms_x):
            lo, hi = xs[i], xs[i + 1]
            off = lo + rng.uniform(0.3, hi - lo - door - 0.3)
            col = tuple(rng.uniform(0.35, 0.8, 3).round(3))
            add([(lo, y, off, y), (off + door, y, hi, y)], col)
    # clutter, kept off the room borders (src/scene.py:507-554 vocabulary)
    margin = 0.9
    rooms = []
    for i in range(rooms_x):
        for j in range(rooms_y):
            x0, x1, y0, y1 = xs[i], xs[i + 1], ys[j], ys[j + 1]
            rooms.append((x0, y0, x1, y1))
            for _ in range(int(rng.integers(1, 4))):
                ox = rng.uniform(x0 + margin, x1 - margin)
                oy = rng.uniform(y0 + margin, y1 - margin)
                col = tuple(rng.uniform(0.2, 0.9, 3).round(3))
                kind = rng.random()
                clamp = lambda px, py: (min(max(px, x0 + margin), x1 - margin),
                                        min(max(py, y0 + margin), y1 - margin))
                if kind < 0.25:
                    h = 0.09
                    a0, b0 = clamp(ox - h, oy - h)
                    a1, b1 = clamp(ox + h, oy + h)
                    add([(a0, b0, a1, b0), (a1, b0, a1, b1), (a1, b1, a0, b1),
                         (a0, b1, a0, b0)], col)
                elif kind < 0.6:
                    ang = rng.uniform(0.0, math.pi)
                    ln = rng.uniform(0.6, 2.0)
                    ex, ey = clamp(ox + ln * math.cos(ang), oy + ln * math.sin(ang))
                    if math.hypot(ex - ox, ey - oy) > 0.3:
                        add([(ox, oy, ex, ey)], col)
                else:
                    ang = rng.uniform(0.0, 2 * math.pi)
                    l1, l2 = rng.uniform(0.5, 1.4, 2)
                    mx, my = clamp(ox + l1 * math.cos(ang), oy + l1 * math.sin(ang))
                    a2 = ang + (math.pi / 2 if rng.random() < 0.5 else -math.pi / 2)
                    ex, ey = clamp(mx + l2 * math.cos(a2), my + l2 * math.sin(a2))
                    segs = []
                    if math.hypot(mx - ox, my - oy) > 0.3:
                        segs.append((ox, oy, mx, my))
                    if math.hypot(ex - mx, ey - my) > 0.3:
                        segs.append((mx, my, ex, ey))
                    add(segs, col)
    raw = np.asarray(raw, dtype=np.float64)
    obj = np.asarray(obj, dtype=np.int64)
    total = float(np.hypot(raw[:, 2] - raw[:, 0], raw[:, 3] - raw[:, 1]).sum())
    ppm = max(1e-9, target_segments / total)
    segs, oid = _subdivide(raw, obj, ppm)
    colors = np.asarray(colors, dtype=np.float64)
    sem = (oid % 65000 + 1).astype(np.uint16)
    return SynthScene(name or f"apartment-{seed}-{rooms_x}x{rooms_y}", segs, sem,
                      colors[oid], np.asarray(rooms))


def config_scene(cfg: str) -> SynthScene:
    """Scene for a BASELINE.json config key (C1..C5)."""
    if cfg == "C1":
        return single_room(250)
    if cfg == "C2":
        return apartment(5, 4, 4, 10_000, name="C2-multiroom-20k-tris")
    if cfg in ("C3", "C4"):
        return apartment(7, 16, 16, 100_000, name="C3-apartment-200k-tris")
    if cfg == "C5":
        return apartment(9, 32, 32, 500_000, name="C5-apartment-1M-tris")
    raise ValueError(f"unknown config {cfg!r}")


def _free_raster(scene: SynthScene, clearance: float, res: float = 0.05):
    """Conservative free-space raster: cells farther than `clearance` (+1 cell)
    from every segment sample point."""
    s = scene.segments
    x0 = float(min(s[:, 0].min(), s[:, 2].min())) - 1.0
    y0 = float(min(s[:, 1].min(), s[:, 3].min())) - 1.0
    x1 = float(max(s[:, 0].max(), s[:, 2].max())) + 1.0
    y1 = float(max(s[:, 1].max(), s[:, 3].max())) + 1.0
    nx, ny = int(math.ceil((x1 - x0) / res)) + 1, int(math.ceil((y1 - y0) / res)) + 1
    blocked = np.zeros((ny, nx), dtype=bool)
    ln = np.hypot(s[:, 2] - s[:, 0], s[:, 3] - s[:, 1])
    k = np.maximum(1, np.ceil(ln / (res * 0.5)).astype(np.int64))
    seg_id = np.repeat(np.arange(len(s)), k + 1)
    f = np.concatenate([np.arange(kk + 1) / kk for kk in k])
    px = s[seg_id, 0] + (s[seg_id, 2] - s[seg_id, 0]) * f
    py = s[seg_id, 1] + (s[seg_id, 3] - s[seg_id, 1]) * f
    blocked[((py - y0) / res).astype(np.int64), ((px - x0) / res).astype(np.int64)] = True
    rad = int(math.ceil(clearance / res)) + 1
    grown = blocked.copy()
    for dy in range(-rad, rad + 1):
        for dx in range(-rad, rad + 1):
            if dx * dx + dy * dy > (rad + 1) ** 2:
                continue
            grown |= np.roll(np.roll(blocked, dy, axis=0), dx, axis=1)
    return ~grown, x0, y0, res


def sample_poses(scene: SynthScene, n: int, seed: int, clearance: float = 0.15, first: int = 0):
    """Start poses of envs first .. first+n-1 inside the rooms, >= clearance
    from every wall (conservative raster test; the simulator re-checks exactly
    on reset).  Heading uniform on (-pi, pi].  Per-env streams derive from
    (seed, global env id) so sharding over ranks does not change any env's
    pose (src/seeding.py:13-23 idea)."""
    free, x0, y0, res = _free_raster(scene, clearance)
    ny, nx = free.shape
    out = np.empty((n, 3))
    for e in range(n):
        rng = np.random.default_rng(np.random.SeedSequence([seed, first + e]))
        for _ in range(10_000):
            r = scene.rooms[int(rng.integers(len(scene.rooms)))]
            x = rng.uniform(r[0] + 0.2, r[2] - 0.2)
            y = rng.uniform(r[1] + 0.2, r[3] - 0.2)
            ci, cj = int((y - y0) / res), int((x - x0) / res)
            if 0 <= ci < ny and 0 <= cj < nx and free[ci, cj]:
                break
        else:
            raise RuntimeError("no free start pose found")
        out[e] = (x, y, math.pi - rng.uniform(0.0, 2.0 * math.pi))
    return out


def random_actions(n_envs: int, n_steps: int, seed: int) -> np.ndarray:
    """Seeded uniform actions over {forward, left, right} as int8 codes 0/1/2
    (tests/test_acceptance.py:91-92 policy)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0xAC7]))
    return rng.integers(0, 3, size=(n_steps, n_envs)).astype(np.int8)


def pointgoal_episodes(env, scene: SynthScene, n: int, seed: int, first: int = 0,
                       n_goals: int = 16):
    """PointGoal episodes for envs first .. first+n-1 of ``env`` (a
    task.BatchEnvironment on ``scene``): goals from a shared pool of
    ``n_goals`` seeded navigable points, starts from ``sample_poses``; each
    env takes the first goal of its own seeded order whose geodesic distance
    gdsp (nav.geodesic_distance on the goal's device field, like the
    reference's episode generator, episodes.py) satisfies Episode.validate
    (1 <= gdsp <= 30 m, gdsp >= euclidean - 2 res).  Everything derives from
    (seed, global env id): sharding does not change an env's episode.
    Returns a list with None for envs no goal fits."""
    import torch

    from . import _native as nat
    from . import nav, task
    grid = env.grid
    goals = sample_poses(scene, n_goals, seed=seed ^ 0x6F41, first=0)[:, :2]
    fields, _ = nav.distance_fields(grid, goals)
    starts = sample_poses(scene, n, seed=seed, first=first)
    k = len(goals)
    pts = torch.as_tensor(np.repeat(starts[:, :2], k, axis=0), device=env.dev)
    fid = torch.as_tensor(np.tile(np.arange(k, dtype=np.int32), n), device=env.dev)
    gd = torch.empty(n * k, dtype=torch.float64, device=env.dev)
    c = grid.ctx
    nat.check(c.lib.nv_nav_geodesic(c.handle, nat.ptr(fields), nat.ptr(fid), nat.ptr(pts), n * k,
                                     nat.ptr(gd), nat.stream_handle(env.dev)))
    gd = gd.cpu().numpy().reshape(n, k)
    out = []
    for e in range(n):
        rng = np.random.default_rng(np.random.SeedSequence([seed, 0x60A1, first + e]))
        ep = None
        for g in rng.permutation(k):
            d = float(gd[e, g])
            eu = float(np.hypot(goals[g, 0] - starts[e, 0], goals[g, 1] - starts[e, 1]))
            if not (math.isfinite(d) and 1.0 <= d <= 30.0 and eu > 0.0
                    and d >= eu - 2.0 * grid.resolution):
                continue
            ep = task.Episode(f"ep{first + e}", env.scene_id or "synthetic",
                              (float(starts[e, 0]), float(starts[e, 1])), float(starts[e, 2]),
                              (float(goals[g, 0]), float(goals[g, 1])), d, eu, d / eu)
            break
        out.append(ep)
    return out
