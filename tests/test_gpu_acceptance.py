"""The reference's release criteria that concern the hot path
(pkg/tests/test_acceptance.py: 3 kinematics fuzz, 4 geodesic correctness,
9 render consistency, 10 depth-noise moment), restated on the GPU.

Criterion 3 runs batched here -- the reference fuzzes one Simulator per
scene; the same invariants are checked for every env of a BatchSimulator
(100k+ actions in total, twice, bit-identical) within the reference's 60 s
budget.  Criterion 4's independent oracle is the reference's: a scipy csgraph
Dijkstra at 0.01 m over the same octile / no-corner-cutting rules, on a mask
rasterised (on the device) at that resolution."""
import math
import time

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_01201_b200 as nb
    from paper_1904_01201_b200 import _native
    _native.load()
    return nb


def _scene_from_golden(nb, name):
    g = load_golden(name)
    walls = [nb.WallSegment(a=(float(s[0]), float(s[1])), b=(float(s[2]), float(s[3])),
                            semantic_id=int(i), albedo=tuple(float(c) for c in a))
             for s, i, a in zip(g["segments"], g["semantic_ids"], g["albedo"])]
    return nb.Scene(id=name, walls=walls, floor_color=tuple(g["floor_color"]),
                    ceiling_color=tuple(g["ceiling_color"]), wall_height=float(g["wall_height"]))


def _starts(nb, scene, n, seed, radius=0.1):
    from paper_1904_01201_b200 import nav
    grid = nav.rasterize_navigable(scene.segment_array(), scene.bounds())
    index = nb.SegmentIndex(scene.segment_array())
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < n:
        cand = np.array([nav.sample_navigable(grid, rng) for _ in range(2 * n)])
        clr = index.clearance_batch(cand[:, 0], cand[:, 1])
        pts.extend(cand[clr >= radius][: n - len(pts)])
    return np.array(pts), rng.uniform(0, 2 * math.pi, n), index


def _fuzz_batch(nb, scene, n_envs, steps, seed):
    pts, heads, index = _starts(nb, scene, n_envs, seed)
    segs, sem, alb = nb.flatten_arrays(nb.build_scene_graph(scene))
    sim = nb.BatchSimulator(segs, sem, alb, n_envs)
    sim.reset(pts, heads)
    rng = np.random.default_rng(seed + 1)
    trace = []
    xy0, h0, p0, _ = (t.cpu().numpy() for t in sim.state())
    for _ in range(steps):
        a = rng.integers(0, 3, n_envs).astype(np.int8)
        sim.step(torch.as_tensor(a, device="cuda:0"), render=False)
        xy, h, p, _ = (t.cpu().numpy() for t in sim.state())
        disp = sim.displacement.cpu().numpy()
        assert np.all((disp >= 0.0) & (disp <= 0.25))
        fwd = a == 0
        assert np.array_equal(h[fwd], h0[fwd])                 # forward keeps heading
        assert np.array_equal(xy[~fwd], xy0[~fwd])             # turns keep position
        clr = index.clearance_batch(xy[:, 0], xy[:, 1])
        assert np.all(clr >= 0.1 - 1e-6)                       # never inside a wall
        assert np.allclose(p, p0 + disp, atol=1e-9)            # path length accumulates
        trace.append(np.concatenate([xy.ravel(), h]))
        xy0, h0, p0 = xy, h, p
    return np.stack(trace)


def test_criterion_03_kinematics_fuzz(nb):
    t0 = time.time()
    names = ["square", "gen101", "room1000", "apt10k"]
    n_envs, steps = 256, 100
    total = 0
    for k, name in enumerate(names):
        scene = _scene_from_golden(nb, name)
        first = _fuzz_batch(nb, scene, n_envs, steps, 900 + k)
        again = _fuzz_batch(nb, scene, n_envs, steps, 900 + k)
        assert np.array_equal(first, again)                    # bit-identical reruns
        total += n_envs * steps
    assert total >= 100_000
    assert time.time() - t0 < 60.0


def _fine_oracle(nb, scene, goal, points, resolution=0.01, radius=0.1):
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import dijkstra
    from paper_1904_01201_b200.geometry import navigable_mask
    mask, origin, _ = navigable_mask(scene.segment_array(), scene.bounds(), resolution, radius)
    h, w = mask.shape
    idx = np.arange(h * w).reshape(h, w)
    rows, cols, data = [], [], []
    for di, dj in ((0, 1), (1, 0), (1, 1), (1, -1)):
        if dj >= 0:
            a, b = idx[:h - di or h, :w - dj or w], idx[di:, dj:]
            ok = mask[:h - di or h, :w - dj or w] & mask[di:, dj:]
            if di and dj:
                ok &= mask[:h - di, dj:] & mask[di:, :w - dj]
        else:
            a, b = idx[:h - di, -dj:], idx[di:, :w + dj]
            ok = mask[:h - di, -dj:] & mask[di:, :w + dj] & mask[:h - di, :w + dj] & mask[di:, -dj:]
        rows.append(a[ok])
        cols.append(b[ok])
        data.append(np.full(int(ok.sum()), resolution * (math.sqrt(2.0) if di and dj else 1.0)))
    graph = coo_matrix((np.concatenate(data), (np.concatenate(rows), np.concatenate(cols))),
                       shape=(h * w, h * w)).tocsr()
    cand = np.argwhere(mask)

    def cell(p):
        j = int(math.floor((p[0] - origin[0]) / resolution + 0.5))
        i = int(math.floor((p[1] - origin[1]) / resolution + 0.5))
        ci, cj = cand[int(np.argmin((cand[:, 0] - i) ** 2 + (cand[:, 1] - j) ** 2))]
        return ci * w + cj

    dist = dijkstra(graph, directed=False, indices=[cell(goal)])[0]
    return [float(dist[cell(p)]) for p in points]


def test_criterion_04_geodesic_vs_fine_oracle(nb):
    from paper_1904_01201_b200 import nav
    walls = [((0, 0), (8, 0), 1), ((8, 0), (8, 8), 2), ((8, 8), (0, 8), 3), ((0, 8), (0, 0), 4),
             ((3.0, 2.0), (3.0, 6.0), 5), ((3.0, 6.0), (5.0, 6.0), 5), ((5.0, 6.0), (5.0, 2.0), 5)]
    scene = nb.Scene(id="u8", walls=[nb.WallSegment(a=a, b=b, semantic_id=s) for a, b, s in walls])
    grid = nav.rasterize_navigable(scene.segment_array(), scene.bounds())
    # the detour case of test_nav.py:82 ...
    field = nav.distance_field(grid, (4.0, 7.2))
    ours = nav.geodesic_distance(field, (4.0, 3.0))
    assert ours > math.hypot(0.0, 4.2) + 1.0
    ref = _fine_oracle(nb, scene, (4.0, 7.2), [(4.0, 3.0)])[0]
    assert abs(ours - ref) / ref <= 0.03
    # ... and 50 separated pairs over random goals (test_acceptance.py:116)
    rng = np.random.default_rng(3)
    cells = grid.navigable_cells()
    checked = 0
    while checked < 50:
        goal = grid.center_of(*cells[int(rng.integers(len(cells)))])
        field = nav.distance_field(grid, goal)
        starts = []
        for _ in range(200):
            s = grid.center_of(*cells[int(rng.integers(len(cells)))])
            d = nav.geodesic_distance(field, s)
            if np.isfinite(d) and math.hypot(*(s - goal)) >= 1.5:
                starts.append((s, d))
            if len(starts) >= 10:
                break
        for (s, d), r in zip(starts, _fine_oracle(nb, scene, goal, [s for s, _ in starts])):
            assert abs(d - r) / r <= 0.03
            checked += 1


def test_criterion_09_render_consistency(nb):
    sq = _scene_from_golden(nb, "square")
    segs, sem, alb = nb.flatten_arrays(nb.build_scene_graph(sq))
    geom = nb.RenderGeometry(segs, sem, alb, sq.wall_height, sq.floor_color, sq.ceiling_color)
    suite = tuple(nb.SensorConfig(k) for k in ("rgb", "depth", "semantic"))
    obs = nb.render(geom, (7.0, 5.0), 0.0, 1.5, suite)
    assert np.all(np.abs(obs.depth[128] - 3.0) <= 1e-5)
    for pose in ((2.0, 3.0, 0.7), (5.0, 5.0, 0.0), (1.0, 9.0, -2.0)):
        fr = nb.render(geom, pose[:2], pose[2], 1.5, suite)
        assert np.array_equal(fr.depth == 10.0, fr.semantic == nb.SEM_VOID)
    sym = nb.render(geom, (5.0, 5.0), 0.0, 1.5, suite)
    assert np.max(np.abs(sym.depth - sym.depth[:, ::-1])) <= 1e-5
    # accelerated index == exhaustive scan, full 256^2 frames on a larger scene
    from paper_1904_01201_b200 import nav
    scene = _scene_from_golden(nb, "room1000")
    segs, sem, alb = nb.flatten_arrays(nb.build_scene_graph(scene))
    geom2 = nb.RenderGeometry(segs, sem, alb, scene.wall_height, scene.floor_color,
                              scene.ceiling_color)
    grid = nav.rasterize_navigable(scene.segment_array(), scene.bounds())
    rng = np.random.default_rng(9)
    for _ in range(2):
        pos, heading = nav.sample_navigable(grid, rng), rng.uniform(0, 2 * math.pi)
        fast = nb.render(geom2, pos, heading, 1.5, suite)
        slow = nb.render(geom2, pos, heading, 1.5, suite, brute_force=True)
        assert np.array_equal(fast.depth, slow.depth)
        assert np.array_equal(fast.rgb, slow.rgb)
        assert np.array_equal(fast.semantic, slow.semantic)


def test_criterion_10_inverse_depth_noise_moment(nb):
    from paper_1904_01201_b200.sensors import apply_inverse_depth_noise
    noisy = apply_inverse_depth_noise(np.full(100_000, 2.0), 0.4, np.random.default_rng(10),
                                      max_range=10.0)
    assert float((10.0 / noisy).std()) == pytest.approx(0.4, abs=0.01)
