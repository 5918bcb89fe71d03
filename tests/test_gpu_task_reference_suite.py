"""The reference's task-layer and navigation tests (pkg/tests/test_task.py,
test_nav.py), restated against this package on the GPU: the Environment
facade over the fused device task step, and the device occupancy grid /
distance fields / geodesic interpolation.  Each test
cites the one it follows.  Tests of the reference that build grids from
hand-made boolean arrays (test_nav.py:161-215) have no counterpart: grids
here are always rasterised on the device from walls."""
import math

import numpy as np
import pytest

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


def rect_walls(x0, y0, x1, y1, sid=1):
    return [((x0, y0), (x1, y0), sid), ((x1, y0), (x1, y1), sid + 1),
            ((x1, y1), (x0, y1), sid + 2), ((x0, y1), (x0, y0), sid + 3)]


def make_scene(nb, walls, scene_id="custom"):
    return nb.Scene(id=scene_id, walls=[nb.WallSegment(a=a, b=b, semantic_id=s) for a, b, s in walls],
                    wall_height=2.5)


@pytest.fixture(scope="module")
def square(nb):
    return make_scene(nb, rect_walls(0.0, 0.0, 10.0, 10.0), "square-10")


def grid_for(scene, resolution=0.05, radius=0.1):
    from paper_1904_01201_b200 import nav
    return nav.rasterize_navigable(scene.segment_array(), scene.bounds(), resolution, radius)


def episode_for(scene, start, heading, goal):  # test_task.py:62-70
    from paper_1904_01201_b200 import nav, task
    field = nav.distance_field(grid_for(scene), goal)
    gdsp = nav.geodesic_distance(field, start)
    eu = math.hypot(goal[0] - start[0], goal[1] - start[1])
    return task.Episode(episode_id="t-0", scene_id=scene.id, start_position=tuple(start),
                        start_heading=heading, goal_position=tuple(goal), gdsp=float(gdsp),
                        euclidean=eu, ratio=float(gdsp / eu))


# --------------------------------------------------------- test_task.py

def test_reset_emits_frame_and_goal(nb, square):  # test_task.py:72
    from paper_1904_01201_b200 import task
    env = task.Environment(square)
    ep = episode_for(square, (2.0, 5.0), 0.7, (7.0, 5.0))
    obs = env.reset(ep)
    assert np.allclose(obs.gps, [0.0, 0.0], atol=1e-12) and obs.compass == 0.0
    assert np.linalg.norm(obs.goal) == pytest.approx(ep.euclidean, abs=1e-9)
    again = env.reset(ep)
    assert np.array_equal(again.depth, obs.depth)
    assert np.array_equal(again.goal, obs.goal)


def test_reset_rejects_goal_in_wall_and_wrong_scene(nb, square):  # test_task.py:84, :94
    from paper_1904_01201_b200 import task
    env = task.Environment(square)
    ep = task.Episode(episode_id="bad", scene_id=square.id, start_position=(2.0, 5.0),
                      start_heading=0.0, goal_position=(10.15, 5.0), gdsp=8.15, euclidean=8.15,
                      ratio=1.0)
    with pytest.raises(task.TaskError, match="not navigable"):
        env.reset(ep)
    ep = task.Episode(episode_id="x", scene_id="other", start_position=(2, 5), start_heading=0.0,
                      goal_position=(7, 5), gdsp=5.0, euclidean=5.0, ratio=1.0)
    with pytest.raises(task.TaskError, match="scene"):
        env.reset(ep)


def test_step_limit_termination(nb, square):  # test_task.py:103
    from paper_1904_01201_b200 import task
    env = task.Environment(square, sensor_configs=())
    env.reset(episode_for(square, (2.0, 5.0), 0.0, (7.0, 5.0)))
    done, count = False, 0
    while not done:
        _, done, _ = env.step(nb.Action.TURN_LEFT)
        count += 1
        assert count <= 500
    assert count == 500
    out = env.outcome
    assert out.terminated_by == "step_limit" and not out.success and out.spl == 0.0
    with pytest.raises(task.TaskError, match="finished"):
        env.step(nb.Action.TURN_LEFT)


def test_stop_success_and_failure_radii(nb, square):  # test_task.py:121
    from paper_1904_01201_b200 import task
    env = task.Environment(square, sensor_configs=())
    ep = episode_for(square, (2.0, 5.0), 0.0, (7.0, 5.0))
    env.reset(ep)
    for _ in range(19):
        env.step(nb.Action.MOVE_FORWARD)
    _, done, info = env.step(nb.Action.STOP)
    assert done and info["outcome"].terminated_by == "stop"
    assert not info["outcome"].success
    env.reset(ep)
    for _ in range(20):
        env.step(nb.Action.MOVE_FORWARD)
    _, done, info = env.step(nb.Action.STOP)
    assert done and info["outcome"].success
    assert info["outcome"].spl == pytest.approx(ep.gdsp / max(5.0, ep.gdsp), abs=1e-6)
    # success implies the stop pose is within 0.2 m geodesic (test_task.py:178)
    from paper_1904_01201_b200 import nav
    assert nav.geodesic_distance(env.field, env.sim.state.position) <= 0.2


def test_reward_stream_telescopes_in_env(nb, square):  # test_task.py:141
    from paper_1904_01201_b200 import nav, task
    env = task.Environment(square, sensor_configs=())
    env.reset(episode_for(square, (2.0, 5.0), 0.3, (7.0, 5.0)))
    rng = np.random.default_rng(0)
    d0 = nav.geodesic_distance(env.field, env.sim.state.position)
    total, steps = 0.0, 0
    acts = (nb.Action.MOVE_FORWARD, nb.Action.TURN_LEFT, nb.Action.TURN_RIGHT)
    for _ in range(60):
        _, done, info = env.step(acts[int(rng.integers(3))])
        total += info["reward"]
        steps += 1
        if done:
            break
    d_end = nav.geodesic_distance(env.field, env.sim.state.position)
    assert total == pytest.approx(d0 - d_end + steps * (-0.01), abs=1e-9)


def test_outcome_determinism(nb, square):  # test_task.py:160
    from paper_1904_01201_b200 import task
    A = nb.Action
    actions = [A.MOVE_FORWARD] * 12 + [A.TURN_LEFT] * 3 + [A.MOVE_FORWARD] * 8 + [A.STOP]
    ep = episode_for(square, (2.0, 5.0), 0.1, (7.0, 5.0))
    outs = [task.run_episode(task.Environment(square, sensor_configs=()), ep, actions)
            for _ in range(2)]
    assert outs[0] == outs[1]


# ---------------------------------------------------------- test_nav.py

def test_rasterize_inset_square_and_boundary_rule(nb, square):  # test_nav.py:29, :41
    grid = grid_for(square)
    ii, jj = np.nonzero(grid.navigable)
    xs, ys = grid.origin[0] + 0.05 * jj, grid.origin[1] + 0.05 * ii
    for v, want in ((xs.min(), 0.1), (xs.max(), 9.9), (ys.min(), 0.1), (ys.max(), 9.9)):
        assert abs(v - want) <= 0.05 + 1e-9
    i, j = grid.cell_of((0.1, 5.0))
    if abs(grid.center_of(i, j)[0] - 0.1) < 1e-12:
        assert grid.navigable[i, j]
    i, j = grid.cell_of((0.05, 5.0))
    assert not grid.navigable[i, j]


def test_rasterize_split_room_two_components(nb):  # test_nav.py:52
    from scipy import ndimage
    walls = rect_walls(0, 0, 10, 10) + [((5.0, 0.0), (5.0, 10.0), 9)]
    grid = grid_for(make_scene(nb, walls))
    _, count = ndimage.label(grid.navigable, structure=[[0, 1, 0], [1, 1, 1], [0, 1, 0]])
    assert count == 2


def test_rasterize_rejects_bad_args(nb, square):  # test_nav.py:62
    from paper_1904_01201_b200 import nav
    with pytest.raises(nav.NavError):
        nav.rasterize_navigable(square.segment_array(), square.bounds(), -1.0)
    with pytest.raises(ValueError):
        nav.rasterize_navigable(square.segment_array(), (5, 5, 5, 5), 0.05)


def test_distance_field_straight_line_and_goal_checks(nb, square):  # test_nav.py:69, :76
    from paper_1904_01201_b200 import nav
    grid = grid_for(square)
    field = nav.distance_field(grid, (2.0, 5.0))
    assert nav.geodesic_distance(field, (7.0, 5.0)) == pytest.approx(5.0, abs=2 * grid.resolution)
    with pytest.raises(nav.NavError, match="not navigable"):
        nav.distance_field(grid, (-3.0, 5.0))


def test_distance_field_unreachable_pocket(nb):  # test_nav.py:143
    from paper_1904_01201_b200 import nav
    walls = rect_walls(0, 0, 10, 10) + rect_walls(4, 4, 6, 6, sid=10)
    grid = grid_for(make_scene(nb, walls))
    field = nav.distance_field(grid, (1.0, 1.0))
    assert math.isinf(nav.geodesic_distance(field, (5.0, 5.0)))


def test_geodesic_identities_and_bounds(nb, square):  # test_nav.py:152, :170
    from paper_1904_01201_b200 import nav
    grid = grid_for(square)
    field = nav.distance_field(grid, (5.0, 5.0))
    assert nav.geodesic_distance(field, grid.center_of(*field.goal_cell)) <= grid.resolution
    i, j = grid.cell_of((3.0, 7.0))
    assert nav.geodesic_distance(field, grid.center_of(i, j)) == pytest.approx(field.dist[i, j],
                                                                              abs=1e-12)
    with pytest.raises(nav.NavError, match="outside grid"):
        nav.geodesic_distance(field, (50.0, 5.0))


def test_sample_navigable_deterministic(nb, square):  # test_nav.py:208
    from paper_1904_01201_b200 import nav
    grid = grid_for(square)
    a = [nav.sample_navigable(grid, np.random.default_rng(9)) for _ in range(10)]
    b = [nav.sample_navigable(grid, np.random.default_rng(9)) for _ in range(10)]
    assert np.array_equal(np.array(a), np.array(b))


def _gen_scene(nb, name):
    from conftest import load_golden
    g = load_golden(name)
    walls = [((float(s[0]), float(s[1])), (float(s[2]), float(s[3])), int(i))
             for s, i in zip(g["segments"], g["semantic_ids"])]
    return make_scene(nb, walls, name)


def test_field_relaxation_triangle_inequality(nb):  # test_nav.py:240
    from paper_1904_01201_b200 import nav
    grid = grid_for(_gen_scene(nb, "gen101"))
    field = nav.distance_field(grid, nav.sample_navigable(grid, np.random.default_rng(4)))
    d, m, res = field.dist, grid.navigable, grid.resolution
    h, w = d.shape
    for di, dj, cost in ((0, 1, res), (1, 0, res), (1, 1, res * math.sqrt(2)),
                         (1, -1, res * math.sqrt(2))):
        if dj >= 0:
            a, b = d[:h - di or h, :w - dj or w], d[di:, dj:]
            ok = m[:h - di or h, :w - dj or w] & m[di:, dj:]
            if di and dj:
                ok &= m[:h - di, dj:] & m[di:, :w - dj]
        else:
            a, b = d[:h - di, -dj:], d[di:, :w + dj]
            ok = m[:h - di, -dj:] & m[di:, :w + dj] & m[:h - di, :w + dj] & m[di:, -dj:]
        fin = ok & np.isfinite(a) & np.isfinite(b)
        assert np.all(np.abs(a[fin] - b[fin]) <= cost + 1e-9)


def test_geodesic_dominates_euclidean(nb):  # test_nav.py:266
    from paper_1904_01201_b200 import nav
    grid = grid_for(_gen_scene(nb, "room1000"))
    rng = np.random.default_rng(12)
    goal = nav.sample_navigable(grid, rng)
    field = nav.distance_field(grid, goal)
    for _ in range(200):
        p = nav.sample_navigable(grid, rng)
        d = nav.geodesic_distance(field, p)
        if np.isfinite(d):
            assert d >= math.hypot(p[0] - goal[0], p[1] - goal[1]) - 2 * grid.resolution
