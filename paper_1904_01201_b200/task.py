"""PointGoal task at the drop-in boundary (reference: pkg/src/navsim/task.py).

``BatchEnvironment`` runs ``Environment.reset/step`` (task.py:123-243) for N
envs of one scene on one GPU: the agent step and the sensors through
nv_step_render, then the task arithmetic -- geodesic distance to the goal
(with the reference's 1 m line-of-sight shortcut), success, SPL, the shaped
reward, termination and the 40-byte EpisodeOutcome records -- through
nv_task_step, all on the caller's stream with no host synchronisation.
Goal fields are built on the device (nav.distance_fields) once per distinct
goal cell, like the reference's FieldCache.  ``Environment`` is the
reference's single-env API over a one-env batch.
"""
from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from . import _native as nat
from . import nav
from . import scene as scene_mod
from .batch import BatchSimulator
from .sensors import EpisodeFrame, Observations, default_sensor_suite, frames_to_host
from .sim import Action, AgentConfig, AgentState, _CODE

MAX_EPISODE_STEPS = 500   # task.py:24
SUCCESS_RADIUS = 0.2      # task.py:25

__all__ = ["MAX_EPISODE_STEPS", "SUCCESS_RADIUS", "TaskError", "Episode", "RewardParams",
           "EpisodeOutcome", "success_test", "spl", "reward", "BatchEnvironment", "Environment",
           "run_episode", "OUTCOME_DTYPE"]


class TaskError(Exception):
    pass


@dataclass(frozen=True)
class Episode:
    episode_id: str
    scene_id: str
    start_position: tuple[float, float]
    start_heading: float
    goal_position: tuple[float, float]
    gdsp: float
    euclidean: float
    ratio: float

    def validate(self, resolution: float = nav.DEFAULT_RESOLUTION) -> None:
        if not (1.0 - 1e-9 <= self.gdsp <= 30.0 + 1e-9):
            raise TaskError(f"episode {self.episode_id}: gdsp {self.gdsp} outside [1, 30] m")
        if self.gdsp < self.euclidean - 2.0 * resolution:
            raise TaskError(f"episode {self.episode_id}: gdsp below euclidean distance")
        if self.euclidean > 0 and abs(self.ratio - self.gdsp / self.euclidean) > 1e-6:
            raise TaskError(f"episode {self.episode_id}: ratio inconsistent with gdsp/euclidean")


@dataclass(frozen=True)
class RewardParams:
    success_reward: float = 10.0
    step_penalty: float = -0.01


@dataclass(frozen=True)
class EpisodeOutcome:
    success: bool
    shortest_path: float
    path_taken: float
    spl: float
    steps: int
    collisions: int
    terminated_by: str     # "stop" | "step_limit"

    def to_json(self) -> str:
        return json.dumps(asdict(self), sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "EpisodeOutcome":
        return cls(**json.loads(text))


# nv_task_step's 40-byte outcome record (include/navsim_b200.h)
OUTCOME_DTYPE = np.dtype([("success", "u1"), ("terminated_by", "u1"), ("pad", "u1", 2),
                          ("steps", "<i4"), ("collisions", "<i4"), ("pad2", "<i4"),
                          ("path_taken", "<f8"), ("shortest_path", "<f8"), ("spl", "<f8")])
assert OUTCOME_DTYPE.itemsize == 40


def success_test(d_stop: float, radius: float = SUCCESS_RADIUS) -> bool:
    return d_stop <= radius


def spl(success: bool, shortest: float, taken: float) -> float:
    if shortest <= 0.0:
        raise TaskError("shortest path must be positive for SPL")
    if taken < 0.0:
        raise TaskError("path taken cannot be negative")
    if not success:
        return 0.0
    return shortest / max(taken, shortest)


def reward(d_prev: float, d_cur: float, reached: bool,
           params: RewardParams = RewardParams()) -> float:
    base = d_prev - d_cur + params.step_penalty
    return base + params.success_reward if reached else base


def outcome_from_record(rec) -> EpisodeOutcome:
    return EpisodeOutcome(success=bool(rec["success"]), shortest_path=float(rec["shortest_path"]),
                          path_taken=float(rec["path_taken"]), spl=float(rec["spl"]),
                          steps=int(rec["steps"]), collisions=int(rec["collisions"]),
                          terminated_by="stop" if int(rec["terminated_by"]) == 1 else "step_limit")


def _scene_arrays(scene):
    """(segments, semantic ids, albedo, wall height, floor, ceiling, bounds, id)."""
    if isinstance(scene, (tuple, list)):
        segs, sem, alb = scene[:3]
        segs = np.asarray(segs, dtype=np.float64).reshape(-1, 4)
        b = (float(min(segs[:, 0].min(), segs[:, 2].min())),
             float(min(segs[:, 1].min(), segs[:, 3].min())),
             float(max(segs[:, 0].max(), segs[:, 2].max())),
             float(max(segs[:, 1].max(), segs[:, 3].max())))
        return segs, sem, alb, 2.5, (0.35, 0.33, 0.30), (0.85, 0.85, 0.85), b, None
    graph = scene_mod.build_scene_graph(scene)
    segs, sem, alb = scene_mod.flatten_arrays(graph)
    return (segs, sem, alb, scene.wall_height, scene.floor_color, scene.ceiling_color,
            scene.bounds(), scene.id)


class BatchEnvironment:
    """N PointGoal environments of one scene, stepped together on one GPU."""

    def __init__(self, scene, n_envs: int, agent: AgentConfig | None = None,
                 sensor_configs=None, reward_params: RewardParams = RewardParams(),
                 resolution: float = nav.DEFAULT_RESOLUTION, device: int = 0,
                 max_steps: int = MAX_EPISODE_STEPS, depth_noise_sigma: float = 0.0,
                 noise_seed: int = 0, env_offset: int = 0):
        import torch
        segs, sem, alb, wall_h, floor, ceil, bounds, sid = _scene_arrays(scene)
        self.scene_id = sid
        self.agent = agent or AgentConfig()
        self.reward_params = reward_params
        self.sim = BatchSimulator(segs, sem, alb, n_envs, self.agent,
                                  default_sensor_suite() if sensor_configs is None
                                  else sensor_configs, wall_h, floor, ceil, device)
        self.n_envs = self.sim.n_envs
        self.dev = self.sim.dev
        c = self.sim.ctx
        self.grid = nav.build_grid(c, bounds, resolution, self.agent.radius)
        if depth_noise_sigma < 0.0:
            from .sensors import SensorError
            raise SensorError("sigma must be non-negative")
        self.depth_noise_sigma = float(depth_noise_sigma)
        self.noise_seed = int(noise_seed)
        self.env_offset = int(env_offset)
        nat.check(c.lib.nv_depth_noise(c.handle, self.depth_noise_sigma,
                                       self.noise_seed & 0xFFFFFFFFFFFFFFFF, self.env_offset))
        nat.check(c.lib.nv_task_config(c.handle, int(max_steps), SUCCESS_RADIUS,
                                       float(reward_params.success_reward),
                                       float(reward_params.step_penalty)))
        self.fused_task = True             # agent + task step in one kernel (nv_task_step_render)
        N = self.n_envs
        self.fields = None                 # f64[k, h, w] device fields, one per goal cell
        self._field_of: dict = {}          # goal cell -> field index (FieldCache)
        self.episodes = [None] * N
        self._goal = np.zeros((N, 2))
        self._gdsp = np.ones(N)
        self._fid = np.zeros(N, dtype=np.int32)
        self.goal_in_frame = torch.zeros((N, 2), dtype=torch.float64, device=self.dev)
        self.reward = torch.zeros(N, dtype=torch.float64, device=self.dev)
        self.dist = torch.zeros(N, dtype=torch.float64, device=self.dev)
        self.done = torch.zeros(N, dtype=torch.uint8, device=self.dev)
        self.outcome = torch.zeros((N, 40), dtype=torch.uint8, device=self.dev)

    # ---------------------------------------------------------------- reset
    def _ensure_fields(self, cells):
        import torch
        new = [tuple(c) for c in cells if tuple(c) not in self._field_of]
        new = list(dict.fromkeys(new))
        if not new:
            return
        cc = np.ascontiguousarray(np.asarray(new, dtype=np.int32))
        f = torch.empty((len(new), self.grid.height, self.grid.width), dtype=torch.float64,
                        device=self.dev)
        c = self.sim.ctx
        nat.check(c.lib.nv_nav_fields(c.handle, nat.ptr(cc), len(cc), nat.ptr(f),
                                      nat.stream_handle(self.dev)))
        base = 0 if self.fields is None else self.fields.shape[0]
        self.fields = f if self.fields is None else torch.cat([self.fields, f], dim=0)
        for k, cell in enumerate(new):
            self._field_of[cell] = base + k

    def reset(self, episodes, mask=None) -> dict:
        """Environment.reset (task.py:179-190) for every env with mask != 0;
        ``episodes`` has one Episode per env (entries of unmasked envs are
        ignored).  Returns the observations dict (device tensors) with the
        goal in each env's episode frame under ``"goal"``."""
        N = self.n_envs
        m = np.ones(N, dtype=bool) if mask is None else np.asarray(mask, dtype=bool).reshape(N)
        idx = np.nonzero(m)[0]
        for e in idx:
            ep = episodes[e]
            if self.scene_id is not None and ep.scene_id != self.scene_id:
                raise TaskError(f"episode {ep.episode_id} is for scene {ep.scene_id!r}, "
                                f"environment holds {self.scene_id!r}")
            ep.validate(self.grid.resolution)
        goals = np.array([episodes[e].goal_position for e in idx], dtype=np.float64).reshape(-1, 2)
        cells = self.grid.snap(goals)
        bad = np.nonzero(cells[:, 0] < 0)[0]
        if len(bad):
            g = goals[bad[0]]
            raise TaskError(f"goal ({g[0]:.3f}, {g[1]:.3f}) is not navigable")
        self._ensure_fields(cells)
        starts = np.zeros((N, 2))
        heads = np.zeros(N)
        for k, e in enumerate(idx):
            ep = episodes[e]
            starts[e] = ep.start_position
            heads[e] = ep.start_heading
            self._goal[e] = goals[k]
            self._gdsp[e] = ep.gdsp
            self._fid[e] = self._field_of[tuple(cells[k])]
            self.episodes[e] = ep
        # _snap_start (task.py:149-156): keep starts that clear the walls,
        # else the nearest navigable cell center
        st, _ = self.sim.reset(starts, heads, mask=m, raise_on_error=False)
        far = np.nonzero(m & (st == nat.NV_ENV_TOO_CLOSE))[0]
        if len(far):
            sc = self.grid.snap(starts[far])
            if (sc[:, 0] < 0).any():
                p = starts[far[int(np.nonzero(sc[:, 0] < 0)[0][0])]]
                raise TaskError(f"start {tuple(p)} not navigable after snapping")
            for k, e in enumerate(far):
                starts[e] = self.grid.center_of(int(sc[k, 0]), int(sc[k, 1]))
            m2 = np.zeros(N, dtype=bool)
            m2[far] = True
            self.sim.reset(starts, heads, mask=m2)
        c = self.sim.ctx
        d0 = np.zeros(N)
        mm = np.ascontiguousarray(m.astype(np.uint8))
        nat.check(c.lib.nv_task_reset(c.handle, nat.ptr(np.ascontiguousarray(self._goal)),
                                      nat.ptr(np.ascontiguousarray(self._gdsp)),
                                      nat.ptr(np.ascontiguousarray(self._fid)),
                                      nat.ptr(self.fields), self.fields.shape[0], nat.ptr(mm),
                                      nat.ptr(d0)))
        self.d0 = d0
        # goal in each episode frame (EpisodeFrame.to_frame, sensors.py:166-168)
        o, h = self.sim.episode_frames()
        o, h = o.cpu().numpy(), h.cpu().numpy()
        gf = self.goal_in_frame.cpu().numpy()
        for e in idx:
            gf[e] = EpisodeFrame(origin=o[e], heading=float(h[e])).to_frame(self._goal[e])
        self.goal_in_frame.copy_(__import__("torch").from_numpy(gf))
        obs = self.sim.render()
        obs["goal"] = self.goal_in_frame
        return obs

    # ----------------------------------------------------------------- step
    def step(self, actions, stream=None):
        """Environment.step for all envs: actions is a device int8 tensor of
        action codes.  Returns (observations, done, info) as device tensors;
        info["outcome"] holds the 40-byte EpisodeOutcome records (valid for
        envs that terminated).  Finished envs stay frozen until reset."""
        c = self.sim.ctx
        sim = self.sim
        if sim.groups and self.fused_task:
            # one call: agent step + task arithmetic, cast, fill; the argument
            # tail (all buffers are owned by this object) is built once
            key = stream
            cached = getattr(self, "_step_args", None)
            if cached is None or cached[0] != key:
                st = nat.stream_handle(self.dev) if stream is None else stream
                g0 = sim.groups[0]
                gps = nat.ptr(sim.gps) if sim.want_gps else None
                comp = nat.ptr(sim.compass) if sim.want_gps else None
                tail = (nat.ptr(g0["rgb"]), nat.ptr(g0["depth"]), nat.ptr(g0["semantic"]), gps,
                        comp, nat.ptr(sim.collided), nat.ptr(sim.displacement),
                        nat.ptr(sim.status), nat.ptr(self.reward), nat.ptr(self.dist),
                        nat.ptr(self.done), nat.ptr(self.outcome), st)
                cached = (key, c.lib.nv_task_step_render, c.handle, g0["cam"], tail)
                self._step_args = cached
            _, fn, h, cam, tail = cached
            rc = fn(h, actions.data_ptr(), cam, *tail)
            if rc:
                nat.check(rc)
            st = tail[-1]
            for g in sim.groups[1:]:
                nat.check(c.lib.nv_render(c.handle, g["cam"], nat.ptr(g["rgb"]),
                                          nat.ptr(g["depth"]), nat.ptr(g["semantic"]), None,
                                          None, st))
        else:
            st = nat.stream_handle(self.dev) if stream is None else stream
            sim.step(actions, render=True, stream=stream)
            nat.check(c.lib.nv_task_step(c.handle, nat.ptr(actions), nat.ptr(sim.status),
                                         nat.ptr(self.reward), nat.ptr(self.dist),
                                         nat.ptr(self.done), nat.ptr(self.outcome), st))
        obs = self.sim.observations()
        obs["goal"] = self.goal_in_frame
        info = {"d": self.dist, "reward": self.reward, "collided": self.sim.collided,
                "displacement": self.sim.displacement, "status": self.sim.status,
                "outcome": self.outcome}
        return obs, self.done, info

    def outcomes(self):
        """Host EpisodeOutcome per env (None for running episodes)."""
        rec = self.outcome.cpu().numpy().view(OUTCOME_DTYPE).reshape(-1)
        done = self.done.cpu().numpy()
        return [outcome_from_record(r) if d else None for r, d in zip(rec, done)]

    def steps(self):
        import torch
        s = torch.empty(self.n_envs, dtype=torch.int32, device=self.dev)
        c = self.sim.ctx
        nat.check(c.lib.nv_task_state(c.handle, nat.ptr(s), None, None, nat.stream_handle(self.dev)))
        return s


class Environment:
    """One simulator bound to the episode lifecycle (task.py:123-250), on the
    GPU through a one-env BatchEnvironment."""

    def __init__(self, scene, agent: AgentConfig | None = None, sensor_configs=None,
                 reward_params: RewardParams = RewardParams(),
                 resolution: float = nav.DEFAULT_RESOLUTION, field_cache=None,
                 depth_noise_sigma: float = 0.0, noise_seed: int = 0, device: int = 0):
        self.scene = scene
        self.agent_config = agent or AgentConfig()
        self._b = BatchEnvironment(scene, 1, self.agent_config, sensor_configs, reward_params,
                                   resolution, device, depth_noise_sigma=depth_noise_sigma,
                                   noise_seed=noise_seed)
        self.grid = self._b.grid
        self.episode = None
        self.steps = 0
        self.done = False
        self._outcome = None

    def _obs(self, o) -> Observations:
        host = frames_to_host(o.get("rgb"), o.get("depth"), o.get("semantic"))
        obs = Observations()
        obs.rgb = None if "rgb" not in host else host["rgb"][0]
        obs.depth = None if "depth" not in host else host["depth"][0]
        obs.semantic = None if "semantic" not in host else host["semantic"][0]
        if "gps" in o:
            obs.gps = o["gps"][0].cpu().numpy().copy()
            obs.compass = float(o["compass"][0].item())
        obs.goal = o["goal"][0].cpu().numpy().copy()
        return obs

    def reset(self, episode: Episode) -> Observations:
        # the noise stream restarts with every episode (task.py:187)
        c = self._b.sim.ctx
        nat.check(c.lib.nv_depth_noise(c.handle, self._b.depth_noise_sigma,
                                       self._b.noise_seed & 0xFFFFFFFFFFFFFFFF, 0))
        obs = self._b.reset([episode])
        self.episode = episode
        self.steps = 0
        self.done = False
        self._outcome = None
        return self._obs(obs)

    def step(self, action: Action):
        import torch
        if self.episode is None:
            raise TaskError("environment must be reset before stepping")
        if self.done:
            raise TaskError("episode is finished; reset before stepping again")
        act = torch.tensor([_CODE[action]], dtype=torch.int8, device=self._b.dev)
        obs, done, info = self._b.step(act)
        self.steps += 1
        self.done = bool(done[0].item())
        out = {"d": float(info["d"][0].item()), "collided": bool(info["collided"][0].item()),
               "reward": float(info["reward"][0].item()), "steps": self.steps,
               "displacement": float(info["displacement"][0].item())}
        if self.done:
            self._outcome = self._b.outcomes()[0]
            out["outcome"] = self._outcome
        return self._obs(obs), self.done, out

    @property
    def outcome(self) -> EpisodeOutcome:
        if self._outcome is None:
            raise TaskError("episode has not terminated")
        return self._outcome

    @property
    def field(self) -> nav.DistanceField:
        """The current episode's goal distance field (task.py:140-141)."""
        if self.episode is None:
            raise TaskError("environment must be reset first")
        key = tuple(self.episode.goal_position)
        if getattr(self, "_field_key", None) != key:
            self._field = nav.distance_field(self.grid, self.episode.goal_position)
            self._field_key = key
        return self._field

    @property
    def sim(self) -> "_EnvAgentView":
        """The bound simulator's agent state (``env.sim.state``, task.py:123-135)."""
        return _EnvAgentView(self._b.sim)


class _EnvAgentView:
    def __init__(self, batch_sim):
        self._s = batch_sim

    @property
    def state(self) -> AgentState:
        xy, h, p, k = (t[0].item() if t.dim() == 1 else t[0].cpu().numpy() for t in self._s.state())
        return AgentState(position=xy, heading=float(h), cumulative_path_length=float(p),
                          collision_count=int(k))


def run_episode(env: Environment, episode: Episode, actions) -> EpisodeOutcome:
    """Replay a fixed action list; the step budget terminates long lists (task.py:246-256)."""
    env.reset(episode)
    for a in actions:
        _, done, _ = env.step(a if isinstance(a, Action) else Action.from_name(a))
        if done:
            break
    if not env.done:
        raise TaskError("action list ended before the episode terminated")
    return env.outcome
