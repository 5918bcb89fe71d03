"""BatchSimulator: N environments stepped and rendered per call, on one GPU.

This is the hot path the benchmark measures: ``Simulator.step`` +
``Simulator.observations`` (sim.py:192-219) for every env at once, driven
through the C ABI (nv_step_render) on the caller's CUDA stream.  Actions,
agent state and frames stay in HBM; PyTorch only owns the buffers and the
stream.  One process per GPU; envs shard across GPUs (see ``dist.py``).
"""
from __future__ import annotations

import math

import numpy as np

from . import _native as nat
from .geometry import _upload_scene
from .sensors import (_CHANNEL_BIT, SensorConfig, SensorError, default_sensor_suite,
                      sensor_groups)


class SimError(Exception):
    pass


class _DevArray:
    """Zero-copy view of a device buffer (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


ACTION_CODES = {"move_forward": 0, "turn_left": 1, "turn_right": 2, "stop": 3}


class BatchSimulator:
    """Device-resident batch of ``n_envs`` agents in one scene.

    Parameters mirror ``Simulator(graph, agent, sensor_configs)`` with the
    scene given as flattened arrays (scene.flatten_arrays output)."""

    def __init__(self, segments, semantic_ids, albedo, n_envs: int, agent=None,
                 sensor_configs=None, wall_height: float = 2.5,
                 floor_color=(0.35, 0.33, 0.30), ceiling_color=(0.85, 0.85, 0.85),
                 device: int = 0):
        import torch
        from .sim import AgentConfig
        self.agent = agent or AgentConfig()
        self.sensor_configs = tuple(default_sensor_suite() if sensor_configs is None
                                    else sensor_configs)
        if self.agent.sensor_height > wall_height:
            raise SimError(f"sensor height {self.agent.sensor_height} exceeds wall height "
                           f"{wall_height}")
        self.wall_height = float(wall_height)
        self.n_envs = int(n_envs)
        self.device = device
        self.dev = f"cuda:{device}"
        self.ctx = nat.Context(device)
        c = self.ctx
        _upload_scene(c, segments, semantic_ids, albedo, wall_height, floor_color, ceiling_color)
        self.n_segments = len(np.asarray(segments).reshape(-1, 4))
        nat.check(c.lib.nv_agent_config(c.handle, float(self.agent.radius),
                                        float(self.agent.forward_step),
                                        math.radians(self.agent.turn_angle),
                                        float(self.agent.sensor_height)))
        nat.check(c.lib.nv_envs_alloc(c.handle, self.n_envs))
        self.groups = []
        N = self.n_envs
        for cam, ((w, h, hfov, max_range), members) in enumerate(
                sensor_groups(self.sensor_configs).items()):
            if cam >= 8:
                raise SensorError("at most 8 distinct camera configurations")
            nat.check(c.lib.nv_camera_config(c.handle, cam, w, h, members[0].focal,
                                             float(max_range)))
            kinds = {m.kind for m in members}
            g = {"cam": cam, "width": w, "height": h, "kinds": kinds,
                 "rgb": torch.empty((N, h, w, 3), dtype=torch.uint8, device=self.dev)
                 if "rgb" in kinds else None,
                 "depth": torch.empty((N, h, w), dtype=torch.float32, device=self.dev)
                 if "depth" in kinds else None,
                 "semantic": torch.empty((N, h, w), dtype=torch.uint16, device=self.dev)
                 if "semantic" in kinds else None}
            self.groups.append(g)
        self.want_gps = any(s.kind == "gps_compass" for s in self.sensor_configs)
        self.gps = torch.empty((N, 2), dtype=torch.float64, device=self.dev)
        self.compass = torch.empty((N,), dtype=torch.float64, device=self.dev)
        self.collided = torch.empty((N,), dtype=torch.uint8, device=self.dev)
        self.displacement = torch.empty((N,), dtype=torch.float64, device=self.dev)
        self.status = torch.empty((N,), dtype=torch.int32, device=self.dev)
        self._reset_done = np.zeros(N, dtype=bool)

    # ------------------------------------------------------------------ reset
    def reset(self, positions, headings, mask=None, raise_on_error: bool = True):
        """Simulator.set_agent_state for every env with mask != 0 (sim.py:172-184).
        Returns (status, clearance) host arrays."""
        N = self.n_envs
        xy = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(N, 2))
        hd = np.ascontiguousarray(np.asarray(headings, dtype=np.float64).reshape(N))
        m = None if mask is None else np.ascontiguousarray(np.asarray(mask, dtype=np.uint8).reshape(N))
        st = np.zeros(N, dtype=np.int32)
        cl = np.zeros(N, dtype=np.float64)
        rc = self.ctx.lib.nv_set_poses(self.ctx.handle, nat.ptr(xy), nat.ptr(hd), nat.ptr(m),
                                       nat.ptr(st), nat.ptr(cl))
        if rc == nat.NV_ERR_ARG and raise_on_error:
            bad = int(np.nonzero(st == nat.NV_ENV_TOO_CLOSE)[0][0])
            raise SimError(f"position ({xy[bad, 0]:.3f}, {xy[bad, 1]:.3f}) is {cl[bad]:.3f} m "
                           f"from the nearest wall; agent radius is {self.agent.radius}")
        if rc not in (nat.NV_OK, nat.NV_ERR_ARG):
            nat.check(rc)
        ok = st == nat.NV_ENV_OK if m is None else (st == nat.NV_ENV_OK) & (m != 0)
        self._reset_done |= ok
        return st, cl

    # ------------------------------------------------------------------- step
    def step(self, actions, render: bool = True, stream=None):
        """One simulator step for all envs: actions is a device int8 tensor of
        action codes (0 forward, 1 left, 2 right, 3 stop).  Enqueues on the
        current stream; returns the (reused) output tensors."""
        import torch
        assert actions.dtype == torch.int8 and actions.is_cuda and actions.numel() == self.n_envs
        c = self.ctx
        st = nat.stream_handle(self.dev) if stream is None else stream
        gps = nat.ptr(self.gps) if self.want_gps else None
        comp = nat.ptr(self.compass) if self.want_gps else None
        if render and self.groups:
            g0 = self.groups[0]
            nat.check(c.lib.nv_step_render(c.handle, nat.ptr(actions), g0["cam"],
                                           nat.ptr(g0["rgb"]), nat.ptr(g0["depth"]),
                                           nat.ptr(g0["semantic"]), gps, comp,
                                           nat.ptr(self.collided), nat.ptr(self.displacement),
                                           nat.ptr(self.status), st))
            for g in self.groups[1:]:
                nat.check(c.lib.nv_render(c.handle, g["cam"], nat.ptr(g["rgb"]),
                                          nat.ptr(g["depth"]), nat.ptr(g["semantic"]), None,
                                          None, st))
        else:
            nat.check(c.lib.nv_step(c.handle, nat.ptr(actions), nat.ptr(self.collided),
                                    nat.ptr(self.displacement), nat.ptr(self.status), st))
            if render and self.want_gps:
                nat.check(c.lib.nv_gps_compass(c.handle, gps, comp, st))
        return self

    def render(self, stream=None):
        """observations() for all envs at the current poses (sim.py:192-200)."""
        c = self.ctx
        st = nat.stream_handle(self.dev) if stream is None else stream
        if self.want_gps and not self.groups:
            nat.check(c.lib.nv_gps_compass(c.handle, nat.ptr(self.gps), nat.ptr(self.compass), st))
        for k, g in enumerate(self.groups):
            nat.check(c.lib.nv_render(c.handle, g["cam"], nat.ptr(g["rgb"]), nat.ptr(g["depth"]),
                                      nat.ptr(g["semantic"]),
                                      nat.ptr(self.gps) if (k == 0 and self.want_gps) else None,
                                      nat.ptr(self.compass) if (k == 0 and self.want_gps) else None,
                                      st))
        return self.observations()

    def observations(self) -> dict:
        out = {}
        for g in self.groups:
            for k in ("rgb", "depth", "semantic"):
                if g[k] is not None:
                    out[k] = g[k]
        if self.want_gps:
            out["gps"] = self.gps
            out["compass"] = self.compass
        return out

    # ------------------------------------------------------------------ state
    def state(self):
        """(positions (N,2), headings, path_length, collision_count) device tensors."""
        import torch
        N = self.n_envs
        xy = torch.empty((N, 2), dtype=torch.float64, device=self.dev)
        h = torch.empty((N,), dtype=torch.float64, device=self.dev)
        p = torch.empty((N,), dtype=torch.float64, device=self.dev)
        k = torch.empty((N,), dtype=torch.int64, device=self.dev)
        nat.check(self.ctx.lib.nv_get_state(self.ctx.handle, nat.ptr(xy), nat.ptr(h), nat.ptr(p),
                                            nat.ptr(k), nat.stream_handle(self.dev)))
        return xy, h, p, k

    def episode_frames(self):
        import torch
        N = self.n_envs
        o = torch.empty((N, 2), dtype=torch.float64, device=self.dev)
        h = torch.empty((N,), dtype=torch.float64, device=self.dev)
        nat.check(self.ctx.lib.nv_get_frame(self.ctx.handle, nat.ptr(o), nat.ptr(h),
                                            nat.stream_handle(self.dev)))
        return o, h

    def step_host(self, actions_host: np.ndarray, channels=None, frames_to_host: bool = False,
                  out=None, stream=None):
        """End-to-end step through the host-buffer C ABI (nv_step_render_host):
        host actions in, host step results out (and host frames if asked).
        Every camera group is rendered (the first one carries the step and
        gps/compass); the frames stay in context-owned device buffers
        (``host_step_frames``).  ``frames_to_host`` copies them into
        ``out['rgb'|'depth'|'semantic']`` and needs a single camera group;
        ``channels`` (NV_CH_* bits) restricts a single group's channels."""
        o = out or {}
        key = (id(o), frames_to_host, channels, stream)
        args = getattr(self, "_host_args", None)
        if args is None or args[0] != key:
            # the argument tuple is built once per (out buffers, mode); a step
            # then costs one pointer conversion and the C call
            if not self.groups:
                raise SensorError("the host-buffer step renders at least one camera sensor")
            if frames_to_host and len(self.groups) > 1:
                raise SensorError("frames_to_host needs a single camera group")
            c = self.ctx
            st = nat.stream_handle(self.dev) if stream is None else stream
            if len(self.groups) == 1:
                g = self.groups[0]
                cam = g["cam"]
                bits = channels if channels is not None else self._group_bits(g)
            else:
                cam = nat.NV_ALL_CAMERAS
                bits = 0
                for g in self.groups:
                    bits |= self._group_bits(g) << (3 * g["cam"])
            tail = (nat.ptr(o.get("rgb")) if frames_to_host else None,
                    nat.ptr(o.get("depth")) if frames_to_host else None,
                    nat.ptr(o.get("semantic")) if frames_to_host else None,
                    nat.ptr(o.get("gps")), nat.ptr(o.get("compass")), nat.ptr(o.get("collided")),
                    nat.ptr(o.get("displacement")), st)
            args = (key, c.lib.nv_step_render_host, c.handle, cam, bits, tail, o)
            self._host_args = args
        _, fn, h, cam, bits, tail, _ = args
        rc = fn(h, actions_host.ctypes.data if hasattr(actions_host, "ctypes") else nat.ptr(actions_host),
                cam, bits, *tail)
        if rc:
            nat.check(rc)
        return o

    @staticmethod
    def _group_bits(g) -> int:
        bits = 0
        for k in g["kinds"]:
            bits |= _CHANNEL_BIT[k]
        return bits

    def host_step_frames(self) -> dict:
        """Device frames written by the last ``step_host`` (all camera
        groups; waits for the frame writers): {kind: torch tensor view}."""
        import ctypes
        import torch
        out = {}
        for g in self.groups:
            p = [ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()]
            nat.check(self.ctx.lib.nv_host_frames(self.ctx.handle, g["cam"], *(ctypes.byref(x) for x in p)))
            N, h, w = self.n_envs, g["height"], g["width"]
            for kind, ptr_, shape, typestr, dt in (
                    ("rgb", p[0], (N, h, w, 3), "|u1", torch.uint8),
                    ("depth", p[1], (N, h, w), "<f4", torch.float32),
                    ("semantic", p[2], (N, h, w), "<u2", torch.uint16)):
                if kind in g["kinds"] and ptr_.value:
                    out[kind] = torch.as_tensor(_DevArray(ptr_.value, shape, typestr), device=self.dev)
        return out

    def launches(self) -> int:
        return self.ctx.launches()
