"""Sensor API at the drop-in boundary (reference: pkg/src/navsim/sensors.py).

``render`` keeps the reference's signature, validation and errors
(sensors.py:105-152); the column cast and the frame fill run on the GPU
(nv_raycast -> nv_fill_frames).  Device frames are u8 RGB / f32 depth / u16
semantic; this facade returns them in the reference's host dtypes (rgb f64 in
[0, 1] within 1/255, depth f64 within f32 rounding, semantic u16 exact).  The
batched, device-resident path is :class:`paper_1904_01201_b200.batch.BatchSimulator`.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .geometry import SegmentIndex, _upload_scene, segment_normals, wrap_angle

SEM_VOID = 0          # _kernels.py:123
SEM_FLOOR = 65534     # _kernels.py:124
SEM_CEILING = 65535   # _kernels.py:125

VISUAL_KINDS = ("rgb", "depth", "semantic")
SENSOR_KINDS = VISUAL_KINDS + ("gps_compass",)
_CHANNEL_BIT = {"rgb": nat.NV_CH_RGB, "depth": nat.NV_CH_DEPTH, "semantic": nat.NV_CH_SEM}


class SensorError(Exception):
    pass


@dataclass(frozen=True)
class SensorConfig:
    kind: str
    width: int = 256
    height: int = 256
    hfov: float = 90.0
    max_range: float = 10.0

    def __post_init__(self):
        if self.kind not in SENSOR_KINDS:
            raise SensorError(f"unknown sensor kind {self.kind!r}")
        if self.kind in VISUAL_KINDS:
            if self.width < 1 or self.height < 1:
                raise SensorError("sensor resolution must be at least 1x1")
            if not (0.0 < self.hfov < 180.0):
                raise SensorError("hfov must be in (0, 180) degrees")
            if self.max_range <= 0.0:
                raise SensorError("max_range must be positive")

    @property
    def focal(self) -> float:
        """(W/2) / tan(hfov/2), sensors.py:55-57 (host f64, passed to the device)."""
        return (self.width * 0.5) / math.tan(math.radians(self.hfov) * 0.5)


def default_sensor_suite():
    return (SensorConfig("rgb"), SensorConfig("depth"), SensorConfig("gps_compass"))


@dataclass
class Observations:
    rgb: np.ndarray | None = None
    depth: np.ndarray | None = None
    semantic: np.ndarray | None = None
    gps: np.ndarray | None = None
    compass: float | None = None
    goal: np.ndarray | None = None


def sensor_groups(configs):
    """Validate and group visual sensors sharing one traversal (sensors.py:113-123)."""
    visual = [c for c in configs if c.kind in VISUAL_KINDS]
    kinds = [c.kind for c in visual]
    if len(set(kinds)) != len(kinds):
        raise SensorError("at most one sensor per visual kind")
    groups: dict = {}
    for c in visual:
        groups.setdefault((c.width, c.height, c.hfov, c.max_range), []).append(c)
    return groups


class RenderGeometry:
    """Device-resident render view of a scene (sensors.py:77-93)."""

    def __init__(self, segments, semantic_ids, albedo, wall_height, floor_color, ceiling_color,
                 device: int = 0):
        self.segments = np.asarray(segments, dtype=np.float64).reshape(-1, 4)
        self.semantic_ids = np.ascontiguousarray(semantic_ids, dtype=np.uint16)
        self.albedo = np.ascontiguousarray(albedo, dtype=np.float64).reshape(-1, 3)
        self.wall_height = float(wall_height)
        self.floor_color = np.asarray(floor_color, dtype=np.float64)
        self.ceiling_color = np.asarray(ceiling_color, dtype=np.float64)
        self._ctx = nat.Context(device)
        _upload_scene(self._ctx, self.segments, self.semantic_ids, self.albedo, self.wall_height,
                      self.floor_color, self.ceiling_color)
        self.index = SegmentIndex(self.segments, _ctx=self._ctx)
        n = segment_normals(self.segments)
        self.normal_x = np.ascontiguousarray(n[:, 0])
        self.normal_y = np.ascontiguousarray(n[:, 1])
        self._cams: dict = {}

    @property
    def context(self):
        return self._ctx

    def camera(self, width, height, focal, max_range) -> int:
        key = (width, height, focal, max_range)
        if key not in self._cams:
            cam = len(self._cams) % 8
            for k, v in list(self._cams.items()):
                if v == cam:
                    del self._cams[k]
            nat.check(self._ctx.lib.nv_camera_config(self._ctx.handle, cam, width, height,
                                                     float(focal), float(max_range)))
            self._cams[key] = cam
        return self._cams[key]


def _column_directions(heading: float, config: SensorConfig):
    """Per-column unnormalised directions with unit forward (sensors.py:96-102)."""
    u = (np.arange(config.width) + 0.5 - config.width * 0.5) / config.focal
    fx, fy = math.cos(heading), math.sin(heading)
    rx, ry = math.sin(heading), -math.cos(heading)
    return fx + u * rx, fy + u * ry


def frames_to_host(rgb, depth, sem):
    """Device u8/f32/u16 frames -> the reference's host dtypes."""
    out = {}
    if rgb is not None:
        out["rgb"] = rgb.cpu().numpy().astype(np.float64) / 255.0
    if depth is not None:
        out["depth"] = depth.cpu().numpy().astype(np.float64)
    if sem is not None:
        out["semantic"] = sem.cpu().numpy()
    return out


def render_device(geom: RenderGeometry, position, heading, sensor_height, configs,
                  brute_force: bool = False):
    """render() returning device tensors {kind: tensor (H, W[, 3])}."""
    import torch
    groups = sensor_groups(configs)
    if not groups:
        return {}
    if sensor_height > geom.wall_height:
        raise SensorError("sensor height must stay below wall height")
    ctx = geom.context
    dev = f"cuda:{ctx.device}"
    out = {}
    for (width, height, hfov, max_range), members in groups.items():
        proto = members[0]
        dirx, diry = _column_directions(heading, proto)
        dx = torch.as_tensor(dirx, device=dev)
        dy = torch.as_tensor(diry, device=dev)
        ox = torch.full((width,), float(position[0]), dtype=torch.float64, device=dev)
        oy = torch.full((width,), float(position[1]), dtype=torch.float64, device=dev)
        t = torch.empty(width, dtype=torch.float64, device=dev)
        i = torch.empty(width, dtype=torch.int64, device=dev)
        st = nat.stream_handle(dev)
        # SegmentIndex.raycast default t_max = 1e9 (geometry.py:165)
        nat.check(ctx.lib.nv_raycast(ctx.handle, nat.ptr(ox), nat.ptr(oy), nat.ptr(dx),
                                     nat.ptr(dy), width, 1e9, int(brute_force), nat.ptr(t),
                                     nat.ptr(i), st))
        kinds = {c.kind for c in members}
        rgb = torch.empty((height, width, 3), dtype=torch.uint8, device=dev) if "rgb" in kinds else None
        dep = torch.empty((height, width), dtype=torch.float32, device=dev) if "depth" in kinds else None
        sem = torch.empty((height, width), dtype=torch.uint16, device=dev) if "semantic" in kinds else None
        cam = geom.camera(width, height, proto.focal, max_range)
        nat.check(ctx.lib.nv_fill_frames(ctx.handle, cam, 1, nat.ptr(t), nat.ptr(i), nat.ptr(dx),
                                         nat.ptr(dy), float(sensor_height), nat.ptr(rgb),
                                         nat.ptr(dep), nat.ptr(sem), st))
        if rgb is not None:
            out["rgb"] = rgb
        if dep is not None:
            out["depth"] = dep
        if sem is not None:
            out["semantic"] = sem
    return out


def render(geom: RenderGeometry, position, heading: float, sensor_height: float, configs,
           brute_force: bool = False) -> Observations:
    """Render all requested visual channels from one GPU traversal per camera
    group (sensors.py:105-152)."""
    dev = render_device(geom, position, heading, sensor_height, configs, brute_force)
    obs = Observations()
    host = frames_to_host(dev.get("rgb"), dev.get("depth"), dev.get("semantic"))
    obs.rgb, obs.depth = host.get("rgb"), host.get("depth")
    obs.semantic = host.get("semantic")
    return obs


@dataclass(frozen=True)
class EpisodeFrame:
    """Episode coordinate frame (sensors.py:155-172)."""

    origin: np.ndarray
    heading: float

    def to_frame(self, p) -> np.ndarray:
        dx, dy = p[0] - self.origin[0], p[1] - self.origin[1]
        c, s = math.cos(-self.heading), math.sin(-self.heading)
        return np.array([c * dx - s * dy, s * dx + c * dy])

    def to_world(self, p) -> np.ndarray:
        c, s = math.cos(self.heading), math.sin(self.heading)
        return np.array([self.origin[0] + c * p[0] - s * p[1],
                         self.origin[1] + s * p[0] + c * p[1]])


def gps_compass(state, frame: EpisodeFrame):
    """Idealised GPS + compass in the episode frame (sensors.py:175-180)."""
    return frame.to_frame(state.position), wrap_angle(state.heading - frame.heading)


# ---------------------------------------------------------------------------
# frame codecs (sensors.py:211-246): PNG encoding on the device, one complete
# PNG per frame (nv_png_encode: quantisation, scanlines, zlib stored blocks,
# Adler-32 and CRC-32 on the GPU); decoding is the consumer's side (PIL).

def apply_inverse_depth_noise(depth, sigma: float, rng: np.random.Generator,
                              max_range: float = 10.0) -> np.ndarray:
    """sensors.apply_inverse_depth_noise (sensors.py:183-205): z' = max_range /
    (max_range / d + eps), eps ~ N(0, sigma), clipped to [0.05, max_range];
    saturated pixels (d >= max_range) pass through; sigma = 0 is the identity;
    sigma < 0 raises SensorError.  Runs on the GPU (nv_depth_noise_apply) in
    f32 with the device's counter-based normals keyed by one draw from
    ``rng`` -- the same ``rng`` state gives the same frame; numpy's normal
    stream itself is not reproduced (parity is the moment test)."""
    if sigma < 0.0:
        raise SensorError("sigma must be non-negative")
    d = np.asarray(depth, dtype=np.float64)
    if sigma == 0.0:
        return d.copy()
    import torch
    seed = int(rng.integers(0, 2 ** 63))
    H, W = (d.shape[-2], d.shape[-1]) if d.ndim >= 2 else (1, d.shape[-1])
    n = int(d.size // (H * W))
    t = torch.as_tensor(d.astype(np.float32)).reshape(n, H, W).to("cuda")
    lib = nat.load()
    nat.check(lib.nv_depth_noise_apply(nat.ptr(t), n, H, W, float(sigma), float(max_range),
                                       seed, 0, 0, nat.stream_handle(t.device)))
    return t.cpu().numpy().astype(np.float64).reshape(d.shape)


PNG_DEPTH, PNG_RGB, PNG_SEMANTIC = 0, 1, 2


def encode_frames(frames, kind: int, max_range: float = 10.0, stream=None):
    """PNG-encode a batch of frames on the GPU.  ``frames``: a CUDA tensor
    [n, H, W] (depth f32/f64, semantic u16) or [n, H, W, 3] (rgb u8/f64).
    Returns (out u8 CUDA tensor [n, size], size): row k is frame k's PNG."""
    import torch
    from . import _native as nat
    if not (isinstance(frames, torch.Tensor) and frames.is_cuda):
        raise SensorError("frames must be a CUDA tensor")
    f = frames.contiguous()
    n, H, W = int(f.shape[0]), int(f.shape[1]), int(f.shape[2])
    src_f64 = 1 if f.dtype == torch.float64 else 0
    want = {PNG_DEPTH: (torch.float32, torch.float64), PNG_RGB: (torch.uint8, torch.float64),
            PNG_SEMANTIC: (torch.uint16, torch.int16)}[kind]
    if f.dtype not in want:
        raise SensorError(f"frames of kind {kind} must be {want}, got {f.dtype}")
    lib = nat.load()
    size = int(lib.nv_png_size(kind, W, H))
    out = torch.empty((n, size), dtype=torch.uint8, device=f.device)
    st = nat.stream_handle(f.device) if stream is None else stream
    nat.check(lib.nv_png_encode(kind, src_f64, nat.ptr(f), n, W, H, float(max_range),
                                nat.ptr(out), size, st))
    return out, size


def _encode_one(arr, kind, max_range=10.0) -> bytes:
    import torch
    t = torch.as_tensor(np.ascontiguousarray(arr))[None].to("cuda")
    out, size = encode_frames(t, kind, max_range)
    return bytes(out[0].cpu().numpy().tobytes())


def depth_to_png(depth: np.ndarray, max_range: float = 10.0) -> bytes:
    """16-bit grayscale PNG; meters scale linearly so max_range -> 65535."""
    d = np.asarray(depth)
    if d.dtype != np.float32:
        d = d.astype(np.float64)
    return _encode_one(d, PNG_DEPTH, max_range)


def rgb_to_png(rgb: np.ndarray) -> bytes:
    r = np.asarray(rgb)
    if r.dtype != np.uint8:
        r = r.astype(np.float64)
    return _encode_one(r, PNG_RGB)


def semantic_to_png(semantic: np.ndarray) -> bytes:
    return _encode_one(np.asarray(semantic, dtype=np.uint16), PNG_SEMANTIC)


def png_to_depth(data: bytes, max_range: float = 10.0) -> np.ndarray:
    import io
    from PIL import Image
    arr = np.asarray(Image.open(io.BytesIO(data)), dtype=np.uint16)
    return arr.astype(np.float64) / 65535.0 * max_range


def png_to_rgb(data: bytes) -> np.ndarray:
    import io
    from PIL import Image
    arr = np.asarray(Image.open(io.BytesIO(data)).convert("RGB"), dtype=np.uint8)
    return arr.astype(np.float64) / 255.0


def png_to_semantic(data: bytes) -> np.ndarray:
    import io
    from PIL import Image
    return np.asarray(Image.open(io.BytesIO(data)), dtype=np.uint16)

