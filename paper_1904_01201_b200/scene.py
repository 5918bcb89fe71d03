"""Scene data model at the drop-in boundary: the input side of scene upload.

Mirrors the reference's in-memory types and the render flattening
(/root/reference/pkg/src/navsim/scene.py:40-76 data model, :233-346 scene
graph, :349-386 flatten).  JSON parsing, validation and procedural generation
are host tooling outside the hot path and are not
rebuilt.  ``flatten_arrays`` also accepts the reference's own SceneGraph
objects (duck-typed), so a reference scene can be handed to this simulator
unchanged.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DEFAULT_WALL_HEIGHT = 2.5   # scene.py:23


@dataclass(frozen=True)
class Transform2D:
    """Rotate by theta, then translate (geometry.py:27-55)."""

    tx: float = 0.0
    ty: float = 0.0
    theta: float = 0.0

    def compose(self, local: "Transform2D") -> "Transform2D":
        c, s = math.cos(self.theta), math.sin(self.theta)
        return Transform2D(self.tx + c * local.tx - s * local.ty,
                           self.ty + s * local.tx + c * local.ty,
                           self.theta + local.theta)

    def apply(self, points) -> np.ndarray:
        p = np.asarray(points, dtype=np.float64)
        c, s = math.cos(self.theta), math.sin(self.theta)
        out = np.empty_like(p)
        out[..., 0] = c * p[..., 0] - s * p[..., 1] + self.tx
        out[..., 1] = s * p[..., 0] + c * p[..., 1] + self.ty
        return out

    @property
    def is_identity(self) -> bool:
        return self.tx == 0.0 and self.ty == 0.0 and self.theta == 0.0


IDENTITY = Transform2D()


@dataclass(frozen=True)
class WallSegment:
    a: tuple
    b: tuple
    semantic_id: int
    albedo: tuple = (0.6, 0.6, 0.6)

    @property
    def length(self) -> float:
        return math.hypot(self.b[0] - self.a[0], self.b[1] - self.a[1])


@dataclass
class Scene:
    id: str
    walls: list
    floor_color: tuple = (0.35, 0.33, 0.30)
    ceiling_color: tuple = (0.85, 0.85, 0.85)
    wall_height: float = DEFAULT_WALL_HEIGHT
    version: int = 1
    navigable_hint: list | None = field(default=None, compare=False)
    warnings: tuple = field(default=(), compare=False)

    def segment_array(self) -> np.ndarray:
        if not self.walls:
            return np.empty((0, 4))
        return np.array([[w.a[0], w.a[1], w.b[0], w.b[1]] for w in self.walls], dtype=np.float64)

    def bounds(self):
        s = self.segment_array()
        if len(s) == 0:
            raise ValueError("scene has no walls")
        return (float(min(s[:, 0].min(), s[:, 2].min())), float(min(s[:, 1].min(), s[:, 3].min())),
                float(max(s[:, 0].max(), s[:, 2].max())), float(max(s[:, 1].max(), s[:, 3].max())))


@dataclass
class ObjectPayload:
    semantic_id: int
    segments: np.ndarray
    albedo: np.ndarray


@dataclass
class RegionPayload:
    name: str


@dataclass
class AgentPayload:
    name: str = "agent"


@dataclass
class SensorPayload:
    kind: str = "sensor"


class SceneNode:
    def __init__(self, name: str, transform: Transform2D = IDENTITY, payload=None):
        self.name = name
        self.transform = transform
        self.payload = payload
        self.parent = None
        self.children: list = []

    def add_child(self, node):
        if node.parent is not None:
            raise ValueError(f"node {node.name} already has a parent")
        p = self
        while p is not None:
            if p is node:
                raise ValueError("adding node would create a cycle")
            p = p.parent
        node.parent = self
        self.children.append(node)
        return node

    def detach(self):
        if self.parent is None:
            raise ValueError("cannot detach the root")
        self.parent.children.remove(self)
        self.parent = None
        return self

    def walk(self):
        yield self
        for ch in self.children:
            yield from ch.walk()

    def find(self, name: str):
        return next((n for n in self.walk() if n.name == name), None)

    def world_transform(self) -> Transform2D:
        chain, n = [], self
        while n is not None:
            chain.append(n.transform)
            n = n.parent
        w = IDENTITY
        for t in reversed(chain):
            w = w.compose(t)
        return w


class SceneGraph:
    def __init__(self, root: SceneNode, scene: Scene):
        self.root = root
        self.scene = scene

    def clone(self) -> "SceneGraph":
        def copy(node):
            twin = SceneNode(node.name, node.transform, node.payload)
            for ch in node.children:
                twin.add_child(copy(ch))
            return twin
        return SceneGraph(copy(self.root), self.scene)

    def object_nodes(self):
        return [n for n in self.root.walk() if _is_object(n.payload)]


def _is_object(payload) -> bool:
    return payload is not None and hasattr(payload, "segments") and hasattr(payload, "semantic_id")


def build_scene_graph(scene) -> SceneGraph:
    """root -> region -> one object node per semantic id, first-seen order
    (scene.py:327-346)."""
    root = SceneNode("root")
    region = root.add_child(SceneNode("region-0", payload=RegionPayload("region-0")))
    groups: dict = {}
    for w in scene.walls:
        groups.setdefault(w.semantic_id, []).append(w)
    for sid, ws in groups.items():
        segs = np.array([[w.a[0], w.a[1], w.b[0], w.b[1]] for w in ws], dtype=np.float64)
        region.add_child(SceneNode(f"object-{sid}", payload=ObjectPayload(
            semantic_id=sid, segments=segs, albedo=np.asarray(ws[0].albedo, dtype=np.float64))))
    return SceneGraph(root, scene)


def flatten_arrays(graph):
    """World-space (segments (n,4), semantic ids (n,) u16, albedo (n,3)) by a
    depth-first, child-order walk composing node transforms (scene.py:349-378)."""
    segs, sems, albs = [], [], []

    def visit(node, world):
        world = world.compose(node.transform)
        p = node.payload
        if _is_object(p):
            local = np.asarray(p.segments, dtype=np.float64)
            if world.is_identity:
                s = local.copy()
            else:
                s = np.concatenate([world.apply(local[:, 0:2]), world.apply(local[:, 2:4])], axis=1)
            segs.append(s)
            sems.append(np.full(len(local), p.semantic_id, dtype=np.uint16))
            albs.append(np.tile(np.asarray(p.albedo, dtype=np.float64), (len(local), 1)))
        for ch in node.children:
            visit(ch, world)

    visit(graph.root, IDENTITY)
    if not segs:
        return np.empty((0, 4)), np.empty(0, dtype=np.uint16), np.empty((0, 3))
    return np.concatenate(segs), np.concatenate(sems), np.concatenate(albs)
