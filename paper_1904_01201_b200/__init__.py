"""navsim hot path, B200-native: batched 2.5D column-raycast rendering (RGB,
depth, semantic) and the swept-disc agent step, as sm_100a CUDA kernels
behind a C ABI (include/navsim_b200.h), with the reference's Python
Simulator / render / SegmentIndex API on top.

Reference: /root/reference/pkg/src/navsim (sim.py, sensors.py, geometry.py,
_kernels.py).  See DESIGN.md.
"""
from .batch import BatchSimulator, SimError
from .geometry import SegmentIndex, segment_normals, wrap_angle
from .scene import (Scene, SceneGraph, SceneNode, Transform2D, WallSegment, build_scene_graph,
                    flatten_arrays)
from .sensors import (SEM_CEILING, SEM_FLOOR, SEM_VOID, EpisodeFrame, Observations,
                      RenderGeometry, SensorConfig, SensorError, default_sensor_suite,
                      gps_compass, render)
from .sim import (Action, AgentConfig, AgentState, Simulator, StepResult, apply_forward,
                  apply_turn, create_simulator)

__version__ = "0.1.0"
