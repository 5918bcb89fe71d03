"""Codec fixtures from the UNMODIFIED reference (sensors.py:211-246).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_golden_codec.py

Renders a few frames with the reference, encodes them with its depth_to_png /
rgb_to_png / semantic_to_png, and stores the f64 inputs plus the samples the
reference's PNGs decode to (PIL) -- the device encoder must decode to the
same samples from the same inputs.
"""
import io
import os

import numpy as np
from PIL import Image

from navsim import sensors as rs
from navsim.scene import Scene, WallSegment, build_scene_graph, flatten_arrays

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    walls = [((0.0, 0.0), (10.0, 0.0), 1, (0.6, 0.5, 0.4)), ((10.0, 0.0), (10.0, 10.0), 2, (0.5, 0.6, 0.4)),
             ((10.0, 10.0), (0.0, 10.0), 3, (0.4, 0.5, 0.6)), ((0.0, 10.0), (0.0, 0.0), 4, (0.6, 0.4, 0.5)),
             ((3.0, 3.0), (5.0, 4.0), 7, (0.9, 0.2, 0.1))]
    sc = Scene(id="codec", walls=[WallSegment(a=a, b=b, semantic_id=s, albedo=c) for a, b, s, c in walls],
               floor_color=(0.3, 0.3, 0.3), ceiling_color=(0.9, 0.9, 0.9))
    segs, sem, alb = flatten_arrays(build_scene_graph(sc))
    geom = rs.RenderGeometry(segs, sem, alb, sc.wall_height, sc.floor_color, sc.ceiling_color)
    W, H = 64, 48
    suite = (rs.SensorConfig("rgb", W, H), rs.SensorConfig("depth", W, H),
             rs.SensorConfig("semantic", W, H))
    out = {"max_range": np.float64(10.0)}
    dep, rgb, sm, qd, qr, qs = [], [], [], [], [], []
    for (x, y, h) in [(7.0, 5.0, 0.0), (2.0, 2.0, 0.8), (5.0, 8.0, -2.0)]:
        o = rs.render(geom, (x, y), h, 1.5, suite)
        dep.append(o.depth); rgb.append(o.rgb); sm.append(o.semantic)
        qd.append(np.asarray(Image.open(io.BytesIO(rs.depth_to_png(o.depth, 10.0))), dtype=np.uint16))
        qr.append(np.asarray(Image.open(io.BytesIO(rs.rgb_to_png(o.rgb))).convert("RGB"), dtype=np.uint8))
        qs.append(np.asarray(Image.open(io.BytesIO(rs.semantic_to_png(o.semantic))), dtype=np.uint16))
    out.update(depth=np.asarray(dep), rgb=np.asarray(rgb), semantic=np.asarray(sm),
               q_depth=np.asarray(qd), q_rgb=np.asarray(qr), q_semantic=np.asarray(qs))
    np.savez_compressed(os.path.join(HERE, "golden_codec.npz"), **out)
    print("codec fixture written")


if __name__ == "__main__":
    main()
