"""Device PNG codecs (nv_png_encode) against the reference's
depth_to_png / rgb_to_png / semantic_to_png (tests/golden/golden_codec.npz):
the device PNGs of the reference's own f64 frames decode (PIL) to exactly the
samples the reference's PNGs decode to; chunk CRCs and the zlib Adler-32
verify; batched encoding of device frames (f32 depth, u8 rgb, u16 semantic)
round-trips within the reference's codec tolerances."""
import io
import os
import struct
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def nb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1904_01201_b200 as nb
    from paper_1904_01201_b200 import _native
    _native.load()
    return nb


def check_png(data: bytes):
    """Chunk CRCs and the zlib stream (Adler-32) verify; returns raw scanlines."""
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    pos, idat = 8, b""
    while pos < len(data):
        ln, typ = struct.unpack(">I4s", data[pos:pos + 8])
        body = data[pos + 8:pos + 8 + ln]
        crc, = struct.unpack(">I", data[pos + 8 + ln:pos + 12 + ln])
        assert crc == zlib.crc32(typ + body), typ
        if typ == b"IDAT":
            idat += body
        pos += 12 + ln
    return zlib.decompress(idat)  # checks the Adler-32


def test_codecs_match_reference(nb):
    from PIL import Image
    from paper_1904_01201_b200 import sensors
    g = dict(np.load(os.path.join(HERE, "golden", "golden_codec.npz")))
    mr = float(g["max_range"])
    for k in range(g["depth"].shape[0]):
        d = sensors.depth_to_png(g["depth"][k], mr)
        check_png(d)
        assert np.array_equal(np.asarray(Image.open(io.BytesIO(d)), dtype=np.uint16), g["q_depth"][k])
        r = sensors.rgb_to_png(g["rgb"][k])
        check_png(r)
        assert np.array_equal(np.asarray(Image.open(io.BytesIO(r)).convert("RGB")), g["q_rgb"][k])
        s = sensors.semantic_to_png(g["semantic"][k])
        check_png(s)
        assert np.array_equal(sensors.png_to_semantic(s), g["q_semantic"][k])
        assert np.array_equal(sensors.png_to_semantic(s), g["semantic"][k])


def test_batched_device_frames_roundtrip(nb):
    from paper_1904_01201_b200 import sensors, synth
    sc = synth.config_scene("C2")
    W, H, n = 128, 96, 12
    suite = (nb.SensorConfig("rgb", W, H), nb.SensorConfig("depth", W, H),
             nb.SensorConfig("semantic", W, H))
    sim = nb.BatchSimulator(sc.segments, sc.semantic_ids, sc.albedo, n, sensor_configs=suite)
    poses = synth.sample_poses(sc, n, seed=8)
    sim.reset(poses[:, :2], poses[:, 2])
    obs = sim.render()
    torch.cuda.synchronize()
    for kind, key in ((sensors.PNG_DEPTH, "depth"), (sensors.PNG_RGB, "rgb"),
                      (sensors.PNG_SEMANTIC, "semantic")):
        out, size = sensors.encode_frames(obs[key], kind, 10.0)
        torch.cuda.synchronize()
        host = out.cpu().numpy()
        src = obs[key].cpu().numpy()
        for e in range(n):
            data = host[e].tobytes()
            raw = check_png(data)
            assert len(raw) == H * (1 + W * (3 if kind == sensors.PNG_RGB else 2))
            if kind == sensors.PNG_DEPTH:
                dec = sensors.png_to_depth(data, 10.0)
                assert np.max(np.abs(dec - src[e].astype(np.float64))) <= 10.0 / 65535 + 1e-6
            elif kind == sensors.PNG_RGB:
                assert np.array_equal(np.round(sensors.png_to_rgb(data) * 255).astype(np.uint8), src[e])
            else:
                assert np.array_equal(sensors.png_to_semantic(data), src[e])
