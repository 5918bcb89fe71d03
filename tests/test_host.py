"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
the correctly rounded host math, synthetic scenes, sharding."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    src = open(os.path.join(ROOT, "include", "navsim_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nv_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    from paper_1904_01201_b200 import _native
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/navsim_b200.h but not exported"
        assert s in _native.SIGNATURES, f"{s} has no ctypes signature"


def test_no_gpu_means_loud_failure():
    import torch
    from paper_1904_01201_b200 import _native
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeUnavailable):
        _native.Context(0)


def test_host_sincos_correctly_rounded_vs_glibc():
    """exact_math.cuh (compiled into the .so host side) vs glibc: equal in the
    vast majority of cases and never more than 1 ulp apart (glibc itself is
    not correctly rounded in ~0.1% of cases)."""
    from paper_1904_01201_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(1)
    xs = np.concatenate([rng.uniform(-math.pi, math.pi, 20000),
                         [0.0, -0.0, math.pi, -math.pi, math.pi / 2, 1e-300]])
    s, c = ctypes.c_double(), ctypes.c_double()
    mism = 0
    for x in xs:
        lib.nv_host_sincos(float(x), ctypes.byref(s), ctypes.byref(c))
        for got, ref in ((s.value, math.sin(x)), (c.value, math.cos(x))):
            if got != ref:
                mism += 1
                assert abs(got - ref) <= math.ulp(ref), (x, got, ref)
    assert mism <= 0.01 * 2 * len(xs)


def test_host_sincos_matches_mpmath():
    mpmath = pytest.importorskip("mpmath")
    from paper_1904_01201_b200 import _native
    lib = _native.load()
    mpmath.mp.prec = 200
    rng = np.random.default_rng(2)
    s, c = ctypes.c_double(), ctypes.c_double()
    # random headings, the table-reduction breakpoints j/64 and the midpoints
    # between them (largest |t|), quadrant boundaries k pi/2, tiny and large
    xs = np.concatenate([rng.uniform(-math.pi, math.pi, 4000),
                         [j / 64 for j in range(-60, 61)], [(j + 0.5) / 64 for j in range(-60, 61)],
                         [k * math.pi / 2 for k in range(-4, 5)],
                         [math.nextafter(k * math.pi / 2, 9) for k in range(-4, 5)],
                         rng.uniform(-1e-3, 1e-3, 200), rng.uniform(-100.0, 100.0, 300)])
    for x in xs:
        lib.nv_host_sincos(float(x), ctypes.byref(s), ctypes.byref(c))
        assert s.value == float(mpmath.sin(mpmath.mpf(float(x)))), x
        assert c.value == float(mpmath.cos(mpmath.mpf(float(x)))), x
    for _ in range(300):
        a, b = rng.uniform(-0.3, 0.3, 2)
        h = lib.nv_host_hypot(float(a), float(b))
        assert h == float(mpmath.sqrt(mpmath.mpf(float(a)) ** 2 + mpmath.mpf(float(b)) ** 2))


def test_synthetic_scene_sizes():
    from paper_1904_01201_b200 import synth
    assert synth.config_scene("C1").n_triangles == 2000
    c2 = synth.config_scene("C2")
    assert 19_000 <= c2.n_triangles <= 21_000
    assert int(c2.semantic_ids.min()) >= 1 and int(c2.semantic_ids.max()) <= 65000


def test_sample_poses_clear_of_walls(oracle_mod):
    from paper_1904_01201_b200 import synth
    sc = synth.config_scene("C2")
    osc = oracle_mod.OracleScene(sc.segments, sc.semantic_ids, sc.albedo)
    poses = synth.sample_poses(sc, 64, seed=3)
    for x, y, h in poses:
        assert osc.clearance((x, y)) >= 0.1
        assert -math.pi < h <= math.pi
    # per-env streams: a prefix of a bigger draw is identical (sharding-invariant)
    assert np.array_equal(synth.sample_poses(sc, 8, seed=3), poses[:8])


def test_env_shards_partition():
    from paper_1904_01201_b200.dist import EnvShard
    for n, w in ((8192, 8), (1000, 3), (5, 8)):
        shards = [EnvShard(n, w, r) for r in range(w)]
        assert shards[0].lo == 0 and shards[-1].hi == n
        for a, b in zip(shards, shards[1:]):
            assert a.hi == b.lo
        assert sum(s.n_local for s in shards) == n


def test_chunked_crc32_matches_zlib():
    """The device PNG encoder's CRC-32 (per-chunk raw CRCs shifted by
    x^(8 * bytes after) mod P, then XOR-combined) equals zlib.crc32; checked
    through the host restatement exported by the library."""
    import ctypes
    import zlib
    from paper_1904_01201_b200 import _native
    lib = _native.load()
    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 4096, 131333):
        b = rng.integers(0, 256, n).astype(np.uint8)
        for chunks in (1, 5, 256):
            got = lib.nv_host_crc32_chunked(b.ctypes.data_as(ctypes.c_void_p), n, chunks)
            assert got == zlib.crc32(b.tobytes())
