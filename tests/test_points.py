"""Product-side point generators (h2g_generate_points, host C++ in libh2g.so)
against the reference's generators (geometry.cpp:42-95): bit for bit.

The benched cloud (BASELINE configs[1]: N = 65,536 on the unit sphere, seed 42)
is pinned by the hash the unmodified reference wrote when it ran the whole
benched configuration (tests/golden/c2_65536_native.json, built with the
reference's own -march=native flags by tools/ref_pin_c2.py)."""
import json
import os

import numpy as np
import pytest

from conftest import has_ref
from oracle import cpu, ref

h2 = pytest.importorskip("paper_2208_10907_b200")
HERE = os.path.dirname(os.path.abspath(__file__))


def fbits(a):
    return ref.fnv64(np.ascontiguousarray(a, dtype=np.float64).view(np.int64).ravel())


def test_benched_sphere_cloud_matches_reference_run():
    with open(os.path.join(HERE, "golden", "c2_65536_native.json")) as f:
        g = json.load(f)
    xyz, q = h2.generate_points("sphere", 65536, 42)
    assert "%016x" % fbits(xyz) == g["points_fnv"]
    assert np.all(q == 1.0)


@pytest.mark.parametrize("geom,n,spheres", [("sphere", 65536, 1), ("sphere", 4096, 8),
                                            ("sphere", 100003, 27), ("cube", 3001, 1),
                                            ("line", 777, 1)])
def test_generators_bitwise_vs_c_oracle(geom, n, spheres):
    a, qa = h2.generate_points(geom, n, 42, spheres)
    b, qb = cpu.generate(geom, n, 42, spheres)
    assert np.array_equal(a.view(np.int64), b.view(np.int64))
    assert np.array_equal(qa, qb)


@pytest.mark.skipif(not has_ref(), reason="reference oracle not built")
@pytest.mark.parametrize("seed", [1, 7, 42, 12345])
def test_sphere_bitwise_vs_live_reference(seed):
    a, _ = h2.generate_points("sphere", 65536, seed)
    b, _ = ref.generate("sphere", 65536, seed)
    assert np.array_equal(a.view(np.int64), b.view(np.int64))


def test_pipeline_clouds_use_the_generators():
    from paper_2208_10907_b200.pipeline import RunConfig, make_cloud
    xyz, _ = make_cloud(RunConfig(n=4096, geometry="sphere", spheres=8, leaf_size=128))
    b, _ = cpu.generate("sphere", 4096, 42, 8)
    assert np.array_equal(xyz.view(np.int64), b.view(np.int64))


def test_baseline_extra_geometries():
    u, _ = h2.generate_points("uniform_sphere", 20000, 42)
    assert np.allclose(np.linalg.norm(u, axis=1), 1.0, atol=1e-14)
    assert abs(u[:, 2].mean()) < 0.02
    e, _ = h2.generate_points("ellipsoids", 50000, 42, 64)
    assert e.min() > -0.25 and e.max() < 1.25
    with pytest.raises(h2.H2GError, match="perfect cube"):
        h2.generate_points("sphere", 100, 42, 5)
    with pytest.raises(h2.H2GError, match="n must be"):
        h2.generate_points("cube", 1, 42)


def test_exp_table_matches_definition():
    """csrc/exp_table.cuh is the 2^(k/128) table re-derived from its definition."""
    import re
    import sys
    sys.path.insert(0, os.path.join(HERE, "..", "tools"))
    import gen_exp_table
    text = open(os.path.join(HERE, "..", "paper_2208_10907_b200", "csrc", "exp_table.cuh")).read()
    vals = [int(v, 16) for v in re.findall(r"0x([0-9a-f]{16})ull", text)]
    assert vals == gen_exp_table.table()


def test_exp_restatement_bitwise_vs_libm():
    """The device exp (common.cuh exp_glibc_core, run on the host) equals the
    libm exp the reference's Yukawa kernel calls (kernels.cpp:36,58), bit for
    bit, over the kernel's argument range and beyond."""
    import math
    from paper_2208_10907_b200 import _lib
    rng = np.random.default_rng(3)
    x = np.concatenate([-rng.uniform(0.0, 4.0, 400_000), rng.uniform(-600.0, 600.0, 50_000),
                        -rng.uniform(0.0, 1e-6, 20_000), -10.0 ** -rng.uniform(0, 20, 20_000),
                        np.array([0.0, -0.0, 1e-17, -1e-300, -2.5, -1.0, 511.9, -511.9])])
    y = _lib.exp_glibc_host(x)
    want = np.array([math.exp(v) for v in x])
    assert np.array_equal(y.view(np.int64), want.view(np.int64))
