"""Parity at the BENCHED configuration (BASELINE configs[1]): N = 65,536 points
of the reference's unit sphere (seed 42), Yukawa exp(-r)/(r + 1e-3), leaf 256,
cap 100, tol 1e-6, b = SplitMix64(7).

The unmodified reference ran this whole configuration once in the development
container (tools/ref_pin_c2.py, 35 min on 8 cores, 40 GB): its ranks per
level, cutoff dims and the FNV of x are in tests/golden/c2_65536_native.json
(built with the reference's own -march=native flags; the -mavx2 -mfma build
gives the same x, c2_65536_avx2.json). The corrected reference
(oracle/_ref_fixed) ran it as well (c2_65536_fixed.json).

* exact QR mode, reference_compat: ranks, cutoff and x bit for bit with the
  unmodified reference (Yukawa through the glibc exp restatement);
* exact QR mode, corrected: bit for bit with the corrected reference;
* the bench's mode (compressed QR, corrected) at N = 65,536: the corrected
  reference is NOT a solver here (its own residual is 4.27: the nodep fill
  scheme itself, not the covered-coupling defect, stops converging between
  16,384 and 32,768 points on this workload). Parity is then
  structural (per-level ranks within 1 % of the reference's, same cutoff
  level) and the residual is no worse than the reference's;
* the bench's mode at N = 16,384, where the corrected algorithm IS a solver
  (5e-7): residual below 100 tol and x within 1e-4 of the exact mode's, which
  is bitwise the corrected reference's algorithm.
"""
import json
import os

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu
h2 = pytest.importorskip("paper_2208_10907_b200")
HERE = os.path.dirname(os.path.abspath(__file__))
N = 65536


def golden(tag):
    path = os.path.join(HERE, "golden", f"c2_{N}_{tag}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    with open(path) as f:
        return json.load(f)


def fbits(a):
    return ref.fnv64(np.ascontiguousarray(a, dtype=np.float64).view(np.int64).ravel())


@pytest.fixture(scope="module")
def cloud():
    xyz, q = h2.generate_points("sphere", N, 42)
    return xyz, q, ref.splitmix_signed(N, 7)


def run(cloud, qr_mode, compat):
    xyz, q, b = cloud
    p = h2.Problem()
    p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
    p.set_options(tol=1e-6, cap=100, qr_mode=qr_mode, reference_compat=compat)
    p.build(xyz, q, 256)
    p.factor()
    x = p.solve(b)
    r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    levels = [[int(l), rk.tolist()] for l, rk in p.factor_levels()]
    lvl, dims = p.cutoff()
    p.close()
    return dict(x=x, r=r, levels=levels, cutoff=(int(lvl), dims.tolist()))


def test_exact_compat_bitwise_vs_unmodified_reference(cloud):
    g = golden("native")
    assert "%016x" % fbits(cloud[0]) == g["points_fnv"]
    out = run(cloud, "exact", True)
    assert out["levels"] == g["levels"]
    assert out["cutoff"] == (g["cutoff_level"], g["cutoff_dims"])
    assert "%016x" % fbits(out["x"]) == g["x_fnv"]


def test_exact_corrected_bitwise_vs_corrected_reference(cloud):
    g = golden("fixed")
    out = run(cloud, "exact", False)
    assert out["levels"] == g["levels"]
    assert "%016x" % fbits(out["x"]) == g["x_fnv"]


def test_bench_mode_vs_corrected_reference(cloud):
    g = golden("fixed")
    xr = np.load(os.path.join(HERE, "golden", f"c2_{N}_fixed.npz"))["x"]
    out = run(cloud, "compressed", False)
    xyz, q, b = cloud
    p = h2.Problem()
    p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
    p.build(xyz, q, 256)
    r_ref = float(np.linalg.norm(p.matvec(xr) - b) / np.linalg.norm(b))  # == dense matvec, bitwise
    p.close()
    assert r_ref > 1.0, r_ref  # the reference algorithm's own regime at this N (4.27)
    assert out["r"] <= r_ref, (out["r"], r_ref)
    assert out["cutoff"][0] == g["cutoff_level"]
    assert [l for l, _ in out["levels"]] == [l for l, _ in g["levels"]]
    for (lvl, rk), (_, rg) in zip(out["levels"], g["levels"]):
        assert abs(sum(rk) - sum(rg)) <= 0.01 * sum(rg), (lvl, sum(rk), sum(rg))


def test_bench_mode_solver_regime_16384():
    """Where the corrected algorithm converges (N = 16,384 of the same
    workload), the bench's compressed mode is a solver to 100 tol and agrees
    with the exact mode (bitwise the corrected reference's algorithm)."""
    n = 16384
    xyz, q = h2.generate_points("sphere", n, 42)
    c = (xyz, q, ref.splitmix_signed(n, 7))
    ex = run(c, "exact", False)
    co = run(c, "compressed", False)
    assert ex["r"] < 1e-4 and co["r"] < 1e-4, (ex["r"], co["r"])
    assert np.linalg.norm(co["x"] - ex["x"]) / np.linalg.norm(ex["x"]) < 1e-4
