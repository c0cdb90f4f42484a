"""CPU checks of bench.py's contract with BASELINE.json (no GPU work)."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_workload_is_baseline_config_1():
    sys.path.insert(0, ROOT)
    import bench
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        cfg = json.load(f)["configs"][1]
    w = bench.WORKLOAD
    assert "N=65,536" in cfg and w["n"] == 65536
    assert "Yukawa" in cfg and w["kernel"] == "yukawa"
    assert "leaf 256" in cfg and w["leaf"] == 256
    assert "max rank 100" in cfg and w["cap"] == 100
    assert "unit sphere" in cfg and w["geometry"].startswith("sphere")
    # diagonal 1e3: scale * (0 + reg) = 1e-3
    assert w["scale"] * w["reg"] == 1e-3
    assert bench.METRIC == "h2ulv_points_per_sec" and bench.UNIT == "points/s"


def test_bench_cli_flags():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl"):
        assert flag in out.stdout
