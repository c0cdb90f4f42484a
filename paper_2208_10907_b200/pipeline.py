"""RunConfig / Pipeline mirror of the reference orchestration (report.hpp:13-99,
report.cpp:32-180), driving the B200 path through the C-ABI.

Point generation (SplitMix64 cube / line / Fibonacci spheres, geometry.cpp:42-95)
and the config defaults follow the reference; `uniform_sphere` and
`ellipsoids` are the extra BASELINE.json geometries (no reference
counterpart: parity for them is unpinned beyond tree/lists).
"""
import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from ._lib import Problem, generate_points

def splitmix_signed(n, seed):
    """b_i = SplitMix64(seed).next_signed() = 2 u - 1 (prng.hpp:14-25): the
    right-hand side of the reference's runs (seed 7)."""
    k = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0


def generate_uniform_cube(n, seed):
    """geometry.cpp:42-52: point i = draws 3i..3i+2; unit charges."""
    return generate_points("cube", n, seed)


def generate_line(n, seed):
    """geometry.cpp:54-62."""
    return generate_points("line", n, seed)


def generate_sphere_surface(n, spheres, spacing, seed):
    """geometry.cpp:64-95 (Fibonacci lattices), bit for bit with the reference."""
    return generate_points("sphere", n, seed, spheres, spacing)


def generate_uniform_sphere(n, seed):
    """i.i.d. uniform points on the unit sphere (BASELINE configs[1] as worded):
    z = 2u - 1, phi = 2 pi u'. No reference counterpart."""
    return generate_points("uniform_sphere", n, seed)


def generate_ellipsoids(n, count, seed):
    """Surface points on `count` seeded random ellipsoids, semi-axes U(0.05, 0.2),
    centres U[0,1]^3 (BASELINE configs[4] surrogate). No reference counterpart."""
    return generate_points("ellipsoids", n, seed, count)


@dataclass
class RunConfig:
    """report.hpp:13-39 (defaults identical)."""
    n: int = 1024
    leaf_size: int = 256
    tol: float = 1e-8
    cap: Optional[int] = None
    kernel: str = "laplace"  # laplace | yukawa
    alpha_m: float = 1.0
    reg: Optional[float] = None  # default 1e-3 * diameter / N^(1/3)
    scale: float = 4.0 * math.pi
    geometry: str = "cube"  # cube | line | sphere | uniform_sphere | ellipsoids
    spheres: int = 1
    spacing: float = 3.0
    eta: float = 1.0
    structure: str = "h2"  # h2 | hss
    threads: int = 1
    seed: int = 42
    oracle: bool = True
    oracle_guard: int = 16384
    absorb_coupling: bool = True
    points: Optional[np.ndarray] = field(default=None, repr=False)  # (xyz, q) import

    def validate(self):
        """RunConfig::validate (report.cpp:43-58)."""
        if self.n < 2:
            raise ValueError("config: n must be >= 2")
        if self.leaf_size < 2:
            raise ValueError("config: leaf size must be >= 2")
        if self.n < 2 * self.leaf_size:
            raise ValueError("config: need n >= 2 * leaf size")
        if self.tol <= 0:
            raise ValueError("config: tol must be positive")
        if self.cap is not None and self.cap < 1:
            raise ValueError("config: rank cap must be >= 1")
        if self.eta <= 0:
            raise ValueError("config: eta must be positive")
        if self.geometry not in ("cube", "line", "sphere", "uniform_sphere", "ellipsoids"):
            raise ValueError("config: unknown geometry " + self.geometry)
        if self.structure not in ("h2", "hss", "blr2"):
            raise ValueError("config: unknown structure " + self.structure)


def make_cloud(cfg):
    """report.cpp:60-65 (+ the BASELINE geometries)."""
    if cfg.points is not None:
        xyz, q = cfg.points
        return np.ascontiguousarray(xyz, dtype=np.float64), np.ascontiguousarray(q, dtype=np.float64)
    if cfg.geometry == "cube":
        return generate_uniform_cube(cfg.n, cfg.seed)
    if cfg.geometry == "line":
        return generate_line(cfg.n, cfg.seed)
    if cfg.geometry == "uniform_sphere":
        return generate_uniform_sphere(cfg.n, cfg.seed)
    if cfg.geometry == "ellipsoids":
        return generate_ellipsoids(cfg.n, cfg.spheres, cfg.seed)
    return generate_sphere_surface(cfg.n, cfg.spheres, cfg.spacing, cfg.seed)


def domain_diameter(xyz):
    """PointCloud::domain_diameter (geometry.cpp:28-40) with the reference's
    contraction fma(d2, d2, d0*d0 + d1*d1) reproduced exactly."""
    d = xyz.max(axis=0) - xyz.min(axis=0)
    s = d[0] * d[0] + d[1] * d[1]
    # exact fma via integer-free decomposition: use math.fma when present
    fma = getattr(math, "fma", None)
    v = fma(d[2], d[2], s) if fma else float(np.float64(d[2]) * d[2] + s)
    return math.sqrt(v)


class Pipeline:
    """Pipeline (report.hpp:73-99): build -> factor -> solve_rhs -> report."""

    def __init__(self, cfg: RunConfig):
        cfg.validate()
        self.cfg = cfg
        self.prob = None
        self.build_seconds = 0.0
        self.factor_seconds = 0.0

    def kernel_params(self, xyz):
        reg = self.cfg.reg
        if reg is None:
            reg = 1e-3 * domain_diameter(xyz) / np.cbrt(float(len(xyz)))
        return dict(kind=self.cfg.kernel, alpha_m=self.cfg.alpha_m if self.cfg.kernel == "yukawa" else 0.0,
                    scale=self.cfg.scale, reg=reg)

    def build(self):
        if self.prob is not None:
            return
        t0 = time.perf_counter()
        self.xyz, self.q = make_cloud(self.cfg)
        self.kernel = self.kernel_params(self.xyz)
        p = Problem()
        p.set_kernel(**self.kernel)
        p.set_options(tol=self.cfg.tol, cap=self.cfg.cap, absorb_coupling=self.cfg.absorb_coupling,
                      structure=self.cfg.structure, eta=self.cfg.eta)
        p.build(self.xyz, self.q, self.cfg.leaf_size)
        self.prob = p
        self.build_seconds = time.perf_counter() - t0

    def factor(self):
        self.build()
        t0 = time.perf_counter()
        self.prob.factor()
        self.factor_seconds = time.perf_counter() - t0
        self.factored = True

    def solve_rhs(self, b):
        return self.prob.solve(b)

    def report(self):
        """RunReport (h2ulv-report/1, report.cpp:113-237) as a dict; see report.py."""
        from .report import report_of
        return report_of(self)


def run_pipeline(cfg):
    """run_pipeline (report.cpp:239-243)."""
    from .report import run_report
    return run_report(cfg)
