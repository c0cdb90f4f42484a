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

from ._lib import Problem

_GOLDEN = 0x9E3779B97F4A7C15
_M64 = 0xFFFFFFFFFFFFFFFF


def _splitmix_stream(seed, count):
    """The first `count` SplitMix64 doubles of a stream (prng.hpp:14-25), vectorised."""
    k = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * np.uint64(_GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def generate_uniform_cube(n, seed):
    """geometry.cpp:42-52: point i = draws 3i..3i+2; unit charges."""
    if n < 2:
        raise ValueError("generate_uniform_cube: n must be >= 2")
    return _splitmix_stream(seed, 3 * n).reshape(n, 3), np.ones(n)


def generate_line(n, seed):
    if n < 2:
        raise ValueError("generate_line: n must be >= 2")
    xyz = np.zeros((n, 3))
    xyz[:, 0] = _splitmix_stream(seed, n)
    return xyz, np.ones(n)


def generate_uniform_sphere(n, seed):
    """i.i.d. uniform points on the unit sphere (BASELINE config 2): z = 2u-1,
    phi = 2 pi u'. No reference counterpart (fed to it as a point cloud)."""
    u = _splitmix_stream(seed, 2 * n).reshape(n, 2)
    z = 2.0 * u[:, 0] - 1.0
    phi = 2.0 * math.pi * u[:, 1]
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1), np.ones(n)


def generate_ellipsoids(n, count, seed):
    """Surface points on `count` seeded random ellipsoids, semi-axes U(0.05, 0.2),
    centres U[0,1]^3 (BASELINE config 5 surrogate). No reference counterpart."""
    u = _splitmix_stream(seed, 6 * count + 2 * n)
    cen = u[: 3 * count].reshape(count, 3)
    ax = 0.05 + 0.15 * u[3 * count: 6 * count].reshape(count, 3)
    v = u[6 * count:].reshape(n, 2)
    which = np.arange(n) % count
    z = 2.0 * v[:, 0] - 1.0
    phi = 2.0 * math.pi * v[:, 1]
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    unit = np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)
    return cen[which] + ax[which] * unit, np.ones(n)


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


def _fib_spheres(n, spheres, spacing, seed):
    """generate_sphere_surface (geometry.cpp:64-95) via libm-equivalent numpy."""
    side = int(round(spheres ** (1.0 / 3.0)))
    if side < 1 or side ** 3 != spheres:
        raise ValueError("generate_sphere_surface: spheres must be a perfect cube count")
    origin = -0.5 * spacing * (side - 1)
    golden = (1.0 + math.sqrt(5.0)) / 2.0
    phases = _splitmix_stream(seed, spheres)
    out = []
    remaining = n
    idx = 0
    for ix in range(side):
        for iy in range(side):
            for iz in range(side):
                left = spheres - idx
                m = (remaining + left - 1) // left
                remaining -= m
                c = (origin + spacing * ix, origin + spacing * iy, origin + spacing * iz)
                phase = phases[idx] * 2.0 * math.pi
                t = np.arange(m, dtype=np.float64)
                z = 1.0 - 2.0 * (t + 0.5) / m
                r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
                phi = 2.0 * math.pi * (t / golden) + phase
                out.append(np.stack([c[0] + r * np.cos(phi), c[1] + r * np.sin(phi), c[2] + z], 1))
                idx += 1
    return np.concatenate(out), np.ones(n)


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
    return _fib_spheres(cfg.n, cfg.spheres, cfg.spacing, cfg.seed)


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
