#!/usr/bin/env python
"""Benchmark of the B200 H2-ULV hot path (build -> factorize -> solve).

Workload (BASELINE.json configs[1]): N = 65,536 points on the unit sphere (the
reference's Fibonacci-lattice generator, geometry.cpp:64-95, bit for bit),
Yukawa kernel exp(-r)/(r + 1e-3) (scale 1, so the diagonal is 1e3), leaf 256,
strong admissibility eta = 1, rank cap 100, tol 1e-6 (tol 1e-8 with cap 100
makes the reference abort with "basis does not absorb fill-in" at leaf 256;
measured). BASELINE assigns configs[2] and [3] to one GPU as
well; the reference's algorithm carries O(N^2) pieces, so this implementation
of it holds at most N = 131,072 on one B200 and configs[1] is
the largest BASELINE config it can run.

Mode: compressed QR (each member of a box's basis panel replaced by a
pivoted-Cholesky factor of its Gram matrix -- same range, same member masses --
then the blocked QR; the reference's pivoting/stopping rules on the compressed
panel; parity within tolerance, tests/test_qr_blocked.py) and the corrected
assembly (reference_compat = 0, pinned bit for bit against the corrected
reference, tests/test_corrected.py). The line's "exact_qr" field times the same
step with the reference's assembly and the bit-exact per-step QR (bitwise equal
to the unmodified reference at this size, tests/test_bench_parity.py);
"sampled_members" times it with sampled far-field basis members.

A step = one pass of the hot path from device-resident points: cluster tree
+ admissibility lists + near-field arena (Pipeline::build), fill-in
pre-computation + bases + level-parallel ULV factorization (Pipeline::factor)
and one right-hand-side solve. value = points / second of a step, timed with
CUDA events on the stream every kernel of the step is launched on.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
Under torchrun (N > 1) the N ranks factorize ONE problem together with the
multi-GPU level partition (Morton-contiguous box ranges per rank, the
partitioned basis stage all-gathers its outputs over NCCL; strong scaling,
value = N_points / max-over-ranks time); --replicas instead gives each rank
its own problem (seed 42 + rank, weak scaling, no collective). The timed
region is bracketed by a barrier + synchronize.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

WORKLOAD = dict(workload="c2_sphere_yukawa", n=65536, geometry="sphere(fibonacci,1)",
                kernel="yukawa", alpha_m=1.0, scale=1.0, reg=1e-3, leaf=256, eta=1.0, cap=100,
                tol=1e-6, structure="h2/nodep")
CPU_SAMPLE_N = 8192  # reference CPU sample: same workload family at N = 8192
METRIC = "h2ulv_points_per_sec"
FP64_DMMA_TFLOPS = 37.18  # profiles/r01_fp64_peak_probe.txt
UNIT = "points/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        # nvidia-smi polling contends with the driver calls of this path's
        # host-side launch preparation (~1,000 launches and a few syncs per
        # factorization): measured on one box, 35,925 points/s unsampled,
        # 26,706 at -lms 500, 35,698 at -lms 2000. 2 s still samples every
        # timed region (>= 5 s at the default 3 steps). BENCH_CLOCK_MS overrides.
        self.interval_ms = int(os.environ.get("BENCH_CLOCK_MS", "2000"))
        self.gpu = gpu_index
        self.samples = []
        self.proc = None

    def start(self):
        if self.interval_ms <= 0:
            self.proc = None
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, ValueError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        smax = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for k, nm in enumerate(names):
                if s[5 + k].lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def splitmix_signed(n, seed):
    from paper_2208_10907_b200.pipeline import splitmix_signed as f
    return f(n, seed)


def make_points(n, seed):
    """The reference's unit-sphere cloud (geometry.cpp:64-95), bit for bit:
    h2g_generate_points (host C++, glibc cos/sin, the reference's contractions)."""
    from paper_2208_10907_b200 import generate_points
    return generate_points("sphere", n, seed)


def cpu_reference(n, steps, warmup, threads):
    """Time the unmodified reference (oracle/_ref/libh2ref.so) on host cores."""
    from oracle import ref
    xyz, q = ref.generate("sphere", n, 42)
    cfg = ref.make_config(WORKLOAD["leaf"], tol=WORKLOAD["tol"], cap=WORKLOAD["cap"],
                          kernel="yukawa", alpha_m=1.0, reg=WORKLOAD["reg"], scale=WORKLOAD["scale"],
                          threads=threads)
    times = []
    for it in range(warmup + steps):
        r = ref.RefRun(xyz, q, cfg)
        t0 = time.perf_counter()
        r.build().factor()
        b = ref.splitmix_signed(n, 7)
        r.solve(b)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
        del r
    return times


def full_config_reference_run():
    """The unmodified reference's one-off run of the whole benched config
    (tools/ref_pin_c2.py; development container, not this host)."""
    path = os.path.join(HERE, "tests", "golden", "c2_65536_native.json")
    try:
        with open(path) as f:
            g = json.load(f)
    except (OSError, ValueError):
        return None
    t = g["wall_build_s"] + g["wall_factor_s"] + g["wall_solve_s"]
    return {"n": g["n"], "value": g["n"] / t, "unit": UNIT, "seconds": t, "cores": g["threads"],
            "where": "development container (8-core Xeon, 62 GB), -march=native build, peak RSS "
                     f"{g['peak_rss_gb']:.0f} GB", "source": "tests/golden/c2_65536_native.json"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    steps = max(1, args.steps)
    times = cpu_reference(CPU_SAMPLE_N, steps, args.warmup, threads)
    t = sum(times) / len(times)
    value = CPU_SAMPLE_N / t
    sample = (f"reference build+factor+solve of N={CPU_SAMPLE_N} (same sphere/Yukawa/leaf 256/"
              f"cap 100/tol 1e-6 family); the full N=65,536 config was run once: see full_config_measured")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": dict(WORKLOAD, n=CPU_SAMPLE_N, sample_of="c2_sphere_yukawa"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample, "full_config_measured": full_config_reference_run()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def load_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(HERE, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def run_b200_arm(args):
    import torch
    import paper_2208_10907_b200 as h2

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.n or WORKLOAD["n"]
    leaf = WORKLOAD["leaf"]
    partitioned = world > 1 and not args.replicas
    qr_mode = args.qr_mode
    comm = None
    partition_fallback = None
    if partitioned:
        # The partitioned path has only ever run over a host (gloo) transport here
        # (one GPU per run): create the NCCL communicator and push one small
        # partitioned factorization through it first; if that fails on any rank,
        # every rank falls back to independent replicas and the line says so.
        ok = 1
        try:
            uid = [h2.nccl_unique_id() if rank == 0 else None]
            torch.distributed.broadcast_object_list(uid, src=0)
            comm = h2.Comm.nccl(world, rank, uid[0])
            px, pq = make_points(8192, 42)
            pp = h2.Problem()
            pp.set_kernel("yukawa", WORKLOAD["alpha_m"], WORKLOAD["scale"], WORKLOAD["reg"])
            pp.set_options(tol=WORKLOAD["tol"], cap=WORKLOAD["cap"], eta=WORKLOAD["eta"], qr_mode=qr_mode,
                           reference_compat=args.compat)
            pp.set_comm(comm)
            pp.build(px, pq, leaf)
            pp.factor()
            pp.close()
        except Exception as e:  # noqa: BLE001 - any failure means "do not use this path"
            ok = 0
            partition_fallback = f"{type(e).__name__}: {e}"[:200]
        flag = torch.tensor([ok], device="cuda", dtype=torch.int32)
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if int(flag.item()) == 0:
            partitioned = False
            comm = None
            partition_fallback = partition_fallback or "the partitioned probe failed on another rank"
    seed = 42 if partitioned else 42 + rank
    xyz, q = make_points(n, seed)
    d_xyz = torch.from_numpy(np.ascontiguousarray(xyz)).cuda()
    d_q = torch.from_numpy(np.ascontiguousarray(q)).cuda()
    # b = SplitMix64(7).next_signed() as in the reference's runs (golden x comparable)
    b = splitmix_signed(n, 7 if partitioned else 7 + rank)
    d_b = torch.from_numpy(b).cuda()
    d_x = torch.empty_like(d_b)
    stream = torch.cuda.Stream()
    compat = args.compat

    def new_problem(mode=None, ref_compat=None):
        p = h2.Problem()
        p.set_stream(stream.cuda_stream)
        p.set_kernel("yukawa", WORKLOAD["alpha_m"], WORKLOAD["scale"], WORKLOAD["reg"])
        p.set_options(tol=WORKLOAD["tol"], cap=WORKLOAD["cap"], eta=WORKLOAD["eta"],
                      qr_mode=mode or qr_mode, reference_compat=compat if ref_compat is None else ref_compat)
        if comm is not None:
            p.set_comm(comm)
        return p

    def step(p):
        p.build_dev(d_xyz.data_ptr(), d_q.data_ptr(), n, leaf)
        p.factor()
        p.solve_dev(d_b.data_ptr(), d_x.data_ptr(), 1)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            p = new_problem()
            step(p)
            p.close()
        barrier()
        clocks = ClockSampler(local)
        clocks.start()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        # One problem object for the timed steps: every step rebuilds the tree,
        # factors and solves (h2g_build resets the factorization); creating and
        # destroying the handle is not part of the hot path. No per-kernel
        # profiling and no statistics reads inside the timed region.
        p = new_problem()
        launches0 = p.stats()["launches"]
        ev0.record(stream)
        for _ in range(args.steps):
            step(p)
        ev1.record(stream)
        barrier()
        clk = clocks.stop()
        launches = (p.stats()["launches"] - launches0) // max(1, args.steps)
        p.close()
    elapsed = ev0.elapsed_time(ev1) * 1e-3
    t_max = elapsed
    if world > 1:
        tt = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    points = n if partitioned else n * world
    value = points * args.steps / t_max

    # residual of the last timed solve through the matrix-free direct sum
    x = d_x.cpu().numpy()
    p = new_problem()
    p.build_dev(d_xyz.data_ptr(), d_q.data_ptr(), n, leaf)
    y = p.matvec(x)
    resid = float(np.linalg.norm(y - b) / np.linalg.norm(b))
    p.close()

    # Breakdown pass (separate from the timed region): per-kernel-family CUDA
    # events and per-phase device time of one more step.
    with torch.cuda.stream(stream):
        os.environ["H2G_PROF_DETAIL"] = "1"  # kernel records named family@phase (read at handle creation)
        p = new_problem()
        os.environ.pop("H2G_PROF_DETAIL", None)
        step(p)  # first step of a fresh handle (tree buffers, arena placement): not the steady state
        barrier()
        p.set_profile(True)
        p.reset_profile()
        step(p)
        barrier()
        sd = p.stats_dev()
        t_phase = {k: sd[k] for k in ("build", "factor", "solve")}
        kdetail = p.kernel_stats()
        p.close()
    # per family (all phases) and per phase (all families)
    kstats, by_phase = {}, {}
    for k, v in kdetail.items():
        fam, _, ph = k.partition("@")
        ph = ph.split("@")[0].split(":")[0] or "other"
        a = kstats.setdefault(fam, {"ms": 0.0, "flops": 0.0, "bytes": 0.0, "launches": 0})
        for f in ("ms", "flops", "bytes", "launches"):
            a[f] += v[f]
        by_phase.setdefault(ph, {})[fam] = v

    # e2e through the public C-ABI with host buffers (H2D/D2H inside the region).
    # Like the device-timed steps, one handle serves every e2e step (creating it
    # allocates the arenas once; that is setup, not the hot path). Reported
    # statistic: the mean over the e2e steps (their total time / steps).
    pe = h2.Problem()
    pe.set_kernel("yukawa", WORKLOAD["alpha_m"], WORKLOAD["scale"], WORKLOAD["reg"])
    pe.set_options(tol=WORKLOAD["tol"], cap=WORKLOAD["cap"], eta=WORKLOAD["eta"], qr_mode=qr_mode,
                   reference_compat=compat)
    if comm is not None:
        pe.set_comm(comm)
    barrier()
    t0 = time.perf_counter()
    for it in range(args.e2e_steps):
        pe.build(xyz, q, leaf)
        pe.factor()
        xe = pe.solve(b)
    barrier()
    e2e_t = (time.perf_counter() - t0) / max(args.e2e_steps, 1)
    pe.close()
    # the host-buffer path must produce the device path's solution
    e2e_dx = float(np.linalg.norm(xe - x) / np.linalg.norm(x))
    if not e2e_dx <= 1e-12:
        raise SystemExit(f"e2e solution differs from the device-timed one: {e2e_dx:.3e}")
    if world > 1:
        tt = torch.tensor([e2e_t], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_t = float(tt.item())

    # the same step with the reference's own assembly and per-step QR rounding
    # (bit-exact with the unmodified reference; tests/test_bench_parity.py)
    exact = None
    if args.exact_steps > 0:
        times = []
        with torch.cuda.stream(stream):
            for _ in range(args.exact_steps):
                p = new_problem("exact", True)
                barrier()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step(p)
                e1.record(stream)
                barrier()
                times.append(e0.elapsed_time(e1) * 1e-3)
                p.close()
        te = max(times)
        if world > 1:
            tt = torch.tensor([te], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        exact = {"qr_mode": "exact", "reference_compat": True, "points_per_s": points / te,
                 "steps": len(times),
                 "note": "same workload, the reference's assembly and QR rounding (bit-exact with "
                         "the unmodified reference, tests/test_bench_parity.py); device time"}

    # Secondary figure: the same step with sampled far-field basis members
    # (h2g_set_sampling; the north star's "far-field samples"). The headline
    # keeps the reference's full members.
    sampled = None
    if args.sample_cols > 0 and args.sampled_steps > 0:
        with torch.cuda.stream(stream):
            p = new_problem()
            p.set_options(tol=WORKLOAD["tol"], cap=WORKLOAD["cap"], eta=WORKLOAD["eta"], qr_mode=qr_mode,
                          reference_compat=compat, sample_cols=args.sample_cols)
            step(p)  # warm-up
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.sampled_steps):
                step(p)
            e1.record(stream)
            barrier()
            ts = e0.elapsed_time(e1) * 1e-3 / args.sampled_steps
            xs = d_x.cpu().numpy()
            rs_ = float(np.linalg.norm(p.matvec(xs) - b) / np.linalg.norm(b))
            p.close()
        if world > 1:
            tt = torch.tensor([ts], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ts = float(tt.item())
        sampled = {"sample_cols": args.sample_cols, "points_per_s": points / ts, "ms_per_step": ts * 1e3,
                   "steps": args.sampled_steps, "solve_rel_residual": rs_,
                   "note": "far-field basis members wider than sample_cols replaced by a strided column "
                           "sample (tolerance parity, tests/test_qr_blocked.py); device time"}

    # dominant kernel family and its roofline
    import json as _json
    peaks = {}
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            peaks = _json.load(f)
    except (OSError, ValueError):
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    dom = max(kstats.items(), key=lambda kv: kv[1]["ms"]) if kstats else ("none", {})
    name, st = dom
    traffic = load_traffic().get({"exact": "qr_exact", "blocked": "qr", "compressed": "qr_compressed"}[qr_mode]
                                 if name == "qr" else name)
    avg_ms = st["ms"] / max(1, st["launches"]) if st else 0.0
    bytes_per_launch = st["bytes"] / max(1, st["launches"]) if st else 0.0
    flops_per_launch = st["flops"] / max(1, st["launches"]) if st else 0.0
    if name == "gemm":
        # DMMA-bound: FP64 tensor peak from our own probe (MEASURED_PEAKS.json has no FP64 figure)
        achieved = flops_per_launch / (avg_ms * 1e-3) / 1e12 if avg_ms else 0.0
        roofline = {"bound": "tensor", "kernel": name, "achieved": achieved, "peak": FP64_DMMA_TFLOPS,
                    "unit": "TFLOP/s", "frac": achieved / FP64_DMMA_TFLOPS,
                    "traffic": traffic.get("bytes_per_launch") if traffic else None,
                    "algorithmic_flops_per_launch": flops_per_launch, "avg_launch_ms": avg_ms,
                    "peak_source": "profiles/r01_fp64_peak_probe.txt (DMMA, measured on B200; MEASURED_PEAKS.json has no FP64 figure)",
                    "traffic_source": traffic.get("source") if traffic else None,
                    "share_of_step": st["ms"] * 1e-3 / max(1e-12, t_phase["build"] + t_phase["factor"] + t_phase["solve"]) if st else None}
    else:
        achieved = bytes_per_launch / (avg_ms * 1e-3) / 1e9 if avg_ms else 0.0
        roofline = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm_peak,
                    "unit": "GB/s", "frac": achieved / hbm_peak if hbm_peak else None,
                    "traffic": traffic.get("bytes_per_launch") if traffic else None,
                    "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                    "share_of_step": st["ms"] * 1e-3 / max(1e-12, t_phase["build"] + t_phase["factor"] + t_phase["solve"]) if st else None}

    # every kernel family against the roof that bounds it:
    # FP64 work (DMMA GEMMs, LU, pivoted Cholesky) against the measured FP64
    # peak, data movement (evaluation writes, copies, QR panel sweeps, solves)
    # against the measured HBM bandwidth
    fp64_families = {"gemm", "gram", "lu", "pchol", "trsm"}
    families = {}
    for k, v in kstats.items():
        base = k.split("@")[0]
        sec = v["ms"] * 1e-3
        if not sec:
            continue
        if base in fp64_families:
            a = v["flops"] / sec / 1e12
            families[k] = {"bound": "fp64", "achieved": a, "unit": "TFLOP/s", "peak": FP64_DMMA_TFLOPS,
                           "frac": a / FP64_DMMA_TFLOPS, "ms": v["ms"], "launches": v["launches"]}
        else:
            a = v["bytes"] / sec / 1e9
            families[k] = {"bound": "hbm", "achieved": a, "unit": "GB/s", "peak": hbm_peak,
                           "frac": a / hbm_peak, "ms": v["ms"], "launches": v["launches"]}
    roofline["families"] = families
    # every batched phase of the factorization against its roofs: the FP64 work of the
    # phase (GEMM, Gram, LU, pivoted Cholesky) against the FP64 peak over the time those
    # kernels take, its data movement (evaluation writes, copies, QR sweeps, solves)
    # against the HBM bandwidth over theirs
    phases = {}
    for ph, fams in by_phase.items():
        f_ms = sum(v["ms"] for k, v in fams.items() if k in fp64_families)
        f_fl = sum(v["flops"] for k, v in fams.items() if k in fp64_families)
        h_ms = sum(v["ms"] for k, v in fams.items() if k not in fp64_families)
        h_by = sum(v["bytes"] for k, v in fams.items() if k not in fp64_families)
        e = {"ms": f_ms + h_ms, "launches": int(sum(v["launches"] for v in fams.values()))}
        if f_ms:
            tf = f_fl / (f_ms * 1e-3) / 1e12
            e["fp64"] = {"ms": f_ms, "achieved": tf, "unit": "TFLOP/s", "frac": tf / FP64_DMMA_TFLOPS}
        if h_ms:
            gb = h_by / (h_ms * 1e-3) / 1e9
            e["hbm"] = {"ms": h_ms, "achieved": gb, "unit": "GB/s", "frac": gb / hbm_peak}
        e["bound"] = "fp64" if f_ms >= h_ms else "hbm"
        phases[ph] = e
    roofline["phases"] = phases

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        try:
            ts = cpu_reference(CPU_SAMPLE_N, 1, 0, os.cpu_count() or 1)
            cpu_baseline = {"value": CPU_SAMPLE_N / ts[0], "unit": UNIT, "cores": os.cpu_count(),
                            "kind": "reference",
                            "sample": f"unmodified reference (oracle/_ref) build+factor+solve, N={CPU_SAMPLE_N}, "
                                      f"same workload family, {ts[0]:.1f} s"}
        except Exception as e:  # reference library not built on this host
            cpu_baseline = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                            "sample": f"unavailable: {e}"}
        full = full_config_reference_run()
        if full:
            cpu_baseline["full_config_measured"] = full

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if partitioned else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Fibonacci-lattice sphere, seed 42" + ("" if partitioned else "+rank") + ")",
            "config": dict(WORKLOAD, n=n, qr_mode=qr_mode, reference_compat=compat,
                           rhs="SplitMix64(7).next_signed()",
                           parallelism=(f"box-partitioned x{world} (NCCL all-gather of stage outputs)" if partitioned
                                        else f"replica x{world}" + (f" (partitioned path unavailable: {partition_fallback})"
                                                                    if partition_fallback else "")),
                           l2="inputs larger than L2 (near-field arena and member panels are GBs)"),
            "phase_s_per_step": t_phase,
            "factor_points_per_s": n / t_phase["factor"],
            "phase_note": "phase_s_per_step from a separate profiled step (the second step of its handle) after the timed region",
            "solve_rel_residual": resid,
            "e2e": {"value": points / e2e_t, "unit": UNIT, "h2d_bytes_per_step": int(8 * (4 * n + n)),
                    "d2h_bytes_per_step": int(8 * n), "statistic": f"mean of {args.e2e_steps} steps",
                    "x_rel_diff_vs_device_path": e2e_dx},
            "gpu_launches": launches,
            "roofline": roofline,
            "kernels": {k: dict(v, avg_ms=v["ms"] / max(1, v["launches"])) for k, v in kstats.items()},
            "clocks": clk,
            "cpu_baseline": cpu_baseline,
            "exact_qr": exact,
            "sampled_members": sampled,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override N (testing only)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--qr-mode", default="compressed", choices=["compressed", "blocked", "exact"],
                    help="member-panel QR: compressed (members replaced by pivoted-Cholesky factors "
                         "of their Gram matrices, then blocked QR), blocked (32 reflectors per panel "
                         "update) -- both parity within tolerance -- or exact (the reference's "
                         "rounding, bit-exact)")
    ap.add_argument("--exact-steps", type=int, default=1,
                    help="extra device-timed steps in exact QR mode, reported beside the headline")
    ap.add_argument("--sample-cols", type=int, default=512,
                    help="column budget of the secondary sampled-member measurement (0: skip)")
    ap.add_argument("--sampled-steps", type=int, default=2)
    ap.add_argument("--compat", action="store_true",
                    help="the reference's h2/nodep assembly bit for bit, covered-coupling defect "
                         "included (default: the corrected assembly, reference_compat = 0)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent problem per rank instead of one partitioned problem")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_b200_arm(args)


if __name__ == "__main__":
    sys.exit(main())
