"""Blocked QR mode (h2g_options.qr_mode = 1, k_qrb.cu): reflectors applied to
the member panel 32 at a time (one read of the panel per step, one write per
block) instead of the reference's per-step read-modify-write. Same pivoting,
tie and stopping rules, different rounding, so parity with the reference is by
tolerance: the solve residual equals the reference's to 1e-6 relative
(Laplace; 5 % for Yukawa, whose kernel entries already differ by 1 ulp) and
the solution equals the exact mode's to 1e-4 relative. Blocked mode is
deterministic (no atomics) and partitions across ranks bit for bit."""
import numpy as np
import pytest

from oracle import cpu, ref

pytestmark = pytest.mark.gpu

h2 = pytest.importorskip("paper_2208_10907_b200")

E2E = ["cube512", "cube1024", "hss1024", "cube2048", "sphere2048_yukawa_cap100", "line1024",
       "spheres8_4096", "c1_cube4096", "sphere4096_yukawa_cap100_tol1e-6_leaf256"]


def solve_case(rec, mode):
    xyz, q = cpu.generate(rec["geometry"], rec["n"], 42, rec["spheres"])
    p = h2.Problem()
    kind = rec["kernel"]
    p.set_kernel(kind, 1.0 if kind == "yukawa" else 0.0, rec["scale"], rec["reg"])
    p.set_options(tol=rec["tol"], cap=rec["cap"], structure=rec["structure"], qr_mode=mode)
    p.build(xyz, q, rec["leaf"])
    p.factor()
    b = ref.splitmix_signed(rec["n"], 7)
    x = p.solve(b)
    r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
    p.close()
    return x, r


@pytest.mark.parametrize("name", E2E)
def test_blocked_residual_matches_reference(golden, name):
    rec = golden[0]["cases"][name]
    xb, rb = solve_case(rec, "blocked")
    xe, _ = solve_case(rec, "exact")
    r_ref = rec["residual"]
    if rec["structure"] == "hss" or r_ref < 1e-6:
        assert rb < 10 * max(r_ref, 1e-12), (rb, r_ref)  # both are solver-accurate
    elif rec["kernel"] == "laplace":
        assert abs(rb - r_ref) <= 1e-6 * r_ref, (rb, r_ref)
        # Different (smaller) ranks where the reference's mass downdates never
        # reach the threshold move x by up to ~1e-5 relative (6e-6 on C1).
        assert np.linalg.norm(xb - xe) <= 1e-4 * np.linalg.norm(xe)
    else:
        assert abs(rb - r_ref) <= 0.05 * r_ref, (rb, r_ref)


def test_blocked_is_deterministic(golden):
    rec = golden[0]["cases"]["c1_cube4096"]
    x1, _ = solve_case(rec, "blocked")
    x2, _ = solve_case(rec, "blocked")
    assert np.array_equal(x1.view(np.int64), x2.view(np.int64))


def test_qr_mode_validation():
    p = h2.Problem()
    with pytest.raises(KeyError):
        p.set_options(qr_mode="fast")
    p.close()


def test_blocked_matches_exact_on_bench_family():
    """The bench workload family (Fibonacci sphere, Yukawa, leaf 256, cap 100,
    tol 1e-6) at N = 16,384: blocked and exact QR give the same solve
    residual to 1e-6 relative and the same per-level rank sums."""
    n = 16384
    xyz, q = h2.generate_points("sphere", n, 42)
    b = np.random.default_rng(7).uniform(-1, 1, n)
    out = {}
    for mode in ("exact", "blocked"):
        p = h2.Problem()
        p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
        p.set_options(tol=1e-6, cap=100, qr_mode=mode)
        p.build(xyz, q, 256)
        p.factor()
        x = p.solve(b)
        r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
        out[mode] = (r, [int(rk.sum()) for _, rk in p.factor_levels()])
        p.close()
    (re, ke), (rb, kb) = out["exact"], out["blocked"]
    assert abs(rb - re) <= 1e-6 * re, (rb, re)
    assert all(abs(a - c) <= 0.01 * a for a, c in zip(ke, kb)), (ke, kb)


# ---- compressed mode (qr_mode = 2, k_pchol.cu) --------------------------------
# Members of width >= 48 are replaced by pivoted-Cholesky factors of their Gram
# matrices (same range, same member masses up to a dropped trace of
# max(64 eps, 0.01 member_tol^2) of each member's mass), then the blocked QR runs
# on the narrow panel. The pivots differ from the reference's, so parity is by
# tolerance: the solve residual matches the reference's to 1e-5 relative
# (Laplace) / 1e-4 (Yukawa) where the reference's own defect sets it, and stays
# solver-accurate where the reference is.

@pytest.mark.parametrize("name", E2E)
def test_compressed_residual_matches_reference(golden, name):
    rec = golden[0]["cases"][name]
    xc, rc = solve_case(rec, "compressed")
    xe, _ = solve_case(rec, "exact")
    r_ref = rec["residual"]
    if rec["structure"] == "hss" or r_ref < 1e-6:
        assert rc < max(100 * r_ref, 1e-9), (rc, r_ref)
    else:
        rtol = 1e-5 if rec["kernel"] == "laplace" else 1e-4
        assert abs(rc - r_ref) <= rtol * r_ref, (rc, r_ref)
        assert np.linalg.norm(xc - xe) <= 1e-4 * np.linalg.norm(xe)


def test_compressed_is_deterministic(golden):
    rec = golden[0]["cases"]["c1_cube4096"]
    x1, _ = solve_case(rec, "compressed")
    x2, _ = solve_case(rec, "compressed")
    assert np.array_equal(x1.view(np.int64), x2.view(np.int64))


def test_compressed_matches_exact_on_bench_family():
    """Bench workload family at N = 16,384: compressed and exact QR give the
    same solve residual to 1e-4 relative and per-level rank sums within 10 %."""
    n = 16384
    xyz, q = h2.generate_points("sphere", n, 42)
    b = np.random.default_rng(7).uniform(-1, 1, n)
    out = {}
    for mode in ("exact", "compressed"):
        p = h2.Problem()
        p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
        p.set_options(tol=1e-6, cap=100, qr_mode=mode)
        p.build(xyz, q, 256)
        p.factor()
        x = p.solve(b)
        r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
        out[mode] = (r, [int(rk.sum()) for _, rk in p.factor_levels()])
        p.close()
    (re, ke), (rc, kc) = out["exact"], out["compressed"]
    assert abs(rc - re) <= 1e-4 * re, (rc, re)
    assert all(abs(c - a) <= 0.1 * a for a, c in zip(ke, kc)), (ke, kc)


@pytest.mark.parametrize("tol", [1e-6, 1e-4])
def test_compressed_basis_keeps_member_stopping_rule(tol):
    """basis_from_members through the compressed mode: members wider than the
    compression threshold (numerically low-rank kernel blocks and one
    full-rank noise member) are replaced by pivoted-Cholesky factors of their
    Gram matrices. The resulting basis must still satisfy the reference's
    per-member rule ||(I - Qs Qs^T) M_i||_F <= member_tol ||M_i||_F
    (member_tol = tol / 2, linalg.cpp:276-297), with a rank within 10 % of the
    exact mode's and Q orthonormal."""
    rng = np.random.default_rng(11)
    dim = 200
    src = rng.uniform(0, 1, (dim, 3))
    members = []
    for w, shift in ((3000, 2.5), (700, 1.5), (64, 4.0), (30, 3.0)):
        tgt = rng.uniform(0, 1, (w, 3)) + np.array([shift, 0, 0])
        d = np.sqrt(((src[:, None, :] - tgt[None, :, :]) ** 2).sum(-1))
        members.append(1.0 / d)
    members.append(1e-3 * rng.standard_normal((dim, 100)))
    concat = np.hstack(members)
    offs = np.cumsum([0] + [m.shape[1] for m in members])
    sq_e, r_e = h2._lib.basis_from_members(concat, offs, tol)
    sq_c, r_c = h2._lib.basis_from_members(concat, offs, tol, qr_mode="compressed")
    assert np.allclose(sq_c.T @ sq_c, np.eye(dim), atol=1e-12)
    qs = sq_c[:, dim - r_c:]
    for mem in members:
        left = mem - qs @ (qs.T @ mem)
        assert np.linalg.norm(left) <= 0.5 * tol * np.linalg.norm(mem) * 1.01, (r_c, r_e)
    assert abs(r_c - r_e) <= max(2, 0.1 * r_e), (r_c, r_e)


@pytest.mark.parametrize("structure", ["hss", "blr2"])
def test_compressed_structure_variants(structure):
    """The compressed mode under the reference's other level-parallel
    structures (weak admissibility; BLR^2's flat top system): solver-accurate
    where the exact mode is, at tol 1e-6 on a 2,048-point cube."""
    n, leaf = 2048, 128
    xyz, q = cpu.generate("cube", n, 42)
    b = ref.splitmix_signed(n, 7)
    res = {}
    for mode in ("exact", "compressed"):
        p = h2.Problem()
        p.set_kernel("laplace", 0.0, 1.0, 1e-3)
        p.set_options(tol=1e-6, structure=structure, qr_mode=mode)
        p.build(xyz, q, leaf)
        p.factor()
        x = p.solve(b)
        res[mode] = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
        p.close()
    assert res["exact"] < 1e-4, res
    assert res["compressed"] < max(10 * res["exact"], 1e-8), res


@pytest.mark.gpu
def test_sampled_far_field_members_solver_regime():
    """h2g_set_sampling (far-field basis members replaced by a strided sample of
    their columns; the reference concatenates every column,
    compression.cpp:153-177, ulv.cpp:476-521): where the corrected algorithm is
    a solver (N = 16,384 of the bench workload, tol 1e-6) the sampled run stays
    one - residual below 100 tol, x within 1e-5 of the full-member run, per-level
    rank sums within 1 % - and the run is deterministic."""
    from oracle import ref
    n = 16384
    xyz, q = h2.generate_points("sphere", n, 42)
    b = ref.splitmix_signed(n, 7)

    def run(sample):
        p = h2.Problem()
        p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
        p.set_options(tol=1e-6, cap=100, qr_mode="compressed", reference_compat=False, sample_cols=sample)
        p.build(xyz, q, 256)
        p.factor()
        x = p.solve(b)
        r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
        ranks = [int(np.sum(rk)) for _, rk in p.factor_levels()]
        p.close()
        return x, r, ranks

    x0, r0, k0 = run(0)
    x1, r1, k1 = run(512)
    x2, r2, k2 = run(512)
    assert r0 < 1e-4 and r1 < 1e-4, (r0, r1)
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x0) < 1e-5
    assert len(k0) == len(k1)
    for a, c in zip(k0, k1):
        assert abs(a - c) <= 0.01 * a + 2, (k0, k1)
    assert np.array_equal(x1.view(np.int64), x2.view(np.int64))


def test_sampling_option_validation():
    p = h2.Problem()
    with pytest.raises(Exception):
        p.set_options(sample_cols=8)
    p.set_options(sample_cols=0)
    p.set_options(sample_cols=512)
    p.close()


def test_nested_transfer_column_members_match_evaluated_ones(monkeypatch):
    """Tolerance modes build the transfer stage's ancestor-partner column members
    from the finer level's members (Vs_c^T times the child's member; Vbig is
    nested) instead of evaluating A(I, c) Vbig_c again at every level
    (ulv.cpp:495-501). Against the evaluated members (H2G_EXACT_SOLVES=1, which
    also turns the other reassociations off) on a 7-level tree in the solver
    regime: fewer kernel evaluations, the same ranks, x equal to 1e-9."""
    from oracle import ref
    n, leaf = 16384, 128
    xyz, q = h2.generate_points("sphere", n, 42)
    b = ref.splitmix_signed(n, 7)

    def run():
        p = h2.Problem()
        p.set_kernel("yukawa", 1.0, 1.0, 1e-3)
        # leaf 128 with cap 100 trips the reference's fill-absorption abort at level 4
        # (ulv.cpp:140-147) in either variant; it is disabled here, the residual is the gate
        p.set_options(tol=1e-6, cap=100, qr_mode="compressed", reference_compat=False,
                      abort_residual_factor=1e30)
        p.build(xyz, q, leaf)
        p.factor()
        x = p.solve(b)
        r = float(np.linalg.norm(p.matvec(x) - b) / np.linalg.norm(b))
        out = (x, r, p.stats()["kernel_evals"], [rk.tolist() for _, rk in p.factor_levels()])
        p.close()
        return out

    monkeypatch.delenv("H2G_EXACT_SOLVES", raising=False)
    xn, rn, en, kn = run()
    monkeypatch.setenv("H2G_EXACT_SOLVES", "1")
    xe, re_, ee, ke = run()
    assert rn < 1e-4 and re_ < 1e-4, (rn, re_)
    assert en < ee, (en, ee)
    assert kn == ke
    assert np.linalg.norm(xn - xe) / np.linalg.norm(xe) < 1e-9
