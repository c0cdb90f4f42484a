"""Explicit ground truth of the level-parallel ULV, level by level, on the GPU
(torch FP64): the generalisation of the reference's dev_diag3 (explicit
A~ = (I - Z) A at the leaf) to every factorized level, at sizes the CPU
cannot hold densely.

For each factorized level: Z from the level's near blocks, A~ = (I - Z) M,
S = [U]^T A~ [V] with the path's own bases, the decoupling of every box's
redundant rows/columns, the exact Schur complement on the skeletons, and its
comparison with the path's merged system of the next level
(h2g_level_block), broken down by child pair kind (near / far at this level).

  python tools/explicit_ulv_gpu.py N [leaf] [tol] [cap] [compat] [qr_mode]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2208_10907_b200 as h2  # noqa: E402

dev = torch.device("cuda")


def main():
    n = int(sys.argv[1])
    leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    tol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
    cap = int(sys.argv[4]) if len(sys.argv) > 4 else 100
    compat = (sys.argv[5] == "1") if len(sys.argv) > 5 else False
    mode = sys.argv[6] if len(sys.argv) > 6 else "exact"
    geom = os.environ.get("GEOM", "sphere")
    kern = os.environ.get("KERN", "yukawa")
    xyz, q = h2.generate_points(geom, n, 42)
    p = h2.Problem()
    p.set_kernel(kern, 1.0 if kern == "yukawa" else 0.0, 1.0, 1e-3)
    p.set_options(tol=tol, cap=cap or None, qr_mode=mode, reference_compat=compat)
    p.build(xyz, q, leaf)
    p.factor()
    L = p.levels
    be, _ = p.nodes()
    X, Q = p.reordered()
    Xt = torch.tensor(X, device=dev)
    Qt = torch.tensor(Q, device=dev)
    M = torch.empty((n, n), dtype=torch.float64, device=dev)
    for i0 in range(0, n, 2048):
        # exact differences (torch.cdist's matmul form loses digits for close points)
        d = torch.sqrt(((Xt[i0:i0 + 2048, None, :] - Xt[None, :, :]) ** 2).sum(-1))
        K = (torch.exp(-d) if kern == "yukawa" else torch.ones_like(d)) / (d + 1e-3)
        M[i0:i0 + 2048] = K * Qt[None, :]
        del d, K
    flv = p.factor_levels()
    print(f"N={n} leaf={leaf} tol={tol} cap={cap} compat={compat} mode={mode} L={L} "
          f"factor levels {[l for l, _ in flv]}", flush=True)

    def rng(l, i):
        k = (1 << l) - 1 + i
        return int(be[k, 0]), int(be[k, 1])

    dims = [rng(L, i)[1] - rng(L, i)[0] for i in range(1 << L)]
    for li, (lvl, ranks) in enumerate(flv):
        m = 1 << lvl
        off = np.concatenate([[0], np.cumsum(dims)]).astype(np.int64)
        nptr, nidx = p.lists(lvl, 0)
        fptr, fidx = p.lists(lvl, 1)
        near = [set(nidx[nptr[k]:nptr[k + 1]].tolist()) for k in range(m)]
        far = [set(fidx[fptr[k]:fptr[k + 1]].tolist()) for k in range(m)]
        sl = lambda k: slice(int(off[k]), int(off[k + 1]))  # noqa: E731
        # A~ = M - Z M, Z_kp = M_kp M_pp^-1 (p near k, p != k)
        At = M.clone()
        for k in range(m):
            for pp in near[k]:
                if pp == k:
                    continue
                Zkp = torch.linalg.solve(M[sl(pp), sl(pp)].T, M[sl(k), sl(pp)].T).T
                At[sl(k)] -= Zkp @ M[sl(pp)]
        # S = U^T A~ V (block diagonal bases)
        for k in range(m):
            U, _ = p.basis(lvl, k, 0)
            At[sl(k)] = torch.tensor(U, device=dev).T @ At[sl(k)]
        for k in range(m):
            V, _ = p.basis(lvl, k, 1)
            At[:, sl(k)] = At[:, sl(k)] @ torch.tensor(V, device=dev)
        S = At
        rk = [int(r) for r in ranks]
        red = torch.zeros(S.shape[0], dtype=torch.bool, device=dev)
        for k in range(m):
            red[int(off[k]):int(off[k + 1]) - rk[k]] = True
        nS = float(torch.linalg.norm(S))
        wr = wc = 0.0
        worst_pairs = []
        for k in range(m):
            rows = slice(int(off[k]), int(off[k + 1]) - rk[k])
            if rows.stop <= rows.start:
                continue
            for i in range(m):
                if i == k:
                    continue
                e_row = float(torch.linalg.norm(S[rows, sl(i)]))
                e_col = float(torch.linalg.norm(S[sl(i), rows]))
                blk = float(torch.linalg.norm(S[sl(k), sl(i)])) + 1e-300
                wr, wc = max(wr, e_row), max(wc, e_col)
                kind = "near" if i in near[k] else ("far" if i in far[k] else "covered")
                worst_pairs.append((max(e_row, e_col) / blk, k, i, kind, e_row, e_col))
        worst_pairs.sort(reverse=True)
        print(f"level {lvl}: |S| {nS:.3e}  worst row-decoupling {wr:.3e}  col-decoupling {wc:.3e}", flush=True)
        for rel, k, i, kind, er, ec in worst_pairs[:4]:
            print(f"   box {k} vs {i} ({kind}): row {er:.2e} col {ec:.2e} (rel to block {rel:.2e})")
        s = ~red
        Srr = S[red][:, red]
        Mn = S[s][:, s] - S[s][:, red] @ torch.linalg.solve(Srr, S[red][:, s])
        del S, At, Srr
        dims = [rk[2 * I] + rk[2 * I + 1] for I in range(m // 2)]
        M = Mn
        if li + 1 >= len(flv):
            break
        # the path's merged system of the next level vs the exact Schur complement
        off2 = np.concatenate([[0], np.cumsum(dims)]).astype(np.int64)
        nptr2, nidx2 = p.lists(lvl - 1, 0)
        worst = []
        for I in range(m // 2):
            for J in nidx2[nptr2[I]:nptr2[I + 1]].tolist():
                B = torch.tensor(p.level_block(li + 1, I, J), device=dev)
                E = M[int(off2[I]):int(off2[I + 1]), int(off2[J]):int(off2[J + 1])]
                e = float(torch.linalg.norm(B - E) / max(1e-300, float(torch.linalg.norm(E))))
                parts = []
                for a in range(2):
                    for b in range(2):
                        ci, cj = 2 * I + a, 2 * J + b
                        r0 = 0 if a == 0 else rk[2 * I]
                        c0 = 0 if b == 0 else rk[2 * J]
                        sub = (slice(r0, r0 + rk[ci]), slice(c0, c0 + rk[cj]))
                        ee = float(torch.linalg.norm(B[sub] - E[sub]))
                        nn = float(torch.linalg.norm(E[sub])) + 1e-300
                        kind = "diag" if ci == cj else ("near" if cj in near[ci] else ("far" if cj in far[ci] else "covered"))
                        parts.append(f"({ci},{cj}) {kind} {ee / nn:.1e}")
                worst.append((e, I, J, parts))
        worst.sort(reverse=True)
        print(f"  merged level {lvl - 1}: worst rel err {worst[0][0]:.3e}", flush=True)
        for e, I, J, parts in worst[:5]:
            print(f"     ({I},{J}) {e:.2e}: " + "; ".join(parts))


if __name__ == "__main__":
    main()
