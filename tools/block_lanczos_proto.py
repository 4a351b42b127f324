"""numpy model of the block thick-restart Lanczos used for large k
(csrc/sc_blanczos.cu): block size b, basis of mb = round_up(m, b) columns,
kr = round_up(k, b) retained Ritz vectors, T = Q^T A Q filled from the
full projections of every block (so no explicit QR coupling is needed),
local CGS2 against the last two blocks + one full CGS pass per block,
CholQR2 of the new block, dense Rayleigh-Ritz via Householder
tridiagonalisation + tridiagonal eigensolver + back-transformation,
residual estimates |W_last s_last| and the reference's verification sweep
from a fresh block (eigen.py:181-239)."""
import sys
import time

import numpy as np
import scipy.sparse as sp


def sytrd(A):
    """Householder tridiagonalisation (LAPACK dsytd2, lower): returns d, e,
    V (reflectors in columns, v[0] = 1 at row i+1), tau."""
    A = A.copy()
    m = A.shape[0]
    d = np.zeros(m)
    e = np.zeros(m - 1)
    tau = np.zeros(m)
    V = np.zeros((m, m))
    for i in range(m - 1):
        x = A[i + 1:, i].copy()
        alpha = x[0]
        xn = np.linalg.norm(x[1:])
        if xn == 0.0:
            t, beta, v = 0.0, alpha, np.zeros_like(x)
            v[0] = 1.0
        else:
            beta = -np.copysign(np.hypot(alpha, xn), alpha)
            t = (beta - alpha) / beta
            v = x / (alpha - beta)
            v[0] = 1.0
        d[i] = A[i, i]
        e[i] = beta
        tau[i] = t
        V[i + 1:, i] = v
        if t != 0.0:
            A22 = A[i + 1:, i + 1:]
            p = t * (A22 @ v)
            w = p - 0.5 * t * (p @ v) * v
            A22 -= np.outer(v, w) + np.outer(w, v)
    d[m - 1] = A[m - 1, m - 1]
    return d, e, V, tau


def dense_topk(T, kout):
    d, e, V, tau = sytrd(T)
    m = len(d)
    Tt = np.diag(d) + np.diag(e, 1) + np.diag(e, -1)
    lam, Z = np.linalg.eigh(Tt)
    order = np.argsort(-lam, kind="stable")[:kout]
    lam, Z = lam[order], Z[:, order].copy()
    for i in range(m - 2, -1, -1):  # Z <- H_i Z
        v = V[i + 1:, i]
        Z[i + 1:] -= tau[i] * np.outer(v, v @ Z[i + 1:])
    return lam, Z


def cgs(Q, W):
    H = Q.T @ W
    return W - Q @ H, H


def cholqr2(W, rng, Qb, scale):
    G = W.T @ W
    R1 = np.linalg.cholesky(G).T
    W = np.linalg.solve(R1.T, W.T).T
    G2 = W.T @ W
    R2 = np.linalg.cholesky(G2).T
    W = np.linalg.solve(R2.T, W.T).T
    return W, G


def block_lanczos(A, k, m=None, b=32, tol=1e-8, max_restarts=300, seed=0, verbose=False):
    n = A.shape[0]
    m = m or min(n, max(2 * k, k + 8))
    kr = -(-k // b) * b
    mb = -(-m // b) * b
    assert mb >= kr + 2 * b
    rng = np.random.default_rng(seed)
    Q = np.zeros((n, mb + b))
    T = np.zeros((mb, mb))
    X = rng.standard_normal((n, b))
    X, _ = np.linalg.qr(X)
    Q[:, :b] = X
    c0 = 0          # first column of the current block
    lock_hi = 0     # columns [0, lock_hi) were a restart's Ritz block
    restarts = 0
    blocks = 0
    scale = 0.0
    pending = None
    t_ritz = t_reorth = 0.0
    while True:
        # ---- one block step
        Qi = Q[:, c0:c0 + b]
        W = A @ Qi
        blocks += 1
        j = c0 + b
        t0 = time.perf_counter()
        first_after_restart = c0 == lock_hi and lock_hi > 0
        if first_after_restart or c0 < 2 * b:
            W, H1 = cgs(Q[:, :j], W)
            W, H2 = cgs(Q[:, :j], W)
            H = H1 + H2
        else:
            lo = c0 - b
            W, L1 = cgs(Q[:, lo:j], W)
            W, L2 = cgs(Q[:, lo:j], W)
            W, F = cgs(Q[:, :j], W)
            H = F.copy()
            H[lo:j] += L1 + L2
        t_reorth += time.perf_counter() - t0
        Hs = H.copy()
        Hs[c0:j] = 0.5 * (H[c0:j] + H[c0:j].T)
        T[:j, c0:j] = Hs
        T[c0:j, :j] = Hs.T
        scale = max(scale, np.abs(Hs[c0:j]).max())
        # CholQR2 of the new block (breakdown: not modelled here)
        Wn, G = cholqr2(W, rng, Q[:, :j], scale)
        if j + b <= mb:
            Q[:, j:j + b] = Wn
            c0 = j
            continue
        # ---- end of sweep: Rayleigh-Ritz on T (mb x mb)
        t0 = time.perf_counter()
        theta, S = dense_topk(T, kr)
        slast = S[mb - b:, :]
        est = np.sqrt(np.einsum("ij,ij->j", slast, G @ slast))
        conv = np.all(est[:k] <= tol * np.maximum(1.0, np.abs(theta[:k])))
        verified = pending is not None and np.all(
            np.abs(theta[:k] - pending) <= np.maximum(1.0, np.abs(theta[:k])) * max(tol, 1e-12))
        if verbose:
            print(f"restart {restarts}: blocks {blocks}, worst est {est[:k].max():.3e}, conv {conv}, "
                  f"verified {verified}", flush=True)
        if conv and verified:
            Y = Q[:, :mb] @ S[:, :k]
            t_ritz += time.perf_counter() - t0
            return theta[:k], Y, dict(restarts=restarts, blocks=blocks, matvecs=blocks * b, t_ritz=t_ritz,
                                      t_reorth=t_reorth)
        if restarts >= max_restarts:
            raise RuntimeError("max restarts")
        restarts += 1
        Y = Q[:, :mb] @ S
        t_ritz += time.perf_counter() - t0
        Q[:, :kr] = Y
        T[:] = 0.0
        T[np.arange(kr), np.arange(kr)] = theta
        if conv:
            pending = theta[:k].copy()
            X = rng.standard_normal((n, b))
            X, _ = cgs(Q[:, :kr], X)
            X, _ = cgs(Q[:, :kr], X)
            X, _ = np.linalg.qr(X)
            Q[:, kr:kr + b] = X
        else:
            pending = None
            Q[:, kr:kr + b] = Wn
        c0 = kr
        lock_hi = kr


def knn_operator(n, d, k, cs, knn, seed=0):
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    from oracle import speclust_oracle as orc
    x, y = orc.blobs(n, d, k, cs, seed=seed)
    sigma = float(np.sqrt(d))
    e = orc.knn_edges(x, knn, sigma)
    rp, col, vals = orc.csr_from_edges(n, e, orc.edge_weights(x, e, sigma))
    deg = orc.degrees(rp, col, vals)
    a = orc.sym_scale_vals(rp, col, vals, deg)
    return sp.csr_matrix((a, col, rp), shape=(n, n)), y


if __name__ == "__main__":
    n, d, kc, cs, knn, k = (int(v) if i != 3 else float(v) for i, v in enumerate(sys.argv[1:7]))
    b = int(sys.argv[7]) if len(sys.argv) > 7 else 32
    A, _ = knn_operator(n, d, kc, cs, knn)
    t0 = time.perf_counter()
    vals, vecs, st = block_lanczos(A, k, b=b, verbose=True)
    print("block", st, "time", time.perf_counter() - t0)
    res = np.linalg.norm(A @ vecs - vecs * vals, axis=0)
    print("max true residual", res.max(), "lambda", vals[0], vals[-1])
    if len(sys.argv) > 8:
        sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
        from oracle import speclust_oracle as orc
        t0 = time.perf_counter()
        v1, u1, r1, s1 = orc.lanczos_topk(lambda z: A @ z, n, k, seed=0)
        print("single", s1, "time", time.perf_counter() - t0)
        print("max eig diff", np.abs(v1 - vals).max())
        qa, _ = np.linalg.qr(u1)
        qb, _ = np.linalg.qr(vecs)
        print("subspace sin", np.linalg.norm(qa - qb @ (qb.T @ qa), 2))
