"""Loss of orthogonality under windowed (delayed block) reorthogonalisation
in the thick-restart Lanczos of eigen.py:152-239 (design experiment).

Mode "full": the reference (recurrence + two CGS passes over the whole basis
every step).  Mode "block": every step the recurrence terms (T's column) and
two CGS passes over the window of the last `s` vectors only; when the window
is full its vectors get two block CGS passes against every older column
(B_old^T V, B_old H: the GEMM form).  Prints the largest |B_old^T V| found at
the block ends (the orthogonality lost inside a window) and the eigenvalues
against the full mode.
"""

import sys

import numpy as np
import scipy.sparse as sps


def operator(name):
    if name == "c1s":
        f = np.load("tests/golden/pipeline_c1s.npz")
        n = len(f["row_ptr"]) - 1
        w = sps.csr_matrix((f["vals"], f["col"], f["row_ptr"]), shape=(n, n))
        k = 20
    elif name == "c2s":
        f = np.load("tests/golden/graph_c2s.npz")
        n = len(f["row_ptr"]) - 1
        w = sps.csr_matrix((f["vals"], f["col"], f["row_ptr"]), shape=(n, n))
        k = 100
    else:
        f = np.load("tests/golden/shape_c4s.npz")
        n = len(f["row_ptr"]) - 1
        w = sps.csr_matrix((np.ones(len(f["col"])), f["col"], f["row_ptr"]), shape=(n, n))
        k = int(name[3:]) if len(name) > 3 else 100
    d = np.asarray(w.sum(axis=1)).ravel()
    di = 1 / np.sqrt(d)
    a = sps.diags(di) @ w @ sps.diags(di)
    return a.tocsr(), k


def lanczos(a, k, mode, s=16, tol=1e-8, seed=0, max_restarts=300, passes=2, adaptive=False, stats=None):
    stats = {} if stats is None else stats
    stats.setdefault('reads', 0)
    last = []
    n = a.shape[0]
    m = min(n, max(2 * k, k + 8))
    rng = np.random.default_rng(seed)
    B = np.zeros((n, m + 1))
    T = np.zeros((m, m))
    q = rng.standard_normal(n)
    B[:, 0] = q / np.linalg.norm(q)
    j = 0
    j0 = 0  # window start: columns < j0 are fully orthogonalised
    scale = 0.0
    pending = None
    restarts = 0
    worst = 0.0
    matvecs = 0

    def cgs2(w, lo, hi):
        for _ in range(2):
            V = B[:, lo:hi]
            w = w - V @ (V.T @ w)
        return w

    def flush(lo, hi):
        # block CGS2 of columns [lo, hi) against [0, lo)
        nonlocal worst
        if lo == 0 or hi <= lo:
            return
        V = B[:, lo:hi]
        H = B[:, :lo].T @ V
        worst = max(worst, np.abs(H).max())
        V -= B[:, :lo] @ H
        if passes == 2:
            V -= B[:, :lo] @ (B[:, :lo].T @ V)
        after = np.abs(B[:, :lo].T @ V).max()
        stats["after"] = max(stats.get("after", 0.0), after)
        stats["reads"] += passes * 2 * lo
        last.append(np.abs(H).max())
        if np.abs(H).max() > 1e-8:
            # re-orthonormalise inside the window (CGS2, in order)
            for c in range(lo, hi):
                v = B[:, c]
                if c > lo:
                    v = cgs2(v, lo, c)
                B[:, c] = v / np.linalg.norm(v)

    while True:
        w = a @ B[:, j]
        matvecs += 1
        alpha = B[:, j] @ w
        T[j, j] = alpha
        w -= B[:, : j + 1] @ T[: j + 1, j]
        if mode == "full":
            w = cgs2(w, 0, j + 1)
            stats["reads"] += 4 * (j + 1)
        else:
            w = cgs2(w, j0, j + 1)
            stats["reads"] += 4 * (j + 1 - j0)
        beta = np.linalg.norm(w)
        scale = max(scale, abs(alpha), beta)
        if j + 1 == m:
            if mode != "full":
                # the last vectors of the sweep: correct before the Ritz step
                flush(j0, j + 1)
                w = cgs2(w, 0, j + 1)
                beta = np.linalg.norm(w)
            theta, S = np.linalg.eigh(T)
            o = np.argsort(-theta, kind="stable")
            theta, S = theta[o], S[:, o]
            est = beta * np.abs(S[m - 1, :k])
            conv = bool(np.all(est <= tol * np.maximum(1, np.abs(theta[:k]))))
            ver = pending is not None and np.all(
                np.abs(theta[:k] - pending) <= np.maximum(1, np.abs(theta[:k])) * max(tol, 1e-12))
            if conv and ver:
                V = B[:, :m] @ S[:, :k]
                V /= np.linalg.norm(V, axis=0)
                return theta[:k], V, restarts, matvecs, worst
            restarts += 1
            if restarts > max_restarts:
                raise RuntimeError("no convergence")
            B[:, :k] = B[:, :m] @ S[:, :k]
            T[:] = 0
            T[np.arange(k), np.arange(k)] = theta[:k]
            if conv:
                pending = theta[:k].copy()
                v = cgs2(rng.standard_normal(n), 0, k)
                B[:, k] = v / np.linalg.norm(v)
            else:
                pending = None
                B[:, k] = w / beta
                T[:k, k] = T[k, :k] = beta * S[m - 1, :k]
            j = k
            j0 = k
            continue
        B[:, j + 1] = w / beta
        T[j, j + 1] = T[j + 1, j] = beta
        j += 1
        if mode != "full" and j - j0 >= s:
            flush(j0, j + 1)
            j0 = j + 1
            if adaptive and last:
                if last[-1] > 1e-9:
                    s = max(2, s // 2)
                elif last[-1] < 1e-12:
                    s = min(32, s * 2)
                stats.setdefault("s_hist", []).append(s)


if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "c1s"
    a, k = operator(name)
    ref = lanczos(a, k, "full")
    print(f"{name}: n={a.shape[0]} k={k} full: restarts {ref[2]} matvecs {ref[3]}")
    st0 = {}
    lanczos(a, k, "full", stats=st0)
    print("  full reads per matvec", st0["reads"] / ref[3])
    for s, passes, adaptive in ((4, 2, False), (8, 2, False), (4, 1, False), (8, 1, False), (4, 1, True)):
        st = {}
        th, V, rs, mv, worst = lanczos(a, k, "block", s=s, passes=passes, adaptive=adaptive, stats=st)
        sh = st.get("s_hist", [s])
        print(f"  passes {passes} adaptive {adaptive} reads/matvec {st['reads'] / mv:.1f} after-flush {st.get('after', 0):.1e} s mean {np.mean(sh):.1f}")
        res = np.linalg.norm(a @ V - V * th, axis=0).max()
        orth = np.abs(V.T @ V - np.eye(k)).max()
        sv = np.linalg.svd(ref[1].T @ V, compute_uv=False)
        ang = np.sqrt(max(0, 1 - sv.min() ** 2))
        print(f"  s={s:3d} restarts {rs} matvecs {mv} max|B_old^T V| {worst:.1e} "
              f"dval {np.abs(th - ref[0]).max():.1e} res {res:.1e} orth {orth:.1e} angle {ang:.1e}")
