"""numpy prototype of the arrowhead divide-and-conquer eigensolver that
csrc/sc_dc.cu implements (design check only; not used by the package).

The Lanczos projected matrix after a thick restart (eigen.py:218-239) is
diag(theta_0..theta_{p-1}) bordered at row/column p by the couplings, followed
by a tridiagonal tail.  Splitting every tridiagonal block at a middle row
turns the merge into an arrowhead eigenproblem (Gu & Eisenstat's tear), so the
whole solve is: arrowhead solves (secular equation per root, Loewner
recomputation of the border for orthogonality, deflation of tiny border
entries and close poles) + products with the child eigenvector blocks.
"""

from __future__ import annotations

import numpy as np

EPS = np.finfo(np.float64).eps


def _secular_root(j, d, z2, alpha, znorm):
    """Root j (0..r) of f(lam) = alpha - lam + sum z2/(lam - d), d ascending.
    Returns (origin index, tau) with lam = d[origin] + tau; origin -1 means
    the apex alpha is the origin (r == 0)."""
    r = len(d)
    if r == 0:
        return -1, 0.0
    if j == 0:
        o = 0
        lo, hi = min(d[0], alpha) - znorm - d[0], 0.0
    elif j == r:
        o = r - 1
        lo, hi = 0.0, max(d[r - 1], alpha) + znorm - d[r - 1]
    else:
        mid = 0.5 * (d[j - 1] + d[j])
        fm = alpha - mid + np.sum(z2 / (mid - d))
        if fm > 0:  # root right of the midpoint: origin at the upper pole
            o = j
            lo, hi = mid - d[j], 0.0
        else:
            o = j - 1
            lo, hi = 0.0, mid - d[j - 1]
    delta = d - d[o]
    a0 = alpha - d[o]
    ilo = j - 1  # nearest pole left of the root (if any)
    ihi = j if j < r else -1
    tau = 0.5 * (lo + hi)
    w1 = w2 = np.inf
    for it in range(200):
        t = tau - delta
        terms = z2 / t
        f = a0 - tau + terms.sum()
        err = abs(a0) + abs(tau) + np.abs(terms).sum()
        if f == 0.0 or abs(f) <= 4 * EPS * err:
            break
        if f > 0:
            lo = tau
        else:
            hi = tau
        if hi - lo <= 2 * EPS * max(abs(lo), abs(hi)):
            break
        # two-pole model matching f and f' at tau (the -1 of the linear
        # term split between the two poles; one pole plus the exact linear
        # term for the extreme roots)
        dterms = z2 / (t * t)
        sl = dterms[: ilo + 1].sum() if ilo >= 0 else 0.0
        sh = dterms[ihi:].sum() if ihi >= 0 else 0.0
        new = None
        if ilo >= 0 and ihi >= 0:
            dl, dh = delta[ilo], delta[ihi]
            s_lo = (sl + 0.5) * t[ilo] ** 2
            s_hi = (sh + 0.5) * t[ihi] ** 2
            c = f - s_lo / (tau - dl) - s_hi / (tau - dh)
            qa = c
            qb = -c * (dl + dh) + s_lo + s_hi
            qc = c * dl * dh - s_lo * dh - s_hi * dl
            new = _quad_in(qa, qb, qc, lo, hi)
        elif ihi >= 0:  # lowest root: poles only to the right, exact -x term
            dh = delta[ihi]
            s_hi = sh * t[ihi] ** 2
            c = f + tau - s_hi / (tau - dh)
            new = _quad_in(-1.0, c + dh, -c * dh + s_hi, lo, hi)
        else:
            dl = delta[ilo]
            s_lo = sl * t[ilo] ** 2
            c = f + tau - s_lo / (tau - dl)
            new = _quad_in(-1.0, c + dl, -c * dl + s_lo, lo, hi)
        width = hi - lo
        if new is None or not (lo < new < hi) or width > 0.5 * w2:
            new = 0.5 * (lo + hi)
        w2, w1 = w1, width
        tau = new
    return o, tau


def _quad_in(a, b, c, lo, hi):
    """A root of a x^2 + b x + c = 0 inside (lo, hi), stable formula."""
    if a == 0.0:
        if b == 0.0:
            return None
        x = -c / b
        return x if lo < x < hi else None
    disc = b * b - 4 * a * c
    if disc < 0:
        return None
    sq = np.sqrt(disc)
    q = -0.5 * (b + np.copysign(sq, b))
    cands = []
    if q != 0.0:
        cands += [q / a, c / q]
    else:
        cands += [0.0]
    for x in cands:
        if lo < x < hi:
            return x
    return None


def arrow_eig(d, z, alpha):
    """[[diag(d), z], [z^T, alpha]] -> (lam ascending, U) with the apex as
    the last coordinate."""
    n = len(d)
    N = n + 1
    if n == 0:
        return np.array([alpha]), np.ones((1, 1))
    perm = np.argsort(d, kind="stable")
    ds = d[perm].astype(float).copy()
    zs = z[perm].astype(float).copy()
    scale = max(np.abs(ds).max(), abs(alpha), np.abs(zs).max())
    tol = 8.0 * EPS * scale
    W = np.eye(n)  # basis of the d-coordinates (columns), sorted order
    kept = []
    defl = []
    pj = -1
    for jj in range(n):
        if abs(zs[jj]) <= tol:
            defl.append(jj)
            continue
        if pj >= 0:
            t = np.hypot(zs[pj], zs[jj])
            c = zs[jj] / t
            s = zs[pj] / t
            tau = (ds[jj] - ds[pj]) * c * s
            if abs(tau) <= tol:
                a = c * W[:, pj] - s * W[:, jj]
                b = s * W[:, pj] + c * W[:, jj]
                dpj = ds[pj] * c * c + ds[jj] * s * s
                djj = ds[pj] * s * s + ds[jj] * c * c
                W[:, pj], W[:, jj] = a, b
                ds[pj], ds[jj] = dpj, djj
                zs[pj], zs[jj] = 0.0, t
                defl.append(pj)
                kept.pop()
        kept.append(jj)
        pj = jj
    kept = np.array(kept, dtype=int)
    dk, zk = ds[kept], zs[kept]
    r = len(kept)
    z2 = zk * zk
    znorm = np.sqrt(z2.sum())
    roots = [_secular_root(j, dk, z2, alpha, znorm) for j in range(r + 1)]
    lam = np.array([(dk[o] if o >= 0 else alpha) + t for o, t in roots])
    # differences lam_j - d_i from the origin representation
    diff = np.empty((r + 1, r))
    for j, (o, t) in enumerate(roots):
        diff[j] = (dk[o] - dk) + t if o >= 0 else (alpha - dk)
    # Loewner: zhat_i^2 = (d_i - lam_0)(lam_r - d_i) prod_{j=1}^{i-1} (d_i-lam_j)/(d_i-d_j)
    #                      * prod_{j=i}^{r-1} (lam_j - d_i)/(d_{j+1} - d_i)
    zh = np.empty(r)
    for i in range(r):
        p = (-diff[0, i]) * diff[r, i]
        for j in range(1, r):
            if j <= i:
                # lam_j < d_i for j <= i (lam_j in (d_{j-1}, d_j))
                p *= (-diff[j, i]) / (dk[i] - dk[j - 1])
            else:
                p *= diff[j, i] / (dk[j] - dk[i])
        zh[i] = np.copysign(np.sqrt(p), zk[i])
    vals = []
    vecs = []
    for j in range(r + 1):
        x = zh / diff[j]
        v = np.zeros(N)
        v[:n] = W[:, kept] @ x
        v[n] = 1.0
        v /= np.linalg.norm(v)
        vals.append(lam[j])
        vecs.append(v)
    for jj in defl:
        v = np.zeros(N)
        v[:n] = W[:, jj]
        vals.append(ds[jj])
        vecs.append(v)
    vals = np.array(vals)
    order = np.argsort(vals, kind="stable")
    vals = vals[order]
    V = np.array(vecs).T[:, order]
    # back to the caller's d order
    out = np.zeros_like(V)
    out[perm] = V[:n]
    out[n] = V[n]
    return vals, out


def tri_eig(a, b):
    """Symmetric tridiagonal (diag a, off-diagonal b) by tearing at the middle row."""
    n = len(a)
    if n == 1:
        return np.array([a[0]]), np.ones((1, 1))
    if n == 2:
        return np.linalg.eigh(np.diag(a) + np.diag(b, 1) + np.diag(b, -1))
    mid = n // 2
    l1, q1 = tri_eig(a[:mid], b[: mid - 1]) if mid > 0 else (np.zeros(0), np.zeros((0, 0)))
    l2, q2 = tri_eig(a[mid + 1:], b[mid + 1:]) if mid + 1 < n else (np.zeros(0), np.zeros((0, 0)))
    d = np.concatenate((l1, l2))
    z = np.concatenate((b[mid - 1] * q1[-1, :] if mid > 0 else [], b[mid] * q2[0, :] if mid + 1 < n else []))
    lam, u = arrow_eig(d, z, a[mid])
    n1 = mid
    Q = np.zeros((n, n))
    Q[:n1] = q1 @ u[:n1]
    Q[mid] = u[-1]
    Q[mid + 1:] = q2 @ u[n1:-1]
    return lam, Q


def thick_eig(T, p):
    """T: arrowhead (rows/cols 0..p-1 diagonal, coupled to p) + tridiagonal tail."""
    m = T.shape[0]
    if p == 0:
        return tri_eig(np.diag(T).copy(), np.diag(T, 1).copy())
    theta = np.diag(T)[:p]
    c = T[:p, p]
    if p + 1 < m:
        l2, q2 = tri_eig(np.diag(T)[p + 1:].copy(), np.diag(T, 1)[p + 1:].copy())
        d = np.concatenate((theta, l2))
        z = np.concatenate((c, T[p, p + 1] * q2[0, :]))
    else:
        l2, q2 = np.zeros(0), np.zeros((0, 0))
        d, z = theta, c
    lam, u = arrow_eig(d, z, T[p, p])
    Q = np.zeros((m, m))
    Q[:p] = u[:p]
    Q[p] = u[-1]
    Q[p + 1:] = q2 @ u[p:-1]
    return lam, Q


def _check(T, p, name):
    lam, Q = thick_eig(T, p)
    ref = np.linalg.eigvalsh(T)
    m = T.shape[0]
    nrm = max(1.0, np.abs(ref).max())
    e_val = np.abs(lam - ref).max() / nrm
    e_orth = np.abs(Q.T @ Q - np.eye(m)).max()
    e_res = np.abs(T @ Q - Q * lam).max() / nrm
    print(f"{name:28s} m={m:5d} val {e_val:.2e} orth {e_orth:.2e} res {e_res:.2e}")
    assert e_val < 1e-13 * m and e_orth < 1e-13 * m and e_res < 1e-13 * m, name


def make_thick(rng, m, p, theta=None, coupling=1e-3, tail_scale=1.0):
    T = np.zeros((m, m))
    if theta is None:
        theta = np.sort(rng.uniform(0.9, 1.0, p))[::-1]
    T[np.arange(p), np.arange(p)] = theta
    T[:p, p] = T[p, :p] = coupling * rng.standard_normal(p)
    a = tail_scale * rng.uniform(-1, 1, m - p)
    b = tail_scale * rng.uniform(0.01, 1, m - p - 1)
    T[np.arange(p, m), np.arange(p, m)] = a
    T[np.arange(p, m - 1), np.arange(p + 1, m)] = b
    T[np.arange(p + 1, m), np.arange(p, m - 1)] = b
    return T


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    for m in (5, 17, 64, 200):
        _check(make_thick(rng, m, 0), 0, "tridiagonal")
        _check(make_thick(rng, m, m // 2), m // 2, "thick")
    # repeated Ritz values (multiplicity), zero couplings, clustered tail
    m = 200
    T = make_thick(rng, m, 100, theta=np.repeat([1.0, 0.99, 0.5], [40, 30, 30]))
    _check(T, 100, "repeated theta")
    T = make_thick(rng, m, 100, coupling=0.0)
    _check(T, 100, "zero couplings")
    T = make_thick(rng, m, 100, coupling=1e-12)
    _check(T, 100, "tiny couplings")
    # Wilkinson-like tail and a tail with zero off-diagonals (split)
    T = make_thick(rng, m, 0)
    T[np.arange(m - 1), np.arange(1, m)] = 1.0
    T[np.arange(1, m), np.arange(m - 1)] = 1.0
    T[np.arange(m), np.arange(m)] = np.abs(np.arange(m) - m // 2)
    _check(T, 0, "wilkinson")
    T = make_thick(rng, m, 50)
    T[[70, 71], [71, 70]] = 0.0
    T[[120, 121], [121, 120]] = 0.0
    _check(T, 50, "split tail")
    # identity-like: all eigenvalues 1 (blocks of components)
    T = np.eye(m)
    _check(T, 0, "identity")
    T = np.eye(m)
    T[:100, 100] = T[100, :100] = 1e-9
    _check(T, 100, "identity + tiny arrow")
    # lanczos matrix of an operator with a 20-fold eigenvalue
    n = 400
    ev = np.concatenate((np.ones(20), rng.uniform(-1, 0.95, n - 20)))
    qq = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (qq * ev) @ qq.T
    q = rng.standard_normal(n)
    Qb = [q / np.linalg.norm(q)]
    al, be = [], []
    for j in range(m):
        w = A @ Qb[-1]
        B = np.array(Qb).T
        w -= B @ (B.T @ w)
        w -= B @ (B.T @ w)
        al.append(Qb[-1] @ A @ Qb[-1])
        bt = np.linalg.norm(w)
        be.append(bt)
        Qb.append(w / bt)
    T = np.diag(al) + np.diag(be[:-1], 1) + np.diag(be[:-1], -1)
    _check(T, 0, "lanczos T (repeated)")
    for m in (1000, 2000):
        p = m // 2
        T = make_thick(rng, m, p, theta=np.sort(1 - 2e-3 * rng.random(p))[::-1], coupling=1e-6)
        _check(T, p, "C3-like clustered")
    print("ok")
