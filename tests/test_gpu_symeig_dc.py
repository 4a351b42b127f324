"""Arrowhead divide-and-conquer projected eigensolver (csrc/sc_dc.cu) against
LAPACK (np.linalg.eigh = dsyevd, the reference's call at eigen.py:189) on the
matrices the thick-restart Lanczos produces (eigen.py:218-239): tridiagonal
(first sweep) and diag(theta) + arrow + tridiagonal tail (after a restart),
with clustered, repeated and deflating spectra, m in {200, 1000, 2000}."""

import time

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


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


def lanczos_T(rng, n, m, mult):
    """Lanczos projected matrix (full reorthogonalisation) of an operator
    with a `mult`-fold top eigenvalue."""
    ev = np.concatenate((np.ones(mult), rng.uniform(-1, 0.95, n - mult)))
    qq = np.linalg.qr(rng.standard_normal((n, n)))[0]
    A = (qq * ev) @ qq.T
    q = rng.standard_normal(n)
    Q = [q / np.linalg.norm(q)]
    al, be = [], []
    for _ in range(m):
        w = A @ Q[-1]
        al.append(Q[-1] @ w)
        B = np.array(Q).T
        w -= B @ (B.T @ w)
        w -= B @ (B.T @ w)
        be.append(np.linalg.norm(w))
        Q.append(w / be[-1])
    return np.diag(al) + np.diag(be[:-1], 1) + np.diag(be[:-1], -1)


def solve(T, p, k):
    from paper_1802_04450_b200 import _native as nat

    lib = nat.load()
    m = T.shape[0]
    Td = torch.from_numpy(np.asfortranarray(T).ravel(order="F").copy()).cuda()
    theta = torch.empty(m, dtype=torch.float64, device="cuda")
    S = torch.empty(m * k, dtype=torch.float64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    nat.check(lib.sc_symeig_arrow_f64(m, p, k, Td.data_ptr(), theta.data_ptr(), S.data_ptr(), st))
    torch.cuda.synchronize()
    return theta.cpu().numpy(), S.cpu().numpy().reshape(k, m).T


def check(T, p, k, tol=1e-13):
    m = T.shape[0]
    theta, S = solve(T, p, k)
    w, V = np.linalg.eigh(T)
    want = w[::-1]
    scale = max(1.0, np.abs(w).max())
    assert np.abs(theta - want).max() <= tol * m * scale
    # eigenvectors: residual, orthonormality, and the subspace of the k
    # largest (when separated from the rest) against LAPACK's
    assert np.abs(T @ S - S * theta[:k]).max() <= tol * m * scale
    assert np.abs(S.T @ S - np.eye(k)).max() <= tol * m
    if k < m and want[k - 1] - want[k] > 1e-6 * scale:
        Vk = V[:, ::-1][:, :k]
        # sin of the largest principal angle: |(I - S S^T) V_k|_2
        assert np.linalg.norm(Vk - S @ (S.T @ Vk), 2) < 1e-10
    return theta, S


@pytest.mark.parametrize("m", [1, 2, 3, 5, 17, 64, 200, 1000, 2000])
def test_tridiagonal(m):
    rng = np.random.default_rng(m)
    check(make_thick(rng, m, 0), 0, max(1, m // 2))


@pytest.mark.parametrize("m", [5, 64, 200, 1000, 2000])
def test_thick_restart_structure(m):
    rng = np.random.default_rng(m + 1)
    p = m // 2
    check(make_thick(rng, m, p), p, p)


@pytest.mark.parametrize("m", [200, 2000])
def test_clustered_c3_like(m):
    # the k wanted Ritz values packed in [0.998, 1] (scaled C3 run)
    rng = np.random.default_rng(7)
    p = m // 2
    theta = np.sort(1 - 2e-3 * rng.random(p))[::-1]
    check(make_thick(rng, m, p, theta=theta, coupling=1e-6), p, p)


def test_repeated_and_deflating():
    rng = np.random.default_rng(3)
    m, p = 200, 100
    check(make_thick(rng, m, p, theta=np.repeat([1.0, 0.99, 0.5], [40, 30, 30])), p, p)
    check(make_thick(rng, m, p, coupling=0.0), p, p)      # verification restart
    check(make_thick(rng, m, p, coupling=1e-12), p, p)
    T = make_thick(rng, m, 50)
    T[[70, 71], [71, 70]] = 0.0                             # breakdown inside the tail
    T[[120, 121], [121, 120]] = 0.0
    check(T, 50, 50)
    check(np.eye(m), 0, 20)
    T = np.eye(m)
    T[:100, 100] = T[100, :100] = 1e-9
    check(T, 100, 100)
    Tw = np.diag(np.abs(np.arange(m) - m // 2).astype(float)) + np.eye(m, k=1) + np.eye(m, k=-1)
    check(Tw, 0, 10)                                        # Wilkinson: close pairs


def test_lanczos_matrix_repeated_eigenvalue():
    rng = np.random.default_rng(11)
    T = lanczos_T(rng, 400, 200, 20)
    theta, _ = check(T, 0, 40)
    assert np.sum(np.abs(theta[:40] - 1.0) < 1e-8) >= 1


def test_speed():
    rng = np.random.default_rng(5)
    out = {}
    for m in (200, 2000):
        p = m // 2
        T = make_thick(rng, m, p, theta=np.sort(1 - 2e-3 * rng.random(p))[::-1], coupling=1e-6)
        solve(T, p, p)
        from paper_1802_04450_b200 import _native as nat

        lib = nat.load()
        Td = torch.from_numpy(np.asfortranarray(T).ravel(order="F").copy()).cuda()
        theta = torch.empty(m, dtype=torch.float64, device="cuda")
        S = torch.empty(m * p, dtype=torch.float64, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        torch.cuda.synchronize()
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            nat.check(lib.sc_symeig_arrow_f64(m, p, p, Td.data_ptr(), theta.data_ptr(), S.data_ptr(), st))
        torch.cuda.synchronize()
        out[m] = (time.perf_counter() - t0) / reps
    print("arrowhead D&C seconds per solve:", out)
    assert out[2000] < 0.25
