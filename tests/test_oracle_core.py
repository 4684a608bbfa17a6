"""Pins of the oracle's building blocks against values fixed by the paper and
by mathematics (never against the oracle itself).  CPU only."""
import itertools
import math

import mpmath
import numpy as np
import pytest
import scipy.linalg

from oracle import phiks_oracle as O
from oracle import dense as D
from paper_2210_07667_b200 import workloads as W


# ---------------------------------------------------------------- μ-mode / Tucker


def _loop_mode_product(T, M, mu):
    """Pure-Python definition: out[..j..] = Σ_k M[j,k] T[..k..]."""
    dims = list(T.shape)
    od = dims.copy()
    od[mu] = M.shape[0]
    out = np.zeros(od, dtype=np.result_type(T, M))
    for idx in itertools.product(*[range(n) for n in od]):
        acc = 0
        for k in range(dims[mu]):
            src = list(idx)
            src[mu] = k
            acc += M[idx[mu], k] * T[tuple(src)]
        out[idx] = acc
    return out


@pytest.mark.parametrize("mu", [0, 1, 2])
def test_mode_product_matches_loop_definition(mu):
    T = W.random_tensor((3, 4, 2), seed=11, complex_=True)
    M = np.random.default_rng(5).standard_normal((5, T.shape[mu]))
    got = O.mu_mode_product(T, M, mu)
    ref = _loop_mode_product(T, M, mu)
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


def test_mode_product_row_swap_example():
    # SPEC-style trivial case: 2x2 tensor [[1,2],[3,4]], mu=1, M = swap -> rows swapped
    T = np.array([[1.0, 2.0], [3.0, 4.0]])
    M = np.array([[0.0, 1.0], [1.0, 0.0]])
    assert np.array_equal(O.mu_mode_product(T, M, 0), np.array([[3.0, 4.0], [1.0, 2.0]]))


def test_tucker_equals_kronecker_matrix():
    # vec(V ×_1 M_1 … ×_d M_d) = (M_d ⊗ … ⊗ M_1) vec(V)
    dims = (3, 4, 5)
    T = W.random_tensor(dims, seed=3)
    mats = [np.random.default_rng(10 + i).standard_normal((n, n)) for i, n in enumerate(dims)]
    kron = np.kron(mats[2], np.kron(mats[1], mats[0]))
    ref = kron @ W.as_flat(T)
    got = W.as_flat(O.tucker(T, mats))
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_tucker_identity_and_2d_formula():
    T = W.random_tensor((4, 6), seed=1)
    assert np.array_equal(O.tucker(T, [np.eye(4), np.eye(6)]), T)
    M1 = np.random.default_rng(1).standard_normal((4, 4))
    M2 = np.random.default_rng(2).standard_normal((6, 6))
    # exp(A1) V exp(A2)^T two-dimensional formula
    assert np.allclose(O.tucker(T, [M1, M2]), M1 @ T @ M2.T, rtol=0, atol=1e-13)


def test_tucker_mode_order_irrelevant():
    T = W.random_tensor((3, 4, 5), seed=4)
    mats = [np.random.default_rng(i).standard_normal((n, n)) for i, n in enumerate(T.shape)]
    a = O.tucker(T, mats)
    b = O.mu_mode_product(O.mu_mode_product(O.mu_mode_product(T, mats[2], 2), mats[0], 0), mats[1], 1)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


# ---------------------------------------------------------------- expm


def test_expm_zero_and_diagonal():
    assert np.array_equal(O.expm_taylor(np.zeros((3, 3))), np.eye(3))
    lam = np.array([1.0, -1.0, 7.5, -30.0])
    E = O.expm_taylor(np.diag(lam))
    assert np.allclose(np.diag(E), np.exp(lam), rtol=1e-14, atol=0)
    assert np.abs(E - np.diag(np.diag(E))).max() == 0.0


def test_expm_jordan_block_closed_form():
    lam, n = -2.5, 6
    J = lam * np.eye(n) + np.diag(np.ones(n - 1), 1)
    ref = np.zeros((n, n))
    for i in range(n):
        for j in range(i, n):
            ref[i, j] = math.exp(lam) / math.factorial(j - i)
    assert np.abs(O.expm_taylor(J) - ref).max() <= 1e-14


@pytest.mark.parametrize("scale", [0.1, 3.0, 40.0])
def test_expm_vs_scipy_pade(scale):
    A = W.random_factors([12], seed=7, scale=scale)[0]
    got, ref = O.expm_taylor(A), scipy.linalg.expm(A)
    assert np.linalg.norm(got - ref, 1) <= 1e-12 * max(np.linalg.norm(ref, 1), 1.0)


def test_expm_half_squared():
    A = W.random_factors([9], seed=8, scale=5.0, complex_=True)[0]
    E = O.expm_taylor(A)
    H = O.expm_taylor(A / 2)
    assert np.linalg.norm(H @ H - E, 1) <= 1e-12 * np.linalg.norm(E, 1)


# ---------------------------------------------------------------- GLL


def test_gll_closed_forms():
    x, w = O.gll_rule(2)
    assert np.allclose(x, [0, 1]) and np.allclose(w, [0.5, 0.5])
    x, w = O.gll_rule(3)
    assert np.allclose(x, [0, 0.5, 1], atol=1e-15) and np.allclose(w, [1 / 6, 2 / 3, 1 / 6], atol=1e-15)
    x, w = O.gll_rule(4)
    r5 = 1 / math.sqrt(5)
    assert np.allclose(x, [0, (1 - r5) / 2, (1 + r5) / 2, 1], atol=1e-15)
    assert np.allclose(w, [1 / 12, 5 / 12, 5 / 12, 1 / 12], atol=1e-15)
    x, w = O.gll_rule(5)
    r37 = math.sqrt(3 / 7)
    assert np.allclose(x, [0, (1 - r37) / 2, 0.5, (1 + r37) / 2, 1], atol=1e-15)
    assert np.allclose(w, [1 / 20, 49 / 180, 16 / 45, 49 / 180, 1 / 20], atol=1e-15)


@pytest.mark.parametrize("q", list(range(2, 33)))
def test_gll_exactness_degree(q):
    x, w = O.gll_rule(q)
    assert x[0] == 0.0 and x[-1] == 1.0 and np.all(np.diff(x) > 0) and np.all(w > 0)
    assert abs(w.sum() - 1.0) <= 1e-14
    for k in range(0, 2 * q - 2):
        assert abs(np.dot(w, x ** k) - 1.0 / (k + 1)) <= 1e-13, k
    # degree 2q-2 is NOT integrated exactly (the rule is exactly of degree 2q-3)
    if q <= 8:
        k = 2 * q - 2
        assert abs(np.dot(w, x ** k) - 1.0 / (k + 1)) > 1e-12


# ---------------------------------------------------------------- kernel k_q


@pytest.mark.parametrize("z", [2.0 + 0j, 0.5 + 0.7j, -1.3 + 0.2j, 3 + 2j])
def test_kernel_q2_closed_form(z):
    # π_2(t) = t(t-1): k_2(z) = [(z^2-z) log(z/(z-1)) - z + 1/2] / (z^2 - z)
    ref = ((z * z - z) * np.log(z / (z - 1)) - z + 0.5) / (z * z - z)
    got = O.kernel_kq(O.gll_rule(2)[0], np.array([z]))[0]
    assert abs(got - ref) <= 1e-13 * abs(ref)


@pytest.mark.parametrize("q,a", [(4, 3.0), (6, -5.0 + 2j), (9, 8.0j), (12, -20.0)])
def test_kernel_hermite_formula_reproduces_quadrature_error(q, a):
    # R_q(f) = (1/2πi) ∮_Γ k_q(z) f(z) dz (Eq. (20), l.795-798) for f(t)=e^{at}
    x, w = O.gll_rule(q)
    exact = (np.exp(a) - 1) / a
    err = exact - np.dot(w, np.exp(a * x))
    r, nz = 1.2, 2048
    z, dz = O.ellipse(r, nz)
    kq = O.kernel_kq(x, z)
    contour = np.sum(kq * np.exp(a * z) * dz) / nz  # (1/2π)∫ k f (r e^{iζ} - ...) dζ
    assert abs(contour - err) <= 1e-7 * abs(err) + 1e-17


# ---------------------------------------------------------------- rectangle


def test_rectangle_contains_spectrum_and_rayleigh_quotients():
    fac = W.random_factors([3, 4, 2], seed=21, scale=4.0, complex_=True)
    rect = O.range_rectangle(fac)
    K = D.assemble_K(fac)
    rng = np.random.default_rng(0)

    def inside(z):
        d = z - rect.center
        return abs(d.real) <= rect.hr * (1 + 1e-12) and abs(d.imag) <= rect.hi * (1 + 1e-12)

    for lam in np.linalg.eigvals(K):
        assert inside(lam)
    for _ in range(200):
        x = rng.standard_normal(K.shape[0]) + 1j * rng.standard_normal(K.shape[0])
        assert inside(np.vdot(x, K @ x) / np.vdot(x, x))


def test_rectangle_fd_laplacian_analytic_eigenvalues():
    n = 10
    A = W.fd_dxx_dirichlet(n)
    rect = O.range_rectangle([A, A])
    h = 1.0 / (n + 1)
    k = np.arange(1, n + 1)
    lam1 = -(4 / h ** 2) * np.sin(k * np.pi * h / 2) ** 2
    lams = (lam1[:, None] + lam1[None, :]).ravel()
    assert rect.hi == 0.0
    assert np.all(np.abs(lams - rect.center.real) <= rect.hr * (1 + 1e-12))
    # trace-shifted rectangle is tight: its real extent equals the spectral spread
    assert rect.center.real - rect.hr <= lams.min() + 1e-9
    assert rect.center.real + rect.hr >= lams.max() - 1e-9


# ---------------------------------------------------------------- remainder bound


def _phi_scalar(ell, z):
    mpmath.mp.dps = 40
    z = mpmath.mpc(z)
    if ell == 0:
        return complex(mpmath.exp(z))
    s = mpmath.mpf(0)
    term = mpmath.mpf(1) / mpmath.factorial(ell)
    k = 0
    while True:
        s += term
        k += 1
        term = term * z / (k + ell)
        if abs(term) < mpmath.mpf(10) ** -45 * max(abs(s), 1):
            break
    return complex(s)


@pytest.mark.parametrize("q", [3, 5, 8])
def test_remainder_bound_dominates_true_scalar_error(q):
    rect = O.Rect(-6.0 - 1.0j, 5.0, 2.0)
    ells = [1, 2, 3]
    B = O.remainder_bounds(rect, ells, [q])[0]
    x, w = O.gll_rule(q)
    for wr in np.linspace(-1, 1, 7):
        for wi in np.linspace(-1, 1, 5):
            lam = rect.center + wr * rect.hr + 1j * wi * rect.hi
            for li, ell in enumerate(ells):
                f = x ** (ell - 1) / math.factorial(ell - 1) * np.exp((1 - x) * lam)
                err = abs(_phi_scalar(ell, lam) - np.dot(w, f))
                assert err <= B[li] * (1 + 1e-6) + 1e-16, (lam, ell, err, B[li])


def test_remainder_bound_zero_operator_exact_rule():
    # K = 0: f_ℓ polynomial of degree ℓ-1 ≤ 2q-3, the rule is exact
    B = O.remainder_bounds(O.Rect(0j, 0.0, 0.0), [1, 2, 3, 4, 5], [6])
    assert np.all(B <= 1e-12)


# ---------------------------------------------------------------- scalar φ identities


@pytest.mark.parametrize("ell", [1, 2, 3, 4, 5])
def test_squaring_identity_scalar(ell):
    # PAPER.md Eq. (12): φ_ℓ(2z) = 2^{-ℓ}(e^z φ_ℓ(z) + Σ_{k=1}^ℓ φ_k(z)/(ℓ-k)!)
    rng = np.random.default_rng(ell)
    for _ in range(20):
        z = complex(rng.uniform(-4, 4), rng.uniform(-4, 4))
        lhs = _phi_scalar(ell, 2 * z)
        rhs = (np.exp(z) * _phi_scalar(ell, z)
               + sum(_phi_scalar(k, z) / math.factorial(ell - k) for k in range(1, ell + 1))) / 2 ** ell
        assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_phi1_closed_form():
    for z in [1.0, -1.0, 0.3 + 2j, -7.0]:
        assert abs(_phi_scalar(1, z) - (np.exp(z) - 1) / z) <= 1e-14 * abs(_phi_scalar(1, z))
