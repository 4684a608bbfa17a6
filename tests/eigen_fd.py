"""Closed-form eigenpairs of the stored FD factor matrices (test helper).

Every BASELINE.json operator is, entry for entry as stored in fp64, either a
tridiagonal Toeplitz matrix (Dirichlet ADR/Laplacian: sub a, diagonal b, super
c, all rows computed identically) or a power-of-two-scaled integer matrix
(Neumann Laplacian s·tridiag(1,-2,1) with 2 in the corner rows), so their
eigenpairs have textbook closed forms evaluated here in 50-digit arithmetic:

  Toeplitz (a·c > 0):  λ_k = b + 2√(ac)·cos(kπ/(n+1)),
                       x_j = (a/c)^{j/2}·sin(jkπ/(n+1)),  j = 1..n
  Neumann:             λ_k = s·(2cos(kπ/(n-1)) − 2),  x_j = cos(jkπ/(n-1)), j = 0..n-1

For a separable tensor e = x^(1) ⊗ … ⊗ x^(d) of eigenvectors,
K e = (Σ_μ λ^(μ)) e (Eq. (3)), hence φ_ℓ(τK) e = φ_ℓ(τλ) e — a
property that holds at any size, used for the full-size parity checks of
configs too large for the oracle.  Pinned by tests/test_eigen_fd.py.
"""
from __future__ import annotations

from typing import Sequence

import mpmath as mp
import numpy as np

mp.mp.dps = 50


def toeplitz_coeffs(A: np.ndarray):
    n = A.shape[0]
    b = A[0, 0]
    a = A[1, 0] if n > 1 else 0.0
    c = A[0, 1] if n > 1 else 0.0
    return a, b, c


def is_toeplitz_tridiag(A: np.ndarray) -> bool:
    a, b, c = toeplitz_coeffs(A)
    n = A.shape[0]
    T = np.diag(np.full(n, b)) + np.diag(np.full(n - 1, a), -1) + np.diag(np.full(n - 1, c), 1)
    return np.array_equal(T, A)


def eigpair(A: np.ndarray, k: int, kind: str):
    """(λ as mpf, x as fp64 array normalised to unit 2-norm) of mode k."""
    n = A.shape[0]
    if kind == "toeplitz":
        a, b, c = (mp.mpf(float(t)) for t in toeplitz_coeffs(A))
        th = mp.mpf(k) * mp.pi / (n + 1)
        lam = b + 2 * mp.sqrt(a * c) * mp.cos(th)
        r = mp.sqrt(a / c)
        x = [r ** j * mp.sin(j * th) for j in range(1, n + 1)]
    elif kind == "neumann":
        s = mp.mpf(float(A[0, 1])) / 2  # corner entry is 2s
        th = mp.mpf(k) * mp.pi / (n - 1)
        lam = s * (2 * mp.cos(th) - 2)
        x = [mp.cos(j * th) for j in range(n)]
    else:
        raise ValueError(kind)
    nrm = mp.sqrt(mp.fsum(t * t for t in x))
    return lam, np.array([float(t / nrm) for t in x])


def separable(vecs: Sequence[np.ndarray]) -> np.ndarray:
    """vec(x^(1) ⊗ … ⊗ x^(d)) in the column-major convention (§2)."""
    out = np.asarray(vecs[0])
    for x in vecs[1:]:
        out = np.kron(np.asarray(x), out)
    return out


def phi(ell: int, z) -> mp.mpf:
    """φ_ℓ(z) = (e^z − Σ_{k<ℓ} z^k/k!)/z^ℓ (Eq. (1)-(2)), 50 digits."""
    z = mp.mpf(z)
    if z == 0:
        return 1 / mp.factorial(ell)
    if abs(z) < mp.mpf("0.5"):
        return mp.fsum(z ** k / mp.factorial(k + ell) for k in range(80))
    return (mp.e ** z - mp.fsum(z ** k / mp.factorial(k) for k in range(ell))) / z ** ell
