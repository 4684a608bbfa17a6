"""Brute-force dense references — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

These assemble the large matrix K that PHIKS never forms (§2 Eq. (3),
l.214-219) and evaluate φ-functions of it directly, for tiny N only.  They
pin the oracle's PHIKS implementation (tests/test_oracle_phiks.py).
"""
from __future__ import annotations

import math
from typing import Dict, Sequence

import numpy as np
import scipy.linalg

N_MAX = 700


def assemble_K(factors: Sequence[np.ndarray]) -> np.ndarray:
    """K = A_d ⊕ … ⊕ A_1 = Σ_μ I_d ⊗ … ⊗ A_μ ⊗ … ⊗ I_1 (Eq. (3))."""
    d = len(factors)
    dims = [a.shape[0] for a in factors]
    N = int(np.prod(dims))
    if N > N_MAX:
        raise ValueError(f"dense oracle capped at N <= {N_MAX}")
    K = np.zeros((N, N), dtype=np.result_type(*factors, np.float64))
    for mu in range(d):
        M = np.ones((1, 1))
        for nu in range(d - 1, -1, -1):
            M = np.kron(M, factors[nu] if nu == mu else np.eye(dims[nu]))
        K = K + M
    return K


def lincomb_augmented(K: np.ndarray, vs: Dict[int, np.ndarray]) -> np.ndarray:
    """exp(K)v_0 + Σ_{ℓ=1}^p φ_ℓ(K) v_ℓ as the first N rows of
    exp([[K, W],[0, J]]) [v_0; e_p] with W = [v_p,…,v_1] and J the p×p
    upper shift (augmented-matrix device, [AMH11] Th. 2.1).
    The exponential is scipy.linalg.expm (Padé; independent of expm_taylor)."""
    N = K.shape[0]
    p = max(vs.keys())
    if p == 0:
        return scipy.linalg.expm(K) @ vs[0]
    dt = np.result_type(K, *vs.values())
    W = np.zeros((N, p), dtype=dt)
    for ell in range(1, p + 1):
        if ell in vs:
            W[:, p - ell] = vs[ell]
    J = np.diag(np.ones(p - 1), 1)
    Aug = np.zeros((N + p, N + p), dtype=dt)
    Aug[:N, :N] = K
    Aug[:N, N:] = W
    Aug[N:, N:] = J
    rhs = np.zeros(N + p, dtype=dt)
    if 0 in vs:
        rhs[:N] = vs[0]
    rhs[-1] = 1.0
    return (scipy.linalg.expm(Aug) @ rhs)[:N]


def phi_taylor_dense(K: np.ndarray, ell: int, terms: int = 400) -> np.ndarray:
    """φ_ℓ(K) = Σ_k K^k/(k+ℓ)! with scaling by powers of two avoided — only
    for ||K|| ≲ 5 (second, independent dense method for cross-checks)."""
    N = K.shape[0]
    S = np.zeros_like(K, dtype=np.result_type(K, np.float64))
    P = np.eye(N, dtype=S.dtype)
    for k in range(terms):
        S = S + P / math.factorial(k + ell)
        P = P @ K
        if np.abs(P).max() / math.factorial(k + 1 + ell) < 1e-300:
            break
    return S
