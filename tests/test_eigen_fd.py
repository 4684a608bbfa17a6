"""Pins of the closed-form eigenpair helper (tests/eigen_fd.py) against the
stored matrices themselves and the oracle, so the full-size property checks
rest on something other than themselves."""
import math

import numpy as np
import pytest

from oracle import phiks_oracle as O
from paper_2210_07667_b200 import workloads as W

import eigen_fd as E


@pytest.mark.parametrize("cfg", [0, 1, 4])
def test_dirichlet_operators_are_exact_toeplitz(cfg):
    for pb in W.config(cfg, small=True).problems:
        for A in pb.A:
            assert E.is_toeplitz_tridiag(A)


@pytest.mark.parametrize("n,k,kind,build", [
    (33, 1, "toeplitz", lambda n: W.fd_dxx_dirichlet(n) + 10.0 * W.fd_dx_dirichlet(n)),
    (64, 7, "toeplitz", lambda n: W.fd_dxx_dirichlet(n) - 10.0 * W.fd_dx_dirichlet(n)),
    (512, 300, "toeplitz", lambda n: W.fd_dxx_dirichlet(n) + 10.0 * W.fd_dx_dirichlet(n)),
    (24, 3, "neumann", lambda n: 2e-3 * W.fd_dxx_neumann(n)),
    (256, 200, "neumann", lambda n: 0.01 * W.fd_dxx_neumann(n)),
])
def test_eigpair_residual(n, k, kind, build):
    A = build(n)
    lam, x = E.eigpair(A, k, kind)
    r = A @ x - float(lam) * x
    assert np.linalg.norm(r) <= 1e-14 * np.abs(A).sum(axis=0).max()
    # matches the eigenvalue numpy finds
    ev = np.linalg.eigvals(A)
    assert np.min(np.abs(ev - float(lam))) <= 1e-9 * np.abs(ev).max()


def test_phi_closed_forms():
    z = -0.37
    assert abs(float(E.phi(0, z)) - np.exp(z)) <= 4e-16
    assert abs(float(E.phi(1, z)) - np.expm1(z) / z) <= 4e-16
    # recurrence φ_{ℓ}(z) = z φ_{ℓ+1}(z) + 1/ℓ! across the series/closed-form switch
    for zz in (-3.0, -0.6, -0.4, 0.2, 2.0):
        for ell in range(5):
            lhs = E.phi(ell, zz)
            rhs = float(zz * E.phi(ell + 1, zz)) + 1.0 / math.factorial(ell)
            assert abs(float(lhs) - rhs) <= 1e-15 * max(1.0, abs(rhs))


def test_property_reproduces_oracle_small():
    # the eigen-tensor property against the oracle on a small ADR problem
    pb = W.config(4, small=True, with_vectors=False).problems[0]
    ks = [(1, 1, 1), (3, 5, 2)]
    rng = np.random.default_rng(0)
    es, lams = [], []
    for kk in ks:
        pairs = [E.eigpair(A, k, "toeplitz") for A, k in zip(pb.A, kk)]
        es.append(E.separable([x for _, x in pairs]))
        lams.append(sum(l for l, _ in pairs))
    c = rng.uniform(-1, 1, size=(len(pb.ells), len(ks)))
    vs = [W.from_flat(sum(c[i, t] * es[t] for t in range(len(ks))), pb.dims) for i in range(len(pb.ells))]
    res = O.phiks(pb.A, pb.tau, "lincomb", pb.ells, vs, n_scales=1)
    exp = sum(float(sum(E.phi(ell, pb.tau * lams[t]) * c[i, t] for i, ell in enumerate(pb.ells))) * es[t]
              for t in range(len(ks)))
    got = W.as_flat(res.out[0])
    assert np.linalg.norm(got - exp) <= 1e-13 * np.linalg.norm(exp)
