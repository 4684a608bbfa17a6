"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no μ-mode products, no
exponentials, no quadrature, no squaring).  It only builds the *inputs* of the
problem statement: the small factor matrices A_μ of the Kronecker sum
K = A_d ⊕ … ⊕ A_1 (§2 Eq. (3), "written as a Kronecker sum") and the
application vectors v, as BASELINE.json's `configs` describe them.  Both
`oracle/` and the product path import it; neither imports the other.

Layout convention (§2, "vec is the operator which stacks the columns
of the input tensor"): an order-d tensor of size n_1×…×n_d is stored
column-major, i.e. element (i_1,…,i_d) lives at i_1 + n_1*(i_2 + n_2*(…)).
A numpy array of shape (n_1,…,n_d) in Fortran order has exactly that layout;
`as_flat` / `from_flat` convert.  Matrices are n×n column-major (Fortran).
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# 1-D finite-difference factor matrices (§4.2 "second order centered
# finite differences", §4.3 "homogeneous Neumann boundary conditions").
# ---------------------------------------------------------------------------


def fd_dxx_dirichlet(n: int) -> np.ndarray:
    """Second derivative, 3-point stencil, homogeneous Dirichlet, n interior
    nodes on (0,1), h = 1/(n+1): tridiag(1,-2,1)/h^2."""
    h = 1.0 / (n + 1)
    A = np.zeros((n, n), order="F")
    i = np.arange(n)
    A[i, i] = -2.0
    A[i[:-1], i[:-1] + 1] = 1.0
    A[i[1:], i[1:] - 1] = 1.0
    return A / (h * h)


def fd_dx_dirichlet(n: int) -> np.ndarray:
    """First derivative, central 3-point stencil (u_{i+1}-u_{i-1})/(2h),
    homogeneous Dirichlet, n interior nodes, h = 1/(n+1)."""
    h = 1.0 / (n + 1)
    A = np.zeros((n, n), order="F")
    i = np.arange(n)
    A[i[:-1], i[:-1] + 1] = 1.0
    A[i[1:], i[1:] - 1] = -1.0
    return A / (2.0 * h)


def fd_dxx_neumann(n: int) -> np.ndarray:
    """Second derivative, 3-point stencil, homogeneous Neumann by ghost-point
    reflection, n nodes including both boundary nodes, h = 1/(n-1)."""
    h = 1.0 / (n - 1)
    A = np.zeros((n, n), order="F")
    i = np.arange(n)
    A[i, i] = -2.0
    A[i[:-1], i[:-1] + 1] = 1.0
    A[i[1:], i[1:] - 1] = 1.0
    A[0, 1] = 2.0
    A[n - 1, n - 2] = 2.0
    return A / (h * h)


def as_flat(T: np.ndarray) -> np.ndarray:
    """Tensor (n_1,…,n_d) -> vec(T) (column-major flatten, §2)."""
    return np.asarray(T).reshape(-1, order="F")


def from_flat(x: np.ndarray, dims: Sequence[int]) -> np.ndarray:
    """vec^{-1}: flat column-major vector -> tensor of shape dims."""
    return np.asarray(x).reshape(tuple(dims), order="F")


def uniform_tensor(dims: Sequence[int], lo: float, hi: float, seed: int) -> np.ndarray:
    """Seeded U[lo,hi] tensor of shape dims (Fortran order, float64)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N = int(np.prod(dims))
    return from_flat(rng.uniform(lo, hi, size=N), dims)


def normal_tensor(dims: Sequence[int], scale: float, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    N = int(np.prod(dims))
    return from_flat(scale * rng.standard_normal(size=N), dims)


# ---------------------------------------------------------------------------
# BASELINE.json configs -> concrete problems
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class Problem:
    """One φ-action request: K = tau*(A_d ⊕ … ⊕ A_1) applied to vectors.

    mode "same": compute φ_ℓ(τK)v for ℓ in ells, on the single vector vs[0]
                 (§3.1, formula (6)).
    mode "lincomb": compute Σ_{ℓ in ells} φ_ℓ(τK) v_ℓ (§3.2,
                 formula (7)); vs[i] pairs with ells[i].
    n_scales: outputs at τ/2^j, j = 0..n_scales-1 (Eq. (13)/(19)).
    """

    name: str
    dims: Tuple[int, ...]
    A: List[np.ndarray]          # factor matrices A_μ (μ = 1..d), unscaled by tau
    tau: float
    mode: str
    ells: Tuple[int, ...]
    vs: List[np.ndarray]         # tensors of shape dims
    n_scales: int = 1


@dataclasses.dataclass
class Workload:
    """A config = one or more independent problems (block-diagonal K̂, §4.4)."""

    name: str
    problems: List[Problem]


def config(idx: int, small: bool = False, with_vectors: bool = True) -> Workload:
    """BASELINE.json configs[idx].  small=True shrinks the grid (same operator
    family, same recipe) so the oracle finishes in seconds — used by the
    parity tests; the full sizes are the bench / sampled-parity workloads."""
    if idx == 0:
        n = 32
        A = fd_dxx_dirichlet(n)
        v = uniform_tensor((n, n), -1.0, 1.0, seed=0)
        p = Problem("cfg0_d2_n32_lap_dirichlet", (n, n), [A, A.copy()], 1e-3,
                    "same", (0, 1, 2, 3), [v], 1)
        return Workload("cfg0", [p])
    if idx == 1:
        n = 64 if small else 512
        eps, alpha = 1.0, (10.0, -5.0)
        A = [eps * fd_dxx_dirichlet(n) + a * fd_dx_dirichlet(n) for a in alpha]
        vs = _uniform_list((n, n), 4, -1.0, 1.0, seed=1)
        p = Problem(f"cfg1_d2_n{n}_adr_lincomb", (n, n), A, 1e-4, "lincomb",
                    (0, 1, 2, 3), vs, 1)
        return Workload("cfg1", [p])
    if idx == 2:
        n = 24 if small else 128
        eps = 0.01
        A = eps * fd_dxx_neumann(n)
        v = normal_tensor((n, n, n), 0.05, seed=2)
        p = Problem(f"cfg2_d3_n{n}_allen_cahn", (n, n, n), [A, A.copy(), A.copy()],
                    1e-2, "same", (1, 2), [v], 4)
        return Workload("cfg2", [p])
    if idx == 3:
        n = 24 if small else 256
        probs = []
        # one vector per species of the block-diagonal Brusselator operator
        rng_vs = _uniform_list((n, n, n), 2, 0.0, 3.0, seed=3)
        for sp, (D, v) in enumerate(zip((2e-3, 1e-3), rng_vs)):
            A = D * fd_dxx_neumann(n)
            probs.append(Problem(f"cfg3_d3_n{n}_brusselator_species{sp}", (n, n, n),
                                 [A, A.copy(), A.copy()], 5e-3, "same", (0, 1, 2), [v], 1))
        return Workload("cfg3", probs)
    if idx == 4:
        dims = (24, 24, 16) if small else (512, 512, 256)
        eps, alpha = 1.0, (10.0, 10.0, -10.0)
        A = [eps * fd_dxx_dirichlet(nm) + a * fd_dx_dirichlet(nm) for nm, a in zip(dims, alpha)]
        vs = _uniform_list(dims, 5, -1.0, 1.0, seed=4) if with_vectors else []
        p = Problem(f"cfg4_d3_{dims[0]}x{dims[1]}x{dims[2]}_adr_etdrk4", tuple(dims), A, 1e-4,
                    "lincomb", (0, 1, 2, 3, 4), vs, 1)
        return Workload("cfg4", [p])
    raise ValueError(f"no config {idx}")


def _uniform_list(dims, count, lo, hi, seed):
    """`count` tensors drawn consecutively from one seeded stream."""
    rng = np.random.Generator(np.random.PCG64(seed))
    N = int(np.prod(dims))
    return [from_flat(rng.uniform(lo, hi, size=N), dims) for _ in range(count)]


def random_factors(dims: Sequence[int], seed: int, scale: float = 1.0,
                   complex_: bool = False) -> List[np.ndarray]:
    """Dense random factor matrices A_μ with ||A_μ||_1 ≈ scale (test inputs)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for n in dims:
        M = rng.standard_normal((n, n))
        if complex_:
            M = M + 1j * rng.standard_normal((n, n))
        M = M * (scale / max(np.abs(M).sum(axis=0).max(), 1e-300))
        out.append(np.asfortranarray(M))
    return out


def random_tensor(dims: Sequence[int], seed: int, complex_: bool = False) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    N = int(np.prod(dims))
    x = rng.uniform(-1.0, 1.0, size=N)
    if complex_:
        x = x + 1j * rng.uniform(-1.0, 1.0, size=N)
    return from_flat(x, dims)
