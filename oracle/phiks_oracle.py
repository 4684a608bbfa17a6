"""PHIKS oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function cites the PAPER.md passage it follows (line numbers refer to
/root/reference/PAPER.md).  No blocking, fusion or reordering beyond what the
paper states; library primitives (numpy tensordot / matmul, numpy.linalg
norms) serve as single steps.

Pins (tests/test_oracle_*.py, all `-m "not gpu"`):
  mu_mode_product / tucker ... pure-Python triple loop on tiny inputs, explicit
                               Kronecker-matrix product
  expm_taylor ................ diagonal closed form, nilpotent Jordan closed
                               form, scipy.linalg.expm (Padé, independent)
  gll_rule ................... closed forms q=2..5, exactness degree 2q-3
  kernel_kq .................. closed form for q=2; Hermite contour formula
                               reproduces the true quadrature error
  range_rectangle ............ contains every Rayleigh quotient / eigenvalue
  remainder_bound ............ dominates the true scalar quadrature error
  select_plan ................ PAPER.md Table 1 (l.1416-1449) values of s, q, T
  phiks_same / phiks_lincomb . dense brute force (augmented-matrix exponential,
                               PAPER.md l.337-351), scalar closed forms
                               phi_1(z)=(e^z-1)/z and the phi recurrence,
                               diagonal A_mu (factorising), K = 0.
No function here is "parity unpinned".
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# Tensor algebra (§2, l.240-270)
# ---------------------------------------------------------------------------


def mu_mode_product(T: np.ndarray, M: np.ndarray, mu: int) -> np.ndarray:
    """μ-mode product T ×_μ M ("×_μ is the so-called μ-mode
    product"): result[i_1..j..i_d] = Σ_k M[j,k] T[i_1..k..i_d].
    `mu` is the 0-based axis (paper's μ = mu+1).  One matmul (tensordot)."""
    out = np.tensordot(M, T, axes=([1], [mu]))  # axis 0 of out is j
    return np.moveaxis(out, 0, mu)


def tucker(T: np.ndarray, mats: Sequence[np.ndarray]) -> np.ndarray:
    """Tucker operator T ×_1 M_1 ×_2 M_2 … ×_d M_d (Eq. (4), l.242-246)."""
    for mu, M in enumerate(mats):
        T = mu_mode_product(T, M, mu)
    return T


# ---------------------------------------------------------------------------
# Small-matrix exponential (§4 l.974-978 delegates to a standard
# scaling-and-squaring routine; the oracle uses the plainest one: Taylor).
# ---------------------------------------------------------------------------


def norm1(X: np.ndarray) -> float:
    return float(np.abs(X).sum(axis=0).max()) if X.size else 0.0


def expm_taylor(X: np.ndarray) -> np.ndarray:
    """exp(X) by scaling and squaring with a Taylor series:
    Y = X/2^σ with ||Y||_1 ≤ 1/2, exp(Y) = Σ_k Y^k/k! summed until the term
    is below 2^-60 of the sum, then σ squarings."""
    n = X.shape[0]
    nrm = norm1(X)
    sigma = 0 if nrm <= 0.5 else int(math.ceil(math.log2(nrm / 0.5)))
    Y = X / (2.0 ** sigma)
    E = np.eye(n, dtype=np.result_type(X, np.float64))
    term = E.copy()
    for k in range(1, 200):
        term = term @ Y / k
        E = E + term
        if norm1(term) <= 2.0 ** -60 * max(norm1(E), 1e-300):
            break
    for _ in range(sigma):
        E = E @ E
    return E


# ---------------------------------------------------------------------------
# Gauss–Lobatto–Legendre rule on [0,1] (§3.3 l.943-956)
# ---------------------------------------------------------------------------


def gll_rule(q: int) -> Tuple[np.ndarray, np.ndarray]:
    """q-point Gauss–Lobatto–Legendre nodes θ_1=0 < … < θ_q=1 and weights on
    [0,1].  Interior nodes: roots of P'_{q-1} (numpy Legendre series roots,
    polished by Newton); weights 2/(q(q-1) P_{q-1}(x_i)^2) on [-1,1], then
    mapped affinely."""
    if q < 2:
        raise ValueError("GLL needs q >= 2")
    L = np.polynomial.legendre.Legendre.basis(q - 1)
    dL = L.deriv()
    d2L = dL.deriv()
    if q > 2:
        xi = np.sort(np.real(dL.roots()))
        for _ in range(5):
            xi = xi - dL(xi) / d2L(xi)
        x = np.concatenate([[-1.0], xi, [1.0]])
    else:
        x = np.array([-1.0, 1.0])
    w = 2.0 / (q * (q - 1) * L(x) ** 2)
    return (x + 1.0) / 2.0, w / 2.0


def nodal_poly(nodes: np.ndarray, z: np.ndarray) -> np.ndarray:
    """π_q(z) = Π_i (z − θ_i), the monic nodal polynomial."""
    z = np.asarray(z)
    out = np.ones(z.shape, dtype=np.complex128)
    for t in nodes:
        out = out * (z - t)
    return out


_GL_CACHE: Dict[int, Tuple[np.ndarray, np.ndarray]] = {}


def _gauss_legendre01(m: int):
    if m not in _GL_CACHE:
        x, w = np.polynomial.legendre.leggauss(m)
        _GL_CACHE[m] = ((x + 1.0) / 2.0, w / 2.0)
    return _GL_CACHE[m]


def kernel_kq(nodes: np.ndarray, z: np.ndarray, m_gl: int = 256) -> np.ndarray:
    """k_q(z) = ∫_0^1 π_q(t) / (π_q(z)(z − t)) dt,
    numerator integral by an m_gl-point Gauss–Legendre rule on [0,1]
    (z must lie off [0,1]; on Γ_r the rule converges like (4r)^(-2 m_gl))."""
    z = np.asarray(z, dtype=np.complex128)
    t, wt = _gauss_legendre01(m_gl)
    pit = nodal_poly(nodes, t).real
    num = (wt * pit)[None, :] / (z.reshape(-1, 1) - t[None, :])
    return (num.sum(axis=1) / nodal_poly(nodes, z.reshape(-1))).reshape(z.shape)


# ---------------------------------------------------------------------------
# Numerical-range rectangle (PAPER.md l.925-940 and the Remark l.582-603)
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class Rect:
    """Ξ = center + [−hr, hr] + i[−hi, hi] (a rectangle in C)."""

    center: complex
    hr: float
    hi: float

    def scaled(self, f: float) -> "Rect":
        return Rect(self.center * f, self.hr * f, self.hi * f)

    def boundary(self, n_side: int) -> np.ndarray:
        """n_side points per side (corners included once per side start)."""
        c, a, b = self.center, self.hr, self.hi
        s = np.linspace(0.0, 1.0, n_side, endpoint=False)
        corners = [complex(-a, -b), complex(a, -b), complex(a, b), complex(-a, b)]
        pts = []
        for k in range(4):
            p0, p1 = corners[k], corners[(k + 1) % 4]
            pts.append(p0 + s * (p1 - p0))
        return c + np.concatenate(pts)


def range_rectangle(factors: Sequence[np.ndarray]) -> Rect:
    """Rectangle Ξ = Ξ_1 + … + Ξ_d ⊇ W(K) = W(A_1)+…+W(A_d).
    Per factor (reading R1): shift by σ_μ = trace(A_μ)/n_μ (Remark,
    l.598-602), then Ξ_μ = σ_μ + [−||H_μ||_2, ||H_μ||_2] + i[−||S_μ||_2, ||S_μ||_2]
    with H_μ, S_μ the Hermitian / skew-Hermitian parts of A_μ − σ_μ I
    ("norms of the Hermitian and the skew-Hermitian parts", l.933-935)."""
    center = 0j
    hr = hi = 0.0
    for A in factors:
        n = A.shape[0]
        sig = complex(np.trace(A)) / n
        B = A - sig * np.eye(n)
        H = (B + B.conj().T) / 2.0
        S = (B - B.conj().T) / 2.0
        center += sig
        hr += float(np.linalg.norm(H, 2))
        hi += float(np.linalg.norm(S, 2))
    return Rect(center, hr, hi)


# ---------------------------------------------------------------------------
# Remainder bound (§3.3 Eq. (21), l.905-960) and plan (l.809-875)
# ---------------------------------------------------------------------------

R_GRID = tuple(float(r) for r in np.geomspace(0.3, 6.0, 16))   # reading R3
N_SIDE = 32                                                    # reading R4
Q_MIN, Q_MAX, S_MAX = 2, 12, 60                                # reading R5
W_CAP = 256.0   # reading R5: scales with max|w| > W_CAP are infeasible for q ≤ Q_MAX
SPECTRAL_SET_C = 1.0 + math.sqrt(2.0)                          # l.908 [CP17]


def n_zeta_for(r: float, wmax: float) -> int:
    """Trapezoid resolution for the ζ-integral (reading R3): power of two
    ≥ 2(|w|_max (r + 1/(16r) + 1/2) + 64), clamped to [128, 4096]."""
    need = 2.0 * (wmax * (r + 1.0 / (16.0 * r) + 0.5) + 64.0)
    n = 128
    while n < need and n < 4096:
        n *= 2
    return n


def ellipse(r: float, nz: int):
    """Γ_r: z(ζ) = r e^{iζ} + 1/2 + e^{−iζ}/(16r), and the factor
    (r e^{iζ} − e^{−iζ}/(16r)) of the parametrised integral (l.886-902)."""
    zeta = 2.0 * np.pi * np.arange(nz) / nz
    e = np.exp(1j * zeta)
    z = r * e + 0.5 + 1.0 / (16.0 * r * e)
    dz = r * e - 1.0 / (16.0 * r * e)
    return z, dz


_KQ_CACHE: Dict[Tuple[int, float, int], np.ndarray] = {}


def _kq_on_ellipse(q: int, r: float, nz: int) -> np.ndarray:
    """k_q at the nz trapezoid points of Γ_r (memoised; depends on q, r, nz only)."""
    key = (q, r, nz)
    if key not in _KQ_CACHE:
        _KQ_CACHE[key] = kernel_kq(gll_rule(q)[0], ellipse(r, nz)[0])
    return _KQ_CACHE[key]


def remainder_bounds(rect: Rect, ells: Sequence[int], qs: Sequence[int],
                     r_grid: Sequence[float] = R_GRID, n_side: int = N_SIDE) -> np.ndarray:
    """B[qi, li] = estimate of ||R_q(f_ℓ(·, X))||_2 for X with W(X) ⊆ rect,
    following Eq. (21) l.910-920: (1+√2)/(2π) sup_{w∈∂Ξ} |∫_0^{2π} k_q(z) f_ℓ(z,w)
    (r e^{iζ} − e^{−iζ}/(16r)) dζ|, sup over sampled boundary points (maximum
    modulus principle, l.938-940), ζ-integral by the trapezoidal rule (l.941),
    minimised over r ∈ r_grid (any r > 1/4 gives a valid bound, l.883).
    f_ℓ(z,w) = z^{ℓ−1}/(ℓ−1)! e^{(1−z)w} (Eq. (2), l.80)."""
    w = rect.boundary(n_side)
    wmax = float(np.abs(w).max())
    best = np.full((len(qs), len(ells)), np.inf)
    if wmax > W_CAP:
        return best
    with np.errstate(over="ignore", invalid="ignore"):
        for r in r_grid:
            nz = n_zeta_for(r, wmax)
            z, dz = ellipse(r, nz)
            E = np.exp(np.outer(1.0 - z, w))                     # (nz, nb)
            kq = np.stack([_kq_on_ellipse(q, r, nz) for q in qs])  # (nq, nz)
            base = kq * dz[None, :]
            for li, ell in enumerate(ells):
                g = base * (z ** (ell - 1) / math.factorial(ell - 1))[None, :]
                vals = np.abs(g @ E).max(axis=1) * SPECTRAL_SET_C / nz
                vals = np.where(np.isfinite(vals), vals, np.inf)
                best[:, li] = np.minimum(best[:, li], vals)
    return best


@dataclasses.dataclass
class Plan:
    s: int
    q: int
    T: int


def tucker_count(mode: str, s: int, s_hat: int, q: int, p: int) -> int:
    """T(s,ŝ,q,p): Eq. (14) q+sp+ŝ (same vector, l.618-620) or Eq. (19)
    qp+sp+ŝ (linear combination, l.775-778)."""
    return (q + s * p + s_hat) if mode == "same" else (q * p + s * p + s_hat)


def tucker_executed(mode: str, s: int, q: int, ells: Sequence[int], n_scales: int,
                    has_v0: bool = False) -> int:
    """Tucker operators phiks_same / phiks_lincomb below actually run (reading R9):
    θ_q = 1 costs none (l.948-952); at the last squaring step j = 1 only the
    combinations that are outputs are formed (l.953-956 "few other
    shrewdnesses"): Ψ_p alone for a linear combination, the requested φ_ℓ for
    the same vector.  Linear combination without v_0, ŝ = 1:
    (q−2)p + sp + 1, the T of PAPER.md Table 1 (l.1436-1446)."""
    p = max(ells)
    if p == 0:
        return n_scales if (mode == "same" or has_v0) else 0
    last = (sum(1 for e in ells if e >= 1) if mode == "same" else 1)
    if mode == "same":
        quad = q - 1
        sq = (s - 1) * p + last if s >= 1 else 0
        return quad + sq + (n_scales if 0 in ells else 0)
    quad = (q - 1) * (p if s >= 1 else 1)
    sq = (s - 1) * p + last if s >= 1 else 0
    return quad + sq + (n_scales if has_v0 else 0)


def q_for_s(mode: str, rect: Rect, p: int, norms: Sequence[float], delta: float, s: int,
            q_min: int = Q_MIN, q_max: int = Q_MAX) -> Optional[int]:
    """Smallest q ∈ [q_min, q_max] meeting the §3.3 criterion at scaling s
    (None if none does).
    same:    ||R_q(f_ℓ(·,K/2^s))|| ||v|| ≤ δ 2^{ℓs}, ℓ=1..p (l.815-826)
    lincomb: Σ_{k=1}^ℓ ||R_q(f_{ℓ−k+1}(·,K/2^s))|| ||v_{p+1−k}|| / 2^{(ℓ−k+1)s} ≤ δ,
             ℓ=1..p (l.854-866); norms[k-1] = ||v_k||."""
    qs = list(range(q_min, q_max + 1))
    ells = list(range(1, p + 1))
    B = remainder_bounds(rect.scaled(2.0 ** -s), ells, qs)  # (nq, p)
    ok = np.ones(len(qs), dtype=bool)
    for li, ell in enumerate(ells):
        if mode == "same":
            ok &= B[:, li] * norms[0] <= delta * 2.0 ** (ell * s)
        else:
            acc = np.zeros(len(qs))
            for k in range(1, ell + 1):
                acc = acc + B[:, ell - k] * norms[p - k] / 2.0 ** ((ell - k + 1) * s)
            ok &= acc <= delta
    idx = np.nonzero(ok)[0]
    return None if idx.size == 0 else qs[int(idx[0])]


def select_plan(mode: str, rect: Rect, p: int, norms: Sequence[float], delta: float,
                s_hat: int, s_min: int = 0, q_min: int = Q_MIN, q_max: int = Q_MAX,
                s_max: int = S_MAX) -> Plan:
    """Choice of s and q (§3.3 l.809-875): for s = s_min, s_min+1, …
    take the smallest admissible q (q_for_s); stop as soon as the Tucker count
    T(s+1) of Eq. (14)/(19) is larger than T(s) and return the s-plan
    (l.830-834, l.867-871; reading R6)."""
    if p == 0:
        return Plan(max(s_min, 0), 0, tucker_count(mode, max(s_min, 0), s_hat, 0, 0))
    prev: Optional[Plan] = None
    for s in range(s_min, s_max + 1):
        q = q_for_s(mode, rect, p, norms, delta, s, q_min, q_max)
        if q is None:
            continue
        cur = Plan(s, q, tucker_count(mode, s, s_hat, q, p))
        if prev is not None and cur.T > prev.T:
            return prev
        prev = cur
    if prev is None:
        raise RuntimeError("plan search exhausted")
    return prev


# ---------------------------------------------------------------------------
# PHIKS (§3.1 Eqs. (11)-(13) and §3.2 Eqs. (17)-(18))
# ---------------------------------------------------------------------------


@dataclasses.dataclass
class Result:
    plan: Plan
    out: Dict                 # same: (ell, j) -> tensor ; lincomb: j -> tensor
    tucker_ops: int


def _node_exponentials(Aq: Sequence[np.ndarray], theta: np.ndarray, s: int):
    """exp((1−θ_i) A_μ / 2^s) for every node and every μ (l.513-517);
    θ = 1 gives the identity and no Tucker operator is formed for it (l.948-952)."""
    return [[expm_taylor((1.0 - th) * A / 2.0 ** s) for A in Aq] if th != 1.0 else None
            for th in theta]


def phiks_same(A: Sequence[np.ndarray], tau: float, V: np.ndarray, ells: Sequence[int],
               n_scales: int, plan: Plan) -> Result:
    """φ_ℓ(τK/2^j) v for ℓ ∈ ells, j = 0..n_scales−1 (§3.1).
    Quadrature Eq. (11) l.547-552 at the scaled matrix τK/2^s, squaring
    Eq. (12) l.554-563 for j = s..1, ℓ = p..1, intermediate scales Eq. (13)
    l.570-580; exp(τK/2^j)v by one Tucker operator each (l.614-616)."""
    Aq = [tau * a for a in A]
    p = max(ells)
    s = plan.s
    assert s >= n_scales - 1
    ops = 0
    out: Dict = {}
    # exp(A_μ/2^j) for j = s..0 via the squaring relation (l.561)
    Es = {s: [expm_taylor(a / 2.0 ** s) for a in Aq]}
    for j in range(s, 0, -1):
        Es[j - 1] = [E @ E for E in Es[j]]
    if p >= 1:
        theta, w = gll_rule(plan.q)
        nodeE = _node_exponentials(Aq, theta, s)
        phi = [None] + [np.zeros_like(V, dtype=np.result_type(V, Aq[0])) for _ in range(p)]
        for i in range(plan.q):
            if nodeE[i] is None:
                TV = V
            else:
                TV = tucker(V, nodeE[i])
                ops += 1
            for ell in range(1, p + 1):
                phi[ell] = phi[ell] + w[i] * theta[i] ** (ell - 1) / math.factorial(ell - 1) * TV
        if s <= n_scales - 1:
            for ell in ells:
                if ell >= 1:
                    out[(ell, s)] = phi[ell]
        for j in range(s, 0, -1):
            new = [None] * (p + 1)
            for ell in range(p, 0, -1):
                if j == 1 and ell not in ells:
                    continue          # level 0 is output only (l.953-956)
                acc = tucker(phi[ell], Es[j])
                ops += 1
                for k in range(1, ell + 1):
                    acc = acc + phi[k] / math.factorial(ell - k)
                new[ell] = acc / 2.0 ** ell
            phi = new
            if j - 1 <= n_scales - 1:
                for ell in ells:
                    if ell >= 1:
                        out[(ell, j - 1)] = phi[ell]
    if 0 in ells:
        for j in range(n_scales):
            out[(0, j)] = tucker(V, Es[j])
            ops += 1
    return Result(plan, out, ops)


def lincomb_nodes_input(theta_i: float, vs: Dict[int, np.ndarray], p: int, s: int, ell: int,
                        zero: np.ndarray) -> np.ndarray:
    """Σ_{k=1}^ℓ θ_i^{ℓ−k}/(ℓ−k)! v_{p+1−k} / 2^{(ℓ−k+1)s} (Eq. (17), l.727-732)."""
    acc = zero
    for k in range(1, ell + 1):
        v = vs.get(p + 1 - k)
        if v is None:
            continue
        acc = acc + theta_i ** (ell - k) / math.factorial(ell - k) * v / 2.0 ** ((ell - k + 1) * s)
    return acc


def phiks_lincomb(A: Sequence[np.ndarray], tau: float, vs: Dict[int, np.ndarray],
                  n_scales: int, plan: Plan) -> Result:
    """exp(τK/2^j) v_0 + Σ_{ℓ=1}^p φ_ℓ(τK/2^j) v_ℓ / 2^{ℓj}, j = 0..n_scales−1
    (§3.2: Φ_j notation l.642-648, quadrature Eq. (17) l.726-733,
    squaring Eq. (18) l.734-746, scales Eq. (19) l.757-761).
    Internally Ψ_ℓ^{(j)} = Φ_j(K) v_{p−ℓ+1,…,p} ("suffix" combinations)."""
    Aq = [tau * a for a in A]
    p = max(vs.keys())
    s = plan.s
    assert s >= n_scales - 1
    ops = 0
    any_v = next(iter(vs.values()))
    zero = np.zeros_like(any_v, dtype=np.result_type(any_v, Aq[0]))
    Es = {s: [expm_taylor(a / 2.0 ** s) for a in Aq]}
    for j in range(s, 0, -1):
        Es[j - 1] = [E @ E for E in Es[j]]
    psi_at: Dict[int, List] = {}
    if p >= 1:
        theta, w = gll_rule(plan.q)
        nodeE = _node_exponentials(Aq, theta, s)
        psi = [None] + [zero.copy() for _ in range(p)]
        for i in range(plan.q):
            for ell in range(1, p + 1):
                if s == 0 and ell != p:
                    continue          # only Ψ_p^{(0)} is an output (l.953-956)
                x = lincomb_nodes_input(theta[i], vs, p, s, ell, zero)
                if nodeE[i] is None:
                    Tx = x
                else:
                    Tx = tucker(x, nodeE[i])
                    ops += 1
                psi[ell] = psi[ell] + w[i] * Tx
        psi_at[s] = psi
        for j in range(s, 0, -1):
            new = [None] * (p + 1)
            for ell in range(p, 0, -1):
                if j == 1 and ell != p:
                    continue          # only Ψ_p^{(0)} is an output (l.953-956, Table 1 T)
                acc = tucker(psi[ell], Es[j])
                ops += 1
                for k in range(1, ell + 1):
                    acc = acc + psi[k] / (math.factorial(ell - k) * 2.0 ** ((ell - k) * j))
                new[ell] = acc
            psi = new
            psi_at[j - 1] = psi
    out: Dict = {}
    for j in range(n_scales):
        acc = zero.copy()
        if p >= 1:
            acc = acc + psi_at[j][p]
        if 0 in vs:
            acc = acc + tucker(vs[0], Es[j])
            ops += 1
        out[j] = acc
    return Result(plan, out, ops)


# ---------------------------------------------------------------------------
# Convenience: full request with the paper's plan selection
# ---------------------------------------------------------------------------


def relative_delta(tol: float, mode: str, norms: Sequence[float]) -> float:
    """Reading R2: the caller's relative tolerance tol becomes the
    absolute δ of §3.3 as δ = tol·||v|| (same vector) or tol·max_ℓ ||v_ℓ||
    (linear combination)."""
    return tol * (norms[0] if mode == "same" else max(norms))


def plan_for(A: Sequence[np.ndarray], tau: float, mode: str, ells: Sequence[int],
             vs: Sequence[np.ndarray], n_scales: int, tol: float = 2.0 ** -53) -> Plan:
    rect = range_rectangle([tau * a for a in A])
    p = max(ells)
    if mode == "same":
        norms = [float(np.linalg.norm(vs[0].ravel()))]
    else:
        d = dict(zip(ells, vs))
        norms = [float(np.linalg.norm(d[k].ravel())) if k in d else 0.0 for k in range(1, p + 1)]
    if p == 0 or max(norms) == 0.0:
        return Plan(max(n_scales - 1, 0), 0 if p == 0 else Q_MIN,
                    tucker_count(mode, max(n_scales - 1, 0), n_scales, 0 if p == 0 else Q_MIN, p))
    delta = relative_delta(tol, mode, norms)
    return select_plan(mode, rect, p, norms, delta, n_scales, s_min=max(n_scales - 1, 0))


def phiks(A, tau, mode, ells, vs, n_scales=1, tol=2.0 ** -53, plan: Optional[Plan] = None) -> Result:
    if plan is None:
        plan = plan_for(A, tau, mode, ells, vs, n_scales, tol)
    if mode == "same":
        return phiks_same(A, tau, vs[0], ells, n_scales, plan)
    return phiks_lincomb(A, tau, dict(zip(ells, vs)), n_scales, plan)
