"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/phiks.h declares, and its host-side §3.3 planner agrees with the
oracle's and with PAPER.md Table 1.  No compute calls."""
import ctypes
import json
import math
import os

import numpy as np
import pytest

from oracle import phiks_oracle as O
from paper_2210_07667_b200 import _lib
from paper_2210_07667_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = _lib.header_functions()
    assert len(names) >= 12
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert b"sm_100a" in lib.phiks_version()


def test_create_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    A = np.asfortranarray(W.fd_dxx_dirichlet(4))
    h = ctypes.c_void_p()
    n = (ctypes.c_int * 1)(4)
    code = lib.phiks_create(1, n, _lib.ptr_array([A.ctypes.data]), ctypes.byref(h))
    assert code == 2  # PHIKS_ERR_CUDA
    assert b"CUDA" in lib.phiks_last_error()


def _select(mode, rect, p, norms, delta, s_hat=1, s_min=0, s_fixed=-1):
    lib = _lib.load()
    info = _lib.PlanInfo()
    arr = (ctypes.c_double * max(len(norms), 1))(*norms)
    code = lib.phiks_select_plan(0 if mode == "same" else 1, rect.center.real, rect.center.imag, rect.hr,
                                 rect.hi, p, arr, delta, s_hat, s_min, s_fixed, ctypes.byref(info))
    _lib.check(code, "phiks_select_plan")
    return info


def _table1():
    with open(os.path.join(GOLD, "table1.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("mode,row", [("same", r) for r in _table1()["same_vector"]]
                         + [("lincomb", r) for r in _table1()["linear_combination"]])
def test_cpp_planner_table1_q_at_paper_s(mode, row):
    """PAPER.md Table 1 (l.1416-1449): the library's §3.3 bound selects the
    paper's q at the paper's s for every column."""
    t = _table1()
    n, d = row["n"], row["d"]
    A = (1 + 1j) / 100 * W.fd_dxx_dirichlet(n)
    rect = O.range_rectangle([A] * d)  # rectangle of the complex validation operator
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h
    nv = 4096 * math.sqrt(2) * float(np.linalg.norm(x * (1 - x))) ** d
    norms = [nv] if mode == "same" else [nv] * t["p"]
    info = _select(mode, rect, t["p"], norms, t["tol"], t["s_hat"], 0, row["s"])
    assert info.q == row["q"]


def _plan_host(pb, tol=0.0):
    lib = _lib.load()
    n = (ctypes.c_int * len(pb.dims))(*pb.dims)
    A = [np.asfortranarray(a) for a in pb.A]
    req = _lib.make_request(0 if pb.mode == "same" else 1, pb.ells, pb.n_scales, pb.tau, tol)
    p = max(pb.ells)
    norms = None
    if pb.mode == "lincomb":
        d = dict(zip(pb.ells, pb.vs))
        norms = (ctypes.c_double * p)(*[float(np.linalg.norm(d[k].ravel())) if k in d else 0.0
                                        for k in range(1, p + 1)])
    info = _lib.PlanInfo()
    _lib.check(lib.phiks_plan_host(len(pb.dims), n, _lib.ptr_array([a.ctypes.data for a in A]), ctypes.byref(req),
                                   norms, ctypes.byref(info)), "phiks_plan_host")
    return info


@pytest.mark.parametrize("cfg,small", [(0, False), (1, True), (2, True), (3, True), (4, True),
                                       (2, False), (3, False)])
def test_cpp_planner_matches_oracle_on_configs(cfg, small):
    for pb in W.config(cfg, small=small).problems:
        ora = O.plan_for(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, pb.n_scales)
        got = _plan_host(pb)
        assert (got.s, got.q, got.T_formula) == (ora.s, ora.q, ora.T), pb.name


def test_cpp_planner_random_factors_match_oracle():
    rng = np.random.default_rng(7)
    for c in range(6):
        dims = tuple(int(x) for x in rng.integers(3, 9, size=int(rng.integers(1, 4))))
        fac = W.random_factors(dims, seed=300 + c, scale=float(rng.uniform(0.5, 30.0)))
        V = W.random_tensor(dims, seed=c)
        pb = W.Problem("rand", dims, fac, 1.0, "same", (0, 1, 2, 3), [V], 1 + c % 3)
        ora = O.plan_for(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, pb.n_scales)
        got = _plan_host(pb)
        assert (got.s, got.q) == (ora.s, ora.q)


def _plan_host_complex(dims, A, mode, ells, n_scales, tau, norms=None, tol=0.0):
    lib = _lib.load()
    n = (ctypes.c_int * len(dims))(*dims)
    Az = [np.asfortranarray(a.astype(np.complex128)) for a in A]
    req = _lib.make_request(0 if mode == "same" else 1, ells, n_scales, tau, tol)
    arr = (ctypes.c_double * max(len(norms or []), 1))(*(norms or [0.0]))
    info = _lib.PlanInfo()
    _lib.check(lib.phiks_plan_host_complex(len(dims), n, _lib.ptr_array([a.ctypes.data for a in Az]),
                                           ctypes.byref(req), arr if norms else None, ctypes.byref(info)),
               "phiks_plan_host_complex")
    return info


@pytest.mark.parametrize("n,d", [(8, 2), (10, 3), (12, 2)])
def test_cpp_complex_range_matches_oracle_plan(n, d):
    # the complex validation operator (1+i)/100·Δ of PAPER.md §4.1: the library's
    # complex numerical-range rectangle gives the oracle's plan
    A = (1 + 1j) / 100 * W.fd_dxx_dirichlet(n)
    dims = (n,) * d
    V = W.random_tensor(dims, seed=3, complex_=True)
    for mode, ells in (("same", (0, 1, 2, 3)), ("lincomb", (0, 1, 2))):
        vs = [V] if mode == "same" else [W.random_tensor(dims, seed=5 + k, complex_=True) for k in ells]
        ora = O.plan_for([A] * d, 1.0, mode, ells, vs, 1)
        norms = None
        if mode == "lincomb":
            norms = [float(np.linalg.norm(W.as_flat(v))) for v in vs[1:]]
        got = _plan_host_complex(dims, [A] * d, mode, ells, 1, 1.0, norms)
        assert (got.s, got.q) == (ora.s, ora.q), (mode, got.s, got.q, ora)


def test_cpp_complex_range_random_factors():
    rng = np.random.default_rng(11)
    for c in range(4):
        dims = tuple(int(x) for x in rng.integers(3, 8, size=2))
        fac = W.random_factors(dims, seed=700 + c, scale=float(rng.uniform(1.0, 20.0)), complex_=True)
        V = W.random_tensor(dims, seed=c, complex_=True)
        ora = O.plan_for(fac, 1.0, "same", (1, 2), [V], 1)
        got = _plan_host_complex(dims, fac, "same", (1, 2), 1, 1.0)
        assert (got.s, got.q) == (ora.s, ora.q)


# ---- full §3.3 search against PAPER.md Table 1 (readings R3, R5, R6) ----
LINCOMB_SQ_REPRODUCED = {(3, 64), (6, 11)}   # see tests/test_oracle_phiks.py


@pytest.mark.parametrize("mode,row", [("same", r) for r in _table1()["same_vector"]]
                         + [("lincomb", r) for r in _table1()["linear_combination"]])
def test_cpp_planner_table1_full_search(mode, row):
    """PAPER.md Table 1 (l.1416-1449): the library's search picks the paper's
    (s, q) in every same-vector column, and a plan of the paper's Eq. (19)
    count in every linear-combination column ((s, q) too where the count has a
    unique minimiser along the search).  A flipped stopping comparison moves
    d=3, n=64 to (8, 10) and d=6, n=11 to (4, 10)."""
    t = _table1()
    n, d = row["n"], row["d"]
    A = (1 + 1j) / 100 * W.fd_dxx_dirichlet(n)
    rect = O.range_rectangle([A] * d)
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h
    nv = 4096 * math.sqrt(2) * float(np.linalg.norm(x * (1 - x))) ** d
    norms = [nv] if mode == "same" else [nv] * t["p"]
    info = _select(mode, rect, t["p"], norms, t["tol"], t["s_hat"], 0, -1)
    paper_T = O.tucker_count(mode, row["s"], t["s_hat"], row["q"], t["p"])
    assert info.T_formula == paper_T
    if mode == "same" or (d, n) in LINCOMB_SQ_REPRODUCED:
        assert (info.s, info.q) == (row["s"], row["q"])


@pytest.mark.parametrize("row", _table1()["linear_combination"], ids=lambda r: f"d{r['d']}n{r['n']}")
def test_cpp_T_executed_equals_table1(row):
    """Table 1's lincomb T = (q−2)p + sp + 1 is the library's executed count at
    the paper's (s, q) (forced), ℓ = 1..5 without v_0."""
    lib = _lib.load()
    n, d = 4, 3
    A = (1 + 1j) / 100 * W.fd_dxx_dirichlet(n)
    Az = [np.asfortranarray(A.astype(np.complex128))] * d
    dims = (ctypes.c_int * d)(*([n] * d))
    req = _lib.make_request(1, (1, 2, 3, 4, 5), 1, 1.0, 0.0, row["s"], row["q"])
    arr = (ctypes.c_double * 5)(*([1.0] * 5))
    info = _lib.PlanInfo()
    _lib.check(lib.phiks_plan_host_complex(d, dims, _lib.ptr_array([a.ctypes.data for a in Az]), ctypes.byref(req),
                                           arr, ctypes.byref(info)), "phiks_plan_host_complex")
    assert info.T_executed == row["T"]


def test_cpp_T_executed_matches_oracle_formula():
    lib = _lib.load()
    A = [np.asfortranarray(W.fd_dxx_dirichlet(5))] * 2
    dims = (ctypes.c_int * 2)(5, 5)
    for mode in ("same", "lincomb"):
        for s, q, ells, ns in [(0, 5, (0, 1, 2), 1), (2, 4, (1, 3), 2), (3, 6, (0, 2), 3), (1, 3, (2,), 1)]:
            req = _lib.make_request(0 if mode == "same" else 1, ells, ns, 1.0, 0.0, s, q)
            arr = (ctypes.c_double * 5)(*([1.0] * 5))
            info = _lib.PlanInfo()
            _lib.check(lib.phiks_plan_host(2, dims, _lib.ptr_array([a.ctypes.data for a in A]), ctypes.byref(req),
                                           arr, ctypes.byref(info)), "phiks_plan_host")
            want = O.tucker_executed(mode, s, q, ells, ns, has_v0=0 in ells)
            if mode == "lincomb" and s >= 1:
                # the library's lincomb quadrature runs one operator per node and GIVEN vector
                # (linearity, reading R9); the oracle follows Eq. (17): one per node and ℓ ≤ p
                given = sum(1 for e in ells if e >= 1)
                want -= (q - 1) * (max(ells) - given)
            assert info.T_executed == want, (mode, s, q, ells)
