"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Tolerance (BASELINE.json north_star): fp64 relative
2-norm error ≤ 1e-12 per output."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, expm, fp64_peak_launch, mode_product, tucker  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-12
DEV = "cuda:0"


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(W.as_flat(x))).to(DEV)


def mat(M):
    return torch.from_numpy(np.asfortranarray(M).reshape(-1, order="F").copy()).to(DEV)


def rel2(got, ref):
    ref = np.asarray(ref).ravel(order="F") if np.asarray(ref).ndim > 1 else np.asarray(ref)
    got = got.detach().cpu().numpy() if isinstance(got, torch.Tensor) else got
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


# ---------------------------------------------------------------- building blocks


@pytest.mark.parametrize("dims", [(7,), (32, 32), (33, 17), (5, 130, 3), (64, 3, 65), (2, 3, 4, 5), (1, 9, 1),
                                  (256, 40), (129, 2, 129),
                                  # large enough for the TMA/mbarrier path (n > 64, even strides)
                                  (256, 300), (130, 130, 40), (96, 200, 66), (100, 100, 70), (66, 258, 34)])
def test_mode_product_every_mode(dims):
    T = W.random_tensor(dims, seed=sum(dims))
    for mu, n in enumerate(dims):
        Ms = [np.random.default_rng(mu + 10 * k).standard_normal((n, n)) for k in range(2)]
        ins = [dev(T), dev(2.0 * T)]
        outs = [torch.empty_like(ins[0]) for _ in range(2)]
        mode_product(dims, mu, ins, [mat(M) for M in Ms], outs)
        torch.cuda.synchronize()
        for k in range(2):
            ref = O.mu_mode_product((1.0 + k) * T, Ms[k], mu)
            assert rel2(outs[k], W.as_flat(ref)) <= 1e-14, (dims, mu, k)


@pytest.mark.parametrize("dims", [(16, 16, 16), (31, 8, 45), (3, 3, 3, 3)])
def test_tucker_matches_oracle(dims):
    T = W.random_tensor(dims, seed=3)
    Ms = [np.random.default_rng(i).standard_normal((n, n)) for i, n in enumerate(dims)]
    out = torch.empty(int(np.prod(dims)), dtype=torch.float64, device=DEV)
    tucker(dims, dev(T), [mat(M) for M in Ms], out)
    assert rel2(out, W.as_flat(O.tucker(T, Ms))) <= 1e-14


@pytest.mark.parametrize("n,scale,c", [(4, 1.0, 1.0), (32, 30.0, 0.37), (65, 400.0, 1.0), (256, 5e3, 0.01),
                                       (300, 2.0, -1.0)])
def test_expm_matches_oracle(n, scale, c):
    A = W.random_factors([n], seed=n, scale=scale)[0]
    E = expm(mat(A), c)
    ref = O.expm_taylor(c * A)
    err = np.abs(E.cpu().numpy().reshape(n, n, order="F") - ref).sum(axis=0).max() / max(O.norm1(ref), 1.0)
    assert err <= 1e-12


def test_expm_fd_operator():
    A = 1e-4 * (W.fd_dxx_dirichlet(512) + 10 * W.fd_dx_dirichlet(512))
    E = expm(mat(A), 0.25)
    ref = O.expm_taylor(0.25 * A)
    assert rel2(E, W.as_flat(ref)) <= 1e-13


def test_fp64_peak_kernel_runs():
    sink = torch.empty(148 * 256, dtype=torch.float64, device=DEV)
    for kind in (0, 1):
        fl = fp64_peak_launch(kind, 148, 100, sink)
        torch.cuda.synchronize()
        assert fl > 0 and torch.isfinite(sink).all()


# ---------------------------------------------------------------- φ-actions


def _run(pb, force=True, n_scales=None):
    n_scales = pb.n_scales if n_scales is None else n_scales
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=n_scales)
    op = PhiKS(pb.A)
    kw = dict(force_s=ref.plan.s, force_q=ref.plan.q) if force else {}
    outs = op.apply(pb.tau, pb.ells, [dev(v) for v in pb.vs], mode=pb.mode, n_scales=n_scales, **kw)
    torch.cuda.synchronize()
    return op, ref, outs


def _compare(pb, ref, outs, n_scales):
    worst = 0.0
    for j in range(n_scales):
        if pb.mode == "same":
            for i, ell in enumerate(pb.ells):
                e = rel2(outs[j * len(pb.ells) + i], W.as_flat(ref.out[(ell, j)]))
                assert e <= TOL, (pb.name, ell, j, e)
                worst = max(worst, e)
        else:
            e = rel2(outs[j], W.as_flat(ref.out[j]))
            assert e <= TOL, (pb.name, j, e)
            worst = max(worst, e)
    return worst


@pytest.mark.parametrize("cfg,small", [(0, False), (1, True), (2, True), (3, True), (4, True)])
def test_configs_small_parity(cfg, small):
    for pb in W.config(cfg, small=small).problems:
        op, ref, outs = _run(pb, force=False)
        st = op.stats()
        assert (st["s"], st["q"]) == (ref.plan.s, ref.plan.q), pb.name   # library's own §3.3 plan
        _compare(pb, ref, outs, pb.n_scales)
        assert st["tucker_ops"] == ref.tucker_ops


def _random_cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    for c in range(n):
        d = int(rng.integers(1, 5))
        dims = tuple(int(x) for x in rng.integers(1, 40 if d <= 2 else 14, size=d))
        fac = W.random_factors(dims, seed=500 + c, scale=float(rng.uniform(0.1, 20.0)))
        mode = "same" if c % 2 == 0 else "lincomb"
        p = int(rng.integers(0, 7))
        ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
        nsc = int(rng.integers(1, 4))
        vs = [W.random_tensor(dims, seed=900 + 7 * c + k) for k in range(1 if mode == "same" else len(ells))]
        out.append(W.Problem(f"rand{c}_{mode}_d{d}", dims, fac, float(rng.uniform(0.05, 2.0)), mode, ells, vs, nsc))
    return out


@pytest.mark.parametrize("pb", _random_cases(16, 42), ids=lambda pb: pb.name)
def test_random_problems_parity(pb):
    op, ref, outs = _run(pb, force=True)
    _compare(pb, ref, outs, pb.n_scales)


def test_host_memory_path_equals_device_path():
    pb = W.config(2, small=True).problems[0]
    op = PhiKS(pb.A)
    d_outs = op.apply(pb.tau, pb.ells, [dev(pb.vs[0])], n_scales=pb.n_scales)
    h_outs = op.apply(pb.tau, pb.ells, [np.asfortranarray(pb.vs[0])], n_scales=pb.n_scales)
    torch.cuda.synchronize()
    for a, b in zip(d_outs, h_outs):
        assert np.array_equal(a.cpu().numpy(), b)


def test_graph_replay_is_bitwise_identical():
    # the second apply on the same buffers replays the captured CUDA graph
    for pb in (W.config(0).problems[0], W.config(1, small=True).problems[0]):
        op = PhiKS(pb.A)
        vs = [dev(v) for v in pb.vs]
        outs = [torch.empty(op.N, dtype=torch.float64, device=DEV) for _ in range(len(pb.ells) if pb.mode == "same"
                                                                                 else 1)]
        first = [o.cpu().numpy().copy() for o in op.apply(pb.tau, pb.ells, vs, mode=pb.mode, outs=outs)]
        for o in outs:
            o.zero_()
        again = [o.cpu().numpy() for o in op.apply(pb.tau, pb.ells, vs, mode=pb.mode, outs=outs)]
        fresh = [o.cpu().numpy() for o in op.apply(pb.tau, pb.ells, vs, mode=pb.mode)]
        for a, b, c in zip(first, again, fresh):
            assert np.array_equal(a, b) and np.array_equal(a, c)


def test_host_async_path_equals_device_path():
    # PHIKS_MEM_HOST_ASYNC: pinned buffers, copies on the handle's streams, two
    # handles in flight (the bench's e2e pattern), then wait()
    pbs = W.config(3, small=True).problems
    ops = [PhiKS(pb.A) for pb in pbs]
    pins, pouts, ref = [], [], []
    for op, pb in zip(ops, pbs):
        x = W.as_flat(pb.vs[0])
        hi = torch.empty(x.size, dtype=torch.float64, pin_memory=True)
        hi.numpy()[:] = x
        pins.append(hi)
        pouts.append([torch.empty(x.size, dtype=torch.float64, pin_memory=True) for _ in pb.ells])
        ref.append([o.cpu().numpy() for o in op.apply(pb.tau, pb.ells, [dev(pb.vs[0])])])
    for rep in range(2):
        for op, pb, hi, ho in zip(ops, pbs, pins, pouts):
            op.apply(pb.tau, pb.ells, [hi.numpy()], outs=[t.numpy() for t in ho], host_async=True)
        for op in ops:
            op.wait()
        for ho, r in zip(pouts, ref):
            for a, b in zip(ho, r):
                assert np.array_equal(a.numpy(), b)


def test_edge_cases():
    # n_μ = 1 everywhere (N = 1): scalar K = Σ a_μ
    fac = [np.array([[-0.3]]), np.array([[0.7]])]
    V = np.array([[2.0]])
    pb = W.Problem("scalar", (1, 1), fac, 1.0, "same", (0, 1, 2, 3), [V], 2)
    op, ref, outs = _run(pb)
    _compare(pb, ref, outs, 2)
    z = 0.4
    assert abs(outs[1].item() - 2.0 * (math.exp(z) - 1) / z) <= 1e-14 * 2
    # K = 0: φ_ℓ(0)v = v/ℓ!
    fac = [np.zeros((3, 3)), np.zeros((4, 4))]
    V = W.random_tensor((3, 4), seed=1)
    pb = W.Problem("zero", (3, 4), fac, 1.0, "same", (0, 1, 2, 3, 4, 5, 6), [V], 1)
    op, ref, outs = _run(pb)
    for i in range(7):
        assert rel2(outs[i], W.as_flat(V) / math.factorial(i)) <= 1e-15
    # zero vector
    pb = W.Problem("zerov", (5, 6), W.random_factors((5, 6), seed=2, scale=3.0), 1.0, "lincomb", (0, 1, 2),
                   [np.zeros((5, 6))] * 3, 1)
    op = PhiKS(pb.A)
    out = op.apply(1.0, (0, 1, 2), [dev(v) for v in pb.vs], mode="lincomb")
    assert float(out[0].abs().max()) == 0.0


def test_errors_are_loud():
    from paper_2210_07667_b200 import PhiksError
    op = PhiKS([W.fd_dxx_dirichlet(8)])
    v = torch.zeros(8, dtype=torch.float64, device=DEV)
    with pytest.raises(PhiksError):
        op.apply(1.0, (2, 1), [v])          # not increasing
    with pytest.raises(PhiksError):
        op.apply(-1.0, (1,), [v])           # tau <= 0
    with pytest.raises(PhiksError):
        op.apply(1.0, (7,), [v])            # order above PHIKS_MAX_P


def test_back_to_back_applies_keep_their_exponentials():
    # the exponential stage runs on a side stream; a second apply with another τ
    # must not overwrite the first apply's exponentials while its Tucker
    # launches still read them (no sync in between), and two handles interleave
    pb = W.config(3, small=True).problems[0]
    big = [W.fd_dxx_neumann(160) * 1e-3] * 3           # above the graph threshold: side-stream path
    v = torch.from_numpy(np.ascontiguousarray(W.random_tensor((160,) * 3, seed=2).reshape(-1, order="F"))).to(DEV)
    op = PhiKS(big)
    ref = []
    for tau in (0.5, 2.0):
        ref.append([o.cpu().numpy() for o in op.apply(tau, (0, 1, 2), [v])])
        torch.cuda.synchronize()
    outs = [op.apply(tau, (0, 1, 2), [v]) for tau in (0.5, 2.0, 0.5)]
    torch.cuda.synchronize()
    for got, exp in zip(outs, [ref[0], ref[1], ref[0]]):
        for a, b in zip(got, exp):
            assert np.array_equal(a.cpu().numpy(), b)
    # two handles interleaved on one stream
    op2 = PhiKS([W.fd_dxx_neumann(160) * 2e-3] * 3)
    r2 = [o.cpu().numpy() for o in op2.apply(1.0, (0, 1, 2), [v])]
    torch.cuda.synchronize()
    seq = []
    for _ in range(3):
        seq.append(op.apply(0.5, (0, 1, 2), [v]))
        seq.append(op2.apply(1.0, (0, 1, 2), [v]))
    torch.cuda.synchronize()
    for k, got in enumerate(seq):
        exp = ref[0] if k % 2 == 0 else r2
        for a, b in zip(got, exp):
            assert np.array_equal(a.cpu().numpy(), b)
    del pb


def test_order_eight_tensor():
    # d = PHIKS_MAX_D = 8, both modes
    dims = (3, 2, 4, 2, 3, 2, 2, 3)
    fac = W.random_factors(dims, seed=88, scale=2.0)
    V = W.random_tensor(dims, seed=8)
    pb = W.Problem("d8_same", dims, fac, 0.7, "same", (0, 1, 2), [V], 2)
    op, ref, outs = _run(pb, force=False)
    _compare(pb, ref, outs, 2)
    vs = [W.random_tensor(dims, seed=20 + k) for k in range(3)]
    pb = W.Problem("d8_lincomb", dims, fac, 0.7, "lincomb", (0, 1, 2), vs, 1)
    op, ref, outs = _run(pb, force=False)
    _compare(pb, ref, outs, 1)


def test_api_error_paths():
    import ctypes
    from paper_2210_07667_b200 import PhiksError, ShardedPhiKS, _lib
    pb = W.config(2, small=True).problems[0]
    op = PhiKS(pb.A)
    v = dev(pb.vs[0])
    # caller workspace too small
    with pytest.raises(PhiksError) as ei:
        op.apply(pb.tau, pb.ells, [v], n_scales=pb.n_scales,
                 workspace=torch.empty(16, dtype=torch.float64, device=DEV))
    assert ei.value.code == 5  # PHIKS_ERR_WORKSPACE
    # wrong vector count / size / dtype
    with pytest.raises(PhiksError):
        op.apply(pb.tau, pb.ells, [v, v], n_scales=pb.n_scales)
    with pytest.raises(ValueError):
        op.apply(pb.tau, pb.ells, [v[:-1].contiguous()], n_scales=pb.n_scales)
    with pytest.raises(TypeError):
        op.apply(pb.tau, pb.ells, [v.float()], n_scales=pb.n_scales)
    # bad mem_kind through the raw ABI
    req = _lib.make_request(0, pb.ells, 1, pb.tau, mem_kind=7)
    arr = _lib.ptr_array([v.data_ptr()])
    outs = [torch.empty_like(v) for _ in pb.ells]
    code = _lib.load().phiks_apply(op._h, ctypes.byref(req), 1, arr, _lib.ptr_array([o.data_ptr() for o in outs]),
                                   None, 0, 0)
    assert code == 1
    # a sharded handle refuses to apply before its peers are attached
    sh = ShardedPhiKS(pb.A, 0, 2, connect=None)
    with pytest.raises(PhiksError):
        sh.apply(pb.tau, pb.ells, [v[: v.numel() // 2].contiguous()], n_scales=pb.n_scales)
    sh.close()
    # n_scales forcing s below ŝ-1
    with pytest.raises(PhiksError):
        op.apply(pb.tau, pb.ells, [v], n_scales=3, force_s=0, force_q=4)


def _table1_rows():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")) as f:
        return json.load(f)["linear_combination"]


@pytest.mark.parametrize("row", _table1_rows(), ids=lambda r: f"d{r['d']}n{r['n']}")
def test_table1_lincomb_tucker_count_executed(row):
    """PAPER.md Table 1 lincomb T = (q−2)p + sp + 1 (l.1436-1446): at the paper's
    (s, q) the library runs exactly T Tucker operators (θ_q = 1 free, only Ψ_p
    at the last squaring step, l.953-956), and the result matches the oracle."""
    dims = (8, 6, 4)
    fac = W.random_factors(dims, seed=row["n"], scale=2.0)
    vs = [W.random_tensor(dims, seed=40 + k) for k in range(5)]
    ells = (1, 2, 3, 4, 5)
    pl = O.Plan(row["s"], row["q"], 0)
    tau = 0.5
    ref = O.phiks_lincomb(fac, tau, dict(zip(ells, vs)), 1, pl)
    assert ref.tucker_ops == row["T"]
    op = PhiKS(fac)
    outs = op.apply(tau, ells, [dev(v) for v in vs], mode="lincomb", n_scales=1, force_s=row["s"],
                    force_q=row["q"])
    torch.cuda.synchronize()
    st = op.stats()
    assert st["tucker_ops"] == row["T"] == st["T_executed"]
    assert rel2(outs[0], W.as_flat(ref.out[0])) <= TOL


@pytest.mark.parametrize("ells,n_scales", [((1, 3), 1), ((2,), 2), ((0, 2, 4), 1), ((1, 2), 3)])
def test_same_vector_last_step_requested_only(ells, n_scales):
    """Same vector: at the last squaring step only the requested φ_ℓ are formed."""
    dims = (9, 7, 5)
    fac = W.random_factors(dims, seed=3, scale=6.0)
    V = W.random_tensor(dims, seed=4)
    pl = O.Plan(3, 5, 0)
    ref = O.phiks_same(fac, 1.0, V, ells, n_scales, pl)
    assert ref.tucker_ops == O.tucker_executed("same", 3, 5, ells, n_scales)
    op = PhiKS(fac)
    outs = op.apply(1.0, ells, [dev(V)], mode="same", n_scales=n_scales, force_s=3, force_q=5)
    torch.cuda.synchronize()
    assert op.stats()["tucker_ops"] == ref.tucker_ops
    for j in range(n_scales):
        for i, ell in enumerate(ells):
            assert rel2(outs[j * len(ells) + i], W.as_flat(ref.out[(ell, j)])) <= TOL


@pytest.mark.parametrize("ells", [(1, 3), (0, 2, 4), (4,), (0, 1, 2, 3, 4, 5)])
@pytest.mark.parametrize("path", ["dmma", "i8"])
def test_lincomb_given_vectors_subset(ells, path):
    """Linear combination with only some v_ℓ given: the quadrature runs one Tucker operator per
    node and GIVEN vector (linearity, reading R9) and matches the oracle's Eq. (17) result."""
    dims = (128, 32, 16)
    fac = [0.4 * W.fd_dxx_neumann(dims[0]), W.fd_dxx_dirichlet(dims[1]) + 2.0 * W.fd_dx_dirichlet(dims[1]),
           0.3 * W.fd_dxx_neumann(dims[2])]
    vs = [W.random_tensor(dims, seed=60 + k) for k in range(len(ells))]
    tau, s, q = 2e-3, 2, 6
    ref = O.phiks(fac, tau, "lincomb", ells, vs, n_scales=2, plan=O.Plan(s, q, 0))
    op = PhiKS(fac)
    op.set_gemm_path(path)
    outs = op.apply(tau, ells, [dev(v) for v in vs], mode="lincomb", n_scales=2, force_s=s, force_q=q)
    torch.cuda.synchronize()
    st = op.stats()
    given = sum(1 for e in ells if e >= 1)
    p = max(ells)
    assert st["tucker_ops"] == st["T_executed"] == (q - 1) * given + (s - 1) * p + 1 + (2 if 0 in ells else 0)
    for j in range(2):
        assert rel2(outs[j], W.as_flat(ref.out[j])) <= TOL, (ells, path, j)


def test_host_async_chained_presplit():
    """Host-memory applies on the chained int8 path with the pre-split combination (two handles in
    flight, the bench's e2e pattern): equal bit for bit to the device-memory path."""
    dims = (128, 128, 16)
    pbs = []
    for k, D in enumerate((2e-3, 1e-3)):
        A = [D * 128.0 ** 2 * W.fd_dxx_neumann(n) / n ** 2 for n in dims]
        pbs.append(W.Problem(f"hc{k}", dims, A, 0.05, "same", (0, 1, 2),
                             [W.uniform_tensor(dims, 0.0, 3.0, seed=60 + k)], 1))
    ops = [PhiKS(pb.A) for pb in pbs]
    for op in ops:
        op.set_gemm_path("i8")
    pins, pouts, ref = [], [], []
    for op, pb in zip(ops, pbs):
        x = W.as_flat(pb.vs[0])
        hi = torch.empty(x.size, dtype=torch.float64, pin_memory=True)
        hi.numpy()[:] = x
        pins.append(hi)
        pouts.append([torch.empty(x.size, dtype=torch.float64, pin_memory=True) for _ in pb.ells])
        ref.append([o.cpu().numpy() for o in op.apply(pb.tau, pb.ells, [dev(pb.vs[0])])])
        st = op.stats()
        assert st["i8_chained_ops"] > 0 and st["presplit_inputs"] > 0, st
    for rep in range(2):
        for op, pb, hi, ho in zip(ops, pbs, pins, pouts):
            op.apply(pb.tau, pb.ells, [hi.numpy()], outs=[t.numpy() for t in ho], host_async=True)
        for op in ops:
            op.wait()
        for ho, r in zip(pouts, ref):
            for a, b in zip(ho, r):
                assert np.array_equal(a.numpy(), b)
