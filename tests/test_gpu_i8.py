"""GPU parity of the int8 tensor-core μ-mode products:
phiks_mode_product_i8 against numpy fp64 on ragged shapes, shared inputs and
matrices, extreme magnitudes, zeros and non-finite values; whole φ-actions on
the int8 path against the CPU oracle and against the DMMA path; the path
selection (phiks_set_gemm_path) and its fallbacks."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, mode_product, mode_product_i8  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def np_mode(x, dims, mu, M):
    X = x.reshape(dims[::-1])  # column-major flat: the last C-order axis is mode 0
    ax = len(dims) - 1 - mu
    return np.moveaxis(np.tensordot(M, X, axes=([1], [ax])), 0, ax).reshape(-1)


def colmajor(M):
    return torch.from_numpy(np.asfortranarray(M).reshape(-1, order="F").copy()).to(DEV)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def dot_bound(xs, dims, mu, M):
    """Per-element |M|·|x| (the scale of an fp64 dot product's error bound)."""
    return np_mode(np.abs(xs), dims, mu, np.abs(M))


@pytest.mark.parametrize("dims,mu", [((40, 33, 17), 0), ((40, 33, 17), 1), ((40, 33, 17), 2), ((256, 9), 0),
                                     ((7, 250), 1), ((130, 64, 5), 1), ((3, 128, 129), 2), ((33, 200, 41), 1),
                                     ((1, 1000, 96), 2), ((129,), 0), ((5, 1, 31), 1), ((512, 40), 0),
                                     ((24, 300, 8), 1), ((64, 7, 449), 2)])  # n > 256: E streamed
@pytest.mark.parametrize("digits", [6, 7])
def test_i8_mode_product_vs_numpy(dims, mu, digits):
    rng = np.random.default_rng(hash((dims, mu, digits)) % 2 ** 32)
    N = int(np.prod(dims))
    n = dims[mu]
    xs = [rng.standard_normal(N) * np.exp(rng.uniform(-4, 4, N)) for _ in range(2)]
    Ms = [rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (n, n))) for _ in range(2)]
    xin = [torch.from_numpy(x).to(DEV) for x in xs]
    Min = [colmajor(M) for M in Ms]
    pairs = [(0, 0), (1, 1), (0, 1), (1, 0)]
    outs = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in pairs]
    mode_product_i8(dims, mu, [xin[a] for a, _ in pairs], [Min[b] for _, b in pairs], outs, slices=digits)
    torch.cuda.synchronize()
    # error bound per element: |Δy| ≤ c·n·2^-(8S-9)·max|e_j|·max|x_c|; check the
    # relative 2-norm and the elementwise bound against the dot-product scale
    for o, (a, b) in zip(outs, pairs):
        ref = np_mode(xs[a], dims, mu, Ms[b])
        got = o.cpu().numpy()
        e = rel(got, ref)
        assert e <= (2e-14 if digits == 7 else 5e-12), (dims, mu, digits, e)
        Xf = xs[a].reshape(dims[::-1])
        ax = len(dims) - 1 - mu
        xmax = np.max(np.abs(Xf), axis=ax, keepdims=True)  # per fiber
        emax = np.max(np.abs(Ms[b]), axis=1)                  # per row j
        scale = np.moveaxis(np.broadcast_to(xmax, Xf.shape), ax, 0)
        scale = np.moveaxis(scale * emax.reshape((-1,) + (1,) * (len(dims) - 1)), 0, ax).reshape(-1)
        bound = n * 2.0 ** (-(8 * digits - 9)) * scale
        assert np.all(np.abs(got - ref) <= bound + 1e-300), (dims, mu, digits)


def test_i8_mode_product_special_values():
    dims, mu = (64, 130), 1
    N = 64 * 130
    n = 130
    rng = np.random.default_rng(7)
    x = rng.standard_normal(N)
    X = x.reshape(130, 64)  # [k, l]
    X[:, 3] = 0.0                      # an all-zero fiber
    X[:, 5] *= 1e300                   # huge
    X[:, 6] *= 1e-300                  # tiny (normal)
    X[:, 7] = 5e-324 * rng.integers(-50, 50, 130)  # subnormal
    X[:, 8] = 0.0
    X[17, 8] = np.nan                  # a NaN poisons its fiber only
    X[:, 9] = 0.0
    X[3, 9] = np.inf
    M = rng.standard_normal((n, n))
    x = X.reshape(-1)
    out = torch.empty(N, dtype=torch.float64, device=DEV)
    mode_product_i8(dims, mu, [torch.from_numpy(x.copy()).to(DEV)], [colmajor(M)], [out], slices=7)
    torch.cuda.synchronize()
    got = out.cpu().numpy().reshape(130, 64)
    with np.errstate(invalid="ignore", over="ignore"):
        ref = np_mode(x, dims, mu, M).reshape(130, 64)
    assert np.all(got[:, 3] == 0.0)
    for c, f in ((5, 1e-300), (6, 1e300)):  # compare rescaled (the 2-norm of 1e300 values overflows)
        assert rel(got[:, c] * f, ref[:, c] * f) <= 1e-14, c
    assert rel(got[:, 7], ref[:, 7]) <= 1e-12  # subnormal inputs keep their (reduced) precision
    assert np.all(np.isnan(got[:, 8])) and np.all(np.isnan(got[:, 9]))
    ok = [c for c in range(64) if c not in (3, 5, 6, 7, 8, 9)]
    assert rel(got[:, ok], ref[:, ok]) <= 1e-14


def test_i8_matches_dmma_building_block_large():
    dims = (256, 256, 64)
    N = int(np.prod(dims))
    g = torch.Generator(device=DEV).manual_seed(3)
    x = torch.rand(N, dtype=torch.float64, device=DEV, generator=g) * 3
    for mu in range(3):
        n = dims[mu]
        M = torch.randn(n * n, dtype=torch.float64, device=DEV, generator=g)
        a = torch.empty_like(x)
        b = torch.empty_like(x)
        mode_product(dims, mu, [x], [M], [a])
        mode_product_i8(dims, mu, [x], [M], [b], slices=7)
        torch.cuda.synchronize()
        assert float(torch.linalg.norm(a - b) / torch.linalg.norm(a)) <= 1e-14, mu


def test_i8_rejects_unsupported():
    x = torch.zeros(600 * 4, dtype=torch.float64, device=DEV)
    M = torch.zeros(600 * 600, dtype=torch.float64, device=DEV)
    with pytest.raises(RuntimeError):  # n_μ > 512
        mode_product_i8((600, 4), 0, [x], [M], [x.clone()], slices=7)
    with pytest.raises(RuntimeError):
        mode_product_i8((4, 4), 0, [x[:16]], [M[:16]], [x[:16].clone()], slices=8)


def _apply(op, pb, path):
    op.set_gemm_path(path)
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in pb.vs]
    outs = op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], op.stats()


def _oracle_outs(pb):
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
    if pb.mode == "same":
        return [W.as_flat(ref.out[(ell, j)]) for j in range(pb.n_scales) for ell in pb.ells]
    return [W.as_flat(ref.out[j]) for j in range(pb.n_scales)]


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_i8_path_apply_parity_small_configs(cfg):
    for pb in W.config(cfg, small=True).problems:
        if max(pb.dims) > 256:
            continue
        op = PhiKS(pb.A)
        got, st = _apply(op, pb, "i8")
        ref = _oracle_outs(pb)
        for k, (g, r) in enumerate(zip(got, ref)):
            assert rel(g, r) <= 1e-12, (pb.name, k, rel(g, r))
        gd, std = _apply(op, pb, "dmma")
        assert std["i8_mode_launches"] == 0
        for g, r in zip(got, gd):
            assert rel(g, r) <= 1e-13


def test_i8_path_apply_random_problems():
    rng = np.random.default_rng(11)
    for c in range(6):
        d = int(rng.integers(2, 4))
        dims = tuple(int(x) for x in rng.integers(24, 140 if d == 3 else 256, size=d))
        fac = W.random_factors(dims, seed=500 + c, scale=float(rng.uniform(0.5, 20.0)))
        mode = "same" if c % 2 == 0 else "lincomb"
        ells = (0, 1, 2) if mode == "same" else (0, 1, 2, 3)
        vs = [W.random_tensor(dims, seed=600 + 7 * c + k) for k in range(1 if mode == "same" else len(ells))]
        pb = W.Problem(f"i8rand{c}", dims, fac, float(rng.uniform(0.2, 1.5)), mode, ells, vs, int(rng.integers(1, 3)))
        op = PhiKS(pb.A)
        got, st = _apply(op, pb, "i8")
        assert st["i8_mode_launches"] > 0, pb.name
        for k, (g, r) in enumerate(zip(got, _oracle_outs(pb))):
            assert rel(g, r) <= 1e-12, (pb.name, k, rel(g, r))


def test_i8_path_blocks_handle_and_fallback():
    # a block-diagonal handle on the int8 path; a mode with n_μ > 512 falls back to DMMA
    dims = (520, 40)
    pbs = []
    for b in range(2):
        fac = W.random_factors(dims, seed=700 + b, scale=4.0 + 6 * b)
        pbs.append(W.Problem(f"blk{b}", dims, fac, 0.5, "same", (0, 1, 2), [W.random_tensor(dims, seed=710 + b)], 1))
    op = PhiKS([pb.A for pb in pbs])
    op.set_gemm_path("i8")
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(pb.vs[0]))).to(DEV) for pb in pbs]
    outs = op.apply(0.5, (0, 1, 2), vs)
    torch.cuda.synchronize()
    st = op.stats()
    assert st["i8_mode_launches"] > 0  # mode 2 (n = 40) on the int8 path, mode 1 (n = 520 > 512) on DMMA
    for b, pb in enumerate(pbs):
        for k, r in enumerate(_oracle_outs(pb)):
            assert rel(outs[b * 3 + k].cpu().numpy(), r) <= 1e-12


def test_i8_path_selection_api():
    pb = W.config(2, small=True).problems[0]
    op = PhiKS(pb.A)
    with pytest.raises(KeyError):
        op.set_gemm_path("fp32")
    _, st = _apply(op, pb, "dmma")
    assert st["i8_mode_launches"] == 0
    _, st = _apply(op, pb, "i8")
    assert st["i8_mode_launches"] > 0


# ---- chained modes: every mode on the int8 path, each product
# writing the next mode's digits with exponents bounded before the product ----
CHAIN_SHAPES = [(128, 96), (128, 48, 32), (256, 16, 64), (128, 16, 16, 16), (256, 128), (128, 128, 16),
                (128, 256, 32, 16), (512, 96), (128, 384, 16)]  # n > 256: E streamed per k-block


@pytest.mark.parametrize("dims", CHAIN_SHAPES)
@pytest.mark.parametrize("mode", ["same", "lincomb"])
def test_i8_chain_apply_parity(dims, mode):
    seed = 800 + sum(dims) + (0 if mode == "same" else 1)
    rng = np.random.default_rng(seed)
    fac = W.random_factors(dims, seed=seed, scale=float(rng.uniform(1.0, 12.0)))
    ells = (0, 1, 2) if mode == "same" else (0, 1, 2, 3)
    vs = [W.random_tensor(dims, seed=seed + 10 + k) for k in range(1 if mode == "same" else len(ells))]
    pb = W.Problem(f"chain{dims}{mode}", dims, fac, float(rng.uniform(0.3, 1.2)), mode, ells, vs, 2)
    op = PhiKS(pb.A)
    op.set_option("chain", 2)  # random (non-Metzler) factors: the guard would keep per-mode splits
    got, st = _apply(op, pb, "i8")
    # every quadrature / squaring batch is chained; lincomb's exp(τK/2^j)v_0 terms (one per
    # scale, several outputs per operator) keep the per-mode path
    assert st["i8_chained_ops"] >= st["tucker_ops"] - (0 if mode == "same" else pb.n_scales) > 0, st
    for k, (g, r) in enumerate(zip(got, _oracle_outs(pb))):
        assert rel(g, r) <= 1e-12, (pb.name, k, rel(g, r))


def test_i8_chain_fd_operators_and_power_of_two_scaling():
    # Neumann / Dirichlet-ADR factors (rows of exp(τA) sum to ~1: tight exponent bounds);
    # φ-actions are linear in v, and scaling v by 2^k shifts every digit exponent by k, so
    # the chained path returns exactly 2^k times the unscaled result
    dims = (128, 64, 32)
    A = [0.7 * W.fd_dxx_neumann(dims[0]), W.fd_dxx_dirichlet(dims[1]) + 3.0 * W.fd_dx_dirichlet(dims[1]),
         0.2 * W.fd_dxx_neumann(dims[2])]
    v = W.uniform_tensor(dims, 0.0, 3.0, seed=901)
    pb = W.Problem("chainfd", dims, A, 2e-3, "same", (0, 1, 2), [v], 2)
    op = PhiKS(pb.A)
    got, st = _apply(op, pb, "i8")
    assert st["i8_chained_ops"] == st["tucker_ops"]
    for k, (g, r) in enumerate(zip(got, _oracle_outs(pb))):
        assert rel(g, r) <= 1e-12, (k, rel(g, r))
    for e in (-1000, 600):
        pbs = W.Problem("chainfd_s", dims, A, 2e-3, "same", (0, 1, 2), [np.ldexp(v, e)], 2)
        gs, _ = _apply(op, pbs, "i8")
        for g0, g1 in zip(got, gs):
            assert np.array_equal(np.ldexp(g0, e), g1), e


def test_i8_chain_zero_and_nonfinite_inputs():
    dims = (128, 32, 16)
    fac = W.random_factors(dims, seed=950, scale=3.0)
    op = PhiKS(fac)
    op.set_option("chain", 2)
    z = np.zeros(dims)
    got, st = _apply(op, W.Problem("z", dims, fac, 0.5, "same", (0, 1), [z], 1), "i8")
    assert st["i8_chained_ops"] > 0
    for g in got:
        assert not np.any(g)
    v = W.random_tensor(dims, seed=951)
    v[tuple(k // 3 for k in v.shape)] = np.nan
    got, _ = _apply(op, W.Problem("nan", dims, fac, 0.5, "same", (0, 1), [v], 1), "i8")
    # a dense Tucker operator spreads the NaN to every output (as fp64 arithmetic does)
    for g in got:
        assert np.all(np.isnan(g))


def test_i8_chain_graph_replay_bitwise():
    # applies of ≤ 4M elements are captured as CUDA graphs the first time and replayed after
    # (DESIGN.md §4): the chained path must replay bit for bit
    dims = (128, 64, 32)
    fac = W.random_factors(dims, seed=970, scale=6.0)
    v = torch.from_numpy(W.as_flat(W.random_tensor(dims, seed=971)).copy()).to(DEV)
    op = PhiKS(fac)
    op.set_gemm_path("i8")
    op.set_option("chain", 2)
    outs = [torch.empty_like(v) for _ in range(3)]
    res = []
    for _ in range(3):
        op.apply(0.4, (0, 1, 2), [v], outs=outs)
        torch.cuda.synchronize()
        res.append([o.cpu().numpy().copy() for o in outs])
    assert op.stats()["i8_chained_ops"] > 0
    for a, b in zip(res[0], res[2]):
        assert np.array_equal(a, b)
