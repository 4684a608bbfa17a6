"""Zero-block skipping of the int8 GEMM (PHIKS_OPT_KSKIP): the exponentials
exp(cτA_μ) of banded factors are numerically banded, and the (64-row n-tile, 128-wide k-block)
blocks of E whose digits are all zero contribute exact integer zeros to the accumulators. The
GEMM skips them, so the results must be bit for bit those of the unskipped GEMM, and the
skipping must actually happen on banded factors and never on dense ones."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, mode_product_i8  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def np_mode(x, dims, mu, M):
    X = x.reshape(dims[::-1])
    ax = len(dims) - 1 - mu
    return np.moveaxis(np.tensordot(M, X, axes=([1], [ax])), 0, ax).reshape(-1)


def colmajor(M):
    return torch.from_numpy(np.asfortranarray(M).reshape(-1, order="F").copy()).to(DEV)


def _run(A, dims, tau, mode, ells, vs, n_scales, kskip):
    op = PhiKS(A)
    op.set_gemm_path("i8")
    op.set_option("kskip", kskip)
    op.set_profiling(True)
    dv = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in vs]
    outs = op.apply(tau, ells, dv, mode=mode, n_scales=n_scales)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], op.stats()


def test_kskip_option_api():
    op = PhiKS([W.fd_dxx_dirichlet(8)] * 2)
    assert op.get_option("kskip") == 1
    op.set_option("kskip", 0)
    assert op.get_option("kskip") == 0
    with pytest.raises(Exception):
        op.set_option("kskip", 2)


@pytest.mark.parametrize("dims,mode,ells,n_scales", [
    ((128, 128, 256), "same", (0, 1, 2), 1),      # configs[3]-shaped last mode (Neumann, D·τ/h² ≈ 0.65)
    ((128, 16, 512), "lincomb", (0, 1, 2, 3), 2),  # n = 512: E streamed per k-block (SE)
    ((384, 256), "same", (1, 2), 2),               # d = 2 (mode 1: 3 k-blocks)
])
def test_kskip_bitwise_banded(dims, mode, ells, n_scales):
    """Banded FD factors: blocks are skipped (the fp64-output launches of the last mode, §4g), the
    outputs equal the unskipped GEMM's bit for bit and the oracle's within 1e-12."""
    D = 2e-3
    A = [D * W.fd_dxx_neumann(n) for n in dims]
    tau = 5e-3
    nv = 1 if mode == "same" else len(ells)
    vs = [W.uniform_tensor(dims, 0.0, 3.0, seed=70 + k) for k in range(nv)]
    on, st_on = _run(A, dims, tau, mode, ells, vs, n_scales, 1)
    off, st_off = _run(A, dims, tau, mode, ells, vs, n_scales, 0)
    assert st_off["i8_kblocks"] > 0 and st_off["i8_kblocks_run"] == st_off["i8_kblocks"], st_off
    assert st_on["i8_kblocks"] == st_off["i8_kblocks"]
    assert st_on["i8_kblocks_run"] < st_on["i8_kblocks"], st_on  # banded exponentials: blocks skipped
    for a, b in zip(on, off):
        assert np.array_equal(a, b)
    ref = O.phiks(A, tau, mode, ells, vs, n_scales=n_scales)
    exp = ([W.as_flat(ref.out[(ell, j)]) for j in range(n_scales) for ell in ells] if mode == "same"
           else [W.as_flat(ref.out[j]) for j in range(n_scales)])
    for g, r in zip(on, exp):
        assert rel(g, r) <= 1e-12


def test_kskip_dense_factors_skip_nothing():
    """Dense random factors: no E digit block is zero, every block runs, results bitwise equal."""
    dims = (256, 128, 32)
    A = W.random_factors(dims, seed=5, scale=2.0)
    vs = [W.random_tensor(dims, seed=6)]
    on, st_on = _run(A, dims, 0.05, "same", (0, 1), vs, 1, 1)
    off, _ = _run(A, dims, 0.05, "same", (0, 1), vs, 1, 0)
    assert st_on["i8_kblocks_run"] == st_on["i8_kblocks"] > 0, st_on
    for a, b in zip(on, off):
        assert np.array_equal(a, b)


def _block_matrix(n, rng, pattern):
    """n×n matrix whose (64-row tile t, 128-wide k-block kb) block is zero where pattern(t, kb)."""
    M = rng.standard_normal((n, n)) * np.exp(rng.uniform(-3, 3, (n, n)))
    for t in range((n + 63) // 64):
        for kb in range((n + 127) // 128):
            if pattern(t, kb):
                M[64 * t:64 * t + 64, 128 * kb:128 * kb + 128] = 0.0
    return M


@pytest.mark.parametrize("dims,mu", [((40, 256, 17), 1), ((512, 40), 0), ((24, 384, 8), 1), ((3, 200, 129), 1),
                                     ((64, 7, 449), 2)])
@pytest.mark.parametrize("pattern", ["band", "gaps", "zero_rows"])
def test_kskip_mode_product_zero_blocks(dims, mu, pattern):
    """The building block (which always skips) on matrices with zero blocks in every position:
    a band, non-contiguous k-block masks, whole zero n-tiles (accumulators still written)."""
    rng = np.random.default_rng(hash((dims, mu, pattern)) % 2 ** 32)
    n = dims[mu]
    N = int(np.prod(dims))
    pats = {
        "band": lambda t, kb: abs(64 * t + 32 - (128 * kb + 64)) > 96,
        "gaps": lambda t, kb: (t + kb) % 2 == 1,
        "zero_rows": lambda t, kb: t % 3 == 1,
    }
    Ms = [_block_matrix(n, rng, pats[pattern]) for _ in range(2)]
    xs = [rng.standard_normal(N) for _ in range(2)]
    xin = [torch.from_numpy(x).to(DEV) for x in xs]
    Min = [colmajor(M) for M in Ms]
    pairs = [(0, 0), (1, 1), (0, 1)]
    outs = [torch.empty(N, dtype=torch.float64, device=DEV) for _ in pairs]
    mode_product_i8(dims, mu, [xin[a] for a, _ in pairs], [Min[b] for _, b in pairs], outs, slices=7)
    torch.cuda.synchronize()
    for o, (a, b) in zip(outs, pairs):
        ref = np_mode(xs[a], dims, mu, Ms[b])
        got = o.cpu().numpy()
        assert rel(got, ref) <= 2e-14, (dims, mu, pattern, rel(got, ref))
        if pattern == "zero_rows":  # rows of a zero n-tile give exact zeros
            Y = got.reshape(dims[::-1])
            ax = len(dims) - 1 - mu
            zr = [j for j in range(n) if (j // 64) % 3 == 1]
            assert np.all(np.take(Y, zr, axis=ax) == 0.0)
