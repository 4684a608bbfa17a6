"""Per-handle execution options (include/phiks.h PHIKS_OPT_*): every setting gives the
oracle's result; the chain guard (reading R15) chains the int8 modes only for Metzler
factors."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, PhiksError  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
TOL = 1e-12


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _apply(op, pb):
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in pb.vs]
    outs = op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], op.stats()


def _oracle_outs(pb):
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
    if pb.mode == "same":
        return [W.as_flat(ref.out[(ell, j)]) for j in range(pb.n_scales) for ell in pb.ells]
    return [W.as_flat(ref.out[j]) for j in range(pb.n_scales)]


def test_option_api():
    op = PhiKS([W.fd_dxx_dirichlet(8)] * 2)
    assert [op.get_option(k) for k in ("split", "chain", "graphs", "presplit")] == [2, 1, 1, 1]
    for name, bad in (("split", 3), ("chain", -1), ("graphs", 2)):
        with pytest.raises(PhiksError):
            op.set_option(name, bad)
    op.set_option("split", 0)
    assert op.get_option("split") == 0


@pytest.mark.parametrize("split", [0, 1, 2])
@pytest.mark.parametrize("path", ["dmma", "i8"])
@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_split_option_parity(split, path, cfg):
    """PHIKS_OPT_SPLIT: quadrature sum and squaring recurrence fused into the last mode's
    epilogue (0), the quadrature as a streaming pass (1), both streaming (2)."""
    for pb in W.config(cfg, small=True).problems:
        op = PhiKS(pb.A)
        op.set_gemm_path(path)
        op.set_option("split", split)
        got, st = _apply(op, pb)
        for k, (g, r) in enumerate(zip(got, _oracle_outs(pb))):
            assert rel(g, r) <= TOL, (pb.name, split, path, k, rel(g, r))


def _fd_problem():
    dims = (128, 64, 32)
    A = [0.7 * W.fd_dxx_neumann(dims[0]), W.fd_dxx_dirichlet(dims[1]) + 3.0 * W.fd_dx_dirichlet(dims[1]),
         0.2 * W.fd_dxx_neumann(dims[2])]
    v = W.uniform_tensor(dims, -1.0, 1.0, seed=31)
    return W.Problem("fd", dims, A, 2e-3, "same", (0, 1, 2), [v], 1)


def _random_problem(scale=20.0, seed=41):
    dims = (128, 64, 32)
    fac = W.random_factors(dims, seed=seed, scale=scale)
    v = W.random_tensor(dims, seed=seed + 1)
    return W.Problem("rand", dims, fac, 0.5, "same", (0, 1, 2), [v], 1)


def test_chain_guard_follows_metzler_factors():
    """Default (guarded): FD Laplacian / ADR factors (off-diagonals ≥ 0) chain; dense random
    factors keep per-mode splits on the int8 path; 0 / 2 switch chaining off / on."""
    for pb, chained_default in ((_fd_problem(), True), (_random_problem(), False)):
        ref = _oracle_outs(pb)
        op = PhiKS(pb.A)
        op.set_gemm_path("i8")
        for opt, want in ((1, chained_default), (0, False), (2, True)):
            op.set_option("chain", opt)
            got, st = _apply(op, pb)
            assert st["i8_mode_launches"] > 0
            assert (st["i8_chained_ops"] > 0) == want, (pb.name, opt, st["i8_chained_ops"])
            for g, r in zip(got, ref):
                assert rel(g, r) <= TOL, (pb.name, opt, rel(g, r))


def test_chain_guard_accuracy_non_metzler():
    """Rows with sign cancellation (dense random factors): the chained exponent bound
    ‖e_j‖₁·max|x| exceeds the true fibre maximum, so chained digits carry fewer bits.  The
    guarded default stays within a small factor of the fp64 DMMA path's error."""
    errs = {}
    for scale in (30.0,):
        pb = _random_problem(scale=scale, seed=77)
        ref = _oracle_outs(pb)
        op = PhiKS(pb.A)
        for key, path, chain in (("dmma", "dmma", 1), ("guarded", "i8", 1), ("forced", "i8", 2)):
            op.set_gemm_path(path)
            op.set_option("chain", chain)
            got, _ = _apply(op, pb)
            errs[key] = max(rel(g, r) for g, r in zip(got, ref))
    assert errs["guarded"] <= TOL and errs["forced"] <= TOL, errs
    assert errs["guarded"] <= 8 * max(errs["dmma"], 1e-16), errs


def test_graphs_option_bitwise():
    pb = W.config(2, small=True).problems[0]
    res = []
    for g in (1, 0):
        op = PhiKS(pb.A)
        op.set_option("graphs", g)
        for _ in range(2):
            got, _ = _apply(op, pb)
        res.append(got)
    for a, b in zip(*res):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("mode", ["same", "lincomb"])
def test_presplit_option_bitwise(mode):
    """PHIKS_OPT_PRESPLIT: the combination producing a squaring level's inputs also writes
    their mode-1 digit planes (one pass fewer); the digits are the ones the split kernel
    would write, so both settings agree bit for bit (and with the oracle)."""
    pb = _fd_problem()
    if mode == "lincomb":
        v = pb.vs[0]
        pb = W.Problem("fd_lin", pb.dims, pb.A, pb.tau, "lincomb", (0, 1, 2, 3),
                       [v, 0.5 * v, W.uniform_tensor(pb.dims, -1.0, 1.0, seed=32), 0.25 * v], 2)
    ref = _oracle_outs(pb)
    res, hits = [], []
    for pre in (1, 0):
        op = PhiKS(pb.A)
        op.set_gemm_path("i8")
        op.set_option("presplit", pre)
        got, st = _apply(op, pb)
        assert st["i8_chained_ops"] > 0 and st["s"] >= 2
        hits.append(st["presplit_inputs"])
        res.append(got)
        for g, r in zip(got, ref):
            assert rel(g, r) <= TOL, (mode, pre, rel(g, r))
    assert hits[0] > 0 and hits[1] == 0, hits
    for a, b in zip(*res):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dims,mode,ells,tau,n_scales", [
    ((384, 128, 16), "same", (1, 2), 4e-3, 2),          # 12 elements per lane, two pre-split inputs
    ((512, 128), "lincomb", (0, 1, 2, 3, 4), 4e-3, 2),  # 16 per lane, four inputs per level, d = 2
    ((256, 128, 16), "lincomb", (1, 2, 3), 4e-3, 2),    # no v_0
    ((256, 128, 16), "lincomb", (0, 1, 2, 3, 4), 3e-5, 4),  # s = 3 < 4 scales: 5 outputs per pass
])
def test_presplit_shapes_bitwise(dims, mode, ells, tau, n_scales):
    """The fused combination + split on the other lane widths and output counts: bitwise equal
    to the separate split, and within the oracle's tolerance."""
    A = [W.fd_dxx_neumann(n) * (0.3 / (k + 1)) for k, n in enumerate(dims)]
    vs = [W.uniform_tensor(dims, -1.0, 1.0, seed=50 + k) for k in range(1 if mode == "same" else len(ells))]
    pb = W.Problem("pre", dims, A, tau, mode, ells, vs, n_scales)
    ref = _oracle_outs(pb)
    res, hits = [], []
    for pre in (1, 0):
        op = PhiKS(pb.A)
        op.set_gemm_path("i8")
        op.set_option("presplit", pre)
        got, st = _apply(op, pb)
        assert st["i8_chained_ops"] > 0 and st["s"] >= 2, st
        hits.append(st["presplit_inputs"])
        res.append(got)
        for g, r in zip(got, ref):
            assert rel(g, r) <= TOL, (dims, pre, rel(g, r))
    assert hits[0] > 0 and hits[1] == 0, hits
    for a, b in zip(*res):
        assert np.array_equal(a, b)


def test_presplit_nonfinite_inputs():
    """A NaN and an Inf in the input: the fused combination + split marks non-finite fibres exactly
    as the split kernel does, so both settings give the same outputs (every output entry depends on
    every input entry through the dense exponentials, so here they are NaN throughout)."""
    pb = _fd_problem()
    v = pb.vs[0].copy()
    v[3, 5, 7] = np.nan
    v[100, 20, 1] = np.inf
    res = []
    for pre in (1, 0):
        op = PhiKS(pb.A)
        op.set_gemm_path("i8")
        op.set_option("presplit", pre)
        outs = op.apply(pb.tau, pb.ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV)],
                        mode=pb.mode, n_scales=pb.n_scales)
        torch.cuda.synchronize()
        st = op.stats()
        assert (st["presplit_inputs"] > 0) == bool(pre)
        res.append([o.cpu().numpy() for o in outs])
    for a, b in zip(*res):
        np.testing.assert_array_equal(a, b)
        assert np.isnan(a).any()


@pytest.mark.parametrize("dims,ells", [
    ((512, 128), (0, 1, 2, 3, 4)),      # 4 inputs per level at n = 512: two warps per fibre (FS = 2)
    ((256, 128, 16), (0, 1, 2, 3, 4)),  # up to 8 outputs per pass at n = 256: two warps per fibre
])
@pytest.mark.parametrize("scale", [1.0, 1e-310])
def test_presplit_warp_pairs_bitwise(dims, ells, scale):
    """The combination + split variants that sum each fibre with two warps (their fibre exponent
    meets in shared memory): bitwise equal to the separate split, also for fibres of subnormal
    magnitude (the exact fp64 maximum path, a second exchange between the two warps)."""
    A = [W.fd_dxx_neumann(n) * (0.3 / (k + 1)) for k, n in enumerate(dims)]
    vs = [W.uniform_tensor(dims, -1.0, 1.0, seed=90 + k) * scale for k in range(len(ells))]
    res, hits = [], []
    for pre in (1, 0):
        op = PhiKS(A)
        op.set_gemm_path("i8")
        op.set_option("presplit", pre)
        outs = op.apply(3e-5, ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in vs],
                        mode="lincomb", n_scales=4)
        torch.cuda.synchronize()
        hits.append(op.stats()["presplit_inputs"])
        res.append([o.cpu().numpy() for o in outs])
    assert hits[0] > 0 and hits[1] == 0, hits
    for a, b in zip(*res):
        assert np.array_equal(a, b)
        assert np.all(np.isfinite(a))
