"""GPU parity for complex factors and tensors (phiks_create_complex) against
the complex-capable oracle: random complex Kronecker sums of order d = 1..4
in both modes and several scales, the paper's complex validation operator
(1+i)/100·Δ of PAPER.md §4.1 l.1071-1082, and complex μ-mode products on
ragged shapes through the Tucker building block."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-12
DEV = "cuda:0"


def cdev(x):
    return torch.from_numpy(np.ascontiguousarray(W.as_flat(x).astype(np.complex128))).to(DEV)


def rel2(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def run_and_compare(pb):
    op = PhiKS(pb.A)
    assert op.complex
    outs = op.apply(pb.tau, pb.ells, [cdev(v) for v in pb.vs], mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    st = op.stats()
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
    assert (st["s"], st["q"]) == (ref.plan.s, ref.plan.q), pb.name
    for j in range(pb.n_scales):
        if pb.mode == "same":
            for i, ell in enumerate(pb.ells):
                e = rel2(outs[j * len(pb.ells) + i].cpu().numpy(), W.as_flat(ref.out[(ell, j)]))
                assert e <= TOL, (pb.name, ell, j, e)
        else:
            e = rel2(outs[j].cpu().numpy(), W.as_flat(ref.out[j]))
            assert e <= TOL, (pb.name, j, e)


def _cases():
    rng = np.random.default_rng(2024)
    out = []
    for c in range(10):
        d = int(rng.integers(1, 5))
        dims = tuple(int(x) for x in rng.integers(1, 48 if d <= 2 else 14, size=d))
        fac = W.random_factors(dims, seed=60 + c, scale=float(rng.uniform(0.2, 15.0)), complex_=True)
        mode = "same" if c % 2 == 0 else "lincomb"
        p = int(rng.integers(0, 5))
        ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
        vs = [W.random_tensor(dims, seed=90 + 5 * c + k, complex_=True)
              for k in range(1 if mode == "same" else len(ells))]
        out.append(W.Problem(f"cplx{c}_{mode}_d{d}", dims, fac, float(rng.uniform(0.1, 1.5)), mode, ells, vs,
                             int(rng.integers(1, 3))))
    return out


@pytest.mark.parametrize("pb", _cases(), ids=lambda pb: pb.name)
def test_complex_random_problems(pb):
    run_and_compare(pb)


@pytest.mark.parametrize("mode", ["same", "lincomb"])
def test_complex_validation_operator(mode):
    # PAPER.md §4.1: (1+i)/100·Δ (Dirichlet), v = 4096(1+i)∏ x(1−x); d = 3, n = 20
    n, d = 20, 3
    A = (1 + 1j) / 100 * W.fd_dxx_dirichlet(n)
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h
    f = x * (1 - x)
    V = 4096 * (1 + 1j) * f
    for _ in range(d - 1):
        V = np.multiply.outer(V, f)
    V = np.asfortranarray(np.transpose(V, tuple(range(d))))
    if mode == "same":
        pb = W.Problem("validation_same", (n,) * d, [A] * d, 1.0, "same", (0, 1, 2, 3, 4, 5), [V], 2)
    else:
        vs = [V] + [W.random_tensor((n,) * d, seed=k, complex_=True) for k in range(5)]
        pb = W.Problem("validation_lincomb", (n,) * d, [A] * d, 1.0, "lincomb", (0, 1, 2, 3, 4, 5), vs, 2)
    run_and_compare(pb)


def test_complex_large_tma_path():
    # sizes that take the TMA kernels on every mode (2n×2n real form on mode 1)
    dims = (96, 80, 66)
    fac = W.random_factors(dims, seed=5, scale=3.0, complex_=True)
    V = W.random_tensor(dims, seed=6, complex_=True)
    pb = W.Problem("cplx_tma", dims, fac, 0.5, "same", (0, 1, 2), [V], 1)
    run_and_compare(pb)


def test_complex_real_factors_agree_with_real_handle():
    # a complex handle on real data gives the real handle's result (imag part 0)
    pb = W.config(2, small=True).problems[0]
    A = [a.astype(np.complex128) for a in pb.A]
    op_c = PhiKS(A)
    op_r = PhiKS(pb.A)
    v = W.as_flat(pb.vs[0])
    oc = op_c.apply(pb.tau, pb.ells, [torch.from_numpy(v.astype(np.complex128)).to(DEV)], n_scales=pb.n_scales)
    orr = op_r.apply(pb.tau, pb.ells, [torch.from_numpy(v.copy()).to(DEV)], n_scales=pb.n_scales)
    torch.cuda.synchronize()
    for a, b in zip(oc, orr):
        a = a.cpu().numpy()
        b = b.cpu().numpy()
        assert np.abs(a.imag).max() == 0.0
        assert rel2(a.real, b) <= 1e-13


def test_complex_validation_operator_d6():
    # PAPER.md Table 1's d = 6 columns (n = 8): six-way complex tensors
    n, d = 8, 6
    A = (1 + 1j) / 100 * W.fd_dxx_dirichlet(n)
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h
    f = x * (1 - x)
    V = 4096 * (1 + 1j) * f
    for _ in range(d - 1):
        V = np.multiply.outer(V, f)
    pb = W.Problem("validation_d6", (n,) * d, [A] * d, 1.0, "same", (0, 1, 2, 3), [V], 1)
    run_and_compare(pb)


# ---- complex handles on the int8 tensor-core path: mode 1 through the 2n × 2n
# real form, modes μ ≥ 2 as one product with K = 2n, [Re M | Im M]·[x ; Jx] ----
@pytest.mark.parametrize("dims,mode", [((40, 48, 24), "same"), ((64, 150), "lincomb"), ((33, 130, 20), "same"),
                                       ((128, 96), "same")])
def test_complex_int8_path(dims, mode):
    seed = 1700 + sum(dims)
    fac = W.random_factors(dims, seed=seed, scale=4.0, complex_=True)
    ells = (0, 1, 2) if mode == "same" else (0, 1, 2, 3)
    vs = [W.random_tensor(dims, seed=seed + 1 + k, complex_=True) for k in range(1 if mode == "same" else len(ells))]
    pb = W.Problem(f"ci8{dims}{mode}", dims, fac, 0.6, mode, ells, vs, 2)
    op = PhiKS(pb.A)
    op.set_gemm_path("i8")
    outs = op.apply(pb.tau, pb.ells, [cdev(v) for v in pb.vs], mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    assert op.stats()["i8_mode_launches"] > 0
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
    for j in range(pb.n_scales):
        if pb.mode == "same":
            for i, ell in enumerate(pb.ells):
                e = rel2(outs[j * len(pb.ells) + i].cpu().numpy(), W.as_flat(ref.out[(ell, j)]))
                assert e <= 1e-12, (pb.name, ell, j, e)
        else:
            e = rel2(outs[j].cpu().numpy(), W.as_flat(ref.out[j]))
            assert e <= 1e-12, (pb.name, j, e)
