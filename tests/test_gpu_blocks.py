"""Block-diagonal K̂ = diag(K_1, …, K_nb) in one handle (phiks_create_blocks,
PAPER.md §4.4's reaction–diffusion species): every block against the oracle,
against a separate handle per block, with different plans per block, in both
modes, and slab-sharded (emulated ranks)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, apply_ranks_serial  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402
from paper_2210_07667_b200.sharding import split_slabs  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-12
DEV = "cuda:0"


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(W.as_flat(x))).to(DEV)


def rel2(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def check_blocks(pbs, force_separate_equal=True):
    tau, ells, mode, ns = pbs[0].tau, pbs[0].ells, pbs[0].mode, pbs[0].n_scales
    op = PhiKS([pb.A for pb in pbs])
    assert op.nblocks == len(pbs)
    vecs = [dev(v) for pb in pbs for v in pb.vs]
    outs = op.apply(tau, ells, vecs, mode=mode, n_scales=ns)
    torch.cuda.synchronize()
    st = op.stats()
    per = len(outs) // len(pbs)
    for b, pb in enumerate(pbs):
        ref = O.phiks(pb.A, tau, mode, ells, pb.vs, n_scales=ns)
        assert st["block_plans"][b] == (ref.plan.s, ref.plan.q), (b, st["block_plans"], ref.plan)
        sep = PhiKS(pb.A).apply(tau, ells, [dev(v) for v in pb.vs], mode=mode, n_scales=ns)
        torch.cuda.synchronize()
        for k in range(per):
            got = outs[b * per + k].cpu().numpy()
            if mode == "same":
                j, i = divmod(k, len(ells))
                exp = W.as_flat(ref.out[(ells[i], j)])
            else:
                exp = W.as_flat(ref.out[k])
            assert rel2(got, exp) <= TOL, (b, k, rel2(got, exp))
            assert rel2(got, sep[k].cpu().numpy()) <= 1e-15, (b, k)
    return op


def test_brusselator_blocks_small():
    pbs = W.config(3, small=True).problems  # two species, different D_s → different plans possible
    check_blocks(pbs)


def test_blocks_lincomb_different_plans():
    dims = (12, 10, 8)
    pbs = []
    for b, scale in enumerate((0.5, 6.0, 30.0)):
        fac = W.random_factors(dims, seed=40 + b, scale=scale)
        vs = [W.random_tensor(dims, seed=100 * b + k) for k in range(4)]
        pbs.append(W.Problem(f"blk{b}", dims, fac, 0.8, "lincomb", (0, 1, 2, 3), vs, 2))
    op = check_blocks(pbs)
    plans = op.stats()["block_plans"]
    assert len(set(plans)) > 1  # the blocks really had different (s, q)


def test_blocks_same_vector_scales():
    dims = (20, 16)
    pbs = []
    for b in range(4):
        fac = W.random_factors(dims, seed=70 + b, scale=2.0 + 5 * b)
        pbs.append(W.Problem(f"blk{b}", dims, fac, 0.6, "same", (0, 1, 2), [W.random_tensor(dims, seed=b)], 3))
    check_blocks(pbs)


def test_blocks_sharded_emulated():
    pbs = W.config(3, small=True).problems
    world = 4
    ranks = [ShardedPhiKS([pb.A for pb in pbs], r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    slabs = [split_slabs(W.as_flat(pb.vs[0]), world) for pb in pbs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(slabs[b][r])).to(DEV) for b in range(len(pbs))]
            for r in range(world)]
    outs = apply_ranks_serial(ranks, pbs[0].tau, pbs[0].ells, vecs, mode="same")
    torch.cuda.synchronize()
    sop = PhiKS([pb.A for pb in pbs])
    sop.set_gemm_path("dmma")  # sharded handles run the DMMA kernel
    single = sop.apply(pbs[0].tau, pbs[0].ells, [dev(pb.vs[0]) for pb in pbs])
    torch.cuda.synchronize()
    for k in range(len(single)):
        got = torch.cat([outs[r][k] for r in range(world)]).cpu().numpy()
        assert rel2(got, single[k].cpu().numpy()) <= 1e-15, k
    for r in ranks:
        r.close()


def test_blocks_complex():
    # complex factors in a block-diagonal handle (phiks_create_blocks_complex)
    dims = (14, 9, 6)
    pbs = []
    for b, scale in enumerate((1.0, 12.0)):
        fac = W.random_factors(dims, seed=300 + b, scale=scale, complex_=True)
        vs = [W.random_tensor(dims, seed=310 + 3 * b + k, complex_=True) for k in range(3)]
        pbs.append(W.Problem(f"cblk{b}", dims, fac, 0.7, "lincomb", (0, 1, 2), vs, 2))
    op = check_blocks(pbs)
    assert op.complex


@pytest.mark.parametrize("world", [2, 3])
def test_blocks_complex_sharded_emulated(world):
    dims = (7, 11, 10)
    pbs = [W.Problem(f"cb{b}", dims, W.random_factors(dims, seed=320 + b, scale=4.0, complex_=True), 0.5, "same",
                     (0, 1, 3), [W.random_tensor(dims, seed=330 + b, complex_=True)], 2) for b in range(2)]
    ranks = [ShardedPhiKS([pb.A for pb in pbs], r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    slabs = [split_slabs(W.as_flat(pb.vs[0]), world, dims) for pb in pbs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(slabs[b][r])).to(DEV) for b in range(len(pbs))]
            for r in range(world)]
    outs = apply_ranks_serial(ranks, 0.5, (0, 1, 3), vecs, mode="same", n_scales=2)
    torch.cuda.synchronize()
    sop = PhiKS([pb.A for pb in pbs])
    sop.set_gemm_path("dmma")
    single = sop.apply(0.5, (0, 1, 3), [dev(pb.vs[0]) for pb in pbs], n_scales=2)
    torch.cuda.synchronize()
    for k in range(len(single)):
        got = torch.cat([outs[r][k] for r in range(world)]).cpu().numpy()
        assert rel2(got, single[k].cpu().numpy()) <= 1e-15, k
    for r in ranks:
        r.close()
