"""GPU parity of the slab-sharded path on ONE GPU.

The ranks are emulated in one process (phiks_apply_ranks_serial): every rank
has its own handle, symmetric region and workspace, and the peer-store
epilogues write into the other ranks' regions exactly as over NVLink; the
phases run rank after rank on one stream, so the cross-rank barriers are
implied by stream order and no kernel waits on another (B200_PROFILING.md).
The gathered slabs must match the oracle to the north-star tolerance
(relative 2-norm ≤ 1e-12) and the single-GPU path bit for bit (the μ-mode
products accumulate every element in the same order).
"""
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


def rel2(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def run_sharded(pb, world, n_scales=None, force=None, path="dmma", chain=1, presplit=None):
    n_scales = pb.n_scales if n_scales is None else n_scales
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    for r in ranks:
        r.set_gemm_path(path)
        r.set_option("chain", chain)
        if presplit is not None:
            r.set_option("presplit", presplit)
    flat = [W.as_flat(v) for v in pb.vs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, world)[r])).to(DEV) for x in flat]
            for r in range(world)]
    outs = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode=pb.mode, n_scales=n_scales)
    torch.cuda.synchronize()
    gathered = [torch.cat([outs[r][i] for r in range(world)]).cpu().numpy() for i in range(len(outs[0]))]
    stats = [r.stats() for r in ranks]
    for r in ranks:
        r.close()
    return gathered, stats


def run_single(pb, n_scales=None):
    n_scales = pb.n_scales if n_scales is None else n_scales
    op = PhiKS(pb.A)
    op.set_gemm_path("dmma")  # like with like: both on the DMMA kernel (same accumulation order)
    outs = op.apply(pb.tau, pb.ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in pb.vs],
                    mode=pb.mode, n_scales=n_scales)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], op.stats()


def compare_oracle(pb, outs, n_scales):
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=n_scales)
    for j in range(n_scales):
        if pb.mode == "same":
            for i, ell in enumerate(pb.ells):
                e = rel2(outs[j * len(pb.ells) + i], W.as_flat(ref.out[(ell, j)]))
                assert e <= TOL, (pb.name, ell, j, e)
        else:
            e = rel2(outs[j], W.as_flat(ref.out[j]))
            assert e <= TOL, (pb.name, j, e)
    return ref


CASES = [(2, 3), (2, 2), (3, 1), (4, 4), (2, 4)]


@pytest.mark.parametrize("cfg,world", [(0, 2), (0, 4), (2, 2), (2, 4), (2, 8), (3, 2), (3, 8), (4, 2), (4, 8), (1, 4)])
def test_sharded_configs_small(cfg, world):
    for pb in W.config(cfg, small=True).problems:
        outs, stats = run_sharded(pb, world)
        ref = compare_oracle(pb, outs, pb.n_scales)
        assert all((s["s"], s["q"]) == (ref.plan.s, ref.plan.q) for s in stats)
        single, _ = run_single(pb)
        for a, b in zip(outs, single):
            assert np.array_equal(a, b), pb.name   # same accumulation order as one GPU


def _random_sharded_cases():
    rng = np.random.default_rng(77)
    cases = []
    for c in range(8):
        world = int(rng.choice([2, 4, 8]))
        d = int(rng.integers(2, 5))
        dims = [int(x) for x in rng.integers(2, 9 if d >= 4 else 20, size=d)]
        dims[-1] = world * int(rng.integers(1, 4))
        dims[-2] = world * int(rng.integers(1, 4))
        dims = tuple(dims)
        mode = "same" if c % 2 == 0 else "lincomb"
        p = int(rng.integers(1, 5))
        ells = tuple(sorted(set([p] + [int(x) for x in rng.integers(0, p + 1, size=2)])))
        vs = [W.random_tensor(dims, seed=300 + 11 * c + k) for k in range(1 if mode == "same" else len(ells))]
        fac = W.random_factors(dims, seed=40 + c, scale=float(rng.uniform(0.5, 8.0)))
        cases.append((W.Problem(f"srand{c}_{mode}_w{world}_d{d}", dims, fac, float(rng.uniform(0.1, 1.5)), mode,
                                ells, vs, int(rng.integers(1, 3))), world))
    return cases


@pytest.mark.parametrize("case", _random_sharded_cases(), ids=lambda c: c[0].name)
def test_sharded_random_problems(case):
    pb, world = case
    outs, _ = run_sharded(pb, world)
    compare_oracle(pb, outs, pb.n_scales)


def test_sharded_many_nodes_chunks():
    # (q-1)·p > 16 quadrature Tucker operators: more than one sub-batch of the T/Y pools
    dims = (8, 8, 8)
    fac = W.random_factors(dims, seed=9, scale=40.0)
    ells = (0, 1, 2, 3, 4, 5, 6)
    vs = [W.random_tensor(dims, seed=k) for k in range(len(ells))]
    pb = W.Problem("chunks", dims, fac, 1.0, "lincomb", ells, vs, 1)
    plan = O.plan_for(fac, 1.0, "lincomb", ells, vs, 1)
    assert (plan.q - 1) * 6 > 16, plan
    outs, _ = run_sharded(pb, 4)
    compare_oracle(pb, outs, 1)


def test_sharded_world1_is_plain_handle():
    pb = W.config(2, small=True).problems[0]
    outs, _ = run_sharded(pb, 1)
    single, _ = run_single(pb)
    for a, b in zip(outs, single):
        assert np.array_equal(a, b)


def run_sharded_ragged(pb, world):
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    flat = [W.as_flat(v) for v in pb.vs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, world, pb.dims)[r])).to(DEV) for x in flat]
            for r in range(world)]
    outs = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    gathered = [torch.cat([outs[r][i] for r in range(world)]).cpu().numpy() for i in range(len(outs[0]))]
    for r in ranks:
        r.close()
    return gathered


@pytest.mark.parametrize("dims,world,mode", [((6, 10, 7), 3, "same"), ((5, 9, 11), 4, "lincomb"),
                                             ((4, 13, 10), 8, "same"), ((30, 25), 6, "lincomb"),
                                             ((3, 4, 9, 9), 2, "same"), ((40, 130, 70), 8, "same")])
def test_sharded_ragged_slabs(dims, world, mode):
    # P does not divide n_d and/or n_{d-1}: block-distributed slabs of different sizes
    fac = W.random_factors(dims, seed=sum(dims) + world, scale=4.0)
    ells = (0, 1, 2)
    vs = [W.random_tensor(dims, seed=7 + k) for k in range(1 if mode == "same" else 3)]
    pb = W.Problem(f"ragged_{dims}_{world}", dims, fac, 0.6, mode, ells, vs, 2)
    outs = run_sharded_ragged(pb, world)
    compare_oracle(pb, outs, 2)
    single, _ = run_single(pb)
    for a, b in zip(outs, single):
        assert rel2(a, b) <= 1e-15


@pytest.mark.parametrize("dims,world,mode", [((6, 8, 8), 2, "same"), ((5, 9, 7), 3, "lincomb"), ((12, 10), 4, "same"),
                                             ((3, 4, 5, 8), 4, "lincomb"), ((70, 66, 40), 8, "same")])
def test_sharded_complex(dims, world, mode):
    fac = W.random_factors(dims, seed=sum(dims), scale=3.0, complex_=True)
    ells = (0, 1, 2)
    vs = [W.random_tensor(dims, seed=11 + k, complex_=True) for k in range(1 if mode == "same" else 3)]
    pb = W.Problem(f"cplx_shard_{dims}_{world}", dims, fac, 0.7, mode, ells, vs, 2)
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    flat = [W.as_flat(v) for v in pb.vs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, world, dims)[r])).to(DEV) for x in flat]
            for r in range(world)]
    outs = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    gathered = [torch.cat([outs[r][i] for r in range(world)]).cpu().numpy() for i in range(len(outs[0]))]
    for r in ranks:
        r.close()
    compare_oracle(pb, gathered, 2)
    sop = PhiKS(pb.A)
    sop.set_gemm_path("dmma")
    single = sop.apply(pb.tau, pb.ells, [torch.from_numpy(np.ascontiguousarray(x)).to(DEV) for x in flat],
                       mode=pb.mode, n_scales=2)
    torch.cuda.synchronize()
    for a, b in zip(gathered, single):
        assert rel2(a, b.cpu().numpy()) <= 1e-15


# ---- the int8 tensor-core path on sharded handles: local modes
# split + GEMM, the two transposition stages as int8 GEMMs whose fp64 epilogue stores into
# the owner ranks' regions ----
@pytest.mark.parametrize("dims,world,mode", [((24, 40, 16), 2, "same"), ((20, 32, 24), 4, "lincomb"),
                                             ((16, 24, 40), 8, "same"), ((36, 20), 4, "same"),
                                             ((12, 10, 18, 16), 8, "lincomb"), ((30, 27, 24), 4, "same"),
                                             ((128, 32, 16), 2, "same"), ((128, 48, 24), 8, "lincomb"),
                                             ((128, 48, 32, 16), 4, "same"), ((128, 128, 16), 4, "lincomb"),
                                             ((512, 32, 16), 2, "same")])  # n > 256: E streamed
def test_sharded_int8_path(dims, world, mode):
    seed = 1300 + sum(dims) + world
    fac = W.random_factors(dims, seed=seed, scale=5.0)
    ells = (0, 1, 2) if mode == "same" else (0, 1, 2, 3)
    vs = [W.random_tensor(dims, seed=seed + 1 + k) for k in range(1 if mode == "same" else len(ells))]
    pb = W.Problem(f"si8_{dims}_{world}_{mode}", dims, fac, 0.7, mode, ells, vs, 2)
    # random (non-Metzler) factors: chaining forced past the guard to exercise the chained stages
    outs, stats = run_sharded(pb, world, path="i8", chain=2)
    assert all(s["i8_mode_launches"] > 0 for s in stats)
    if dims[0] == 128:  # modes 1..d−2 chained into the peer-store stage
        assert all(s["i8_chained_ops"] > 0 for s in stats)
    compare_oracle(pb, outs, pb.n_scales)
    single, _ = run_single(pb)
    for a, b in zip(outs, single):
        assert rel2(a, b) <= 1e-13


@pytest.mark.parametrize("dims,world,mode", [((6, 8, 8), 2, "same"), ((5, 9, 7), 3, "lincomb"),
                                             ((40, 66, 48), 4, "same"), ((3, 4, 5, 8), 4, "lincomb")])
def test_sharded_complex_int8(dims, world, mode):
    # complex sharded handles on the int8 path: local K = 2n products, and the two transposition
    # stages as K = 2n products whose epilogue stores into the owners (no copy pass, §4f)
    fac = W.random_factors(dims, seed=3 + sum(dims), scale=3.0, complex_=True)
    ells = (0, 1, 2)
    vs = [W.random_tensor(dims, seed=21 + k, complex_=True) for k in range(1 if mode == "same" else 3)]
    pb = W.Problem(f"cplx_shard_i8_{dims}_{world}", dims, fac, 0.7, mode, ells, vs, 2)
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    for r in ranks:
        r.set_gemm_path("i8")
    flat = [W.as_flat(v) for v in pb.vs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, world, dims)[r])).to(DEV) for x in flat]
            for r in range(world)]
    outs = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    assert all(r.stats()["i8_mode_launches"] > 0 for r in ranks)
    gathered = [torch.cat([outs[r][i] for r in range(world)]).cpu().numpy() for i in range(len(outs[0]))]
    for r in ranks:
        r.close()
    compare_oracle(pb, gathered, 2)


# ---- sharded digit stages: stage 0 exchanges the next-mode exponent maxima
# across the ranks and writes mode d's digit planes straight into the owners' pools; stage 1
# reads them (no fp64 transposition buffer, no re-split) ----
def _fd_factors(dims):
    out = []
    for k, n in enumerate(dims):
        if k % 2 == 0:
            out.append((0.5 + 0.3 * k) * W.fd_dxx_neumann(n))
        else:
            out.append(W.fd_dxx_dirichlet(n) + (2.0 + k) * W.fd_dx_dirichlet(n))
    return out


@pytest.mark.parametrize("dims,world,mode,kind", [((128, 64, 16), 2, "same", "fd"),
                                                  ((256, 64, 32), 2, "lincomb", "fd"),
                                                  ((128, 128, 16), 4, "same", "rand"),
                                                  ((128, 256, 16), 8, "lincomb", "fd"),
                                                  ((128, 16, 64, 16), 2, "same", "rand"),
                                                  ((256, 256, 32), 8, "same", "fd")])
def test_sharded_digit_stages(dims, world, mode, kind):
    seed = 1700 + sum(dims) + world
    fac = _fd_factors(dims) if kind == "fd" else W.random_factors(dims, seed=seed, scale=4.0)
    tau = 2e-3 if kind == "fd" else 0.6
    ells = (0, 1, 2) if mode == "same" else (0, 1, 2, 3)
    vs = [W.random_tensor(dims, seed=seed + 1 + k) for k in range(1 if mode == "same" else len(ells))]
    pb = W.Problem(f"sdig_{dims}_{world}_{mode}", dims, fac, tau, mode, ells, vs, 2)
    chain = 1 if kind == "fd" else 2  # Metzler FD factors chain under the default guard
    outs, stats = run_sharded(pb, world, path="i8", chain=chain)
    assert all(s["shard_digit_ops"] == s["tucker_ops"] > 0 for s in stats), \
        [(s["shard_digit_ops"], s["tucker_ops"]) for s in stats]
    compare_oracle(pb, outs, pb.n_scales)
    # one GPU, chained int8: the same digits (the exponent maxima are global either way) and
    # exact integer products; only the combination passes group their sums differently
    op = PhiKS(pb.A)
    op.set_gemm_path("i8")
    op.set_option("chain", chain)
    single = op.apply(pb.tau, pb.ells, [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in pb.vs],
                      mode=pb.mode, n_scales=pb.n_scales)
    torch.cuda.synchronize()
    for a, b in zip(outs, single):
        assert rel2(a, b.cpu().numpy()) <= 1e-13


@pytest.mark.parametrize("dims,world,mode", [((128, 64, 16), 2, "same"), ((256, 128, 32), 4, "lincomb")])
def test_sharded_presplit_bitwise(dims, world, mode):
    """PHIKS_OPT_PRESPLIT on slab-sharded handles: the combination that completes a squaring
    level's inputs writes their mode-1 digits (mode 1 is local to the slab); same results bit for
    bit as the separate split."""
    fac = _fd_factors(dims)
    ells = (0, 1, 2) if mode == "same" else (0, 1, 2, 3)
    vs = [W.random_tensor(dims, seed=1900 + k) for k in range(1 if mode == "same" else len(ells))]
    pb = W.Problem(f"spre_{dims}_{world}_{mode}", dims, fac, 2e-3, mode, ells, vs, 2)
    res = []
    for pre in (1, 0):
        outs, stats = run_sharded(pb, world, path="i8", chain=1, presplit=pre)
        hits = [st["presplit_inputs"] for st in stats]
        assert all(h > 0 for h in hits) if pre else all(h == 0 for h in hits), (pre, hits)
        res.append(outs)
    compare_oracle(pb, res[0], pb.n_scales)
    for a, b in zip(*res):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("path", ["dmma", "i8"])
def test_ranks_serial_filtered_replay(path):
    """phiks_apply_ranks_serial_ex (projection timing, include/phiks.h): stage A alone (which = 1)
    then the rest (which = 2) reproduces a full apply bit for bit, and so does the rest alone once
    both workspace halves hold the exponentials of earlier full applies."""
    pb = W.config(3, small=True).problems[0]
    world = 4
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    for r in ranks:
        r.set_gemm_path(path)
    flat = [W.as_flat(v) for v in pb.vs]
    vecs = [[torch.from_numpy(np.ascontiguousarray(split_slabs(x, world)[r])).to(DEV) for x in flat]
            for r in range(world)]

    def run(which):
        o = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode=pb.mode, n_scales=pb.n_scales, which=which)
        torch.cuda.synchronize()
        return [t.cpu().numpy() for k in range(world) for t in o[k]]
    full = run(0)
    run(0)
    for which in (2, 2):
        for a, b in zip(full, run(which)):
            assert np.array_equal(a, b)
    with pytest.raises(Exception):
        run(3)
    for r in ranks:
        r.close()
