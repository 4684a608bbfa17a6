"""Parity at BASELINE.json's FULL sizes, through the same C-ABI calls bench.py
times.

* configs[1] (2-D 512², lincomb of 4), configs[2] (3-D 128³, 4 scales) and
  configs[3] (3-D 256³, both Brusselator species — the bench workload): every
  output against the oracle on the same seeded inputs, relative 2-norm ≤ 1e-12,
  with the library's own §3.3 plan equal to the oracle's.
* configs[4] (512×512×256, 67 M unknowns; the oracle is too slow): the
  eigen-tensor property φ_ℓ(τK)e = φ_ℓ(τλ)e (tests/eigen_fd.py, pinned in
  tests/test_eigen_fd.py) on combinations of separable eigen-tensors of the
  stored ADR factors, same operator and request as the config.
* the maximum factor size n = 4096 (PHIKS_MAX_N) by the same property.
* configs[3] slab-sharded over 8 emulated ranks: bit-identical to one GPU.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, apply_ranks_serial  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402
from paper_2210_07667_b200.sharding import split_slabs  # noqa: E402

import eigen_fd as E  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 1e-12
DEV = "cuda:0"


def rel2(got, ref):
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(W.as_flat(x))).to(DEV)


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_full_config_parity(cfg):
    for pb in W.config(cfg).problems:
        op = PhiKS(pb.A)
        outs = op.apply(pb.tau, pb.ells, [to_dev(v) for v in pb.vs], mode=pb.mode, n_scales=pb.n_scales)
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
        del outs, op
        torch.cuda.empty_cache()


def _eigen_case(A, ks, kind, n_vec, seed):
    es, lams = [], []
    for kk in ks:
        pairs = [E.eigpair(M, k, kind) for M, k in zip(A, kk)]
        es.append(E.separable([x for _, x in pairs]))
        lams.append(sum(l for l, _ in pairs))
    c = np.random.default_rng(seed).uniform(-1, 1, size=(n_vec, len(ks)))
    vs = [sum(c[i, t] * es[t] for t in range(len(ks))) for i in range(n_vec)]
    return es, lams, c, vs


def test_config4_full_eigen_property():
    pb = W.config(4, with_vectors=False).problems[0]
    ks = [(1, 1, 1), (2, 7, 3), (60, 200, 100), (512, 511, 256)]
    es, lams, c, vs = _eigen_case(pb.A, ks, "toeplitz", len(pb.ells), seed=4)
    op = PhiKS(pb.A)
    out = op.apply(pb.tau, pb.ells, [torch.from_numpy(v).to(DEV) for v in vs], mode="lincomb")[0]
    torch.cuda.synchronize()
    exp = sum(float(sum(E.phi(ell, pb.tau * lams[t]) * c[i, t] for i, ell in enumerate(pb.ells))) * es[t]
              for t in range(len(ks)))
    e = rel2(out.cpu().numpy(), exp)
    assert e <= TOL, e


def test_max_n_eigen_property():
    n = 4096
    A = W.fd_dxx_dirichlet(n) + 10.0 * W.fd_dx_dirichlet(n)
    fac = [A, A.copy()]
    ks = [(1, 1), (5, 2), (3000, 4096)]
    es, lams, c, _ = _eigen_case(fac, ks, "toeplitz", 1, seed=9)
    v = sum(c[0, t] * es[t] for t in range(len(ks)))
    tau, ells = 1e-6, (0, 1, 2, 3)
    op = PhiKS(fac)
    outs = op.apply(tau, ells, [torch.from_numpy(v).to(DEV)], mode="same", n_scales=2)
    torch.cuda.synchronize()
    for j in range(2):
        for i, ell in enumerate(ells):
            exp = sum(float(E.phi(ell, tau / 2 ** j * lams[t]) * c[0, t]) * es[t] for t in range(len(ks)))
            e = rel2(outs[j * len(ells) + i].cpu().numpy(), exp)
            assert e <= TOL, (ell, j, e)


def test_config3_full_sharded8_equals_single():
    pb = W.config(3).problems[0]
    x = W.as_flat(pb.vs[0])
    op = PhiKS(pb.A)
    op.set_gemm_path("dmma")  # the sharded handle runs the DMMA kernel: same arithmetic, bitwise equal
    single = [o.cpu().numpy() for o in op.apply(pb.tau, pb.ells, [to_dev(pb.vs[0])], n_scales=1)]
    del op
    world = 8
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    vecs = [[torch.from_numpy(np.ascontiguousarray(s)).to(DEV)] for s in split_slabs(x, world)]
    for r in ranks:
        r.set_gemm_path("dmma")
    outs = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode="same", n_scales=1)
    torch.cuda.synchronize()
    for i in range(len(pb.ells)):
        got = torch.cat([outs[r][i] for r in range(world)]).cpu().numpy()
        assert np.array_equal(got, single[i]), i
    # the default (int8) path on the sharded handle: peer-store epilogues of the int8 GEMM
    for r in ranks:
        r.set_gemm_path("auto")
    outs = apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode="same", n_scales=1)
    torch.cuda.synchronize()
    assert all(r.stats()["i8_mode_launches"] > 0 for r in ranks)
    for i in range(len(pb.ells)):
        got = torch.cat([outs[r][i] for r in range(world)]).cpu().numpy()
        assert rel2(got, single[i]) <= 1e-13, i
    for r in ranks:
        r.close()


@pytest.mark.skipif(not __import__("os").environ.get("PHIKS_SLOW_TESTS"),
                    reason="~5 min of oracle time; scripts/fullsize_cfg4_parity.py records the result in profiles/")
def test_config4_full_oracle_parity():
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import fullsize_cfg4_parity as F
    res = F.run()
    assert res["library_plan"]["s"] == res["oracle_plan"]["s"] and res["library_plan"]["q"] == res["oracle_plan"]["q"]
    assert res["library_plan"]["tucker_ops"] == res["oracle_plan"]["tucker_ops"]
    assert res["rel_2norm_err"] <= TOL, res
