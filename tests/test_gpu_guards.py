"""Out-of-bounds write detection without compute-sanitizer (closed on this
pool): every output, and the caller-provided workspace, is a slice of a
larger buffer whose guard zones hold a sentinel; after the call the guards
must be untouched and the results must still match the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import phiks_oracle as O  # noqa: E402
from paper_2210_07667_b200 import PhiKS, ShardedPhiKS, apply_ranks_serial, mode_product  # noqa: E402
from paper_2210_07667_b200 import workloads as W  # noqa: E402
from paper_2210_07667_b200.sharding import split_slabs  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
G = 4096          # guard doubles on each side
SENT = 1.2345e300


class Guarded:
    def __init__(self, n):
        self.buf = torch.full((n + 2 * G,), SENT, dtype=torch.float64, device=DEV)
        self.t = self.buf[G:G + n]

    def intact(self):
        b = self.buf.cpu().numpy()
        return bool(np.all(b[:G] == SENT) and np.all(b[-G:] == SENT))


@pytest.mark.parametrize("dims", [(7,), (33, 17), (5, 130, 3), (64, 3, 65), (256, 2, 66), (130, 129), (3, 257, 5),
                                  (66, 64, 2), (2, 3, 4, 5)])
def test_mode_product_writes_stay_in_bounds(dims):
    N = int(np.prod(dims))
    X = W.random_tensor(dims, seed=1)
    x = torch.from_numpy(np.ascontiguousarray(W.as_flat(X))).to(DEV)
    for mu, n in enumerate(dims):
        M = np.random.default_rng(mu).standard_normal((n, n))
        Md = torch.from_numpy(np.asfortranarray(M).reshape(-1, order="F").copy()).to(DEV)
        out = Guarded(N)
        mode_product(dims, mu, [x], [Md], [out.t])
        torch.cuda.synchronize()
        assert out.intact(), (dims, mu)
        ref = W.as_flat(O.mu_mode_product(X, M, mu))
        got = out.t.cpu().numpy()
        assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)


@pytest.mark.parametrize("cfg", [0, 1, 2])
def test_apply_outputs_and_workspace_stay_in_bounds(cfg):
    import ctypes
    from paper_2210_07667_b200 import _lib
    pb = W.config(cfg, small=True).problems[0]
    op = PhiKS(pb.A)
    ref = O.phiks(pb.A, pb.tau, pb.mode, pb.ells, pb.vs, n_scales=pb.n_scales)
    nout = len(pb.ells) * pb.n_scales if pb.mode == "same" else pb.n_scales
    outs = [Guarded(op.N) for _ in range(nout)]
    vs = [torch.from_numpy(np.ascontiguousarray(W.as_flat(v))).to(DEV) for v in pb.vs]
    # caller workspace of exactly the size the library asks for, inside guards
    norms = [float(np.linalg.norm(v)) for v in pb.vs[1:]] if pb.mode == "lincomb" else None
    plan = op.plan(pb.tau, pb.ells, mode=pb.mode, n_scales=pb.n_scales, vec_norms=norms)
    req = _lib.make_request(op._mode(pb.mode), pb.ells, pb.n_scales, pb.tau)
    info = _lib.PlanInfo(plan["s"], plan["q"], 0, 0)
    nbytes = ctypes.c_size_t()
    _lib.check(_lib.load().phiks_workspace_size(op._h, ctypes.byref(req), ctypes.byref(info), ctypes.byref(nbytes)),
               "phiks_workspace_size")
    ws = Guarded((nbytes.value + 7) // 8)
    op.apply(pb.tau, pb.ells, vs, mode=pb.mode, n_scales=pb.n_scales, outs=[o.t for o in outs], workspace=ws.t)
    torch.cuda.synchronize()
    assert ws.intact()
    assert all(o.intact() for o in outs)
    for j in range(pb.n_scales):
        if pb.mode == "same":
            for i, ell in enumerate(pb.ells):
                got = outs[j * len(pb.ells) + i].t.cpu().numpy()
                exp = W.as_flat(ref.out[(ell, j)])
                assert np.linalg.norm(got - exp) <= 1e-12 * np.linalg.norm(exp)
        else:
            got = outs[j].t.cpu().numpy()
            exp = W.as_flat(ref.out[j])
            assert np.linalg.norm(got - exp) <= 1e-12 * np.linalg.norm(exp)


def test_sharded_outputs_stay_in_bounds():
    pb = W.config(3, small=True).problems[0]
    world = 4
    ranks = [ShardedPhiKS(pb.A, r, world, connect=None) for r in range(world)]
    ShardedPhiKS.connect_local(ranks)
    slabs = split_slabs(W.as_flat(pb.vs[0]), world)
    vecs = [[torch.from_numpy(np.ascontiguousarray(s)).to(DEV)] for s in slabs]
    outs = [[Guarded(ranks[0].N) for _ in pb.ells] for _ in range(world)]
    apply_ranks_serial(ranks, pb.tau, pb.ells, vecs, mode="same", outs=[[o.t for o in row] for row in outs])
    torch.cuda.synchronize()
    assert all(o.intact() for row in outs for o in row)
    ref = O.phiks(pb.A, pb.tau, "same", pb.ells, pb.vs)
    for i, ell in enumerate(pb.ells):
        got = np.concatenate([outs[r][i].t.cpu().numpy() for r in range(world)])
        exp = W.as_flat(ref.out[(ell, 0)])
        assert np.linalg.norm(got - exp) <= 1e-12 * np.linalg.norm(exp)
    for r in ranks:
        r.close()
