"""Slab sharding without a GPU.

The library's own geometry of the two peer-store launches
(phiks_shard_layout, the same function its launches use) drives a simulation
of the sharded Tucker operator in which the local contractions are the
oracle's μ-mode products and the peer stores are numpy scatters — exchanged
between processes with torch.distributed (gloo, world size 2) in the last
test.  The gathered result must equal the oracle's Tucker operator on the
global tensor (Eq. (4)); that pins the slab/transposed-slab index
arithmetic of the CUDA path's epilogue (kernels.cu remote_store).
"""
import ctypes
import os
import socket

import numpy as np
import pytest

from oracle import phiks_oracle as O
from paper_2210_07667_b200 import _lib
from paper_2210_07667_b200 import workloads as W
from paper_2210_07667_b200.sharding import slab_bounds, split_slabs


def layout(dims, rank, world, stage):
    lib = _lib.load()
    out = (ctypes.c_int64 * 7)()
    n = (ctypes.c_int * len(dims))(*dims)
    _lib.check(lib.phiks_shard_layout(len(dims), n, rank, world, stage, out), "phiks_shard_layout")
    return dict(zip(("L", "n", "R", "cb", "rstride", "roff", "colstride"), list(out)))


def local_mode_product(x_flat, L, n, R, M):
    """(L, n, R) column-major view: y[l, j, r] = Σ_k M[j, k] x[l, k, r] (oracle)."""
    X = x_flat.reshape((L, n, R), order="F")
    return O.mu_mode_product(X, M, 1)


def peer_store(Y, lay, world):
    """What the remote epilogue does: element (l, j, r) -> (rank k, offset)."""
    L, n, R = Y.shape
    l, j, r = np.meshgrid(np.arange(L), np.arange(n), np.arange(R), indexing="ij")
    k = j // lay["cb"]
    off = l + lay["rstride"] * r + lay["roff"] + lay["colstride"] * (j - k * lay["cb"])
    return [(off[k == q], Y[k == q]) for q in range(world)]


def sharded_tucker_stage(slab, dims, mats, rank, world, stage, exchange):
    """One stage for one rank; `exchange(parts)` returns what this rank receives."""
    lay = layout(dims, rank, world, stage)
    M = mats[len(dims) - 2 + stage]
    Y = local_mode_product(slab, lay["L"], lay["n"], lay["R"], M)
    return exchange(peer_store(Y, lay, world))


def local_prefix(slab, dims, mats, world):
    """modes 1..d-2 on the slab (local dims (n_1..n_{d-1}, n_d/P))."""
    ld = list(dims)
    ld[-1] //= world
    T = W.from_flat(slab, ld)
    for mu in range(len(dims) - 2):
        T = O.mu_mode_product(T, mats[mu], mu)
    return W.as_flat(T)


def simulate(dims, mats, x, world):
    """All ranks in one process; the exchange is a plain numpy scatter."""
    N = int(np.prod(dims))
    Nl = N // world
    slabs = [local_prefix(s.copy(), dims, mats, world) for s in split_slabs(x, world)]
    for stage in (0, 1):
        recv = [np.full(Nl, np.nan) for _ in range(world)]
        for r in range(world):
            lay = layout(dims, r, world, stage)
            Y = local_mode_product(slabs[r], lay["L"], lay["n"], lay["R"], mats[len(dims) - 2 + stage])
            for q, (off, val) in enumerate(peer_store(Y, lay, world)):
                assert np.all(np.isnan(recv[q][off])), "two stores hit one element"
                recv[q][off] = val
        assert not any(np.isnan(v).any() for v in recv), "an element received no store"
        slabs = recv
    return np.concatenate(slabs)


CASES = [((6, 8), 2), ((5, 4, 8), 2), ((5, 4, 8), 4), ((3, 8, 8), 8), ((2, 3, 4, 4), 2), ((4, 6, 2), 2)]


@pytest.mark.parametrize("dims,world", CASES)
def test_sharded_tucker_simulation_equals_oracle(dims, world):
    mats = W.random_factors(dims, seed=7, scale=1.0)
    x = W.as_flat(W.random_tensor(dims, seed=3))
    got = simulate(dims, mats, x, world)
    ref = W.as_flat(O.tucker(W.from_flat(x, dims), mats))
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)


def test_layout_world1_is_identity_transposition():
    # world = 1: the two stages are the plain mode-(d-1) and mode-d products
    dims = (5, 6, 7)
    s0, s1 = layout(dims, 0, 1, 0), layout(dims, 0, 1, 1)
    assert (s0["L"], s0["n"], s0["R"]) == (5, 6, 7) and s0["colstride"] == 5 and s0["rstride"] == 30
    assert (s1["L"], s1["n"], s1["R"]) == (30, 7, 1) and s1["colstride"] == 30 and s1["roff"] == 0


def test_slab_bounds_partition():
    N, world = 4096, 8
    b = [slab_bounds(N, world, r) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == N
    assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
    with pytest.raises(ValueError):
        slab_bounds(10, 3, 0)


def test_create_sharded_rejects_bad_arguments():
    lib = _lib.load()
    A = np.asfortranarray(W.fd_dxx_dirichlet(8))
    ptrs = _lib.ptr_array([A.ctypes.data] * 3)
    h = ctypes.c_void_p()
    n3 = (ctypes.c_int * 3)(8, 8, 8)
    n_bad = (ctypes.c_int * 3)(8, 3, 8)   # n_{d-1} = 3 < world = 4
    n1 = (ctypes.c_int * 1)(8)
    assert lib.phiks_create_sharded(3, n3, ptrs, 0, 9, ctypes.byref(h)) == 1   # world > 8
    assert lib.phiks_create_sharded(3, n3, ptrs, 2, 2, ctypes.byref(h)) == 1   # rank >= world
    assert lib.phiks_create_sharded(3, n_bad, ptrs, 0, 4, ctypes.byref(h)) == 1
    assert lib.phiks_create_sharded(1, n1, ptrs, 0, 2, ctypes.byref(h)) == 1   # d = 1
    out = (ctypes.c_int64 * 7)()
    assert lib.phiks_shard_layout(3, n_bad, 0, 4, 0, out) == 1
    assert lib.phiks_shard_layout(3, n3, 0, 4, 2, out) == 1


# ---------------------------------------------------------------------------
# world size 2 over gloo: each process is one rank, the exchange is a real
# collective (all_gather_object of the (offset, value) parts).
# ---------------------------------------------------------------------------
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, dims, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mats = W.random_factors(dims, seed=11, scale=1.0)
        x = W.as_flat(W.random_tensor(dims, seed=5))
        lo, hi = slab_bounds(x.size, world, rank)
        slab = local_prefix(x[lo:hi].copy(), dims, mats, world)

        def exchange(parts):
            got = [None] * world
            dist.all_gather_object(got, parts)
            recv = np.full(hi - lo, np.nan)
            for src in range(world):
                off, val = got[src][rank]
                recv[off] = val
            return recv

        for stage in (0, 1):
            slab = sharded_tucker_stage(slab, dims, mats, rank, world, stage, exchange)
        full = [None] * world
        dist.all_gather_object(full, slab)
        # the plan input of the lincomb mode: local sums of squares summed in rank order
        ss = [None] * world
        dist.all_gather_object(ss, float(np.sum(x[lo:hi] ** 2)))
        q.put((rank, np.concatenate(full), float(np.sqrt(sum(ss)))))
    finally:
        dist.destroy_process_group()


def test_sharded_tucker_gloo_world2():
    import torch.multiprocessing as mp
    dims = (4, 6, 8)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, dims, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mats = W.random_factors(dims, seed=11, scale=1.0)
    x = W.as_flat(W.random_tensor(dims, seed=5))
    ref = W.as_flat(O.tucker(W.from_flat(x, dims), mats))
    for rank, full, nrm in res:
        np.testing.assert_allclose(full, ref, rtol=1e-13, atol=1e-13)
        assert abs(nrm - np.linalg.norm(x)) <= 1e-13 * np.linalg.norm(x)


# ---------------------------------------------------------------------------
# ragged slabs (P not dividing n_d or n_{d-1}): phiks_shard_layout_ex
# ---------------------------------------------------------------------------
from paper_2210_07667_b200.sharding import block_range  # noqa: E402


def layout_ex(dims, rank, world, stage):
    lib = _lib.load()
    out = (ctypes.c_int64 * (4 + 3 * world))()
    n = (ctypes.c_int * len(dims))(*dims)
    _lib.check(lib.phiks_shard_layout_ex(len(dims), n, rank, world, stage, out), "phiks_shard_layout_ex")
    v = list(out)
    return {"L": v[0], "n": v[1], "R": v[2], "colstride": v[3], "kstart": v[4:4 + world],
            "kstride": v[4 + world:4 + 2 * world], "kroff": v[4 + 2 * world:4 + 3 * world]}


def owner(j, n, world):
    return next(k for k in range(world) if j < block_range(n, world, k)[1])


def peer_store_ex(Y, lay, world):
    L, n, R = Y.shape
    l, j, r = np.meshgrid(np.arange(L), np.arange(n), np.arange(R), indexing="ij")
    k = np.vectorize(lambda jj: owner(jj, n, world))(j)
    ks = np.asarray(lay["kstart"])[k]
    kst = np.asarray(lay["kstride"])[k]
    kro = np.asarray(lay["kroff"])[k]
    off = l + kst * r + kro + lay["colstride"] * (j - ks)
    return [(off[k == q], Y[k == q]) for q in range(world)]


def simulate_ragged(dims, mats, x, world):
    d = len(dims)
    L0 = int(np.prod(dims[:-2]))
    na, nd = dims[-2], dims[-1]
    slabs = []
    for r, s in enumerate(split_slabs(x, world, dims)):
        ld = list(dims)
        a, b = block_range(nd, world, r)
        ld[-1] = b - a
        T = W.from_flat(s.copy(), ld)
        for mu in range(d - 2):
            T = O.mu_mode_product(T, mats[mu], mu)
        slabs.append(W.as_flat(T))
    sizes = [[L0 * (block_range(na, world, k)[1] - block_range(na, world, k)[0]) * nd for k in range(world)],
             [L0 * na * (block_range(nd, world, k)[1] - block_range(nd, world, k)[0]) for k in range(world)]]
    for stage in (0, 1):
        recv = [np.full(sizes[stage][k], np.nan) for k in range(world)]
        for r in range(world):
            lay = layout_ex(dims, r, world, stage)
            Y = local_mode_product(slabs[r], lay["L"], lay["n"], lay["R"], mats[d - 2 + stage])
            for q, (off, val) in enumerate(peer_store_ex(Y, lay, world)):
                assert np.all(np.isnan(recv[q][off])), "two stores hit one element"
                recv[q][off] = val
        assert not any(np.isnan(v).any() for v in recv), "an element received no store"
        slabs = recv
    return np.concatenate(slabs)


@pytest.mark.parametrize("dims,world", [((5, 7, 10), 3), ((6, 9), 4), ((3, 10, 9), 8), ((2, 3, 5, 9), 2),
                                        ((4, 8, 8), 4)])
def test_ragged_sharded_tucker_simulation_equals_oracle(dims, world):
    mats = W.random_factors(dims, seed=17, scale=1.0)
    x = W.as_flat(W.random_tensor(dims, seed=4))
    got = simulate_ragged(dims, mats, x, world)
    ref = W.as_flat(O.tucker(W.from_flat(x, dims), mats))
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-13)


def test_layout_ex_matches_uniform_layout():
    dims, world = (5, 8, 16), 4
    for stage in (0, 1):
        for r in range(world):
            a, b = layout(dims, r, world, stage), layout_ex(dims, r, world, stage)
            assert (a["L"], a["n"], a["R"], a["colstride"]) == (b["L"], b["n"], b["R"], b["colstride"])
            assert all(s == a["rstride"] for s in b["kstride"]) and all(o == a["roff"] for o in b["kroff"])
            assert b["kstart"] == [k * a["cb"] for k in range(world)]
