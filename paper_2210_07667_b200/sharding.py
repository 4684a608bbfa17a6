"""Slab sharding of PHIKS across the GPUs of one box.

Rank r of P owns the slab i_d ∈ [r·n_d/P, (r+1)·n_d/P) of the outermost mode,
i.e. the contiguous elements [r·N/P, (r+1)·N/P) of every column-major tensor.
The library does the rest (include/phiks.h, "Slab sharding"): modes 1..d-2 on
the slab, the mode-(d-1) product storing straight into the peer that owns
each column in the transposed layout, the mode-d product there, and the
stores back — over NVLink peer memory mapped with CUDA IPC.  This module only
marshals: it exchanges the IPC handles over torch.distributed (the plumbing)
and cuts global tensors into slabs.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np

from . import _lib


def block_range(n: int, world: int, rank: int):
    """[start, start+count) of rank's share of n indices: n // world each, one
    more for the first n % world ranks (the library's distribution)."""
    q, rem = divmod(n, world)
    start = rank * q + min(rank, rem)
    return start, start + q + (1 if rank < rem else 0)


def slab_bounds(N: int, world: int, rank: int, dims=None):
    """[lo, hi) of rank's slab in the flat column-major array: the block of the
    outermost mode (dims[-1]) it owns.  Without dims, N % world == 0 is required."""
    if dims is None:
        if N % world:
            raise ValueError("N must be divisible by world (pass dims for ragged slabs)")
        c = N // world
        return rank * c, (rank + 1) * c
    M = N // int(dims[-1])
    a, b = block_range(int(dims[-1]), world, rank)
    return M * a, M * b


def split_slabs(x, world: int, dims=None) -> list:
    """Views of the world slabs of a flat global tensor (numpy or torch)."""
    N = x.shape[0] if hasattr(x, "shape") else len(x)
    return [x[slice(*slab_bounds(N, world, r, dims))] for r in range(world)]


def _PhiKS():
    from . import PhiKS
    return PhiKS


class ShardedPhiKS:
    """Rank `rank` of a `world`-way slab-sharded φ-action handle.

    connect="dist": exchange IPC handles with torch.distributed (one process
    per GPU; every rank constructs its handle collectively).  connect=None:
    leave unconnected (same-process emulation: see connect_local)."""

    def __init__(self, factors: Sequence[np.ndarray], rank: int, world: int, connect: Optional[str] = "dist",
                 group=None):
        self.op = _PhiKS()(factors, rank=rank, world=world)
        self.rank, self.world = rank, world
        self.N = self.op.N  # this rank's slab (ragged slabs differ between ranks)
        self.dims = self.op.dims
        if connect == "dist" and world > 1:
            self.connect_dist(group)

    # -- peers -------------------------------------------------------------
    def ipc_handle(self) -> bytes:
        buf = (ctypes.c_char * _lib.IPC_HANDLE_BYTES)()
        _lib.check(_lib.load().phiks_shard_ipc_handle(self.op._h, buf), "phiks_shard_ipc_handle")
        return bytes(buf)

    def base(self) -> int:
        b = ctypes.c_void_p()
        _lib.check(_lib.load().phiks_shard_base(self.op._h, ctypes.byref(b)), "phiks_shard_base")
        return int(b.value or 0)

    def peer_base(self, k: int) -> int:
        b = ctypes.c_void_p()
        _lib.check(_lib.load().phiks_shard_peer_base(self.op._h, int(k), ctypes.byref(b)), "phiks_shard_peer_base")
        return int(b.value or 0)

    def open_peers(self, handles: Sequence[bytes]):
        if len(handles) != self.world:
            raise ValueError("one handle per rank")
        blob = b"".join(bytes(h).ljust(_lib.IPC_HANDLE_BYTES, b"\0") for h in handles)
        buf = ctypes.create_string_buffer(blob, len(blob))
        _lib.check(_lib.load().phiks_shard_open_peers(self.op._h, buf), "phiks_shard_open_peers")

    def connect_dist(self, group=None):
        import torch.distributed as dist
        gathered: List[Optional[bytes]] = [None] * self.world
        dist.all_gather_object(gathered, self.ipc_handle(), group=group)
        self.open_peers(gathered)

    @staticmethod
    def connect_local(ranks: Sequence["ShardedPhiKS"]):
        """Attach the ranks of one process to each other (emulation on one GPU)."""
        bases = [r.base() for r in ranks]
        for r in ranks:
            _lib.check(_lib.load().phiks_shard_set_peer_bases(r.op._h, _lib.ptr_array(bases)),
                       "phiks_shard_set_peer_bases")

    # -- compute (local slabs) -----------------------------------------------
    def apply(self, *a, **kw):
        return self.op.apply(*a, **kw)

    def plan(self, *a, **kw):
        return self.op.plan(*a, **kw)

    def stats(self) -> dict:
        return self.op.stats()

    def set_profiling(self, on: bool = True):
        self.op.set_profiling(on)

    def set_gemm_path(self, path: str):
        """int8 / DMMA / auto for the Tucker products of this rank (phiks_set_gemm_path)."""
        self.op.set_gemm_path(path)

    def set_option(self, name: str, value: int):
        """Execution option of this rank's handle (PHIKS_OPT_*, include/phiks.h)."""
        self.op.set_option(name, value)

    def wait(self):
        self.op.wait()

    def close(self):
        self.op.close()


def apply_ranks_serial(ranks: Sequence[ShardedPhiKS], tau: float, ells: Sequence[int], vecs: Sequence[Sequence],
                       mode: str = "same", n_scales: int = 1, tol: float = 0.0, outs=None, stream=None,
                       which: int = 0):
    """Run every rank's apply phase by phase on ONE GPU (phiks_apply_ranks_serial_ex).
    vecs[k]: rank k's local input slabs (device tensors); returns outs[k].  which: 0 every kernel,
    1 / 2 only / all but stage A (projection timing, include/phiks.h)."""
    import torch
    from . import PhiKS, _check_dev, _stream_ptr
    world = len(ranks)
    m = PhiKS._mode(mode)
    nouts = ranks[0].op.nblocks * (len(ells) * n_scales if m == _lib.MODE_SAME_VECTOR else n_scales)
    cplx = ranks[0].op.complex
    dt = torch.complex128 if cplx else torch.float64
    if outs is None:
        outs = [[torch.empty(ranks[k].N, dtype=dt, device=vecs[k][0].device) for _ in range(nouts)]
                for k in range(world)]
    vptr = [_check_dev(v, ranks[k].N, cplx) for k in range(world) for v in vecs[k]]
    optr = [_check_dev(o, ranks[k].N, cplx) for k in range(world) for o in outs[k]]
    req = _lib.make_request(m, ells, n_scales, tau, tol)
    hs = (ctypes.c_void_p * world)(*[r.op._h.value for r in ranks])
    _lib.check(_lib.load().phiks_apply_ranks_serial_ex(hs, world, ctypes.byref(req), len(vecs[0]),
                                                       _lib.ptr_array(vptr), _lib.ptr_array(optr),
                                                       _stream_ptr(stream), int(which)), "phiks_apply_ranks_serial_ex")
    return outs
