"""CUDA IPC plumbing of the slab-sharded handle across PROCESSES (one GPU):
two ranks exchange their symmetric-region handles over torch.distributed
(gloo), map each other's region (phiks_shard_open_peers) and each reads the
pattern the other wrote.  Only host-synchronised copies — no kernel waits on
another process (B200_PROFILING.md), so this is safe on one GPU; the
device-side barrier and peer-store kernels are covered by the emulated-rank
tests (tests/test_gpu_sharded.py)."""
import ctypes
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
CTRL = 4096  # first pooled tensor of the region (csrc/host.h kCtrlBytes)


def _cudart():
    for name in ("libcudart.so", "libcudart.so.12"):
        try:
            return ctypes.CDLL(name)
        except OSError:
            continue
    import glob
    for p in glob.glob("/usr/local/cuda/lib64/libcudart.so*"):
        return ctypes.CDLL(p)
    raise OSError("libcudart not found")


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_07667_b200 import ShardedPhiKS
        from paper_2210_07667_b200 import workloads as W
        A = W.fd_dxx_neumann(8)
        op = ShardedPhiKS([A, A, A], rank, world)  # connect="dist": all_gather_object of the IPC handles
        rt = _cudart()
        rt.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        mine = np.arange(64, dtype=np.float64) + 1000.0 * (rank + 1)
        assert rt.cudaMemcpy(ctypes.c_void_p(op.base() + CTRL), mine.ctypes.data, mine.nbytes, 1) == 0
        assert op.peer_base(rank) == op.base()
        dist.barrier()
        got = {}
        for k in range(world):
            buf = np.empty(64)
            assert rt.cudaMemcpy(buf.ctypes.data, ctypes.c_void_p(op.peer_base(k) + CTRL), buf.nbytes, 2) == 0
            got[k] = buf
        dist.barrier()
        op.close()
        q.put((rank, {k: v.tolist() for k, v in got.items()}))
    finally:
        dist.destroy_process_group()


def test_ipc_exchange_between_processes():
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got in res.items():
        for k in range(world):
            np.testing.assert_array_equal(np.array(got[k]), np.arange(64) + 1000.0 * (k + 1))
