"""B200-native PHIKS: actions of φ-functions of Kronecker sums on FP64 tensor cores.

User API (thin marshalling over the C ABI of include/phiks.h; PyTorch only
provides device memory and streams):

    from paper_2210_07667_b200 import PhiKS
    op = PhiKS([A1, A2, A3])                    # numpy factor matrices A_μ
    outs = op.apply(tau, [0, 1, 2], [v])        # φ_ℓ(τK)v, torch fp64 cuda tensors
    comb = op.apply(tau, [0, 1, 2], [v0, v1, v2], mode="lincomb")

Tensors are column-major n_1×…×n_d (§2 vec convention): a torch
tensor of shape (n_d, …, n_1) in C order, or any contiguous tensor with N
elements in that order.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import MEM_DEVICE, MEM_HOST, MODE_LINCOMB, MODE_SAME_VECTOR, PhiksError

__all__ = ["PhiKS", "ShardedPhiKS", "PhiksError", "mode_product", "tucker", "expm", "fp64_peak_launch", "version",
           "apply_ranks_serial"]


def _torch():
    import torch
    return torch


def _stream_ptr(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


def _check_dev(t, N: Optional[int] = None, complex_: bool = False):
    torch = _torch()
    dt = torch.complex128 if complex_ else torch.float64
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dt and t.is_contiguous()):
        raise TypeError(f"expected a contiguous {dt} CUDA tensor")
    if N is not None and t.numel() != N:
        raise ValueError(f"tensor has {t.numel()} elements, expected {N}")
    return t.data_ptr()


def version() -> str:
    return _lib.load().phiks_version().decode()


class PhiKS:
    """Handle on K = A_d ⊕ … ⊕ A_1 (phiks_create / phiks_destroy)."""

    def __init__(self, factors: Sequence, rank: int = 0, world: int = 1):
        """factors: [A_1, …, A_d] for K = A_d ⊕ … ⊕ A_1, or a list of such lists
        for a block-diagonal K̂ = diag(K_1, …, K_nb) (§4.4; every block
        with the same dims; vectors and outputs are then given block-major)."""
        lib = _lib.load()
        blocks = [list(f) for f in factors] if (len(factors) and not hasattr(factors[0], "shape")
                                                 and isinstance(factors[0], (list, tuple))) else [list(factors)]
        self.nblocks = len(blocks)
        self.d = len(blocks[0])
        self.dims = tuple(int(np.asarray(a).shape[0]) for a in blocks[0])
        self.rank, self.world = int(rank), int(world)
        # complex factors (§4.1's validation operator is complex): complex128 throughout
        self.complex = any(np.iscomplexobj(a) for blk in blocks for a in blk)
        dt = np.complex128 if self.complex else np.float64
        self._A = [np.asfortranarray(np.asarray(a, dtype=dt)) for blk in blocks for a in blk]
        for blk in blocks:
            if len(blk) != self.d or tuple(int(np.asarray(a).shape[0]) for a in blk) != self.dims:
                raise ValueError("every block needs the same dims")
        for a in self._A:
            if a.ndim != 2 or a.shape[0] != a.shape[1]:
                raise ValueError("factor matrices must be square")
        n_arr = (ctypes.c_int * self.d)(*self.dims)
        a_arr = _lib.ptr_array([a.ctypes.data for a in self._A])
        h = ctypes.c_void_p()
        if self.complex:
            if self.world == 1:
                _lib.check(lib.phiks_create_blocks_complex(self.nblocks, self.d, n_arr, a_arr, ctypes.byref(h)),
                           "phiks_create_complex")
            else:
                _lib.check(lib.phiks_create_sharded_blocks_complex(self.nblocks, self.d, n_arr, a_arr, self.rank,
                                                                   self.world, ctypes.byref(h)),
                           "phiks_create_sharded_complex")
        elif self.world == 1:
            _lib.check(lib.phiks_create_blocks(self.nblocks, self.d, n_arr, a_arr, ctypes.byref(h)), "phiks_create")
        else:
            _lib.check(lib.phiks_create_sharded_blocks(self.nblocks, self.d, n_arr, a_arr, self.rank, self.world,
                                                       ctypes.byref(h)), "phiks_create_sharded")
        self._h = h
        # N: elements of the tensors apply() takes (the local slab when sharded)
        self.N = int(np.prod(self.dims))
        if self.world > 1:
            cnt = ctypes.c_int64()
            _lib.check(lib.phiks_shard_info(self._h, None, None, ctypes.byref(cnt), None), "phiks_shard_info")
            self.N = int(cnt.value)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.load().phiks_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------
    def plan(self, tau: float, ells: Sequence[int], mode: str = "same", n_scales: int = 1,
             tol: float = 0.0, vec_norms: Optional[Sequence[float]] = None) -> dict:
        lib = _lib.load()
        req = _lib.make_request(self._mode(mode), ells, n_scales, tau, tol)
        info = _lib.PlanInfo()
        norms = None
        if vec_norms is not None:
            norms = (ctypes.c_double * len(vec_norms))(*vec_norms)
        _lib.check(lib.phiks_plan(self._h, ctypes.byref(req), norms, ctypes.byref(info)), "phiks_plan")
        return {"s": info.s, "q": info.q, "T_formula": info.T_formula, "T_executed": info.T_executed}

    @staticmethod
    def _mode(mode) -> int:
        if mode in ("same", MODE_SAME_VECTOR):
            return MODE_SAME_VECTOR
        if mode in ("lincomb", MODE_LINCOMB):
            return MODE_LINCOMB
        raise ValueError(f"unknown mode {mode!r}")

    def apply(self, tau: float, ells: Sequence[int], vecs: Sequence, mode: str = "same", n_scales: int = 1,
              tol: float = 0.0, outs: Optional[Sequence] = None, force_s: int = -1, force_q: int = -1,
              stream=None, workspace=None, host_async: bool = False):
        """Run phiks_apply.  vecs/outs are contiguous fp64 CUDA tensors
        (PHIKS_MEM_DEVICE) or numpy arrays (PHIKS_MEM_HOST; then outs are
        returned as numpy arrays).  host_async=True (numpy arrays over PINNED
        memory only) returns before the copies finish (PHIKS_MEM_HOST_ASYNC);
        call wait() before reading the outputs.  Returns the list of outputs:
        same-vector → outs[j*len(ells)+i] = φ_{ells[i]}(τK/2^j)v; lincomb → outs[j]."""
        lib = _lib.load()
        m = self._mode(mode)
        host = isinstance(vecs[0], np.ndarray)
        nouts = self.nblocks * (len(ells) * n_scales if m == MODE_SAME_VECTOR else n_scales)
        dt = np.complex128 if self.complex else np.float64
        if host:
            vecs = [np.ascontiguousarray(np.asarray(v, dtype=dt).reshape(-1, order="F")) for v in vecs]
            for v in vecs:
                if v.size != self.N:
                    raise ValueError("vector size mismatch")
            if outs is None:
                outs = [np.empty(self.N, dtype=dt) for _ in range(nouts)]
            vptr = [v.ctypes.data for v in vecs]
            optr = [o.ctypes.data for o in outs]
            sptr = _stream_ptr(stream) if stream is not None else 0
        else:
            torch = _torch()
            tdt = torch.complex128 if self.complex else torch.float64
            vptr = [_check_dev(v, self.N, self.complex) for v in vecs]
            if outs is None:
                outs = [torch.empty(self.N, dtype=tdt, device=vecs[0].device) for _ in range(nouts)]
            optr = [_check_dev(o, self.N, self.complex) for o in outs]
            sptr = _stream_ptr(stream)
        kind = (_lib.MEM_HOST_ASYNC if host_async else MEM_HOST) if host else MEM_DEVICE
        req = _lib.make_request(m, ells, n_scales, tau, tol, force_s, force_q, kind)
        ws_ptr, ws_bytes = (None, 0)
        if workspace is not None:
            ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
        code = lib.phiks_apply(self._h, ctypes.byref(req), len(vecs), _lib.ptr_array(vptr), _lib.ptr_array(optr),
                               ws_ptr, ws_bytes, sptr)
        _lib.check(code, "phiks_apply")
        return list(outs)

    def stats(self) -> dict:
        st = _lib.Stats()
        _lib.check(_lib.load().phiks_get_stats(self._h, ctypes.byref(st)), "phiks_get_stats")
        return {"s": st.plan.s, "q": st.plan.q, "T_formula": st.plan.T_formula, "T_executed": st.plan.T_executed,
                "kernel_launches": st.kernel_launches, "tucker_ops": st.tucker_ops,
                "mu_mode_flops": st.mu_mode_flops, "expm_flops": st.expm_flops,
                "workspace_bytes": st.workspace_bytes, "total_kernel_launches": st.total_kernel_launches,
                "mode_product_launches": st.mode_product_launches, "mode_product_ms": st.mode_product_ms,
                "mode_product_flops": st.mode_product_flops, "expm_launches": st.expm_launches,
                "expm_ms": st.expm_ms,
                "block_plans": [(st.block_plan[b].s, st.block_plan[b].q) for b in range(max(st.nblocks, 1))],
                "i8_mode_launches": st.i8_mode_launches, "i8_launches": st.i8_launches, "i8_ms": st.i8_ms,
                "i8_flops": st.i8_flops, "i8_gemm_launches": st.i8_gemm_launches, "i8_gemm_ms": st.i8_gemm_ms,
                "i8_chained_ops": st.i8_chained_ops, "shard_digit_ops": st.shard_digit_ops,
                "presplit_inputs": st.presplit_inputs,
                "i8_kblocks": st.i8_kblocks, "i8_kblocks_run": st.i8_kblocks_run}

    GEMM_PATHS = {"auto": 0, "dmma": 1, "i8": 2}

    def set_gemm_path(self, path: str):
        """μ-mode-product path of the Tucker launches: "auto", "dmma" or "i8"."""
        _lib.check(_lib.load().phiks_set_gemm_path(self._h, self.GEMM_PATHS[path]), "phiks_set_gemm_path")

    OPTIONS = {"split": 0, "chain": 1, "graphs": 2, "presplit": 3, "kskip": 4}

    def set_option(self, name: str, value: int):
        """Execution option of the handle (include/phiks.h PHIKS_OPT_*): "split" 0/1/2,
        "chain" 0 (off) / 1 (guarded, default) / 2 (forced), "graphs" 0/1, "presplit" 0/1,
        "kskip" 0/1 (zero E digit blocks skipped by the int8 GEMM, default 1)."""
        _lib.check(_lib.load().phiks_set_option(self._h, self.OPTIONS[name], int(value)), "phiks_set_option")

    def get_option(self, name: str) -> int:
        v = ctypes.c_int()
        _lib.check(_lib.load().phiks_get_option(self._h, self.OPTIONS[name], ctypes.byref(v)), "phiks_get_option")
        return v.value

    def set_profiling(self, on: bool = True):
        _lib.check(_lib.load().phiks_set_profiling(self._h, 1 if on else 0), "phiks_set_profiling")

    def wait(self):
        """Block until the last apply (kernels and host copies) has finished."""
        _lib.check(_lib.load().phiks_wait(self._h), "phiks_wait")


# ----------------------------------------------------------------------
def mode_product(dims: Sequence[int], mu: int, ins: Sequence, Ms: Sequence, outs: Sequence, stream=None):
    """Batched μ-mode product out_b = in_b ×_{mu+1} M_b (0-based mu)."""
    lib = _lib.load()
    N = int(np.prod(dims))
    n_arr = (ctypes.c_int * len(dims))(*dims)
    _lib.check(lib.phiks_mode_product(len(dims), n_arr, int(mu), len(ins),
                                      _lib.ptr_array([_check_dev(t, N) for t in ins]),
                                      _lib.ptr_array([_check_dev(M) for M in Ms]),
                                      _lib.ptr_array([_check_dev(t, N) for t in outs]), _stream_ptr(stream)),
               "phiks_mode_product")


def mode_product_i8(dims: Sequence[int], mu: int, ins: Sequence, Ms: Sequence, outs: Sequence, slices: int = 8,
                    workspace=None, stream=None):
    """mode_product on the int8 tensor cores (exact 7-bit slicing)."""
    lib = _lib.load()
    torch = _torch()
    N = int(np.prod(dims))
    n_arr = (ctypes.c_int * len(dims))(*dims)
    need = ctypes.c_size_t(0)
    _lib.check(lib.phiks_mode_product_i8_workspace(len(dims), n_arr, int(mu), int(slices), len(ins),
                                                   ctypes.byref(need)), "phiks_mode_product_i8_workspace")
    if workspace is None or workspace.numel() < need.value:
        workspace = torch.empty(max(need.value, 1), dtype=torch.uint8, device=ins[0].device)
    _lib.check(lib.phiks_mode_product_i8(len(dims), n_arr, int(mu), int(slices), len(ins),
                                         _lib.ptr_array([_check_dev(t, N) for t in ins]),
                                         _lib.ptr_array([_check_dev(M) for M in Ms]),
                                         _lib.ptr_array([_check_dev(t, N) for t in outs]), workspace.data_ptr(),
                                         workspace.numel(), _stream_ptr(stream)), "phiks_mode_product_i8")
    return workspace


def tucker(dims: Sequence[int], x, Ms: Sequence, out, scratch=None, stream=None):
    lib = _lib.load()
    torch = _torch()
    N = int(np.prod(dims))
    if scratch is None and len(dims) > 1:
        scratch = torch.empty(2 * N, dtype=torch.float64, device=x.device)
    n_arr = (ctypes.c_int * len(dims))(*dims)
    _lib.check(lib.phiks_tucker(len(dims), n_arr, _check_dev(x, N), _lib.ptr_array([_check_dev(M) for M in Ms]),
                                _check_dev(out, N), scratch.data_ptr() if scratch is not None else None,
                                _stream_ptr(stream)), "phiks_tucker")


def expm(A, c: float = 1.0, stream=None):
    """exp(c·A) for a square fp64 CUDA matrix stored column-major (n*n elements)."""
    lib = _lib.load()
    torch = _torch()
    n = int(round(A.numel() ** 0.5))
    E = torch.empty_like(A)
    scratch = torch.empty(8 * n * n + 256, dtype=torch.float64, device=A.device)
    _lib.check(lib.phiks_expm(n, _check_dev(A), float(c), E.data_ptr(), scratch.data_ptr(), _stream_ptr(stream)),
               "phiks_expm")
    return E


def fp64_peak_launch(kind: int, blocks: int, iters: int, sink, stream=None) -> float:
    """Launch the DMMA (kind 0) / DFMA (kind 1) microbenchmark; returns its flop count."""
    lib = _lib.load()
    fl = ctypes.c_double()
    _lib.check(lib.phiks_fp64_peak_launch(int(kind), int(blocks), int(iters), _check_dev(sink), _stream_ptr(stream),
                                          ctypes.byref(fl)), "phiks_fp64_peak_launch")
    return fl.value


from .sharding import ShardedPhiKS, apply_ranks_serial  # noqa: E402
