"""ctypes binding of libphiks.so (include/phiks.h).  Argument marshalling only:
every compute step runs in the library's CUDA kernels.  There is no fallback:
if the library is missing or no CUDA device is present, calls raise."""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PHIKS_LIB_PATH") or os.path.join(_HERE, "libphiks.so")  # override: experiments only
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "phiks.h")

MODE_SAME_VECTOR = 0
MODE_LINCOMB = 1
MEM_DEVICE = 0
MEM_HOST = 1
MEM_HOST_ASYNC = 2
MAX_D, MAX_P, MAX_SCALES, MAX_N, MAX_BLOCKS = 8, 6, 16, 4096, 4
IPC_HANDLE_BYTES = 64
MAX_RANKS = 8

_STATUS = {0: "PHIKS_OK", 1: "PHIKS_ERR_ARG", 2: "PHIKS_ERR_CUDA", 3: "PHIKS_ERR_PLAN",
           4: "PHIKS_ERR_NOMEM", 5: "PHIKS_ERR_WORKSPACE", 6: "PHIKS_ERR_LIMIT"}


class PhiksError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(code, code)}: {msg}")
        self.code = code


class Request(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("n_ells", ctypes.c_int), ("ells", ctypes.POINTER(ctypes.c_int)),
                ("n_scales", ctypes.c_int), ("tau", ctypes.c_double), ("tol", ctypes.c_double),
                ("force_s", ctypes.c_int), ("force_q", ctypes.c_int), ("mem_kind", ctypes.c_int)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("s", ctypes.c_int), ("q", ctypes.c_int), ("T_formula", ctypes.c_int),
                ("T_executed", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("plan", PlanInfo), ("kernel_launches", ctypes.c_int64), ("tucker_ops", ctypes.c_int64),
                ("mu_mode_flops", ctypes.c_double), ("expm_flops", ctypes.c_double),
                ("workspace_bytes", ctypes.c_size_t), ("total_kernel_launches", ctypes.c_int64),
                ("mode_product_launches", ctypes.c_int64), ("mode_product_ms", ctypes.c_double),
                ("mode_product_flops", ctypes.c_double), ("expm_launches", ctypes.c_int64),
                ("expm_ms", ctypes.c_double), ("nblocks", ctypes.c_int), ("block_plan", PlanInfo * 4),
                ("i8_mode_launches", ctypes.c_int64), ("i8_launches", ctypes.c_int64), ("i8_ms", ctypes.c_double),
                ("i8_flops", ctypes.c_double), ("i8_gemm_launches", ctypes.c_int64), ("i8_gemm_ms", ctypes.c_double),
                ("i8_chained_ops", ctypes.c_int64), ("shard_digit_ops", ctypes.c_int64),
                ("presplit_inputs", ctypes.c_int64),
                ("i8_kblocks", ctypes.c_int64), ("i8_kblocks_run", ctypes.c_int64)]


_lib = None


def load() -> ctypes.CDLL:
    """Load libphiks.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built — run __graft_entry__.build() (make -C paper_2210_07667_b200/csrc)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    P = ctypes.POINTER
    lib.phiks_create.argtypes = [i, P(i), P(vp), P(vp)]
    lib.phiks_destroy.argtypes = [vp]
    lib.phiks_plan.argtypes = [vp, P(Request), P(d), P(PlanInfo)]
    lib.phiks_apply.argtypes = [vp, P(Request), i, P(vp), P(vp), vp, ctypes.c_size_t, vp]
    lib.phiks_workspace_size.argtypes = [vp, P(Request), P(PlanInfo), P(ctypes.c_size_t)]
    lib.phiks_get_stats.argtypes = [vp, P(Stats)]
    lib.phiks_mode_product.argtypes = [i, P(i), i, i, P(vp), P(vp), P(vp), vp]
    lib.phiks_tucker.argtypes = [i, P(i), vp, P(vp), vp, vp, vp]
    lib.phiks_expm.argtypes = [i, vp, d, vp, vp, vp]
    lib.phiks_fp64_peak_launch.argtypes = [i, i, ctypes.c_int64, vp, vp, P(d)]
    lib.phiks_plan_host.argtypes = [i, P(i), P(vp), P(Request), P(d), P(PlanInfo)]
    lib.phiks_select_plan.argtypes = [i, d, d, d, d, i, P(d), d, i, i, i, P(PlanInfo)]
    lib.phiks_set_profiling.argtypes = [vp, i]
    lib.phiks_create_sharded.argtypes = [i, P(i), P(vp), i, i, P(vp)]
    lib.phiks_create_blocks.argtypes = [i, i, P(i), P(vp), P(vp)]
    lib.phiks_create_sharded_blocks.argtypes = [i, i, P(i), P(vp), i, i, P(vp)]
    lib.phiks_create_sharded_complex.argtypes = [i, P(i), P(vp), i, i, P(vp)]
    lib.phiks_create_blocks_complex.argtypes = [i, i, P(i), P(vp), P(vp)]
    lib.phiks_create_sharded_blocks_complex.argtypes = [i, i, P(i), P(vp), i, i, P(vp)]
    lib.phiks_shard_info.argtypes = [vp, P(i), P(i), P(ctypes.c_int64), P(ctypes.c_size_t)]
    lib.phiks_shard_ipc_handle.argtypes = [vp, vp]
    lib.phiks_shard_open_peers.argtypes = [vp, vp]
    lib.phiks_shard_base.argtypes = [vp, P(vp)]
    lib.phiks_shard_set_peer_bases.argtypes = [vp, P(vp)]
    lib.phiks_apply_ranks_serial.argtypes = [P(vp), i, P(Request), i, P(vp), P(vp), vp]
    lib.phiks_apply_ranks_serial_ex.argtypes = [P(vp), i, P(Request), i, P(vp), P(vp), vp, i]
    lib.phiks_wait.argtypes = [vp]
    lib.phiks_set_gemm_path.argtypes = [vp, i]
    lib.phiks_set_option.argtypes = [vp, i, i]
    lib.phiks_get_option.argtypes = [vp, i, P(i)]
    lib.phiks_mode_product_i8_workspace.argtypes = [i, P(i), i, i, i, P(ctypes.c_size_t)]
    lib.phiks_mode_product_i8.argtypes = [i, P(i), i, i, i, P(vp), P(vp), P(vp), vp, ctypes.c_size_t, vp]
    lib.phiks_create_complex.argtypes = [i, P(i), P(vp), P(vp)]
    lib.phiks_plan_host_complex.argtypes = [i, P(i), P(vp), P(Request), P(d), P(PlanInfo)]
    lib.phiks_shard_peer_base.argtypes = [vp, i, P(vp)]
    lib.phiks_shard_layout.argtypes = [i, P(i), i, i, i, P(ctypes.c_int64)]
    lib.phiks_shard_layout_ex.argtypes = [i, P(i), i, i, i, P(ctypes.c_int64)]
    lib.phiks_last_error.restype = ctypes.c_char_p
    lib.phiks_version.restype = ctypes.c_char_p
    for name in ("phiks_create", "phiks_destroy", "phiks_plan", "phiks_apply", "phiks_workspace_size",
                 "phiks_get_stats", "phiks_mode_product", "phiks_tucker", "phiks_expm",
                 "phiks_fp64_peak_launch", "phiks_plan_host", "phiks_select_plan", "phiks_set_profiling",
                 "phiks_create_sharded", "phiks_shard_info", "phiks_shard_ipc_handle", "phiks_shard_open_peers",
                 "phiks_shard_base", "phiks_shard_set_peer_bases", "phiks_apply_ranks_serial", "phiks_apply_ranks_serial_ex", "phiks_shard_layout", "phiks_wait", "phiks_shard_peer_base", "phiks_create_complex", "phiks_plan_host_complex", "phiks_create_blocks",
                 "phiks_create_sharded_blocks", "phiks_shard_layout_ex",
                 "phiks_create_sharded_complex", "phiks_create_blocks_complex",
                 "phiks_create_sharded_blocks_complex",
                 "phiks_mode_product_i8_workspace", "phiks_mode_product_i8", "phiks_set_gemm_path",
                 "phiks_set_option", "phiks_get_option"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def header_functions() -> list:
    """Names of the functions include/phiks.h declares."""
    import re
    src = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(phiks_[a-z0-9_]+)\s*\(", src)))


def check(code: int, where: str) -> None:
    if code != 0:
        raise PhiksError(code, where, load().phiks_last_error().decode())


def ptr_array(ptrs: Sequence[int]):
    arr = (ctypes.c_void_p * max(len(ptrs), 1))()
    for k, p in enumerate(ptrs):
        arr[k] = ctypes.c_void_p(int(p))
    return arr


def make_request(mode: int, ells: Sequence[int], n_scales: int, tau: float, tol: float = 0.0,
                 force_s: int = -1, force_q: int = -1, mem_kind: int = MEM_DEVICE):
    ells_arr = (ctypes.c_int * len(ells))(*[int(e) for e in ells])
    req = Request(mode, len(ells), ctypes.cast(ells_arr, ctypes.POINTER(ctypes.c_int)), int(n_scales),
                  float(tau), float(tol), int(force_s), int(force_q), int(mem_kind))
    req._keep = ells_arr  # keep the array alive with the struct
    return req
