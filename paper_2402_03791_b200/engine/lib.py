"""ctypes binding of ``libzpp.so`` (the C ABI in ``include/zpp.h``).

This is the only way the engine reaches the GPU: there is no CPU or eager
fallback.  If the shared library is missing or a call fails, a RuntimeError is
raised with ``zpp_last_error()``.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_float, c_int, c_longlong, c_uint64, c_ulonglong, c_void_p

_PKG = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(_PKG, "libzpp.so")

c_size = c_longlong
c_stream = c_uint64
P = c_void_p

_SIGS = {
    "zpp_last_error": (c_char_p, []),
    "zpp_num_sms": (c_int, []),
    "zpp_version": (c_int, []),
    "zpp_gemm": (c_int, [P, c_int, c_size, P, c_int, c_size, P, c_size, c_int, c_int, c_int, c_int,
                         P, P, c_size, P, c_size, c_stream]),
    "zpp_gemm_set_cta_group": (c_int, [c_int]),
    "zpp_gemm_set_streamk": (c_int, [c_int]),
    "zpp_attn_fwd": (c_int, [P, P, P, c_int, c_int, c_int, c_int, c_stream]),
    "zpp_attn_bwd": (c_int, [P, P, P, P, P, P, c_int, c_int, c_int, c_int, c_stream]),
    "zpp_attn_bwd_workspace_floats": (c_longlong, [c_int, c_int, c_int, c_int]),
    "zpp_layernorm_fwd": (c_int, [P, P, P, P, P, P, c_int, c_int, c_float, c_stream]),
    "zpp_layernorm_bwd": (c_int, [P, P, P, P, P, P, P, P, P, P, c_int, c_int, c_int, c_stream]),
    "zpp_layernorm_bwd_workspace_floats": (c_longlong, [c_int, c_int]),
    "zpp_norm_param_grads": (c_int, [P, P, P, P, P, P, P, c_int, c_int, c_int, c_stream]),
    "zpp_rmsnorm_fwd": (c_int, [P, P, P, P, c_int, c_int, c_float, c_stream]),
    "zpp_rmsnorm_bwd": (c_int, [P, P, P, P, P, P, P, P, c_int, c_int, c_int, c_stream]),
    "zpp_swiglu_fwd": (c_int, [P, P, c_int, c_int, c_stream]),
    "zpp_swiglu_bwd": (c_int, [P, P, P, c_int, c_int, c_stream]),
    "zpp_rope": (c_int, [P, c_int, c_int, c_int, c_int, c_float, c_int, c_stream]),
    "zpp_colsum_acc": (c_int, [P, c_size, P, P, c_int, c_int, c_int, c_stream]),
    "zpp_gelu_fwd": (c_int, [P, P, c_size, c_stream]),
    "zpp_embed_fwd": (c_int, [P, P, P, P, c_int, c_int, c_int, c_stream]),
    "zpp_embed_bwd": (c_int, [P, P, P, P, c_int, c_int, c_int, c_int, c_stream]),
    "zpp_xent_fwd_bwd": (c_int, [P, c_size, P, P, c_int, c_int, c_float, c_stream]),
    "zpp_cast_scale_f32_bf16": (c_int, [P, P, c_size, c_float, c_stream]),
    "zpp_accum_bf16_f32": (c_int, [P, P, c_size, c_stream]),
    "zpp_accum_f32_f32": (c_int, [P, P, c_size, c_stream]),
    "zpp_adamw": (c_int, [P, P, P, P, P, c_size, c_float, c_float, c_float, c_float, c_float, c_int,
                          c_stream]),
    "zpp_init_param": (c_int, [P, P, c_size, c_ulonglong, c_size, c_float, c_float, c_stream]),
    "zpp_zero": (c_int, [P, c_size, c_stream]),
    "zpp_preload_kernels": (c_int, []),
    "zpp_nccl_load": (c_int, [c_char_p]),
    "zpp_nccl_unique_id": (c_int, [c_char_p]),
    "zpp_comm_init": (c_int, [c_char_p, c_int, c_int, POINTER(c_void_p)]),
    "zpp_comm_destroy": (c_int, [P]),
    "zpp_allgather": (c_int, [P, P, P, c_size, c_int, c_stream]),
    "zpp_reduce_scatter": (c_int, [P, P, P, c_size, c_int, c_stream]),
    "zpp_allreduce": (c_int, [P, P, P, c_size, c_int, c_stream]),
    "zpp_send": (c_int, [P, P, c_size, c_int, c_int, c_stream]),
    "zpp_recv": (c_int, [P, P, c_size, c_int, c_int, c_stream]),
}

EPI_BF16, EPI_BF16_GELU, EPI_BF16_DGELU, EPI_F32, EPI_F32_ACC = range(5)

_lib = None


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def load() -> ctypes.CDLL:
    """Load libzpp.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libzpp.so not found at {LIB_PATH}: build it with "
                           "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load().zpp_last_error().decode(errors="replace")
        raise RuntimeError(f"libzpp {what} failed (rc={rc}): {msg}")


_DEBUG_SYNC = os.environ.get("ZPP_DEBUG_SYNC") == "1"


def call(name: str, *args) -> None:
    if _DEBUG_SYNC:  # debugging aid: log and synchronize every launch
        import sys
        import torch
        print(f"[zpp] {name}", file=sys.stderr, flush=True)
        check(getattr(load(), name)(*args), name)
        torch.cuda.synchronize()
        print(f"[zpp] {name} done", file=sys.stderr, flush=True)
        return
    check(getattr(load(), name)(*args), name)


def nccl_path() -> str:
    import nvidia.nccl  # the NCCL torch itself loads (pip nvidia-nccl-cu12)
    for base in list(getattr(nvidia.nccl, "__path__", [])):
        p = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    raise RuntimeError("libnccl.so.2 from the nvidia-nccl wheel not found")


def load_nccl() -> None:
    call("zpp_nccl_load", nccl_path().encode())
