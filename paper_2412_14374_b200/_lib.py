"""ctypes binding of libpp200.so (include/pp200.h).

The library is the only compute path: there is no CPU or eager-PyTorch
fallback.  ``lib()`` raises ``RuntimeError`` when the shared object is
missing, and every wrapper raises ``ExecutorFault``-compatible
``PC Error`` on a non-zero status.
"""
from __future__ import annotations

import ctypes
import pathlib
import threading

HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = HERE / "libpp200.so"

PC_F32, PC_F64, PC_BF16, PC_I32 = 0, 1, 2, 3

EPI_BIAS = 1
EPI_GELU = 2
EPI_RESIDUAL = 4
EPI_GELU_GRAD = 8
EPI_ACCUM = 16
EPI_RELU = 32
EPI_RELU_GRAD = 64
EPI_SPLITK_ZERO_C = 128
EPI_SPLITK_ORDERED = 256

_c_i = ctypes.c_int
_c_i64 = ctypes.c_int64
_c_p = ctypes.c_void_p
_c_f = ctypes.c_float
_c_d = ctypes.c_double

# name -> argtypes (all return int status unless listed in _RESTYPES)
SIGNATURES: dict[str, list] = {
    "pc_version": [],
    "pc_device_sm_count": [],
    "pc_gemm": [_c_i, _c_i, _c_i, _c_i, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64,
                _c_p, _c_i64, _c_i, _c_p, _c_p, _c_i64, _c_p, _c_i64, _c_p],
    "pc_gemm_set_tile_n": [_c_i],
    "pc_gemm_tile_choice": [_c_i, _c_i64, _c_i64, _c_i64, _c_i, ctypes.POINTER(_c_i),
                            ctypes.POINTER(_c_i), ctypes.POINTER(_c_i)],
    "pc_gemm_set_tma_store": [_c_i],
    "pc_gemm_set_cta_pair": [_c_i],
    "pc_gemm_set_ablation": [_c_i],
    "pc_fill": [_c_i, _c_i64, _c_d, _c_p, _c_p],
    "pc_ewise": [_c_i, _c_i, _c_i64, _c_p, _c_p, _c_i64, _c_p, _c_p],
    "pc_sumsq_half": [_c_i, _c_i64, _c_p, _c_p, _c_p],
    "pc_sum_f32": [_c_i64, _c_p, _c_p, _c_p],
    "pc_col_sum": [_c_i, _c_i, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i, _c_p, _c_i64, _c_p],
    "pc_reduce_workspace_bytes": [_c_i64, _c_i64, ctypes.POINTER(_c_i64)],
    "pc_copy2d": [_c_i, _c_i64, _c_i64, _c_p, _c_i64, _c_i, _c_p, _c_i64, _c_p],
    "pc_accumulate": [_c_i, _c_i, _c_i64, _c_p, _c_p, _c_p],
    "pc_peer_alloc": [_c_i64, ctypes.POINTER(_c_p), _c_p],
    "pc_peer_free": [_c_p],
    "pc_peer_open": [_c_p, ctypes.POINTER(_c_p)],
    "pc_peer_close": [_c_p],
    "pc_stream_write_u32": [_c_p, ctypes.c_uint32, _c_p],
    "pc_stream_wait_u32": [_c_p, ctypes.c_uint32, _c_p],
    "pc_peer_copy": [_c_p, _c_p, _c_i64, _c_p],
    "pc_peer_wait": [_c_p, _c_p, _c_p],
    "pc_host_word_alloc": [ctypes.POINTER(_c_p), ctypes.POINTER(_c_p)],
    "pc_host_word_free": [_c_p],
    "pc_graph_kernel_nodes": [_c_p, ctypes.POINTER(_c_i64)],
    "pc_sgd_update": [_c_i, _c_i64, _c_p, _c_p, _c_d, _c_p, _c_p, _c_p],
    "pc_cast": [_c_i, _c_i, _c_i64, _c_p, _c_p, _c_p],
    "pc_timestamp": [_c_p, _c_p],
    "pc_layernorm_fwd": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_f, _c_p],
    "pc_layernorm_bwd": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                         _c_p, _c_p, _c_i64, _c_p],
    "pc_layernorm_bwd_acc": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                             _c_p, _c_p, _c_i, _c_p, _c_i64, _c_p],
    "pc_layernorm_partial_rows": [_c_i64, _c_i64, ctypes.POINTER(_c_i64)],
    "pc_layernorm_bwd_partials": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                  _c_p, _c_i64, _c_p],
    "pc_layernorm_param_grads": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_i,
                                 _c_p, _c_i64, _c_p],
    "pc_layernorm_param_bias_grads": [_c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                                      _c_p, _c_p, _c_p, _c_i, _c_p],
    "pc_rmsnorm_fwd": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_f, _c_p],
    "pc_rmsnorm_bwd": [_c_i, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p, _c_p,
                       _c_i64, _c_p],
    "pc_rope": [_c_i, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_f, _c_i, _c_p],
    "pc_swiglu_fwd": [_c_i, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p],
    "pc_swiglu_bwd": [_c_i, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p],
    "pc_gqa_kv": [_c_i, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_i, _c_p],
    "pc_embedding_fwd": [_c_i, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p],
    "pc_embedding_bwd_workspace_bytes": [_c_i64, ctypes.POINTER(_c_i64)],
    "pc_embedding_bwd": [_c_i, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_p,
                         _c_i64, _c_p],
    "pc_embedding_bwd_acc": [_c_i, _c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_p, _c_p, _c_p, _c_i,
                             _c_p, _c_i64, _c_p],
    "pc_xent_fwd_bwd": [_c_i, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_p, _c_p],
    "pc_attention_fwd": [_c_i, _c_i, _c_i, _c_i, _c_i, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_p],
    "pc_attention_bwd": [_c_i, _c_i, _c_i, _c_i, _c_i, _c_p, _c_i64, _c_p, _c_p, _c_i64, _c_p,
                         _c_p, _c_p, _c_i64, _c_p],
    "pc_attention_gqa_fwd": [_c_i, _c_i, _c_i, _c_i, _c_i, _c_i, _c_p, _c_i64, _c_p, _c_i64, _c_p,
                             _c_p],
    "pc_attention_gqa_bwd": [_c_i, _c_i, _c_i, _c_i, _c_i, _c_i, _c_p, _c_i64, _c_p, _c_p, _c_i64,
                             _c_p, _c_p, _c_p, _c_i64, _c_p],
    "pc_attention_set_impl": [_c_i],
    "pc_attention_tune": [_c_i, _c_i],
    "pc_gemm_set_max_split": [_c_i],
    "pc_gemm_wgrad_pair": [_c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64,
                           _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_i, _c_p, _c_i64, _c_p],
    "pc_colsum_set_cluster": [_c_i],
    "pc_lmhead_xent_workspace": [_c_i64, _c_i64, _c_i64, ctypes.POINTER(_c_i64), ctypes.POINTER(_c_i64)],
    "pc_lmhead_xent_fwd": [_c_i64, _c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_p,
                           _c_i64, _c_p, _c_i64, _c_p, _c_p],
    "pc_lmhead_xent_bwd": [_c_i64, _c_i64, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p, _c_i64, _c_p,
                           _c_i64, _c_p, _c_i64, _c_i, _c_p],
    "pc_p2p_available": [],
    "pc_p2p_unique_id": [_c_p],
    "pc_p2p_comm_init": [ctypes.POINTER(_c_p), _c_i, _c_p, _c_i],
    "pc_p2p_send": [_c_p, _c_p, _c_i64, _c_i, _c_p],
    "pc_p2p_recv": [_c_p, _c_p, _c_i64, _c_i, _c_p],
    "pc_p2p_abort": [_c_p],
    "pc_p2p_destroy": [_c_p],
}

EW_ADD, EW_MUL, EW_RELU, EW_RELU_GRAD = 1, 2, 3, 4
_RESTYPES = {"pc_last_error": ctypes.c_char_p}


class PCError(RuntimeError):
    """Non-zero status from a libpp200 entry point."""


_lock = threading.Lock()
_lib = None


def lib_path() -> pathlib.Path:
    return LIB_PATH


def lib():
    """Load libpp200.so once; fail loudly if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2412_14374_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        L.pc_last_error.restype = ctypes.c_char_p
        L.pc_last_error.argtypes = []
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = ctypes.c_int
        _lib = L
        return _lib


def exported_symbols() -> list[str]:
    return ["pc_last_error", *SIGNATURES]


# C-ABI calls that launch at least one kernel, counted for bench.py's gpu_launches.
_NON_LAUNCH = {"pc_version", "pc_device_sm_count", "pc_gemm_set_tile_n", "pc_gemm_tile_choice", "pc_attention_set_impl", "pc_attention_tune",
               "pc_gemm_set_tma_store", "pc_gemm_set_cta_pair", "pc_gemm_set_max_split", "pc_colsum_set_cluster", "pc_gemm_set_ablation",
               "pc_embedding_bwd_workspace_bytes", "pc_reduce_workspace_bytes", "pc_p2p_available", "pc_p2p_unique_id",
               "pc_p2p_comm_init", "pc_p2p_abort", "pc_p2p_destroy",
               "pc_peer_alloc", "pc_peer_free", "pc_peer_open", "pc_peer_close",
               "pc_stream_write_u32", "pc_stream_wait_u32", "pc_graph_kernel_nodes",
               "pc_host_word_alloc", "pc_host_word_free", "pc_lmhead_xent_workspace",
               "pc_layernorm_partial_rows"}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    if name not in _NON_LAUNCH:
        launch_count += 1
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = lib().pc_last_error().decode(errors="replace")
        raise PCError(f"{name} failed ({rc}): {msg}")
