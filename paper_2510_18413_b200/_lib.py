"""ctypes binding of the C ABI (include/adamas_b200.h).

The product path is the CUDA library only: if libadamas_b200.so is missing or
fails to load this module raises — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

ADAMAS_OK = 0
ADAMAS_ERR_CONFIG = 1
ADAMAS_ERR_RUNTIME = 2
ADAMAS_F32 = 0
ADAMAS_BF16 = 1
ADAMAS_STATUS_DEGENERATE = 1
ADAMAS_STATUS_SYNC_TIMEOUT = 4
ADAMAS_STATUS_PEER_TIMEOUT = 8
ADAMAS_STATUS_BAD_SELECTION = 16
TUNING_FIELDS = ("qsplit", "cluster", "P", "stages", "smem_kb", "exact_encode", "dbg", "no_pdl", "composed",
                 "require_fused")

EXPORTED = [
    "adamas_version", "adamas_last_error", "adamas_cache_create", "adamas_cache_destroy",
    "adamas_cache_seq_len", "adamas_cache_truncate", "adamas_cache_buffers", "adamas_cache_status",
    "adamas_cache_append", "adamas_cache_append_coded", "adamas_cache_codes_ref",
    "adamas_encode_query", "adamas_score", "adamas_topk", "adamas_sparse_attention",
    "adamas_decode_step", "adamas_decode_step_batched", "adamas_codes_ref_to_planes",
    "adamas_codes_planes_to_ref", "adamas_debug_trace", "adamas_seq_local_candidates",
    "adamas_seq_select_attend", "adamas_lse_merge", "adamas_seq_select_attend_merge", "adamas_cache_save_adkv", "adamas_cache_load_adkv",
    "adamas_score_metric", "adamas_hsel_create", "adamas_hsel_destroy", "adamas_hsel_build",
    "adamas_hsel_codes_ref", "adamas_hsel_select", "adamas_dot_topk", "adamas_page_select",
    "adamas_attention_f64", "adamas_topk_f64", "adamas_pages_create", "adamas_pages_destroy",
    "adamas_pages_build", "adamas_pages_select", "adamas_mailbox_create", "adamas_mailbox_ipc_handle",
    "adamas_mailbox_connect", "adamas_mailbox_connect_local", "adamas_mailbox_status", "adamas_mailbox_destroy",
    "adamas_seq_p2p_local", "adamas_seq_p2p_select_attend", "adamas_seq_p2p_merge", "adamas_seq_step_p2p",
    "adamas_set_tuning", "adamas_get_tuning",
]


class ConfigError(ValueError):
    """Mirror of adamas::ConfigError (include/adamas/common.hpp:19-22)."""


class AdamasRuntimeError(RuntimeError):
    pass


_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    lib = os.environ.get("ADAMAS_LIB", LIB)  # A/B experiments may point at another build of the same ABI
    if not os.path.exists(lib):
        raise ImportError(f"{lib} is not built; run __graft_entry__.build() (no CPU fallback exists)")
    L = C.CDLL(lib)
    vp, i32, i64, sz = C.c_void_p, C.c_int, C.c_int64, C.c_size_t
    L.adamas_version.restype = C.c_char_p
    L.adamas_last_error.restype = C.c_char_p
    L.adamas_cache_create.argtypes = [C.POINTER(vp), i32, i32, i32, i64, i32]
    L.adamas_cache_destroy.argtypes = [vp]
    L.adamas_cache_seq_len.argtypes = [vp, C.POINTER(i64)]
    L.adamas_cache_truncate.argtypes = [vp, i64]
    L.adamas_cache_buffers.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
    L.adamas_cache_status.argtypes = [vp, vp, C.POINTER(i32)]
    L.adamas_cache_append.argtypes = [vp, vp, vp, i64, vp]
    L.adamas_cache_append_coded.argtypes = [vp, vp, vp, vp, i64, vp]
    L.adamas_cache_codes_ref.argtypes = [vp, i64, i64, vp, vp]
    L.adamas_encode_query.argtypes = [vp, vp, i32, vp, vp]
    L.adamas_score.argtypes = [vp, vp, i32, vp, vp]
    L.adamas_topk.argtypes = [vp, i32, i64, i64, vp, vp]
    L.adamas_sparse_attention.argtypes = [vp, vp, i32, vp, i64, vp, vp, vp]
    L.adamas_decode_step.argtypes = [vp, vp, i32, vp, vp, i64, vp, vp, vp]
    L.adamas_decode_step_batched.argtypes = [C.POINTER(vp), i32, vp, i32, vp, vp, i64, vp, vp, vp]
    L.adamas_codes_ref_to_planes.argtypes = [vp, i64, vp]
    L.adamas_codes_planes_to_ref.argtypes = [vp, i64, vp]
    L.adamas_debug_trace.argtypes = [vp]
    L.adamas_seq_local_candidates.argtypes = [vp, vp, i32, vp, vp, i32, i64, i64, vp, vp]
    L.adamas_seq_select_attend.argtypes = [vp, vp, i32, vp, i32, i64, i64, i64, vp, vp, vp]
    L.adamas_lse_merge.argtypes = [vp, i32, i32, vp, vp]
    L.adamas_seq_select_attend_merge.argtypes = [vp, vp, i32, vp, i32, i64, i64, i64, vp, i32, vp, vp, vp]
    L.adamas_cache_save_adkv.argtypes = [vp, i32, C.c_char_p, vp]
    L.adamas_score_metric.argtypes = [vp, vp, i32, i32, vp, vp]
    L.adamas_cache_load_adkv.argtypes = [vp, C.POINTER(C.c_char_p), i32, vp]
    L.adamas_hsel_create.argtypes = [C.POINTER(vp), i32, i32, i32]
    L.adamas_hsel_destroy.argtypes = [vp]
    L.adamas_hsel_build.argtypes = [vp, vp, i64, i64, vp]
    L.adamas_hsel_codes_ref.argtypes = [vp, i64, i64, vp, vp]
    L.adamas_hsel_select.argtypes = [vp, vp, i64, i64, i32, i64, vp, vp]
    L.adamas_dot_topk.argtypes = [vp, vp, i64, i64, i64, i64, i32, i64, vp, vp, vp]
    L.adamas_pages_create.argtypes = [C.POINTER(vp), i64, i32]
    L.adamas_pages_destroy.argtypes = [vp]
    L.adamas_pages_build.argtypes = [vp, vp, i64, i64, vp]
    L.adamas_pages_select.argtypes = [vp, vp, i64, i64, i64, vp, vp, vp]
    L.adamas_mailbox_create.argtypes = [C.POINTER(vp), i32, i32, i32, i64]
    L.adamas_mailbox_ipc_handle.argtypes = [vp, vp]
    L.adamas_mailbox_connect.argtypes = [vp, vp]
    L.adamas_mailbox_connect_local.argtypes = [C.POINTER(vp), i32]
    L.adamas_mailbox_status.argtypes = [vp, C.POINTER(i32)]
    L.adamas_mailbox_destroy.argtypes = [vp]
    L.adamas_seq_p2p_local.argtypes = [vp, vp, vp, i32, vp, vp, i32, i64, vp]
    L.adamas_seq_p2p_select_attend.argtypes = [vp, vp, vp, i32, i64, i64, vp, vp]
    L.adamas_seq_p2p_merge.argtypes = [vp, vp, vp]
    L.adamas_seq_step_p2p.argtypes = [vp, vp, vp, i32, vp, vp, i32, i64, i64, vp, vp, vp]
    L.adamas_topk_f64.argtypes = [vp, i64, i64, i64, vp, vp]
    L.adamas_set_tuning.argtypes = [C.POINTER(i32), i32]
    L.adamas_get_tuning.argtypes = [C.POINTER(i32), i32]
    L.adamas_page_select.argtypes = [vp, vp, i64, i64, i64, i64, i32, i64, i64, vp, vp, vp]
    L.adamas_attention_f64.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp, i64, vp, vp, vp]
    for name in EXPORTED:
        if not hasattr(L, name):
            raise ImportError(f"{lib} does not export {name}")
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == ADAMAS_OK:
        return
    msg = load().adamas_last_error().decode()
    if rc == ADAMAS_ERR_CONFIG:
        raise ConfigError(msg)
    raise AdamasRuntimeError(msg)
