"""Python mirror of the reference operator API over the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/adamas/*.hpp) so parity tests read like the
reference's own tests; tensors are torch CUDA tensors (device memory and
streams are torch's plumbing), every computation runs in the sm_100a kernels
of libadamas_b200.so.

    reference (namespace adamas)            here
    KvCache(head_dim, bits)                 KvCache(n_kv_heads, capacity, dtype, head_dim, bits)
    KvCache::update(k, v, pack(encode(k)))  KvCache.update(keys, values)
    KvCache::update(k, v, code)             KvCache.update_coded(keys, values, codes_ref)
    KvCache::code_words(i)                  KvCache.code_words(start, n)
    pack(encode(q))                         KvCache.encode_query(q)
    score_all(q_code, cache, manhattan)     KvCache.score_all(q_codes)
    top_k(scores, k)                        top_k(scores, k)
    sparse_attention(q, cache, sel)         KvCache.sparse_attention(q, idx)
    select(adamas) + attend (sweep.cpp)     KvCache.decode_step(q, k_new, v_new, budget)
"""
from __future__ import annotations

import contextlib
import ctypes as C

import torch

from ._lib import (ADAMAS_BF16, ADAMAS_F32, ADAMAS_STATUS_BAD_SELECTION, ADAMAS_STATUS_DEGENERATE,
                   ADAMAS_STATUS_PEER_TIMEOUT, ADAMAS_STATUS_SYNC_TIMEOUT, TUNING_FIELDS, AdamasRuntimeError,
                   ConfigError, check, load)

HEAD_DIM = 128
_DTYPES = {torch.float32: ADAMAS_F32, torch.bfloat16: ADAMAS_BF16}


def _stream(stream=None) -> C.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def _need(t: torch.Tensor, dtype, shape_tail, what):
    if not t.is_cuda:
        raise ConfigError(f"{what}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ConfigError(f"{what}: dtype {t.dtype} != cache dtype {dtype}")
    if tuple(t.shape[-len(shape_tail):]) != tuple(shape_tail):
        raise ConfigError(f"{what}: shape {tuple(t.shape)} does not end in {shape_tail}")
    if not t.is_contiguous():
        raise ConfigError(f"{what}: must be contiguous")


class KvCache:
    """Device KV cache of one layer: K, V and 32 B codes per token per kv-head."""

    def __init__(self, n_kv_heads: int, capacity: int, dtype=torch.bfloat16, head_dim: int = HEAD_DIM,
                 bits: int = 2):
        self.L = load()
        if dtype not in _DTYPES:
            raise ConfigError(f"unsupported dtype {dtype}")
        h = C.c_void_p()
        check(self.L.adamas_cache_create(C.byref(h), n_kv_heads, head_dim, bits, capacity, _DTYPES[dtype]))
        self.h = h
        self.n_kv = n_kv_heads
        self.capacity = capacity
        self.dtype = dtype
        self.head_dim = head_dim
        self.bits = bits

    def close(self):
        if getattr(self, "h", None):
            self.L.adamas_cache_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ------------------------------------------------------------------
    @property
    def seq_len(self) -> int:
        v = C.c_int64()
        check(self.L.adamas_cache_seq_len(self.h, C.byref(v)))
        return v.value

    def truncate(self, n: int) -> None:
        check(self.L.adamas_cache_truncate(self.h, n))

    # -- ADKV snapshots (save_snapshot / load_snapshot, kv_cache.cpp:111-165) ----
    def save_snapshot(self, kv_head: int, path: str, stream=None) -> None:
        check(self.L.adamas_cache_save_adkv(self.h, kv_head, str(path).encode(), _stream(stream)))

    def load_snapshots(self, paths, stream=None) -> int:
        """Appends one reference snapshot per kv-head; returns seq_len."""
        arr = (C.c_char_p * len(paths))(*[str(x).encode() for x in paths])
        check(self.L.adamas_cache_load_adkv(self.h, arr, len(paths), _stream(stream)))
        return self.seq_len

    def buffers(self):
        k, v, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(self.L.adamas_cache_buffers(self.h, C.byref(k), C.byref(v), C.byref(c)))
        return k.value, v.value, c.value

    def keys(self) -> torch.Tensor:
        """View of the device key array [n_kv][capacity][128] (no copy)."""
        return self._view(self.buffers()[0])

    def values(self) -> torch.Tensor:
        return self._view(self.buffers()[1])

    def _view(self, addr):
        return _DeviceView(addr, (self.n_kv, self.capacity, self.head_dim), self.dtype).tensor()

    def status(self, stream=None) -> int:
        s = C.c_int()
        check(self.L.adamas_cache_status(self.h, _stream(stream), C.byref(s)))
        return s.value

    def raise_on_status(self, stream=None) -> None:
        """Reads and clears the sticky status word; raises what the reference
        would have thrown: ConfigError for a zero / non-finite vector
        (quantizer.cpp:46-47) or a bad gather (kv_cache.cpp:90-91,
        attention.cpp:42), a runtime error for a timed-out exchange."""
        st = self.status(stream)
        if st & ADAMAS_STATUS_BAD_SELECTION:
            raise ConfigError("KvCache: gather indices must be strictly increasing and in range "
                              "(or the selection is empty)")
        if st & ADAMAS_STATUS_DEGENERATE:
            raise ConfigError("degenerate scale: zero or non-finite vector encoded")
        if st & (ADAMAS_STATUS_SYNC_TIMEOUT | ADAMAS_STATUS_PEER_TIMEOUT):
            raise AdamasRuntimeError(f"device exchange timed out (status {st:#x}): results invalid")

    def raise_on_degenerate(self, stream=None) -> None:
        """quantizer.cpp:46-47: a zero / non-finite vector is a ConfigError."""
        self.raise_on_status(stream)

    # -- operators ----------------------------------------------------------------
    def update(self, keys: torch.Tensor, values: torch.Tensor, stream=None) -> int:
        """keys/values [n_tokens][n_kv][128] -> appended with their codes; returns seq_len."""
        _need(keys, self.dtype, (self.n_kv, self.head_dim), "update keys")
        _need(values, self.dtype, (self.n_kv, self.head_dim), "update values")
        n = keys.numel() // (self.n_kv * self.head_dim)
        check(self.L.adamas_cache_append(self.h, _ptr(keys), _ptr(values), n, _stream(stream)))
        return self.seq_len

    def update_coded(self, keys, values, codes_ref: torch.Tensor, stream=None) -> int:
        _need(keys, self.dtype, (self.n_kv, self.head_dim), "update keys")
        _need(values, self.dtype, (self.n_kv, self.head_dim), "update values")
        _need(codes_ref, torch.int16, (self.n_kv, 16), "update codes")
        n = keys.numel() // (self.n_kv * self.head_dim)
        check(self.L.adamas_cache_append_coded(self.h, _ptr(keys), _ptr(values), _ptr(codes_ref), n,
                                               _stream(stream)))
        return self.seq_len

    def code_words(self, start: int = 0, n: int | None = None, stream=None) -> torch.Tensor:
        """Reference-layout code words [n_kv][n][16] (int16 holding u16 bits)."""
        if n is None:
            n = self.seq_len - start
        out = torch.empty((self.n_kv, n, 16), dtype=torch.int16, device="cuda")
        check(self.L.adamas_cache_codes_ref(self.h, start, n, _ptr(out), _stream(stream)))
        return out

    def encode_query(self, q: torch.Tensor, stream=None) -> torch.Tensor:
        """pack(encode(q)) per head: q [n_q][128] -> int16 [n_q][16] reference words."""
        _need(q, self.dtype, (self.head_dim,), "encode_query q")
        n_q = q.numel() // self.head_dim
        out = torch.empty((n_q, 16), dtype=torch.int16, device="cuda")
        check(self.L.adamas_encode_query(self.h, _ptr(q), n_q, _ptr(out), _stream(stream)))
        return out

    METRICS = {"manhattan": 0, "euclidean_sq": 1, "hamming_1bit": 2}

    def score_all(self, q_codes: torch.Tensor, metric: str = "manhattan", stream=None) -> torch.Tensor:
        """int32 [n_q][seq_len] distances (estimator.cpp:45-59): Metric::manhattan
        (default), Metric::euclidean_sq, or the 1-bit pipeline's l1 ("hamming_1bit")."""
        if metric not in self.METRICS:
            raise ConfigError(f"unknown metric {metric}")
        n_q = q_codes.shape[0]
        out = torch.empty((n_q, self.seq_len), dtype=torch.int32, device="cuda")
        check(self.L.adamas_score_metric(self.h, _ptr(q_codes.contiguous()), n_q, self.METRICS[metric], _ptr(out),
                                         _stream(stream)))
        return out

    def sparse_attention(self, q: torch.Tensor, idx: torch.Tensor, with_lse: bool = False, validate: bool = True,
                         stream=None):
        """fp32 [n_q][128]; idx int32 [n_q][k] ascending (-1 ends a row).

        Rows are validated on the device (strictly increasing, in range, not
        empty); with validate=True (the reference's behaviour) a bad row raises
        ConfigError here, which synchronizes the stream."""
        _need(q, self.dtype, (self.head_dim,), "sparse_attention q")
        n_q = q.numel() // self.head_dim
        idx = idx.to(torch.int32).contiguous()
        out = torch.empty((n_q, self.head_dim), dtype=torch.float32, device="cuda")
        lse = torch.empty((n_q, 2), dtype=torch.float32, device="cuda") if with_lse else None
        check(self.L.adamas_sparse_attention(self.h, _ptr(q), n_q, _ptr(idx), idx.shape[-1], _ptr(out),
                                             _ptr(lse), _stream(stream)))
        if validate:
            self.raise_on_status(stream)
        return (out, lse) if with_lse else out

    def decode_step(self, q, k_new, v_new, budget: int, want_idx: bool = True, out=None, idx=None,
                    stream=None):
        """One fused decode step (append, encode, scan, select, attend)."""
        _need(q, self.dtype, (self.head_dim,), "decode q")
        _need(k_new, self.dtype, (self.n_kv, self.head_dim), "decode k_new")
        _need(v_new, self.dtype, (self.n_kv, self.head_dim), "decode v_new")
        n_q = q.numel() // self.head_dim
        if out is None:
            out = torch.empty((n_q, self.head_dim), dtype=torch.float32, device="cuda")
        if want_idx and idx is None:
            idx = torch.empty((n_q, budget), dtype=torch.int32, device="cuda")
        check(self.L.adamas_decode_step(self.h, _ptr(q), n_q, _ptr(k_new), _ptr(v_new), budget, _ptr(out),
                                        _ptr(idx if want_idx else None), _stream(stream)))
        return (out, idx) if want_idx else out


def top_k(scores: torch.Tensor, k: int, stream=None) -> torch.Tensor:
    """top_k per row (estimator.cpp:75-90): int32 [n_rows][k], -1 past min(k, n)."""
    L = load()
    s = scores.to(torch.int32).contiguous()
    if s.dim() == 1:
        s = s.unsqueeze(0)
    out = torch.empty((s.shape[0], k), dtype=torch.int32, device="cuda")
    check(L.adamas_topk(_ptr(s), s.shape[0], s.shape[1], k, _ptr(out), _stream(stream)))
    return out


def get_tuning() -> dict:
    vals = (C.c_int * len(TUNING_FIELDS))()
    check(load().adamas_get_tuning(vals, len(TUNING_FIELDS)))
    return dict(zip(TUNING_FIELDS, list(vals)))


def set_tuning(**kw) -> None:
    """Launch-plan overrides (include/adamas_b200.h adamas_set_tuning)."""
    cur = get_tuning()
    for k, v in kw.items():
        if k not in cur:
            raise ConfigError(f"unknown tuning field {k}")
        cur[k] = int(v)
    vals = (C.c_int * len(TUNING_FIELDS))(*[cur[f] for f in TUNING_FIELDS])
    check(load().adamas_set_tuning(vals, len(TUNING_FIELDS)))


@contextlib.contextmanager
def tuning(**kw):
    """Temporarily override launch-plan fields: `with tuning(cluster=4): ...`."""
    saved = get_tuning()
    set_tuning(**kw)
    try:
        yield
    finally:
        set_tuning(**saved)


def decode_step_batched(caches, q, k_new, v_new, budget, out=None, idx=None, want_idx=True, stream=None):
    """One fused launch over independent sequences (per-request caches)."""
    L = load()
    n = len(caches)
    arr = (C.c_void_p * n)(*[c.h for c in caches])
    n_q = q.shape[-2]
    if out is None:
        out = torch.empty((n, n_q, HEAD_DIM), dtype=torch.float32, device="cuda")
    if want_idx and idx is None:
        idx = torch.empty((n, n_q, budget), dtype=torch.int32, device="cuda")
    check(L.adamas_decode_step_batched(arr, n, _ptr(q), n_q, _ptr(k_new), _ptr(v_new), budget, _ptr(out),
                                       _ptr(idx if want_idx else None), _stream(stream)))
    return (out, idx) if want_idx else out


class _DeviceView:
    """Wraps a raw device address as a torch tensor via __cuda_array_interface__."""

    def __init__(self, addr, shape, dtype):
        self.addr, self.shape, self.dtype = addr, shape, dtype

    @property
    def __cuda_array_interface__(self):
        typestr = {torch.float32: "<f4", torch.bfloat16: "<u2"}[self.dtype]
        return {"shape": self.shape, "typestr": typestr, "data": (self.addr, False), "version": 3}

    def tensor(self) -> torch.Tensor:
        t = torch.as_tensor(self, device="cuda")
        return t.view(torch.bfloat16) if self.dtype == torch.bfloat16 else t
