"""ctypes bindings for the CPU checkers in oracle/ — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module, and only as the checker or the timed CPU
baseline — never as part of the product path (paper_2510_18413_b200 must not
import it).

* ``Oracle``    — liboracle.so, the C restatement (adamas_oracle.c).
* ``Reference`` — _ref/libadamas_ref.so, the unmodified reference library
                  compiled from /root/reference/proj/src plus ref_shim.cpp.
* ``synth``     — the shared integer synthetic generator (bit-identical to
                  or_synth_value in adamas_oracle.c and the CUDA generator).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBORACLE = os.path.join(HERE, "liboracle.so")
LIBREF = os.path.join(HERE, "_ref", "libadamas_ref.so")

_u64 = np.uint64


def synth(seed: int, first: int, n: int) -> np.ndarray:
    """float32 Irwin-Hall(4) values; see or_synth_value (adamas_oracle.c)."""
    with np.errstate(over="ignore"):
        idx = np.arange(first, first + n, dtype=np.uint64)
        z = _u64(seed) ^ (idx * _u64(0xD1B54A32D192ED03))
        z = z + _u64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> _u64(30))) * _u64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _u64(27))) * _u64(0x94D049BB133111EB)
        z = z ^ (z >> _u64(31))
        m = _u64(0xFFFF)
        s = (z & m) + ((z >> _u64(16)) & m) + ((z >> _u64(32)) & m) + (z >> _u64(48))
    return ((s.astype(np.int64) - 131070).astype(np.float64) / 37837.0).astype(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (nearest-even), returned as float32 values."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def build(with_ref: bool | None = None) -> None:
    """make liboracle.so (and _ref/ when /root/reference is present)."""
    targets = ["all"]
    if with_ref is None:
        with_ref = os.path.isdir("/root/reference/proj/src")
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


_D = C.c_double
_SZ = C.c_size_t


class Oracle:
    """The C restatement of the reference hot path."""

    def __init__(self, path: str = LIBORACLE):
        if not os.path.exists(path):
            build(with_ref=False)
        L = C.CDLL(path)
        self.L = L
        L.or_fwht.argtypes = [C.POINTER(_D), _SZ, C.c_int]
        L.or_compute_thresholds.argtypes = [C.POINTER(_D), _SZ, C.c_int, C.POINTER(_D)]
        L.or_bucketize.argtypes = [C.POINTER(_D), _SZ, C.POINTER(_D), C.c_int, C.POINTER(C.c_uint8)]
        L.or_pack.argtypes = [C.POINTER(C.c_uint8), _SZ, C.c_int, C.POINTER(C.c_uint16), C.POINTER(_SZ)]
        L.or_unpack.argtypes = [C.POINTER(C.c_uint16), _SZ, C.c_int, C.POINTER(C.c_uint8)]
        L.or_encode_pack.argtypes = [C.POINTER(_D), _SZ, C.POINTER(C.c_uint16)]
        L.or_l1_2bit.argtypes = [C.POINTER(C.c_uint16), C.POINTER(C.c_uint16), _SZ]
        L.or_l1_2bit.restype = C.c_uint32
        L.or_score_all.argtypes = [C.POINTER(C.c_uint16), C.POINTER(C.c_uint16), _SZ, _SZ, C.POINTER(C.c_int32)]
        L.or_top_k.argtypes = [C.POINTER(C.c_int32), _SZ, _SZ, C.POINTER(C.c_int64)]
        L.or_top_k.restype = _SZ
        L.or_full_attention.argtypes = [C.POINTER(_D)] * 3 + [_SZ, _SZ, C.POINTER(_D)]
        L.or_sparse_attention.argtypes = [C.POINTER(_D)] * 3 + [_SZ, _SZ, C.POINTER(C.c_int64), _SZ, C.POINTER(_D)]
        L.or_output_error.argtypes = [C.POINTER(_D), C.POINTER(_D), _SZ]
        L.or_output_error.restype = _D
        L.or_synth_fill.argtypes = [C.c_uint64, C.c_uint64, _SZ, C.POINTER(C.c_float)]

    # -- transform / quantizer ---------------------------------------------
    def fwht(self, x, normalized=True):
        y = np.array(x, dtype=np.float64, copy=True)
        rc = self.L.or_fwht(_p(y, _D), y.size, int(normalized))
        if rc:
            raise ValueError("ConfigError: fwht dimension")
        return y

    def compute_thresholds(self, x, bits=2):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(7, dtype=np.float64)
        if self.L.or_compute_thresholds(_p(x, _D), x.size, bits, _p(out, _D)):
            raise ValueError("ConfigError: thresholds")
        return out[: (1 << bits) - 1].copy()

    def bucketize(self, x, t, bits=2):
        x = np.ascontiguousarray(x, dtype=np.float64)
        t = np.ascontiguousarray(t, dtype=np.float64)
        out = np.zeros(x.size, dtype=np.uint8)
        self.L.or_bucketize(_p(x, _D), x.size, _p(t, _D), bits, _p(out, C.c_uint8))
        return out

    def pack(self, codes, bits=2):
        c = np.ascontiguousarray(codes, dtype=np.uint8)
        per = 16 // bits
        out = np.zeros((c.size + per - 1) // per, dtype=np.uint16)
        n = _SZ(0)
        if self.L.or_pack(_p(c, C.c_uint8), c.size, bits, _p(out, C.c_uint16), C.byref(n)):
            raise ValueError("ConfigError: pack")
        return out[: n.value]

    def unpack(self, words, bits=2):
        w = np.ascontiguousarray(words, dtype=np.uint16)
        out = np.zeros(w.size * (16 // bits), dtype=np.uint8)
        self.L.or_unpack(_p(w, C.c_uint16), w.size, bits, _p(out, C.c_uint8))
        return out

    def encode_pack(self, x):
        """pack(encode(x)) for one vector; raises on degenerate input."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros((x.size + 7) // 8, dtype=np.uint16)
        if self.L.or_encode_pack(_p(x, _D), x.size, _p(out, C.c_uint16)):
            raise ValueError("ConfigError: encode")
        return out

    def encode_pack_rows(self, X):
        X = np.ascontiguousarray(X, dtype=np.float64)
        return np.stack([self.encode_pack(r) for r in X.reshape(-1, X.shape[-1])]).reshape(
            X.shape[:-1] + ((X.shape[-1] + 7) // 8,))

    # -- estimator -----------------------------------------------------------
    def l1_2bit(self, q, k):
        q = np.ascontiguousarray(q, dtype=np.uint16)
        k = np.ascontiguousarray(k, dtype=np.uint16)
        return int(self.L.or_l1_2bit(_p(q, C.c_uint16), _p(k, C.c_uint16), q.size))

    def score_all(self, qwords, cache_words):
        q = np.ascontiguousarray(qwords, dtype=np.uint16)
        cw = np.ascontiguousarray(cache_words, dtype=np.uint16)
        S = cw.shape[0]
        out = np.zeros(S, dtype=np.int32)
        self.L.or_score_all(_p(q, C.c_uint16), _p(cw, C.c_uint16), S, q.size, _p(out, C.c_int32))
        return out

    def top_k(self, scores, k):
        s = np.ascontiguousarray(scores, dtype=np.int32)
        out = np.zeros(max(min(k, s.size), 1), dtype=np.int64)
        n = self.L.or_top_k(_p(s, C.c_int32), s.size, k, _p(out, C.c_int64))
        return out[:n].copy()

    # -- attention -----------------------------------------------------------
    def full_attention(self, q, K, V):
        q = np.ascontiguousarray(q, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        V = np.ascontiguousarray(V, dtype=np.float64)
        out = np.zeros(q.size, dtype=np.float64)
        if self.L.or_full_attention(_p(q, _D), _p(K, _D), _p(V, _D), K.shape[0], q.size, _p(out, _D)):
            raise ValueError("ConfigError: full_attention")
        return out

    def sparse_attention(self, q, K, V, idx):
        q = np.ascontiguousarray(q, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        V = np.ascontiguousarray(V, dtype=np.float64)
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros(q.size, dtype=np.float64)
        if self.L.or_sparse_attention(_p(q, _D), _p(K, _D), _p(V, _D), K.shape[0], q.size,
                                      _p(idx, C.c_int64), idx.size, _p(out, _D)):
            raise ValueError("ConfigError: sparse_attention")
        return out

    def output_error(self, a, e):
        a = np.ascontiguousarray(a, dtype=np.float64)
        e = np.ascontiguousarray(e, dtype=np.float64)
        return float(self.L.or_output_error(_p(a, _D), _p(e, _D), a.size))

    def synth(self, seed, first, n):
        out = np.zeros(n, dtype=np.float32)
        self.L.or_synth_fill(seed, first, n, _p(out, C.c_float))
        return out

    # -- composite -------------------------------------------------------------
    def decode_head(self, q, K, V, cache_words, budget):
        """One head: (scores, ascending indices, attention output)."""
        qw = self.encode_pack(q)
        scores = self.score_all(qw, cache_words)
        idx = self.top_k(scores, budget)
        out = self.sparse_attention(q, K, V, idx)
        return qw, scores, idx, out


class Reference:
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self, path: str = LIBREF):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference; run make -C oracle ref)")
        L = C.CDLL(path)
        self.L = L
        L.ref_simd_level.restype = C.c_char_p
        L.ref_fwht.argtypes = [C.POINTER(_D), _SZ, C.c_int]
        L.ref_compute_thresholds.argtypes = [C.POINTER(_D), _SZ, C.c_int, C.POINTER(_D)]
        L.ref_pack.argtypes = [C.POINTER(C.c_uint8), _SZ, C.c_int, C.POINTER(C.c_uint16), C.POINTER(_SZ)]
        L.ref_encode_pack.argtypes = [C.POINTER(_D), _SZ, C.POINTER(C.c_uint16)]
        L.ref_manhattan_packed.argtypes = [C.POINTER(C.c_uint16), C.POINTER(C.c_uint16), _SZ]
        L.ref_manhattan_packed.restype = C.c_uint32
        L.ref_cache_new.argtypes = [_SZ, C.c_int]
        L.ref_cache_new.restype = C.c_void_p
        L.ref_cache_free.argtypes = [C.c_void_p]
        L.ref_cache_update.argtypes = [C.c_void_p, C.POINTER(_D), C.POINTER(_D), C.POINTER(C.c_uint16)]
        L.ref_cache_seq_len.argtypes = [C.c_void_p]
        L.ref_cache_seq_len.restype = _SZ
        L.ref_score_all.argtypes = [C.c_void_p, C.POINTER(C.c_uint16), C.POINTER(C.c_int32)]
        L.ref_top_k.argtypes = [C.POINTER(C.c_int32), _SZ, _SZ, C.POINTER(C.c_int64)]
        L.ref_top_k.restype = _SZ
        L.ref_sparse_attention.argtypes = [C.c_void_p, C.POINTER(_D), C.POINTER(C.c_int64), _SZ, C.POINTER(_D)]
        L.ref_full_attention.argtypes = [C.POINTER(_D)] * 3 + [_SZ, _SZ, C.POINTER(_D)]
        L.ref_decode_head.argtypes = [C.c_void_p, C.POINTER(_D), _SZ, C.POINTER(C.c_int64), C.POINTER(_SZ), C.POINTER(_D)]
        L.ref_layer_build.argtypes = [_SZ, _SZ, _SZ, C.c_int, C.c_uint64, C.c_int]
        L.ref_layer_build.restype = C.c_void_p
        L.ref_layer_free.argtypes = [C.c_void_p]
        L.ref_layer_decode.argtypes = [C.c_void_p, _SZ, C.c_int, C.c_int, C.POINTER(_D)]
        L.ref_score_all_metric.argtypes = [C.c_void_p, C.POINTER(C.c_uint16), C.c_int, C.POINTER(C.c_int32)]
        L.ref_encode_pack_bits.argtypes = [C.POINTER(_D), _SZ, C.c_int, C.POINTER(C.c_uint16)]
        L.ref_save_snapshot.argtypes = [C.c_void_p, C.c_char_p]
        L.ref_load_snapshot.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.ref_load_snapshot.restype = C.c_void_p
        L.ref_cache_rows.argtypes = [C.c_void_p, _SZ, C.POINTER(_D), C.POINTER(_D)]
        L.ref_cache_code_words.argtypes = [C.c_void_p, _SZ, C.POINTER(C.c_uint16)]
        vp = C.c_void_p
        spec_t = [C.c_uint64, _SZ, _SZ, _SZ, C.c_int, _D, _D, _SZ, _D]
        L.ref_workload_instance.argtypes = spec_t + [_SZ, vp, vp, vp, C.POINTER(C.c_uint64), C.POINTER(C.c_int64)]
        L.ref_run_sweep.argtypes = spec_t + [vp, _SZ, vp, vp, vp, vp, vp, vp, _SZ, C.c_int,
                                             C.c_char_p, _SZ, C.POINTER(_SZ), C.c_char_p, _SZ, C.POINTER(_SZ),
                                             C.c_char_p, _SZ, C.POINTER(_SZ)]
        L.ref_last_error.restype = C.c_char_p
        L.ref_rows_to_csv.argtypes = [vp, vp, vp, _SZ, C.c_char_p, _SZ]
        L.ref_rows_to_csv.restype = _SZ
        L.ref_top_k_by_score.argtypes = [vp, _SZ, _SZ, vp]
        L.ref_top_k_by_score.restype = _SZ
        L.ref_page_select.argtypes = [vp, vp, _SZ, _SZ, _SZ, _SZ, vp, C.POINTER(_SZ)]
        L.ref_adamas_select.argtypes = [vp, vp, _SZ, _SZ, C.c_int, C.c_int, C.c_int, _SZ, vp, C.POINTER(_SZ), vp, vp]

    # -- sweep harness (workload.cpp, sweep.cpp, baselines.cpp) -------------------
    _KINDS = {"adamas": 0, "window": 1, "quest": 2, "oracle": 3}
    _DISTS = {"gaussian": 0, "gaussian_with_outliers": 1, "planted_needle": 2}

    @classmethod
    def _spec_args(cls, w):
        return [w.seed, w.seq_len, w.head_dim, w.num_queries, cls._DISTS[w.distribution], w.outlier_frac,
                w.outlier_scale, w.position, w.snr]

    def workload_instance(self, w, qi):
        """Workload(w).instance(qi) (workload.cpp:125-155) -> (seed, query, keys, values, needle or None)."""
        q = np.zeros(w.head_dim)
        K = np.zeros((w.seq_len, w.head_dim))
        V = np.zeros((w.seq_len, w.head_dim))
        seed = C.c_uint64(0)
        needle = C.c_int64(-1)
        rc = self.L.ref_workload_instance(*self._spec_args(w), qi, q.ctypes.data, K.ctypes.data, V.ctypes.data,
                                          C.byref(seed), C.byref(needle))
        if rc:
            raise ValueError("ConfigError: workload")
        return seed.value, q, K, V, (None if needle.value < 0 else needle.value)

    def run_sweep(self, w, sweep):
        """run_sweep (sweep.cpp:189-253) -> (rows CSV, rows JSON, needle summary CSV or None)."""
        pol = sweep.policies
        budgets = np.array(sweep.budgets, dtype=np.uint64)
        kinds = np.array([self._KINDS[p.kind] for p in pol], np.int32)
        bits = np.array([p.bits for p in pol], np.int32)
        metrics = np.array([0 if p.metric in ("l1", "manhattan") else 1 for p in pol], np.int32)
        had = np.array([int(p.with_hadamard) for p in pol], np.int32)
        sinks = np.array([p.sink for p in pol], np.uint64)
        pages = np.array([p.page_size for p in pol], np.uint64)
        cap = 1 << 16
        while True:
            bufs = [C.create_string_buffer(cap) for _ in range(3)]
            lens = [_SZ(0) for _ in range(3)]
            rc = self.L.ref_run_sweep(*self._spec_args(w), budgets.ctypes.data, budgets.size, kinds.ctypes.data,
                                      bits.ctypes.data, metrics.ctypes.data, had.ctypes.data, sinks.ctypes.data,
                                      pages.ctypes.data, len(pol), int(sweep.measure_output_error),
                                      bufs[0], cap, C.byref(lens[0]), bufs[1], cap, C.byref(lens[1]),
                                      bufs[2], cap, C.byref(lens[2]))
            if rc:
                raise (ValueError if rc == 1 else RuntimeError)(self.L.ref_last_error().decode())
            if max(x.value for x in lens) < cap:
                break
            cap = max(x.value for x in lens) + 1
        csv, js, nd = (b.value.decode() for b in bufs)
        return csv, js, (nd if lens[2].value else None)

    def rows_to_csv(self, recall, output_error=None):
        """rows_to_csv over rows carrying these recall / output_error values."""
        r = np.ascontiguousarray(recall, dtype=np.float64)
        e = np.zeros_like(r) if output_error is None else np.ascontiguousarray(output_error, dtype=np.float64)
        has = np.full(r.size, 0 if output_error is None else 1, np.int32)
        n = self.L.ref_rows_to_csv(r.ctypes.data, e.ctypes.data, has.ctypes.data, r.size, None, 0)
        buf = C.create_string_buffer(n + 1)
        self.L.ref_rows_to_csv(r.ctypes.data, e.ctypes.data, has.ctypes.data, r.size, buf, n + 1)
        return buf.value.decode()

    def top_k_by_score(self, scores, k):
        s = np.ascontiguousarray(scores, dtype=np.float64)
        out = np.zeros(min(k, s.size), np.int64)
        n = self.L.ref_top_k_by_score(s.ctypes.data, s.size, k, out.ctypes.data)
        return out[:n]

    def page_select(self, q, K, page_size, k):
        q = np.ascontiguousarray(q, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        out = np.zeros(max(k, K.shape[0]), np.int64)
        n = _SZ(0)
        rc = self.L.ref_page_select(q.ctypes.data, K.ctypes.data, K.shape[0], K.shape[1], page_size, k,
                                    out.ctypes.data, C.byref(n))
        if rc:
            raise ValueError("ConfigError: page_select: " + self.L.ref_last_error().decode())
        return out[:n.value]

    def adamas_select(self, q, K, bits, metric, with_hadamard, k, want_codes=False):
        """select's adamas branch (sweep.cpp:87-98) -> indices (and key / query codes in
        the reference formats when want_codes)."""
        q = np.ascontiguousarray(q, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        S, d = K.shape
        cb = d if bits == 3 else 2 * ((d + 16 // bits - 1) // (16 // bits))
        kc = np.zeros((S, cb), np.uint8) if want_codes else None
        qc = np.zeros(cb, np.uint8) if want_codes else None
        out = np.zeros(max(min(k, S), 1), np.int64)
        n = _SZ(0)
        rc = self.L.ref_adamas_select(q.ctypes.data, K.ctypes.data, S, d, bits, metric, int(with_hadamard), k,
                                      out.ctypes.data, C.byref(n), None if kc is None else kc.ctypes.data,
                                      None if qc is None else qc.ctypes.data)
        if rc:
            raise ValueError("ConfigError: adamas_select: " + self.L.ref_last_error().decode())
        if want_codes:
            return out[:n.value], kc, qc
        return out[:n.value]

    # -- ablation metrics (estimator.cpp:45-59, kernels.hpp:24-32) ---------------
    def encode_pack_bits(self, x, bits):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(x.size * bits // 16, dtype=np.uint16)
        if self.L.ref_encode_pack_bits(_p(x, _D), x.size, bits, _p(out, C.c_uint16)):
            raise ValueError("ConfigError: encode")
        return out

    def score_all_metric(self, K, q, bits, metric):
        """score_all(pack(encode(q, bits)), cache of K with bits-wide codes, metric)."""
        K = np.ascontiguousarray(K, dtype=np.float64)
        c = self.L.ref_cache_new(K.shape[1], bits)
        try:
            zero = np.zeros(K.shape[1])
            for i in range(K.shape[0]):
                w = self.encode_pack_bits(K[i], bits)
                if self.L.ref_cache_update(c, _p(K[i], _D), _p(zero, _D), _p(w, C.c_uint16)):
                    raise ValueError("ConfigError: update")
            qw = self.encode_pack_bits(q, bits)
            out = np.zeros(K.shape[0], np.int32)
            if self.L.ref_score_all_metric(c, _p(qw, C.c_uint16), metric, _p(out, C.c_int32)):
                raise ValueError("ConfigError: score_all")
            return out
        finally:
            self.L.ref_cache_free(c)

    # -- ADKV snapshots (kv_cache.cpp:111-165) ------------------------------------
    def cache_from_rows(self, K, V, words):
        """A reference KvCache (one head) holding rows K, V with the given code words."""
        K = np.ascontiguousarray(K, dtype=np.float64)
        V = np.ascontiguousarray(V, dtype=np.float64)
        W = np.ascontiguousarray(words, dtype=np.uint16)
        c = self.L.ref_cache_new(K.shape[1], 2)
        for i in range(K.shape[0]):
            if self.L.ref_cache_update(c, _p(K[i], _D), _p(V[i], _D), _p(W[i], C.c_uint16)):
                raise ValueError("ConfigError: update")
        return c

    def save_snapshot(self, cache, path):
        rc = self.L.ref_save_snapshot(cache, str(path).encode())
        if rc:
            raise (ValueError if rc == 1 else RuntimeError)("save_snapshot")

    def load_snapshot(self, path):
        """(K, V, words) of the reference's load_snapshot."""
        rc = C.c_int(0)
        c = self.L.ref_load_snapshot(str(path).encode(), C.byref(rc))
        if rc.value:
            raise (ValueError if rc.value == 1 else RuntimeError)("load_snapshot")
        try:
            n = self.L.ref_cache_seq_len(c)
            K = np.zeros((n, 128)); V = np.zeros((n, 128)); W = np.zeros((n, 16), np.uint16)
            for i in range(n):
                self.L.ref_cache_rows(c, i, _p(K[i], _D), _p(V[i], _D))
                self.L.ref_cache_code_words(c, i, _p(W[i], C.c_uint16))
        finally:
            self.L.ref_cache_free(c)
        return K, V, W

    def cache_free(self, cache):
        self.L.ref_cache_free(cache)

    def simd_level(self) -> str:
        return self.L.ref_simd_level().decode()

    def fwht(self, x, normalized=True):
        y = np.array(x, dtype=np.float64, copy=True)
        if self.L.ref_fwht(_p(y, _D), y.size, int(normalized)):
            raise ValueError("ConfigError")
        return y

    def compute_thresholds(self, x, bits=2):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros(7, dtype=np.float64)
        if self.L.ref_compute_thresholds(_p(x, _D), x.size, bits, _p(out, _D)):
            raise ValueError("ConfigError")
        return out[: (1 << bits) - 1].copy()

    def encode_pack(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.zeros((x.size + 7) // 8, dtype=np.uint16)
        if self.L.ref_encode_pack(_p(x, _D), x.size, _p(out, C.c_uint16)):
            raise ValueError("ConfigError")
        return out

    def manhattan_packed(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.uint16)
        b = np.ascontiguousarray(b, dtype=np.uint16)
        return int(self.L.ref_manhattan_packed(_p(a, C.c_uint16), _p(b, C.c_uint16), a.size))

    def top_k(self, scores, k):
        s = np.ascontiguousarray(scores, dtype=np.int32)
        out = np.zeros(max(min(k, s.size), 1), dtype=np.int64)
        n = self.L.ref_top_k(_p(s, C.c_int32), s.size, k, _p(out, C.c_int64))
        return out[:n].copy()

    def full_attention(self, q, K, V):
        q = np.ascontiguousarray(q, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        V = np.ascontiguousarray(V, dtype=np.float64)
        out = np.zeros(q.size, dtype=np.float64)
        if self.L.ref_full_attention(_p(q, _D), _p(K, _D), _p(V, _D), K.shape[0], q.size, _p(out, _D)):
            raise ValueError("ConfigError")
        return out

    def decode_head(self, q, K, V, budget):
        """Builds a reference KvCache over (K, V) with encode+pack per row (the
        build_cache loop, sweep.cpp:38-50) and runs the reference decode step.
        Returns (cache code words, scores, indices, output)."""
        K = np.ascontiguousarray(K, dtype=np.float64)
        V = np.ascontiguousarray(V, dtype=np.float64)
        q = np.ascontiguousarray(q, dtype=np.float64)
        S, d = K.shape
        c = self.L.ref_cache_new(d, 2)
        try:
            words = np.zeros((S, (d + 7) // 8), dtype=np.uint16)
            for i in range(S):
                words[i] = self.encode_pack(K[i])
                if self.L.ref_cache_update(c, _p(K[i], _D), _p(V[i], _D), _p(words[i], C.c_uint16)):
                    raise ValueError("ConfigError")
            qw = self.encode_pack(q)
            scores = np.zeros(S, dtype=np.int32)
            if self.L.ref_score_all(c, _p(qw, C.c_uint16), _p(scores, C.c_int32)):
                raise ValueError("ConfigError")
            idx = np.zeros(max(min(budget, S), 1), dtype=np.int64)
            n = _SZ(0)
            out = np.zeros(d, dtype=np.float64)
            if self.L.ref_decode_head(c, _p(q, _D), budget, _p(idx, C.c_int64), C.byref(n), _p(out, _D)):
                raise ValueError("ConfigError")
            return words, qw, scores, idx[: n.value].copy(), out
        finally:
            self.L.ref_cache_free(c)

    # -- CPU decode benchmark -------------------------------------------------
    def layer_build(self, n_heads, seq_len, d, bf16, seed, threads):
        return self.L.ref_layer_build(n_heads, seq_len, d, int(bf16), seed, threads)

    def layer_decode(self, layer, budget, threads, steps):
        out = np.zeros(steps, dtype=np.float64)
        if self.L.ref_layer_decode(layer, budget, threads, steps, _p(out, _D)):
            raise RuntimeError("reference decode failed")
        return out

    def layer_free(self, layer):
        self.L.ref_layer_free(layer)
