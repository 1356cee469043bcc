"""GPU backend for the sweep harness.

The reference's harness (proj/src/sweep.cpp) runs every (policy, budget,
query) cell of a sweep on one CPU thread. This module is the same harness
surface with the per-cell work on the GPU, batched over all queries of a
sweep:

  HarnessSelector      build_cache + the adamas branch of select
                       (sweep.cpp:38-50, :87-98) -> adamas_hsel_* (C ABI)
  dot_topk             top_k_by_score over dot scores: the oracle policy and
                       every row's recall reference (sweep.cpp:202-214)
  page_select          the quest baseline (baselines.cpp:34-91)
  attention_f64        full_attention / attend_subset for output_error
                       (attention.cpp:8-57, sweep.cpp:120-131)
  run_sweep            run_sweep (sweep.cpp:189-253) over caller-supplied
                       instances (the synthetic workload generator is the
                       harness's, workload.cpp; it stays out of scope)
  needle_report, rows_to_csv, rows_to_json, needle_summary_to_csv
                       the emitters (sweep.cpp:255-336), byte-identical

Selections are identical index sets to the reference's (same fp64 operations
in the same order on the device), so the recall / selected_count / needle
columns are byte-identical; output_error uses the device exp() and agrees to
~1e-15 relative. Numbers are printed the way the reference's JSON library
prints them (format_number: Grisu2 as in nlohmann::json 3.11.3, the version
this repo pins against since the reference does not vendor its copy).
"""
from __future__ import annotations

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional, Sequence

import numpy as np
import torch

from ._lib import ConfigError, check, load

METRICS = {"l1": 0, "manhattan": 0, "l2": 1, "euclidean_sq": 1}
KINDS = ("adamas", "window", "quest", "oracle")
DISTRIBUTIONS = ("gaussian", "gaussian_with_outliers", "planted_needle")


# ----------------------------------------------------------------------------- config records
@dataclass
class WorkloadSpec:
    """WorkloadSpec (workload.hpp:56-67): the description of a synthetic workload."""

    seed: int = 0
    seq_len: int = 1
    head_dim: int = 64
    num_queries: int = 1
    distribution: str = "gaussian"
    outlier_frac: float = 0.01
    outlier_scale: float = 10.0
    position: int = 0
    snr: float = 10.0

    def validate(self) -> None:  # workload.cpp:64-80
        if self.seq_len < 1:
            raise ConfigError("workload: seq_len must be at least 1")
        d = self.head_dim
        if d < 2 or d & (d - 1):
            raise ConfigError("workload: head_dim must be a power of two >= 2")
        if self.num_queries < 1:
            raise ConfigError("workload: num_queries must be at least 1")
        if self.distribution not in DISTRIBUTIONS:
            raise ConfigError("unknown distribution: " + str(self.distribution))
        if self.distribution == "gaussian_with_outliers":
            if not 0.0 <= self.outlier_frac <= 1.0:
                raise ConfigError("workload: outlier_frac must lie in [0, 1]")
            if self.outlier_scale <= 0.0:
                raise ConfigError("workload: outlier_scale must be positive")
        if self.distribution == "planted_needle":
            if self.position >= self.seq_len:
                raise ConfigError("workload: needle position out of range")
            if self.snr <= 0.0:
                raise ConfigError("workload: snr must be positive")


@dataclass
class PolicySpec:
    """PolicySpec (sweep.hpp:15-33)."""

    kind: str = "adamas"
    bits: int = 2
    metric: str = "l1"
    with_hadamard: bool = True
    sink: int = 4
    page_size: int = 16

    def label(self) -> str:  # sweep.cpp:146-161
        if self.kind == "adamas":
            name = f"adamas-{self.bits}bit-{'l1' if METRICS[self.metric] == 0 else 'l2'}"
            return name if self.with_hadamard else name + "-nohadamard"
        if self.kind == "window":
            return f"window-sink{self.sink}"
        if self.kind == "quest":
            return f"quest-p{self.page_size}"
        if self.kind == "oracle":
            return "oracle"
        return "?"

    def validate(self) -> None:  # sweep.cpp:163-168
        if self.kind not in KINDS:
            raise ConfigError("unknown policy kind: " + str(self.kind))
        if self.metric not in METRICS:
            raise ConfigError("unknown metric: " + str(self.metric))
        if self.kind == "adamas" and not 1 <= self.bits <= 3:
            raise ConfigError("policy: adamas bits must be 1, 2, or 3")
        if self.kind == "quest" and self.page_size == 0:
            raise ConfigError("policy: quest page_size must be positive")


@dataclass
class SweepConfig:
    """SweepConfig (sweep.hpp:35-44)."""

    budgets: list = field(default_factory=list)
    policies: list = field(default_factory=list)
    measure_output_error: bool = True

    def validate(self) -> None:  # sweep.cpp:170-179
        if not self.budgets:
            raise ConfigError("sweep: at least one budget required")
        for i, b in enumerate(self.budgets):
            if b == 0:
                raise ConfigError("sweep: budgets must be positive")
            if i > 0 and b <= self.budgets[i - 1]:
                raise ConfigError("sweep: budgets must be strictly ascending")
        if not self.policies:
            raise ConfigError("sweep: at least one policy required")
        for p in self.policies:
            p.validate()


@dataclass
class Instance:
    """WorkloadInstance (workload.hpp:69-80). Instances that share key/value
    tensors (Gaussian workloads) must hold the SAME array objects: like the
    reference's pointer identity check (sweep.cpp:62), sharing is by identity."""

    seed: int
    query: np.ndarray
    keys: np.ndarray
    values: np.ndarray
    needle_position: Optional[int] = None


@dataclass
class ResultRow:
    """ResultRow (sweep.hpp:46-56)."""

    policy: str
    budget: int
    seed: int
    recall: float = 0.0
    output_error: Optional[float] = None
    selected_count: int = 0
    needle_hit: Optional[bool] = None


@dataclass
class NeedleSummaryRow:
    policy: str
    budget: int
    needle_fraction: float = 0.0
    queries: int = 0


# ----------------------------------------------------------------------------- device helpers
def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(a, device) -> torch.Tensor:
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)).to(device)


_STAGING = {}  # (device, bytes) -> two pinned staging buffers, reused across sweeps
_STAGE_BYTES = 64 << 20


def _dev_stack(arrays, device) -> torch.Tensor:
    """Stack host fp64 matrices straight into one device tensor. Large sets go
    through two reused pinned 64 MB buffers: host threads fill one (numpy
    copies release the GIL) while the DMA engine drains the other."""
    shape = arrays[0].shape
    out = torch.empty((len(arrays), *shape), dtype=torch.float64, device=device)
    per = int(np.prod(shape)) * 8
    if len(arrays) * per < _STAGE_BYTES or per > _STAGE_BYTES:
        for i, a in enumerate(arrays):
            out[i].copy_(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)))
        return out
    from concurrent.futures import ThreadPoolExecutor
    chunk = _STAGE_BYTES // per
    key = (str(device), chunk, tuple(shape))
    if key not in _STAGING:
        _STAGING[key] = [torch.empty((chunk, *shape), dtype=torch.float64).pin_memory() for _ in range(2)]
    bufs = _STAGING[key]
    done = [None, None]
    stream = torch.cuda.current_stream(device)
    with ThreadPoolExecutor(max_workers=8) as pool:
        for k, c0 in enumerate(range(0, len(arrays), chunk)):
            c1 = min(len(arrays), c0 + chunk)
            b = bufs[k & 1]
            if done[k & 1] is not None:
                done[k & 1].synchronize()  # the DMA out of this buffer has finished
            hb = b.numpy()
            list(pool.map(lambda i: np.copyto(hb[i - c0], arrays[i], casting="same_kind"), range(c0, c1)))
            out[c0:c1].copy_(b[:c1 - c0], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            done[k & 1] = ev
    return out


class HarnessSelector:
    """One adamas policy's code store: build_cache over n_inst key matrices,
    then select for any number of queries (sweep.cpp:38-50, :87-98)."""

    def __init__(self, head_dim: int, bits: int = 2, with_hadamard: bool = True):
        self.h = None
        self.L = load()
        self.head_dim, self.bits, self.with_hadamard = head_dim, bits, with_hadamard
        h = C.c_void_p()
        check(self.L.adamas_hsel_create(C.byref(h), head_dim, bits, int(with_hadamard)))
        self.h = h
        self.n_inst = self.seq_len = 0

    def close(self):
        if self.h:
            self.L.adamas_hsel_destroy(self.h)
            self.h = None

    __del__ = close

    def build(self, keys: torch.Tensor) -> None:
        """keys: device fp64 [n_inst][seq_len][head_dim] (or [seq_len][head_dim])."""
        if keys.dim() == 2:
            keys = keys.unsqueeze(0)
        keys = keys.contiguous()
        self.n_inst, self.seq_len = keys.shape[0], keys.shape[1]
        check(self.L.adamas_hsel_build(self.h, _ptr(keys), self.n_inst, self.seq_len, _stream()))

    def codes_ref(self, first: int = 0, n: Optional[int] = None) -> torch.Tensor:
        """Built codes in the reference's formats (uint16 words / uint8 bytes)."""
        n = self.n_inst * self.seq_len - first if n is None else n
        d = self.head_dim
        if self.bits == 3:
            out = torch.empty((n, d), dtype=torch.uint8, device="cuda")
        else:
            per = 16 // self.bits
            out = torch.empty((n, (d + per - 1) // per), dtype=torch.int16, device="cuda")
        check(self.L.adamas_hsel_codes_ref(self.h, first, n, _ptr(out), _stream()))
        return out

    def select(self, queries: torch.Tensor, budget: int, metric: str = "l1", rows_per_inst: int = 1) -> torch.Tensor:
        """int64 [n_rows][budget] ascending indices (-1 past min(budget, seq_len))."""
        queries = queries.contiguous()
        n_rows = queries.shape[0]
        idx = torch.empty((n_rows, budget), dtype=torch.int64, device=queries.device)
        check(self.L.adamas_hsel_select(self.h, _ptr(queries), n_rows, rows_per_inst, METRICS[metric], budget,
                                        _ptr(idx), _stream()))
        return idx


def dot_topk(queries, keys, k: int, rows_per_inst: int = 1, want_scores: bool = False):
    """top_k_by_score(dot(q, k_i), k) per row (baselines.cpp:21-32)."""
    L = load()
    n_rows, d = queries.shape
    n_inst, S = keys.shape[0], keys.shape[1]
    idx = torch.empty((n_rows, k), dtype=torch.int64, device=queries.device)
    sc = torch.empty((n_rows, S), dtype=torch.float64, device=queries.device) if want_scores else None
    check(L.adamas_dot_topk(_ptr(queries), _ptr(keys), n_rows, rows_per_inst, n_inst, S, d, k, _ptr(idx), _ptr(sc),
                            _stream()))
    return (idx, sc) if want_scores else idx


def topk_scores(scores, k: int):
    """top_k_by_score over precomputed fp64 scores [n_rows][n]."""
    L = load()
    idx = torch.empty((scores.shape[0], k), dtype=torch.int64, device=scores.device)
    check(L.adamas_topk_f64(_ptr(scores), scores.shape[0], scores.shape[1], k, _ptr(idx), _stream()))
    return idx


class PageSelector:
    """The quest baseline's state: PageSummaries of n_inst key matrices
    (baselines.cpp:34-54), built once, then page_select per budget (:71-91)."""

    def __init__(self, page_size: int, head_dim: int):
        self.h = None
        self.L = load()
        h = C.c_void_p()
        check(self.L.adamas_pages_create(C.byref(h), page_size, head_dim))
        self.h = h

    def close(self):
        if self.h:
            self.L.adamas_pages_destroy(self.h)
            self.h = None

    __del__ = close

    def build(self, keys: torch.Tensor) -> None:
        keys = keys.contiguous()
        check(self.L.adamas_pages_build(self.h, _ptr(keys), keys.shape[0], keys.shape[1], _stream()))

    def select(self, queries: torch.Tensor, budget: int, rows_per_inst: int = 1):
        """(idx [n_rows][budget], counts [n_rows])."""
        queries = queries.contiguous()
        n = queries.shape[0]
        idx = torch.empty((n, budget), dtype=torch.int64, device=queries.device)
        counts = torch.zeros(n, dtype=torch.int64, device=queries.device)
        check(self.L.adamas_pages_select(self.h, _ptr(queries), n, rows_per_inst, budget, _ptr(idx), _ptr(counts),
                                         _stream()))
        return idx, counts


def page_select(queries, keys, page_size: int, budget: int, rows_per_inst: int = 1):
    """Quest page selection (baselines.cpp:71-91) -> (idx [n_rows][budget], counts [n_rows])."""
    L = load()
    n_rows, d = queries.shape
    n_inst, S = keys.shape[0], keys.shape[1]
    idx = torch.empty((n_rows, budget), dtype=torch.int64, device=queries.device)
    counts = torch.zeros(n_rows, dtype=torch.int64, device=queries.device)
    check(L.adamas_page_select(_ptr(queries), _ptr(keys), n_rows, rows_per_inst, n_inst, S, d, page_size, budget,
                               _ptr(idx), _ptr(counts), _stream()))
    return idx, counts


def attention_f64(queries, keys, values, rows_per_inst: int = 1, idx=None, counts=None):
    """full_attention over all rows (idx None) or the selected rows (attention.cpp:8-38)."""
    L = load()
    n_rows, d = queries.shape
    n_inst, S = keys.shape[0], keys.shape[1]
    out = torch.empty((n_rows, d), dtype=torch.float64, device=queries.device)
    stride = 0 if idx is None else idx.shape[1]
    check(L.adamas_attention_f64(_ptr(queries), _ptr(keys), _ptr(values), n_rows, rows_per_inst, n_inst, S, d,
                                 _ptr(idx), stride, _ptr(counts), _ptr(out), _stream()))
    return out


# ----------------------------------------------------------------------------- host arithmetic
def output_error(approx: np.ndarray, exact: np.ndarray) -> float:
    """attention.cpp:47-57, sums in index order (np.cumsum accumulates left to right)."""
    d = approx - exact
    diff = float(np.cumsum(d * d)[-1])
    ref = math.sqrt(float(np.cumsum(exact * exact)[-1]))
    return math.sqrt(diff) / max(ref, 1e-30)


def recall_against(selected: np.ndarray, oracle: np.ndarray) -> float:
    """sweep.cpp:113-118 (both sorted ascending, distinct)."""
    if oracle.size == 0:
        return 1.0
    common = np.intersect1d(selected, oracle, assume_unique=True).size
    return float(common) / float(oracle.size)


# ----------------------------------------------------------------------------- run_sweep
def _group_rows(instances: Sequence[Instance]):
    """(unique key tensors in first-use order, instance index of every row)."""
    uniq, of = [], []
    seen = {}
    for inst in instances:
        key = id(inst.keys)
        if key not in seen:
            seen[key] = len(uniq)
            uniq.append(inst)
        of.append(seen[key])
    return uniq, of


def run_sweep(instances: Sequence[Instance], sweep: SweepConfig, device: str = "cuda") -> list:
    """run_sweep (sweep.cpp:189-253) over the given per-query instances, every
    selection on the GPU. Row order: policies in config order, budgets in
    config order, queries ascending."""
    sweep.validate()
    if not instances:
        raise ConfigError("run_sweep: no instances")
    uniq, of = _group_rows(instances)
    n_q, n_inst = len(instances), len(uniq)
    S, d = uniq[0].keys.shape
    for u in uniq:
        if u.keys.shape != (S, d) or u.values.shape != (S, d):
            raise ConfigError("run_sweep: every instance must share seq_len and head_dim")
    # rows of one instance must be contiguous and equally many (Gaussian: one
    # instance for all; needle: one per query); otherwise sweep per instance
    rpi = n_q // n_inst
    if n_q % n_inst or any(of[r] != r // rpi for r in range(n_q)):
        return _run_sweep_grouped(instances, sweep, device)
    K = _dev_stack([u.keys for u in uniq], device)
    V = _dev_stack([u.values for u in uniq], device) if sweep.measure_output_error else None
    Q = _dev(np.stack([i.query for i in instances]), device)
    budgets = list(sweep.budgets)
    _, dots = dot_topk(Q, K, 0, rpi, want_scores=True)  # dot scores once, top-k per budget
    oracle = {b: topk_scores(dots, b).cpu().numpy() for b in budgets}
    del dots
    exact = attention_f64(Q, K, V, rpi).cpu().numpy() if sweep.measure_output_error else None
    rows = []
    for pol in sweep.policies:
        label = pol.label()
        sel_state = None
        if pol.kind == "adamas":  # prepare_state (sweep.cpp:60-78): errors are not cell-qualified
            sel_state = HarnessSelector(d, pol.bits, pol.with_hadamard)
            sel_state.build(K)
        elif pol.kind == "quest":
            sel_state = PageSelector(pol.page_size, d)
            sel_state.build(K)
        try:
            for b in budgets:
                try:
                    idx, counts = _select(pol, sel_state, Q, K, b, rpi, S, oracle)
                except ConfigError as e:
                    raise ConfigError(f"policy={label} budget={b}: {e}") from None
                if counts is None:  # every row holds min(b, S) indices, -1 padded to b
                    counts = torch.full((Q.shape[0],), min(b, S), dtype=torch.int64, device=Q.device)
                approx = None
                if exact is not None:
                    approx = attention_f64(Q, K, V, rpi, idx, counts).cpu().numpy()
                idx_h = idx.cpu().numpy()
                cnt_h = counts.cpu().numpy()
                common = _common_counts(idx_h, oracle[b])
                n_orc = min(b, S)
                for qi, inst in enumerate(instances):
                    n = int(cnt_h[qi])
                    row = ResultRow(policy=label, budget=b, seed=inst.seed)
                    # recall_against (sweep.cpp:113-118); n_orc > 0 always (b, S >= 1)
                    row.recall = float(common[qi]) / float(n_orc)
                    row.selected_count = n
                    if approx is not None:
                        row.output_error = output_error(approx[qi], exact[qi])
                    if inst.needle_position is not None:
                        row.needle_hit = bool((idx_h[qi, :n] == inst.needle_position).any())
                    rows.append(row)
        finally:
            if sel_state is not None:
                sel_state.close()
    return rows


def _common_counts(sel: np.ndarray, orc: np.ndarray) -> np.ndarray:
    """|sel_r ∩ orc_r| per row; rows hold distinct indices, -1 padded."""
    m = np.concatenate([sel, orc], axis=1)
    m.sort(axis=1)
    return ((m[:, 1:] == m[:, :-1]) & (m[:, 1:] >= 0)).sum(axis=1)


def _select(pol, selector, Q, K, b, rpi, S, oracle):
    """(idx [n_rows][w] on the device, counts or None when every row holds min(b, S))."""
    if pol.kind == "adamas":
        return selector.select(Q, b, pol.metric, rpi), None
    if pol.kind == "oracle":
        return torch.as_tensor(oracle[b], device=Q.device), None
    if pol.kind == "quest":
        return selector.select(Q, b, rpi)
    # window (baselines.cpp:8-19; sweep.cpp:100-104): index arithmetic only
    sink = min(pol.sink, b)
    recent = b - sink
    if sink + recent >= S:
        row = np.arange(S, dtype=np.int64)
    else:
        row = np.concatenate([np.arange(sink), np.arange(S - recent, S)]).astype(np.int64)
    idx = torch.as_tensor(np.tile(row, (Q.shape[0], 1)), device=Q.device)
    counts = torch.full((Q.shape[0],), row.size, dtype=torch.int64, device=Q.device)
    return idx, counts


def _run_sweep_grouped(instances, sweep, device):
    """Instances whose sharing pattern is not one-per-group: one sweep per
    instance group, rows re-interleaved into the reference's order."""
    uniq, of = _group_rows(instances)
    per_group = []
    for g in range(len(uniq)):
        members = [i for i, x in enumerate(of) if x == g]
        per_group.append((members, run_sweep([instances[i] for i in members], sweep, device)))
    n_q = len(instances)
    n_cells = len(sweep.policies) * len(sweep.budgets)
    out = [None] * (n_cells * n_q)
    for members, rows in per_group:
        m = len(members)
        for c in range(n_cells):
            for j, qi in enumerate(members):
                out[c * n_q + qi] = rows[c * m + j]
    return out


# ----------------------------------------------------------------------------- reports / emitters
def needle_report(rows: Sequence[ResultRow]) -> list:
    """sweep.cpp:255-272."""
    if not rows:
        raise ConfigError("needle_report: no rows")
    summary, index = [], {}
    for row in rows:
        if row.needle_hit is None:
            raise ConfigError("needle_report: rows are not from a planted-needle workload")
        key = (row.policy, row.budget)
        if key not in index:
            index[key] = len(summary)
            summary.append(NeedleSummaryRow(policy=row.policy, budget=row.budget))
        cell = summary[index[key]]
        cell.needle_fraction += 1.0 if row.needle_hit else 0.0
        cell.queries += 1
    for cell in summary:
        cell.needle_fraction /= float(cell.queries)
    return summary


def csv_escape(field_: str) -> str:
    """sweep.cpp:139-148 (RFC 4180 quoting)."""
    if not any(c in field_ for c in ',"\n'):
        return field_
    return '"' + field_.replace('"', '""') + '"'


def rows_to_csv(rows: Sequence[ResultRow]) -> str:
    """sweep.cpp:280-297."""
    out = ["policy,budget,seed,recall,output_error,selected_count\n"]
    for r in rows:
        err = format_number(r.output_error) if r.output_error is not None else ""
        out.append(f"{csv_escape(r.policy)},{r.budget},{r.seed},{format_number(r.recall)},{err},{r.selected_count}\n")
    return "".join(out)


def rows_to_json(rows: Sequence[ResultRow]) -> str:
    """sweep.cpp:299-313: nlohmann ordered_json dump(2) of the row objects."""
    if not rows:
        return "[]\n"
    items = []
    for r in rows:
        err = format_number(r.output_error) if r.output_error is not None else "null"
        items.append("  {\n"
                     f"    \"policy\": {json.dumps(r.policy)},\n"
                     f"    \"budget\": {r.budget},\n"
                     f"    \"seed\": {r.seed},\n"
                     f"    \"recall\": {format_number(r.recall)},\n"
                     f"    \"output_error\": {err},\n"
                     f"    \"selected_count\": {r.selected_count}\n"
                     "  }")
    return "[\n" + ",\n".join(items) + "\n]\n"


def needle_summary_to_csv(rows: Sequence[NeedleSummaryRow]) -> str:
    """sweep.cpp:320-334."""
    out = ["policy,budget,needle_fraction,queries\n"]
    for r in rows:
        out.append(f"{csv_escape(r.policy)},{r.budget},{format_number(r.needle_fraction)},{r.queries}\n")
    return "".join(out)


# ----------------------------------------------------------------------------- format_number
# nlohmann::json's double -> text (json.hpp 3.11.3, dtoa_impl): Grisu2 with
# 64-bit "DiyFp" arithmetic and a table of cached powers of ten, then %g-like
# formatting with fixed notation for exponents in [-4, 15). Grisu2 always
# round-trips but is not always the shortest representation, so Python's repr
# differs in ~1% of cases; this is a restatement of the published algorithm
# (Loitsch, PLDI 2010) in nlohmann's variant.
_MASK64 = (1 << 64) - 1
_ALPHA, _GAMMA = -60, -32


def _cached_power(k: int):
    """(f, e) with f * 2^e ~= 10^k, f a normalized 64-bit significand rounded to nearest."""
    v = Fraction(10) ** k
    e = v.numerator.bit_length() - v.denominator.bit_length() - 63
    while Fraction(2) ** (e + 63) > v:
        e -= 1
    while Fraction(2) ** (e + 64) <= v:
        e += 1
    scaled = v / (Fraction(2) ** e)
    f = scaled.numerator // scaled.denominator
    rem = scaled - f
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and f & 1):
        f += 1
    if f >> 64:
        f >>= 1
        e += 1
    return f, e


_CACHED = [(*_cached_power(k), k) for k in range(-300, 325, 8)]


def _diy_mul(xf, xe, yf, ye):
    return ((xf * yf + (1 << 63)) >> 64) & _MASK64, xe + ye + 64


def _normalize(f, e):
    s = 64 - f.bit_length()
    return (f << s) & _MASK64, e - s


def _boundaries(value: float):
    bits = int.from_bytes(np.float64(value).tobytes(), "little")
    E, F = bits >> 52, bits & ((1 << 52) - 1)
    if E == 0:
        vf, ve = F, 1 - 1075
    else:
        vf, ve = F + (1 << 52), E - 1075
    closer = F == 0 and E > 1
    pf, pe = 2 * vf + 1, ve - 1
    if closer:
        mf, me = 4 * vf - 1, ve - 2
    else:
        mf, me = 2 * vf - 1, ve - 1
    wpf, wpe = _normalize(pf, pe)
    wmf, wme = (mf << (me - wpe)) & _MASK64, wpe
    wf, we = _normalize(vf, ve)
    return (wmf, wme), (wf, we), (wpf, wpe)


def _grisu2(value: float):
    (mmf, mme), (vf, ve), (mpf, mpe) = _boundaries(value)
    f = _ALPHA - mpe - 1
    k = int(f * 78913 / (1 << 18)) + (1 if f > 0 else 0)  # C++ truncating division
    index = (300 + k + 7) // 8
    cf, ce, ck = _CACHED[index]
    wf, we = _diy_mul(vf, ve, cf, ce)
    lf, le = _diy_mul(mmf, mme, cf, ce)
    hf, he = _diy_mul(mpf, mpe, cf, ce)
    m_minus, m_plus = lf + 1, hf - 1
    dec_exp = -ck
    delta = m_plus - m_minus
    dist = m_plus - wf
    one_e = he
    one_f = 1 << -one_e
    p1 = m_plus >> -one_e
    p2 = m_plus & (one_f - 1)
    buf = []
    n = len(str(p1))
    pow10 = 10 ** (n - 1)

    def rnd(rest, ten_k):
        while rest < dist and delta - rest >= ten_k and (rest + ten_k < dist or dist - rest > rest + ten_k - dist):
            buf[-1] = chr(ord(buf[-1]) - 1)
            rest += ten_k

    while n > 0:
        d, p1 = divmod(p1, pow10)
        buf.append(chr(48 + d))
        n -= 1
        rest = (p1 << -one_e) + p2
        if rest <= delta:
            dec_exp += n
            rnd(rest, pow10 << -one_e)
            return "".join(buf), dec_exp
        pow10 //= 10
    m = 0
    while True:
        p2 *= 10
        d, p2 = p2 >> -one_e, p2 & (one_f - 1)
        buf.append(chr(48 + d))
        m += 1
        delta *= 10
        dist *= 10
        if p2 <= delta:
            break
    dec_exp -= m
    rnd(p2, one_f)
    return "".join(buf), dec_exp


def format_number(v: float) -> str:
    """nlohmann::json(v).dump() for a double (sweep.cpp:133-137)."""
    v = float(v)
    if not math.isfinite(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    v = abs(v)
    if v == 0.0:
        return sign + "0.0"
    digits, dec_exp = _grisu2(v)
    k = len(digits)
    n = k + dec_exp
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    mant = digits if k == 1 else digits[0] + "." + digits[1:]
    e = n - 1
    return sign + mant + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"
