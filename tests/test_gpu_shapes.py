"""-m gpu: parity at the BASELINE.json shapes bench.py times, with the
launcher's AUTOMATIC plan (no tuning overrides), so the kernel instances the
bench measures are the ones checked:

  config 1  LongChat 32 x 128, S = 32768, bf16, budgets 64 / 128 / 256
            (fused_decode_kernel<bf16, 1, 2, false, 4>, 32 clusters of 4), and
            several layers' caches decoded back to back in ONE CUDA graph with
            PDL between the launches, as in the bench
  config 2  Llama-3.1-8B GQA 32 q / 8 kv, S = 131072, bf16, budget 128
            (automatic q-split)
  config 3  16 requests x 32K, Llama shape, one batched launch
  config 4  1M tokens, 8 kv / 32 q, 8-way sequence split simulated on one GPU
            through the peer-memory protocol (simulate_step_p2p)

Every q-head's indices are compared bit-exact with the CPU oracle
(estimator.cpp:45-90 semantics) and its output within 1e-2 relative (bf16 K/V,
attention.cpp:8-45). Inputs are drawn on the GPU (torch) and copied to the
host per kv-head for the oracle."""
import numpy as np
import pytest
import torch

from tests.gpu_helpers import rel_err

pytestmark = pytest.mark.gpu
TOL_BF16 = 1e-2


def _randn(gen, *shape):
    return torch.randn(shape, generator=gen, device="cuda").to(torch.bfloat16)


def _fill(gpu, K, V, cap):
    """cache holding K, V [S][n_kv][128] (bulk append in 8192-token pieces)."""
    c = gpu.KvCache(K.shape[1], cap, torch.bfloat16)
    for s0 in range(0, K.shape[0], 8192):
        c.update(K[s0:s0 + 8192].contiguous(), V[s0:s0 + 8192].contiguous())
    return c


def _oracle(oracle, heads_kv, q, budget, G):
    """Per q-head reference decode; heads_kv(hk) -> (K_h, V_h) float64 [S][128]
    (host copies of exactly what the device holds)."""
    n_q = q.shape[0]
    idx, out = [None] * n_q, [None] * n_q
    for hk in range(n_q // G):
        Kh, Vh = heads_kv(hk)
        words = oracle.encode_pack_rows(Kh)
        for g in range(G):
            h = hk * G + g
            _, _, i, o = oracle.decode_head(q[h].astype(np.float64), Kh, Vh, words, budget)
            idx[h], out[h] = i, o
    return np.stack(idx), np.stack(out)


def _check(got_idx, got_out, eidx, eout, budget, S):
    keep = min(budget, S)
    bad = np.nonzero((got_idx[:, :keep] != eidx).any(axis=1))[0]
    assert bad.size == 0, f"indices differ in q-heads {bad[:8].tolist()} (of {got_idx.shape[0]})"
    assert (got_idx[:, keep:] == -1).all()
    err = rel_err(got_out, eout).max()
    assert err <= TOL_BF16, err


def _host_head(K, hk, S):
    return K[:S, hk].double().cpu().numpy()


@pytest.fixture(scope="module")
def longchat(gpu):
    """Config 1: four layers' caches of S - 1 = 32767 tokens (32 kv-heads)."""
    S, n, layers = 32768, 32, 4
    gen = torch.Generator(device="cuda").manual_seed(11)
    Ks = [_randn(gen, S, n, 128) for _ in range(layers)]
    Vs = [_randn(gen, S, n, 128) for _ in range(layers)]
    caches = [_fill(gpu, K[:S - 1], V[:S - 1], S + 1) for K, V in zip(Ks, Vs)]
    return S, n, Ks, Vs, caches, gen


@pytest.mark.parametrize("budget", [64, 128, 256])
def test_config1_longchat_auto_plan(gpu, oracle, longchat, budget):
    S, n, Ks, Vs, caches, gen = longchat
    assert gpu.get_tuning()["cluster"] == 0 and gpu.get_tuning()["qsplit"] == 0  # the automatic plan
    c, K, V = caches[0], Ks[0], Vs[0]
    q = _randn(gen, n, 128)
    out, idx = c.decode_step(q, K[S - 1].contiguous(), V[S - 1].contiguous(), budget)
    torch.cuda.synchronize()
    c.raise_on_status()
    eidx, eout = _oracle(oracle, lambda hk: (_host_head(K, hk, S), _host_head(V, hk, S)),
                         q.float().cpu().numpy(), budget, 1)
    _check(idx.cpu().numpy(), out.cpu().numpy(), eidx, eout, budget, S)
    c.truncate(S - 1)


def test_config1_layers_in_one_graph(gpu, oracle, longchat):
    """Four distinct caches decoded back to back inside one CUDA graph (PDL
    between the launches, the bench's timed structure), replayed twice."""
    S, n, Ks, Vs, caches, gen = longchat
    budget, L = 128, len(caches)
    qs = _randn(gen, L, n, 128)
    out = torch.empty((L, n, 128), dtype=torch.float32, device="cuda")
    idx = torch.empty((L, n, budget), dtype=torch.int32, device="cuda")
    kn = [K[S - 1].contiguous() for K in Ks]
    vn = [V[S - 1].contiguous() for V in Vs]

    def step(st):
        for l, c in enumerate(caches):
            c.decode_step(qs[l], kn[l], vn[l], budget, out=out[l], idx=idx[l], stream=st)
        for c in caches:
            c.truncate(S - 1)

    step(torch.cuda.current_stream())  # eager first (configures the kernels)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(torch.cuda.current_stream())
    out.zero_()
    idx.fill_(-7)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for l in range(L):
        caches[l].raise_on_status()
        eidx, eout = _oracle(oracle, lambda hk: (_host_head(Ks[l], hk, S), _host_head(Vs[l], hk, S)),
                             qs[l].float().cpu().numpy(), budget, 1)
        _check(idx[l].cpu().numpy(), out[l].cpu().numpy(), eidx, eout, budget, S)


def test_config2_llama_gqa_128k(gpu, oracle):
    S, n_kv, n_q, budget = 131072, 8, 32, 128
    gen = torch.Generator(device="cuda").manual_seed(22)
    K, V = _randn(gen, S, n_kv, 128), _randn(gen, S, n_kv, 128)
    c = _fill(gpu, K[:S - 1], V[:S - 1], S + 1)
    for step in range(2):  # two steps: the second re-appends at S - 1 after a truncate
        q = _randn(gen, n_q, 128)
        out, idx = c.decode_step(q, K[S - 1].contiguous(), V[S - 1].contiguous(), budget)
        torch.cuda.synchronize()
        c.raise_on_status()
        eidx, eout = _oracle(oracle, lambda hk: (_host_head(K, hk, S), _host_head(V, hk, S)),
                             q.float().cpu().numpy(), budget, n_q // n_kv)
        _check(idx.cpu().numpy(), out.cpu().numpy(), eidx, eout, budget, S)
        c.truncate(S - 1)


def test_config3_batched_16_requests(gpu, oracle):
    R, S, n_kv, n_q, budget = 16, 32768, 8, 32, 128
    gen = torch.Generator(device="cuda").manual_seed(33)
    Ks = [_randn(gen, S, n_kv, 128) for _ in range(R)]
    Vs = [_randn(gen, S, n_kv, 128) for _ in range(R)]
    caches = [_fill(gpu, K[:S - 1], V[:S - 1], S + 1) for K, V in zip(Ks, Vs)]
    q = _randn(gen, R, n_q, 128)
    kn = torch.stack([K[S - 1] for K in Ks]).contiguous()
    vn = torch.stack([V[S - 1] for V in Vs]).contiguous()
    out, idx = gpu.decode_step_batched(caches, q, kn, vn, budget)
    torch.cuda.synchronize()
    for r in range(R):
        caches[r].raise_on_status()
        eidx, eout = _oracle(oracle, lambda hk: (_host_head(Ks[r], hk, S), _host_head(Vs[r], hk, S)),
                             q[r].float().cpu().numpy(), budget, n_q // n_kv)
        _check(idx[r].cpu().numpy(), out[r].cpu().numpy(), eidx, eout, budget, S)


def test_config4_1m_sequence_split_8way(gpu, oracle):
    """8 shards of 131072 tokens (the bench's per-rank share), tail shard
    appends; peer-memory protocol with the fused merge; global indices from
    every rank bit-exact against the single-device oracle over all 1M tokens."""
    from paper_2510_18413_b200.seqshard import Mailbox, SeqShardedDecoder, simulate_step_p2p
    W, per, n_kv, n_q, budget = 8, 131072, 8, 32, 128
    S = W * per  # after the tail shard's append
    gen = torch.Generator(device="cuda").manual_seed(44)
    Ks = [_randn(gen, per, n_kv, 128) for _ in range(W)]
    Vs = [_randn(gen, per, n_kv, 128) for _ in range(W)]
    lengths = [per] * (W - 1) + [per - 1]
    decs = []
    for r in range(W):
        c = _fill(gpu, Ks[r][:lengths[r]], Vs[r][:lengths[r]], per + 4)
        decs.append(SeqShardedDecoder(c, r, W, lengths))
    boxes = [Mailbox(r, W, n_q, budget) for r in range(W)]
    Mailbox.connect_local(boxes)
    q = _randn(gen, n_q, 128)
    outs, gidx = simulate_step_p2p(decs, boxes, [q] * W, Ks[-1][per - 1].contiguous(), Vs[-1][per - 1].contiguous(),
                                   want_idx=True)
    torch.cuda.synchronize()

    def heads_kv(hk):
        return (torch.cat([K[:, hk] for K in Ks]).double().cpu().numpy(),
                torch.cat([V[:, hk] for V in Vs]).double().cpu().numpy())

    eidx, eout = _oracle(oracle, heads_kv, q.float().cpu().numpy(), budget, n_q // n_kv)
    for r in range(W):
        _check(gidx[r].cpu().numpy(), outs[r].cpu().numpy(), eidx, eout, budget, S)
