"""CPU multi-process checks (gloo, world sizes 2 and 4) of the shard layer
(dist.py), plus direct checks of the sequence-shard top-k protocol's host model.

Sequence sharding must select exactly the single-device global top-k of the
same fp32 scores (the ranks' shares, mapped to global indices, union to
oracle.topk_select's set -- ties to the smaller global index, sink / window on
global positions) and produce the single-device output; KV-head sharding needs
no collective and its per-rank outputs concatenate to the full output.  Local
compute is the oracle-backed provider tests/oracle_ops.py (protocol:
tests/shard_model.py); the CUDA kernels are compared with the same model in
tests/test_gpu_shard.py.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import shard_model as SM


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bits_t(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)


# cases: (world, Ns, lens_full, k, sink, window, tie_period)
SEQ_CASES = {
    "w2_ragged": (2, 256, [512, 412], 60, 0, 0, 0),
    "w4_ties_sink_window": (4, 128, [512, 300], 90, 3, 5, 37),
}


def _case(name):
    import datagen
    world, Ns, lens_full, k, sink, window, period = SEQ_CASES[name]
    B, H_q, H_kv, L, P = 2, 8, 2, 16, 8
    N = Ns * world
    lens_full = np.array(lens_full, dtype=np.int32)
    c = datagen.make_case(B, H_q, H_kv, N, 128, seed=5, seq_lens=lens_full)
    if period:      # repeated K/V rows -> equal scores across the shards (heavy exact ties)
        for j in range(period, N):
            c["K"][:, :, j] = c["K"][:, :, j % period]
            c["V"][:, :, j] = c["V"][:, :, j % period]
    W = datagen.make_projections(77, L, P, 128)
    return world, Ns, lens_full, k, sink, window, B, H_q, H_kv, L, P, c, W


def _seq_worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_ops
        from paper_2602_06283_b200.dist import SeqShardDecoder, seq_shard_config
        from paper_2602_06283_b200.ops import Config
        world, Ns, lens_full, k, sink, window, B, H_q, H_kv, L, P, c, W = _case(name)
        cfg = seq_shard_config(Config(B=B, H_q=H_q, H_kv=H_kv, N_max=Ns * world, L=L, P=P, tau=0.5),
                               world, rank)
        sl = slice(rank * Ns, (rank + 1) * Ns)
        K = _bits_t(c["K"][:, :, sl].copy())
        V = _bits_t(c["V"][:, :, sl].copy())
        dec = SeqShardDecoder(cfg, _bits_t(W), K, V, k, ops=oracle_ops, sink=sink, window=window)
        dec.prefill()
        out, lse = dec.step(_bits_t(c["q"]), torch.from_numpy(lens_full))
        share = {(b, r): (dec.idx[b, r, :dec.cnt[b, r]].numpy() + rank * Ns).tolist()
                 for b in range(B) for r in range(H_kv)}
        q.put((rank, out.numpy(), lse.numpy(), share))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("name", sorted(SEQ_CASES))
def test_sequence_shard_exact_topk_and_combine(name):
    world, Ns, lens_full, k, sink, window, B, H_q, H_kv, L, P, c, W = _case(name)
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_worker, args=(r, world, port, name, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = [qu.get(timeout=840) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    ref = O.decode_step(c["q"], c["K"], c["V"], W, lens_full, tau=0.5, k=k, sm_scale=1 / np.sqrt(128))
    q, Kf, Vf = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    for b in range(B):
        for r in range(H_kv):
            s32 = ref["scores"][(b, r)].astype(np.float32).astype(np.float64)   # the product's fp32 scores
            S_ref = O.topk_select(s32, k, int(lens_full[b]), sink, window)
            union = sorted(sum((res[x][3][(b, r)] for x in range(world)), []))
            assert union == S_ref.tolist()
            for rank in range(world):
                out, lse = res[rank][1], res[rank][2]
                for h in range(r * (H_q // H_kv), (r + 1) * (H_q // H_kv)):
                    y, l = O.sparse_attention(q[b, h], Kf[b, r], Vf[b, r], S_ref, 1 / np.sqrt(128))
                    # partial states travel in the product's fp32 exchange buffers
                    assert np.max(np.abs(out[b, h] - y)) < 1e-6
                    assert abs(lse[b, h] - l) < 1e-6


# ---------------------------------------------------------------------------
# the protocol's host model directly: G shards, brute-force reference
# ---------------------------------------------------------------------------
def _protocol(shard_keys, k, Q=64, shards=None):
    G = len(shard_keys)
    digs = [SM.digest(kk, k, shards or G, Q) for kk in shard_keys]
    st = [SM.bracket(digs, k) for _ in range(G)]
    rounds = 0
    while not all(s["resolved"] for s in st):
        msgs = [SM.window(shard_keys[s], st[s]) for s in range(G)]
        st = [SM.resolve(msgs, s, st[s]) for s in range(G)]
        rounds += 1
        assert rounds <= 3
    out = []
    for s in range(G):
        out += [j + s * len(shard_keys[0]) for j in SM.emit(shard_keys[s], st[s])]
    return sorted(out), rounds


def _reference(keys_full, k):
    order = sorted(range(len(keys_full)), key=lambda j: (-keys_full[j], j))
    valid = [j for j in order if keys_full[j] != 0]
    return sorted(valid[:min(k, len(valid))])


@pytest.mark.parametrize("G,Ns,k,kind", [
    (2, 300, 57, "gauss"), (4, 256, 400, "gauss"), (8, 128, 100, "ties"), (3, 200, 590, "ties"),
    (4, 512, 1000, "all_equal"),     # window > 2048 keys: histogram rounds
    (8, 512, 4000, "wide_ties"),     # > 2048 bracket keys over many values: 2-3 rounds
    (4, 100, 1000, "gauss"),         # k > #valid
    (5, 64, 7, "invalid_tail"),
    (2, 4096, 4000, "outliers"),     # wide [min, max]: the digest bins are coarse -> 3 rounds
    (4, 2048, 3000, "outliers_eq"),
])
def test_shard_protocol_model_exact(G, Ns, k, kind):
    r = np.random.default_rng(G * 1000 + Ns + k)
    N = G * Ns
    if kind == "gauss":
        s = r.standard_normal(N).astype(np.float32)
    elif kind == "ties":
        s = r.integers(0, 12, N).astype(np.float32)
    elif kind == "all_equal":
        s = np.full(N, 3.25, dtype=np.float32)
    elif kind == "wide_ties":
        s = (r.integers(0, 3000, N) * 1e-3 + 1.0).astype(np.float32)
    elif kind == "outliers":
        s = (1.0 + 1e-3 * r.standard_normal(N)).astype(np.float32)
        s[5], s[N - 3] = 1e30, -1e30
    elif kind == "outliers_eq":
        s = np.full(N, 2.0, dtype=np.float32)
        s[7], s[9] = 1e30, -5.0
    else:
        s = r.standard_normal(N).astype(np.float32)
        s[N - 70:] = -np.inf
    keys = SM.row_keys(s, N, 0, N)
    got, rounds = _protocol([keys[i * Ns:(i + 1) * Ns] for i in range(G)], k)
    assert got == _reference(keys, k)
    # the same selection as the oracle's Alg. 3 TopK on the same fp32 scores
    assert got == O.topk_select(s.astype(np.float64), k, N).tolist()


def test_shard_protocol_model_forced_keys():
    """Sink / local window on global positions, shards in rank order."""
    G, Ns, k, sink, window = 4, 100, 50, 7, 13
    N = G * Ns
    n = N - 37
    s = np.random.default_rng(3).integers(0, 5, N).astype(np.float32)
    shard_keys = [SM.row_keys(s[i * Ns:(i + 1) * Ns], n, i * Ns, Ns, sink, window) for i in range(G)]
    got, _ = _protocol(shard_keys, k)
    assert got == O.topk_select(s.astype(np.float64), k, n, sink, window).tolist()


def test_digest_pairs_are_exact_counts():
    s = np.random.default_rng(11).standard_normal(5000).astype(np.float32)
    keys = SM.row_keys(s, 5000, 0, 5000)
    for (e, c) in SM.digest(keys, 700, 4, 64):
        if e:
            assert c == sum(1 for x in keys if x >= e)


# ---------------------------------------------------------------------------
# KV-head sharding
# ---------------------------------------------------------------------------
def _kv_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        from paper_2602_06283_b200.dist import kv_head_shard, kv_head_shard_config
        from paper_2602_06283_b200.ops import Config
        B, H_q, H_kv, N, L, P, k = 1, 8, 4, 256, 16, 8, 40
        c = datagen.make_case(B, H_q, H_kv, N, 128, seed=9)
        W = datagen.make_projections(78, L, P, 128)
        cfg = Config(B=B, H_q=H_q, H_kv=H_kv, N_max=N, L=L, P=P)
        sc = kv_head_shard_config(cfg, world, rank)
        qs, Ks, Vs = kv_head_shard(cfg, world, rank, _bits_t(c["q"]), _bits_t(c["K"]), _bits_t(c["V"]))
        bits = lambda t: t.view(torch.int16).numpy().view(np.uint16)
        r = O.decode_step(bits(qs), bits(Ks), bits(Vs), W, c["seq_lens"], tau=0.5, k=k,
                          sm_scale=1 / np.sqrt(128))
        q.put((rank, sc.H_q, sc.H_kv, {h: r["y"][(0, h)] for h in range(sc.H_q)}))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_kv_head_shard_no_collective():
    import datagen
    world = 2
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_kv_worker, args=(r, world, port, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([qu.get(timeout=540) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = datagen.make_case(1, 8, 4, 256, 128, seed=9)
    W = datagen.make_projections(78, 16, 8, 128)
    ref = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=0.5, k=40, sm_scale=1 / np.sqrt(128))
    for rank, Hq_s, Hkv_s, ys in res:
        assert Hq_s == 4 and Hkv_s == 2
        for h, y in ys.items():
            assert np.array_equal(y, ref["y"][(0, rank * Hq_s + h)])
