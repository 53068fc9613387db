"""CPU multi-process checks (gloo, world size 2) of the shard layer (dist.py).

Sequence sharding must select exactly the single-device global top-k (the
shares of the ranks, mapped to global indices, union to the oracle's set) and
produce the single-device output; KV-head sharding needs no collective and
its per-rank outputs concatenate to the full output.  Local compute is the
oracle-backed provider tests/oracle_ops.py; the CUDA resolve kernel itself is
covered by test_gpu_parity.py::test_topk_resolve_virtual_shards.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bits_t(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16)


def _seq_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle_ops
        from paper_2602_06283_b200.dist import SeqShardDecoder
        from paper_2602_06283_b200.ops import Config
        B, H_q, H_kv, Ns, L, P, k = 2, 8, 2, 256, 16, 8, 60
        N = Ns * world
        lens_full = np.array([N, N - 100], dtype=np.int32)        # ragged: shard 1 of b=1 partial
        c = datagen.make_case(B, H_q, H_kv, N, 128, seed=5, seq_lens=lens_full)
        W = datagen.make_projections(77, L, P, 128)
        cfg = Config(B=B, H_q=H_q, H_kv=H_kv, N_max=Ns, L=L, P=P, tau=0.5)
        sl = slice(rank * Ns, (rank + 1) * Ns)
        K = _bits_t(c["K"][:, :, sl].copy())
        V = _bits_t(c["V"][:, :, sl].copy())
        dec = SeqShardDecoder(cfg, _bits_t(W), K, V, k, ops=oracle_ops)
        dec.prefill()
        lens = torch.from_numpy(np.clip(lens_full - rank * Ns, 0, Ns).astype(np.int32))
        out, lse, idx, cnt = dec.step(_bits_t(c["q"]), lens)
        share = {(b, r): (idx[b, r, :cnt[b, r]].numpy() + rank * Ns).tolist()
                 for b in range(B) for r in range(H_kv)}
        q.put((rank, out.numpy(), lse.numpy(), share))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_sequence_shard_exact_topk_and_combine():
    import datagen
    import oracle as O
    world = 2
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_worker, args=(r, world, port, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = [qu.get(timeout=540) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    B, H_q, H_kv, Ns, L, P, k = 2, 8, 2, 256, 16, 8, 60
    N = Ns * world
    lens_full = np.array([N, N - 100], dtype=np.int32)
    c = datagen.make_case(B, H_q, H_kv, N, 128, seed=5, seq_lens=lens_full)
    W = datagen.make_projections(77, L, P, 128)
    ref = O.decode_step(c["q"], c["K"], c["V"], W, lens_full, tau=0.5, k=k,
                        sm_scale=1 / np.sqrt(128))
    for b in range(B):
        for r in range(H_kv):
            union = sorted(res[0][3][(b, r)] + res[1][3][(b, r)])
            assert union == ref["sel"][(b, r)].tolist()
    for rank in range(world):
        out, lse = res[rank][1], res[rank][2]
        for b in range(B):
            for h in range(H_q):
                # partial states travel in the product's fp32 exchange buffers
                assert np.max(np.abs(out[b, h] - ref["y"][(b, h)])) < 1e-6
                assert abs(lse[b, h] - ref["lse"][(b, h)]) < 1e-6


def _kv_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle as O
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
    import oracle as O
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
