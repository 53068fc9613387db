"""GPU: the exact sequence-shard top-k (socket_topk_digest / _bracket / _window
/ _resolve / _emit) and top-k over rows longer than one cluster's shared memory.

  * every protocol kernel against the host model tests/shard_model.py on the
    same fp32 scores: digests, brackets, resolved states and emits bit for bit,
    window messages as multisets;
  * configs[3] at full size on one GPU through dist.VirtualShards (8 shards of
    131072 keys, 1M-token rows, k = 104858): the global selection equals the
    oracle's Alg. 3 TopK of the same fp32 scores and the single-device
    socket_topk of the 1M-key rows; outputs against the oracle's attention;
  * the same with heavy exact ties at full size.
"""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle as O
import shard_model as SM
from helpers import bits_to_dev

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_2602_06283_b200.ops")
from paper_2602_06283_b200 import Config  # noqa: E402
from paper_2602_06283_b200.dist import VirtualShards, seq_shard_config  # noqa: E402

DEV = "cuda"


def _u32(t):
    return [int(x) & 0xFFFFFFFF for x in t.reshape(-1).tolist()]


def _synthetic(kind, rows, N, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    if kind == "gauss":
        return torch.randn((rows, N), generator=g, device=DEV)
    if kind == "ties":
        return torch.randint(0, 40, (rows, N), generator=g, device=DEV).float() / 40
    if kind == "outliers":
        s = 1.0 + 1e-3 * torch.randn((rows, N), generator=g, device=DEV)
        s[:, 5] = 1e30
        s[:, N - 3] = -1e30
        return s
    raise ValueError(kind)


@pytest.mark.parametrize("kind,G,Ns,k,sink,window", [
    ("gauss", 4, 8192, 3000, 0, 0), ("ties", 4, 8192, 5000, 2, 9), ("outliers", 2, 16384, 9000, 0, 0),
    ("ties", 8, 2048, 300, 0, 0),
])
def test_shard_kernels_match_host_model(kind, G, Ns, k, sink, window):
    B, H_kv = 2, 2
    cfg_full = Config(B=B, H_q=8, H_kv=H_kv, N_max=G * Ns, L=16, P=8)
    full = _synthetic(kind, B * H_kv, G * Ns, 7).view(B, H_kv, G * Ns).contiguous()
    lens = torch.tensor([G * Ns, G * Ns - Ns // 2 - 13], dtype=torch.int32, device=DEV)
    shard_cfg = [seq_shard_config(cfg_full, G, r) for r in range(G)]
    scores = []
    for r in range(G):
        sc = full[:, :, r * Ns:(r + 1) * Ns].clone()
        # past each row's valid length the score kernel writes -inf; garbage must be ignored too
        n_loc = (lens - r * Ns).clamp(0, Ns)
        for b in range(B):
            sc[b, :, int(n_loc[b]):] = 1e9
        scores.append(sc.contiguous())
    # round 1: digests
    digs = [ops.topk_digest(shard_cfg[r], scores[r], lens, k, G, 64, sink=sink, window=window) for r in range(G)]
    keys = {}
    for r in range(G):
        for b in range(B):
            for h in range(H_kv):
                kk = SM.row_keys(scores[r][b, h].cpu().numpy(), int(lens[b]), r * Ns, Ns, sink, window)
                keys[(r, b, h)] = kk
                ref = SM.digest(kk, k, G, 64)
                got = _u32(digs[r][b, h])
                assert got == [x for p in ref for x in p]
    all_d = torch.stack(digs)
    states = [ops.topk_bracket(shard_cfg[r], all_d, k) for r in range(G)]
    model = {}
    for b in range(B):
        for h in range(H_kv):
            digs_m = [SM.digest(keys[(r, b, h)], k, G, 64) for r in range(G)]
            model[(b, h)] = [SM.bracket(digs_m, k) for _ in range(G)]
            for r in range(G):
                assert _u32(states[r][b, h]) == [x & 0xFFFFFFFF for x in SM.state_to_words(model[(b, h)][r])]
    for _ in range(3):
        msgs = [ops.topk_window(shard_cfg[r], scores[r], lens, states[r], sink=sink, window=window)
                for r in range(G)]
        all_m = torch.stack(msgs)
        for r in range(G):
            ops.topk_resolve(shard_cfg[r], all_m, r, states[r])
        for b in range(B):
            for h in range(H_kv):
                mm = [SM.window(keys[(r, b, h)], model[(b, h)][r]) for r in range(G)]
                for r in range(G):
                    got = SM.words_to_msg(_u32(msgs[r][b, h]))
                    if model[(b, h)][r]["resolved"]:
                        continue
                    for f in ("lo", "hi", "above", "wc", "mode", "sh"):
                        assert got[f] == mm[r][f], f
                    pay = sorted(got["payload"]) if got["mode"] == 0 else got["payload"]
                    assert pay == mm[r]["payload"]
                model[(b, h)] = [SM.resolve(mm, r, model[(b, h)][r]) for r in range(G)]
                for r in range(G):
                    assert _u32(states[r][b, h]) == [x & 0xFFFFFFFF for x in SM.state_to_words(model[(b, h)][r])]
    for b in range(B):
        for h in range(H_kv):
            assert all(st["resolved"] for st in model[(b, h)])
    union = {(b, h): [] for b in range(B) for h in range(H_kv)}
    for r in range(G):
        idx, cnt = ops.topk_emit(shard_cfg[r], scores[r], lens, k, states[r], sink=sink, window=window)
        for b in range(B):
            for h in range(H_kv):
                sel = idx[b, h, :int(cnt[b, h])].tolist()
                assert sel == SM.emit(keys[(r, b, h)], model[(b, h)][r])
                union[(b, h)] += [j + r * Ns for j in sel]
    # == Alg. 3 TopK of the concatenated fp32 scores (oracle), and == socket_topk on one device
    idx_f, cnt_f = ops.topk(cfg_full, full, lens, k, sink, window)
    for b in range(B):
        for h in range(H_kv):
            s = full[b, h].double().cpu().numpy()
            ref = O.topk_select(s, k, int(lens[b]), sink, window).tolist()
            assert union[(b, h)] == ref
            assert idx_f[b, h, :int(cnt_f[b, h])].tolist() == ref


@pytest.mark.parametrize("kind", ["ties", "gauss"])
def test_long_row_topk_1m_keys(kind):
    """Rows of 2^20 keys (configs[3] on one device): key slices in the workspace."""
    N, k = 1 << 20, 104858
    cfg = Config(B=1, H_q=32, H_kv=8, N_max=N, L=60, P=8)
    s = _synthetic(kind, 8, N, 11).view(1, 8, N).contiguous()
    lens = torch.tensor([N - 1000], dtype=torch.int32, device=DEV)
    assert ops.workspace_bytes(cfg, 3, k) == 8 * N * 4
    idx, cnt, sel = ops.topk(cfg, s, lens, k, 16, 64, want_scores=True)
    for r in (0, 5):
        sn = s[0, r].double().cpu().numpy()
        ref = O.topk_select(sn, k, N - 1000, 16, 64)
        assert int(cnt[0, r]) == len(ref)
        assert np.array_equal(idx[0, r, :len(ref)].cpu().numpy(), ref)
        assert np.array_equal(sel[0, r, :len(ref)].cpu().numpy(), sn[ref].astype(np.float32))


@pytest.mark.timeout(900)
def test_virtual_shards_configs3_full_size():
    """BASELINE configs[3]: 1M-token context sequence-sharded over 8 shards
    (8 x 131072 keys, 32 q / 8 kv heads, L = 60, P = 8, k = 104858), on one
    GPU through the same kernels and message flow as 8 ranks."""
    G, Ns, k, L = 8, 131072, 104858, 60
    N = G * Ns
    cfg = Config(B=1, H_q=32, H_kv=8, N_max=N, L=L, P=8, tau=0.5)
    q, K, V = datagen.torch_make_cache(1, 32, 8, N, 128, seed=91)
    Wb = datagen.make_projections(4242, L, 8, 128)
    W = bits_to_dev(Wb)
    lens = torch.tensor([N - 777], dtype=torch.int32, device=DEV)
    vs = VirtualShards(cfg, W, K, V, k, G)
    vs.prefill()
    out, lse = vs.step(q, lens)
    torch.cuda.synchronize()
    full = torch.cat([s.scores for s in vs.shards], dim=2)       # [1, 8, N] fp32, the shards' scores
    idx_f, cnt_f = ops.topk(cfg, full, lens, k)
    for r in (0, 3, 7):
        sel = vs.global_selection(0, r)
        sn = full[0, r].double().cpu().numpy()
        ref = O.topk_select(sn, k, N - 777)
        assert sel == ref.tolist()
        assert idx_f[0, r, :int(cnt_f[0, r])].tolist() == sel
        # scores of sampled keys against the oracle (Eq. 4 x ||v||, fp32 vs float64)
        js = np.random.default_rng(r).choice(N - 777, 64, replace=False)
        Kb = K[0, r, js].view(torch.int16).cpu().numpy().view(np.uint16)
        Vb = V[0, r, js].view(torch.int16).cpu().numpy().view(np.uint16)
        qb = q[0, r * 4:(r + 1) * 4].view(torch.int16).cpu().numpy().view(np.uint16)
        Wd, codes = O.widen(Wb), O.hash_keys(O.widen(Kb), O.widen(Wb))[0]
        T = sum(O.soft_bucket_probs(O.widen(qb)[h], Wd, 0.5) for h in range(4))
        s_ref = O.soft_scores(T, codes) * O.value_norms(O.widen(Vb))
        assert np.max(np.abs(sn[js] - s_ref) / s_ref) <= 1e-5
        # outputs of the group's heads over the selected set
        S = np.asarray(sel)
        Ks = O.widen(K[0, r, S].view(torch.int16).cpu().numpy().view(np.uint16))
        Vs = O.widen(V[0, r, S].view(torch.int16).cpu().numpy().view(np.uint16))
        for h in range(r * 4, r * 4 + 4):
            y, l = O.sparse_attention(O.widen(q[0, h].view(torch.int16).cpu().numpy().view(np.uint16)),
                                      Ks, Vs, np.arange(len(S)), cfg.scale)
            assert np.max(np.abs(out[0, h].float().cpu().numpy() - y)) <= 2e-3
            assert abs(float(lse[0, h]) - l) <= 1e-3


def test_virtual_shards_full_size_heavy_ties():
    """The protocol at configs[3] sizes on scores with massive exact ties (40
    levels): every shard's share unions to the single-device selection."""
    G, Ns, k = 8, 131072, 104858
    N = G * Ns
    cfg = Config(B=1, H_q=32, H_kv=8, N_max=N, L=60, P=8)
    full = _synthetic("ties", 8, N, 5).view(1, 8, N).contiguous()
    lens = torch.tensor([N], dtype=torch.int32, device=DEV)
    sc = [seq_shard_config(cfg, G, r) for r in range(G)]
    parts = [full[:, :, r * Ns:(r + 1) * Ns].contiguous() for r in range(G)]
    all_d = torch.stack([ops.topk_digest(sc[r], parts[r], lens, k, G) for r in range(G)])
    st = [ops.topk_bracket(sc[r], all_d, k) for r in range(G)]
    rounds = 0
    while not all(bool((x[..., 3] != 0).all()) for x in st):
        all_m = torch.stack([ops.topk_window(sc[r], parts[r], lens, st[r]) for r in range(G)])
        for r in range(G):
            ops.topk_resolve(sc[r], all_m, r, st[r])
        rounds += 1
        assert rounds <= 3
    idx_f, cnt_f = ops.topk(cfg, full, lens, k)
    got = [[] for _ in range(8)]
    for r in range(G):
        idx, cnt = ops.topk_emit(sc[r], parts[r], lens, k, st[r])
        for h in range(8):
            got[h] += (idx[0, h, :int(cnt[0, h])].long() + r * Ns).tolist()
    for h in range(8):
        assert got[h] == idx_f[0, h, :int(cnt_f[0, h])].tolist()
    ref = O.topk_select(full[0, 2].double().cpu().numpy(), k, N)
    assert got[2] == ref.tolist()


def _random_protocol_cases(n_cases=40, seed=4242):
    """Seeded cases of the exact sequence-shard top-k: 2..8 shards, 32..20000
    keys per shard, any k (also k > keys per shard), ragged rows that end inside
    any shard (or are empty), sink / window, four score distributions."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_cases):
        G = int(rng.integers(2, 9))
        Ns = 32 * int(rng.integers(1, 626))
        N = G * Ns
        B, H = int(rng.integers(1, 4)), int(rng.choice([1, 2, 4]))
        lens = [int(rng.integers(0, N + 1)) if rng.random() < 0.5 else N for _ in range(B)]
        sink, window = (int(rng.integers(0, 16)), int(rng.integers(0, 200))) if rng.random() < 0.4 else (0, 0)
        k = int(rng.integers(max(1, sink + window), N + 1))
        kind = str(rng.choice(["gauss", "ties", "outliers", "levels3"]))
        out.append((G, Ns, B, H, lens, sink, window, k, kind, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("G,Ns,B,H,lens,sink,window,k,kind,seed", _random_protocol_cases())
def test_shard_protocol_random_cases(G, Ns, B, H, lens, sink, window, k, kind, seed):
    """The digest / bracket / window / resolve / emit exchange on seeded random
    shapes: every shard's share unions to the oracle's Alg. 3 TopK of the whole
    row (same fp32 scores) and to the single-device socket_topk, in at most 3
    window rounds."""
    N = G * Ns
    cfg = Config(B=B, H_q=H, H_kv=H, N_max=N, L=16, P=8)
    if kind == "levels3":   # three exact values: massive ties at the threshold
        g = torch.Generator(device=DEV).manual_seed(seed)
        full = torch.randint(0, 3, (B * H, N), generator=g, device=DEV).float()
    else:
        full = _synthetic(kind, B * H, N, seed)
    full = full.view(B, H, N).contiguous()
    lt = torch.tensor(lens, dtype=torch.int32, device=DEV)
    sc = [seq_shard_config(cfg, G, r) for r in range(G)]
    parts = [full[:, :, r * Ns:(r + 1) * Ns].contiguous() for r in range(G)]
    all_d = torch.stack([ops.topk_digest(sc[r], parts[r], lt, k, G, sink=sink, window=window)
                         for r in range(G)])
    st = [ops.topk_bracket(sc[r], all_d, k) for r in range(G)]
    rounds = 0
    while not all(bool((x[..., 3] != 0).all()) for x in st):
        all_m = torch.stack([ops.topk_window(sc[r], parts[r], lt, st[r], sink=sink, window=window)
                             for r in range(G)])
        for r in range(G):
            ops.topk_resolve(sc[r], all_m, r, st[r])
        rounds += 1
        assert rounds <= 3
    got = [[[] for _ in range(H)] for _ in range(B)]
    for r in range(G):
        idx, cnt = ops.topk_emit(sc[r], parts[r], lt, k, st[r], sink=sink, window=window)
        for b in range(B):
            for h in range(H):
                got[b][h] += (idx[b, h, :int(cnt[b, h])].long() + r * Ns).tolist()
    idx_f, cnt_f = ops.topk(cfg, full, lt, k, sink, window)
    for b in range(B):
        for h in range(H):
            ref = O.topk_select(full[b, h].double().cpu().numpy(), k, lens[b], sink, window).tolist()
            assert got[b][h] == ref
            assert idx_f[b, h, :int(cnt_f[b, h])].tolist() == ref
