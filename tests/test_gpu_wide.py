"""NEXT-2: P > 8 (wide, uint16) codes -- the RULER setting of Table 6 (P = 10-12,
L = 60, "600 bits/token") and P = 16.

Same acceptance as the byte-code path: codes bit-exact (near-zero projection
margins logged), tables within the Alg. 2 ulp budget (+2 ulp for the factored
half-tables, each rounded once), scores <= 1e-5 relative, top-k identical on
identical scores (near-ties vs fp64 documented), attention <= 2e-3.
"""
import math

import numpy as np
import pytest
import torch

import datagen
import oracle as O
from helpers import bits_to_dev, rel_err

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_2602_06283_b200.ops")
from paper_2602_06283_b200 import Config, KV_SHARED, PER_QHEAD, SocketDecoder  # noqa: E402
from paper_2602_06283_b200._lib import SocketError  # noqa: E402

DEV = "cuda"


def make(B, H_q, H_kv, N, L, P, seed, mode=KV_SHARED, lens=None, tau=0.5):
    c = datagen.make_case(B, H_q, H_kv, N, 128, seed, seq_lens=lens)
    W = datagen.make_projections(5000 + seed, L, P, 128)
    cfg = Config(B=B, H_q=H_q, H_kv=H_kv, N_max=N, L=L, P=P, tau=tau, group_mode=mode)
    d = dict(q=bits_to_dev(c["q"]), K=bits_to_dev(c["K"]), V=bits_to_dev(c["V"]), W=bits_to_dev(W),
             seq_lens=torch.from_numpy(c["seq_lens"]).to(DEV))
    return cfg, c, W, d


def plain(cfg, codes):
    return ops.unpack_codes(cfg, codes).cpu().numpy().view(np.uint16).astype(np.int64)


def check_codes(got, ref, margin, P):
    diff = got != ref
    for b, h, l, j in zip(*np.nonzero(diff)):
        flipped = got[b, h, l, j] ^ ref[b, h, l, j]
        for i in range(P):
            if flipped >> i & 1:
                assert margin[b, h, l, i, j] < 1e-5
    assert diff.sum() <= max(2, diff.size // 100000)


@pytest.mark.parametrize("L,P,N", [(60, 10, 1024), (60, 12, 512), (16, 16, 256), (5, 9, 96), (33, 11, 160)])
def test_wide_codes_prefill_and_append(L, P, N):
    cfg, c, W, d = make(2, 2, 2, N, L, P, seed=L + P)
    codes = ops.alloc_codes(cfg, DEV)
    assert codes.numel() == 2 * 2 * N * max(32, cfg.code_slots) * P // 8   # packed: Lp * P bits per key
    vn = torch.zeros((2, 2, N), dtype=torch.float32, device=DEV)
    ops.hash_keys(cfg, d["K"], d["W"], codes, V=d["V"], vnorm=vn)
    ref, margin = O.hash_keys(O.widen(c["K"]), O.widen(W))
    check_codes(plain(cfg, codes), ref, margin, P)
    codes2 = ops.alloc_codes(cfg, DEV)
    js = [0, 31, 33, N - 1]
    for j in js:
        ops.hash_keys(cfg, d["K"], d["W"], codes2, V=d["V"], vnorm=vn, n_begin=j, n_count=1)
    got2 = plain(cfg, codes2)
    check_codes(got2[..., js], ref[..., js], margin[..., js], P)
    other = np.ones(N, bool)
    other[js] = False
    assert np.all(got2[..., other] == 0)


def test_wide_pack_unpack_roundtrip():
    cfg = Config(B=2, H_q=2, H_kv=2, N_max=96, L=60, P=12)
    x = torch.randint(0, 4096, (2, 2, 60, 96), dtype=torch.int32, device=DEV).to(torch.int16)
    assert torch.equal(ops.unpack_codes(cfg, ops.pack_codes(cfg, x)), x)


def table_tol(tau, P):
    ulp = 2.0 ** -24
    amax = 2.0 / (math.sqrt(128) * tau)
    return (P * (3 + 3 * amax) + 6) * ulp


@pytest.mark.parametrize("P,L,mode,tau", [(10, 60, KV_SHARED, 0.5), (12, 20, PER_QHEAD, 0.3),
                                          (16, 3, PER_QHEAD, 0.5), (9, 8, KV_SHARED, 0.7)])
def test_wide_tables(P, L, mode, tau):
    cfg, c, W, d = make(1, 4, 1, 64, L, P, seed=P, mode=mode, tau=tau)
    got = ops.query_tables(cfg, d["q"], d["W"]).cpu().numpy()
    ref = O.selection_tables(O.widen(c["q"]), O.widen(W), tau, 1, mode)
    assert np.max(rel_err(got, ref)) < table_tol(tau, P)


@pytest.mark.parametrize("P,L,mode,lens", [(10, 60, KV_SHARED, [4096, 3000]), (12, 60, PER_QHEAD, [2048, 17]),
                                           (16, 16, PER_QHEAD, [4096, 4096]), (11, 8, KV_SHARED, [100, 4096]),
                                           (9, 33, PER_QHEAD, [4096, 1000]), (10, 20, KV_SHARED, [0, 4095]),
                                           # KV_SHARED half-table images beyond shared memory: tiled
                                           # over (32-slot group, head chunk) with parked partials
                                           (16, 16, KV_SHARED, [4096, 2000]), (13, 60, KV_SHARED, [4096, 4096]),
                                           (14, 40, KV_SHARED, [3000, 4096])])
def test_wide_scores(P, L, mode, lens):
    N = 4096
    cfg, c, W, d = make(2, 8, 2, N, L, P, seed=P * L, mode=mode, lens=lens)
    codes_ref, _ = O.hash_keys(O.widen(c["K"]), O.widen(W))
    codes = ops.pack_codes(cfg, torch.from_numpy(codes_ref.astype(np.uint16).view(np.int16)).to(DEV))
    vn_ref = O.value_norms(O.widen(c["V"]))
    vnorm = torch.from_numpy(vn_ref.astype(np.float32)).to(DEV)
    got = ops.score(cfg, d["q"], d["W"], codes, vnorm, d["seq_lens"]).cpu().numpy()
    T = O.selection_tables(O.widen(c["q"]), O.widen(W), 0.5, 2, mode)
    for b in range(2):
        for r in range(cfg.H_sel):
            g = r if mode == KV_SHARED else r // 4
            w = O.soft_scores(T[b, r], codes_ref[b, g])
            s = O.masked_value_scores(w, vn_ref[b, g].astype(np.float32).astype(np.float64), lens[b])
            fin = np.isfinite(s)
            assert np.array_equal(np.isfinite(got[b, r]), fin)
            if fin.any():
                assert np.max(rel_err(got[b, r][fin], s[fin])) <= 1e-5


@pytest.mark.parametrize("mode,L,P", [(KV_SHARED, 60, 10), (PER_QHEAD, 60, 10), (KV_SHARED, 16, 16)])
def test_wide_decode_step_end_to_end(mode, L, P):
    """RULER-setting step (L = 60, P = 10, 600 bits/token) and P = 16 with a
    group-summed selection (tiled half-tables) through SocketDecoder
    (socket_decode_step): scores, top-k and attention vs the oracle."""
    H_q, H_kv, N, k = 8, 2, 4096, 512
    cfg, c, W, d = make(1, H_q, H_kv, N, L, P, seed=41, mode=mode)
    dec = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=k)
    assert dec.fused           # socket_decode_step: PDL-chained kernels with the wide score
    dec.prefill()
    out, lse = dec.step(d["q"], d["seq_lens"])
    ref = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=0.5, k=k, sm_scale=cfg.scale,
                        group_mode=mode)
    idx, cnt, sc = dec.idx.cpu().numpy(), dec.cnt.cpu().numpy(), dec.scores.cpu().numpy()
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    for r in range(cfg.H_sel):
        s_ref = ref["scores"][(0, r)]
        assert np.max(rel_err(sc[0, r], s_ref)) <= 1e-5
        S_gpu, S_ref = idx[0, r, :cnt[0, r]], ref["sel"][(0, r)]
        assert len(S_gpu) == len(S_ref) == k
        kth = np.sort(s_ref[S_ref])[0]
        for j in np.setxor1d(S_gpu, S_ref):
            assert abs(s_ref[j] - kth) <= 1e-5 * kth
    G = H_q // H_kv
    for h in range(H_q):
        r = h // G if mode == KV_SHARED else h
        S = idx[0, r, :cnt[0, r]]
        y, _ = O.sparse_attention(q[0, h], K[0, h // G], V[0, h // G], S, cfg.scale)
        assert np.max(np.abs(out[0, h].float().cpu().numpy() - y)) <= 2e-3


def _random_score_cases(n_cases=30, seed=5150):
    """Seeded socket_score cases: P 1..16 (byte and packed codes), L 1..64, both
    selection modes, 1..8 heads per row, tau, ragged / empty rows, a key mask."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n_cases:
        NH, H_kv = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4]))
        B = int(rng.integers(1, 4))
        N = 32 * int(rng.integers(1, 97))
        L, P = int(rng.integers(1, 65)), int(rng.integers(1, 17))
        mode = PER_QHEAD if rng.random() < 0.3 else KV_SHARED
        if B * NH * H_kv * N * (1 << max(0, P - 8)) > 4_000_000:
            continue
        lens = [int(rng.integers(0, N + 1)) if rng.random() < 0.4 else N for _ in range(B)]
        out.append((B, NH * H_kv, H_kv, N, L, P, mode, float(rng.choice([0.25, 0.5, 1.0])), lens,
                    bool(rng.random() < 0.3), int(rng.integers(0, 1 << 20))))
    return out


@pytest.mark.parametrize("B,H_q,H_kv,N,L,P,mode,tau,lens,masked,seed", _random_score_cases())
def test_score_random_cases(B, H_q, H_kv, N, L, P, mode, tau, lens, masked, seed):
    """Eq. 4 scores of seeded random configurations (every score kernel: byte
    codes, group-summed P <= 10, factored P >= 11, tiled KV_SHARED images) within
    1e-5 relative of the oracle's, -inf exactly where the oracle has it."""
    cfg, c, W, d = make(B, H_q, H_kv, N, L, P, seed, mode=mode, lens=lens, tau=tau)
    codes_ref, _ = O.hash_keys(O.widen(c["K"]), O.widen(W))
    plain_codes = codes_ref.astype(np.uint8) if P <= 8 else codes_ref.astype(np.uint16).view(np.int16)
    codes = ops.pack_codes(cfg, torch.from_numpy(plain_codes).to(DEV))
    vn_ref = O.value_norms(O.widen(c["V"]))
    vnorm = torch.from_numpy(vn_ref.astype(np.float32)).to(DEV)
    mask = None
    if masked:
        mask = (torch.rand((B, N), generator=torch.Generator().manual_seed(seed)) > 0.25).to(torch.uint8)
    got = ops.score(cfg, d["q"], d["W"], codes, vnorm, d["seq_lens"],
                    mask=None if mask is None else mask.to(DEV)).cpu().numpy()
    T = O.selection_tables(O.widen(c["q"]), O.widen(W), tau, H_kv, mode)
    G = H_q // H_kv
    for b in range(B):
        for r in range(cfg.H_sel):
            g = r if mode == KV_SHARED else r // G
            w = O.soft_scores(T[b, r], codes_ref[b, g])
            s = O.masked_value_scores(w, vn_ref[b, g].astype(np.float32).astype(np.float64), lens[b],
                                      None if mask is None else mask[b].numpy())
            fin = np.isfinite(s)
            assert np.array_equal(np.isfinite(got[b, r]), fin)
            if fin.any():
                assert np.max(rel_err(got[b, r][fin], s[fin])) <= 1e-5
