"""GPU parity: every stage of the CUDA path (through the C ABI) against the
float64 oracle on identical seeded inputs.  Tolerances are the north star's
(BASELINE.json) and DESIGN.md "Numerics":
  codes   bit-exact except bits whose oracle margin < 1e-5 (logged)
  tables  <= 2e-6 relative
  scores  <= 1e-5 relative (fp32 vs float64)
  top-k   identical when both sides select from the same fp32 scores;
          vs float64 scores: symmetric difference only at documented near-ties
  output  <= 2e-3 absolute (bf16), lse <= 1e-3 absolute
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
from paper_2602_06283_b200 import _lib  # noqa: E402

DEV = "cuda"


def chained(cfg, on=True):
    """cfg with SOCKET_FLAG_CHAINED_STEP: socket_decode_step never uses the one-launch kernel."""
    import dataclasses
    return dataclasses.replace(cfg, flags=1) if on else cfg


def make(B, H_q, H_kv, N, L, P, seed=0, seq_lens=None, variant="gauss", tau=0.5, mode=KV_SHARED,
         n_needle=0):
    c = datagen.make_case(B, H_q, H_kv, N, 128, seed, variant=variant, seq_lens=seq_lens,
                          n_needle=n_needle)
    W = datagen.make_projections(1000 + seed, L, P, 128)
    cfg = Config(B=B, H_q=H_q, H_kv=H_kv, N_max=N, L=L, P=P, tau=tau, group_mode=mode)
    dev = dict(q=bits_to_dev(c["q"]), K=bits_to_dev(c["K"]), V=bits_to_dev(c["V"]),
               W=bits_to_dev(W), seq_lens=torch.from_numpy(c["seq_lens"]).to(DEV))
    return cfg, c, W, dev


# ---------------------------------------------------------------------------
# Alg. 1 codes and norms
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("B,H,N,L,P", [(1, 1, 4096, 16, 8), (2, 2, 1024, 60, 8), (1, 2, 512, 8, 4),
                                       (1, 1, 256, 64, 8), (1, 1, 256, 3, 2), (1, 1, 128, 100, 8),
                                       (2, 1, 96, 33, 7), (1, 3, 64, 128, 8)])
def test_codes_bit_exact(B, H, N, L, P):
    cfg, c, W, d = make(B, H, H, N, L, P, seed=L + P)
    codes = ops.alloc_codes(cfg, DEV)
    vnorm = torch.zeros((B, H, N), dtype=torch.float32, device=DEV)
    ops.hash_keys(cfg, d["K"], d["W"], codes, V=d["V"], vnorm=vnorm)
    got = ops.unpack_codes(cfg, codes).cpu().numpy().astype(np.int64)
    ref, margin = O.hash_keys(O.widen(c["K"]), O.widen(W))
    diff = got != ref
    if diff.any():
        # a flipped code must be explained by a near-zero projection of that key/table
        bi, hi, li, ji = np.nonzero(diff)
        for b, h, l, j in zip(bi, hi, li, ji):
            flipped = (got[b, h, l, j] ^ ref[b, h, l, j])
            for i in range(P):
                if flipped >> i & 1:
                    assert margin[b, h, l, i, j] < 1e-5, (b, h, l, j, i, margin[b, h, l, i, j])
        print(f"logged {int(diff.sum())} near-zero-margin code flips")
    assert diff.sum() <= max(2, diff.size // 100000)
    vn_ref = O.value_norms(O.widen(c["V"]))
    assert np.max(rel_err(vnorm.cpu().numpy(), vn_ref)) < 1e-6


def test_hash_partial_ranges_touch_only_their_rows():
    cfg, c, W, d = make(1, 2, 2, 256, 16, 8, seed=5)
    codes = ops.alloc_codes(cfg, DEV)
    ref, _ = O.hash_keys(O.widen(c["K"]), O.widen(W))
    ops.hash_keys(cfg, d["K"], d["W"], codes, n_begin=37, n_count=1)    # append-style
    ops.hash_keys(cfg, d["K"], d["W"], codes, n_begin=100, n_count=61)  # ragged range
    got = ops.unpack_codes(cfg, codes).cpu().numpy().astype(np.int64)
    inside = np.zeros(256, bool)
    inside[37] = True
    inside[100:161] = True
    assert np.array_equal(got[..., inside], ref[..., inside])
    assert np.all(got[..., ~inside] == 0)


@pytest.mark.parametrize("L,P", [(60, 8), (16, 8), (8, 5)])
def test_hash_tensor_core_partial_ranges(L, P):
    """Prefill ranges >= 128 keys go through the tcgen05 kernel, including ranges
    that start and end inside 128-key tiles; rows outside stay untouched."""
    cfg, c, W, d = make(2, 2, 2, 640, L, P, seed=L + 3)
    codes = ops.alloc_codes(cfg, DEV)
    ops.hash_keys(cfg, d["K"], d["W"], codes, n_begin=37, n_count=300)
    ops.hash_keys(cfg, d["K"], d["W"], codes, n_begin=384, n_count=256)
    got = ops.unpack_codes(cfg, codes).cpu().numpy().astype(np.int64)
    ref, margin = O.hash_keys(O.widen(c["K"]), O.widen(W))
    inside = np.zeros(640, bool)
    inside[37:337] = True
    inside[384:640] = True
    assert np.all(got[..., ~inside] == 0)
    diff = (got != ref) & inside
    for b, h, l, j in zip(*np.nonzero(diff)):
        flipped = got[b, h, l, j] ^ ref[b, h, l, j]
        for i in range(P):
            if flipped >> i & 1:
                assert margin[b, h, l, i, j] < 1e-5
    assert diff.sum() <= 2


def test_append_path_codes_and_norms():
    """The append path (n_count = 1, decode step) writes codes equal to the
    oracle's (margin rule) and value norms bit-identical to the prefill path."""
    cfg, c, W, d = make(2, 4, 2, 128, 60, 8, seed=6)
    codes = ops.alloc_codes(cfg, DEV)
    vn = torch.zeros((2, 2, 128), dtype=torch.float32, device=DEV)
    ops.hash_keys(cfg, d["K"], d["W"], codes, V=d["V"], vnorm=vn)
    codes2 = ops.alloc_codes(cfg, DEV)
    vn2 = torch.zeros_like(vn)
    js = [0, 31, 32, 77, 127]
    for j in js:
        ops.hash_keys(cfg, d["K"], d["W"], codes2, V=d["V"], vnorm=vn2, n_begin=j, n_count=1)
        assert torch.equal(vn2[:, :, j], vn[:, :, j])
    got = ops.unpack_codes(cfg, codes2).cpu().numpy().astype(np.int64)[..., js]
    ref, margin = O.hash_keys(O.widen(c["K"]), O.widen(W))
    ref, margin = ref[..., js], margin[..., js]
    diff = got != ref
    for b, h, l, jj in zip(*np.nonzero(diff)):
        flipped = got[b, h, l, jj] ^ ref[b, h, l, jj]
        for i in range(8):
            if flipped >> i & 1:
                assert margin[b, h, l, i, jj] < 1e-5


def test_pack_unpack_roundtrip():
    for L in (3, 16, 60, 100):
        cfg = Config(B=2, H_q=2, H_kv=2, N_max=96, L=L, P=8)
        plain = torch.randint(0, 256, (2, 2, L, 96), dtype=torch.uint8, device=DEV)
        assert torch.equal(ops.unpack_codes(cfg, ops.pack_codes(cfg, plain)), plain)


# ---------------------------------------------------------------------------
# Alg. 2 tables
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("P,mode,tau", [(8, KV_SHARED, 0.5), (8, PER_QHEAD, 0.3), (4, KV_SHARED, 0.7),
                                        (1, PER_QHEAD, 0.5), (8, KV_SHARED, 0.05)])
def test_tables(P, mode, tau):
    cfg, c, W, d = make(2, 8, 2, 64, 60, P, seed=P, tau=tau, mode=mode)
    got = ops.query_tables(cfg, d["q"], d["W"]).cpu().numpy()
    ref = O.selection_tables(O.widen(c["q"]), O.widen(W), tau, 2, mode)
    assert got.shape == ref.shape
    assert np.max(rel_err(got, ref)) < table_tol(tau, P)


def table_tol(tau, P):
    """each fp32 factor sigma(+-a) carries <= 3 ulp from
    tanhf/expf/add/div plus 3 ulp * |a| propagated from u, |a| <= 2/(sqrt(128) tau);
    a table entry is a product of P factors (exact in fp64) rounded once, summed
    over <= 8 heads in fp32: P*(3 + 3|a|_max) + 4 ulp."""
    ulp = 2.0 ** -24
    amax = 2.0 / (math.sqrt(128) * tau)
    return (P * (3 + 3 * amax) + 4) * ulp


# ---------------------------------------------------------------------------
# Eq. 4 / Alg. 4 scores
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("L,mode,lens", [(16, KV_SHARED, [4096]), (60, KV_SHARED, [3000, 4096]),
                                         (60, PER_QHEAD, [2500, 17]), (8, KV_SHARED, [4096, 0]),
                                         (64, KV_SHARED, [4090]), (33, PER_QHEAD, [1000])])
def test_scores(L, mode, lens):
    B = len(lens)
    cfg, c, W, d = make(B, 8, 2, 4096, L, 8, seed=L, seq_lens=lens, mode=mode)
    codes_ref, _ = O.hash_keys(O.widen(c["K"]), O.widen(W))
    codes = ops.pack_codes(cfg, torch.from_numpy(codes_ref.astype(np.uint8)).to(DEV))
    vn_ref = O.value_norms(O.widen(c["V"]))
    vnorm = torch.from_numpy(vn_ref.astype(np.float32)).to(DEV)
    mask = torch.ones((B, 4096), dtype=torch.uint8, device=DEV)
    mask[:, 7::97] = 0
    got = ops.score(cfg, d["q"], d["W"], codes, vnorm, d["seq_lens"], mask=mask).cpu().numpy()
    T = O.selection_tables(O.widen(c["q"]), O.widen(W), 0.5, 2, mode)
    G = 4
    for b in range(B):
        for r in range(cfg.H_sel):
            g = r if mode == KV_SHARED else r // G
            w = O.soft_scores(T[b, r], codes_ref[b, g])
            s = O.masked_value_scores(w, vn_ref[b, g].astype(np.float32).astype(np.float64),
                                      lens[b], mask[b].cpu().numpy())
            fin = np.isfinite(s)
            assert np.array_equal(np.isfinite(got[b, r]), fin)
            assert np.all(np.isneginf(got[b, r][~fin]))
            if fin.any():
                assert np.max(rel_err(got[b, r][fin], s[fin])) <= 1e-5


def test_score_rejects_more_than_64_tables():
    cfg, c, W, d = make(1, 4, 1, 64, 100, 8, seed=2)
    codes = ops.alloc_codes(cfg, DEV)
    vn = torch.ones((1, 1, 64), dtype=torch.float32, device=DEV)
    from paper_2602_06283_b200._lib import SocketError
    with pytest.raises(SocketError) as e:
        ops.score(cfg, d["q"], d["W"], codes, vn, d["seq_lens"])
    assert e.value.status == 2   # SOCKET_EUNSUPPORTED


# ---------------------------------------------------------------------------
# Top-k
# ---------------------------------------------------------------------------
def _check_topk_same_scores(cfg, scores, lens, k, sink=0, window=0):
    idx, cnt = ops.topk(cfg, scores, torch.tensor(lens, dtype=torch.int32, device=DEV), k, sink, window)
    s = scores.cpu().numpy().astype(np.float64)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            ref = O.topk_select(s[b, r], k, lens[b], sink, window)
            assert cnt[b, r] == len(ref)
            assert np.array_equal(idx[b, r, :cnt[b, r]], ref)
            assert np.all(idx[b, r, cnt[b, r]:] == -1)


@pytest.mark.parametrize("N,k,lens,sink,window", [
    (4096, 512, [4096], 0, 0), (4096, 512, [4096, 3001], 16, 32), (32768, 3277, [32768], 0, 0),
    (1024, 1024, [1024, 700], 0, 0), (256, 100, [0, 50, 256], 0, 0), (131072, 13107, [131072], 0, 0),
    (2048, 7, [2048], 3, 4),
])
def test_topk_identical_on_same_scores(N, k, lens, sink, window):
    B = len(lens)
    cfg = Config(B=B, H_q=8, H_kv=2, N_max=N, L=16, P=8)
    g = torch.Generator(device=DEV).manual_seed(N + k)
    scores = torch.rand((B, 2, N), generator=g, device=DEV)
    for b, n in enumerate(lens):
        scores[b, :, n:] = -math.inf
    scores[:, :, 5::13] = -math.inf                        # masked keys
    _check_topk_same_scores(cfg, scores, lens, k, sink, window)


def test_topk_heavy_ties():
    """Massive exact ties (scores in {0, .25, .5, .75}): ties go to smaller index."""
    cfg = Config(B=2, H_q=4, H_kv=4, N_max=8192, L=16, P=8)
    g = torch.Generator(device=DEV).manual_seed(3)
    scores = (torch.randint(0, 4, (2, 4, 8192), generator=g, device=DEV).float() / 4)
    _check_topk_same_scores(cfg, scores, [8192, 5000], 1500)
    scores = torch.full((2, 4, 8192), 0.5, device=DEV)      # all equal
    _check_topk_same_scores(cfg, scores, [8192, 8192], 777)


def test_topk_negative_and_large_scores():
    cfg = Config(B=1, H_q=1, H_kv=1, N_max=4096, L=16, P=8)
    g = torch.Generator(device=DEV).manual_seed(4)
    scores = torch.randn((1, 1, 4096), generator=g, device=DEV) * 1e3
    _check_topk_same_scores(cfg, scores, [4096], 333)


# ---------------------------------------------------------------------------
# sparse attention
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [KV_SHARED, PER_QHEAD])
def test_sparse_decode_on_gpu_selection(mode):
    lens = [4096, 1999]
    cfg, c, W, d = make(2, 8, 2, 4096, 16, 8, seed=11, seq_lens=lens, mode=mode)
    k = 512
    g = torch.Generator(device=DEV).manual_seed(9)
    scores = torch.rand((2, cfg.H_sel, 4096), generator=g, device=DEV)
    for b, n in enumerate(lens):
        scores[b, :, n:] = -math.inf
    idx, cnt = ops.topk(cfg, scores, d["seq_lens"], k)
    out, lse = ops.sparse_decode(cfg, d["q"], d["K"], d["V"], idx, cnt, k)
    out = out.float().cpu().numpy()
    lse = lse.cpu().numpy()
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(2):
        for h in range(8):
            r = h // 4 if mode == KV_SHARED else h
            S = idx[b, r, :cnt[b, r]]
            y, l = O.sparse_attention(q[b, h], K[b, h // 4], V[b, h // 4], S, cfg.scale)
            assert np.max(np.abs(out[b, h] - y)) <= 2e-3
            assert abs(lse[b, h] - l) <= 1e-3


def test_sparse_full_budget_equals_dense_and_sdpa():
    N = 1024
    cfg, c, W, d = make(1, 8, 2, N, 16, 8, seed=12)
    idx = torch.arange(N, dtype=torch.int32, device=DEV).repeat(1, 2, 1).contiguous()
    cnt = torch.full((1, 2), N, dtype=torch.int32, device=DEV)
    out_s, lse_s = ops.sparse_decode(cfg, d["q"], d["K"], d["V"], idx, cnt, N)
    out_d, lse_d = ops.dense_decode(cfg, d["q"], d["K"], d["V"], d["seq_lens"])
    assert torch.equal(out_s, out_d)
    qq = d["q"].float().view(1, 8, 1, 128)
    KK = d["K"].float().repeat_interleave(4, dim=1)
    VV = d["V"].float().repeat_interleave(4, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(qq, KK, VV, scale=cfg.scale).view(1, 8, 128)
    assert (out_d.float() - ref).abs().max().item() <= 2e-3


def test_empty_selection_gives_zero_and_neg_inf():
    cfg, c, W, d = make(2, 4, 1, 256, 16, 8, seed=13, seq_lens=[0, 256])
    dec = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=64)
    dec.prefill()
    out, lse = dec.step(d["q"], d["seq_lens"])
    assert torch.all(out[0] == 0) and torch.all(torch.isneginf(lse[0]))
    assert torch.all(torch.isfinite(lse[1]))


def test_lse_combine_matches_union():
    """Partials from disjoint index sets merged == attention over the union."""
    cfg, c, W, d = make(1, 4, 1, 2048, 16, 8, seed=14)
    k = 300
    sel = torch.randperm(2048, generator=torch.Generator().manual_seed(1))[:2 * k].sort().values
    parts = []
    for a in (sel[:k], sel[k:]):
        idx = a.to(torch.int32).view(1, 1, k).to(DEV)
        cnt = torch.full((1, 1), k, dtype=torch.int32, device=DEV)
        p = torch.empty((1, 4, 130), dtype=torch.float32, device=DEV)
        ops.sparse_decode(cfg, d["q"], d["K"], d["V"], idx, cnt, k, partial=p, want_out=False)
        parts.append(p)
    out, lse = ops.lse_combine(cfg, torch.stack(parts))
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    for h in range(4):
        y, l = O.sparse_attention(q[0, h], K[0, 0], V[0, 0], sel.numpy(), cfg.scale)
        assert np.max(np.abs(out[0, h].float().cpu().numpy() - y)) <= 2e-3
        assert abs(lse[0, h].item() - l) <= 1e-3


# ---------------------------------------------------------------------------
# end to end
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [KV_SHARED, PER_QHEAD])
def test_decode_step_c1_end_to_end(mode):
    """BASELINE config 1: single head, n=4096, L=16, P=8, k=512 (+ a GQA case)."""
    for (H_q, H_kv) in ((1, 1), (8, 2)):
        cfg, c, W, d = make(1, H_q, H_kv, 4096, 16, 8, seed=21 + H_q, mode=mode,
                            variant="needle", n_needle=64)
        dec = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=512)
        dec.prefill()
        out, lse = dec.step(d["q"], d["seq_lens"])
        ref = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=0.5, k=512,
                            sm_scale=cfg.scale, group_mode=mode)
        idx, cnt = dec.idx.cpu().numpy(), dec.cnt.cpu().numpy()
        sc = dec.scores.cpu().numpy()
        q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
        for r in range(cfg.H_sel):
            s_ref = ref["scores"][(0, r)]
            fin = np.isfinite(s_ref)
            assert np.max(rel_err(sc[0, r][fin], s_ref[fin])) <= 1e-5
            S_gpu = idx[0, r, :cnt[0, r]]
            S_ref = ref["sel"][(0, r)]
            assert len(S_gpu) == len(S_ref)
            kth = np.sort(s_ref[S_ref])[0]
            for j in np.setxor1d(S_gpu, S_ref):          # documented near-ties only
                assert abs(s_ref[j] - kth) <= 1e-5 * kth, (j, s_ref[j], kth)
        G = H_q // H_kv
        for h in range(H_q):
            r = h // G if mode == KV_SHARED else h
            S = idx[0, r, :cnt[0, r]]
            y, l = O.sparse_attention(q[0, h], K[0, h // G], V[0, h // G], S, cfg.scale)
            assert np.max(np.abs(out[0, h].float().cpu().numpy() - y)) <= 2e-3
            if np.array_equal(S, ref["sel"][(0, r)]):
                assert np.max(np.abs(out[0, h].float().cpu().numpy() - ref["y"][(0, h)])) <= 2e-3


def test_cuda_graph_replay_matches_eager():
    cfg, c, W, d = make(2, 8, 2, 2048, 60, 8, seed=31)
    dec = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=205)
    dec.prefill()
    out_e, lse_e = [t.clone() for t in dec.step(d["q"], d["seq_lens"], append=True)]
    dec.capture(d["q"], d["seq_lens"], append=True)
    out_g, lse_g = dec.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_e, out_g) and torch.equal(lse_e, lse_g)     # deterministic


@pytest.mark.parametrize("B,k", [(16, 3277)])
def test_full_size_c2_sampled(B, k):
    """BASELINE config 2 at full size (32 q / 8 kv heads, 32K, L=60, P=8,
    10x sparsity), launch configuration of bench.py; sampled rows vs oracle."""
    N, L, P = 32768, 60, 8
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=L, P=P, tau=0.5)
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=77)
    Wb = datagen.make_projections(4242, L, P, 128)
    W = bits_to_dev(Wb)
    lens = torch.full((B,), N, dtype=torch.int32, device=DEV)
    dec = SocketDecoder(cfg, W, K, V, k=k)
    dec.prefill()
    out, lse = dec.step(q, lens, append=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    for (b, g) in [(0, 0), (B - 1, 7), (int(rng.integers(B)), int(rng.integers(8)))]:
        Kb = K[b, g].view(torch.int16).cpu().numpy().view(np.uint16)
        Vb = V[b, g].view(torch.int16).cpu().numpy().view(np.uint16)
        qb = q[b, g * 4:(g + 1) * 4].view(torch.int16).cpu().numpy().view(np.uint16)
        ref = O.decode_step(qb[None], Kb[None, None], Vb[None, None], Wb, np.array([N]), tau=0.5,
                            k=k, sm_scale=cfg.scale)
        s_ref = ref["scores"][(0, 0)]
        assert np.max(rel_err(dec.scores[b, g].cpu().numpy(), s_ref)) <= 1e-5
        S_gpu = dec.idx[b, g, :dec.cnt[b, g]].cpu().numpy()
        S_ref = ref["sel"][(0, 0)]
        kth = np.sort(s_ref[S_ref])[0]
        for j in np.setxor1d(S_gpu, S_ref):
            assert abs(s_ref[j] - kth) <= 1e-5 * kth
        qf, Kf, Vf = O.widen(qb), O.widen(Kb), O.widen(Vb)
        for h in range(4):
            y, _ = O.sparse_attention(qf[h], Kf, Vf, S_gpu, cfg.scale)
            assert np.max(np.abs(out[b, g * 4 + h].float().cpu().numpy() - y)) <= 2e-3


def test_decode_step_fused_matches_unfused():
    """socket_decode_step (small batch: the one-launch cluster kernel) gives the
    stage-by-stage calls' codes, norms, scores and selection bit for bit; the
    attention is split per cluster CTA instead of per decode split, so out and
    lse agree to fp32 / bf16 rounding."""
    cfg, c, W, d = make(2, 8, 2, 4096, 60, 8, seed=41)
    a = SocketDecoder(cfg, d["W"], d["K"].clone(), d["V"].clone(), k=409)
    b = SocketDecoder(cfg, d["W"], d["K"].clone(), d["V"].clone(), k=409)
    a.prefill()
    b.prefill()
    oa, la = [t.clone() for t in a.step(d["q"], d["seq_lens"], append=True)]
    ob, lb = [t.clone() for t in b.step_unfused(d["q"], d["seq_lens"], append=True)]
    assert torch.equal(a.codes, b.codes) and torch.equal(a.vnorm, b.vnorm)
    assert torch.equal(a.scores, b.scores)
    assert torch.equal(a.idx, b.idx) and torch.equal(a.cnt, b.cnt)
    assert (oa.float() - ob.float()).abs().max().item() <= 2e-3
    assert ((la - lb).abs() <= 1e-3).all()


@pytest.mark.parametrize("one_launch", [True, False])
def test_decode_step_ragged_sink_window_mask_vs_oracle(one_launch):
    """socket_decode_step with ragged lengths (the append hashes key seq_lens[b]-1
    of each sequence), sink/window forcing and a key mask, against the oracle --
    through the one-launch cluster kernel and through the PDL-chained kernels."""
    lens = [3000, 4096, 1]
    cfg, c, W, d = make(3, 8, 2, 4096, 16, 8, seed=43, seq_lens=lens)
    cfg = chained(cfg, not one_launch)
    k, sink, window = 300, 4, 16
    dec = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=k, sink=sink, window=window)
    dec.prefill(n_tokens=4096)
    mask = torch.ones((3, 4096), dtype=torch.uint8, device=DEV)
    mask[:, 100:200] = 0
    out, lse = dec.step(d["q"], d["seq_lens"], append=True, mask=mask)
    ref = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=0.5, k=k, sm_scale=cfg.scale,
                        sink=sink, window=window, mask=mask.cpu().numpy())
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    idx, cnt = dec.idx.cpu().numpy(), dec.cnt.cpu().numpy()
    sc = dec.scores.cpu().numpy()
    for b in range(3):
        for r in range(2):
            s_ref = ref["scores"][(b, r)]
            fin = np.isfinite(s_ref)
            assert np.array_equal(np.isfinite(sc[b, r]), fin)
            assert np.max(rel_err(sc[b, r][fin], s_ref[fin])) <= 1e-5
            S_ref = ref["sel"][(b, r)]
            S = idx[b, r, :cnt[b, r]]
            assert len(S) == len(S_ref)
            kth = np.sort(s_ref[S_ref])[0] if len(S_ref) else 0
            for j in np.setxor1d(S, S_ref):
                assert abs(s_ref[j] - kth) <= 1e-5 * abs(kth)
            forced = [j for j in range(lens[b]) if (j < sink or j >= lens[b] - window) and mask[b, j]]
            assert set(forced) <= set(S.tolist())
            for h in range(r * 4, r * 4 + 4):
                y, _ = O.sparse_attention(q[b, h], K[b, r], V[b, r], S, cfg.scale)
                assert np.max(np.abs(out[b, h].float().cpu().numpy() - y)) <= 2e-3


@pytest.mark.parametrize("one_launch", [True, False])
def test_decode_step_with_new_rows(one_launch):
    """socket_decode_step(k_new, v_new) stores the new token's rows into the
    cache at seq_lens[b] - 1 and gives exactly the result of writing them first."""
    lens = [2048, 1500]
    cfg, c, W, d = make(2, 8, 2, 2048, 60, 8, seed=51, seq_lens=lens)
    cfg = chained(cfg, not one_launch)
    g = torch.Generator(device=DEV).manual_seed(3)
    k_new = torch.randn((2, 2, 128), generator=g, device=DEV).to(torch.bfloat16)
    v_new = torch.randn((2, 2, 128), generator=g, device=DEV).to(torch.bfloat16)
    Ka, Va = d["K"].clone(), d["V"].clone()
    Kb, Vb = d["K"].clone(), d["V"].clone()
    for b in range(2):
        Kb[b, :, lens[b] - 1] = k_new[b]
        Vb[b, :, lens[b] - 1] = v_new[b]
    a = SocketDecoder(cfg, d["W"], Ka, Va, k=300)
    bb = SocketDecoder(cfg, d["W"], Kb, Vb, k=300)
    a.prefill()
    bb.prefill()
    oa, la = [t.clone() for t in a.step(d["q"], d["seq_lens"], append=True, k_new=k_new, v_new=v_new)]
    ob, lb = [t.clone() for t in bb.step(d["q"], d["seq_lens"], append=True)]
    assert torch.equal(Ka, Kb) and torch.equal(Va, Vb)
    assert torch.equal(a.codes, bb.codes) and torch.equal(a.vnorm, bb.vnorm)
    assert torch.equal(a.idx, bb.idx) and torch.equal(oa, ob) and torch.equal(la, lb)


@pytest.mark.parametrize("one_launch", [True, False])
def test_decode_step_host_inputs_equal_device_inputs(one_launch):
    """q, k_new and v_new in pinned host memory (read in place by the one-launch
    kernel, staged by the copy kernel on the chained path) give bit-identical
    caches, selections and outputs to the same inputs on the device."""
    lens = [2048, 1777]
    cfg, c, W, d = make(2, 8, 2, 2048, 60, 8, seed=57, seq_lens=lens)
    cfg = chained(cfg, not one_launch)
    g = torch.Generator(device=DEV).manual_seed(5)
    k_new = torch.randn((2, 2, 128), generator=g, device=DEV).to(torch.bfloat16)
    v_new = torch.randn((2, 2, 128), generator=g, device=DEV).to(torch.bfloat16)
    Ka, Va = d["K"].clone(), d["V"].clone()
    Kb, Vb = d["K"].clone(), d["V"].clone()
    a = SocketDecoder(cfg, d["W"], Ka, Va, k=300)
    bb = SocketDecoder(cfg, d["W"], Kb, Vb, k=300)
    a.prefill()
    bb.prefill()
    qh, kh, vh = (t.cpu().pin_memory() for t in (d["q"], k_new, v_new))
    oa, la = [t.clone() for t in a.step(qh, d["seq_lens"], append=True, k_new=kh, v_new=vh)]
    ob, lb = [t.clone() for t in bb.step(d["q"], d["seq_lens"], append=True, k_new=k_new, v_new=v_new)]
    torch.cuda.synchronize()
    assert torch.equal(Ka, Kb) and torch.equal(Va, Vb)
    assert torch.equal(a.codes, bb.codes) and torch.equal(a.vnorm, bb.vnorm)
    assert torch.equal(a.idx, bb.idx) and torch.equal(oa, ob) and torch.equal(la, lb)


@pytest.mark.parametrize("B", [4, 8])   # 8 rows: one-launch kernel reading host memory; 16: chained
def test_host_step_graph_matches_device_step(B):
    """bind_host / host_step (pinned host inputs -> graph step -> pinned host
    output) gives the device step's output."""
    cfg, c, W, d = make(B, 8, 2, 2048, 60, 8, seed=53)
    K2, V2 = d["K"].clone(), d["V"].clone()
    a = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=256)
    a.prefill()
    b = SocketDecoder(cfg, d["W"], K2, V2, k=256)
    b.prefill()
    n = 2048
    k_row, v_row = K2[:, :, n - 1].cpu(), V2[:, :, n - 1].cpu()   # bind_host's warm-up rewrites a's
    q_h, k_h, v_h, out_h = a.bind_host(d["seq_lens"])
    q_h.copy_(d["q"].cpu())
    k_h.copy_(k_row)
    v_h.copy_(v_row)
    a.host_step()
    torch.cuda.synchronize()
    ob, _ = b.step(d["q"], d["seq_lens"], append=True)
    assert torch.equal(out_h, ob.cpu())


def one_vs_chained(cfg, d, k, sink=0, window=0):
    """(codes, vnorm, scores, idx, cnt, out, lse) of one appended step through the
    one-launch row-spread kernel (SOCKET_FLAG_ONE_LAUNCH) and through the
    PDL-chained kernels."""
    import dataclasses
    res = []
    for flags in (_lib.FLAG_ONE_LAUNCH, _lib.FLAG_CHAINED_STEP):
        cf = dataclasses.replace(cfg, flags=flags)
        assert ops.decode_step_launches(cf) == (1 if flags == _lib.FLAG_ONE_LAUNCH else 4)
        dec = SocketDecoder(cf, d["W"], d["K"].clone(), d["V"].clone(), k=k, sink=sink, window=window)
        dec.prefill()
        out, lse = dec.step(d["q"], d["seq_lens"], append=True)
        res.append([t.clone() for t in (dec.codes, dec.vnorm, dec.scores, dec.idx, dec.cnt, out, lse)])
    return res


@pytest.mark.parametrize("B,H_q,H_kv,N,L,lens,scoring,sink,window", [
    (1, 1, 1, 4096, 16, [4096], 0, 0, 0),          # configs[0], NH = 1, Lp = 16 (replicated LUT columns)
    (1, 8, 1, 2048, 8, [1000], 0, 0, 0),           # NH = 8, Lp = 8
    (2, 8, 2, 1024, 33, [1024, 0], 0, 2, 8),       # empty sequence, sink/window, Lp = 64
    (1, 4, 2, 8192, 60, [8190], 1, 0, 0),          # hard-LSH tables, n not a multiple of 32
    (4, 8, 2, 2048, 60, [2048, 1, 700, 2047], 0, 0, 4),
    (2, 32, 8, 4096, 60, [4096, 3001], 0, 0, 0),   # 16 rows (the default one-launch grid), 9 CTAs per row
    (4, 32, 8, 2048, 60, [2048, 77, 2000, 1500], 0, 64, 128),   # 32 rows, 4 CTAs per row
    (1, 32, 8, 16384, 60, [16384], 0, 0, 0),       # 18 CTAs per row (B = 1 production geometry)
    (3, 32, 8, 4096, 60, [4096, 4000, 3333], 0, 0, 0),   # 24 rows, 6 CTAs per row: ceil(64 / 6) = 11
    # tables per CTA, rounded to 12 so that the float4 LUT-column stores stay 16-B aligned
    (5, 32, 8, 2048, 60, [2048, 2048, 1500, 999, 2047], 0, 0, 0),   # 40 rows, 3 CTAs per row
])
def test_one_launch_step_matches_chained(B, H_q, H_kv, N, L, lens, scoring, sink, window):
    """The one-launch row-spread step and the PDL-chained kernels agree on every
    output: codes, norms, scores and the selection bit for bit, attention to
    fp32 / bf16 rounding."""
    import dataclasses
    cfg, c, W, d = make(B, H_q, H_kv, N, L, 8, seed=61 + L, seq_lens=lens)
    cfg = dataclasses.replace(cfg, scoring=scoring)
    k = max(sink + window, min(N // 8, 512))
    a, b = one_vs_chained(cfg, d, k, sink, window)
    for x, y in zip(a[:5], b[:5]):
        assert torch.equal(x, y)
    assert (a[5].float() - b[5].float()).abs().max().item() <= 2e-3
    fin = torch.isfinite(b[6])
    assert torch.equal(torch.isfinite(a[6]), fin)
    # the attention weights are rounded to bf16 per tile relative to the running
    # max, which depends on the split: lse agrees within the 1e-3 bar of DESIGN 5
    assert ((a[6][fin] - b[6][fin]).abs() <= 1e-3).all()


@pytest.mark.parametrize("case", ["all_tie", "forced_only", "all_valid", "hard_ties"])
def test_one_launch_selection_modes(case):
    """The one-launch kernel's top-k branches against the chained kernels and the
    oracle's TopK on the same fp32 scores: every key tied (refinement levels down
    to a one-value bin, ties to the smaller index), only forced sink / window keys
    (k_eff <= #forced), k >= #valid (everything), and hard-LSH collision counts."""
    import dataclasses
    B, H_q, H_kv, N = 1, 8, 2, 8192
    cfg, c, W, d = make(B, H_q, H_kv, N, 60, 8, seed=97)
    k, sink, window = 1000, 0, 0
    if case == "all_tie":
        d["W"] = torch.zeros_like(d["W"])                  # every code 255, uniform tables
        d["V"] = d["V"][:, :, :1].expand_as(d["V"]).contiguous()   # every norm equal
    elif case == "forced_only":
        k, sink, window = 96, 48, 48
    elif case == "all_valid":
        d["seq_lens"] = torch.tensor([900], dtype=torch.int32, device=DEV)
    elif case == "hard_ties":
        cfg = dataclasses.replace(cfg, scoring=1)
    a, b = one_vs_chained(cfg, d, k, sink, window)
    for x, y in zip(a[:5], b[:5]):
        assert torch.equal(x, y)
    assert (a[5].float() - b[5].float()).abs().max().item() <= 2e-3
    n = int(d["seq_lens"][0])
    for r in range(H_kv):
        s = a[2][0, r].double().cpu().numpy()
        ref = O.topk_select(s, k, n, sink=sink, window=window)
        assert a[3][0, r, :a[4][0, r]].cpu().numpy().tolist() == list(ref)
    if case == "all_tie":
        assert a[3][0, 0, :k].cpu().numpy().tolist() == list(range(k))


def _random_one_launch_shapes(n_shapes=40, seed=2026):
    """Seeded shapes the one-launch kernel accepts, spread over its geometry:
    1..74 selection rows (2..74 CTAs per row), 1/2/4/8 heads per row, L with and
    without 4-table alignment, ragged and empty rows, sink / window."""
    import dataclasses
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n_shapes:
        NH = int(rng.choice([1, 2, 4, 8]))
        H_kv = int(rng.choice([1, 2, 4, 8]))
        B = int(rng.integers(1, 10))
        if B * H_kv > 74:
            continue
        N = int(rng.choice([256, 512, 1024, 2048, 4096])) + 32 * int(rng.integers(0, 8))
        L = int(rng.choice([8, 13, 16, 24, 31, 33, 45, 60, 64]))
        lens = [int(rng.integers(0, N + 1)) if rng.random() < 0.4 else N for _ in range(B)]
        sink, window = (int(rng.integers(0, 8)), int(rng.integers(0, 32))) if rng.random() < 0.3 else (0, 0)
        k = max(sink + window, int(rng.integers(1, max(2, N // 4))))
        cfg = Config(B=B, H_q=NH * H_kv, H_kv=H_kv, N_max=N, L=L, P=8, flags=_lib.FLAG_ONE_LAUNCH)
        try:
            if ops.decode_step_launches(cfg) != 1:   # host-only geometry query (no GPU needed)
                continue
        except Exception:   # noqa: BLE001 -- library not built: nothing to parametrize
            return out
        out.append((B, NH * H_kv, H_kv, N, L, lens, sink, window, k))
    return out


@pytest.mark.parametrize("B,H_q,H_kv,N,L,lens,sink,window,k", _random_one_launch_shapes())
def test_one_launch_random_shapes(B, H_q, H_kv, N, L, lens, sink, window, k):
    """Seeded random geometries of the one-launch row-spread kernel against the
    chained kernels (bit-identical codes, norms, scores and selection; attention
    to bf16 rounding).  A fixed shape list once missed a misaligned store that
    only 6 CTAs per row produced."""
    cfg, c, W, d = make(B, H_q, H_kv, N, L, 8, seed=7 * B + L, seq_lens=lens)
    a, b = one_vs_chained(cfg, d, k, sink, window)
    for x, y in zip(a[:5], b[:5]):
        assert torch.equal(x, y)
    # each path against the oracle's Eq. 2 on the common selection (DESIGN 5,
    # R-28): 2e-3 absolute, plus one bf16 ulp of the output, plus the bf16
    # rounding of the softmax weights fed to the tensor cores, 2^-8 sum_i a_i |v_i - y|
    # (a_i the exact weights) -- with k down to ~20 keys both terms exceed 2e-3
    Kb, Vb, qb = O.widen(c["K"]), O.widen(c["V"]), O.widen(c["q"])
    G = H_q // H_kv
    for bb in range(B):
        for g in range(H_kv):
            S = b[3][bb, g, :int(b[4][bb, g])].cpu().numpy()
            for h in range(g * G, (g + 1) * G):
                y, lse = O.sparse_attention(qb[bb, h], Kb[bb, g], Vb[bb, g], S, cfg.scale)
                ulp = 2.0 ** (np.floor(np.log2(np.maximum(np.abs(y), 2.0 ** -126))) - 7)
                wr = 0.0
                if len(S):
                    z = cfg.scale * (Kb[bb, g][S] @ qb[bb, h])
                    al = np.exp(z - z.max())
                    al /= al.sum()
                    wr = 2.0 ** -8 * (al[:, None] * np.abs(Vb[bb, g][S] - y)).sum(axis=0)
                tol = 2e-3 + ulp + wr
                for out, ls in ((a[5], a[6]), (b[5], b[6])):
                    assert (np.abs(out[bb, h].float().cpu().numpy() - y) <= tol).all()
                    # lse: 1e-3, plus the bf16 weights' relative error in l, log(1 + 2^-9) < 2^-8
                    if np.isfinite(lse):
                        assert abs(float(ls[bb, h]) - lse) <= 1e-3 + 2.0 ** -8
                    else:
                        assert not torch.isfinite(ls[bb, h])


def _random_step_cases(n_cases=40, seed=2027):
    """Seeded decode-step cases over the chained path's geometry: batch 1..16,
    1..8 KV heads, 1..8 heads per row, both selection modes, N 64..8288, L 1..64,
    P 1..12 (P > 8: packed wide codes), tau, ragged / empty rows, sink / window,
    a key mask, any k <= N."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n_cases:
        NH, H_kv = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8]))
        B = int(rng.integers(1, 17))
        N = int(rng.choice([64, 128, 256, 512, 1024, 2048, 4096, 8192])) + 32 * int(rng.integers(0, 4))
        if B * NH * H_kv * N > 1_500_000:
            continue
        mode = PER_QHEAD if rng.random() < 0.25 else KV_SHARED
        L = int(rng.integers(1, 65))
        P = int(rng.integers(1, 9)) if rng.random() < 0.8 else int(rng.integers(9, 13))
        tau = float(rng.choice([0.25, 0.5, 1.0]))
        lens = [int(rng.integers(0, N + 1)) if rng.random() < 0.4 else N for _ in range(B)]
        sink, window = (int(rng.integers(0, 8)), int(rng.integers(0, 64))) if rng.random() < 0.3 else (0, 0)
        k = int(rng.integers(max(1, sink + window), N + 1))
        masked = bool(rng.random() < 0.3)
        out.append((B, NH * H_kv, H_kv, N, L, P, mode, tau, lens, sink, window, k, masked))
    return out


@pytest.mark.parametrize("B,H_q,H_kv,N,L,P,mode,tau,lens,sink,window,k,masked", _random_step_cases())
def test_chained_step_random_cases_vs_oracle(B, H_q, H_kv, N, L, P, mode, tau, lens, sink, window, k, masked):
    """socket_decode_step through the PDL-chained kernels on seeded random shapes,
    against the oracle: codes bit-exact up to near-zero projection margins, scores
    within 1e-5 relative, the selection identical to the oracle's TopK of the
    GPU's own fp32 scores, attention within the R-28 bound on that selection."""
    cfg, c, W, d = make(B, H_q, H_kv, N, L, P, seed=1000 + 13 * B + L + P, seq_lens=lens, tau=tau, mode=mode)
    cfg = chained(cfg)
    dec = SocketDecoder(cfg, d["W"], d["K"], d["V"], k=k, sink=sink, window=window)
    dec.prefill()
    mask = None
    if masked:
        g = torch.Generator().manual_seed(B * 7919 + N)
        mask = (torch.rand((B, N), generator=g) > 0.2).to(torch.uint8).to(DEV)
    out, lse = dec.step(d["q"], d["seq_lens"], append=True, mask=mask)
    codes = ops.unpack_codes(cfg, dec.codes).cpu().numpy().astype(np.int64)
    ref_codes, margin = O.hash_keys(O.widen(c["K"]), O.widen(W))
    for b, h, l, j in zip(*np.nonzero(codes != ref_codes)):
        flipped = codes[b, h, l, j] ^ ref_codes[b, h, l, j]
        assert all(margin[b, h, l, i, j] < 1e-5 for i in range(P) if flipped >> i & 1)
    ref = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=tau, k=k, sm_scale=cfg.scale,
                        group_mode=mode, sink=sink, window=window, codes=codes,
                        mask=None if mask is None else mask.cpu().numpy())
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    sc, idx, cnt = dec.scores.cpu().numpy(), dec.idx.cpu().numpy(), dec.cnt.cpu().numpy()
    G = H_q // H_kv
    for b in range(B):
        n = lens[b]
        for r in range(cfg.H_sel):
            s_ref = ref["scores"][(b, r)]
            fin = np.isfinite(s_ref)
            assert np.array_equal(np.isfinite(sc[b, r]), fin)
            if fin.any():
                assert np.max(rel_err(sc[b, r][fin], s_ref[fin])) <= 1e-5
            S = idx[b, r, :cnt[b, r]]
            assert S.tolist() == list(O.topk_select(sc[b, r].astype(np.float64), k, n, sink, window))
            g = r if mode == KV_SHARED else r // G
            for h in (range(g * G, (g + 1) * G) if mode == KV_SHARED else [r]):
                y, l_ref = O.sparse_attention(q[b, h], K[b, g], V[b, g], S, cfg.scale)
                tol = 2e-3 + 2.0 ** (np.floor(np.log2(np.maximum(np.abs(y), 2.0 ** -126))) - 7)
                if len(S):
                    z = cfg.scale * (K[b, g][S] @ q[b, h])
                    al = np.exp(z - z.max())
                    al /= al.sum()
                    tol = tol + 2.0 ** -8 * (al[:, None] * np.abs(V[b, g][S] - y)).sum(axis=0)
                assert (np.abs(out[b, h].float().cpu().numpy() - y) <= tol).all()
                if np.isfinite(l_ref):
                    assert abs(float(lse[b, h]) - l_ref) <= 1e-3 + 2.0 ** -8
                else:
                    assert not math.isfinite(float(lse[b, h]))


def _random_hash_cases(n_cases=30, seed=31337):
    """Seeded prefill / append hashing cases: L 1..128, P 1..16, B x H up to 8
    rows, N up to 3000, 1-3 key ranges each (short ranges take the CUDA-core
    kernel, >= 128 keys the tcgen05 GEMM; L > 64 the CUDA-core fallback)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_cases):
        B, H = int(rng.integers(1, 3)), int(rng.choice([1, 2, 4]))
        N = 32 * int(rng.integers(1, 94))
        L = int(rng.choice([1, 3, 8, 16, 31, 33, 60, 64, 100, 128]))
        P = int(rng.integers(1, 17)) if L <= 64 else int(rng.integers(1, 9))
        ranges, start = [], 0
        for _ in range(int(rng.integers(1, 4))):
            if start >= N:
                break
            b0 = int(rng.integers(start, N))
            cnt = int(rng.integers(1, N - b0 + 1))
            ranges.append((b0, cnt))
            start = b0 + cnt
        out.append((B, H, N, L, P, ranges, int(rng.integers(0, 1 << 20))))
    return out


@pytest.mark.parametrize("B,H,N,L,P,ranges,seed", _random_hash_cases())
def test_hash_random_ranges_vs_oracle(B, H, N, L, P, ranges, seed):
    """Alg. 1 codes (and value norms) of seeded random key ranges, bit-exact
    against the oracle up to near-zero projection margins; keys outside the
    ranges stay untouched."""
    cfg, c, W, d = make(B, H, H, N, L, P, seed=seed)
    codes = ops.alloc_codes(cfg, DEV)
    vnorm = torch.full((B, H, N), -1.0, dtype=torch.float32, device=DEV)
    for b0, cnt in ranges:
        ops.hash_keys(cfg, d["K"], d["W"], codes, V=d["V"], vnorm=vnorm, n_begin=b0, n_count=cnt)
    got = ops.unpack_codes(cfg, codes).cpu().numpy().astype(np.int64)
    ref, margin = O.hash_keys(O.widen(c["K"]), O.widen(W))
    inside = np.zeros(N, bool)
    for b0, cnt in ranges:
        inside[b0:b0 + cnt] = True
    assert np.all(got[..., ~inside] == 0)
    vn = vnorm.cpu().numpy()
    assert np.all(vn[..., ~inside] == -1.0)
    vn_ref = O.value_norms(O.widen(c["V"]))
    assert np.max(rel_err(vn[..., inside], vn_ref[..., inside])) < 1e-6
    for b, h, l, j in zip(*np.nonzero((got != ref) & inside)):
        flipped = got[b, h, l, j] ^ ref[b, h, l, j]
        assert all(margin[b, h, l, i, j] < 1e-5 for i in range(P) if flipped >> i & 1)


def _random_topk_cases(n_cases=30, seed=777):
    """Seeded socket_topk cases over its cluster geometries: 1..130 rows, rows of
    32..700000 keys (slices in shared memory up to 16 x 40960 keys, beyond in the
    workspace), any k, ragged / empty rows, sink / window, ties."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n_cases:
        big = rng.random() < 0.15
        N = 32 * int(rng.integers(20480, 21900)) if big else 32 * int(rng.integers(1, 2049))
        B = 1 if big else int(rng.integers(1, 17))
        H = 1 if big else int(rng.choice([1, 2, 4, 8]))
        if B * H * N > 3_000_000:
            continue
        lens = [int(rng.integers(0, N + 1)) if rng.random() < 0.4 else N for _ in range(B)]
        sink, window = (int(rng.integers(0, 16)), int(rng.integers(0, 300))) if rng.random() < 0.3 else (0, 0)
        k = int(rng.integers(max(1, sink + window), N + 1))
        kind = str(rng.choice(["gauss", "ties", "levels2"]))
        out.append((B, H, N, lens, sink, window, k, kind, int(rng.integers(0, 1 << 30))))
    return out


@pytest.mark.parametrize("B,H,N,lens,sink,window,k,kind,seed", _random_topk_cases())
def test_topk_random_cases(B, H, N, lens, sink, window, k, kind, seed):
    """socket_topk on seeded random shapes equals the oracle's Alg. 3 TopK of the
    same fp32 scores (ties to the smaller index, forced sink / window first),
    and the -1 padding past cnt."""
    cfg = Config(B=B, H_q=H, H_kv=H, N_max=N, L=16, P=8)
    g = torch.Generator(device=DEV).manual_seed(seed)
    if kind == "gauss":
        s = torch.randn((B, H, N), generator=g, device=DEV)
    elif kind == "ties":
        s = torch.randint(0, 50, (B, H, N), generator=g, device=DEV).float() * 0.25
    else:
        s = torch.randint(0, 2, (B, H, N), generator=g, device=DEV).float()
    lt = torch.tensor(lens, dtype=torch.int32, device=DEV)
    idx, cnt = ops.topk(cfg, s, lt, k, sink, window)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(B):
        for h in range(H):
            ref = O.topk_select(s[b, h].double().cpu().numpy(), k, lens[b], sink, window)
            assert idx[b, h, :cnt[b, h]].tolist() == ref.tolist()
            assert np.all(idx[b, h, cnt[b, h]:] == -1)


def _random_sparse_cases(n_cases=24, seed=99):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n_cases:
        NH, H_kv = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8]))
        B = int(rng.integers(1, 9))
        N = 32 * int(rng.integers(1, 257))
        if B * NH * H_kv * N > 2_000_000:
            continue
        mode = PER_QHEAD if rng.random() < 0.3 else KV_SHARED
        k = int(rng.integers(1, N + 1))
        out.append((B, NH * H_kv, H_kv, N, mode, k, int(rng.integers(0, 1 << 20))))
    return out


@pytest.mark.parametrize("B,H_q,H_kv,N,mode,k,seed", _random_sparse_cases())
def test_sparse_decode_random_selections(B, H_q, H_kv, N, mode, k, seed):
    """socket_sparse_decode (and its fused split merge) on seeded random
    selections -- random subsets of any size up to k per row, empty rows, -1
    padding -- against the oracle's Eq. 2 (R-28 bound)."""
    cfg, c, W, d = make(B, H_q, H_kv, N, 16, 8, seed=seed, mode=mode)
    rng = np.random.default_rng(seed)
    H_sel = cfg.H_sel
    idx = np.full((B, H_sel, k), -1, np.int32)
    cnt = np.zeros((B, H_sel), np.int32)
    for b in range(B):
        for r in range(H_sel):
            m = 0 if rng.random() < 0.1 else int(rng.integers(1, k + 1))
            idx[b, r, :m] = np.sort(rng.choice(N, m, replace=False))
            cnt[b, r] = m
    out, lse = ops.sparse_decode(cfg, d["q"], d["K"], d["V"], torch.from_numpy(idx).to(DEV),
                                 torch.from_numpy(cnt).to(DEV), k)
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    G = H_q // H_kv
    for b in range(B):
        for h in range(H_q):
            g, r = h // G, (h // G if mode == KV_SHARED else h)
            S = idx[b, r, :cnt[b, r]]
            y, l_ref = O.sparse_attention(q[b, h], K[b, g], V[b, g], S, cfg.scale)
            tol = 2e-3 + 2.0 ** (np.floor(np.log2(np.maximum(np.abs(y), 2.0 ** -126))) - 7)
            if len(S):
                z = cfg.scale * (K[b, g][S] @ q[b, h])
                al = np.exp(z - z.max())
                al /= al.sum()
                tol = tol + 2.0 ** -8 * (al[:, None] * np.abs(V[b, g][S] - y)).sum(axis=0)
            assert (np.abs(out[b, h].float().cpu().numpy() - y) <= tol).all()
            if np.isfinite(l_ref):
                assert abs(float(lse[b, h]) - l_ref) <= 1e-3 + 2.0 ** -8
            else:
                assert not math.isfinite(float(lse[b, h]))


@pytest.mark.parametrize("B,H_q,H_kv,N,L,lens,sink,window,k", _random_one_launch_shapes(16, seed=9091))
def test_one_launch_random_shapes_new_rows(B, H_q, H_kv, N, L, lens, sink, window, k):
    """The same geometries with the new token's K/V rows passed to the step
    (k_new / v_new): the one-launch kernel stores them into the cache at
    seq_lens[b] - 1 exactly as the chained kernels do, and every output agrees."""
    import dataclasses
    cfg, c, W, d = make(B, H_q, H_kv, N, L, 8, seed=11 * B + L, seq_lens=lens)
    g = torch.Generator(device=DEV).manual_seed(B * 31 + L)
    k_new = torch.randn((B, H_kv, 128), generator=g, device=DEV).to(torch.bfloat16)
    v_new = torch.randn((B, H_kv, 128), generator=g, device=DEV).to(torch.bfloat16)
    res = []
    for flags in (_lib.FLAG_ONE_LAUNCH, _lib.FLAG_CHAINED_STEP):
        cf = dataclasses.replace(cfg, flags=flags)
        dec = SocketDecoder(cf, d["W"], d["K"].clone(), d["V"].clone(), k=k, sink=sink, window=window)
        dec.prefill()
        out, lse = dec.step(d["q"], d["seq_lens"], append=True, k_new=k_new, v_new=v_new)
        res.append([t.clone() for t in (dec.K, dec.V, dec.codes, dec.vnorm, dec.scores, dec.idx, dec.cnt,
                                         out, lse)])
    a, b = res
    for x, y in zip(a[:7], b[:7]):
        assert torch.equal(x, y)
    for bb in range(B):
        if 0 < lens[bb] <= N:
            assert torch.equal(a[0][bb, :, lens[bb] - 1], k_new[bb])
            assert torch.equal(a[1][bb, :, lens[bb] - 1], v_new[bb])
    ya, yb = a[7].float(), b[7].float()
    mag = torch.maximum(ya.abs(), yb.abs()).clamp_min(2.0 ** -126)
    # two correct paths: each within the R-28 bound of Eq. 2, so at most twice apart
    assert ((ya - yb).abs() <= 4e-3 + 2 * torch.exp2(torch.floor(torch.log2(mag)) - 7) + 2.0 ** -7 * mag).all()
    fin = torch.isfinite(b[8])
    assert torch.equal(torch.isfinite(a[8]), fin)
    assert ((a[8][fin] - b[8][fin]).abs() <= 2e-3 + 2.0 ** -7).all()


@pytest.mark.parametrize("case", range(12))
def test_partials_and_lse_combine_random_splits(case):
    """A row's selection split at random over G = 2..8 disjoint parts (as the
    sequence shards split it): socket_sparse_decode's partial states of each
    part, merged by socket_lse_combine, equal the oracle's Eq. 2 over the union
    (R-28 bound); empty parts and empty rows included."""
    rng = np.random.default_rng(600 + case)
    G = int(rng.integers(2, 9))
    B, H_kv, NH = int(rng.integers(1, 4)), int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4, 8]))
    N = 32 * int(rng.integers(2, 200))
    mode = PER_QHEAD if rng.random() < 0.3 else KV_SHARED
    cfg, c, W, d = make(B, NH * H_kv, H_kv, N, 16, 8, seed=700 + case, mode=mode)
    k = int(rng.integers(1, N + 1))
    H_sel = cfg.H_sel
    owner = rng.integers(0, G, size=(B, H_sel, N))
    sel = [[np.sort(rng.choice(N, 0 if rng.random() < 0.1 else int(rng.integers(1, k + 1)), replace=False))
            for _ in range(H_sel)] for _ in range(B)]
    parts = []
    for s in range(G):
        idx = np.full((B, H_sel, k), -1, np.int32)
        cnt = np.zeros((B, H_sel), np.int32)
        for b in range(B):
            for r in range(H_sel):
                mine = [j for j in sel[b][r] if owner[b, r, j] == s]
                idx[b, r, :len(mine)] = mine
                cnt[b, r] = len(mine)
        part = torch.empty((B, cfg.H_q, 130), dtype=torch.float32, device=DEV)
        ops.sparse_decode(cfg, d["q"], d["K"], d["V"], torch.from_numpy(idx).to(DEV), torch.from_numpy(cnt).to(DEV),
                          k, partial=part, want_out=False)
        parts.append(part)
    out, lse = ops.lse_combine(cfg, torch.stack(parts))
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    G_h = cfg.H_q // H_kv
    for b in range(B):
        for h in range(cfg.H_q):
            g = h // G_h
            S = sel[b][g if mode == KV_SHARED else h]
            y, l_ref = O.sparse_attention(q[b, h], K[b, g], V[b, g], S, cfg.scale)
            tol = 2e-3 + 2.0 ** (np.floor(np.log2(np.maximum(np.abs(y), 2.0 ** -126))) - 7)
            if len(S):
                z = cfg.scale * (K[b, g][S] @ q[b, h])
                al = np.exp(z - z.max())
                al /= al.sum()
                tol = tol + 2.0 ** -8 * (al[:, None] * np.abs(V[b, g][S] - y)).sum(axis=0)
            assert (np.abs(out[b, h].float().cpu().numpy() - y) <= tol).all()
            if np.isfinite(l_ref):
                assert abs(float(lse[b, h]) - l_ref) <= 1e-3 + 2.0 ** -8
            else:
                assert not math.isfinite(float(lse[b, h]))
