"""Hard-LSH scoring (Eq. 3) on the GPU path and the Fig. 2 ranking
harness (metrics P:825-847) at GPU scale.

Hard scores are integer collision counts (times an fp32 norm), so the GPU and
the oracle agree bit for bit once the oracle's double product is rounded to
fp32; the top-k over them (massive exact ties, broken by index, R-15) must
then be identical.
"""
import dataclasses
import json
import os

import numpy as np
import pytest
import torch

import datagen
import oracle as O
from oracle import ranking as RK
from helpers import bits_to_dev

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_2602_06283_b200.ops")
from paper_2602_06283_b200 import Config, KV_SHARED, PER_QHEAD  # noqa: E402

DEV = "cuda"
HARD = 1


def make(B, H_q, H_kv, N, L, P, seed, mode, lens=None):
    c = datagen.make_case(B, H_q, H_kv, N, 128, seed, seq_lens=lens)
    W = datagen.make_projections(2000 + seed, L, P, 128)
    cfg = Config(B=B, H_q=H_q, H_kv=H_kv, N_max=N, L=L, P=P, group_mode=mode, scoring=HARD)
    d = dict(q=bits_to_dev(c["q"]), K=bits_to_dev(c["K"]), V=bits_to_dev(c["V"]), W=bits_to_dev(W),
             seq_lens=torch.from_numpy(c["seq_lens"]).to(DEV))
    return cfg, c, W, d


@pytest.mark.parametrize("mode,P,L", [(KV_SHARED, 8, 60), (PER_QHEAD, 8, 16), (KV_SHARED, 5, 33)])
def test_hard_tables_one_hot(mode, P, L):
    cfg, c, W, d = make(2, 8, 2, 64, L, P, seed=P + L, mode=mode)
    got = ops.query_tables(cfg, d["q"], d["W"]).cpu().numpy()
    ref = O.selection_tables_hard(O.widen(c["q"]), O.widen(W), 2, mode)
    # the query's own bucket is a sign decision: allow only flips of near-zero projections
    x = np.einsum("lpt,bht->bhlp", O.widen(W), O.widen(c["q"]))
    xa = np.einsum("lpt,bht->bhlp", np.abs(O.widen(W)), np.abs(O.widen(c["q"])))
    near = (np.abs(x) <= 1e-12 * xa).any(axis=-1)          # [B, H_q, L]
    diff = np.any(got != ref, axis=-1)                       # [B, H_sel, L]
    if mode == KV_SHARED:
        near = near.reshape(2, 2, 4, L).any(axis=2)
    assert not np.any(diff & ~near)


@pytest.mark.parametrize("mode,lens", [(KV_SHARED, [4096, 3000]), (PER_QHEAD, [2500, 4096])])
def test_hard_scores_bit_exact_and_topk_identical(mode, lens):
    L, P, N, k = 60, 8, 4096, 512
    cfg, c, W, d = make(2, 8, 2, N, L, P, seed=3, mode=mode, lens=lens)
    codes_ref, _ = O.hash_keys(O.widen(c["K"]), O.widen(W))
    codes = ops.pack_codes(cfg, torch.from_numpy(codes_ref.astype(np.uint8)).to(DEV))
    vn = O.value_norms(O.widen(c["V"])).astype(np.float32)
    vnorm = torch.from_numpy(vn).to(DEV)
    got = ops.score(cfg, d["q"], d["W"], codes, vnorm, d["seq_lens"]).cpu().numpy()
    T = O.selection_tables_hard(O.widen(c["q"]), O.widen(W), 2, mode)
    idx, cnt = ops.topk(cfg, torch.from_numpy(got).to(DEV), d["seq_lens"], k)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    for b in range(2):
        for r in range(cfg.H_sel):
            g = r if mode == KV_SHARED else r // 4
            w = O.soft_scores(T[b, r], codes_ref[b, g])                       # integer counts
            s = O.masked_value_scores(w, vn[b, g].astype(np.float64), lens[b])
            s32 = s.astype(np.float32)                                       # one rounding
            assert np.array_equal(got[b, r], s32)
            S = O.topk_select(s32.astype(np.float64), k, lens[b])
            assert cnt[b, r] == len(S) and np.array_equal(idx[b, r, :cnt[b, r]], S)


def test_ranking_harness_soft_beats_hard():
    """Fig. 2 at GPU scale: standard Gaussian keys, ground truth = exact q.k
    top-k.  Soft (SOCKET, tau = 0.5) vs hard LSH selections from the GPU path
    with unit value norms (the plain Eq. 3 / Eq. 4 rankers), averaged over
    queries; soft must win on all three metrics at every k."""
    d, N, L, P, n_q = 128, 4096, 60, 8, 32
    ks = [32, 64, 128, 256, 512]
    r = np.random.default_rng(77)
    K = r.standard_normal((N, d)).astype(np.float32)
    Q = r.standard_normal((n_q, d)).astype(np.float32)
    kdev = torch.from_numpy(K).to(DEV).to(torch.bfloat16)
    qdev = torch.from_numpy(Q).to(DEV).to(torch.bfloat16)
    Kw = kdev.float().cpu().numpy().astype(np.float64)            # the bf16 values both sides see
    Qw = qdev.float().cpu().numpy().astype(np.float64)
    W = datagen.make_projections(4242, L, P, d)
    Wd = bits_to_dev(W)
    base = Config(B=n_q, H_q=1, H_kv=1, N_max=N, L=L, P=P, tau=0.5)
    Kc = kdev.view(1, 1, N, d).expand(n_q, 1, N, d).contiguous()
    codes = ops.alloc_codes(base, DEV)
    ops.hash_keys(base, Kc, Wd, codes)
    ones = torch.ones((n_q, 1, N), dtype=torch.float32, device=DEV)
    lens = torch.full((n_q,), N, dtype=torch.int32, device=DEV)
    q3 = qdev.view(n_q, 1, d)
    res = {}
    for name, cfg in (("soft", base), ("hard", dataclasses.replace(base, scoring=HARD))):
        s = ops.score(cfg, q3, Wd, codes, ones, lens)
        sc = s.cpu().numpy()
        for k in ks:
            idx, cnt = ops.topk(cfg, s, lens, k)
            idx = idx.cpu().numpy()
            m = {"precision": [], "jaccard": [], "ndcg": []}
            for i in range(n_q):
                dots = Kw @ Qw[i]
                truth = np.argsort(-dots, kind="stable")[:k]
                sel = idx[i, 0, :k]
                m["precision"].append(RK.precision(sel, truth))
                m["jaccard"].append(RK.jaccard(sel, truth))
                m["ndcg"].append(RK.ndcg(RK.ranked_selection(sc[i, 0], sel), RK.graded_relevance(dots)))
            res.setdefault(name, {})[k] = {key: float(np.mean(v)) for key, v in m.items()}
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(res, open("gpurun_out/ranking_fig2.json", "w"), indent=1)
    for k in ks:
        for key in ("precision", "jaccard", "ndcg"):
            assert res["soft"][k][key] > res["hard"][k][key], (k, key, res["soft"][k], res["hard"][k])


def _random_hard_cases(n_cases=20, seed=1234):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_cases):
        NH, H_kv = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4]))
        B = int(rng.integers(1, 4))
        N = 32 * int(rng.integers(1, 129))
        mode = PER_QHEAD if rng.random() < 0.3 else KV_SHARED
        lens = [int(rng.integers(0, N + 1)) if rng.random() < 0.4 else N for _ in range(B)]
        k = int(rng.integers(1, N + 1))
        out.append((B, NH * H_kv, H_kv, N, int(rng.integers(1, 65)), int(rng.integers(1, 9)), mode, lens, k,
                    int(rng.integers(0, 1 << 20))))
    return out


@pytest.mark.parametrize("B,H_q,H_kv,N,L,P,mode,lens,k,seed", _random_hard_cases())
def test_hard_scores_random_cases(B, H_q, H_kv, N, L, P, mode, lens, k, seed):
    """Eq. 3 collision counts x ||v|| on seeded random shapes: bit-exact against
    the oracle after its one fp32 rounding, and the top-k over these massively
    tied scores identical to the oracle's TopK (ties to the smaller index)."""
    cfg, c, W, d = make(B, H_q, H_kv, N, L, P, seed, mode, lens=lens)
    codes_ref, _ = O.hash_keys(O.widen(c["K"]), O.widen(W))
    codes = ops.pack_codes(cfg, torch.from_numpy(codes_ref.astype(np.uint8)).to(DEV))
    vn = O.value_norms(O.widen(c["V"])).astype(np.float32)
    got = ops.score(cfg, d["q"], d["W"], codes, torch.from_numpy(vn).to(DEV), d["seq_lens"]).cpu().numpy()
    T = O.selection_tables_hard(O.widen(c["q"]), O.widen(W), H_kv, mode)
    idx, cnt = ops.topk(cfg, torch.from_numpy(got).to(DEV), d["seq_lens"], k)
    idx, cnt = idx.cpu().numpy(), cnt.cpu().numpy()
    G = H_q // H_kv
    for b in range(B):
        for r in range(cfg.H_sel):
            g = r if mode == KV_SHARED else r // G
            w = O.soft_scores(T[b, r], codes_ref[b, g])
            s32 = O.masked_value_scores(w, vn[b, g].astype(np.float64), lens[b]).astype(np.float32)
            assert np.array_equal(got[b, r], s32)
            S = O.topk_select(s32.astype(np.float64), k, lens[b])
            assert cnt[b, r] == len(S) and np.array_equal(idx[b, r, :cnt[b, r]], S)
