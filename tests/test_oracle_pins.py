"""Pins for the CPU oracle (tests/-only): every oracle function is checked here
against something other than itself -- closed forms, limits the paper states,
special cases that reduce to a library routine, or brute force on tiny inputs.

Citations: P:L = /root/reference/PAPER.md line L.  R-n = DESIGN.md reading n.
"""
import math

import numpy as np
import pytest
import scipy.integrate
import scipy.special
import scipy.stats
import torch

import oracle as O


def rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


# ---------------------------------------------------------------------------
# Alg. 1 codes
# ---------------------------------------------------------------------------
def test_codes_axis_projections_closed_form():
    """W rows = unit axis vectors e_{t(l,i)}: sign(W k) is sign of a coordinate,
    so b = sum_i [k_{t(l,i)} >= 0] 2^i (R-3: sign(0)=+1, R-4: LSB = row 0)."""
    L, P, d, N = 5, 6, 16, 40
    r = rng(1)
    t = r.integers(0, d, size=(L, P))
    W = np.zeros((L, P, d))
    for l in range(L):
        for i in range(P):
            W[l, i, t[l, i]] = r.uniform(0.5, 2.0)       # positive scale keeps the sign
    K = r.standard_normal((N, d))
    K[3, :] = 0.0                                        # exact zeros -> all bits 1
    K[7, t[0, 0]] = 0.0
    codes, _ = O.hash_keys(K, W)
    for l in range(L):
        for j in range(N):
            expect = sum((1 << i) for i in range(P) if K[j, t[l, i]] >= 0)
            assert codes[l, j] == expect
    assert np.all(codes[:, 3] == (1 << P) - 1)


def test_codes_all_positive_and_antipodal_and_equal_keys():
    """all projections positive -> 2^P-1; k and -k -> complementary
    ids (XOR = 2^P-1); identical keys -> identical ids; permutation equivariance."""
    L, P, d, N = 7, 8, 32, 50
    r = rng(2)
    W = np.abs(r.standard_normal((L, P, d)))
    Kpos = np.abs(r.standard_normal((N, d))) + 0.01
    c, _ = O.hash_keys(Kpos, W)
    assert np.all(c == 255)
    W = r.standard_normal((L, P, d))
    K = r.standard_normal((N, d))
    c1, m = O.hash_keys(K, W)
    c2, _ = O.hash_keys(-K, W)
    assert np.all(m > 0)
    assert np.all((c1 ^ c2) == (1 << P) - 1)
    K2 = np.concatenate([K, K[:5]])
    c3, _ = O.hash_keys(K2, W)
    assert np.all(c3[:, N:] == c3[:, :5])
    perm = r.permutation(N)
    c4, _ = O.hash_keys(K[perm], W)
    assert np.all(c4 == c1[:, perm])


def test_value_norms_library():
    V = rng(3).standard_normal((3, 17, 128))
    assert np.allclose(O.value_norms(V), np.linalg.norm(V, axis=-1), rtol=1e-14, atol=0)


# ---------------------------------------------------------------------------
# Alg. 2 soft bucket probabilities
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("P", [1, 2, 4, 8, 10])
def test_tables_factorized_equals_corner_softmax(P):
    """Literal corner enumeration (Alg. 2) == product of logistic factors (exact
    algebraic identity); SPEC acceptance S:544 bound 1e-10."""
    r = rng(10 + P)
    d, L = 64, 6
    W = r.standard_normal((L, P, d))
    q = r.standard_normal(d)
    for tau in (0.3, 0.5, 0.7, 2.0):
        a = O.soft_bucket_probs(q, W, tau)
        b = O.soft_bucket_probs_factorized(q, W, tau)
        assert np.max(np.abs(a - b)) <= 1e-10


def test_tables_P1_closed_form():
    """P=1: two corners c = -1, +1; p(+1) = e^{u/t}/(e^{u/t}+e^{-u/t}) = sigma(2u/t)."""
    r = rng(4)
    d = 128
    W = r.standard_normal((3, 1, d))
    q = r.standard_normal(d)
    tau = 0.5
    p = O.soft_bucket_probs(q, W, tau)
    for l in range(3):
        u = math.tanh(float(W[l, 0] @ q)) / math.sqrt(d)
        p1 = 1.0 / (1.0 + math.exp(-2.0 * u / tau))
        assert abs(p[l, 1] - p1) < 1e-15 and abs(p[l, 0] - (1 - p1)) < 1e-15


def test_tables_rows_stochastic_argmax_is_hard_bucket():
    """Rows sum to 1; argmax_r p(r|q) = hard bucket of q ('the
    dominant query bucket under soft collision and the hard bucket for q coincide')."""
    r = rng(5)
    d, L, P = 128, 60, 8
    W = r.standard_normal((L, P, d))
    q = r.standard_normal(d)
    p = O.soft_bucket_probs(q, W, 0.5)
    assert np.allclose(p.sum(axis=1), 1.0, atol=1e-12)
    assert np.all(p > 0)
    assert np.all(np.argmax(p, axis=1) == O.hash_query(q, W))
    # the same argument applied to a second table-set, to make the check non-trivial
    W2 = r.standard_normal((L, P, d))
    assert np.all(np.argmax(O.soft_bucket_probs(q, W2, 0.3), axis=1) == O.hash_query(q, W2))


def test_tables_uniform_when_Wq_zero_and_tau_large():
    """Wq = 0 -> all logits equal -> uniform 1/R; tau -> inf ->
    uniform."""
    d, L, P = 32, 4, 8
    W = rng(6).standard_normal((L, P, d))
    assert np.allclose(O.soft_bucket_probs(np.zeros(d), W, 0.5), 1 / 256, atol=1e-15)
    p = O.soft_bucket_probs(rng(7).standard_normal(d), W, 1e6)
    assert np.max(np.abs(p - 1 / 256)) < 1e-8


def test_tables_tau_to_zero_is_one_hot_hard_bucket():
    """tau -> 0: p(b_q|q) -> 1 ('SOCKET reduces to traditional LSH' P:608)."""
    r = rng(8)
    d, L, P = 128, 30, 8
    W = r.standard_normal((L, P, d))
    q = r.standard_normal(d)
    x = W @ q
    keep = np.min(np.abs(np.tanh(x)), axis=1) > 0.05    # tables with a clear logit gap
    p = O.soft_bucket_probs(q, W, 1e-4)
    bq = O.hash_query(q, W)
    assert keep.sum() > 5
    assert np.all(p[keep, bq[keep]] > 1 - 1e-6)


# ---------------------------------------------------------------------------
# Eq. 3 / Eq. 4 / Alg. 4 scores
# ---------------------------------------------------------------------------
def _tables_for(q, W, tau):
    return O.soft_bucket_probs(q, W, tau)


def test_soft_score_tau_zero_equals_hard_collision_count():
    """tau -> 0: w_hat_j -> s_hard(j) = #{l : b_j = b_q} (Eq. 3 vs Eq. 4 limit,
    P:462-464)."""
    r = rng(9)
    d, L, P, N = 128, 40, 4, 300
    W = r.standard_normal((L, P, d))
    q = r.standard_normal(d)
    # keep only tables with a clear gap so the limit is reached at tau=1e-4
    x = W @ q
    W = W[np.min(np.abs(np.tanh(x)), axis=1) > 0.05]
    K = r.standard_normal((N, d))
    codes, _ = O.hash_keys(K, W)
    T = _tables_for(q, W, 1e-4)
    w = O.soft_scores(T, codes)
    h = O.hard_scores(O.hash_query(q, W), codes)
    assert np.max(np.abs(w - h)) < 1e-4
    K[0] = q                                          # a key equal to q collides everywhere
    codes, _ = O.hash_keys(K, W)
    assert O.hard_scores(O.hash_query(q, W), codes)[0] == W.shape[0]


def test_soft_score_tau_inf_is_L_over_R():
    r = rng(11)
    d, L, P, N = 64, 20, 8, 100
    W = r.standard_normal((L, P, d))
    codes, _ = O.hash_keys(r.standard_normal((N, d)), W)
    w = O.soft_scores(_tables_for(r.standard_normal(d), W, 1e7), codes)
    assert np.max(np.abs(w - L / 256)) < 1e-8


def _mu_tau(cos, qnorm, d, tau):
    """Population per-bit soft collision factor (DESIGN.md pin P-4, derived):
    x = w.q ~ N(0,|q|^2), key bit = [w.k >= 0];
    mu = E_x[ sigma(a tanh x) Phi(z) + sigma(-a tanh x) (1 - Phi(z)) ],
    a = 2/(sqrt(d) tau), z = rho x / (|q| sqrt(1 - rho^2))."""
    a = 2.0 / (math.sqrt(d) * tau)
    s = math.sqrt(1 - cos * cos)

    def f(x):
        z = cos * x / (qnorm * s)
        pz = scipy.stats.norm.cdf(z)
        sp = scipy.special.expit(a * math.tanh(x))
        return (sp * pz + (1 - sp) * (1 - pz)) * scipy.stats.norm.pdf(x, scale=qnorm)

    val, _ = scipy.integrate.quad(f, -12 * qnorm, 12 * qnorm, limit=400, points=[0.0])
    return val


@pytest.mark.parametrize("cos,tau", [(0.525, 0.5), (0.9, 0.5), (-0.3, 0.5), (0.525, 0.002), (0.9, 0.002)])
def test_soft_scores_converge_to_collision_kernel(cos, tau):
    """North star: soft scores converge toward the collision-probability kernel as
    L grows.  With i.i.d. Gaussian rows, E_W[p^(l)(b_j|q)] = mu_tau^P exactly and
    w_hat/L concentrates at rate L^-1/2.  As tau -> 0, mu_tau -> 1 -
    theta/pi, the SRP collision probability, i.e. the angular kernel
    of Eq. 7."""
    d, P, L = 128, 8, 6000
    r = rng(int(1000 * (cos + 2) + 1e4 * tau))
    q = r.standard_normal(d)
    e = r.standard_normal(d)
    e -= (e @ q) / (q @ q) * q
    e /= np.linalg.norm(e)
    k = cos * q / np.linalg.norm(q) + math.sqrt(1 - cos * cos) * e
    k *= 7.0                                           # key norm is irrelevant to signs
    W = r.standard_normal((L, P, d))
    codes, _ = O.hash_keys(k[None, :], W)              # [L, 1]
    T = O.soft_bucket_probs(q, W, tau)                 # [L, R]
    per_table = T[np.arange(L), codes[:, 0]]
    w_hat = O.soft_scores(T, codes)[0]
    assert abs(w_hat - per_table.sum()) < 1e-9
    mean, se = w_hat / L, per_table.std(ddof=1) / math.sqrt(L)
    mu = _mu_tau(cos, np.linalg.norm(q), d, tau) ** P
    assert abs(mean - mu) < 5 * se, (mean, mu, se)
    # hard collisions (Eq. 3) obey the SRP identity E[1{b_j=b_q}] = (1-theta/pi)^P
    srp = (1 - math.acos(cos) / math.pi) ** P
    hard = O.hard_scores(O.hash_query(q, W), codes)[0] / L
    se_h = math.sqrt(srp * (1 - srp) / L)
    assert abs(hard - srp) < 5 * se_h
    if tau <= 0.002:
        assert abs(_mu_tau(cos, np.linalg.norm(q), d, tau) - (1 - math.acos(cos) / math.pi)) < 2e-3


def test_masked_value_scores_alg4():
    """Alg. 4: masked -> -inf; ||v||=0 -> 0; uniform norm keeps the
    ranking of w_hat (positive rescaling)."""
    w = np.array([0.3, 0.1, 0.5, 0.2, 0.4])
    vn = np.array([1.0, 0.0, 2.0, 1.0, 1.0])
    s = O.masked_value_scores(w, vn, n=4, mask=np.array([1, 1, 1, 0, 1]))
    assert s[0] == 0.3 and s[1] == 0.0 and s[2] == 1.0
    assert np.isneginf(s[3]) and np.isneginf(s[4])
    s2 = O.masked_value_scores(w, np.full(5, 3.0), n=5)
    assert np.all(np.argsort(-s2, kind="stable") == np.argsort(-w, kind="stable"))


def test_kv_shared_tables_are_sum_of_head_scores():
    """KV_SHARED (R-14): sum_l T_g[l, b_j] == sum_{h in g} w_hat_h(j), where the
    right side is scored head by head (linearity of Eq. 4)."""
    r = rng(12)
    B, H_q, H_kv, d, L, P, N = 1, 8, 2, 32, 9, 8, 64
    W = r.standard_normal((L, P, d))
    q = r.standard_normal((B, H_q, d))
    K = r.standard_normal((N, d))
    codes, _ = O.hash_keys(K, W)
    Tg = O.selection_tables(q, W, 0.5, H_kv, O.GROUP_KV_SHARED)
    Th = O.selection_tables(q, W, 0.5, H_kv, O.GROUP_PER_QHEAD)
    for g in range(H_kv):
        lhs = O.soft_scores(Tg[0, g], codes)
        rhs = sum(O.soft_scores(Th[0, h], codes) for h in range(g * 4, g * 4 + 4))
        assert np.allclose(lhs, rhs, rtol=1e-13)


# ---------------------------------------------------------------------------
# Top-k (Alg. 3 l.244; P:686 sink/window)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(12))
def test_topk_matches_bruteforce_with_ties(seed):
    r = rng(100 + seed)
    N = int(r.integers(1, 10))
    s = r.integers(0, 4, size=N).astype(np.float64)     # heavy exact ties
    n = int(r.integers(0, N + 1))
    s[n:] = -np.inf
    if N > 3:
        s[r.integers(0, n + 1)] = -np.inf if n > 0 else s[0]
    k = int(r.integers(1, N + 1))
    sink = int(r.integers(0, 2))
    window = int(r.integers(0, 2))
    if sink + window > k:
        sink, window = 0, 0
    got = O.topk_select(s, k, n, sink, window)
    exp = O.topk_bruteforce(s, k, n, sink, window)
    assert np.array_equal(got, exp)


def test_topk_special_cases():
    r = rng(13)
    s = r.standard_normal(50)
    assert np.array_equal(O.topk_select(s, 50, 50), np.arange(50))            # k = N: all
    assert np.array_equal(O.topk_select(s, 1, 50), [np.argmax(s)])           # k = 1: argmax
    assert np.array_equal(O.topk_select(s * 3.5, 7, 50), O.topk_select(s, 7, 50))  # rescale
    assert len(O.topk_select(np.full(5, -np.inf), 3, 0)) == 0                # all masked
    s2 = s.copy()
    s2[20:] = -np.inf
    assert np.array_equal(O.topk_select(s2, 30, 20), np.arange(20))          # k > n_valid
    assert np.array_equal(O.topk_select(s, 30, 20), np.arange(20))           # j >= n invalid
    assert np.array_equal(O.topk_bruteforce(s[:8], 3, 5), O.topk_select(s[:8], 3, 5))


# ---------------------------------------------------------------------------
# Eq. 1 / Eq. 2 attention
# ---------------------------------------------------------------------------
def test_sparse_attention_full_budget_equals_sdpa():
    """k = n: Eq. 2 == Eq. 1 == torch SDPA (fp64), SPEC S:542 bound 1e-6 rel."""
    r = rng(14)
    d, N = 128, 300
    q, K, V = r.standard_normal(d), r.standard_normal((N, d)), r.standard_normal((N, d))
    sm = 1 / math.sqrt(d)
    y, lse = O.sparse_attention(q, K, V, np.arange(N), sm)
    yt = torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(q)[None, None, None], torch.tensor(K)[None, None], torch.tensor(V)[None, None],
        scale=sm)[0, 0, 0].numpy()
    assert np.max(np.abs(y - yt)) <= 1e-6 * np.max(np.abs(yt))
    assert abs(lse - scipy.special.logsumexp(sm * (K @ q))) < 1e-12
    y2, _ = O.dense_attention(q, K, V, N, sm)
    assert np.array_equal(y, y2)


def test_sparse_attention_special_cases():
    r = rng(15)
    d, N = 16, 40
    q, K, V = r.standard_normal(d), r.standard_normal((N, d)), r.standard_normal((N, d))
    y, _ = O.sparse_attention(q, K, V, np.array([7]), 0.3)
    assert np.allclose(y, V[7], rtol=0, atol=1e-15)                   # k = 1 -> v
    S = np.array([1, 5, 9, 30])
    y, lse = O.sparse_attention(np.zeros(d), K, V, S, 1.0)             # equal logits
    assert np.allclose(y, V[S].mean(axis=0), atol=1e-15)
    assert abs(lse - math.log(4)) < 1e-15
    y, lse = O.sparse_attention(q, K, V, np.array([], dtype=np.int64), 1.0)
    assert np.all(y == 0) and np.isneginf(lse)


def test_lse_combine_equals_union():
    """Softmax over a disjoint union == LSE merge of the parts (Flash-Decode)."""
    r = rng(16)
    d, N = 32, 200
    q, K, V = r.standard_normal(d), r.standard_normal((N, d)), r.standard_normal((N, d))
    S = np.sort(r.choice(N, 60, replace=False))
    parts = [O.sparse_attention(q, K, V, S[a:b], 0.2) for a, b in [(0, 10), (10, 11), (11, 60)]]
    parts.append(O.sparse_attention(q, K, V, S[:0], 0.2))            # empty part
    y, lse = O.lse_combine(parts)
    y0, lse0 = O.sparse_attention(q, K, V, S, 0.2)
    assert np.max(np.abs(y - y0)) < 1e-13 and abs(lse - lse0) < 1e-13


# ---------------------------------------------------------------------------
# end-to-end decode step
# ---------------------------------------------------------------------------
def test_decode_step_full_budget_is_dense_and_modes_agree_when_G1():
    import datagen
    c = datagen.make_case(B=2, H_q=4, H_kv=4, N_max=96, d=64, seed=3, seq_lens=[96, 61])
    W = datagen.make_projections(9, 6, 8, 64)
    sm = 1 / 8.0
    a = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=0.5, k=96, sm_scale=sm,
                      group_mode=O.GROUP_KV_SHARED)
    b = O.decode_step(c["q"], c["K"], c["V"], W, c["seq_lens"], tau=0.5, k=96, sm_scale=sm,
                      group_mode=O.GROUP_PER_QHEAD)
    q, K, V = O.widen(c["q"]), O.widen(c["K"]), O.widen(c["V"])
    for bb in range(2):
        for h in range(4):
            yd, _ = O.dense_attention(q[bb, h], K[bb, h], V[bb, h], int(c["seq_lens"][bb]), sm)
            assert np.allclose(a["y"][(bb, h)], yd, atol=1e-14)
            assert np.array_equal(a["sel"][(bb, h)], b["sel"][(bb, h)])


@pytest.mark.slow
def test_soft_ranking_beats_hard_on_gaussian_keys():
    """Fig. 2 qualitative claim, as a sanity check: precision of the
    selected set against the exact q.k top-k is higher for soft than hard LSH,
    averaged over seeds (standard Gaussian keys)."""
    d, N, L, P, k = 128, 4096, 60, 8, 256
    soft_p, hard_p = [], []
    for seed in range(6):
        r = rng(500 + seed)
        W = r.standard_normal((L, P, d))
        q, K = r.standard_normal(d), r.standard_normal((N, d))
        codes, _ = O.hash_keys(K, W)
        truth = set(np.argsort(-(K @ q), kind="stable")[:k])
        ws = O.soft_scores(O.soft_bucket_probs(q, W, 0.5), codes)
        wh = O.hard_scores(O.hash_query(q, W), codes)
        soft_p.append(len(truth & set(O.topk_select(ws, k, N))) / k)
        hard_p.append(len(truth & set(O.topk_select(wh, k, N))) / k)
    assert np.mean(soft_p) > np.mean(hard_p)


def test_golden_table6_defaults_are_the_build_defaults():
    """tests/golden/table6_defaults.json: the build's defaults P=8,
    L=60 and tau in [0.3, 0.7] come from Table 6."""
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table6_defaults.json")))
    from paper_2602_06283_b200.ops import Config
    c = Config(B=1, H_q=1, H_kv=1, N_max=32)
    row = g["rows"][0]
    assert (c.P, c.L) == (row["P"], row["L"]) and row["tau"][0] <= c.tau <= row["tau"][1]


# ---------------------------------------------------------------------------
# Hard-LSH tables (Eq. 3) and the Fig. 2 ranking metrics
# ---------------------------------------------------------------------------
def test_hard_tables_give_eq3_collision_counts():
    """sum_l T_hard[l, b_j] is Eq. 3's collision count; tables are one-hot per
    head (KV_SHARED: sums to G); tau -> 0 soft tables tend to them."""
    r = rng(21)
    B, H_q, H_kv, d, L, P, N = 2, 4, 2, 64, 12, 6, 300
    W = r.standard_normal((L, P, d))
    q = r.standard_normal((B, H_q, d))
    K = r.standard_normal((N, d))
    codes, _ = O.hash_keys(K, W)
    Tp = O.selection_tables_hard(q, W, H_kv, O.GROUP_PER_QHEAD)
    assert np.array_equal(Tp.sum(axis=-1), np.ones((B, H_q, L)))
    for b in range(B):
        for h in range(H_q):
            assert np.array_equal(O.soft_scores(Tp[b, h], codes), O.hard_scores(O.hash_query(q[b, h], W), codes))
    Tg = O.selection_tables_hard(q, W, H_kv, O.GROUP_KV_SHARED)
    assert np.array_equal(Tg.sum(axis=-1), np.full((B, H_kv, L), H_q // H_kv))
    assert np.array_equal(Tg[:, 1], Tp[:, 2] + Tp[:, 3])
    # a key equal to the query collides in every table
    K[7] = q[0, 0]
    codes, _ = O.hash_keys(K, W)
    assert O.soft_scores(Tp[0, 0], codes)[7] == L
    # tau -> 0: soft tables -> one-hot at the hard bucket (on tables with a clear margin)
    x = W @ q[0, 0]
    keep = np.min(np.abs(np.tanh(x)), axis=1) > 0.05
    Ts = O.selection_tables(q[:1, :1], W[keep], 1e-4, 1, O.GROUP_PER_QHEAD)[0, 0]
    Th = O.selection_tables_hard(q[:1, :1], W[keep], 1, O.GROUP_PER_QHEAD)[0, 0]
    assert np.max(np.abs(Ts - Th)) < 1e-6


def test_ranking_metrics_closed_forms():
    """P:825-847 definitions on hand-checkable cases."""
    from oracle import ranking as RK
    assert RK.precision([1, 2, 3, 4], [3, 4, 5, 6]) == 0.5
    assert RK.jaccard([1, 2, 3, 4], [3, 4, 5, 6]) == 2 / 6
    assert RK.jaccard([1, 2], [1, 2]) == 1.0 and RK.jaccard([1], [2]) == 0.0
    # DCG of relevances (1, 0, 1): (2^1-1)/log2(2) + 0 + (2^1-1)/log2(4) = 1.5
    assert abs(RK.dcg([1, 0, 1]) - 1.5) < 1e-15
    rel = np.array([0.0, 1.0, 0.5, 0.25])
    assert abs(RK.ndcg([1, 2, 3], rel) - 1.0) < 1e-15            # ideal order
    worse = RK.dcg(rel[[3, 2, 1]]) / RK.dcg([1.0, 0.5, 0.25])
    assert abs(RK.ndcg([3, 2, 1], rel) - worse) < 1e-15 and worse < 1.0
    assert np.array_equal(RK.ranked_selection([0.1, 0.9, 0.5, 0.9], [0, 1, 2, 3]), [1, 3, 2, 0])
    g = RK.graded_relevance([2.0, -1.0, 0.5])
    assert np.allclose(g, [1.0, 0.0, 0.5])


# ---------------------------------------------------------------------------
# Eq. 6 sampling estimator
# ---------------------------------------------------------------------------
def test_sampling_estimator_inverse_cdf_by_hand():
    """Tiny case worked by hand: s = (1, 2, 1) -> C = (1, 3, 4); u = (0.1, 0.3,
    0.8) -> targets (0.4, 1.2, 3.2) -> J = (0, 1, 2); a key past n or with -inf
    score is never drawn."""
    s = np.array([1.0, 2.0, 1.0, 5.0, -np.inf])
    vn = np.array([1.0, 2.0, 4.0, 1.0, 1.0])
    V = np.eye(5, 3)
    J, T = O.sampling_estimator(s, vn, V, 3, np.array([0.1, 0.3, 0.8]))
    assert list(J) == [0, 1, 2]
    # a~ = w_hat / sum w_hat with w_hat = (1, 1, 0.25); p = s / sum s = (1, 2, 1) / 4
    a = np.array([1.0, 1.0, 0.25]) / 2.25
    p = np.array([0.25, 0.5, 0.25])
    ref = (a[0] / p[0] * V[0] + a[1] / p[1] * V[1] + a[2] / p[2] * V[2]) / 3
    assert np.allclose(T, ref, atol=1e-15)
    Jn, Tn = O.sampling_estimator(np.full(4, -np.inf), np.ones(4), np.ones((4, 2)), 4, np.array([0.5]))
    assert list(Jn) == [-1] and np.all(Tn == 0)


def test_sampling_estimator_is_unbiased():
    """E[T] = sum_j a~_j v_j = y_{tau,L}(q): stratified draws
    u_m = (m + 1/2)/M converge at O(1/M); iid draws average to it within 5 sigma."""
    r = rng(31)
    N, d = 40, 8
    s = r.uniform(0.1, 2.0, N)
    vn = r.uniform(0.5, 3.0, N)
    V = r.standard_normal((N, d))
    w_hat = s / vn
    y = (w_hat / w_hat.sum()) @ V
    M = 1 << 16
    _, T = O.sampling_estimator(s, vn, V, N, (np.arange(M) + 0.5) / M)
    assert np.max(np.abs(T - y)) < 2e-3
    runs = np.stack([O.sampling_estimator(s, vn, V, N, r.uniform(size=256))[1] for _ in range(400)])
    se = runs.std(axis=0, ddof=1) / np.sqrt(runs.shape[0])
    assert np.all(np.abs(runs.mean(axis=0) - y) < 5 * se + 1e-12)


# ---------------------------------------------------------------------------
# input widening (bf16 bits -> float64)
# ---------------------------------------------------------------------------
def test_widen_hand_values():
    """Exact values of hand-picked bf16 bit patterns: the bf16 format is the top
    16 bits of an IEEE binary32 (sign, 8 exponent bits, 7 fraction bits)."""
    cases = {
        0x0000: 0.0, 0x3F80: 1.0, 0xC000: -2.0, 0x3F81: 1.0 + 2.0 ** -7, 0x4049: 3.140625,
        0x0001: 2.0 ** -133,                          # smallest subnormal: 2^-126 * 2^-7
        0x0080: 2.0 ** -126,                          # smallest normal
        0x7F7F: (2.0 - 2.0 ** -7) * 2.0 ** 127,      # max finite
        0xFF7F: -(2.0 - 2.0 ** -7) * 2.0 ** 127,
    }
    got = O.widen(np.array(list(cases), dtype=np.uint16))
    assert np.array_equal(got, np.array(list(cases.values())))
    neg0 = O.widen(np.array([0x8000], dtype=np.uint16))[0]
    assert neg0 == 0.0 and math.copysign(1.0, neg0) == -1.0
    inf = O.widen(np.array([0x7F80, 0xFF80], dtype=np.uint16))
    assert inf[0] == math.inf and inf[1] == -math.inf


def test_widen_round_trips_datagen_rounding():
    """widen inverts datagen's fp32 -> bf16 rounding on values that are already
    bf16 (the rounding is then exact), and stays within half a bf16 ulp of the
    fp32 input otherwise (round-to-nearest)."""
    import datagen
    r = rng(77)
    x = r.standard_normal(20000).astype(np.float32) * np.float32(10.0) ** r.integers(-30, 30, 20000).astype(np.float32)
    bits = datagen.bf16_bits_from_f32(x)
    w = O.widen(bits)
    assert np.array_equal(datagen.bf16_bits_from_f32(w.astype(np.float32)), bits)
    ulp = np.abs(w) * 2.0 ** -8
    assert np.all(np.abs(w - x.astype(np.float64)) <= ulp * (1 + 1e-12) + 1e-45)
    # the sign is the top bit, the magnitude the rest
    assert np.array_equal(np.signbit(w), (bits >> 15).astype(bool))
