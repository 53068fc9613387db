"""SOCKET oracle: a plain, slow, obviously-correct CPU reference in float64.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py` (its `cpu_baseline` leg and `--impl reference`) may import this
module.  The product path (`paper_2602_06283_b200/`, `csrc/`) never imports,
links or executes it, and the two share no code: no kernels, headers, helpers,
table generators, pre- or post-processing.  Inputs come from `datagen/`, which
holds none of the method's arithmetic.

Citations: "P:L" is /root/reference/PAPER.md line L (arxiv 2602.06283, SOCKET).
Every function follows the paper's algorithm in its own order and notation;
library primitives (matmul, exp, tanh, a stable sort) serve as single steps.
Where the paper is silent or ambiguous the reading used is the one listed in
DESIGN.md ("Readings of the paper", R-n), cited inline.

Pins (what keeps this oracle honest) live in tests/test_oracle_pins.py.  Every
function below is pinned there by something other than itself: closed forms,
limits, brute force on tiny inputs, or library routines (see DESIGN.md
"Oracle pins").  No function here is "parity unpinned".

Shapes (decode step):
  q [B][H_q][d], K, V [B][H_kv][N][d], W [L][P][d], seq_lens [B], mask [B][N]
  G = H_q / H_kv (GQA group), g(h) = h // G.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

GROUP_KV_SHARED = 0   # one selection per KV head from the group-summed tables (R-14)
GROUP_PER_QHEAD = 1   # one selection per query head (literal single-query paper setting)


# ---------------------------------------------------------------------------
# input widening (bf16 bits -> float64, exact)
# ---------------------------------------------------------------------------
def widen(bits) -> np.ndarray:
    """bf16 bit patterns (uint16) -> float64, exactly."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# Alg. 1  PrecomputeKeyHashes (prefill)
# ---------------------------------------------------------------------------
def hash_keys(K: np.ndarray, W: np.ndarray):
    """Alg. 1: b_j^(l) = encode(sign(W^(l) k_j)).

    K [..., N, d] float64, W [L, P, d] float64.
    Returns (codes [..., L, N] int64 in [0, 2^P), margin [..., L, P, N]).

    P:203  h^(l)(k_j) <- sign(W^(l) k_j) in {+-1}^P
    P:204  "Encode h^(l)(k_j) as a bucket id b_j^(l) in [R]"
    Readings: sign(0) = +1 (R-3); bit i of the id is hyperplane row i, least
    significant first (R-4).
    margin = |x| / sum_t |W_t k_t| (relative distance of the projection from
    its sign boundary; used to log near-zero projections, north star).
    """
    L, P, d = W.shape
    # x[..., l, i, j] = sum_t W[l, i, t] * K[..., j, t]   (one matmul)
    x = np.einsum("lpt,...nt->...lpn", W, K)
    xabs = np.einsum("lpt,...nt->...lpn", np.abs(W), np.abs(K))
    bits = (x >= 0.0).astype(np.int64)                    # sign(x) = +1  <=>  bit 1
    codes = np.zeros(bits.shape[:-2] + bits.shape[-1:], dtype=np.int64)
    for i in range(P):                                     # bit i <- row i (LSB first)
        codes += bits[..., i, :] << i
    with np.errstate(invalid="ignore", divide="ignore"):
        margin = np.where(xabs > 0, np.abs(x) / xabs, 0.0)
    return codes, margin


def hash_query(q: np.ndarray, W: np.ndarray) -> np.ndarray:
    """Hard bucket of a query (same rule as Alg. 1): b_q^(l)."""
    codes, _ = hash_keys(q[None, :], W)
    return codes[:, 0]


def value_norms(V: np.ndarray) -> np.ndarray:
    """||v_j||_2, Alg. 3 line P:244 and Alg. 4 P:1492.  V [..., N, d]."""
    return np.sqrt(np.sum(V * V, axis=-1))


# ---------------------------------------------------------------------------
# Alg. 2  SoftBucketProbs (decoding)
# ---------------------------------------------------------------------------
def corners(P: int) -> np.ndarray:
    """c_r in {+-1}^P for r in [R]; c_{r,i} = +1 iff bit i of r is set (R-5)."""
    R = 1 << P
    r = np.arange(R)[:, None]
    i = np.arange(P)[None, :]
    return np.where((r >> i) & 1, 1.0, -1.0)


def soft_bucket_probs(q: np.ndarray, W: np.ndarray, tau: float) -> np.ndarray:
    """Alg. 2, literally: enumerate all R = 2^P corners.

    P:217  u^(l)(q) <- (1/sqrt(d)) tanh(W^(l) q)
    P:219  logit^(l)(r) <- u^(l)(q)^T c_r / tau
    P:221  p^(l)(.|q) <- softmax(logit^(l)(1..R))
    q [d], W [L, P, d].  Returns p [L, R] float64.
    """
    L, P, d = W.shape
    u = np.tanh(W @ q) / math.sqrt(d)                      # [L, P]
    logit = (u @ corners(P).T) / tau                       # [L, R]
    logit = logit - logit.max(axis=1, keepdims=True)       # overflow-safe softmax
    e = np.exp(logit)
    return e / e.sum(axis=1, keepdims=True)


def soft_bucket_probs_factorized(q: np.ndarray, W: np.ndarray, tau: float) -> np.ndarray:
    """Same distribution as Alg. 2 via the exact product form.

    Because logit(r) = sum_i u_i c_{r,i} / tau is linear in the corner, the
    corner softmax factorizes:  p(r) = prod_i sigma(2 u_i c_{r,i} / tau)
    (SPEC.md l.139 design note; pinned against the literal enumeration).
    """
    L, P, d = W.shape
    u = np.tanh(W @ q) / math.sqrt(d)                      # [L, P]
    C = corners(P)                                          # [R, P]
    z = 2.0 * u[:, None, :] * C[None, :, :] / tau          # [L, R, P]
    return np.prod(1.0 / (1.0 + np.exp(-z)), axis=2)


def selection_tables(q: np.ndarray, W: np.ndarray, tau: float, H_kv: int,
                     group_mode: int) -> np.ndarray:
    """Per-selection-row tables T[b][row][l][r].

    q [B, H_q, d].  PER_QHEAD: T[b, h] = p_{b,h}.  KV_SHARED (reading R-14):
    T[b, g] = sum_{h in group g} p_{b,h}, so that sum_l T[g, l, b_j] =
    sum_{h in g} w_hat_h(j) -- one selection per KV head from the group's
    summed soft collision scores.
    """
    B, H_q, d = q.shape
    G = H_q // H_kv
    p = np.stack([np.stack([soft_bucket_probs(q[b, h], W, tau) for h in range(H_q)])
                  for b in range(B)])                      # [B, H_q, L, R]
    if group_mode == GROUP_PER_QHEAD:
        return p
    return p.reshape(B, H_kv, G, *p.shape[2:]).sum(axis=2)  # [B, H_kv, L, R]


def selection_tables_hard(q: np.ndarray, W: np.ndarray, H_kv: int,
                          group_mode: int) -> np.ndarray:
    """Hard-LSH tables (Eq. 3): T[b][row][l][r] = [r == b_q^(l)],
    summed over the group's query heads in KV_SHARED mode (reading R-14), so
    that sum_l T[row, l, b_j^(l)] is the collision count of Eq. 3 (summed over
    the group).  b_q^(l) is the query's own bucket by the key rule of Alg. 1
    (hash_query).  q [B, H_q, d]."""
    B, H_q, d = q.shape
    L, P, _ = W.shape
    G = H_q // H_kv
    T = np.zeros((B, H_q, L, 1 << P), dtype=np.float64)
    for b in range(B):
        for h in range(H_q):
            bq = hash_query(q[b, h], W)                     # [L]
            T[b, h, np.arange(L), bq] = 1.0
    if group_mode == GROUP_PER_QHEAD:
        return T
    return T.reshape(B, H_kv, G, L, 1 << P).sum(axis=2)


# ---------------------------------------------------------------------------
# Eq. 4 / Alg. 3 / Alg. 4  soft collision scores
# ---------------------------------------------------------------------------
def soft_scores(T: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Eq. 4: w_hat_j = sum_{l=1..L} p^(l)(b_j^(l) | q).  T [L, R], codes [L, N]."""
    L = T.shape[0]
    w = np.zeros(codes.shape[1], dtype=np.float64)
    for l in range(L):                                      # ascending l
        w += T[l, codes[l]]
    return w


def hard_scores(bq: np.ndarray, codes: np.ndarray) -> np.ndarray:
    """Eq. 3: s_hard(k_j, q) = sum_l 1[b_j^(l) = b_q^(l)]."""
    return np.sum(codes == bq[:, None], axis=0).astype(np.float64)


def masked_value_scores(w_hat: np.ndarray, vnorm: np.ndarray, n: int,
                        mask=None) -> np.ndarray:
    """Alg. 4: -inf if m_j = 0 else ||v_j|| * w_hat_j.

    m_j = 0 for j >= n (positions past the sequence length) or mask[j] = 0.
    Value-norm weighting per Alg. 3 l.244 / Alg. 4 l.1503 (reading R-8).
    """
    N = w_hat.shape[0]
    s = vnorm * w_hat
    valid = np.arange(N) < n
    if mask is not None:
        valid &= np.asarray(mask[:N]) != 0
    return np.where(valid, s, -np.inf)


# ---------------------------------------------------------------------------
# TopK (Alg. 3 l.244) with forced sink / local window
# ---------------------------------------------------------------------------
def topk_select(s: np.ndarray, k: int, n: int, sink: int = 0, window: int = 0) -> np.ndarray:
    """S_k = TopK(s) under the total order (score descending, index ascending).

    Readings: ties go to the smaller index (R-15); -inf keys are never
    selected and k_eff = min(k, #valid) (R-16); the first `sink` and last
    `window` valid positions of [0, n) are forced in and counted inside k (R-17).
    Returns the selected indices in ascending order (int64).
    """
    N = s.shape[0]
    j = np.arange(N)
    valid = ~np.isneginf(s) & (j < n)                       # m_j = 0: -inf or past n (Alg. 4)
    forced = valid & ((j < sink) | ((j >= n - window) & (j < n)))
    n_valid = int(valid.sum())
    k_eff = min(k, n_valid)
    order = np.lexsort((j, -s))                             # primary -s, secondary j (stable)
    chosen = list(j[forced])
    for idx in order:
        if len(chosen) >= k_eff:
            break
        if valid[idx] and not forced[idx]:
            chosen.append(idx)
    return np.sort(np.asarray(chosen, dtype=np.int64))


# ---------------------------------------------------------------------------
# Eq. 2 sparse attention, Eq. 1 dense attention
# ---------------------------------------------------------------------------
def sparse_attention(q: np.ndarray, K: np.ndarray, V: np.ndarray, S: np.ndarray,
                     sm_scale: float):
    """Eq. 2: y = sum_{i in S} alpha_i v_i, alpha = softmax over S of exact logits.

    Exact logits z_i = sm_scale * q^T k_i ("exact attention ... using only this
    subset"; "standard softmax normalization over the selected subset",
    P:309) -- reading R-1 of Alg. 3's garbled alpha line.  sm_scale: R-2.
    Returns (y [d], lse) with lse = log sum_{i in S} exp(z_i); empty S gives
    (0, -inf).
    """
    d = q.shape[0]
    if len(S) == 0:
        return np.zeros(d), -np.inf
    z = sm_scale * (K[S] @ q)
    m = z.max()
    e = np.exp(z - m)
    l = e.sum()
    y = (e[:, None] * V[S]).sum(axis=0) / l
    return y, m + math.log(l)


def dense_attention(q, K, V, n: int, sm_scale: float, mask=None):
    """Eq. 1 (with sm_scale, R-2): attention over every valid key j < n."""
    valid = np.arange(K.shape[0]) < n
    if mask is not None:
        valid &= np.asarray(mask[:K.shape[0]]) != 0
    return sparse_attention(q, K, V, np.nonzero(valid)[0], sm_scale)


def sampling_estimator(s: np.ndarray, vnorm: np.ndarray, V: np.ndarray, n: int,
                       u: np.ndarray):
    """Eq. 6 sampling-based estimator, literally.

    s [N] masked value scores s_j = ||v_j|| w_hat_j (Alg. 4; -inf invalid),
    vnorm [N], V [N, d], n = sequence length, u [M] uniforms in [0, 1).
      w_hat_j = s_j / ||v_j||  (0 where ||v_j|| = 0 or j invalid; reading R-24)
      a~_j = w_hat_j / sum_i w_hat_i
      p_j  = a~_j ||v_j|| / sum_i a~_i ||v_i||
      J_m  = min{ j : sum_{i<=j} p_i > u_m }                  (inverse CDF, J_m ~ p)
      T    = (1/M) sum_m (a~_{J_m} / p_{J_m}) v_{J_m}          (Eq. 6)
    Returns (J [M] int64, T [d]); a row without mass gives J = -1 and T = 0.
    The inverse CDF is evaluated on the unnormalised cumulative sums
    (sum_{i<=j} s_i > u_m sum_i s_i), the same event in exact arithmetic.
    """
    N = s.shape[0]
    valid = (np.arange(N) < n) & np.isfinite(s) & (s > 0)
    sv = np.where(valid, s, 0.0)
    vn = np.asarray(vnorm, dtype=np.float64)
    w_hat = np.where(valid & (vn > 0), sv / np.where(vn > 0, vn, 1.0), 0.0)
    M = u.shape[0]
    if sv.sum() <= 0 or w_hat.sum() <= 0:
        return np.full(M, -1, dtype=np.int64), np.zeros(V.shape[1])
    a = w_hat / w_hat.sum()
    p = a * vn / np.sum(a * vn)
    C = np.cumsum(sv)                                   # sum_{i<=j} s_i, j ascending
    J = np.searchsorted(C, u * C[-1], side="right")     # first j with C_j > u C_n
    J = np.minimum(J, N - 1)
    T = np.zeros(V.shape[1])
    for m in range(M):
        T += (a[J[m]] / p[J[m]]) * V[J[m]]
    return J.astype(np.int64), T / M


def lse_combine(parts):
    """Merge split softmax states: parts = [(y_s, lse_s)] over disjoint subsets.

    y = sum_s exp(lse_s - M) y_s / sum_s exp(lse_s - M); lse = M + log sum exp(lse_s - M).
    (Exact identity of softmax over a disjoint union; pinned in tests.)
    """
    lses = np.array([p[1] for p in parts])
    if np.all(np.isneginf(lses)):
        return np.zeros_like(parts[0][0]), -np.inf
    M = lses.max()
    wts = np.exp(lses - M)
    y = sum(w * p[0] for w, p in zip(wts, parts)) / wts.sum()
    return y, M + math.log(wts.sum())


# ---------------------------------------------------------------------------
# full decode step (hash -> tables -> scores -> top-k -> sparse attention)
# ---------------------------------------------------------------------------
def decode_step(q_bits, K_bits, V_bits, W_bits, seq_lens, *, tau: float, k: int,
                sm_scale: float, group_mode: int = GROUP_KV_SHARED, sink: int = 0,
                window: int = 0, mask=None, codes=None, rows=None):
    """One SOCKET decode step for every (b, head), Alg. 1 -> 2 -> 3.

    q_bits [B,H_q,d], K_bits/V_bits [B,H_kv,N,d], W_bits [L,P,d] (bf16 bits).
    codes: optional precomputed [B,H_kv,L,N] (else Alg. 1 is run here).
    rows: optional list of (b, selection-row) pairs to restrict the work to
    (used to sample full-size cases); None = all.
    Returns dict with codes, vnorm, scores, sel (dict (b,row)->idx), y, lse.
    """
    q = widen(q_bits)
    K = widen(K_bits)
    V = widen(V_bits)
    W = widen(W_bits)
    B, H_q, d = q.shape
    H_kv, N = K.shape[1], K.shape[2]
    G = H_q // H_kv
    H_sel = H_q if group_mode == GROUP_PER_QHEAD else H_kv
    if rows is None:
        rows = [(b, r) for b in range(B) for r in range(H_sel)]
    out = {"scores": {}, "sel": {}, "y": {}, "lse": {}, "w_hat": {}}
    code_cache, vnorm = {}, {}
    for (b, r) in rows:
        g = r if group_mode == GROUP_KV_SHARED else r // G
        if (b, g) not in vnorm:
            vnorm[(b, g)] = value_norms(V[b, g])
            code_cache[(b, g)] = (hash_keys(K[b, g], W)[0] if codes is None
                                  else np.asarray(codes[b, g], dtype=np.int64))
        cg = code_cache[(b, g)]
        heads = list(range(g * G, (g + 1) * G)) if group_mode == GROUP_KV_SHARED else [r]
        T = sum(soft_bucket_probs(q[b, h], W, tau) for h in heads)
        w_hat = soft_scores(T, cg)
        m = None if mask is None else mask[b]
        s = masked_value_scores(w_hat, vnorm[(b, g)], int(seq_lens[b]), m)
        S = topk_select(s, k, int(seq_lens[b]), sink, window)
        out["w_hat"][(b, r)] = w_hat
        out["scores"][(b, r)] = s
        out["sel"][(b, r)] = S
        for h in heads:
            y, lse = sparse_attention(q[b, h], K[b, g], V[b, g], S, sm_scale)
            out["y"][(b, h)] = y
            out["lse"][(b, h)] = lse
    out["codes"] = code_cache
    out["vnorm"] = vnorm
    return out


# ---------------------------------------------------------------------------
# brute-force characterisation of the selection (used only as a pin)
# ---------------------------------------------------------------------------
def topk_bruteforce(s, k, n, sink=0, window=0):
    """Enumerate all subsets; return the unique S with |S| = k_eff that contains
    the forced set and in which every non-forced member beats every valid
    non-member under (score desc, index asc).  Tiny inputs only."""
    N = len(s)
    valid = [not (np.isneginf(s[j])) and j < n for j in range(N)]
    forced = {j for j in range(N) if valid[j] and (j < sink or n - window <= j < n)}
    k_eff = min(k, sum(valid))

    def beats(a, b):
        return s[a] > s[b] or (s[a] == s[b] and a < b)

    found = []
    for S in itertools.combinations([j for j in range(N) if valid[j]], k_eff):
        S = set(S)
        if not forced <= S:
            continue
        free = S - forced
        if all(beats(a, b) for a in free for b in range(N) if valid[b] and b not in S):
            found.append(sorted(S))
    assert len(found) == 1, found
    return np.array(found[0], dtype=np.int64)
