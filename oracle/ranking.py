"""Ranking-quality metrics of Fig. 2, as defined in the
paper's appendix "Definition of metrics used in fig. ranking_metrics"
(P:825-847).  TEST INFRASTRUCTURE ONLY (see socket_oracle.py header): the
ranking harness (tests/test_ranking_gpu.py) scores the GPU path's selections
with these; the product path never imports them.

Readings (R-22): the "relevant set" R is the exact top-k of the
ground-truth relevance q.k_j ("ground-truth relevance is defined by
dot-product similarity"); the graded relevance r_j fed to NDCG is q.k_j
min-max scaled to [0, 1] over the row (the paper gives no scale, and 2^{q.k}
would overflow); IDCG is the DCG of the k most relevant items of the whole
row in decreasing relevance order; a method's ranked list is its selected set
in decreasing order of its own score (ties: smaller index first).
"""
from __future__ import annotations

import numpy as np


def precision(selected, relevant) -> float:
    """|S_k intersect R| / k, k = |S_k|."""
    S = set(int(x) for x in selected)
    return len(S & set(int(x) for x in relevant)) / max(1, len(S))


def jaccard(a, b) -> float:
    """|A intersect B| / |A union B|."""
    A, B = set(int(x) for x in a), set(int(x) for x in b)
    u = A | B
    return len(A & B) / len(u) if u else 1.0


def dcg(rel_in_rank_order) -> float:
    """sum_{i=1..k} (2^{r_i} - 1) / log2(i + 1)."""
    r = np.asarray(rel_in_rank_order, dtype=np.float64)
    i = np.arange(1, r.size + 1, dtype=np.float64)
    return float(np.sum((np.power(2.0, r) - 1.0) / np.log2(i + 1.0)))


def ndcg(ranked, relevance) -> float:
    """DCG / IDCG; `ranked` is the method's list (best first),
    `relevance` the graded relevance of every item of the row."""
    rel = np.asarray(relevance, dtype=np.float64)
    k = len(ranked)
    ideal = np.sort(rel)[::-1][:k]
    idcg = dcg(ideal)
    return dcg(rel[np.asarray(ranked, dtype=np.int64)]) / idcg if idcg > 0 else 1.0


def graded_relevance(dots) -> np.ndarray:
    """q.k_j min-max scaled to [0, 1] over the row (reading R-22)."""
    x = np.asarray(dots, dtype=np.float64)
    lo, hi = x.min(), x.max()
    return (x - lo) / (hi - lo) if hi > lo else np.zeros_like(x)


def ranked_selection(scores, selected) -> np.ndarray:
    """Selected indices ordered by score descending, ties to the smaller index."""
    sel = np.asarray(selected, dtype=np.int64)
    s = np.asarray(scores, dtype=np.float64)[sel]
    order = np.lexsort((sel, -s))
    return sel[order]
