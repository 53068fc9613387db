"""Oracle-backed local-ops provider with the call signatures of
paper_2602_06283_b200.ops, used ONLY by the CPU (gloo) tests of the shard
layer (tests/test_dist_gloo.py).  It lets dist.py's orchestration -- the
collectives, rank order, shard offsets and the exact sequence-shard top-k
protocol (tests/shard_model.py) -- be checked on CPU processes; the CUDA
kernels themselves are covered by the -m gpu tests.
"""
import numpy as np
import torch

import oracle as O
import shard_model as SM


def _w(t):
    return O.widen(t.contiguous().view(torch.int16).numpy().view(np.uint16))


def alloc_codes(cfg, device):
    return torch.zeros((cfg.B, cfg.H_kv, cfg.L, cfg.N_max), dtype=torch.int64)


def hash_keys(cfg, K, W, codes, V=None, vnorm=None, n_begin=0, n_count=None):
    n_count = cfg.N_max - n_begin if n_count is None else n_count
    sl = slice(n_begin, n_begin + n_count)
    c, _ = O.hash_keys(_w(K)[:, :, sl], _w(W))
    codes[..., sl] = torch.from_numpy(c)
    if V is not None:
        vnorm[..., sl] = torch.from_numpy(O.value_norms(_w(V)[:, :, sl])).float()
    return codes


def score(cfg, q, W, codes, vnorm, seq_lens, mask=None, out=None, ws=None):
    T = O.selection_tables(_w(q), _w(W), cfg.tau, cfg.H_kv, cfg.group_mode)
    G = cfg.H_q // cfg.H_kv
    s = np.empty((cfg.B, cfg.H_sel, cfg.N_max))
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            g = r if cfg.group_mode == O.GROUP_KV_SHARED else r // G
            w = O.soft_scores(T[b, r], codes[b, g].numpy())
            n = max(0, min(int(seq_lens[b]) - cfg.index_base, cfg.N_max))   # global lengths
            s[b, r] = O.masked_value_scores(w, vnorm[b, g].double().numpy(), n)
    # the product's scores are fp32: round so the protocol sees the same kind of keys
    t = torch.from_numpy(s).float()
    if out is not None:
        out.copy_(t)
        return out
    return t


def topk(cfg, scores, seq_lens, k, sink=0, window=0, idx=None, cnt=None, sel_scores=None,
         want_scores=False):
    B, H = scores.shape[:2]
    idx = torch.full((B, H, k), -1, dtype=torch.int32)
    cnt = torch.zeros((B, H), dtype=torch.int32)
    sc = torch.full((B, H, k), -np.inf, dtype=torch.float64)
    for b in range(B):
        for r in range(H):
            s = scores[b, r].numpy()
            S = O.topk_select(s, k, int(seq_lens[b]), sink, window)
            idx[b, r, :len(S)] = torch.from_numpy(S.astype(np.int32))
            cnt[b, r] = len(S)
            sc[b, r, :len(S)] = torch.from_numpy(s[S])
    return (idx, cnt, sc) if want_scores else (idx, cnt)


def _keys(cfg, scores, seq_lens, b, r, sink, window):
    return SM.row_keys(scores[b, r].float().numpy(), int(seq_lens[b]), cfg.index_base, cfg.N_max,
                       sink, window)


def topk_digest(cfg, scores, seq_lens, k, shards, Q=64, sink=0, window=0, digest=None, ws=None):
    d = torch.zeros((cfg.B, cfg.H_sel, Q, 2), dtype=torch.int64)
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            d[b, r] = torch.tensor(SM.digest(_keys(cfg, scores, seq_lens, b, r, sink, window), k, shards, Q))
    return d


def topk_bracket(cfg, all_digests, k, state=None):
    st = torch.zeros((cfg.B, cfg.H_sel, 8), dtype=torch.int64)
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            digs = [[tuple(int(x) for x in p) for p in all_digests[s, b, r].tolist()]
                    for s in range(all_digests.shape[0])]
            st[b, r] = torch.tensor(SM.state_to_words(SM.bracket(digs, k)))
    if state is not None:
        state.copy_(st)
        return state
    return st


def topk_window(cfg, scores, seq_lens, state, sink=0, window=0, msg=None, ws=None):
    m = torch.zeros((cfg.B, cfg.H_sel, 8 + SM.CAP), dtype=torch.int64)
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            st = SM.words_to_state(state[b, r].tolist())
            m[b, r] = torch.tensor(SM.msg_to_words(SM.window(_keys(cfg, scores, seq_lens, b, r, sink, window), st)))
    return m


def topk_resolve(cfg, all_msgs, rank, state):
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            msgs = [SM.words_to_msg(all_msgs[s, b, r].tolist()) for s in range(all_msgs.shape[0])]
            st = SM.resolve(msgs, rank, SM.words_to_state(state[b, r].tolist()))
            state[b, r] = torch.tensor(SM.state_to_words(st))
    return state


def topk_emit(cfg, scores, seq_lens, k, state, sink=0, window=0, idx=None, cnt=None, sel_scores=None,
              ws=None):
    for b in range(cfg.B):
        for r in range(cfg.H_sel):
            sel = SM.emit(_keys(cfg, scores, seq_lens, b, r, sink, window), SM.words_to_state(state[b, r].tolist()))
            idx[b, r] = -1
            if sel is None:
                cnt[b, r] = -1
                continue
            idx[b, r, :len(sel)] = torch.tensor(sel, dtype=torch.int32)
            cnt[b, r] = len(sel)
    return idx, cnt


def sparse_decode(cfg, q, K, V, idx, cnt, k, out=None, lse=None, partial=None, ws=None,
                  want_out=True):
    qd, Kd, Vd = _w(q), _w(K), _w(V)
    G = cfg.H_q // cfg.H_kv
    for b in range(cfg.B):
        for h in range(cfg.H_q):
            r = h // G if cfg.group_mode == O.GROUP_KV_SHARED else h
            S = idx[b, r, :int(cnt[b, r])].numpy().astype(np.int64)
            y, l = O.sparse_attention(qd[b, h], Kd[b, h // G], Vd[b, h // G], S, cfg.scale)
            # (m, l, o) = (lse, 1, y) is a valid partial state; empty -> (-inf, 0, 0)
            partial[b, h, 0] = l
            partial[b, h, 1] = 0.0 if np.isneginf(l) else 1.0
            partial[b, h, 2:] = torch.from_numpy(y)
    return None, None


def lse_combine(cfg, partials, out=None, lse=None):
    G = partials.shape[0]
    out = torch.empty((cfg.B, cfg.H_q, cfg.d), dtype=torch.float64)
    lse = torch.empty((cfg.B, cfg.H_q), dtype=torch.float64)
    for b in range(cfg.B):
        for h in range(cfg.H_q):
            parts = []
            for s in range(G):
                m, l, o = partials[s, b, h, 0].item(), partials[s, b, h, 1].item(), partials[s, b, h, 2:].numpy()
                parts.append((o / l if l > 0 else np.zeros_like(o), m + np.log(l) if l > 0 else -np.inf))
            y, ls = O.lse_combine(parts)
            out[b, h] = torch.from_numpy(np.asarray(y, dtype=np.float64))
            lse[b, h] = ls
    return out, lse
