"""Host model of the sequence-shard top-k protocol (include/socket_b200.h:
socket_topk_digest / _bracket / _window / _resolve / _emit), written from
DESIGN.md "Multi-GPU" in plain Python integers.  TEST INFRASTRUCTURE ONLY:

  * the CPU (gloo) tests run dist.py's orchestration with this model as the
    local provider (tests/oracle_ops.py), so the protocol's exactness -- the
    union of the shards' emits equals the oracle's single-device top-k -- is
    checked at world sizes 2 and 4 with heavy ties, on CPU;
  * the GPU tests compare the CUDA kernels' digests, states and emits with
    this model on the same fp32 scores (bit-exact; message keys as a multiset).

It shares no code with the CUDA path.  Keys are the monotone u32 image of the
fp32 scores (larger score <=> larger key), 0 = invalid (-inf), 0xFFFFFFFF =
forced sink / local-window key.
"""
import numpy as np

BINS = 2048
CAP = 2048
FULL = 0xFFFFFFFF


def row_keys(scores_row, n_glob, index_base, N_max, sink=0, window=0):
    """Keys of the local valid prefix of one row (python ints)."""
    n = max(0, min(int(n_glob) - int(index_base), N_max))
    s = np.ascontiguousarray(scores_row[:n], dtype=np.float32)
    u = s.view(np.uint32).astype(np.uint64)
    k = np.where(u & 0x80000000, (~u) & 0xFFFFFFFF, u | 0x80000000)
    out = []
    for j in range(n):
        if s[j] == -np.inf:
            out.append(0)
            continue
        pos = index_base + j
        if pos < sink or pos >= n_glob - window:
            out.append(FULL)
        else:
            out.append(int(k[j]))
    return out


def digest(keys, k, shards, Q):
    tvalid = sum(1 for x in keys if x != 0)
    tforced = sum(1 for x in keys if x == FULL)
    reg = [x for x in keys if x != 0 and x != FULL]
    pairs = [(0, 0)] * Q
    pairs[0] = (1, tvalid)
    pairs[1] = (FULL, tforced)
    if reg:
        gmin, gmax = min(reg), max(reg)
        span = gmax - gmin
        sh = 0 if span < BINS else span.bit_length() - 11
        pairs[2] = ((gmax + 1) & FULL, tforced)
        hist = [0] * BINS
        for x in reg:
            hist[(x - gmin) >> sh] += 1
        suff = [0] * (BINS + 1)
        suff[BINS] = tforced
        for b in range(BINS - 1, -1, -1):
            suff[b] = suff[b + 1] + hist[b]
        k_loc = min(k, tvalid)
        nt = Q - 3
        m1 = max(1, nt * 3 // 4)
        m2 = nt - m1
        R1 = min(k_loc, 2 * ((k + shards - 1) // shards))
        if k_loc > tforced:
            for t_i in range(nt):
                if t_i < m1:
                    t = ((t_i + 1) * R1 + m1 - 1) // m1
                else:
                    t = R1 + ((t_i - m1 + 1) * (k_loc - R1) + m2 - 1) // max(m2, 1)
                t = max(t, 1)
                if t > tforced:
                    lo = max(b for b in range(BINS) if suff[b] >= t)
                    pairs[3 + t_i] = (gmin + (lo << sh), suff[lo])
    return pairs


def bracket(digests, k):
    """digests: list over shards of pair lists.  Returns the initial state dict."""
    valid = sum(d[0][1] for d in digests)
    k_eff = min(k, valid)
    if k_eff == 0:
        return dict(lo=1, hi=0, k_eff=0, resolved=1, T=FULL, quota=0, need=0, gt=0)
    lo_best, hi_best = 0, 1 << 32
    for d in digests:
        for (x, _) in d:
            if x == 0:
                continue
            Ls = Us = 0
            for ds in digests:
                lower = max([c for (e, c) in ds if e != 0 and e >= x], default=0)
                upper = min([c for (e, c) in ds if e != 0 and e <= x], default=FULL)
                Ls += lower
                Us += upper
            if Ls >= k_eff:
                lo_best = max(lo_best, x)
            if Us + 1 <= k_eff:
                hi_best = min(hi_best, x)
    return dict(lo=lo_best, hi=0 if hi_best == 1 << 32 else hi_best, k_eff=k_eff, resolved=0,
                T=0, quota=0, need=0, gt=0)


def _hi(st):
    return (1 << 32) if st["hi"] == 0 else st["hi"]


def _shift(lo, hi):
    sh = 0
    while ((hi - lo - 1) >> sh) >= CAP:
        sh += 1
    return sh


def window(keys, st):
    """Message dict: above, wc, mode (0 keys / 1 hist), sh, payload."""
    lo, hi = st["lo"], _hi(st)
    if st["resolved"]:
        return dict(lo=lo, hi=st["hi"], above=0, wc=0, mode=0, sh=0, payload=[])
    above = sum(1 for x in keys if x != 0 and x >= hi)
    win = [x for x in keys if x != 0 and lo <= x < hi]
    if len(win) <= CAP:
        return dict(lo=lo, hi=st["hi"], above=above, wc=len(win), mode=0, sh=0, payload=sorted(win))
    sh = _shift(lo, hi)
    h = [0] * CAP
    for x in win:
        h[(x - lo) >> sh] += 1
    return dict(lo=lo, hi=st["hi"], above=above, wc=len(win), mode=1, sh=sh, payload=h)


def resolve(msgs, rank, st):
    """msgs: list over shards.  Returns the new state (a copy)."""
    st = dict(st)
    if st["resolved"]:
        return st
    lo, hi = st["lo"], _hi(st)
    need = st["k_eff"] - sum(m["above"] for m in msgs)
    sh = _shift(lo, hi)
    G = len(msgs)
    gt, eq = [0] * G, [0] * G
    if all(m["mode"] == 0 for m in msgs):
        union = sorted((x for m in msgs for x in m["payload"]), reverse=True)
        T = union[need - 1]
        for s, m in enumerate(msgs):
            gt[s] = sum(1 for x in m["payload"] if x > T)
            eq[s] = sum(1 for x in m["payload"] if x == T)
    else:
        H = [[0] * CAP for _ in range(G)]
        for s, m in enumerate(msgs):
            if m["mode"] == 1:
                H[s] = list(m["payload"])
            else:
                for x in m["payload"]:
                    H[s][(x - lo) >> sh] += 1
        tot = [sum(H[s][b] for s in range(G)) for b in range(CAP)]
        run, bstar = 0, None
        for b in range(CAP - 1, -1, -1):
            if run < need <= run + tot[b]:
                bstar = b
                break
            run += tot[b]
        if sh != 0:
            nlo = lo + (bstar << sh)
            nhi = min(hi, nlo + (1 << sh))
            st["lo"], st["hi"] = nlo, (0 if nhi == 1 << 32 else nhi)
            return st
        T = lo + bstar
        for s in range(G):
            gt[s] = sum(H[s][b] for b in range(bstar + 1, CAP))
            eq[s] = H[s][bstar]
    gt_tot = sum(m["above"] for m in msgs) + sum(gt)
    ties = st["k_eff"] - gt_tot
    before = sum(eq[:rank])
    q = min(ties - before, eq[rank]) if ties > before else 0
    st.update(resolved=1, T=T, quota=q, need=need, gt=msgs[rank]["above"] + gt[rank])
    return st


def emit(keys, st):
    """Local indices (ascending) of this shard's share; None if unresolved."""
    if not st["resolved"]:
        return None
    T, q = st["T"], st["quota"]
    out, taken = [], 0
    for j, x in enumerate(keys):
        if x != 0 and x > T:
            out.append(j)
        elif x != 0 and x == T and taken < q:
            out.append(j)
            taken += 1
    return out


# ---- tensor encodings (the library's buffer formats) -------------------------
def state_to_words(st):
    return [st["lo"], st["hi"], st["k_eff"], st["resolved"], st["T"], st["quota"], st["need"], st["gt"]]


def words_to_state(w):
    w = [int(x) & FULL for x in w]
    return dict(lo=w[0], hi=w[1], k_eff=w[2], resolved=w[3], T=w[4], quota=w[5], need=w[6], gt=w[7])


def msg_to_words(m):
    w = [m["lo"], m["hi"], m["above"], m["wc"], m["mode"], m["sh"], 0, 0] + list(m["payload"])
    return w + [0] * (8 + CAP - len(w))


def words_to_msg(w):
    w = [int(x) & FULL for x in w]
    mode = w[4]
    payload = w[8:8 + CAP] if mode == 1 else w[8:8 + w[3]]
    return dict(lo=w[0], hi=w[1], above=w[2], wc=w[3], mode=mode, sh=w[5], payload=payload)
