"""BASELINE configs[4] sweep and the 128K point of configs[2] on one B200.

    python tools/sweep.py [--out gpurun_out/sweep.json]

For each (ctx, batch, L, P, sparsity) point: the fused SOCKET decode step
(CUDA graph replay, L2 flushed before each step) vs our dense split-KV decode
and torch SDPA on the same cache; reports tokens/s, speedup and the score and
decode kernels' HBM fractions (back-to-back launches).  Bits/token = L * P.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, KV_SHARED, PER_QHEAD, SocketDecoder, ops  # noqa: E402
from paper_2602_06283_b200 import _lib  # noqa: E402

HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def timed(fn, flush, reps=10, inner=1):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1) / inner
    return tot / reps


def point(ctx, batch, L, P, sparsity, flush, cache, mode=None, H_q=32, H_kv=8):
    k = int(round(ctx / sparsity))
    key = (ctx, batch, H_q, H_kv)
    if key not in cache:
        cache.clear()
        torch.cuda.empty_cache()
        cache[key] = datagen.torch_make_cache(batch, H_q, H_kv, ctx, 128, seed=5)
    q, K, V = cache[key]
    W = torch.from_numpy(datagen.make_projections(4242, L, P, 128).view("int16")).cuda().view(torch.bfloat16)
    cfg = Config(B=batch, H_q=H_q, H_kv=H_kv, N_max=ctx, L=L, P=P, tau=0.5,
                 group_mode=KV_SHARED if mode is None else mode)
    lens = torch.full((batch,), ctx, dtype=torch.int32, device="cuda")
    dec = SocketDecoder(cfg, W, K, V, k=k)
    dec.prefill()
    if dec.fused:
        dec.capture(q, lens, append=True)
        t_step = timed(dec.replay, flush)
    else:                                   # P > 8: stage by stage (eager)
        t_step = timed(lambda: dec.step(q, lens, append=True), flush)
    lut = ops.build_lut(cfg, q, W)
    t_score = timed(lambda: ops.score_lut(cfg, lut, dec.codes, dec.vnorm, lens, out=dec.scores), flush, 5, 10)
    ops.topk(cfg, dec.scores, lens, k, idx=dec.idx, cnt=dec.cnt)
    t_dec = timed(lambda: ops.sparse_decode(cfg, q, K, V, dec.idx, dec.cnt, k, out=dec.out, lse=dec.lse,
                                            ws=dec.ws_dec), flush, 5, 10)
    ws = ops.workspace(cfg, _lib.OP_DENSE_DECODE, 1, q.device)
    t_dense = timed(lambda: ops.dense_decode(cfg, q, K, V, lens, ws=ws), flush)
    qq = q.view(batch, H_q, 1, 128)
    t_sdpa = timed(lambda: torch.nn.functional.scaled_dot_product_attention(qq, K, V, scale=cfg.scale,
                                                                             enable_gqa=True), flush)
    code_bytes = ops.codes_bytes(cfg) // (batch * H_kv * ctx)      # stored bytes per key (packed for P > 8)
    score_bytes = batch * H_kv * ctx * (code_bytes + 4) + batch * cfg.H_sel * ctx * 4
    dec_bytes = batch * cfg.H_sel * k * 516 + batch * H_q * 512
    best_dense = min(t_dense, t_sdpa)
    return {
        "ctx": ctx, "batch": batch, "H_q": H_q, "H_kv": H_kv,
        "selection": "per_qhead" if cfg.group_mode == PER_QHEAD else "kv_shared",
        "launches": ops.decode_step_launches(cfg), "L": L, "P": P, "bits_per_token": L * P,
        "stored_bits_per_token": code_bytes * 8, "sparsity": sparsity, "k": k,
        "step_ms": round(t_step, 4), "tokens_per_s": round(batch / (t_step * 1e-3), 1),
        "dense_ms": round(best_dense, 4), "dense_impl": "ours" if t_dense <= t_sdpa else "torch_sdpa",
        "speedup_vs_dense": round(best_dense / t_step, 3),
        "score_ms": round(t_score, 4), "score_frac": round(score_bytes / (t_score * 1e-3) / 1e9 / HBM, 3),
        "decode_ms": round(t_dec, 4), "decode_frac": round(dec_bytes / (t_dec * 1e-3) / 1e9 / HBM, 3),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.json")
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    pts = []
    cache = {}
    # configs[0]: single head, n = 4096, L = 16, P = 8, k = 512 (latency)
    pts.append(point(4096, 1, 16, 8, 8, flush, cache, H_q=1, H_kv=1))
    print(json.dumps(pts[-1]), flush=True)
    # configs[4]: 64K context (B = 4), L x bits and sparsity sweep (bits/token 64..1024)
    for (L, P) in [(16, 8), (32, 8), (60, 8), (64, 8), (8, 8), (60, 10)]:
        for s in ([5, 10, 20, 33, 50] if L == 60 and P == 8 else [10, 33]):
            pts.append(point(65536, 4, L, P, s, flush, cache))
            print(json.dumps(pts[-1]), flush=True)
    # 768 and 1024 bits/token (P = 12, 16): factored half-table lookups (DESIGN 4.6),
    # both selection modes (KV_SHARED sums G = 4 heads per lookup; PER_QHEAD reads
    # each code once per query head)
    for (P, mode) in [(12, KV_SHARED), (16, KV_SHARED), (16, PER_QHEAD)]:
        for s in (10, 33):
            pts.append(point(65536, 4, 64, P, s, flush, cache, mode=mode))
            print(json.dumps(pts[-1]), flush=True)
    # configs[2] per-GPU shard on one GPU: 128K context, B = 8, all 8 KV heads (G = 1)
    for s in (5, 10, 33):
        pts.append(point(131072, 8, 60, 8, s, flush, cache))
        print(json.dumps(pts[-1]), flush=True)
    # configs[1] batch sweep at 32K
    for bsz in (1, 4):
        for s in (5, 10):
            pts.append(point(32768, bsz, 60, 8, s, flush, cache))
            print(json.dumps(pts[-1]), flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    json.dump(pts, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
