"""Small-batch step timing: the one-launch cluster kernel vs the multi-kernel
path (socket_cfg.flags = SOCKET_FLAG_CHAINED_STEP), CUDA-graph replay, L2 flushed before each step.

    python tools/fused_check.py [--batch 1 2] [--ctx 32768] [--sparsity 10 5]
"""
import argparse
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder, ops  # noqa: E402
from paper_2602_06283_b200 import _lib  # noqa: E402


def timed(fn, flush, reps=20):
    for _ in range(3):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--ctx", type=int, nargs="+", default=[32768])
    ap.add_argument("--sparsity", type=float, nargs="+", default=[10, 5])
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for N in a.ctx:
        for B in a.batch:
            q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=3)
            W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
            lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
            cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5)
            for sp in a.sparsity:
                k = int(round(N / sp))
                res = {"ctx": N, "batch": B, "sparsity": sp, "k": k}
                outs = {}
                for mode in ("fused", "multi"):
                    cm = dataclasses.replace(cfg, flags=_lib.FLAG_CHAINED_STEP if mode == "multi" else 0)
                    dec = SocketDecoder(cm, W, K, V, k=k)
                    dec.prefill()
                    dec.capture(q, lens, append=True)
                    res[mode + "_us"] = round(timed(dec.replay, flush), 2)
                    dec.replay()
                    torch.cuda.synchronize()
                    outs[mode] = (dec.out.float().clone(), dec.idx.clone(), dec.scores.clone())
                    del dec
                res["same_idx"] = bool(torch.equal(outs["fused"][1], outs["multi"][1]))
                res["same_scores"] = bool(torch.equal(outs["fused"][2], outs["multi"][2]))
                res["max_out_diff"] = float((outs["fused"][0] - outs["multi"][0]).abs().max())
                ws = ops.workspace(cfg, _lib.OP_DENSE_DECODE, 1, q.device)
                res["dense_ours_us"] = round(timed(lambda: ops.dense_decode(cfg, q, K, V, lens, ws=ws), flush), 2)
                qq = q.view(B, 32, 1, 128)
                res["dense_sdpa_us"] = round(timed(lambda: torch.nn.functional.scaled_dot_product_attention(
                    qq, K, V, scale=cfg.scale, enable_gqa=True), flush), 2)
                print(json.dumps(res), flush=True)
            del q, K, V
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
