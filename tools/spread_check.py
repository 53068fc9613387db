"""One-launch row-spread step vs the chained kernels:
selection / scores / codes identical, outputs close, and graph-replayed step
times (L2 flushed before every replay).

    python tools/spread_check.py [--batch 1 2 4] [--ctx 32768 65536] [--sparsity 10 5 33]
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
from paper_2602_06283_b200 import Config, SocketDecoder, _lib  # noqa: E402

MODES = {"spread": _lib.FLAG_ONE_LAUNCH, "chained": _lib.FLAG_CHAINED_STEP}


def timed(fn, flush, reps=60):
    """Mean of reps CUDA-event timings (events tick in ~2 us quanta on this part:
    the mean resolves below a quantum, the median does not)."""
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return sum(ts) / len(ts) * 1e3


def run(B, N, sp, flush, modes, ragged=False, sink=0, window=0, hard=False, time_it=True):
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=3)
    W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
    lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
    if ragged:
        g = torch.Generator().manual_seed(B * 7 + N)
        lens = torch.randint(N // 3, N + 1, (B,), generator=g, dtype=torch.int32).cuda()
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5, scoring=int(hard))
    k = int(round(N / sp))
    res = {"B": B, "N": N, "sparsity": sp, "k": k, "ragged": ragged, "sink": sink, "window": window,
           "hard": hard}
    outs = {}
    for mode in modes:
        cm = dataclasses.replace(cfg, flags=MODES[mode])
        dec = SocketDecoder(cm, W, K.clone(), V.clone(), k=k, sink=sink, window=window)
        dec.prefill()
        dec.capture(q, lens, append=True)
        if time_it:
            res[mode + "_us"] = round(timed(dec.replay, flush), 2)
        dec.replay()
        torch.cuda.synchronize()
        outs[mode] = (dec.out.float().clone(), dec.idx.clone(), dec.scores.clone(), dec.cnt.clone(),
                      dec.lse.clone(), dec.codes.clone(), dec.vnorm.clone())
        del dec
    ref = outs["chained"]
    for mode in modes:
        if mode == "chained":
            continue
        o = outs[mode]
        res[mode + "_same_idx"] = bool(torch.equal(o[1], ref[1]))
        res[mode + "_same_cnt"] = bool(torch.equal(o[3], ref[3]))
        res[mode + "_same_scores"] = bool(torch.equal(o[2], ref[2]))
        res[mode + "_same_codes"] = bool(torch.equal(o[5], ref[5]) and torch.equal(o[6], ref[6]))
        res[mode + "_out_diff"] = float((o[0] - ref[0]).abs().max())
        res[mode + "_lse_diff"] = float((o[4] - ref[4]).abs().max())
    print(json.dumps(res), flush=True)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 2, 4])
    ap.add_argument("--ctx", type=int, nargs="+", default=[32768, 65536, 131072])
    ap.add_argument("--sparsity", type=float, nargs="+", default=[10, 5, 33])
    ap.add_argument("--modes", default="spread,chained")
    ap.add_argument("--edge", action="store_true", help="ragged / sink-window / hard cases first")
    ap.add_argument("--noflush", action="store_true", help="no L2 flush between timed replays")
    ap.add_argument("--lib", default=None, help="an experiment build (tools/variant_build.py)")
    a = ap.parse_args()
    if a.lib:
        _lib.LIB_PATH = a.lib
    flush = torch.empty(256 << 20 if not a.noflush else 16, dtype=torch.uint8, device="cuda")
    modes = a.modes.split(",")
    if a.edge:
        run(1, 4096, 8, flush, ["spread", "chained"], time_it=False)
        run(1, 32768, 10, flush, ["spread", "chained"], ragged=True, time_it=False)
        run(2, 32768, 10, flush, ["spread", "chained"], ragged=True, sink=64, window=128, time_it=False)
        run(1, 32768, 10, flush, ["spread", "chained"], hard=True, time_it=False)
        run(1, 8192, 1.0, flush, ["spread", "chained"], time_it=False)
    for N in a.ctx:
        for B in a.batch:
            for sp in a.sparsity:
                run(B, N, sp, flush, modes)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
