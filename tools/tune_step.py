"""Small-batch tuning sweep: fused step / top-k / sparse decode times under
different cluster-size and split targets (env knobs read at launch time).

    python tools/tune_step.py [--batch 1 4 16] [--sparsity 5 10]

Every time is a CUDA-graph replay (no host launch overhead); the step is
timed with the L2 flushed before each replay, the single kernels as 10
back-to-back launches inside one graph.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder, ops  # noqa: E402


def graph_of(fn, n):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    return g


def time_graph(g, flush, reps, per):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps / per * 1e3   # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 4, 16])
    ap.add_argument("--sparsity", type=float, nargs="+", default=[5, 10])
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--topk-ctas", type=int, nargs="+", default=[148, 64, 32])
    ap.add_argument("--decode-target", type=int, nargs="+", default=[592, 296, 148])
    a = ap.parse_args()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    N = a.ctx
    for bsz in a.batch:
        q, K, V = datagen.torch_make_cache(bsz, 32, 8, N, 128, seed=1)
        W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
        lens = torch.full((bsz,), N, dtype=torch.int32, device="cuda")
        cfg = Config(B=bsz, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5)
        for sp in a.sparsity:
            k = int(round(N / sp))
            res = {"batch": bsz, "sparsity": sp, "k": k, "topk_us": {}, "decode_us": {}, "step_us": {}}
            dec = SocketDecoder(cfg, W, K, V, k=k)
            dec.prefill()
            dec.step(q, lens, append=True)
            torch.cuda.synchronize()
            for tc in a.topk_ctas:
                os.environ["SOCKET_TOPK_MIN_CTAS"] = str(tc)
                g = graph_of(lambda: ops.topk(cfg, dec.scores, lens, k, idx=dec.idx, cnt=dec.cnt), 10)
                res["topk_us"][tc] = round(time_graph(g, None, 10, 10), 2)
            os.environ.pop("SOCKET_TOPK_MIN_CTAS")
            for dt in a.decode_target:
                os.environ["SOCKET_DECODE_TARGET"] = str(dt)
                ws = ops.workspace(cfg, 4, k, q.device)
                g = graph_of(lambda: ops.sparse_decode(cfg, q, K, V, dec.idx, dec.cnt, k, out=dec.out,
                                                       lse=dec.lse, ws=ws), 10)
                res["decode_us"][dt] = round(time_graph(g, flush, 10, 10), 2)
            os.environ.pop("SOCKET_DECODE_TARGET")
            for tc in a.topk_ctas:
                for dt in a.decode_target:
                    os.environ["SOCKET_TOPK_MIN_CTAS"] = str(tc)
                    os.environ["SOCKET_DECODE_TARGET"] = str(dt)
                    d2 = SocketDecoder(cfg, W, K, V, k=k)
                    d2.codes, d2.vnorm = dec.codes, dec.vnorm
                    d2.capture(q, lens, append=True)
                    res["step_us"][f"{tc}/{dt}"] = round(time_graph(d2.graph, flush, 20, 1), 2)
                    del d2
            os.environ.pop("SOCKET_TOPK_MIN_CTAS")
            os.environ.pop("SOCKET_DECODE_TARGET")
            print(json.dumps(res), flush=True)
            del dec
        del q, K, V
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
