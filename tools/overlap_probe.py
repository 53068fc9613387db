"""Does splitting the batch into G concurrent step chains (one graph, G forked
streams) hide the latency-bound stages (prologue, top-k) of one chain behind the
HBM-bound stages (score, decode) of another?

    python tools/overlap_probe.py [--batch 16] [--ctx 32768] [--sparsity 10] [--chains 1,2,4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--sparsity", type=float, default=10.0)
ap.add_argument("--chains", default="1,2,4,8")
ap.add_argument("--reps", type=int, default=30)
a = ap.parse_args()
B, N = a.batch, a.ctx
k = int(round(N / a.sparsity))
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
cur = torch.cuda.current_stream()


def build(G, stagger):
    bs = B // G
    decs = []
    for g in range(G):
        cfg = Config(B=bs, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5, flags=1)
        d = SocketDecoder(cfg, W, K[g * bs:(g + 1) * bs], V[g * bs:(g + 1) * bs], k=k)
        d.prefill()
        decs.append((d, q[g * bs:(g + 1) * bs].contiguous(), lens[g * bs:(g + 1) * bs].contiguous()))
    streams = [torch.cuda.Stream() for _ in range(G)]
    for d, qq, ll in decs:                      # warm-up outside the graph
        d.step(qq, ll, append=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cap):
        ev0 = torch.cuda.Event()
        ev0.record(cap)
        prev = ev0
        for (d, qq, ll), s in zip(decs, streams):
            s.wait_event(prev if stagger else ev0)
            with torch.cuda.stream(s):
                d.step(qq, ll, append=True)
            if stagger:
                e = torch.cuda.Event()
                e.record(s)
                prev = e
        for s in streams:
            cap.wait_stream(s)
    return g, decs


def timeit(g):
    ts = []
    for i in range(a.reps + 3):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2] * 1e3


res = {}
for G in [int(x) for x in a.chains.split(",")]:
    if B % G:
        continue
    g, decs = build(G, False)
    res[f"G{G}"] = timeit(g)
    print(f"chains={G} (B/chain={B // G}) concurrent: {res[f'G{G}']:.1f} us", flush=True)
    del g, decs
    torch.cuda.empty_cache()
print(res)
