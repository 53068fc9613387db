"""Phase timing of topk_cluster_kernel from in-kernel clock64 stamps.

    python tools/trace_topk.py [--batch 1 4 16] [--ctx 32768] [--sparsity 10]

Builds a -DSK_TRACE copy of the library (build/trace/libsocket_trace.so; the
product library is untouched), runs score + top-k on the bench workload and
prints, per phase, the median / max over CTAs of the cycles spent (stamp i+1 -
stamp i of the same CTA).  Stamps: see TK_TRACE(i) in csrc/topk.cu.
"""
import argparse
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_06283_b200 import build as B  # noqa: E402

PHASES = ["pdl_wait", "load", "stat_sync", "hist", "hist_sync", "ghist_scan", "cand", "cand_sync",
          "gather_select", "count", "count_sync", "emit", "tail", "final_sync"]


def build_trace():
    out = os.path.join(ROOT, "build", "trace")
    os.makedirs(out, exist_ok=True)
    objs = []
    for s in B._sources():
        o = os.path.join(out, os.path.basename(s)[:-3] + ".o")
        cmd = [B.nvcc()] + B.ARCH + B.NVCC_FLAGS + ["-DSK_TRACE", "-c", s, "-o", o]
        subprocess.run(cmd, check=True)
        objs.append(o)
    lib = os.path.join(out, "libsocket_trace.so")
    subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-o", lib] + objs + ["-lcudart"], check=True)
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1, 4, 16])
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--sparsity", type=float, default=10.0)
    ap.add_argument("--hard", action="store_true")
    a = ap.parse_args()
    libpath = build_trace()
    from paper_2602_06283_b200 import _lib
    _lib.LIB_PATH = libpath
    L = _lib.lib()
    L.socket_debug_topk_trace.restype = ctypes.c_int
    import datagen
    from paper_2602_06283_b200 import Config, SocketDecoder, ops
    for bsz in a.batch:
        N = a.ctx
        k = int(round(N / a.sparsity))
        q, K, V = datagen.torch_make_cache(bsz, 32, 8, N, 128, seed=1)
        W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
        cfg = Config(B=bsz, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5, scoring=int(a.hard))
        lens = torch.full((bsz,), N, dtype=torch.int32, device="cuda")
        dec = SocketDecoder(cfg, W, K, V, k=k)
        dec.prefill()
        dec.step(q, lens)
        for _ in range(3):
            ops.topk(cfg, dec.scores, lens, k, idx=dec.idx, cnt=dec.cnt)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops.topk(cfg, dec.scores, lens, k, idx=dec.idx, cnt=dec.cnt)
        e1.record()
        torch.cuda.synchronize()
        buf = (ctypes.c_ulonglong * (4096 * 16))()
        assert L.socket_debug_topk_trace(buf, 4096 * 16) == 0
        t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16).astype(np.int64)
        n_cta = cfg.B * 8 * 1
        valid = t[:, 0] != 0
        t = t[valid]
        print(f"B={bsz} N={N} k={k}: {t.shape[0]} CTAs, event time {e0.elapsed_time(e1) * 1e3:.1f} us, "
              f"total cycles median {np.median(t[:, 14] - t[:, 0]):.0f} max {np.max(t[:, 14] - t[:, 0]):.0f}")
        stamps = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14]
        for i in range(len(stamps) - 1):
            d = t[:, stamps[i + 1]] - t[:, stamps[i]]
            d = d[(t[:, stamps[i + 1]] != 0) & (t[:, stamps[i]] != 0)]
            if d.size:
                print(f"   {PHASES[i]:14s} median {np.median(d):8.0f}  max {np.max(d):8.0f} cycles")
        del dec, q, K, V
        torch.cuda.empty_cache()
        _ = n_cta


if __name__ == "__main__":
    main()
