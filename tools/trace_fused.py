"""Phase timing of the fused small-batch step kernel (FU_STAMP in csrc/fused.cu).

    python tools/trace_fused.py [--batch 1] [--ctx 32768] [--sparsity 10]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from trace_topk import build_trace  # noqa: E402

PH = ["stage q/W", "DMMA+sigma+half+append", "LUT to cluster", "cluster sync", "score slice",
      "top-k", "attend + merge"]
TK = ["stat_sync", "hist", "hist_sync", "ghist_scan", "cand", "cand_sync", "gather_select", "count",
      "emit", "tail", "final_sync"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--sparsity", type=float, default=10)
    a = ap.parse_args()
    libpath = build_trace()
    from paper_2602_06283_b200 import _lib
    _lib.LIB_PATH = libpath
    L = _lib.lib()
    import datagen
    from paper_2602_06283_b200 import Config, SocketDecoder
    B, N = a.batch, a.ctx
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
    W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5)
    lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
    dec = SocketDecoder(cfg, W, K, V, k=int(N / a.sparsity))
    dec.prefill()
    for _ in range(3):
        dec.step(q, lens, append=True)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (4096 * 8))()
    assert L.socket_debug_fused_trace(buf, 4096 * 8) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 8).astype(np.int64)
    t = t[t[:, 0] != 0]
    print(f"B={B} N={N}: {len(t)} CTAs, total cycles median {np.median(t[:, 7] - t[:, 0]):.0f} "
          f"max {np.max(t[:, 7] - t[:, 0]):.0f}")
    for i in range(7):
        d = t[:, i + 1] - t[:, i]
        print(f"   {PH[i]:24s} median {np.median(d):8.0f}  max {np.max(d):8.0f} cycles")
    # top-k sub-phases (TK_TRACE stamps 2..13 of topk_core; 0/1 are not stamped here)
    tb = (ctypes.c_ulonglong * (4096 * 16))()
    if L.socket_debug_fused_topk_trace(tb, 4096 * 16) == 0:
        u = np.frombuffer(tb, dtype=np.uint64).reshape(4096, 16).astype(np.int64)
        u = u[u[:, 2] != 0]
        for i in range(2, 13):
            ok = (u[:, i + 1] != 0) & (u[:, i] != 0)
            if ok.any():
                d = u[ok, i + 1] - u[ok, i]
                print(f"     topk {TK[i - 2]:14s} median {np.median(d):8.0f}  max {np.max(d):8.0f} cycles")


if __name__ == "__main__":
    main()
