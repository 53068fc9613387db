"""Phase timing of the one-launch row-spread step (SP_STAMP in csrc/spread.cu).

    python tools/trace_spread.py [--batch 1] [--ctx 32768] [--sparsity 10]
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

PH = ["prefetch+tables+norms", "barrier 1", "LUT load + range", "scores + hist", "barrier 2",
      "locate + candidates", "barrier 3", "resolve + offsets", "emit", "attention + merge"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, nargs="+", default=[1])
    ap.add_argument("--ctx", type=int, nargs="+", default=[32768])
    ap.add_argument("--sparsity", type=float, default=10)
    a = ap.parse_args()
    libpath = build_trace()
    from paper_2602_06283_b200 import _lib
    _lib.LIB_PATH = libpath
    L = _lib.lib()
    import datagen
    from paper_2602_06283_b200 import Config, SocketDecoder
    for N in a.ctx:
        for B in a.batch:
            q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
            W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
            cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=60, P=8, tau=0.5, flags=_lib.FLAG_ONE_LAUNCH)
            lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
            dec = SocketDecoder(cfg, W, K, V, k=int(round(N / a.sparsity)))
            dec.prefill()
            flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            dec.capture(q, lens, append=True)
            ev = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dec.replay()
                e1.record()
                torch.cuda.synchronize()
                ev.append(e0.elapsed_time(e1) * 1e3)
            buf = (ctypes.c_ulonglong * (4096 * 32))()
            assert L.socket_debug_spread_trace(buf, 4096 * 32) == 0
            t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 32).astype(np.int64)
            t = t[t[:, 0] != 0]
            gt = t[:, 23]
            ge = t[:, 24]
            print(f"   last replay: CUDA events {ev[-1]:.1f} us, in-kernel span (first CTA start -> last CTA end, "
                  f"globaltimer) {(ge.max() - gt.min()) / 1e3:.1f} us")
            print(f"B={B} N={N}: {len(t)} CTAs, start skew (globaltimer) {(gt.max() - gt.min()) / 1e3:.2f} us; "
                  f"total cycles median {np.median(t[:, 10] - t[:, 0]):.0f} max {np.max(t[:, 10] - t[:, 0]):.0f}")
            ct = t[:, 21]
            print(f"   final-bin candidates per row: median {np.median(ct):.0f} max {ct.max()}")
            for i in range(10):
                ok = (t[:, i + 1] != 0) & (t[:, i] != 0)
                d = t[ok, i + 1] - t[ok, i]
                if len(d):
                    print(f"   {PH[i]:24s} median {np.median(d):8.0f}  min {np.min(d):8.0f}  max {np.max(d):8.0f} cycles")
            for nm, i0, i1 in (("start -> tables staged", 0, 11), ("staged -> dmma+sigma+append", 11, 16),
                               ("-> half tables", 16, 17), ("-> LUT columns", 17, 18), ("LUT columns -> barrier1", 18, 1),
                               ("barrier3 -> cands gathered", 7, 19), ("-> T resolved", 19, 20), ("-> offsets", 20, 8),
                               ("emit -> attention loop done", 9, 12), ("attn done -> partial written", 12, 13),
                               ("partial -> ticket", 13, 14), ("ticket -> end", 14, 10),
                               ("last: ticket -> staged", 14, 22), ("last: staged -> end", 22, 10)):
                ok = (t[:, i0] != 0) & (t[:, i1] != 0)
                d = t[ok, i1] - t[ok, i0]
                if len(d):
                    print(f"     {nm:28s} median {np.median(d):8.0f}  min {np.min(d):8.0f}  max {np.max(d):8.0f}")
            del dec, q, K, V
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
