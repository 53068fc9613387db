"""Where the host-I/O step's time goes (B = 16 bench workload):
device graph vs host graph (H2D copy + graph, output written to pinned host)
vs its parts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
from paper_2602_06283_b200 import Config, SocketDecoder  # noqa: E402

B, N = int(sys.argv[1]) if len(sys.argv) > 1 else 16, 32768
_st = torch.cuda.Stream()
torch.cuda.set_stream(_st)      # a non-default stream, as in bench.py
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N)
dec = SocketDecoder(cfg, W, K, V, k=3277)
dec.prefill()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, n=30):
    for _ in range(5):
        flush.zero_()
        fn()
    torch.cuda.synchronize()
    tot = 0
    for _ in range(n):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / n * 1e3


dec.capture(q, lens, append=True)
print(f"device graph (append, out on device)    {timeit(dec.replay):7.1f} us")
k_row, v_row = K[:, :, N - 1].cpu(), V[:, :, N - 1].cpu()
qh, kh, vh, oh = dec.bind_host(lens)
qh.copy_(q.cpu())                # real inputs (zeros would make every score tie)
kh.copy_(k_row)
vh.copy_(v_row)
dec._in_d.copy_(dec._in_h)
print(f"host_step (H2D + graph, out -> host)    {timeit(dec.host_step):7.1f} us")
print(f"graph only (out -> host)                {timeit(dec.graph_host.replay):7.1f} us")
print(f"H2D copy only ({dec._in_h.numel() * 2 // 1024} KB)                 "
      f"{timeit(lambda: dec._in_d.copy_(dec._in_h, non_blocking=True)):7.1f} us")
