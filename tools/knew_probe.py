import sys, os, torch
sys.path.insert(0, os.getcwd())
import datagen
from paper_2602_06283_b200 import Config, SocketDecoder
B, N = 16, 32768
q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=1)
W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
cfg = Config(B=B, H_q=32, H_kv=8, N_max=N)
dec = SocketDecoder(cfg, W, K, V, k=3277); dec.prefill()
kd = K[:, :, N - 1].contiguous(); vd = V[:, :, N - 1].contiguous()
torch.cuda.synchronize()
dec.step(q, lens, append=True)
torch.cuda.synchronize()
dec.step(q, lens, append=True, k_new=kd, v_new=vd)
torch.cuda.synchronize()
