import sys, json, dataclasses
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch, datagen
from paper_2602_06283_b200 import Config, SocketDecoder, _lib, ops
from spread_check import timed
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for (B, Hq, Hkv, N) in [(16, 4, 1, 32768), (16, 8, 2, 32768), (16, 16, 4, 32768), (8, 4, 1, 131072)]:
    k = N // 10
    q, K, V = datagen.torch_make_cache(B, Hq, Hkv, N, 128, seed=2)
    W = torch.from_numpy(datagen.make_projections(4242, 60, 8, 128).view("int16")).cuda().view(torch.bfloat16)
    lens = torch.full((B,), N, dtype=torch.int32, device="cuda")
    res = {}
    outs = {}
    for name, fl in (("default", 0), ("chained", 1)):
        cfg = Config(B=B, H_q=Hq, H_kv=Hkv, N_max=N, L=60, P=8, flags=fl)
        dec = SocketDecoder(cfg, W, K.clone(), V.clone(), k=k)
        dec.prefill()
        dec.capture(q, lens, append=True)
        res[name + "_us"] = round(timed(dec.replay, flush), 2)
        res[name + "_launches"] = ops.decode_step_launches(cfg)
        dec.replay(); torch.cuda.synchronize()
        outs[name] = (dec.idx.clone(), dec.out.float().clone())
    res["same_idx"] = bool(torch.equal(outs["default"][0], outs["chained"][0]))
    res["out_diff"] = float((outs["default"][1] - outs["chained"][1]).abs().max())
    print(json.dumps({"B": B, "H_q": Hq, "H_kv": Hkv, "N": N, **res}), flush=True)
