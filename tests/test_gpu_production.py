"""GPU parity at the production launch configurations (the shapes bench.py
times), sampled rows against the float64 oracle at the north-star tolerances
(scores 1e-5 relative, selection identical except documented near-ties,
outputs 2e-3 absolute, lse 1e-3):

  * the decode step at B = 1 (32 q / 8 kv heads) for 32K, 64K and 128K
    context: the one-launch row-spread kernel (18 CTAs per row, 1824 / 3648 /
    7296-key slices), and at B = 2 (9 CTAs per row, the default one-launch grid);
  * the chained 128K per-GPU step of configs[2] (B = 8, k = 13107 and 26214);
  * the wide-code (P = 10, 600 bits/token) step and score kernel at B = 16, 32K;
  * bind_host() leaves the cache untouched (its warm-up runs without append).
"""
import numpy as np
import pytest
import torch

import datagen
import oracle as O
from helpers import bits_to_dev, rel_err

pytestmark = pytest.mark.gpu

ops = pytest.importorskip("paper_2602_06283_b200.ops")
from paper_2602_06283_b200 import Config, SocketDecoder  # noqa: E402

DEV = "cuda"


def _bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def check_rows(dec, cfg, q, K, V, Wb, N, k, rows, P=8):
    """Sampled (b, kv head) units of a KV_SHARED step against oracle.decode_step.

    Codes: bit-exact except bits whose oracle margin |x| / sum|W_t k_t| < 1e-5
    (fp32 vs float64 sign of a near-zero projection); the
    keys holding such a flip are excluded from the score check (their score
    differs by a table entry) and may differ in the selection.  All other
    scores within 1e-5 relative; the selection identical on the GPU's own fp32
    scores, and against float64 only at near-ties or flipped keys."""
    G = cfg.H_q // cfg.H_kv
    plain = ops.unpack_codes(cfg, dec.codes)
    for (b, g) in rows:
        Kb, Vb = _bits(K[b, g]), _bits(V[b, g])
        qb = _bits(q[b, g * G:(g + 1) * G])
        n = int(dec_lens(dec, b))
        ref = O.decode_step(qb[None], Kb[None, None], Vb[None, None], Wb, np.array([n]), tau=cfg.tau,
                            k=k, sm_scale=cfg.scale)
        got_codes = plain[b, g].long().cpu().numpy() & ((1 << P) - 1)
        ref_codes = ref["codes"][(0, 0)]
        flip_l, flip_j = np.nonzero(got_codes[:, :n] != ref_codes[:, :n])
        flipped = set(flip_j.tolist())
        if flipped:   # every flipped bit must sit on a near-zero projection
            js = np.array(sorted(flipped))
            _, margin = O.hash_keys(O.widen(Kb[js]), O.widen(Wb))
            pos = {j: i for i, j in enumerate(js)}
            for l, j in zip(flip_l, flip_j):
                x = int(got_codes[l, j]) ^ int(ref_codes[l, j])
                for i in range(P):
                    if x >> i & 1:
                        assert margin[l, i, pos[j]] < 1e-5, (l, i, j, margin[l, i, pos[j]])
            print(f"unit {(b, g)}: {len(flip_l)} code(s) flipped at near-zero margins, keys {sorted(flipped)}")
        s_ref = ref["scores"][(0, 0)]
        s_gpu = dec.scores[b, g].cpu().numpy()
        fin = np.isfinite(s_ref)
        assert np.array_equal(np.isfinite(s_gpu), fin)
        ok = fin.copy()
        ok[list(flipped)] = False
        assert np.max(rel_err(s_gpu[ok], s_ref[ok])) <= 1e-5
        S_gpu = dec.idx[b, g, :dec.cnt[b, g]].cpu().numpy()
        S_ref = ref["sel"][(0, 0)]
        assert len(S_gpu) == len(S_ref)
        # same fp32 scores -> identical selection; vs float64 only near-ties / flipped keys differ
        assert np.array_equal(S_gpu, O.topk_select(s_gpu.astype(np.float64), k, n))
        kth = np.sort(s_ref[S_ref])[0]
        kth_gpu = np.sort(s_gpu[S_gpu])[0]
        for j in np.setxor1d(S_gpu, S_ref):
            # a flipped key moves its own score, and (when it crosses) the k-th value too
            assert (abs(s_ref[j] - kth) <= 1e-5 * kth or j in flipped or
                    (flipped and abs(s_ref[j] - kth_gpu) <= 1e-5 * kth_gpu)), j
        qf, Kf, Vf = O.widen(qb), O.widen(Kb), O.widen(Vb)
        for h in range(G):
            y, l = O.sparse_attention(qf[h], Kf, Vf, S_gpu, cfg.scale)
            assert np.max(np.abs(dec.out[b, g * G + h].float().cpu().numpy() - y)) <= 2e-3
            assert abs(float(dec.lse[b, g * G + h]) - l) <= 1e-3


def dec_lens(dec, b):
    return dec._lens[b]


def run(B, N, k, L=60, P=8, flags=0, seed=0, lens=None):
    cfg = Config(B=B, H_q=32, H_kv=8, N_max=N, L=L, P=P, tau=0.5, flags=flags)
    q, K, V = datagen.torch_make_cache(B, 32, 8, N, 128, seed=seed)
    Wb = datagen.make_projections(4242 + P, L, P, 128)
    if lens is None:
        lens = [N] * B
    lt = torch.tensor(lens, dtype=torch.int32, device=DEV)
    dec = SocketDecoder(cfg, bits_to_dev(Wb), K, V, k=k)
    dec._lens = lens
    dec.prefill()
    dec.step(q, lt, append=True)
    torch.cuda.synchronize()
    return dec, cfg, q, K, V, Wb


@pytest.mark.parametrize("N,sparsity", [(32768, 10), (65536, 10), (131072, 33)])
def test_one_launch_step_b1_production(N, sparsity):
    k = int(round(N / sparsity))
    dec, cfg, q, K, V, Wb = run(1, N, k, seed=N, lens=[N - 5])
    # one launch: the row-spread kernel (18 CTAs per row, 1824 .. 7296-key slices)
    assert ops.decode_step_launches(cfg) == 1
    check_rows(dec, cfg, q, K, V, Wb, N, k, [(0, 0), (0, 5), (0, 7)])


@pytest.mark.parametrize("sparsity", [10, 5])
def test_one_launch_step_b2_production(sparsity):
    N = 32768
    k = int(round(N / sparsity))
    dec, cfg, q, K, V, Wb = run(2, N, k, seed=7 + sparsity, lens=[N - 3, N - 2000])
    assert ops.decode_step_launches(cfg) == 1   # 16 selection rows (<= 32): the row-spread kernel
    check_rows(dec, cfg, q, K, V, Wb, N, k, [(0, 1), (1, 6)])


@pytest.mark.parametrize("k", [13107, 26214])
def test_chained_step_128k_configs2(k):
    N = 131072
    dec, cfg, q, K, V, Wb = run(8, N, k, seed=k, lens=[N, N - 1, N - 100, N, N, N, N - 31, N])
    assert ops.decode_step_launches(cfg) == 4
    check_rows(dec, cfg, q, K, V, Wb, N, k, [(0, 0), (2, 3), (7, 7)])


def test_wide_codes_step_b16_32k():
    """P = 10 (uint16 codes, group-summed tables of score_wide2_kernel), bench shape."""
    N, k = 32768, 3277
    dec, cfg, q, K, V, Wb = run(16, N, k, P=10, seed=3)
    check_rows(dec, cfg, q, K, V, Wb, N, k, [(0, 0), (15, 7)], P=10)


def test_bind_host_leaves_cache_untouched():
    N, k = 4096, 400
    cfg = Config(B=2, H_q=32, H_kv=8, N_max=N, L=60, P=8)
    q, K, V = datagen.torch_make_cache(2, 32, 8, N, 128, seed=8)
    W = bits_to_dev(datagen.make_projections(4250, 60, 8, 128))
    lens = torch.full((2,), N, dtype=torch.int32, device=DEV)
    dec = SocketDecoder(cfg, W, K, V, k=k)
    dec.prefill()
    K0, V0, c0, v0 = K.clone(), V.clone(), dec.codes.clone(), dec.vnorm.clone()
    dec.bind_host(lens)
    torch.cuda.synchronize()
    assert torch.equal(K, K0) and torch.equal(V, V0)
    assert torch.equal(dec.codes, c0) and torch.equal(dec.vnorm, v0)


def test_append_past_capacity_is_skipped():
    """seq_lens[b] > N_max: the step must not write outside row b's cache."""
    N, k = 2048, 200
    cfg = Config(B=2, H_q=8, H_kv=2, N_max=N, L=16, P=8)
    q, K, V = datagen.torch_make_cache(2, 8, 2, N, 128, seed=12)
    W = bits_to_dev(datagen.make_projections(4251, 16, 8, 128))
    for flags in (0, 1):
        c = Config(**{**cfg.__dict__, "flags": flags})
        dec = SocketDecoder(c, W, K, V, k=k)
        dec.prefill()
        K0, c0, v0 = K.clone(), dec.codes.clone(), dec.vnorm.clone()
        lens = torch.tensor([N + 1, N + 40], dtype=torch.int32, device=DEV)
        kn = torch.ones((2, 2, 128), dtype=torch.bfloat16, device=DEV)
        dec.step(q, lens, append=True, k_new=kn, v_new=kn)
        torch.cuda.synchronize()
        assert torch.equal(K, K0) and torch.equal(dec.codes, c0) and torch.equal(dec.vnorm, v0)
