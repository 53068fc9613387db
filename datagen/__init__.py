"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the SOCKET method (no hashing, no soft
probabilities, no scoring, no selection, no attention).  It only draws random
numbers and rounds them to bf16, so that `oracle/` (test infrastructure) and
the CUDA path (`paper_2602_06283_b200`) can consume bit-identical inputs
without sharing any code.

Input recipe:
  * q, K, V ~ N(0, 1), rounded to bf16 (round-to-nearest-even).  This is the
    value distribution of the paper's ranking study (Fig. 2 caption, PAPER.md
    l.147-149: "Keys are randomly generated using a standard Gaussian
    distribution").
  * W^(l) ~ N(0, 1) i.i.d. rows (Alg. 1), drawn from a fixed
    seed, rounded to bf16; one W shared by every head and batch (DESIGN.md
    reading R-12).
  * Variants: "gauss" (default), "unitq" (q rescaled to unit norm, the small
    signal regime of PAPER.md l.670), "needle" (k/8 keys planted near q so the
    selection is non-trivial).

Two back-ends draw the same *distribution*:
  * numpy PCG64 (host) for small, oracle-sized cases; and
  * torch generators (device) for BASELINE-sized caches that are too large to
    draw on the host.  For those, the host copy of any sampled slice is taken
    from the device tensor, so the two sides still see identical bits.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "bf16_bits_from_f32",
    "f32_from_bf16_bits",
    "make_projections",
    "make_case",
    "torch_make_cache",
]


def bf16_bits_from_f32(x: np.ndarray) -> np.ndarray:
    """Round float32 values to bf16 (round-to-nearest-even); return uint16 bits."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    lsb = (b >> 16) & 1
    r = ((b + 0x7FFF + lsb) >> 16).astype(np.uint16)
    return r


def f32_from_bf16_bits(bits: np.ndarray) -> np.ndarray:
    """Widen bf16 bits (uint16) to float32 exactly."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def make_projections(seed: int, L: int, P: int, d: int) -> np.ndarray:
    """W[L][P][d] as bf16 bits; fp32 N(0,1) draws from PCG64(seed) rounded to bf16."""
    rng = np.random.Generator(np.random.PCG64(seed))
    w = rng.standard_normal((L, P, d), dtype=np.float32)
    return bf16_bits_from_f32(w)


def make_case(B: int, H_q: int, H_kv: int, N_max: int, d: int, seed: int,
              variant: str = "gauss", seq_lens=None, n_needle: int = 0):
    """Draw one synthetic decode case on the host.

    Returns dict of uint16 bf16-bit arrays q[B][H_q][d], K/V[B][H_kv][N_max][d]
    and int32 seq_lens[B].  Rows j >= seq_lens[b] are still filled with random
    data (they must be ignored by both sides).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    q = rng.standard_normal((B, H_q, d), dtype=np.float32)
    K = rng.standard_normal((B, H_kv, N_max, d), dtype=np.float32)
    V = rng.standard_normal((B, H_kv, N_max, d), dtype=np.float32)
    if variant == "unitq":
        q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    elif variant == "needle":
        # Plant n_needle keys per (b, kv-head) near the direction of the
        # group's first query head: k = 4*q/|q| + 0.5*noise.
        G = H_q // H_kv
        for b in range(B):
            for g in range(H_kv):
                qd = q[b, g * G] / np.linalg.norm(q[b, g * G])
                pos = rng.choice(N_max, size=min(n_needle, N_max), replace=False)
                K[b, g, pos] = 4.0 * qd + 0.5 * rng.standard_normal((len(pos), d), dtype=np.float32)
    elif variant != "gauss":
        raise ValueError(f"unknown variant {variant!r}")
    if seq_lens is None:
        seq_lens = np.full((B,), N_max, dtype=np.int32)
    seq_lens = np.asarray(seq_lens, dtype=np.int32)
    return {
        "q": bf16_bits_from_f32(q),
        "K": bf16_bits_from_f32(K),
        "V": bf16_bits_from_f32(V),
        "seq_lens": seq_lens,
    }


def torch_make_cache(B: int, H_q: int, H_kv: int, N_max: int, d: int, seed: int,
                     device="cuda"):
    """Draw a BASELINE-sized cache directly in device memory (torch generator).

    Same distribution as make_case(variant="gauss"); used for sizes the host
    cannot draw in seconds.  Returns bf16 tensors q, K, V.
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    q = torch.randn((B, H_q, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    K = torch.empty((B, H_kv, N_max, d), device=device, dtype=torch.bfloat16)
    V = torch.empty((B, H_kv, N_max, d), device=device, dtype=torch.bfloat16)
    # draw in slabs to bound the fp32 temporary
    for b in range(B):
        K[b] = torch.randn((H_kv, N_max, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
        V[b] = torch.randn((H_kv, N_max, d), generator=g, device=device, dtype=torch.float32).to(torch.bfloat16)
    return q, K, V
