"""Shared test helpers (host <-> device marshalling of datagen bits)."""
import numpy as np
import torch


def bits_to_dev(bits: np.ndarray, device="cuda") -> torch.Tensor:
    """uint16 bf16 bit pattern array -> bf16 CUDA tensor with identical bits."""
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to(device).view(torch.bfloat16)


def dev_to_bits(t: torch.Tensor) -> np.ndarray:
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def rel_err(a, b, floor=0.0):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), floor)
