"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO attention arithmetic: only seeded random draws, dtype
rounding of the draws, and the construction of special-case inputs.  Both the
oracle (tests, bench cpu_baseline) and the product path consume exactly the
tensors returned here.  Recipe:

  * Q, K, V, dO iid N(0, 1), layout [B, H, N, d], generated in float32 by a
    seeded torch CPU generator, then rounded (RN) to the kernel dtype.  The
    oracle upcasts the *rounded* values to float64 (R18).
  * seeds: q = base+0, k = base+1, v = base+2, dO = base+3.
  * stress variants: logit scale multiplier (std of QK^T*scale ~ sigma) and a
    +300 overflow case.
"""
from __future__ import annotations

import torch

_DT = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32}


def torch_dtype(name: str) -> torch.dtype:
    return _DT[name]


def randn(shape, seed: int, dtype: str = "bf16", std: float = 1.0) -> torch.Tensor:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    x = torch.randn(*shape, generator=g, dtype=torch.float32)
    if std != 1.0:
        x = x * std
    return x.to(_DT[dtype])


def qkv(b: int, h: int, n: int, d: int, dtype: str = "bf16", seed: int = 0, std: float = 1.0,
        with_do: bool = True):
    """Seeded (q, k, v, do) CPU tensors of shape [B, H, N, d] in `dtype`."""
    shape = (b, h, n, d)
    q = randn(shape, seed + 0, dtype, std)
    k = randn(shape, seed + 1, dtype, std)
    v = randn(shape, seed + 2, dtype)
    do = randn(shape, seed + 3, dtype) if with_do else None
    return q, k, v, do


def identical_keys(n: int, d: int, dtype: str = "bf16", seed: int = 0):
    """Every key row equal (one random row repeated); q, v random."""
    q = randn((1, 1, n, d), seed, dtype)
    k_row = randn((1, 1, 1, d), seed + 1, dtype)
    k = k_row.expand(1, 1, n, d).contiguous()
    v = randn((1, 1, n, d), seed + 2, dtype)
    return q, k, v


def one_hot_logit(n: int, d: int, j_star: int, alpha: float = 32.0, dtype: str = "bf16", seed: int = 0):
    """Every Q row = alpha*e_0; K row j_star = alpha*e_0, other K rows 0.
    alpha = 32 is exact in bf16/fp16."""
    q = torch.zeros((1, 1, n, d), dtype=torch.float32)
    q[..., 0] = alpha
    k = torch.zeros((1, 1, n, d), dtype=torch.float32)
    k[0, 0, j_star, 0] = alpha
    v = randn((1, 1, n, d), seed + 2, dtype)
    return q.to(_DT[dtype]), k.to(_DT[dtype]), v
