"""Benchmark FLOP accounting and the causal block census, as the paper defines them.

TEST INFRASTRUCTURE ONLY (see oracle/ref_attention.py header).

* FLOPs: forward = 4 * seqlen^2 * head_dim * heads, times batch
  (the batch factor is omitted at P:619; BASELINE.json multiplies by B, R9);
  halved with a causal mask; backward = 2.5 x forward; fwd+bwd = 3.5 x forward.
* Causal census: a (row block i, column block j) pair is
  Skip if every column index exceeds every row index, Full if no column index
  exceeds any row index, Partial otherwise.  Brute force over every pair and
  every element, written as the definition (slow, small inputs only).
"""
from __future__ import annotations


def attention_flops(batch: int, heads: int, seqlen: int, head_dim: int, causal: bool,
                    pass_: str = "fwd") -> float:
    f = 4.0 * seqlen * seqlen * head_dim * heads * batch
    if causal:
        f /= 2.0
    mult = {"fwd": 1.0, "bwd": 2.5, "fwd_bwd": 3.5}[pass_]
    return f * mult


def causal_census(n: int, br: int, bc: int):
    """Classify every block pair of an N x N causal score matrix by checking
    every element (j > i is masked).  Returns dict(full, partial, skip) counts
    and the per-row-block list of computed column blocks."""
    tr = -(-n // br)
    tc = -(-n // bc)
    full = partial = skip = 0
    computed = []
    for i in range(tr):
        rows = range(i * br, min(n, (i + 1) * br))
        cols_done = []
        for j in range(tc):
            cols = range(j * bc, min(n, (j + 1) * bc))
            masked = [c > r for r in rows for c in cols]
            if all(masked):
                skip += 1
            elif any(masked):
                partial += 1
                cols_done.append(j)
            else:
                full += 1
                cols_done.append(j)
        computed.append(cols_done)
    return {"full": full, "partial": partial, "skip": skip, "computed": computed}
