"""Helpers shared by the GPU parity tests (comparison rules of DESIGN.md §4)."""
import math

import numpy as np
import torch

# BASELINE.json north_star tolerances
TOL = {
    "bf16": {"O": 1e-2, "grad": 5e-2, "L": 1e-3},
    "fp16": {"O": 2e-3, "grad": 1e-2, "L": 1e-3},
}
MANT = {"bf16": 7, "fp16": 10}


def half_ulp(ref: np.ndarray, dtype: str) -> np.ndarray:
    """Half a unit in the last place of the dtype at |ref| (R14): the error a
    correctly rounded output of the exact value may already carry."""
    a = np.abs(ref)
    e = np.floor(np.log2(np.maximum(a, 2.0 ** -14)))
    return 2.0 ** (e - MANT[dtype] - 1)


def o_excess(o_gpu: torch.Tensor, o_ref: np.ndarray, dtype: str) -> float:
    err = np.abs(o_gpu.double().cpu().numpy() - o_ref)
    return float(np.max(err - half_ulp(o_ref, dtype)))


def max_abs(a, b) -> float:
    a = a.double().cpu().numpy() if isinstance(a, torch.Tensor) else a
    b = b.double().cpu().numpy() if isinstance(b, torch.Tensor) else b
    return float(np.max(np.abs(a - b)))


def grad_ok(g_gpu: torch.Tensor, g_ref: np.ndarray, dtype: str, floor: float = 0.0, degenerate: bool = False):
    """Per-tensor rule (R15): max-abs error <= c * max|g_ref|.

    `floor` (2^-8 of the largest of the three gradients, `grad_floor`) replaces
    max|g_ref| only where the exact gradient vanishes (e.g. dQ = dK = 0 at N = 1,
    dQ = 0 for identical keys): the caller must declare such a case with
    `degenerate=True`, and a non-degenerate reference below the floor fails."""
    err = max_abs(g_gpu, g_ref)
    ref_max = float(np.max(np.abs(g_ref))) if g_ref.size else 0.0
    if ref_max >= floor:
        lim = TOL[dtype]["grad"] * ref_max
    elif degenerate:
        lim = TOL[dtype]["grad"] * floor
    else:
        return False, err, f"reference max {ref_max} below the floor {floor} in a case not declared degenerate"
    return err <= lim, err, lim


def grad_floor(*refs) -> float:
    return 2.0 ** -8 * max(float(np.max(np.abs(r))) for r in refs)


def to_np(t: torch.Tensor) -> np.ndarray:
    return t.double().cpu().numpy()


def scale_for(d: int) -> float:
    return 1.0 / math.sqrt(d)
