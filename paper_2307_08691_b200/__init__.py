"""B200 (sm_100a) FlashAttention-2 hot path — thin Python binding over the C ABI.

Argument marshalling only: every step of the attention path runs in the CUDA
kernels of ``libfa2_sm100.so`` (see include/fa2.h).  PyTorch supplies device
memory and the current stream.  There is no CPU fallback: if the library is
missing or the device is not sm_100, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

__all__ = ["lib", "forward", "backward", "forward_fp8", "forward_varlen", "backward_varlen", "backward_varlen_workspace_size",
           "backward_preprocess", "backward_workspace_size",
           "attention_step_host", "step_arena_size", "kv_block_range", "set_timing_events", "FA2Error", "LIB_PATH"]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FA2_LIB_PATH") or os.path.join(HERE, "libfa2_sm100.so")

FA2_BF16, FA2_FP16 = 0, 1
_STATUS = {0: "FA2_OK", 1: "FA2_ERR_INVALID_ARG", 2: "FA2_ERR_UNSUPPORTED", 3: "FA2_ERR_WORKSPACE", 4: "FA2_ERR_CUDA"}


class FA2Error(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{_STATUS.get(status, status)}: {detail}")
        self.status = status
        self.detail = detail


_lib = None


def lib() -> ctypes.CDLL:
    """Load libfa2_sm100.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FA2Error(-1, f"{LIB_PATH} not built (run `python -c 'import __graft_entry__ as g; g.build()'`)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, f, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t
        L.fa2_forward.argtypes = [vp, vp, vp, vp, vp, i, i, i, i, i, f, i, vp]
        L.fa2_forward.restype = i
        L.fa2_forward_gqa.argtypes = [vp, vp, vp, vp, vp, i, i, i, i, i, i, f, i, vp]
        L.fa2_forward_gqa.restype = i
        L.fa2_backward_gqa.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, i, i, i, i, i, i, f, i, vp]
        L.fa2_backward_gqa.restype = i
        L.fa2_backward_deterministic.argtypes = L.fa2_backward_gqa.argtypes
        L.fa2_backward_deterministic.restype = i
        L.fa2_forward_ex.argtypes = [vp, vp, vp, vp, vp, i, i, i, i, i, i, i, f, i, vp]
        L.fa2_forward_ex.restype = i
        L.fa2_forward_varlen.argtypes = [vp, vp, vp, vp, vp, vp, vp, i, i, i, i, i, i, i, i, i, f, i, vp]
        L.fa2_forward_varlen.restype = i
        L.fa2_forward_fp8.argtypes = [vp, vp, vp, vp, vp, i, i, i, i, i, i, f, f, f, f, vp]
        L.fa2_forward_fp8.restype = i
        L.fa2_backward_ex.argtypes = [vp] * 10 + [sz, i, i, i, i, i, i, i, f, i, i, vp]
        L.fa2_backward_ex.restype = i
        L.fa2_backward_varlen.argtypes = [vp] * 11 + [vp, sz, i, i, i, i, i, i, i, i, i, f, i, i, vp]
        L.fa2_backward_varlen.restype = i
        L.fa2_backward_varlen_workspace_size.argtypes = [i, i, i, i]
        L.fa2_backward_varlen_workspace_size.restype = sz
        L.fa2_backward.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, i, i, i, i, i, f, i, vp]
        L.fa2_backward.restype = i
        L.fa2_backward_preprocess.argtypes = [vp, vp, vp, i, i, i, i, i, vp]
        L.fa2_backward_preprocess.restype = i
        L.fa2_backward_workspace_size.argtypes = [i, i, i, i]
        L.fa2_backward_workspace_size.restype = sz
        L.fa2_step_arena_size.argtypes = [i, i, i, i]
        L.fa2_step_arena_size.restype = sz
        L.fa2_attention_step_host.argtypes = [vp] * 9 + [vp, sz, i, i, i, i, i, f, i, vp]
        L.fa2_attention_step_host.restype = i
        L.fa2_kv_block_range.argtypes = [i, i, i, i, i, ctypes.POINTER(i), ctypes.POINTER(i)]
        L.fa2_kv_block_range.restype = i
        us = ctypes.POINTER(ctypes.c_ushort)
        L.fa2_tile_schedule.argtypes = [i, i, i, i, i, us, us, i, ctypes.POINTER(i)]
        L.fa2_tile_schedule.restype = i
        L.fa2_status_string.argtypes = [i]
        L.fa2_status_string.restype = ctypes.c_char_p
        L.fa2_last_error_detail.argtypes = []
        L.fa2_last_error_detail.restype = ctypes.c_char_p
        L.fa2_debug_set_trace.argtypes = [vp]
        L.fa2_debug_set_trace.restype = None
        L.fa2_set_timing_events.argtypes = [vp]
        L.fa2_set_timing_events.restype = None
        L.fa2_last_launch_count.argtypes = []
        L.fa2_last_launch_count.restype = i
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise FA2Error(status, lib().fa2_last_error_detail().decode())


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.bfloat16:
        return FA2_BF16
    if t.dtype == torch.float16:
        return FA2_FP16
    raise FA2Error(2, f"unsupported dtype {t.dtype}")


def _stream(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def _shape(q):
    if q.dim() != 4:
        raise FA2Error(1, "expected [B, H, N, d] tensors")
    return tuple(q.shape)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _need(t, shape, dtype, device, name):
    """Every buffer handed to the library: a contiguous tensor of the expected shape,
    dtype and device (the C layer checks only NULL and 16-byte alignment)."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise FA2Error(1, f"{name} must be a torch.Tensor")
    shape = tuple(int(x) for x in shape)
    if (tuple(t.shape) != shape or t.dtype != dtype or not t.is_contiguous() or t.device != device):
        raise FA2Error(1, f"{name} must be a contiguous {shape} {dtype} tensor on {device} "
                          f"(got {tuple(t.shape)} {t.dtype} on {t.device}, contiguous={t.is_contiguous()})")


def _need_cuda(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise FA2Error(1, f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise FA2Error(1, f"{name} must be contiguous")


def _need_workspace(ws, device, name="workspace"):
    """Scratch buffers: contiguous, on the device.  Their size is checked by the C
    layer, which knows the minimum (e.g. the backward workspace without the GQA
    split's extra accumulators) and returns FA2_ERR_WORKSPACE when it is short."""
    import torch
    if not isinstance(ws, torch.Tensor) or ws.device != device or not ws.is_contiguous():
        raise FA2Error(1, f"{name} must be a contiguous tensor on {device}")


def _kv_heads(q, k):
    hkv = k.shape[1] if k.dim() == 4 else -1
    if hkv < 1 or q.shape[1] % hkv:
        raise FA2Error(1, f"key/value heads ({hkv}) must divide query heads ({q.shape[1]})")
    return hkv


def _kv_check(q, k, v, dtype=None):
    """q: contiguous [B, H, N_q, d] CUDA tensor; k, v: [B, H_kv, N_k, d] with H_kv | H,
    q's dtype (or `dtype`) and device.  Returns (H_kv, N_k)."""
    import torch
    _need_cuda(q, "q")
    if not isinstance(k, torch.Tensor) or k.dim() != 4 or k.shape[0] != q.shape[0] or k.shape[3] != q.shape[3]:
        raise FA2Error(1, f"k must be [B, H_kv, N_k, d] matching q {tuple(q.shape)}")
    Hkv = _kv_heads(q, k)
    dt = q.dtype if dtype is None else dtype
    _need(k, k.shape, dt, q.device, "k")
    _need(v, k.shape, dt, q.device, "v")
    return Hkv, k.shape[2]


def forward(q, k, v, causal: bool = False, softmax_scale: float | None = None, out=None, lse=None, stream=None):
    """O, L for [B,H,N_q,d] bf16/fp16 CUDA tensors (Alg. 1).  k, v are
    [B,H_kv,N_k,d]: H_kv < H heads is MQA/GQA; N_k != N_q uses the
    bottom-right causal alignment (fa2_forward_ex, R22).
    Returns (o, lse[B,H,N_q] fp32)."""
    import torch
    B, H, N, d = _shape(q)
    Hkv, Nk = _kv_check(q, k, v)
    _dtype_code(q)
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    o = torch.empty_like(q) if out is None else out
    L = torch.empty((B, H, N), dtype=torch.float32, device=q.device) if lse is None else lse
    _need(o, q.shape, q.dtype, q.device, "out")
    _need(L, (B, H, N), torch.float32, q.device, "lse")
    if Nk == N:
        _check(lib().fa2_forward_gqa(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), B, H, Hkv, N, d, int(bool(causal)),
                                     scale, _dtype_code(q), ctypes.c_void_p(_stream(stream))))
    else:
        _check(lib().fa2_forward_ex(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), B, H, Hkv, N, Nk, d,
                                    int(bool(causal)), scale, _dtype_code(q), ctypes.c_void_p(_stream(stream))))
    return o, L


def backward_workspace_size(B: int, H: int, N: int, d: int) -> int:
    return int(lib().fa2_backward_workspace_size(B, H, N, d))


def backward(q, k, v, o, lse, do, causal: bool = False, softmax_scale: float | None = None,
             dq=None, dk=None, dv=None, workspace=None, stream=None, deterministic: bool = False):
    """dQ, dK, dV (Alg. 2).  With H_kv < H key/value heads, dK/dV are
    summed over each group of query heads.  deterministic=True calls
    fa2_backward_deterministic (fixed dQ summation order, bitwise reproducible).
    Returns (dq, dk, dv)."""
    import torch
    B, H, N, d = _shape(q)
    Hkv, Nk = _kv_check(q, k, v)
    _dtype_code(q)
    for t, n in ((o, "o"), (do, "do")):
        _need(t, q.shape, q.dtype, q.device, n)
    _need(lse, (B, H, N), torch.float32, q.device, "lse")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    _need(dq, q.shape, q.dtype, q.device, "dq")
    _need(dk, k.shape, k.dtype, q.device, "dk")
    _need(dv, k.shape, k.dtype, q.device, "dv")
    wsz = backward_workspace_size(B, H, N, d)
    if workspace is None:
        workspace = torch.empty(wsz, dtype=torch.uint8, device=q.device)
    _need_workspace(workspace, q.device)
    args = (_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(do), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(workspace),
            workspace.numel() * workspace.element_size())
    st = ctypes.c_void_p(_stream(stream))
    if Nk == N:
        fn = lib().fa2_backward_deterministic if deterministic else lib().fa2_backward_gqa
        _check(fn(*args, B, H, Hkv, N, d, int(bool(causal)), scale, _dtype_code(q), st))
    else:
        _check(lib().fa2_backward_ex(*args, B, H, Hkv, N, Nk, d, int(bool(causal)), scale, int(bool(deterministic)),
                                     _dtype_code(q), st))
    return dq, dk, dv


def forward_fp8(q, k, v, descale_q: float = 1.0, descale_k: float = 1.0, descale_v: float = 1.0,
                causal: bool = False, softmax_scale: float | None = None, out=None, lse=None, stream=None):
    """FP8 forward (fa2_forward_fp8): q [B,H,N,128], k/v [B,H_kv,N,128] torch.float8_e4m3fn
    CUDA tensors representing descale_x * x.  Returns (o [B,H,N,128] bf16, lse [B,H,N] fp32)."""
    import torch
    B, H, N, d = _shape(q)
    if q.dtype != torch.float8_e4m3fn:
        raise FA2Error(1, "q must be torch.float8_e4m3fn")
    Hkv, Nk = _kv_check(q, k, v, dtype=torch.float8_e4m3fn)
    if Nk != N:
        raise FA2Error(1, "FP8 forward: k/v with N_k == N_q")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    o = torch.empty((B, H, N, d), dtype=torch.bfloat16, device=q.device) if out is None else out
    L = torch.empty((B, H, N), dtype=torch.float32, device=q.device) if lse is None else lse
    _need(o, (B, H, N, d), torch.bfloat16, q.device, "out")
    _need(L, (B, H, N), torch.float32, q.device, "lse")
    _check(lib().fa2_forward_fp8(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), B, H, Hkv, N, d, int(bool(causal)), scale,
                                 float(descale_q), float(descale_k), float(descale_v), ctypes.c_void_p(_stream(stream))))
    return o, L


def _varlen_check(q, k, v, cu_q, cu_k):
    import torch
    if q.dim() != 3 or k.dim() != 3 or k.shape[2] != q.shape[2]:
        raise FA2Error(1, "varlen tensors are packed [total, heads, d]")
    Hkv = k.shape[1]
    if Hkv < 1 or q.shape[1] % Hkv:
        raise FA2Error(1, f"key/value heads ({Hkv}) must divide query heads ({q.shape[1]})")
    _need_cuda(q, "q")
    _dtype_code(q)
    _need(k, k.shape, q.dtype, q.device, "k")
    _need(v, k.shape, q.dtype, q.device, "v")
    for c, n in ((cu_q, "cu_seqlens_q"), (cu_k, "cu_seqlens_k")):
        if c.dtype != torch.int32 or c.dim() != 1 or not c.is_contiguous() or c.device != q.device:
            raise FA2Error(1, f"{n} must be a contiguous int32 tensor on {q.device}")
    if cu_q.numel() != cu_k.numel() or cu_q.numel() < 2:
        raise FA2Error(1, "cu_seqlens_q and cu_seqlens_k must both have B+1 >= 2 entries")
    return cu_q.numel() - 1, Hkv


def forward_varlen(q, k, v, cu_seqlens_q, cu_seqlens_k, max_seqlen_q: int, max_seqlen_k: int, causal: bool = False,
                   softmax_scale: float | None = None, out=None, lse=None, stream=None):
    """Packed variable-length batch (fa2_forward_varlen): q [T_q,H,d], k/v
    [T_k,H_kv,d], cu_seqlens_* int32 [B+1] on the device.  Returns (o [T_q,H,d],
    lse [H,T_q] fp32)."""
    import torch
    B, Hkv = _varlen_check(q, k, v, cu_seqlens_q, cu_seqlens_k)
    Tq, H, d = q.shape
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    o = torch.empty_like(q) if out is None else out
    L = torch.empty((H, Tq), dtype=torch.float32, device=q.device) if lse is None else lse
    _need(o, q.shape, q.dtype, q.device, "out")
    _need(L, (H, Tq), torch.float32, q.device, "lse")
    _check(lib().fa2_forward_varlen(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(L), _ptr(cu_seqlens_q),
                                    _ptr(cu_seqlens_k), B, H, Hkv, Tq, k.shape[0], int(max_seqlen_q),
                                    int(max_seqlen_k), d, int(bool(causal)), scale, _dtype_code(q),
                                    ctypes.c_void_p(_stream(stream))))
    return o, L


def backward_varlen_workspace_size(B: int, H: int, total_q: int, d: int) -> int:
    return int(lib().fa2_backward_varlen_workspace_size(B, H, total_q, d))


def backward_varlen(q, k, v, o, lse, do, cu_seqlens_q, cu_seqlens_k, max_seqlen_q: int, max_seqlen_k: int,
                    causal: bool = False, softmax_scale: float | None = None, dq=None, dk=None, dv=None,
                    workspace=None, stream=None, deterministic: bool = False):
    """Backward of forward_varlen (fa2_backward_varlen).  Returns (dq, dk, dv)."""
    import torch
    B, Hkv = _varlen_check(q, k, v, cu_seqlens_q, cu_seqlens_k)
    Tq, H, d = q.shape
    for t, n in ((o, "o"), (do, "do")):
        _need(t, q.shape, q.dtype, q.device, n)
    _need(lse, (H, Tq), torch.float32, q.device, "lse")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    _need(dq, q.shape, q.dtype, q.device, "dq")
    _need(dk, k.shape, k.dtype, q.device, "dk")
    _need(dv, k.shape, k.dtype, q.device, "dv")
    wsz = backward_varlen_workspace_size(B, H, Tq, d)
    if workspace is None:
        workspace = torch.empty(wsz, dtype=torch.uint8, device=q.device)
    _need_workspace(workspace, q.device)
    _check(lib().fa2_backward_varlen(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(do), _ptr(dq), _ptr(dk),
                                     _ptr(dv), _ptr(cu_seqlens_q), _ptr(cu_seqlens_k), _ptr(workspace),
                                     workspace.numel() * workspace.element_size(), B, H, Hkv, Tq, k.shape[0],
                                     int(max_seqlen_q), int(max_seqlen_k), d, int(bool(causal)), scale,
                                     int(bool(deterministic)), _dtype_code(q), ctypes.c_void_p(_stream(stream))))
    return dq, dk, dv


def backward_preprocess(o, do, stream=None):
    """D = rowsum(dO o O), [B,H,N] fp32."""
    import torch
    B, H, N, d = _shape(o)
    _need_cuda(o, "o")
    _dtype_code(o)
    _need(do, o.shape, o.dtype, o.device, "do")
    out = torch.empty((B, H, N), dtype=torch.float32, device=o.device)
    _check(lib().fa2_backward_preprocess(_ptr(o), _ptr(do), _ptr(out), B, H, N, d, _dtype_code(o),
                                         ctypes.c_void_p(_stream(stream))))
    return out


def step_arena_size(B: int, H: int, N: int, d: int) -> int:
    return int(lib().fa2_step_arena_size(B, H, N, d))


def attention_step_host(q_h, k_h, v_h, do_h, outs, arena, causal: bool, softmax_scale: float | None = None,
                        stream=None):
    """One end-to-end fwd+bwd step through HOST (pinned) tensors.  `outs` is a
    dict with optional host tensors o, lse, dq, dk, dv to receive results."""
    import torch
    B, H, N, d = _shape(q_h)
    _dtype_code(q_h)
    cpu = torch.device("cpu")
    for t, n in ((q_h, "q"), (k_h, "k"), (v_h, "v"), (do_h, "do")):
        _need(t, q_h.shape, q_h.dtype, cpu, n + " (host)")
    for n, t in outs.items():
        if n not in ("o", "lse", "dq", "dk", "dv"):
            raise FA2Error(1, f"unknown output {n!r}")
        if t is not None:
            _need(t, (B, H, N) if n == "lse" else q_h.shape, torch.float32 if n == "lse" else q_h.dtype, cpu,
                  n + " (host)")
    if not isinstance(arena, torch.Tensor) or not arena.is_cuda:
        raise FA2Error(1, "arena must be a CUDA tensor")
    _need_workspace(arena, arena.device, "arena")
    scale = 1.0 / math.sqrt(d) if softmax_scale is None else float(softmax_scale)
    g = outs.get
    _check(lib().fa2_attention_step_host(_ptr(q_h), _ptr(k_h), _ptr(v_h), _ptr(do_h), _ptr(g("o")),
                                         _ptr(g("lse")), _ptr(g("dq")), _ptr(g("dk")), _ptr(g("dv")),
                                         _ptr(arena), arena.numel() * arena.element_size(), B, H, N, d,
                                         int(bool(causal)), scale, _dtype_code(q_h),
                                         ctypes.c_void_p(_stream(stream))))


def set_timing_events(events):
    """Benchmark hook: `events` is a list of 6 torch.cuda.Event (created with
    enable_timing=True) or None.  See fa2_set_timing_events in include/fa2.h.
    Returns the ctypes array, which the caller must keep alive while in use."""
    if events is None:
        lib().fa2_set_timing_events(None)
        return None
    arr = (ctypes.c_void_p * 6)(*[ctypes.c_void_p(e.cuda_event) for e in events])
    lib().fa2_set_timing_events(ctypes.cast(arr, ctypes.c_void_p))
    return arr


def tile_schedule(pass_: int, heads: int, N: int, heads_per_tile: int = 1, grid: int = 148):
    """Host balanced schedule of the causal square forward (pass_=0) / backward (1):
    returns (order, start) with CTA c running order[start[c]:start[c+1]]."""
    per_head = -(-N // (256 if pass_ == 0 else 128))
    cap = max(1, per_head * heads)
    order = (ctypes.c_ushort * cap)()
    start = (ctypes.c_ushort * (grid + 1))()
    nt = ctypes.c_int(0)
    _check(lib().fa2_tile_schedule(pass_, heads, N, heads_per_tile, grid, order, start, cap, ctypes.byref(nt)))
    return list(order[:nt.value]), list(start)


def kv_block_range(N: int, Br: int, Bc: int, i: int, causal: bool):
    """Host tile map: (n_blocks, first_masked) for query row block i."""
    nb, fm = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().fa2_kv_block_range(N, Br, Bc, i, int(bool(causal)), ctypes.byref(nb), ctypes.byref(fm)))
    return nb.value, fm.value
