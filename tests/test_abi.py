"""CPU tests of the C-ABI library: it builds, loads, exports every symbol that
include/fa2.h declares, validates arguments before touching CUDA, and its
host-side tile map agrees with the oracle's brute-force causal census."""
import ctypes
import os
import re

import pytest

import paper_2307_08691_b200 as fa2
from oracle import flops as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2307_08691_b200 import build
    build.build()
    return fa2.lib()


def header_functions():
    txt = open(os.path.join(ROOT, "include", "fa2.h")).read()
    return re.findall(r"FA2_API\s+[\w\s\*]+?\b(fa2_\w+)\s*\(", txt)


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n
    # and nothing else leaks out of the .so besides the declared C symbols
    out = os.popen(f"nm -D --defined-only {fa2.LIB_PATH}").read()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert set(names) <= exported
    assert all(not s.startswith("_Z") for s in exported), [s for s in exported if s.startswith("_Z")][:5]


def test_status_strings(L):
    for code, name in [(0, b"FA2_OK"), (1, b"FA2_ERR_INVALID_ARG"), (2, b"FA2_ERR_UNSUPPORTED"),
                       (3, b"FA2_ERR_WORKSPACE"), (4, b"FA2_ERR_CUDA")]:
        assert L.fa2_status_string(code) == name


FAKE = [ctypes.c_void_p(4096 * (i + 1)) for i in range(9)]   # aligned, never dereferenced


def fwd(L, B=1, H=1, N=128, d=64, causal=0, scale=0.125, dtype=0, ptrs=None):
    p = ptrs or FAKE
    return L.fa2_forward(p[0], p[1], p[2], p[3], p[4], B, H, N, d, causal, scale, dtype, None)


def test_forward_validation(L):
    assert fwd(L, d=96) == 2
    assert fwd(L, d=256) == 2
    assert fwd(L, dtype=7) == 2
    assert fwd(L, N=0) == 1
    assert fwd(L, B=0) == 1
    assert fwd(L, H=-1) == 1
    assert fwd(L, scale=0.0) == 1
    assert fwd(L, scale=float("nan")) == 1
    assert fwd(L, scale=float("inf")) == 1
    assert fwd(L, ptrs=[None] + FAKE[1:]) == 1
    mis = list(FAKE)
    mis[2] = ctypes.c_void_p(4096 + 8)
    assert fwd(L, ptrs=mis) == 1
    assert b"16-byte" in L.fa2_last_error_detail()
    # valid arguments reach CUDA; with no GPU in this container that is FA2_ERR_CUDA / UNSUPPORTED
    assert fwd(L) in (2, 4)


def test_backward_validation(L):
    ws = L.fa2_backward_workspace_size(2, 3, 100, 64)
    npad = 128
    sem = (2 * 3 * (npad // 32) * 4 + 15) // 16 * 16   # 4 counters per 128-row tile
    base = 2 * 3 * npad * 64 * 4 + 2 * 2 * 3 * npad * 4 + sem
    # + room for the GQA split's fp32 dK/dV accumulators (256-byte aligned)
    assert ws == (base + 255) // 256 * 256 + 2 * 3 * 100 * 64 * 8
    assert L.fa2_backward_workspace_size(1, 1, 1, 96) == 0
    args = FAKE[:9]
    r = L.fa2_backward(*args, ctypes.c_void_p(1 << 20), base - 1, 2, 3, 100, 64, 0, 0.125, 0, None)
    assert r == 3   # the base layout is the minimum (the split room is optional)
    r = L.fa2_backward(*args, None, ws, 2, 3, 100, 64, 0, 0.125, 0, None)
    assert r == 3
    r = L.fa2_backward(*args[:5], None, *args[6:9], ctypes.c_void_p(1 << 20), ws, 2, 3, 100, 64, 0, 0.125, 0, None)
    assert r == 1
    r = L.fa2_backward(*args, ctypes.c_void_p(1 << 20), ws, 2, 3, 100, 80, 0, 0.125, 0, None)
    assert r == 2


def test_step_arena_size(L):
    t = 2 * 3 * 100 * 64 * 2
    t16 = (t + 255) // 256 * 256
    lb = (2 * 3 * 100 * 4 + 255) // 256 * 256
    assert L.fa2_step_arena_size(2, 3, 100, 64) == 9 * t16 + lb + L.fa2_backward_workspace_size(2, 3, 100, 64)


@pytest.mark.parametrize("N", [1, 17, 127, 128, 129, 256, 300, 1000])
@pytest.mark.parametrize("Br,Bc", [(128, 128), (64, 128), (128, 64), (32, 16)])
@pytest.mark.parametrize("causal", [False, True])
def test_kv_block_range_matches_census(L, N, Br, Bc, causal):
    """The library's host tile map vs the oracle's element-by-element census."""
    if causal:
        c = F.causal_census(N, Br, Bc)
    tr = -(-N // Br)
    tc = -(-N // Bc)
    for i in range(tr):
        nb, fm = fa2.kv_block_range(N, Br, Bc, i, causal)
        if causal:
            assert nb == len(c["computed"][i])
            assert c["computed"][i] == list(range(nb))
        else:
            assert nb == tc
        # first masked block: first computed block containing a masked or out-of-range column
        rows = range(i * Br, min(N, (i + 1) * Br))
        want = nb
        for j in range(nb):
            cols = range(j * Bc, (j + 1) * Bc)
            if any(cc >= N or (causal and cc > r) for r in rows for cc in cols):
                want = j
                break
        assert fm == want, (i, nb, fm, want)


def test_kv_block_range_errors(L):
    with pytest.raises(fa2.FA2Error):
        fa2.kv_block_range(100, 128, 128, 1, False)
    with pytest.raises(fa2.FA2Error):
        fa2.kv_block_range(0, 128, 128, 0, False)


def test_gqa_validation(L):
    p = FAKE
    # H must be a positive multiple of H_kv
    assert L.fa2_forward_gqa(p[0], p[1], p[2], p[3], p[4], 1, 6, 4, 128, 64, 0, 0.125, 0, None) == 1
    assert L.fa2_forward_gqa(p[0], p[1], p[2], p[3], p[4], 1, 6, 0, 128, 64, 0, 0.125, 0, None) == 1
    assert L.fa2_forward_gqa(p[0], p[1], p[2], p[3], p[4], 1, 6, 3, 128, 96, 0, 0.125, 0, None) == 2
    ws = ctypes.c_void_p(1 << 20)
    assert L.fa2_backward_gqa(*p[:9], ws, 1 << 30, 1, 8, 3, 128, 64, 0, 0.125, 0, None) == 1
    # the deterministic entry point validates exactly like fa2_backward_gqa
    assert L.fa2_backward_deterministic(*p[:9], ws, 1 << 30, 1, 8, 3, 128, 64, 0, 0.125, 0, None) == 1
    assert L.fa2_backward_deterministic(*p[:9], ws, 16, 1, 8, 2, 128, 64, 0, 0.125, 0, None) == 3
    assert L.fa2_backward_deterministic(*p[:9], ws, 1 << 30, 1, 8, 2, 128, 96, 0, 0.125, 0, None) == 2
    assert L.fa2_backward_deterministic(*p[:9], ws, 1 << 30, 1, 8, 2, 128, 64, 1, 0.125, 0, None) in (2, 4)
    # valid GQA arguments reach CUDA (no device here)
    assert L.fa2_forward_gqa(p[0], p[1], p[2], p[3], p[4], 1, 8, 2, 128, 64, 1, 0.125, 0, None) in (2, 4)


def test_rectangular_and_varlen_validation(L):
    p = FAKE
    cu = ctypes.c_void_p(4096)
    # N_k < 1
    assert L.fa2_forward_ex(p[0], p[1], p[2], p[3], p[4], 1, 2, 2, 128, 0, 64, 0, 0.125, 0, None) == 1
    # valid rectangular arguments reach CUDA
    assert L.fa2_forward_ex(p[0], p[1], p[2], p[3], p[4], 1, 2, 1, 100, 300, 64, 1, 0.125, 0, None) in (2, 4)
    vl = lambda *a: L.fa2_forward_varlen(p[0], p[1], p[2], p[3], p[4], *a)
    assert vl(None, cu, 2, 4, 2, 100, 100, 60, 60, 64, 0, 0.125, 0, None) == 1          # NULL cu_seqlens
    assert vl(ctypes.c_void_p(4097), cu, 2, 4, 2, 100, 100, 60, 60, 64, 0, 0.125, 0, None) == 1   # misaligned
    assert vl(cu, cu, 2, 4, 3, 100, 100, 60, 60, 64, 0, 0.125, 0, None) == 1            # H % H_kv
    assert vl(cu, cu, 2, 4, 2, 0, 100, 60, 60, 64, 0, 0.125, 0, None) == 1              # total_q < 1
    assert vl(cu, cu, 2, 4, 2, 100, 100, 101, 60, 64, 0, 0.125, 0, None) == 1           # max > total
    assert vl(cu, cu, 2, 4, 2, 100, 100, 60, 60, 96, 0, 0.125, 0, None) == 2            # d
    assert vl(cu, cu, 2, 4, 2, 100, 100, 60, 60, 64, 1, 0.125, 0, None) in (2, 4)       # valid
    # varlen workspace: padded rows H * pad128(T_q + 127 B), dq_acc + D + L2 + counters + tile offsets
    B, H, T, d = 3, 4, 1000, 64
    rows = H * (-(-(T + 127 * B) // 128) * 128)
    r16 = lambda x: (x + 15) // 16 * 16
    want = rows * d * 4 + 2 * rows * 4 + r16(rows // 32 * 4) + r16((B + 1) * 4)
    assert L.fa2_backward_varlen_workspace_size(B, H, T, d) == (want + 255) // 256 * 256 + T * H * d * 8
    ws = ctypes.c_void_p(1 << 20)
    bv = lambda nbytes, *a: L.fa2_backward_varlen(*p[:9], cu, cu, ws, nbytes, *a)
    assert bv(want - 1, B, H, 2, T, T, 500, 500, d, 0, 0.125, 0, 0, None) == 3
    assert bv(want, B, H, 2, T, T, 500, 500, d, 0, 0.125, 0, 0, None) in (2, 4)


def test_fp8_validation(L):
    p = FAKE
    assert L.fa2_forward_fp8(p[0], p[1], p[2], p[3], p[4], 1, 2, 2, 128, 64, 0, 0.1, 1.0, 1.0, 1.0, None) == 2   # d
    assert L.fa2_forward_fp8(p[0], p[1], p[2], p[3], p[4], 1, 2, 2, 128, 128, 0, 0.1, 0.0, 1.0, 1.0, None) == 1  # descale
    assert L.fa2_forward_fp8(p[0], p[1], p[2], p[3], p[4], 1, 2, 2, 128, 128, 0, 0.1, 1.0, float("inf"), 1.0, None) == 1
    assert L.fa2_forward_fp8(p[0], p[1], p[2], p[3], p[4], 1, 3, 2, 128, 128, 0, 0.1, 1.0, 1.0, 1.0, None) == 1  # H % H_kv
    assert L.fa2_forward_fp8(p[0], p[1], p[2], p[3], p[4], 1, 2, 1, 128, 128, 1, 0.1, 1.0, 1.0, 1.0, None) in (2, 4)
