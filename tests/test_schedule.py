"""CPU tests of the host-side balanced tile schedule (fa2_tile_schedule)
used by the causal square forward and arrival-order backward launches.  The tile work
model here is written independently from the causal skip rule: a forward
tile (two 128-row sub-tiles of a 256-row block) visits, per sub-tile, the key blocks up
to the one holding its last row; a backward key block nb visits the query tiles >= nb."""
import pytest

import paper_2307_08691_b200 as fa2

G = 148


def fwd_work(N, t):
    nmb = -(-N // 256)
    mb = nmb - 1 - t % nmb
    w = 1
    for i in range(2):
        r0 = mb * 256 + i * 128
        if r0 < N:
            last = min(N - 1, r0 + 127)
            w += min(-(-N // 128), last // 128 + 1)
    return w


def bwd_work(N, t, nh):
    nnb = -(-N // 128)
    return (nnb - t % nnb) * nh + 1


@pytest.fixture(scope="module")
def L():
    from paper_2307_08691_b200 import build
    build.build()
    return fa2.lib()


# the paper's sweep shapes: hidden 2048, B = 16k / N; heads = B * H
@pytest.mark.parametrize("N,H", [(512, 16), (2048, 16), (8192, 16), (16384, 16), (1024, 32), (8192, 32),
                                 (4096, 32), (300, 16), (65536, 1)])
@pytest.mark.parametrize("pass_", [0, 1])
def test_schedule_is_a_balanced_permutation(L, N, H, pass_):
    heads = max(1, 16384 // N) * H
    order, start = fa2.tile_schedule(pass_, heads, N, 1, G)
    T = len(order)
    assert T == heads * (-(-N // (256 if pass_ == 0 else 128)))
    # every tile exactly once, CTA ranges contiguous and ordered
    assert sorted(order) == list(range(T))
    assert start[0] == 0 and start[G] == T
    assert all(start[c] <= start[c + 1] for c in range(G))
    work = (lambda t: fwd_work(N, t)) if pass_ == 0 else (lambda t: bwd_work(N, t, 1))
    loads = [sum(work(t) for t in order[start[c]:start[c + 1]]) for c in range(G)]
    mean = sum(work(t) for t in range(T)) / G
    stride = [sum(work(t) for t in range(c, T, G)) for c in range(G)]
    biggest = max(work(t) for t in range(T))
    # greedy longest-first within windows: within one tile of the mean, and never
    # worse than the stride schedule it replaces
    assert max(loads) <= max(mean + biggest, max(stride))
    assert max(loads) <= max(stride)
    if T >= 4 * G:
        assert max(loads) / mean <= 1.10, (max(loads) / mean, max(stride) / mean)


def test_schedule_gqa_backward_weights_heads(L):
    # a backward tile visiting 4 query heads carries 4x the query tiles
    order, start = fa2.tile_schedule(1, 16, 8192, 4, G)
    T = len(order)
    loads = [sum(bwd_work(8192, t, 4) for t in order[start[c]:start[c + 1]]) for c in range(G)]
    mean = sum(bwd_work(8192, t, 4) for t in range(T)) / G
    assert sorted(order) == list(range(T)) and max(loads) / mean <= 1.10


def test_schedule_errors(L):
    with pytest.raises(fa2.FA2Error):
        fa2.tile_schedule(2, 16, 1024, 1, G)
    with pytest.raises(fa2.FA2Error):
        fa2.tile_schedule(0, 16, 1024, 1, 161)
    with pytest.raises(fa2.FA2Error):   # 16 * 65536 / 128 = 8192 fits; twice that does not
        fa2.tile_schedule(1, 32, 65536, 1, G)
