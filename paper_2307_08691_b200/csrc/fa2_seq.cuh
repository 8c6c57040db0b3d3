// Sequence geometry shared by the forward and backward kernels: the fixed-length
// layout [B, H, N, d] (N_q rows for q/o/dO/dQ, N_k rows for k/v/dK/dV) and the
// packed variable-length layout [T, H, d] with per-sequence row offsets
// cu_seqlens (R22, R23).
//
// Tiles are loaded through 3-D TMA views in memory order:
//   fixed:  {d, N, B*heads}   coordinates (c, row, b*heads + head)
//   packed: {d, heads, T}     coordinates (c, head, row)
// so the row coordinate is dimension 1 or 2; both give the same 128-row x 128-B
// swizzled SMEM tile (box {64, 128, 1} or {64, 1, 128}).
#pragma once
#include <type_traits>
#include "sm100_ptx.cuh"

namespace fa2 {

// Balanced static tile schedule (causal, square fixed-length paths of the forward and the
// arrival-order backward).  Causal work tiles differ in length, and the static stride
// schedule (CTA c takes tiles c, c + G, ...) leaves the busiest CTA with 1.15-1.4x the
// mean work at the paper's shapes.  The host assigns tiles greedily (heaviest first, to
// the least-loaded CTA) inside windows of heads whose K/V (forward) or Q/dO (backward)
// fit in L2 together, and passes every CTA's list as a kernel parameter: no device
// memory, no global state on the device.  n == 0: static stride schedule.
constexpr int kSchedMaxTiles = 8192;
constexpr int kSchedMaxCtas = 160;
struct TileSched {
  int n;                               // number of tiles (0: no table)
  uint16_t start[kSchedMaxCtas + 1];   // CTA c's tiles: order[start[c] .. start[c + 1])
  uint16_t order[kSchedMaxTiles];
};
struct NoSched {
  int n;
};
template <bool ON>
using SchedT = typename std::conditional<ON, TileSched, NoSched>::type;

// n-th work tile of this CTA (-1: none left)
template <class S>
FA2_DEVICE int sched_tile(const S& sc, int n, int num_tiles) {
  if constexpr (std::is_same<S, TileSched>::value) {
    if (sc.n > 0) {
      const int i = sc.start[blockIdx.x] + n;
      return i < sc.start[blockIdx.x + 1] ? sc.order[i] : -1;
    }
  }
  const int t = blockIdx.x + n * gridDim.x;
  return t < num_tiles ? t : -1;
}

struct SeqGeom {
  const int* cu_q;     // packed: [B+1] query row offsets (device); nullptr: fixed lengths
  const int* cu_k;     // packed: [B+1] key row offsets
  int Nq, Nk;          // fixed lengths (packed: the maxima, which size the tile grid)
};

// One sequence (batch entry) as a work tile sees it.
struct Seq {
  int bc;    // batch coordinate of the TMA views / stride arithmetic (0 when packed)
  int q0;    // first query row of the sequence in its tensor's row dimension
  int k0;    // first key row
  int nq;    // query rows N_q(b)
  int nk;    // key rows N_k(b)
  int off;   // causal offset N_k - N_q: row i sees key j iff j <= i + off (bottom-right, R22)
};

// GEN ("general geometry") is a compile-time property of the kernel instantiation.
// GEN == false: the square fixed-length layout (N_q == N_k == Nq, causal offset 0),
// whose lengths are kernel parameters (constant-bank operands) -- the benchmark path
// keeps exactly the arithmetic of the square case.  GEN == true: N_q != N_k and/or
// the packed variable-length layout, resolved at run time.
template <bool GEN>
FA2_DEVICE Seq seq_of(const SeqGeom& g, int b) {
  Seq s;
  if constexpr (!GEN) {
    s.bc = b; s.q0 = 0; s.k0 = 0; s.nq = g.Nq; s.nk = g.Nq; s.off = 0;
    return s;
  }
  if (g.cu_q == nullptr) {
    s.bc = b; s.q0 = 0; s.k0 = 0; s.nq = g.Nq; s.nk = g.Nk;
  } else {
    s.bc = 0;
    s.q0 = __ldg(g.cu_q + b);
    s.k0 = __ldg(g.cu_k + b);
    s.nq = __ldg(g.cu_q + b + 1) - s.q0;
    s.nk = __ldg(g.cu_k + b + 1) - s.k0;
  }
  s.off = s.nk - s.nq;
  return s;
}

// Load one 128-row x 64-column box of head `head` (of `heads`), rows [row, row+128).
template <bool GEN>
FA2_DEVICE void tma_load_rows(void* smem_dst, const CUtensorMap* m, uint64_t* bar, const SeqGeom& g, int c, int row,
                              int head, int bc, int heads, uint64_t policy) {
  if (GEN && g.cu_q != nullptr) ptx::tma_load_3d_hint(smem_dst, m, bar, c, head, row, policy);
  else ptx::tma_load_3d_hint(smem_dst, m, bar, c, row, bc * heads + head, policy);
}

}  // namespace fa2
