// FlashAttention-2 backward pass (Alg. 2) for sm_100a.
//
//   fa2_bwd_preprocess : D_i = rowsum(dO o O)_i (Alg. 2 line 4),
//                        L2_i = L_i * log2(e) (padded rows: +inf), zero dQ_acc.
//   fa2_bwd_kernel     : one persistent CTA per SM; a work tile is one key/value
//                        block K_j, V_j of 128 rows (the "column block" worker of
//                        P:489-496); it walks the query blocks i (B_r rows):
//       S^T   = K_j Q_i^T                   tcgen05 SS -> TMEM   (Alg. 2 l.10)
//       dP^T  = V_j dO_i^T                  tcgen05 SS -> TMEM   (l.13)
//       P^T   = exp(S^T - L_i)              (l.11, one thread = one key row)
//       dS^T  = P^T o (dP^T - D_i)          (l.14, D_i broadcast per query row)
//       dV_j += P^T dO_i                    tcgen05 SS, TMEM accumulator (l.12)
//       dK_j += dS^T Q_i                    tcgen05 SS, TMEM accumulator (l.17)
//       dQ_i += dS K_j                      tcgen05 SS -> TMEM -> fp32 TMA
//                                           reduce-add into dQ_acc (l.15-16;
//                                           the atomic add of P:494-496)
//     dK_j, dV_j are written once at the end (l.19); the softmax scale is
//     applied to dK and dQ (dS carries it, R1).
//   fa2_dq_convert     : dQ = cast(dQ_acc).
//
// Orientation: key rows are TMEM lanes (M = 128), query blocks of B_r = 128 rows.
// This file holds the d = 64 kernel (dQ = dS K, M = B_r = 128, TMEM S^T | dP^T | dV
// | dK | dQ | P^T); d = 128 runs fa2_bwd128_kernel (fa2_bwd128_sm100.cuh, dQ^T =
// K^T dS^T over the dP^T columns) or, opt-in, the CTA-pair fa2_bwd_pair_kernel
// (fa2_bwd2_sm100.cuh).
//
// Warp roles (512 threads): warps 0-7 two compute warpgroups (each owns half of
// the query columns of P^T / dS^T); warps 8-11 dQ readout + reduce-add; warp 12
// MMA issuer; warp 13 TMA producer; warps 14-15 idle.
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "fa2_seq.cuh"

namespace fa2 {

constexpr int kBwdThreads = 512;
__host__ __device__ constexpr int bwd_bm(int d) { return d == 128 ? 64 : 128; }

struct BwdMaps {
  CUtensorMap q, k, v, dout, dq_acc;
};

struct BwdParams {
  const float* lse;     // unused by the main kernel (L2 in workspace); kept for reference
  const float* dvec;    // workspace: [acc_rows] D, followed by [acc_rows] L*log2(e)
  void* dk;
  void* dv;
  float* dq_acc;        // fp32 dQ accumulator [acc_rows, D] (padded query rows, RowParams)
  int BH;              // B * H (query heads)
  int H, Hkv, group;    // query heads, key/value heads, H / Hkv (GQA; group == 1 for MHA)
  int num_n_blocks;     // ceil(N / 128)
  int num_tiles;        // BH * num_n_blocks
  float scale;
  float scale_log2;
  unsigned long long* trace;  // optional clock64 trace (CTA 0, first work tile), nullptr in production
  int* dq_sem;          // deterministic mode: one counter per 128-row tile of the padded workspace
  int det_cyclic;       // deterministic schedule (see bwd_q_tile): 1 for the square fixed layout when
                        // num_n_blocks <= gridDim.x
  SeqGeom geom;                  // sequence geometry (fa2_seq.cuh)
  long long k_bs, k_hs, k_rs;    // dK / dV strides in elements: batch, key/value head, row
  long long acc_bs, acc_hs;      // padded workspace rows per batch entry (fixed layout) and per query head
  long long acc_rows;            // rows of dq_acc (and of D, L*log2e) in total
  const int* tile_off;           // packed: [B+1] prefix sums of ceil(N_q(b) / 128); nullptr: fixed layout
  // GQA load balance: the query heads of a key/value group are split over `hsplit` work
  // tiles; with hsplit > 1 the tiles reduce-add fp32 partial dK, dV into dk_acc, dv_acc
  // (same element layout as dk, dv; zeroed beforehand, cast by fa2_dkv_convert).
  int hsplit;
  float* dk_acc;
  float* dv_acc;
};

// A backward work tile: key block nb (128 rows) of key/value head kvh of sequence b,
// visited with query tiles i0 .. i0+nqt-1 of query heads kvh*group + h0 .. + h0+nh-1
// (the whole group unless hsplit > 1).
struct BwdTile {
  int b, kvh, nb;
  Seq sq;
  int nqb;        // query tiles of the sequence, ceil(N_q / 128)
  int i0, nqt;    // first query tile and number of query tiles (per query head)
  int h0, nh;     // query heads of the group handled by this tile
};
FA2_DEVICE void bwd_decode(const BwdParams& p, bool causal, int t, int& bh, int& nb);
// Returns false when the key block lies past the sequence's keys (nothing to do).
// nqt == 0 (no query row sees the block, i.e. N_q == 0): dK = dV = 0 for its rows.
template <bool GEN>
FA2_DEVICE bool bwd_tile(const BwdParams& p, bool causal, int t, BwdTile& w) {
  int bh, nb;
  bwd_decode(p, causal, t, bh, nb);   // bh = (b * Hkv + kvh) * hsplit + split
  const int split = bh % p.hsplit;
  bh /= p.hsplit;
  w.nh = p.group / p.hsplit;
  w.h0 = split * w.nh;
  w.b = bh / p.Hkv;
  w.kvh = bh % p.Hkv;
  w.nb = nb;
  w.sq = seq_of<GEN>(p.geom, w.b);
  if (nb * 128 >= w.sq.nk) return false;
  w.nqb = (w.sq.nq + 127) / 128;
  int i0 = 0;
  if (causal) {   // first query row that sees key nb*128: row >= nb*128 - (N_k - N_q) (R22)
    const int first_row = nb * 128 - w.sq.off;
    i0 = first_row > 0 ? first_row / 128 : 0;
  }
  w.i0 = i0;
  w.nqt = w.nqb > i0 ? w.nqb - i0 : 0;
  return true;
}
// Padded workspace row of query row 0 of (sequence b, query head hq): rows of dq_acc,
// D and L*log2e; every sequence starts at a multiple of 128.
template <bool GEN>
FA2_DEVICE long long bwd_acc_row0(const BwdParams& p, const BwdTile& w, int hq) {
  if (GEN && p.tile_off != nullptr) return hq * p.acc_hs + 128LL * __ldg(p.tile_off + w.b);
  return w.sq.bc * p.acc_bs + hq * p.acc_hs;
}
// dK / dV row `kv_row` (sequence-relative) of the tile's key/value head, in elements
template <bool GEN>
FA2_DEVICE long long bwd_kv_off(const BwdParams& p, const BwdTile& w, int kv_row) {
  if constexpr (!GEN) return (static_cast<long long>(w.b * p.Hkv + w.kvh) * w.sq.nk + kv_row) * p.k_rs;
  return w.sq.bc * p.k_bs + w.kvh * p.k_hs + (w.sq.k0 + kv_row) * p.k_rs;
}

// ---------------------------------------------------------------------------
// Work schedule shared by every warp role of both backward kernels.
//
// A work tile t is (head bh, key block nb), t = bh * num_n_blocks + nb; CTA b takes
// t = b, b + grid, ...  Within a tile the query tiles are visited in steps s = 0 .. nqt-1.
//
// Deterministic mode (P:494-496 accumulate dQ_i with atomics, whose
// order is arbitrary): every dQ tile (query head bhq, query tile i) receives the
// contributions of its key blocks in a FIXED order, enforced by a counter per tile:
// the dQ issuer of key block nb waits until dq_sem[bhq, i] == rank(nb, i), issues its
// fp32 reduce-adds, waits for them to complete, then stores rank + 1.
//   det_cyclic = 1 (num_n_blocks <= grid, so a CTA holds at most one tile of any head,
//   and the grid is a multiple of num_n_blocks so a head's tiles run side by side):
//     non-causal: step s visits i = (nb + s) mod n, causal: i = nb + s; rank = s, i.e.
//     the predecessor of (nb, step s) is (nb + 1, step s - 1): the CTAs of one head wait
//     on one another's previous step only, and no skew accumulates.  Causal work tiles
//     alternate heavy/light key blocks between iterations to balance the CTAs.
//   det_cyclic = 0 (a head spans more than the grid): rank = nb (ascending key blocks);
//     every wait points to a lower work tile, so progress is guaranteed.
// ---------------------------------------------------------------------------
FA2_DEVICE void bwd_decode(const BwdParams& p, bool causal, int t, int& bh, int& nb) {
  bh = t / p.num_n_blocks;
  nb = t % p.num_n_blocks;
  if (causal && p.dq_sem != nullptr && p.det_cyclic && ((t / static_cast<int>(gridDim.x)) & 1))
    nb = p.num_n_blocks - 1 - nb;
}
FA2_DEVICE int bwd_q_tile(const BwdParams& p, bool causal, const BwdTile& w, int s) {
  if (causal) return w.i0 + s;
  if (p.dq_sem != nullptr && p.det_cyclic) return w.nb + s < w.nqb ? w.nb + s : w.nb + s - w.nqb;
  return s;
}
// One counter per dQ tile: dq_sem[bhq * n_q_blocks + i] = number of key blocks whose
// contribution has landed.  The dQ issuer of key block nb spins (acquire) until the
// counter equals its rank, issues the tile's reduce-adds, waits for them to COMPLETE,
// then stores rank + 1 (release).  A blocked issuer holds no pending release, and the
// waits point to (key block + 1, step - 1) in the cyclic schedule or to a lower work
// tile in the ascending one, so the wait graph is acyclic and every CTA progresses.
// (Finer-grained counters per part of a tile, with deferred releases, were measured
// slower: tools/bench_det.py.)
// 4 counters per 128-row dQ tile (the CTA-pair kernel uses one per query half and d half)
FA2_DEVICE int* dq_sem_ptr(const BwdParams& p, long long acc_row0, int i) { return p.dq_sem + (acc_row0 / 128 + i) * 4; }
FA2_DEVICE int dq_rank(const BwdParams& p, int nb, int s) { return p.det_cyclic ? s : nb; }
FA2_DEVICE void dq_sem_wait(const int* sem, int rank) {
  while (ptx::ld_acquire_gpu(sem) != rank) {
  }
  ptx::fence_proxy_async_global();
}
// after the tile's reduce-adds were committed (one or more bulk groups)
FA2_DEVICE void dq_sem_release(int* sem, int rank) {
  ptx::bulk_wait<0>();
  ptx::fence_proxy_async_global();
  ptx::st_release_gpu(sem, rank + 1);
}

// Debug timeline: trace[ev * 64 + h] = clock64() for CTA 0's first 64 query tiles.
#define FA2_BTRACE(ev, h)                                                                       \
  do {                                                                                          \
    if (p.trace != nullptr && blockIdx.x == 0 && (h) < 64) p.trace[(ev) * 64 + (h)] = clock64(); \
  } while (0)

// ---------------------------------------------------------------------------
// Row geometry of the backward workspace, shared by preprocess and dQ convert.
// Workspace rows are "padded query rows": fixed layout (b*H + h) * N_pad + r; packed
// layout h * acc_hs + 128 * tile_off[b] + r (every sequence starts at a multiple of
// 128 so that whole 128-row query tiles address contiguous, aligned rows).
// ---------------------------------------------------------------------------
struct RowParams {
  const void* o;          // q-layout tensors: O and dO (preprocess), dQ (convert)
  const void* dout;
  void* dq;
  const float* lse;       // fixed [B,H,N_q]; packed [H,T_q]
  float* dvec;            // [acc_rows] D
  float* lse2;            // [acc_rows] L * log2(e) (+inf on padding rows and rows that saw no key)
  float* dq_acc;          // [acc_rows, D] fp32
  int* dq_sem;            // [acc_rows / 128] deterministic-mode counters (or nullptr)
  int B, H, Nq;           // Nq: fixed query length
  const int* cu_q;        // packed: [B+1]; nullptr for the fixed layout
  const int* tile_off;    // packed: [B+1] prefix sums of ceil(N_q(b) / 128)
  long long acc_hs;       // fixed: N_pad (rows per (b, h)); packed: rows per query head
  long long acc_rows;     // total workspace rows
  long long o_bs, o_hs, o_rs, l_bs, l_hs;   // strides (elements) of the q layout and of L
};

// Padded workspace row R -> element offsets of that query row in the q layout (O, dO)
// and in L; false for padding rows.  32-bit index arithmetic: the host guarantees
// acc_rows < 2^31.  Fixed layout: R = bh * N_pad + r with bh = b*H + h, so the q-layout
// offset is bh * N_q * d + r * d and the L offset bh * N_q + r.
FA2_DEVICE bool acc_row_ref(const RowParams& p, long long R, long long& q_off, long long& l_off) {
  const unsigned hs = static_cast<unsigned>(p.acc_hs), Ru = static_cast<unsigned>(R);
  const unsigned hd = Ru / hs, pr = Ru - hd * hs;   // fixed: (b*H + h, r); packed: (h, padded row)
  if (p.cu_q == nullptr) {
    if (pr >= static_cast<unsigned>(p.Nq)) return false;
    q_off = static_cast<long long>(hd) * p.o_hs + static_cast<long long>(pr) * p.o_rs;
    l_off = static_cast<long long>(hd) * p.l_hs + pr;
    return true;
  }
  if (pr >= 128u * static_cast<unsigned>(__ldg(p.tile_off + p.B))) return false;
  int lo = 0, hi = p.B;   // largest b with 128 * tile_off[b] <= pr (skips empty sequences)
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (128u * static_cast<unsigned>(__ldg(p.tile_off + mid)) <= pr) lo = mid; else hi = mid;
  }
  const int q0 = __ldg(p.cu_q + lo);
  const int r = static_cast<int>(pr - 128u * static_cast<unsigned>(__ldg(p.tile_off + lo)));
  if (r >= __ldg(p.cu_q + lo + 1) - q0) return false;
  q_off = static_cast<long long>(hd) * p.o_hs + static_cast<long long>(q0 + r) * p.o_rs;
  l_off = static_cast<long long>(hd) * p.l_hs + q0 + r;
  return true;
}

// packed layout: tile_off[b] = sum_{b' < b} ceil(N_q(b') / 128), one block
__global__ void __launch_bounds__(1024) fa2_tile_prefix(const int* __restrict__ cu_q, int B, int* __restrict__ tile_off) {
  __shared__ int part[1024];
  const int per = (B + 1023) / 1024;
  const int b0 = threadIdx.x * per, b1 = min(B, b0 + per);
  int sum = 0;
  for (int b = b0; b < b1; ++b) sum += (cu_q[b + 1] - cu_q[b] + 127) / 128;
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {   // inclusive Hillis-Steele scan
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x == 0 ? 0 : part[threadIdx.x - 1];
  for (int b = b0; b < b1; ++b) {
    tile_off[b] = run;
    run += (cu_q[b + 1] - cu_q[b] + 127) / 128;
  }
  if (threadIdx.x == 1023) tile_off[B] = part[1023];
}

// ---------------------------------------------------------------------------
// Preprocess: one warp per padded workspace row R.
//   dvec[R] = sum_c dO[row, c] * O[row, c]     (real rows)       else 0
//   lse2[R] = L[row] * log2(e)                 (real rows, finite L; +inf otherwise:
//             padding rows and rows that saw no key, R23, so P = 0 there)
//   dq_acc[R, :] = 0 ; dq_sem[R / 128] = 0 at the first row of a tile (deterministic mode)
// fa2_backward_preprocess uses it with lse2 == dq_acc == nullptr and N_pad == N_q.
// ---------------------------------------------------------------------------
template <int D, bool BF16>
__global__ void __launch_bounds__(256) fa2_bwd_preprocess(const RowParams p) {
  // D / 8 threads per padded workspace row, 16-byte loads of O and dO (8 elements each), the
  // row sum reduced over the row's lanes: enough bytes in flight per SM for HBM (one warp
  // per row with 4-8 byte loads ran at ~2.7 TB/s)
  constexpr int TPR = D / 8;
  const long long gt = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  const long long R = gt / TPR;
  const int sub = static_cast<int>(gt % TPR);
  const bool in = R < p.acc_rows;
  long long q_off = 0, l_off = 0;
  const bool real = in && acc_row_ref(p, R, q_off, l_off);
  float acc = 0.f;
  if (real) {
    const uint4 a = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.o) + q_off + sub * 8);
    const uint4 c = *reinterpret_cast<const uint4*>(reinterpret_cast<const uint16_t*>(p.dout) + q_off + sub * 8);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = ptx::unpack2<BF16>(av[e]), y = ptx::unpack2<BF16>(cv[e]);
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
  }
#pragma unroll
  for (int off = TPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (!in) return;
  if (sub == 0) {
    p.dvec[R] = acc;
    if (p.lse2 != nullptr) {
      const float l = real ? p.lse[l_off] : INFINITY;
      p.lse2[R] = l == -INFINITY ? INFINITY : l * 1.4426950408889634f;
    }
    if (p.dq_sem != nullptr && R % 32 == 0) p.dq_sem[R / 32] = 0;   // 4 counters per 128-row tile
  }
  if (p.dq_acc != nullptr) {
    float4* z = reinterpret_cast<float4*>(p.dq_acc + R * D + sub * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// dQ = cast(dq_acc) for every real query row: one thread per 8 elements of the q layout
// (fixed: [B,H,N_q,D] in order; packed: [T_q,H,D] in order).
template <int D, bool BF16>
__global__ void __launch_bounds__(256) fa2_dq_convert(const RowParams p, long long rows_out) {
  const long long i8 = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;  // index of 8-element group
  if (i8 >= rows_out * (D / 8)) return;
  const long long row = i8 / (D / 8);
  const int c = static_cast<int>(i8 % (D / 8)) * 8;
  long long R;
  if (p.cu_q == nullptr) {            // row = (b*H + h)*N_q + r   (rows_out < 2^31, host-checked)
    const unsigned ru = static_cast<unsigned>(row), nq = static_cast<unsigned>(p.Nq);
    const unsigned bh = ru / nq;
    R = static_cast<long long>(bh) * p.acc_hs + (ru - bh * nq);
  } else {                            // row = t*H + h
    const unsigned ru = static_cast<unsigned>(row), hh = static_cast<unsigned>(p.H);
    const int t = static_cast<int>(ru / hh), h = static_cast<int>(ru - (ru / hh) * hh);
    int lo = 0, hi = p.B;             // the sequence b with cu_q[b] <= t < cu_q[b+1] (largest such b)
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (__ldg(p.cu_q + mid) <= t) lo = mid; else hi = mid;
    }
    R = h * p.acc_hs + 128LL * __ldg(p.tile_off + lo) + (t - __ldg(p.cu_q + lo));
  }
  const float4* src = reinterpret_cast<const float4*>(p.dq_acc + R * D + c);
  const float4 a = src[0], b = src[1];
  uint4 out;
  out.x = ptx::pack2<BF16>(a.x, a.y);
  out.y = ptx::pack2<BF16>(a.z, a.w);
  out.z = ptx::pack2<BF16>(b.x, b.y);
  out.w = ptx::pack2<BF16>(b.z, b.w);
  reinterpret_cast<uint4*>(p.dq)[i8] = out;
}

// dQ = cast(dq_acc) for the d = 128 kernel's chunked accumulator (FA2_BWD_DQ_LSU): inside each
// 128-row tile of the padded workspace, element (q, c) sits at float (q / 4) * 512 + c * 4 + q % 4
// (the layout its register-direct red.global.add.v4 writes).  One thread per 4 workspace rows
// x 8 columns: eight float4 loads of 128 contiguous bytes, four 16-byte stores.
template <bool BF16>
__global__ void __launch_bounds__(256) fa2_dq_convert_chunked(const RowParams p) {
  constexpr int D = 128;
  const long long t = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  if (t >= (p.acc_rows / 4) * (D / 8)) return;
  const long long R0 = (t / (D / 8)) * 4;
  const int c = static_cast<int>(t % (D / 8)) * 8;
  const float4* src = reinterpret_cast<const float4*>(p.dq_acc + (R0 / 128) * (128 * D) + ((R0 % 128) / 4) * (4 * D)) + c;
  float4 f[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = src[k];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    long long q_off = 0, l_off = 0;
    if (!acc_row_ref(p, R0 + j, q_off, l_off)) continue;
    float e[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) e[k] = j == 0 ? f[k].x : j == 1 ? f[k].y : j == 2 ? f[k].z : f[k].w;
    uint4 out;
    out.x = ptx::pack2<BF16>(e[0], e[1]);
    out.y = ptx::pack2<BF16>(e[2], e[3]);
    out.z = ptx::pack2<BF16>(e[4], e[5]);
    out.w = ptx::pack2<BF16>(e[6], e[7]);
    *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.dq) + q_off + c) = out;
  }
}

// GQA split: dK, dV = cast(dk_acc, dv_acc), n8 groups of 8 elements each (same layouts)
template <bool BF16>
__global__ void __launch_bounds__(256)
fa2_dkv_convert(const float* __restrict__ dk_acc, const float* __restrict__ dv_acc, void* __restrict__ dk,
                void* __restrict__ dv, long long n8) {
  const long long i8 = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  if (i8 >= 2 * n8) return;
  const bool is_v = i8 >= n8;
  const long long j = is_v ? i8 - n8 : i8;
  const float4* src = reinterpret_cast<const float4*>((is_v ? dv_acc : dk_acc) + j * 8);
  const float4 a = src[0], b = src[1];
  uint4 out;
  out.x = ptx::pack2<BF16>(a.x, a.y);
  out.y = ptx::pack2<BF16>(a.z, a.w);
  out.z = ptx::pack2<BF16>(b.x, b.y);
  out.w = ptx::pack2<BF16>(b.z, b.w);
  reinterpret_cast<uint4*>(is_v ? dv : dk)[j] = out;
}

template <int D>
struct BwdSmem {
  static constexpr int BM = bwd_bm(D);
  static constexpr bool DST_TMEM = (D == 128);    // dS^T also kept in TMEM (A operand of the dK MMA)
  static constexpr int KV_TILE = 128 * D * 2;     // K_j or V_j
  static constexpr int Q_TILE = BM * D * 2;       // Q_i or dO_i
  static constexpr int Q_SUB = BM * 128;          // one 64-column swizzle box of a Q/dO tile
  static constexpr int DS_TILE = 128 * BM * 2;    // dS^T (bf16), B operand of the dQ MMA
  static constexpr int DQ_TILE = BM * D * 4;      // fp32 staging for the dQ reduce-add
  static constexpr int STAGES = 3;                // Q_i / dO_i / L_i / D_i ring
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_TILE;
  static constexpr int OFF_Q = OFF_V + KV_TILE;
  static constexpr int OFF_DO = OFF_Q + STAGES * Q_TILE;
  static constexpr int OFF_DST = OFF_DO + STAGES * Q_TILE;
  static constexpr int OFF_DQ = OFF_DST + DS_TILE;
  static constexpr int OFF_VEC = OFF_DQ + DQ_TILE;                 // [STAGES][2][BM] floats: L2, D
  static constexpr int OFF_BAR = OFF_VEC + STAGES * 2 * BM * 4;
  // kv_full kv_empty q_full[S] q_empty[S] s_full s_consumed ds_ready ds_empty dq_full dq_empty dkv_full dkv_empty
  static constexpr int NBAR = 10 + 2 * STAGES;
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

template <int D, bool BF16, bool CAUSAL, bool GEN>
__global__ void __launch_bounds__(kBwdThreads, 1)
fa2_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
               const __grid_constant__ CUtensorMap tm_dq, const BwdParams p,
               const __grid_constant__ SchedT<CAUSAL && !GEN> sched) {
  using L = BwdSmem<D>;
  constexpr int BM = L::BM;
  constexpr int STAGES = L::STAGES;
  constexpr bool DQT = (D == 128);          // dQ produced transposed
  constexpr bool DST_TMEM = L::DST_TMEM;
  constexpr int NSUB = D / 64;
  constexpr int HALF = BM / 2;               // query columns per compute warpgroup
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sDO = smem + L::OFF_DO;
  uint8_t* sDST = smem + L::OFF_DST;
  uint8_t* sDQ = smem + L::OFF_DQ;
  float* sVec = reinterpret_cast<float*>(smem + L::OFF_VEC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* kv_full = bars + 0;
  uint64_t* kv_empty = bars + 1;
  uint64_t* q_full = bars + 2;              // [STAGES]
  uint64_t* q_empty = q_full + STAGES;      // [STAGES]
  uint64_t* s_full = q_empty + STAGES;
  uint64_t* s_consumed = s_full + 1;
  uint64_t* ds_ready = s_full + 2;
  uint64_t* ds_empty = s_full + 3;
  uint64_t* dq_full = s_full + 4;
  uint64_t* dq_empty = s_full + 5;
  uint64_t* dkv_full = s_full + 6;
  uint64_t* dkv_empty = s_full + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(kv_empty, 1);
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&q_full[s], 1); ptx::mbar_init(&q_empty[s], 1); }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(s_consumed, 8);
    ptx::mbar_init(ds_ready, 8);
    ptx::mbar_init(ds_empty, 1);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_empty, 4);
    ptx::mbar_init(dkv_full, 1);
    ptx::mbar_init(dkv_empty, 8);
    ptx::fence_mbar_init();
  }
  if (warp == 13 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q); ptx::tma_prefetch_desc(&tm_k); ptx::tma_prefetch_desc(&tm_v);
    ptx::tma_prefetch_desc(&tm_do); ptx::tma_prefetch_desc(&tm_dq);
  }
  if (warp == 0) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns.  d=128 (BM=64): S^T 0, dP^T 64, dV 128, dK 256, dQ^T 384, P^T 448, dS^T 480 (= 512)
  //                d=64 (BM=128): S^T 0, dP^T 128, dV 256, dK 320, dQ 384, P^T 448 (= 512)
  constexpr uint32_t T_ST = 0, T_DPT = BM, T_DV = 2 * BM, T_DK = 2 * BM + D, T_DQ = 2 * BM + 2 * D;
  constexpr uint32_t T_PT = T_DQ + 64, T_DST = T_PT + BM / 2;
  static_assert(T_PT + BM / 2 + (DST_TMEM ? BM / 2 : 0) <= 512, "TMEM budget");

  static_assert(BM == 128, "query tiles of 128 rows (bwd_tile / bwd_q_tile assume B_r == B_c)");
  const float* gD = p.dvec;
  const float* gL2 = p.dvec + p.acc_rows;

  if (warp < 8) {
    // ====================== compute warpgroups: P^T, dS^T ======================
    ptx::setmaxnreg_inc<144>();   // 144*384 + 80*128 == 128*512 (compute + dQ warpgroups / control warps)
    const int wg = warp / 4;
    const int r = threadIdx.x % 128;                   // key row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t sVec_a = ptx::smem_u32(sVec), sDST_a = ptx::smem_u32(sDST);
    uint32_t g = 0;          // global query-tile counter
    int it = 0;
    for (int n_ = 0, t; (t = sched_tile(sched, n_, p.num_tiles)) >= 0; ++n_) {
      BwdTile w;
      if (!bwd_tile<GEN>(p, CAUSAL, t, w)) continue;
      const int nb = w.nb, nqt = w.nqt, nk = w.sq.nk, off = w.sq.off;
      const int kv_row = nb * 128 + r;
      if (nqt == 0) {   // no query row sees this key block (N_q == 0): dV = dK = 0
        if (p.hsplit == 1 && kv_row < nk) {   // (split: the zeroed fp32 accumulators already hold 0)
          uint4* z = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(wg == 0 ? p.dv : p.dk) + bwd_kv_off<GEN>(p, w, kv_row) * 2);
          for (int e = 0; e < D / 8; ++e) z[e] = make_uint4(0u, 0u, 0u, 0u);
        }
        continue;
      }
      for (int x = 0; x < nqt * w.nh; ++x, ++g) {
        const int i = bwd_q_tile(p, CAUSAL, w, x % nqt);   // query tile (of query head kvh*group + x/nqt)
        const int slot = g % STAGES;
        ptx::mbar_wait(&q_full[slot], (g / STAGES) & 1);
        ptx::mbar_wait(s_full, g & 1);
        if (threadIdx.x == 0) FA2_BTRACE(0, g);
        ptx::tc_fence_after();
        const uint32_t vL2 = sVec_a + slot * 2 * BM * 4;     // L_i * log2(e) for the BM query rows
        const uint32_t vD = vL2 + BM * 4;                     // D_i
        // causal tiles crossing the (bottom-right aligned, R22) diagonal and the ragged key tail; query
        // rows past N_q need no mask (L*log2e = +inf in the workspace -> P = 0)
        const bool need_mask = (CAUSAL && nb * 128 + 127 > i * BM + off) || (nb * 128 + 128 > nk);
        uint32_t pk[HALF / 2], dk[HALF / 2];
#pragma unroll
        for (int ch = 0; ch < HALF / 32; ++ch) {
          const int c0 = wg * HALF + ch * 32;          // first query column of this chunk
          uint32_t sv[32], dpv[32];
          ptx::tmem_ld_x32(tmem + lane_base + T_ST + c0, sv);
          ptx::tmem_ld_x32(tmem + lane_base + T_DPT + c0, dpv);
          ptx::tmem_wait_ld();
          if (ch == HALF / 32 - 1) {
            // every TMEM read of S^T / dP^T for this tile is done: the MMA warp may overwrite them
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(s_consumed);
            if (threadIdx.x == 0) FA2_BTRACE(1, g);
          }
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            float pp[2], dd[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = c0 + 2 * e + h;
              float pv = ptx::ex2(fmaf(__uint_as_float(sv[2 * e + h]), p.scale_log2, -ptx::lds_f32(vL2 + c * 4)));
              if (need_mask) {
                const int q_row = i * BM + c;
                if ((CAUSAL && kv_row > q_row + off) || kv_row >= nk) pv = 0.f;
              }
              pp[h] = pv;
              dd[h] = pv * (__uint_as_float(dpv[2 * e + h]) - ptx::lds_f32(vD + c * 4));
            }
            pk[ch * 16 + e] = ptx::pack2<BF16>(pp[0], pp[1]);
            dk[ch * 16 + e] = ptx::pack2<BF16>(dd[0], dd[1]);
          }
        }
        // the previous tile's dV/dK/dQ MMAs must have finished reading P^T / dS^T
        if (g > 0) ptx::mbar_wait(ds_empty, (g - 1) & 1);
        if (threadIdx.x == 0) FA2_BTRACE(2, g);
        ptx::tc_fence_after();
#pragma unroll
        for (int ch = 0; ch < HALF / 32; ++ch) {
          const int c0 = wg * HALF + ch * 32;
          // P^T (and dS^T) rows into TMEM: A operands of the dV (dK) MMAs, 2 values per column
          ptx::tmem_st_x16(tmem + lane_base + T_PT + c0 / 2, pk + ch * 16);
          if constexpr (DST_TMEM) ptx::tmem_st_x16(tmem + lane_base + T_DST + c0 / 2, dk + ch * 16);
          // dS^T row into SMEM (B operand of the dQ MMA): 32 columns = 4 x 16-B chunks, 128-B swizzle
          const int region = c0 / 64;                    // 64-column (128-B) region
          const int cc0 = (c0 % 64) / 8;                 // first 16-B chunk within the 128-B row
          const uint32_t roff = region * (128 * 128) + (r / 8) * 1024 + (r % 8) * 128;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const int b = ch * 16 + 4 * q4;
            ptx::sts_v4(sDST_a + roff + (((cc0 + q4) ^ (r % 8)) * 16), dk[b], dk[b + 1], dk[b + 2], dk[b + 3]);
          }
        }
        ptx::tmem_wait_st();
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ds_ready);
        if (threadIdx.x == 0) FA2_BTRACE(3, g);
      }
      // ---- epilogue: dV_j (warpgroup 0), dK_j * scale (warpgroup 1) ----
      ptx::mbar_wait(dkv_full, it & 1);
      ptx::tc_fence_after();
      if (p.hsplit > 1) {
        // this tile covers part of the group's query heads: fp32 reduce-add of the partial
        // dV / dK (GQA load-balance split; fa2_dkv_convert casts the sums)
        const uint32_t tsrc = tmem + lane_base + (wg == 0 ? T_DV : T_DK);
        const float mul = wg == 0 ? 1.f : p.scale;
        float* acc = (wg == 0 ? p.dv_acc : p.dk_acc) + bwd_kv_off<GEN>(p, w, kv_row);
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld_x32(tsrc + ch * 32, v);
          ptx::tmem_wait_ld();
          if (kv_row < nk) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              ptx::red_add_v4_f32(acc + ch * 32 + 4 * e, __uint_as_float(v[4 * e]) * mul, __uint_as_float(v[4 * e + 1]) * mul,
                                  __uint_as_float(v[4 * e + 2]) * mul, __uint_as_float(v[4 * e + 3]) * mul);
          }
        }
      } else {
        const uint32_t tsrc = tmem + lane_base + (wg == 0 ? T_DV : T_DK);
        const float mul = wg == 0 ? 1.f : p.scale;
        uint8_t* dst = reinterpret_cast<uint8_t*>(wg == 0 ? p.dv : p.dk) + bwd_kv_off<GEN>(p, w, kv_row) * 2;
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld_x32(tsrc + ch * 32, v);
          ptx::tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = ptx::pack2<BF16>(__uint_as_float(v[2 * e]) * mul, __uint_as_float(v[2 * e + 1]) * mul);
          if (kv_row < nk) {
            uint4* o = reinterpret_cast<uint4*>(dst + ch * 64);
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(dkv_empty);
      ++it;
    }
  } else if (warp < 12) {
    // ====================== dQ readout + fp32 reduce-add ======================
    ptx::setmaxnreg_inc<144>();
    const int r = threadIdx.x - 256;                    // 0..127 == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const bool leader = (r == 0);
    const uint32_t sDQ_a = ptx::smem_u32(sDQ);
    uint32_t g = 0;
    for (int n_ = 0, t; (t = sched_tile(sched, n_, p.num_tiles)) >= 0; ++n_) {
      BwdTile w;
      if (!bwd_tile<GEN>(p, CAUSAL, t, w) || w.nqt == 0) continue;
      const int nb = w.nb, nqt = w.nqt;
      for (int x = 0; x < nqt * w.nh; ++x, ++g) {
        const int i = bwd_q_tile(p, CAUSAL, w, x % nqt);
        const long long acc0 = bwd_acc_row0<GEN>(p, w, w.kvh * p.group + w.h0 + x / nqt);   // query head of the group
        ptx::mbar_wait(dq_full, g & 1);
        if (leader) FA2_BTRACE(7, g);
        ptx::tc_fence_after();
        uint32_t v[64];
        ptx::tmem_ld_x32(tmem + lane_base + T_DQ, v);
        ptx::tmem_ld_x32(tmem + lane_base + T_DQ + 32, v + 32);
        ptx::tmem_wait_ld();
        // dQ accumulator in TMEM is free for the next tile's dQ MMA
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(dq_empty);
        // staging buffer free? (the previous reduce-add has finished reading it); in
        // deterministic mode also wait for this key block's turn on dQ tile (bhq, i)
        if (leader) ptx::bulk_wait_read<0>();
        ptx::named_bar_sync(1, 128);
        if constexpr (DQT) {
          // TMEM lane r = head-dim column d; 64 columns = the BM = 64 query rows
          const uint32_t box = sDQ_a + (r / 32) * (BM * 128) + (r % 4) * 4;
#pragma unroll
          for (int q = 0; q < 64; ++q)
            ptx::sts_f32(box + q * 128 + ((((r % 32) / 4) ^ (q % 8)) * 16), __uint_as_float(v[q]) * p.scale);
        } else {
          // TMEM lane r = query row; 64 columns = head dim (two 32-column fp32 boxes)
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t row = sDQ_a + ch * (BM * 128) + r * 128;
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const uint32_t* w = v + ch * 32 + 4 * c4;
              ptx::sts_v4(row + ((c4 ^ (r % 8)) * 16), __float_as_uint(__uint_as_float(w[0]) * p.scale),
                          __float_as_uint(__uint_as_float(w[1]) * p.scale), __float_as_uint(__uint_as_float(w[2]) * p.scale),
                          __float_as_uint(__uint_as_float(w[3]) * p.scale));
            }
          }
        }
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 128);
        if (leader) {
#pragma unroll
          // deterministic mode: wait for this key block's turn on dQ tile (bhq, i)
          if (p.dq_sem != nullptr) dq_sem_wait(dq_sem_ptr(p, acc0, i), dq_rank(p, nb, x % nqt));
#pragma unroll
          for (int b = 0; b < D / 32; ++b)
            ptx::tma_reduce_add_2d(&tm_dq, sDQ + b * (BM * 128), b * 32, static_cast<int>(acc0 + i * BM));
          ptx::bulk_commit();
          if (p.dq_sem != nullptr) dq_sem_release(dq_sem_ptr(p, acc0, i), dq_rank(p, nb, x % nqt));
          FA2_BTRACE(8, g);
        }
      }
    }
    if (leader) ptx::bulk_wait<0>();
  } else if (warp == 12) {
    ptx::setmaxnreg_dec<80>();
    // ================== MMA issuer: whole warp, one elected lane issues ==================
    constexpr uint32_t IDESC_S = ptx::idesc_f16(BF16, 128, BM, false, false);   // S^T, dP^T
    constexpr uint32_t IDESC_G = ptx::idesc_f16(BF16, 128, D, false, true);     // dV, dK
    constexpr uint32_t IDESC_Q = ptx::idesc_f16(BF16, 128, 64, true, true);     // dQ^T or dQ
    // base descriptors; per-MMA descriptors add (byte offset >> 4) to the start-address field
    const uint64_t dK_k = ptx::sw128_desc(ptx::smem_u32(sK), 16, 1024);         // K_j, K-major
    const uint64_t dV_k = ptx::sw128_desc(ptx::smem_u32(sV), 16, 1024);         // V_j, K-major
    const uint64_t dK_mn = ptx::sw128_desc(ptx::smem_u32(sK), 128 * 128, 1024); // K_j, MN-major
    const uint64_t dQ_k = ptx::sw128_desc(ptx::smem_u32(sQ), 16, 1024);
    const uint64_t dO_k = ptx::sw128_desc(ptx::smem_u32(sDO), 16, 1024);
    const uint64_t dQ_mn = ptx::sw128_desc(ptx::smem_u32(sQ), L::Q_SUB, 1024);
    const uint64_t dO_mn = ptx::sw128_desc(ptx::smem_u32(sDO), L::Q_SUB, 1024);
    const uint64_t dS_k = ptx::sw128_desc(ptx::smem_u32(sDST), 16, 1024);
    const uint64_t dS_mn = ptx::sw128_desc(ptx::smem_u32(sDST), 128 * 128, 1024);
    uint32_t g = 0;
    int it = 0;
    uint32_t dkv_uses = 0;
    auto issue_grads = [&](uint32_t h, bool first_in_tile) {
      const uint32_t slot = h % STAGES;
      ptx::mbar_wait(ds_ready, h & 1);
      FA2_BTRACE(5, h);
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        // dV += P^T dO_i (A = P^T in TMEM);  dK += dS^T Q_i (A = dS^T in TMEM or SMEM); B: MN-major [BM x D]
#pragma unroll
        for (int k = 0; k < BM / 16; ++k) {
          const uint32_t boff = (slot * L::Q_TILE + k * 2048) >> 4;
          const uint32_t acc = (!first_in_tile || k > 0) ? 1u : 0u;
          ptx::mma_ts(tmem + T_DV, tmem + T_PT + k * 8, dO_mn + boff, IDESC_G, acc);
          if constexpr (DST_TMEM)
            ptx::mma_ts(tmem + T_DK, tmem + T_DST + k * 8, dQ_mn + boff, IDESC_G, acc);
          else
            ptx::mma_ss(tmem + T_DK, dS_k + (((k / 4) * (128 * 128) + (k % 4) * 32) >> 4), dQ_mn + boff, IDESC_G, acc);
        }
        ptx::mma_commit(&q_empty[slot]);
      }
      __syncwarp();
      FA2_BTRACE(12, h);
      if (h > 0) ptx::mbar_wait(dq_empty, (h - 1) & 1);
      FA2_BTRACE(13, h);
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        // dQ^T = K^T dS^T (A = K_j MN-major, B = dS^T MN-major), or dQ = dS K (A = dS^T as MN-major, B = K_j MN-major)
#pragma unroll
        for (int k = 0; k < 128 / 16; ++k) {
          const uint32_t off = (k * 2048) >> 4;
          if constexpr (DQT) ptx::mma_ss(tmem + T_DQ, dK_mn + off, dS_mn + off, IDESC_Q, k > 0 ? 1u : 0u);
          else ptx::mma_ss(tmem + T_DQ, dS_mn + off, dK_mn + off, IDESC_Q, k > 0 ? 1u : 0u);
        }
        ptx::mma_commit(dq_full);
        ptx::mma_commit(ds_empty);
      }
      __syncwarp();
      FA2_BTRACE(6, h);
    };
    for (int n_ = 0, t; (t = sched_tile(sched, n_, p.num_tiles)) >= 0; ++n_) {
      BwdTile w;
      if (!bwd_tile<GEN>(p, CAUSAL, t, w) || w.nqt == 0) continue;
      ptx::mbar_wait(kv_full, it & 1);
      bool have_prev = false;
      const int cnt = w.nqt * w.nh;   // query tiles of every query head of the tile
      for (int x = 0; x < cnt; ++x, ++g) {
        const uint32_t slot = g % STAGES;
        FA2_BTRACE(10, g);
        ptx::mbar_wait(&q_full[slot], (g / STAGES) & 1);
        FA2_BTRACE(11, g);
        if (g > 0) ptx::mbar_wait(s_consumed, (g - 1) & 1);
        FA2_BTRACE(9, g);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          // S^T = K_j Q_i^T ; dP^T = V_j dO_i^T   (both operands K-major, K = D)
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t akv = ((k / 4) * (128 * 128) + (k % 4) * 32) >> 4;
            const uint32_t aq = (slot * L::Q_TILE + (k / 4) * L::Q_SUB + (k % 4) * 32) >> 4;
            ptx::mma_ss(tmem + T_ST, dK_k + akv, dQ_k + aq, IDESC_S, k > 0 ? 1u : 0u);
            ptx::mma_ss(tmem + T_DPT, dV_k + akv, dO_k + aq, IDESC_S, k > 0 ? 1u : 0u);
          }
          ptx::mma_commit(s_full);
        }
        __syncwarp();
        FA2_BTRACE(4, g);
        if (have_prev) issue_grads(g - 1, x - 1 == 0);
        else if (dkv_uses > 0) {
          // first query tile of this work tile: previous dK/dV must be drained first
          ptx::mbar_wait(dkv_empty, (dkv_uses - 1) & 1);
        }
        have_prev = true;
      }
      issue_grads(g - 1, cnt - 1 == 0);
      ++dkv_uses;
      if (ptx::elect_one()) {
        ptx::mma_commit(dkv_full);
        ptx::mma_commit(kv_empty);
      }
      __syncwarp();
      ++it;
    }
  } else if (warp == 13) {
    ptx::setmaxnreg_dec<80>();
    // ============================ TMA producer ============================
    if (lane == 0) {
      uint32_t g = 0;
      int it = 0;
      const uint64_t pol_q = ptx::l2_policy_evict_last();
      const uint64_t pol_kv = ptx::l2_policy_evict_first();
      for (int n_ = 0, t; (t = sched_tile(sched, n_, p.num_tiles)) >= 0; ++n_) {
        BwdTile w;
        if (!bwd_tile<GEN>(p, CAUSAL, t, w) || w.nqt == 0) continue;
        const int nb = w.nb, nqt = w.nqt;
        if (it > 0) ptx::mbar_wait(kv_empty, (it - 1) & 1);
        ptx::mbar_arrive_expect_tx(kv_full, 2 * L::KV_TILE);
        for (int s = 0; s < NSUB; ++s) {
          tma_load_rows<GEN>(sK + s * 128 * 128, &tm_k, kv_full, p.geom, s * 64, w.sq.k0 + nb * 128, w.kvh, w.sq.bc, p.Hkv, pol_kv);
          tma_load_rows<GEN>(sV + s * 128 * 128, &tm_v, kv_full, p.geom, s * 64, w.sq.k0 + nb * 128, w.kvh, w.sq.bc, p.Hkv, pol_kv);
        }
        for (int x = 0; x < nqt * w.nh; ++x, ++g) {
          const int i = bwd_q_tile(p, CAUSAL, w, x % nqt), hq = w.kvh * p.group + w.h0 + x / nqt;
          const int slot = g % STAGES;
          if (g >= STAGES) ptx::mbar_wait(&q_empty[slot], ((g / STAGES) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&q_full[slot], 2 * L::Q_TILE + 2 * BM * 4);
          for (int s = 0; s < NSUB; ++s) {
            tma_load_rows<GEN>(sQ + slot * L::Q_TILE + s * L::Q_SUB, &tm_q, &q_full[slot], p.geom, s * 64, w.sq.q0 + i * BM,
                          hq, w.sq.bc, p.H, pol_q);
            tma_load_rows<GEN>(sDO + slot * L::Q_TILE + s * L::Q_SUB, &tm_do, &q_full[slot], p.geom, s * 64,
                          w.sq.q0 + i * BM, hq, w.sq.bc, p.H, pol_q);
          }
          float* vdst = sVec + slot * 2 * BM;
          const long long voff = bwd_acc_row0<GEN>(p, w, hq) + static_cast<long long>(i) * BM;
          ptx::bulk_load_1d(vdst, gL2 + voff, BM * 4, &q_full[slot]);
          ptx::bulk_load_1d(vdst + BM, gD + voff, BM * 4, &q_full[slot]);
        }
        ++it;
      }
    }
  } else {
    ptx::setmaxnreg_dec<80>();   // warps 14-15 idle (complete the control warpgroup)
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 512);
  }
}

}  // namespace fa2
