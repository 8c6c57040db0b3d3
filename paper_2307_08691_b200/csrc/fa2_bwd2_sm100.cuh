// FlashAttention-2 backward (Alg. 2) on a CTA pair (cluster of 2,
// tcgen05 cta_group::2): the d = 128, square fixed-length, arrival-order path.
//
// Why a pair.  On one SM (fa2_bwd128_sm100.cuh) every 128 x 128 tile
// sends 64 KB of fp32 dQ partials to L2, and the chip's L2 fp32 reduction rate (~5.9 TB/s,
// ~20 B/clk/SM; tools/micro/tmaio.cu) then needs >= ~3300 cycles per tile against a
// 2560-cycle MMA floor.  Here a work tile is a 256-row key block split over the pair (CTA r
// owns key rows [256 nb2 + 128 r, +128)), and dQ_i = dS_i K_j contracts over all 256 keys
// in ONE M = 128 cta_group::2 MMA whose output rows are split between the CTAs (CTA r:
// query rows [64 r, 64 r + 64) of the tile, all of d).  Each CTA then reduce-adds 32 KB per
// tile instead of 64 KB; the price is 16 KB of dS sent to the peer CTA per tile.
//
// Per query tile i (128 rows) and query head (all heads of the GQA group),
// every MMA issued by the leader CTA (rank 0):
//   S^T  = K_j Q_i^T     M=256 N=128 K=d   A = own K (SS)       B = own 64 query rows, all d
//   dP^T = V_j dO_i^T    M=256 N=128 K=d   A = own V            B = own 64 dO rows, all d
//   dV  += P^T dO_i      M=256 N=d   K=128 A = P^T (TMEM, TS)   B = all 128 dO rows, own 64 d
//   dK  += dS^T Q_i      M=256 N=d   K=128 A = dS^T (TMEM, TS)  B = all 128 Q rows, own 64 d
//   dQ_i = dS_i K_j      M=128 N=d   K=256 A = dS (own 64 query rows x 256 keys, SMEM)
//                                          B = K (256 keys x own 64 d, SMEM)
// dQ lands in each CTA's TMEM as 64 rows x 128 d folded onto 128 lanes x 64 columns
// (lanes 0-63: d [0,64), lanes 64-127: d [64,128), lane % 64 = query row).
//
// TMEM (512 columns per CTA): S^T [0,128) | dP^T [128,256) | dV [256,384) | dK [384,512).
// P^T overwrites S^T [0,64) (packed pairs), dS^T overwrites dP^T [128,192), dQ lands in
// [192,256) (dP^T columns the dS phase has consumed).
//
// The dS exchange and the dQ reduce-add run on the TMA engine, not the LSU (st.async /
// red.global through the LSU stall the compute warps' own shared-memory traffic behind
// them): the warpgroup holding the peer's query half stages its 16 KB in shared memory and
// one thread bulk-copies it into the peer's A slot (completion bytes on the peer's
// dsx_full); the dQ warps stage 8 KB rounds and bulk reduce-add them.  The dS buffer is
// single: dQ(x) is issued right after dK(x), before anything of step x + 1 needs it.
// MMA issue order (steady state, step x):
//   dK(x) [dS^T(x) in TMEM], dQ(x) [dS(x) in both CTAs' A slots], dV(x+1) [P^T(x+1)],
//   dP^T(x+1) [dQ(x) read out of TMEM], S^T(x+2)
// so the compute warps derive P^T(x+1) while dK(x) / dQ(x) run, and dS^T(x+1) is the only
// phase the chain waits for.
//
// Shared memory per CTA (1024-B aligned boxes of 128-B swizzled rows):
//   K   32 KB  own key rows, d halves 0 | 1               (A of S^T, K-major)
//   V   32 KB  own key rows                               (A of dP^T)
//   Kd  32 KB  K rows of CTA 0 | CTA 1, own d half        (B of dQ, MN-major)
//   QS  16 KB  own 64 query rows, d halves 0 | 1          (B of S^T)
//   QK  16 KB  128 query rows, own d half                 (B of dK, MN-major)
//   DOP 16 KB  own 64 dO rows, d halves 0 | 1             (B of dP^T)
//   DOV 16 KB  128 dO rows, own d half                    (B of dV)
//   DS  32 KB  dS of the own query half: keys of CTA 0 | CTA 1 (A of dQ, MN-major)
//   XS  16 KB  staging of the dS rows the peer needs (bulk-copied into its DS slot)
//   DQ  16 KB  2 x 8 KB fp32 staging of the dQ reduce-add (one per d half)
//   VEC 2 KB   L_i * log2(e), D_i (2 stages)
//
// dQ_acc layout (workspace, fp32): inside every 128-row tile of the padded rows, element
// (q, c) at float ((q / 64) * 32 + c / 4) * 256 + (q % 64) * 4 + c % 4: each CTA's 64 rows
// are one contiguous 32 KB range, a d half of them 16 KB, and the staging rounds copy
// verbatim; fa2_dq_convert_pair casts it back.
//
// Barriers the leader's MMA warp waits on live in the leader: TMA loads of both CTAs
// complete on them (cta_group::2 TMA), warps of both CTAs arrive on them remotely.
// Barriers released by MMAs (s_full, dp_full, dq_full, dkv_full, ds_free, *_empty) are
// signalled in both CTAs by multicast tcgen05.commit.  L_i / D_i are per-CTA (local).
//
// Warp roles (512 threads per CTA): warps 0-7 compute (P^T, dS^T; warpgroup w owns query
// columns [64 w, 64 w + 64)), warps 8-11 dQ read-out + reduce-add, warp 12 MMA issuer
// (leader only), warp 13 TMA producer, warp 14 dS-exchange bookkeeping, warp 15 idle.
#pragma once
#include "fa2_bwd_sm100.cuh"
#include "sm100_pair.cuh"

// FMA-pipe exponential pairs per 16 in the P^T phase (unmasked tiles)
#ifndef FA2_BWD_PAIR_EMU
#define FA2_BWD_PAIR_EMU 4
#endif

namespace fa2 {

struct BwdPairSmem {
  static constexpr int BOX128 = 128 * 128;      // 128 rows x 128 B
  static constexpr int BOX64 = 64 * 128;        // 64 rows x 128 B
  static constexpr int DQ_BUF = 8192;           // one dQ reduce round: 8 KB fp32
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + 2 * BOX128;
  static constexpr int OFF_KD = OFF_V + 2 * BOX128;
  static constexpr int OFF_QS = OFF_KD + 2 * BOX128;
  static constexpr int OFF_QK = OFF_QS + 2 * BOX64;
  static constexpr int OFF_DOP = OFF_QK + BOX128;
  static constexpr int OFF_DOV = OFF_DOP + 2 * BOX64;
  static constexpr int OFF_DS = OFF_DOV + BOX128;      // A0 | A1 (dQ's A operand)
  static constexpr int OFF_XS = OFF_DS + 2 * BOX128;   // outgoing dS rows (staging)
  static constexpr int OFF_DQ = OFF_XS + BOX128;       // [2] dQ staging, one per d half
  static constexpr int OFF_VEC = OFF_DQ + 2 * DQ_BUF;  // [2][2][128] floats: L2, D
  static constexpr int OFF_BAR = OFF_VEC + 2 * 2 * 128 * 4;
  static constexpr int NBAR = 32;
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  // no alignment slack: the dynamic shared window starts 1024-B aligned (checked in the kernel)
  static constexpr int ALLOC = BYTES;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

// A pair work tile: key block nb2 (256 rows) of key/value head kvh of batch b, visited
// with query tiles i0 .. nqb-1 of query heads kvh*group + h0 .. + h0+nh-1 (the whole group
// unless the GQA load balance splits it over hsplit tiles, BwdParams::hsplit).
// nqt < 0: the key block lies past its sequence's keys (varlen: the tile grid is sized by the
// longest sequence) -- no work and no rows; nqt == 0: no query row sees it (N_q == 0) -- dK =
// dV = 0 are written, nothing else runs.
struct PairTile {
  int b, kvh, nb2, i0, nqt, h0, nh;
  Seq sq;
};
template <bool GEN>
FA2_DEVICE PairTile pair_tile(const BwdParams& p, bool causal, int t) {
  PairTile w;
  int bh = t / p.num_n_blocks;   // (b * Hkv + kvh) * hsplit + split
  const int split = bh % p.hsplit;
  bh /= p.hsplit;
  w.nh = p.group / p.hsplit;
  w.h0 = split * w.nh;
  w.nb2 = t % p.num_n_blocks;
  // deterministic cyclic causal: alternate heavy / light key blocks between the grid's rounds
  // (all key blocks of a head run in the same round, so this only permutes them over pairs)
  if (causal && p.dq_sem != nullptr && p.det_cyclic && ((t / static_cast<int>(gridDim.x / 2)) & 1))
    w.nb2 = p.num_n_blocks - 1 - w.nb2;
  w.b = bh / p.Hkv;
  w.kvh = bh % p.Hkv;
  w.sq = seq_of<GEN>(p.geom, w.b);
  const int nqb = (w.sq.nq + 127) / 128;
  int i0 = 0;
  if (causal) {   // first query tile that sees key 256 nb2 (CTA 0's first key): row >= 256 nb2 - off (R22)
    const int first_row = w.nb2 * 256 - w.sq.off;
    i0 = first_row > 0 ? first_row / 128 : 0;
  }
  w.i0 = i0;
  w.nqt = w.nb2 * 256 >= w.sq.nk ? -1 : (nqb > i0 ? nqb - i0 : 0);
  return w;
}
// first padded dQ_acc / L / D row of query head hq of the tile's sequence (RowParams layout)
template <bool GEN>
FA2_DEVICE long long pair_acc_row0(const BwdParams& p, const PairTile& w, int hq) {
  if (GEN && p.tile_off != nullptr) return hq * p.acc_hs + 128LL * __ldg(p.tile_off + w.b);
  return w.sq.bc * p.acc_bs + hq * p.acc_hs;
}
// dK / dV element offset of sequence-relative key row kv_row of the tile's key/value head
template <bool GEN>
FA2_DEVICE long long pair_kv_off(const BwdParams& p, const PairTile& w, int kv_row) {
  if constexpr (!GEN) return (static_cast<long long>(w.b * p.Hkv + w.kvh) * w.sq.nk + kv_row) * 128;
  return w.sq.bc * p.k_bs + w.kvh * p.k_hs + (w.sq.k0 + kv_row) * p.k_rs;
}
// Deterministic mode (R21, §6.4): every dQ half-tile (query head,
// query tile i, query half r, d half) receives the pair key blocks' contributions in a fixed
// order, enforced by its own counter (4 per 128-row tile).  Key blocks are 256 rows, query
// tiles 128, so a head has T_r = 2 T_c2 query tiles.
//   det_cyclic (T_r even and the head's key blocks fit the pair grid, which is then a
//   multiple of them, so they run side by side):
//     non-causal: step s visits query tile i = (2 nb2 + s) mod T_r; tile i is visited by
//     key block nb2 at s = (i - 2 nb2) mod T_r, one of every other step, so rank = s / 2
//     and the predecessor of (nb2, s) is (nb2 + 1, s - 2);
//     causal: i = 2 nb2 + s (from the first tile that sees the block), rank = i / 2 - nb2
//     (descending key blocks), predecessor (nb2 + 1, s - 2).
//     The waits point to a neighbour's earlier step: no skew accumulates.
//   otherwise: i = i0 + s, rank = nb2 (ascending key blocks: every wait points to a lower
//   work tile, so progress is guaranteed).
FA2_DEVICE int pair_q_tile(const BwdParams& p, bool causal, const PairTile& w, int s) {
  if (causal || p.dq_sem == nullptr || !p.det_cyclic) return w.i0 + s;
  const int nqb = w.nqt, i = 2 * w.nb2 + s;   // non-causal: every query tile, nqb even
  return i < nqb ? i : i - nqb;
}
FA2_DEVICE int pair_rank(const BwdParams& p, bool causal, const PairTile& w, int i, int s) {
  if (!p.det_cyclic) return w.nb2;
  return causal ? (i >> 1) - w.nb2 : (s >> 1);
}

// GEN: N_q != N_k and/or the packed variable-length layout (fa2_seq.cuh), resolved per work
// tile; the square fixed-length path keeps its constant lengths.
template <bool BF16, bool CAUSAL, bool GEN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kBwdThreads, 1)
fa2_bwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q64, const __grid_constant__ CUtensorMap tm_q128,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_do64, const __grid_constant__ CUtensorMap tm_do128,
                    const __grid_constant__ CUtensorMap tm_dk, const __grid_constant__ CUtensorMap tm_dv,
                    const BwdParams p, const __grid_constant__ SchedT<CAUSAL && !GEN> sched) {
  using L = BwdPairSmem;
  constexpr int D = 128, BM = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if (ptx::smem_u32(smem) & 1023u) __trap();   // SW128 tiles and descriptors need 1024-B alignment
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sKd = smem + L::OFF_KD;
  uint8_t* sQS = smem + L::OFF_QS;
  uint8_t* sQK = smem + L::OFF_QK;
  uint8_t* sDOP = smem + L::OFF_DOP;
  uint8_t* sDOV = smem + L::OFF_DOV;
  uint8_t* sDS = smem + L::OFF_DS;
  uint8_t* sXS = smem + L::OFF_XS;
  uint8_t* sDQ = smem + L::OFF_DQ;
  float* sVec = reinterpret_cast<float*>(smem + L::OFF_VEC);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  // leader-side (the MMA warp waits; arrivals / tx from both CTAs)
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;
  uint64_t* qk_full = bars + 2;
  uint64_t* dop_full = bars + 3;
  uint64_t* dov_full = bars + 4;
  uint64_t* p_ready = bars + 5;     // 16 arrivals: 8 compute warps x 2 CTAs
  uint64_t* ds_ready = bars + 6;    // 16
  uint64_t* dq_empty = bars + 7;    // 8: 4 dQ warps x 2 CTAs
  uint64_t* dkv_empty = bars + 8;   // 16
  uint64_t* dsx_ready = bars + 9;   // CTA 1's dsx_full completed (relayed by its warp 14)
  // released by the MMAs (multicast commit: both CTAs)
  uint64_t* kv_empty = bars + 10;
  uint64_t* q_empty = bars + 11;
  uint64_t* qk_empty = bars + 12;
  uint64_t* dop_empty = bars + 13;
  uint64_t* dov_empty = bars + 14;
  uint64_t* s_full = bars + 15;
  uint64_t* dp_full = bars + 16;
  uint64_t* dq_full = bars + 17;
  uint64_t* dkv_full = bars + 18;
  uint64_t* ds_free = bars + 19;    // dQ(x) complete: both CTAs' A slots may be rewritten
  // local
  uint64_t* vec_full = bars + 20;   // [2]
  uint64_t* vec_empty = bars + 22;  // [2]
  uint64_t* dsx_full = bars + 24;   // the peer's dS rows have landed in this CTA's A slot (tx bytes)
  uint64_t* xs_full = bars + 25;    // 4: the staging warpgroup's rows are in XS
  uint64_t* xs_empty = bars + 26;   // 1: the bulk copy has read XS
  uint64_t* s_consumed = bars + 27; // (leader) 8: warpgroup 1 of both CTAs has loaded S^T cols [64,128)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = pair::cta_rank();
  const int pair_id = static_cast<int>(pair::cluster_id()), npairs = static_cast<int>(pair::num_clusters());

  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(q_full, 1);
    ptx::mbar_init(qk_full, 1);
    ptx::mbar_init(dop_full, 1);
    ptx::mbar_init(dov_full, 1);
    ptx::mbar_init(p_ready, 16);
    ptx::mbar_init(ds_ready, 16);
    ptx::mbar_init(dq_empty, 8);
    ptx::mbar_init(dkv_empty, 16);
    ptx::mbar_init(dsx_ready, 1);
    ptx::mbar_init(kv_empty, 1);
    ptx::mbar_init(q_empty, 1);
    ptx::mbar_init(qk_empty, 1);
    ptx::mbar_init(dop_empty, 1);
    ptx::mbar_init(dov_empty, 1);
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(dp_full, 1);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dkv_full, 1);
    ptx::mbar_init(ds_free, 1);
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&vec_full[s], 1);
      ptx::mbar_init(&vec_empty[s], 8);
    }
    ptx::mbar_init(dsx_full, 1);
    ptx::mbar_init(xs_full, 4);
    ptx::mbar_init(xs_empty, 1);
    ptx::mbar_init(s_consumed, 8);
    ptx::fence_mbar_init();
  }
  if (warp == 13 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q64); ptx::tma_prefetch_desc(&tm_q128); ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v); ptx::tma_prefetch_desc(&tm_do64); ptx::tma_prefetch_desc(&tm_do128);
  }
  if (warp == 0)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(ptx::smem_u32(tmem_slot)), "r"(512));
  ptx::tc_fence_before();
  pair::cluster_sync();   // barriers initialised and TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t T_S = 0, T_DQ = 64, T_DP = 128, T_DV = 256, T_DK = 384;

  if (warp < 8) {
    // ====================== compute warpgroups: P^T, dS^T ======================
    ptx::setmaxnreg_inc<152>();
    const int wg = warp / 4;
    const int r = threadIdx.x % 128;                   // key row within the CTA's block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t sVec_a = ptx::smem_u32(sVec);
    const int c0 = wg * 64;                             // this warpgroup's 64 query columns
    // dS row r, query columns [c0, c0 + 64) (128-B swizzled MN-major rows) belong to the CTA
    // whose dQ rows they are: the own query half (wg == rank) goes into this CTA's A slot
    // A_rank, the other half is staged in XS and bulk-copied into the peer's A slot A_rank
    const bool own_half = static_cast<uint32_t>(wg) == rank;
    const uint32_t row_off = (r / 8) * 1024 + (r % 8) * 128;
    const uint32_t ds_row = own_half ? ptx::smem_u32(sDS) + rank * L::BOX128 + row_off : ptx::smem_u32(sXS) + row_off;
    const uint32_t pbar = 2 + (warp % 4);   // named barrier of the two warps sharing these TMEM lanes
    const float sl2 = p.scale_log2;
    uint32_t g = 0;
    int it = 0;
    for (int n_ = 0, t; (t = pair::sched_tile_pair(sched, n_, p.num_tiles, pair_id, npairs)) >= 0; ++n_) {
      const PairTile w = pair_tile<GEN>(p, CAUSAL, t);
      if (w.nqt < 0) continue;
      const int kv_row = w.nb2 * 256 + static_cast<int>(rank) * 128 + r;   // sequence-relative
      const int nk = w.sq.nk;
      if (w.nqt == 0) {   // no query row sees this key block (N_q == 0): dV = dK = 0
        if (p.hsplit == 1 && kv_row < nk) {   // (split: the zeroed fp32 accumulators already hold 0)
          uint4* z = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(wg == 0 ? p.dv : p.dk) + pair_kv_off<GEN>(p, w, kv_row) * 2);
          for (int e = 0; e < D / 8; ++e) z[e] = make_uint4(0u, 0u, 0u, 0u);
        }
        continue;
      }
      const int nx = w.nqt * w.nh;
      // debug tile timeline (trace[4096 + (cta * 32 + n) * 8 + k]): start / end globaltimer and
      // clock64, tile index, query-tile steps, SM id
      const bool ttr = p.trace != nullptr && threadIdx.x == 0 && n_ < 32;
      unsigned long long* const trow = ttr ? p.trace + 4096 + (blockIdx.x * 32 + n_) * 8 : nullptr;
      if (ttr) {
        unsigned long long gt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        unsigned sm; asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        trow[0] = gt; trow[1] = clock64(); trow[4] = t; trow[5] = nx; trow[6] = sm;
      }
      for (int x = 0; x < nx; ++x, ++g) {
        const int i = pair_q_tile(p, CAUSAL, w, x % w.nqt);
        const uint32_t slot = g & 1;
        const uint32_t vL2 = sVec_a + slot * 2 * BM * 4 + c0 * 4, vD = vL2 + BM * 4;
        // mask: causal tiles crossing the diagonal and the ragged key tail (query rows past N
        // need none: their L*log2e is +inf, so P = 0)
        const int kv_first = w.nb2 * 256 + static_cast<int>(rank) * 128;
        const bool need_mask = (CAUSAL && kv_first + 127 > i * BM + w.sq.off) || (kv_first + 128 > nk);
        ptx::mbar_wait(&vec_full[slot], (g >> 1) & 1);
        ptx::mbar_wait(s_full, g & 1);
        if (threadIdx.x == 0) FA2_BTRACE(0, g);
        ptx::tc_fence_after();
        // ---- P^T = exp2(S^T * scale*log2e - L*log2e), masked ----
        float pf[64];
        const float2 sl2x2 = make_float2(sl2, sl2);
        auto p_block = [&](auto emu_tag) {
          constexpr int EMU = decltype(emu_tag)::value;
          // both 32-column chunks of S^T in one round trip (tcgen05.wait::ld waits for all)
          uint32_t sva[64];
          ptx::tmem_ld_x32(tmem + lane_base + T_S + c0, sva);
          ptx::tmem_ld_x32(tmem + lane_base + T_S + c0 + 32, sva + 32);
          ptx::tmem_wait_ld();
          if (wg == 1) {   // S^T cols [64,128) are in registers: dQ(x-1) may land there
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) pair::arrive_remote(s_consumed, 0);
          }
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t* sv = sva + ch * 32;
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
              const float4 l4 = ptx::lds_v4f(vL2 + (ch * 32 + e4 * 4) * 4);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = ch * 32 + e4 * 4 + 2 * h;   // column within the warpgroup's 64
                const float2 x2 = ptx::ffma2(make_float2(__uint_as_float(sv[e - ch * 32]), __uint_as_float(sv[e - ch * 32 + 1])),
                                             sl2x2, h == 0 ? make_float2(-l4.x, -l4.y) : make_float2(-l4.z, -l4.w));
                float2 pr;
                if ((e / 2) % 16 < EMU) {
                  pr = ptx::exp2_poly2(x2);
                } else {
                  pr.x = ptx::ex2(x2.x);
                  pr.y = ptx::ex2(x2.y);
                }
                if (!EMU && need_mask) {
                  const int q_row = i * BM + c0 + e;
                  if ((CAUSAL && kv_row > q_row + w.sq.off) || kv_row >= nk) pr.x = 0.f;
                  if ((CAUSAL && kv_row > q_row + 1 + w.sq.off) || kv_row >= nk) pr.y = 0.f;
                }
                pf[e] = pr.x;
                pf[e + 1] = pr.y;
              }
            }
          }
        };
        // rows that see no key (R23) carry L*log2e = +inf: the polynomial would give 2^-125
        // instead of 0, so the general geometry keeps MUFU everywhere
        if (need_mask || GEN) p_block(std::integral_constant<int, 0>{});
        else p_block(std::integral_constant<int, FA2_BWD_PAIR_EMU>{});
        if (threadIdx.x == 0) FA2_BTRACE(15, g);
        {
          // packed P^T, contiguous: query columns [0,64) at TMEM cols [0,32), [64,128) at [32,64)
          // (A operand of dV); warpgroup 1 overwrites S^T columns warpgroup 0 reads, so it waits
          // for its partner warp (same lanes) to have loaded them
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) pk[e] = ptx::pack2<BF16>(pf[2 * e], pf[2 * e + 1]);
          if (wg == 0) ptx::named_bar_arrive(pbar, 64);
          else ptx::named_bar_sync(pbar, 64);
          ptx::tmem_st_x32(tmem + lane_base + T_S + wg * 32, pk);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair::arrive_remote(p_ready, 0);
        if (threadIdx.x == 0) FA2_BTRACE(1, g);
        // ---- dS^T = P^T o (dP^T - D) ----
        ptx::mbar_wait(dp_full, g & 1);
        if (threadIdx.x == 0) FA2_BTRACE(2, g);
        ptx::tc_fence_after();
        uint32_t dk[32];
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          uint32_t dv[32];
          ptx::tmem_ld_x32(tmem + lane_base + T_DP + c0 + ch * 32, dv);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 d4 = ptx::lds_v4f(vD + (ch * 32 + e4 * 4) * 4);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int e = e4 * 4 + 2 * h;
              const float2 t2 = ptx::fadd2(make_float2(__uint_as_float(dv[e]), __uint_as_float(dv[e + 1])),
                                           h == 0 ? make_float2(-d4.x, -d4.y) : make_float2(-d4.z, -d4.w));
              const float2 s2 = ptx::fmul2(make_float2(pf[ch * 32 + e], pf[ch * 32 + e + 1]), t2);
              dk[ch * 16 + e / 2] = ptx::pack2<BF16>(s2.x, s2.y);
            }
          }
        }
        if (threadIdx.x == 0) FA2_BTRACE(11, g);
        // packed dS^T of this warpgroup's 64 query columns over the first 32 of its own dP^T
        // columns (A operand of dK)
        ptx::tmem_st_x32(tmem + lane_base + T_DP + c0, dk);
        // dS rows -> shared memory (A operand of dQ): the own A slot is rewritten once dQ of
        // the previous step has completed; the staging buffer once warp 15's bulk copy of the
        // previous step has read it
        if (own_half) {
          if (g > 0) ptx::mbar_wait(ds_free, (g - 1) & 1);
        } else {
          if (g > 0) ptx::mbar_wait(xs_empty, (g - 1) & 1);
        }
        if (threadIdx.x == 0) FA2_BTRACE(12, g);
#pragma unroll
        for (int q8 = 0; q8 < 8; ++q8)
          ptx::sts_v4(ds_row + ((q8 ^ (r % 8)) * 16), dk[4 * q8], dk[4 * q8 + 1], dk[4 * q8 + 2], dk[4 * q8 + 3]);
        ptx::fence_proxy_async_smem();
        ptx::tmem_wait_st();
        if (threadIdx.x == 0) FA2_BTRACE(13, g);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (!own_half) ptx::mbar_arrive(xs_full);
          pair::arrive_remote(ds_ready, 0);
          ptx::mbar_arrive(&vec_empty[slot]);
        }
        if (threadIdx.x == 0) FA2_BTRACE(3, g);
      }
      // ---- epilogue: dV_j (warpgroup 0), dK_j * scale (warpgroup 1) ----
      if (ttr) trow[7] = clock64();   // debug: epilogue start (before the last MMAs' completion wait)
      ptx::mbar_wait(dkv_full, it & 1);
      ptx::tc_fence_after();
      if (p.hsplit > 1) {
        // this tile covers part of the group's query heads: fp32 reduce-add of the partial
        // dV / dK (fa2_dkv_convert casts the sums)
        const uint32_t tsrc = tmem + lane_base + (wg == 0 ? T_DV : T_DK);
        const float mul = wg == 0 ? 1.f : p.scale;
        float* acc = (wg == 0 ? p.dv_acc : p.dk_acc) + pair_kv_off<GEN>(p, w, kv_row);
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
      } else if (p.geom.cu_q == nullptr) {
        // fixed layout: dV (warpgroup 0), then dK (warpgroup 1), packed into the SW128 boxes of
        // the free own dS slot A_rank (d 0-63) and XS (d 64-127) -- both free once the tile's
        // last dQ completed, which dkv_full implies -- and written by TMA tensor stores (rows
        // past N_k are clipped by the tensor map); 16-byte per-row stores took ~7000 cycles
        const uint32_t tsrc = tmem + lane_base + (wg == 0 ? T_DV : T_DK);
        const float mul = wg == 0 ? 1.f : p.scale;
        uint32_t pk[D / 32][16];
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld_x32(tsrc + ch * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[ch][e] = ptx::pack2<BF16>(__uint_as_float(v[2 * e]) * mul, __uint_as_float(v[2 * e + 1]) * mul);
        }
        // dV / dK are out of TMEM: the next tile's MMAs may overwrite them
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair::arrive_remote(dkv_empty, 0);
        if (wg == 1) ptx::named_bar_sync(7, 256);   // warpgroup 0's stores have read the staging
        const uint32_t st0 = ptx::smem_u32(sDS) + rank * L::BOX128 + r * 128, st1 = ptx::smem_u32(sXS) + r * 128;
#pragma unroll
        for (int c = 0; c < 16; ++c)
          ptx::sts_v4((c < 8 ? st0 : st1) + (((c % 8) ^ (r % 8)) * 16), pk[c / 4][4 * (c % 4)], pk[c / 4][4 * (c % 4) + 1],
                      pk[c / 4][4 * (c % 4) + 2], pk[c / 4][4 * (c % 4) + 3]);
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(wg == 0 ? 6 : 8, 128);
        if (r == 0) {
          const CUtensorMap* m = wg == 0 ? &tm_dv : &tm_dk;
          const int krow = w.sq.k0 + w.nb2 * 256 + static_cast<int>(rank) * 128, z = w.sq.bc * p.Hkv + w.kvh;
          ptx::tma_store_3d(m, sDS + rank * L::BOX128, 0, krow, z);
          ptx::tma_store_3d(m, sXS, 64, krow, z);
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();
        }
        ptx::named_bar_sync(wg == 0 ? 6 : 8, 128);
        if (wg == 0) {
          ptx::named_bar_arrive(7, 256);
          ptx::named_bar_sync(9, 256);   // warpgroup 1's stores have read the staging too
        } else {
          ptx::named_bar_arrive(9, 256);
        }
        if (ttr) {
          unsigned long long gt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          trow[2] = gt; trow[3] = clock64();
        }
        ++it;
        continue;
      } else {
        const uint32_t tsrc = tmem + lane_base + (wg == 0 ? T_DV : T_DK);
        const float mul = wg == 0 ? 1.f : p.scale;
        uint8_t* dst = reinterpret_cast<uint8_t*>(wg == 0 ? p.dv : p.dk) + pair_kv_off<GEN>(p, w, kv_row) * 2;
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld_x32(tsrc + ch * 32, v);
          ptx::tmem_wait_ld();
          uint32_t o16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) o16[e] = ptx::pack2<BF16>(__uint_as_float(v[2 * e]) * mul, __uint_as_float(v[2 * e + 1]) * mul);
          if (kv_row < nk) {
            uint4* o = reinterpret_cast<uint4*>(dst + ch * 64);
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = make_uint4(o16[4 * e], o16[4 * e + 1], o16[4 * e + 2], o16[4 * e + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) pair::arrive_remote(dkv_empty, 0);
      if (ttr) {
        unsigned long long gt; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        trow[2] = gt; trow[3] = clock64();
      }
      ++it;
    }
    if (r == 0) ptx::bulk_wait<0>();   // the dK / dV tensor stores have completed
  } else if (warp < 12) {
    // ====================== dQ read-out + fp32 bulk reduce-add ======================
    // lane L holds query row L % 64 of this CTA's half and d half L / 64 (64 columns); the two
    // warps of a d half stage their 16 KB in two 8 KB rounds ([c/4][64 rows][4] floats, the
    // accumulator's own layout) and one of them bulk reduce-adds each round
    ptx::setmaxnreg_inc<152>();
    const int quarter = warp % 4;
    const int row = (quarter % 2) * 32 + lane;          // query row within this CTA's 64
    const int dh = quarter / 2;                          // d half held by this lane
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const bool issuer = (quarter % 2 == 0) && lane == 0;
    const uint32_t hbar = 11 + dh;                       // the 64 threads of this d half
    uint8_t* const stage = sDQ + dh * L::DQ_BUF;
    const uint32_t stage_a = ptx::smem_u32(stage) + row * 16;
    const bool leader = (threadIdx.x == 256);
    uint32_t g = 0;
    for (int n_ = 0, t; (t = pair::sched_tile_pair(sched, n_, p.num_tiles, pair_id, npairs)) >= 0; ++n_) {
      const PairTile w = pair_tile<GEN>(p, CAUSAL, t);
      if (w.nqt <= 0) continue;
      const int nx = w.nqt * w.nh;
      for (int x = 0; x < nx; ++x, ++g) {
        const int i = pair_q_tile(p, CAUSAL, w, x % w.nqt);
        const int hq = w.kvh * p.group + w.h0 + x / w.nqt;
        const long long acc0 = pair_acc_row0<GEN>(p, w, hq);
        // this CTA's 32 KB of the tile (query rows [64 rank, +64)), this d half's 16 KB
        float* const acc = p.dq_acc + (acc0 + static_cast<long long>(i) * BM) * D + (rank * 32 + dh * 16) * 256;
        // deterministic mode: this d half's counter of the dQ half-tile (see pair_rank)
        int* const sem = p.dq_sem == nullptr ? nullptr : p.dq_sem + (acc0 / 128 + i) * 4 + rank * 2 + dh;
        const int drank = pair_rank(p, CAUSAL, w, i, x % w.nqt);
        ptx::mbar_wait(dq_full, g & 1);
        if (leader) FA2_BTRACE(9, g);
        ptx::tc_fence_after();
        uint32_t v[64];
        ptx::tmem_ld_x32(tmem + lane_base + T_DQ, v);
        ptx::tmem_ld_x32(tmem + lane_base + T_DQ + 32, v + 32);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair::arrive_remote(dq_empty, 0);
        if (leader) FA2_BTRACE(10, g);
        if (sem != nullptr && issuer) dq_sem_wait(sem, drank);   // the previous contribution landed
#pragma unroll
        for (int rd = 0; rd < 2; ++rd) {
          if (issuer) ptx::bulk_wait_read<0>();          // the staging buffer's last round was read
          ptx::named_bar_sync(hbar, 64);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const int j = rd * 32 + j4 * 4;
            ptx::sts_v4(stage_a + j4 * 1024, __float_as_uint(__uint_as_float(v[j]) * p.scale),
                        __float_as_uint(__uint_as_float(v[j + 1]) * p.scale),
                        __float_as_uint(__uint_as_float(v[j + 2]) * p.scale),
                        __float_as_uint(__uint_as_float(v[j + 3]) * p.scale));
          }
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(hbar, 64);
          if (issuer) {
            ptx::bulk_reduce_add_f32(acc + rd * 2048, stage, L::DQ_BUF);
            ptx::bulk_commit();
          }
        }
        // complete, then rank + 1 (deferring the release to the next step measured slower:
        // 773 -> 651 TFLOP/s non-causal, 676 -> 529 causal)
        if (sem != nullptr && issuer) dq_sem_release(sem, drank);
        if (leader) FA2_BTRACE(16, g);
      }
    }
    if (issuer) ptx::bulk_wait<0>();
  } else if (warp == 12) {
    // ================== MMA issuer (leader CTA): whole warp, one elected lane ==================
    ptx::setmaxnreg_dec<56>();   // 12 x 152 + 4 x 56 = 2048 registers per lane slot
    if (rank == 0) {
      constexpr uint32_t IDESC_S = ptx::idesc_f16(BF16, 256, 128, false, false);   // S^T, dP^T
      constexpr uint32_t IDESC_G = ptx::idesc_f16(BF16, 256, D, false, true);      // dV, dK
      constexpr uint32_t IDESC_Q = ptx::idesc_f16(BF16, 128, D, true, true);       // dQ
      // descriptors are rebuilt from the 32-bit shared-window base at every issue (a few
      // integer ops) instead of keeping eight 64-bit values live in this 56-register warp
      const uint32_t sb = ptx::smem_u32(smem);
      auto kmaj = [&](int off) { return ptx::sw128_desc(sb + off, 16, 1024); };
      auto mnmaj = [&](int off) { return ptx::sw128_desc(sb + off, L::BOX128, 1024); };
      // each issue step: wait (whole warp), fence, one elected lane issues + commits
      auto issue_s = [&]() {   // S^T = K Q^T: K = d, 4 steps per 64-column box
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t offa = (k / 4) * L::BOX128 + (k % 4) * 32;
            const uint32_t offb = (k / 4) * L::BOX64 + (k % 4) * 32;
            pair::mma_ss2(tmem + T_S, kmaj(L::OFF_K) + (offa >> 4), kmaj(L::OFF_QS) + (offb >> 4), IDESC_S, k > 0 ? 1u : 0u);
          }
          pair::commit_both(s_full);
          pair::commit_both(q_empty);
        }
        __syncwarp();
      };
      auto issue_dp = [&]() {   // dP^T = V dO^T
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t offa = (k / 4) * L::BOX128 + (k % 4) * 32;
            const uint32_t offb = (k / 4) * L::BOX64 + (k % 4) * 32;
            pair::mma_ss2(tmem + T_DP, kmaj(L::OFF_V) + (offa >> 4), kmaj(L::OFF_DOP) + (offb >> 4), IDESC_S, k > 0 ? 1u : 0u);
          }
          pair::commit_both(dp_full);
          pair::commit_both(dop_empty);
        }
        __syncwarp();
      };
      auto issue_dv = [&](bool acc) {   // dV += P^T dO (A: packed P^T at TMEM cols [0,64))
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BM / 16; ++k)
            pair::mma_ts2(tmem + T_DV, tmem + T_S + k * 8, mnmaj(L::OFF_DOV) + ((k * 2048) >> 4), IDESC_G, (acc || k > 0) ? 1u : 0u);
          pair::commit_both(dov_empty);
        }
        __syncwarp();
      };
      auto issue_dk = [&](bool acc) {   // dK += dS^T Q (A: packed dS^T at TMEM cols [128,160) | [192,224))
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BM / 16; ++k)
            pair::mma_ts2(tmem + T_DK, tmem + T_DP + (k / 4) * 64 + (k % 4) * 8, mnmaj(L::OFF_QK) + ((k * 2048) >> 4), IDESC_G,
                          (acc || k > 0) ? 1u : 0u);
          pair::commit_both(qk_empty);
        }
        __syncwarp();
      };
      // dQ = dS K over the pair's 256 keys into S^T cols [64,128), once the dS rows of both
      // query halves sit in both CTAs' A slots
      auto issue_dq = [&](uint32_t y) {
        ptx::mbar_wait(dsx_full, y & 1);                   // CTA 1's rows landed here
        FA2_BTRACE(21, y);
        pair::wait_cluster(dsx_ready, y & 1);              // CTA 0's rows landed in CTA 1
        FA2_BTRACE(22, y);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll 1   // rolled: sixteen hoisted 64-bit descriptor pairs would not fit the warp's registers
          for (int k = 0; k < 256 / 16; ++k) {
            const uint32_t off = ((k / 8) * L::BOX128 + (k % 8) * 2048) >> 4;
            pair::mma_ss2(tmem + T_DQ, mnmaj(L::OFF_DS) + off, mnmaj(L::OFF_KD) + off, IDESC_Q, k > 0 ? 1u : 0u);
          }
          pair::commit_both(dq_full);
          pair::commit_both(ds_free);
        }
        __syncwarp();
      };
      // Issue order, step x (steady state):
      //   dK(x) [dS^T(x)], dP^T(x+1) [dK(x) read dS^T(x), in order],
      //   dQ(x) [dS(x) in both CTAs' A slots; P(x+1) has loaded S^T cols [64,128)],
      //   dV(x+1) [P^T(x+1)], S^T(x+2) [dQ(x) read out]
      // dQ(x) completes well before the compute warps rewrite the (single) A slots with
      // dS(x+1), and the exchange of dS(x) overlaps dK(x) / dP^T(x+1) and P(x+1).
      uint32_t g = 0;
      int it = 0;
      for (int n_ = 0, t; (t = pair::sched_tile_pair(sched, n_, p.num_tiles, pair_id, npairs)) >= 0; ++n_) {
        const PairTile w = pair_tile<GEN>(p, CAUSAL, t);
        if (w.nqt <= 0) continue;
        const uint32_t n = static_cast<uint32_t>(w.nqt * w.nh);
        const uint32_t g0 = g, end = g0 + n;
        // prologue: S^T(g0), dP^T(g0), dV(g0), S^T(g0+1)
        ptx::mbar_wait(kv_full, it & 1);
        ptx::mbar_wait(q_full, g0 & 1);
        if (g0 > 0) pair::wait_cluster(dq_empty, (g0 - 1) & 1);   // previous tile's last dQ read out
        issue_s();
        ptx::mbar_wait(dop_full, g0 & 1);
        issue_dp();
        if (it > 0) pair::wait_cluster(dkv_empty, (it - 1) & 1);  // previous dK / dV drained
        ptx::mbar_wait(dov_full, g0 & 1);
        pair::wait_cluster(p_ready, g0 & 1);
        issue_dv(false);
        if (g0 + 1 < end) {
          ptx::mbar_wait(q_full, (g0 + 1) & 1);
          issue_s();
        }
        for (uint32_t x = g0; x < end; ++x) {
          pair::wait_cluster(ds_ready, x & 1);
          FA2_BTRACE(7, x);
          ptx::mbar_wait(qk_full, x & 1);
          issue_dk(x > g0);
          if (x + 1 < end) {
            ptx::mbar_wait(dop_full, (x + 1) & 1);
            issue_dp();
            pair::wait_cluster(s_consumed, (x + 1) & 1);
          }
          FA2_BTRACE(8, x);
          // dQ(x) lands where dQ(x-1) was: its read-out was waited for before S^T(x+1) --
          // except at the tile's last step, where no S^T follows
          if (x + 1 == end && x > g0) pair::wait_cluster(dq_empty, (x - 1) & 1);
          issue_dq(x);
          FA2_BTRACE(5, x);
          if (x + 1 < end) {
            ptx::mbar_wait(dov_full, (x + 1) & 1);
            pair::wait_cluster(p_ready, (x + 1) & 1);
            FA2_BTRACE(4, x + 1);
            issue_dv(true);
            if (x + 2 < end) {
              ptx::mbar_wait(q_full, (x + 2) & 1);
              pair::wait_cluster(dq_empty, x & 1);                 // dQ(x) read out of [64,128)
              issue_s();
            }
            FA2_BTRACE(6, x + 1);
          }
        }
        g = end;
        if (ptx::elect_one()) {
          pair::commit_both(dkv_full);
          pair::commit_both(kv_empty);
        }
        __syncwarp();
        ++it;
      }
    }
  } else if (warp == 13) {
    // ============================ TMA producer (both CTAs) ============================
    ptx::setmaxnreg_dec<56>();
    if (lane == 0) {
      const float* gD = p.dvec;
      const float* gL2 = p.dvec + p.acc_rows;
      const uint64_t pol_q = ptx::l2_policy_evict_last();
      const uint64_t pol_kv = ptx::l2_policy_evict_first();
      const int ro = static_cast<int>(rank);
      // rows [row, row + box) of head `head` (of `heads`) at column c, in this tile's sequence:
      // fixed layout {d, N, B*heads}, packed {d, heads, T} (fa2_seq.cuh tma_load_rows)
      auto load = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c, int row, int head, int heads,
                      const Seq& sq, uint64_t pol) {
        if (GEN && p.geom.cu_q != nullptr) pair::tma_load_pair(dst, m, bar, c, head, row, pol);
        else pair::tma_load_pair(dst, m, bar, c, row, sq.bc * heads + head, pol);
      };
      uint32_t g = 0;
      int it = 0;
      for (int n_ = 0, t; (t = pair::sched_tile_pair(sched, n_, p.num_tiles, pair_id, npairs)) >= 0; ++n_) {
        const PairTile w = pair_tile<GEN>(p, CAUSAL, t);
        if (w.nqt <= 0) continue;
        if (it > 0) ptx::mbar_wait(kv_empty, (it - 1) & 1);
        ++it;
        if (rank == 0) ptx::mbar_arrive_expect_tx(kv_full, 2 * 6 * L::BOX128);
        const int k0 = w.sq.k0 + w.nb2 * 256;
        for (int s = 0; s < 2; ++s) {
          load(sK + s * L::BOX128, &tm_k, kv_full, s * 64, k0 + ro * 128, w.kvh, p.Hkv, w.sq, pol_kv);
          load(sV + s * L::BOX128, &tm_v, kv_full, s * 64, k0 + ro * 128, w.kvh, p.Hkv, w.sq, pol_kv);
          load(sKd + s * L::BOX128, &tm_k, kv_full, ro * 64, k0 + s * 128, w.kvh, p.Hkv, w.sq, pol_kv);
        }
        const int nx = w.nqt * w.nh;
        for (int x = 0; x < nx; ++x, ++g) {
          const int i = pair_q_tile(p, CAUSAL, w, x % w.nqt);
          const int hq = w.kvh * p.group + w.h0 + x / w.nqt;
          const int q0 = w.sq.q0 + i * BM;
          const uint32_t slot = g & 1;
          // L_i * log2(e), D_i: this CTA's own copy (local barrier)
          if (g >= 2) ptx::mbar_wait(&vec_empty[slot], ((g >> 1) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&vec_full[slot], 2 * BM * 4);
          const long long voff = pair_acc_row0<GEN>(p, w, hq) + static_cast<long long>(i) * BM;
          ptx::bulk_load_1d(sVec + slot * 2 * BM, gL2 + voff, BM * 4, &vec_full[slot]);
          ptx::bulk_load_1d(sVec + slot * 2 * BM + BM, gD + voff, BM * 4, &vec_full[slot]);
          // Q_i rows of this CTA's query half, all d (released after S^T(i))
          if (g >= 1) ptx::mbar_wait(q_empty, (g - 1) & 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(q_full, 2 * 2 * L::BOX64);
          for (int s = 0; s < 2; ++s) load(sQS + s * L::BOX64, &tm_q64, q_full, s * 64, q0 + ro * 64, hq, p.H, w.sq, pol_q);
          // dO_i rows of this CTA's query half, all d (released after dP^T(i))
          if (g >= 1) ptx::mbar_wait(dop_empty, (g - 1) & 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(dop_full, 2 * 2 * L::BOX64);
          for (int s = 0; s < 2; ++s) load(sDOP + s * L::BOX64, &tm_do64, dop_full, s * 64, q0 + ro * 64, hq, p.H, w.sq, pol_q);
          // dO_i all rows, this CTA's d half (released after dV(i))
          if (g >= 1) ptx::mbar_wait(dov_empty, (g - 1) & 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(dov_full, 2 * L::BOX128);
          load(sDOV, &tm_do128, dov_full, ro * 64, q0, hq, p.H, w.sq, pol_q);
          // Q_i all rows, this CTA's d half (released after dK(i))
          if (g >= 1) ptx::mbar_wait(qk_empty, (g - 1) & 1);
          if (rank == 0) ptx::mbar_arrive_expect_tx(qk_full, 2 * L::BOX128);
          load(sQK, &tm_q128, qk_full, ro * 64, q0, hq, p.H, w.sq, pol_q);
        }
      }
    }
  } else if (warp == 14) {
    // ============ dS exchange bookkeeping (both CTAs) ============
    // each step the peer bulk-copies 16 KB into this CTA's A slot, completing on dsx_full;
    // CTA 1 relays its completion to the leader (whose MMA warp waits on local barriers)
    ptx::setmaxnreg_dec<56>();
    if (lane == 0) {
      uint32_t g = 0;
      for (int n_ = 0, t; (t = pair::sched_tile_pair(sched, n_, p.num_tiles, pair_id, npairs)) >= 0; ++n_) {
        const PairTile w = pair_tile<GEN>(p, CAUSAL, t);
        const int nx = w.nqt > 0 ? w.nqt * w.nh : 0;
        for (int x = 0; x < nx; ++x, ++g) {
          ptx::mbar_arrive_expect_tx(dsx_full, L::BOX128);
          ptx::mbar_wait(dsx_full, g & 1);
          FA2_BTRACE(20, g);
          if (rank == 1) pair::arrive_remote(dsx_ready, 0);
        }
      }
    }
  } else {
    // ============ warp 15: dS exchange issuer (both CTAs) ============
    // bulk-copies the staged rows (own keys, the peer's query half) into the peer's A slot
    // A_rank once the peer's dQ of the previous step has released it (ds_free, multicast)
    ptx::setmaxnreg_dec<56>();
    if (lane == 0) {
      const uint32_t peer = rank ^ 1u;
      const uint32_t peer_slot = pair::map_cta(ptx::smem_u32(sDS) + rank * L::BOX128, peer);
      const uint32_t peer_bar = pair::map_cta(ptx::smem_u32(dsx_full), peer);
      uint32_t g = 0;
      for (int n_ = 0, t; (t = pair::sched_tile_pair(sched, n_, p.num_tiles, pair_id, npairs)) >= 0; ++n_) {
        const PairTile w = pair_tile<GEN>(p, CAUSAL, t);
        const int nx = w.nqt > 0 ? w.nqt * w.nh : 0;
        for (int x = 0; x < nx; ++x, ++g) {
          ptx::mbar_wait(xs_full, g & 1);
          FA2_BTRACE(17, g);
          if (g > 0) ptx::mbar_wait(ds_free, (g - 1) & 1);
          FA2_BTRACE(18, g);
          pair::bulk_copy_to_cta(peer_slot, sXS, L::BOX128, peer_bar);
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();
          FA2_BTRACE(19, g);
          ptx::mbar_arrive(xs_empty);
        }
      }
      ptx::bulk_wait<0>();
    }
  }
  __syncwarp();
  ptx::tc_fence_before();
  pair::cluster_sync();
  if (warp == 0) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
  }
}

// dQ = cast(dq_acc) for the pair kernel's accumulator layout (see the header comment):
// one thread per (padded workspace row, 8 columns).
template <bool BF16>
__global__ void __launch_bounds__(256) fa2_dq_convert_pair(const RowParams p) {
  constexpr int D = 128;
  const long long t = static_cast<long long>(blockIdx.x) * 256 + threadIdx.x;
  if (t >= p.acc_rows * (D / 8)) return;
  const long long R = t / (D / 8);
  const int c = static_cast<int>(t % (D / 8)) * 8;
  long long q_off = 0, l_off = 0;
  if (!acc_row_ref(p, R, q_off, l_off)) return;
  const int q = static_cast<int>(R % 128);
  const float* src = p.dq_acc + (R / 128) * (128 * D) + ((q / 64) * 32 + c / 4) * 256 + (q % 64) * 4;
  const float4 a = *reinterpret_cast<const float4*>(src);
  const float4 b = *reinterpret_cast<const float4*>(src + 256);
  uint4 out;
  out.x = ptx::pack2<BF16>(a.x, a.y);
  out.y = ptx::pack2<BF16>(a.z, a.w);
  out.z = ptx::pack2<BF16>(b.x, b.y);
  out.w = ptx::pack2<BF16>(b.z, b.w);
  *reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(p.dq) + q_off + c) = out;
}

}  // namespace fa2
