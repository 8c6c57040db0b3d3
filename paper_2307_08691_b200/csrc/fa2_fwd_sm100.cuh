// FlashAttention-2 forward pass (Alg. 1) for sm_100a.
//
// One persistent CTA per SM walks a static list of work tiles.  A work tile is
// (b*h, m_block): 2 query sub-tiles Q0, Q1 of 128 rows each (256 rows, the
// "outer loop over row blocks").  For each key/value block K_j, V_j
// (B_c = 128 rows, the inner loop P:354-362):
//
//   S_i  = Q_i K_j^T                 tcgen05.mma SS, fp32 accumulator in TMEM
//   m, P~, l update (online softmax)  softmax warpgroup i, one thread = one row
//   O_i  = diag(e^{m_old-m_new}) O_i + P~ V_j   tcgen05.mma TS (P~ from TMEM)
//
// The O rescale factor is e^{m_old - m_new} (no inverse; R3).  It is
// applied lazily: the running max a row uses for its exponentials is only
// moved when the true max exceeds it by more than 2^8 (log2 domain), which is
// exact because l and O always share that max.  O is divided by
// l once at the end (tweak 1) and only L = m + log l is stored
// (tweak 2).  Causal blocks entirely above the diagonal are never
// visited and the mask is only evaluated on blocks that straddle the diagonal
// or the ragged tail.
//
// Warp roles (384 threads; FwdCfg):
//   warps 0-3   softmax WG 0: rows of Q0 (TMEM lanes 0-127), also O0 rescale + epilogue
//   warps 4-7   softmax WG 1: rows of Q1
//   warp  8     MMA issuer (one elected thread)
//   warp  9     TMA producer of Q and K, warp 10 TMA producer of V (one thread each)
//   warp  11    idle
//
// TMEM columns: S0 [0,128), S1 [128,256), O0 [256,256+D), O1 [256+D,256+2D);
// P~_i (16-bit) is written over the first 64 columns of S_i (d = 64: own columns).
//
// Alternatives measured on B200 and removed: two warps per row with the
// row max exchanged through SMEM; B_c = 64 with double-buffered P~ and one MMA issuer per
// sub-tile.
#pragma once
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <type_traits>
#include "fa2_seq.cuh"

namespace fa2 {

// Column pairs (out of every 16) whose exponential runs as a polynomial on the
// FMA pipe instead of MUFU.EX2 (unmasked blocks only).  Measured best on B200
// (tools/fwd_ms.py sweep over 2/4/6/8): 4 at d = 128 (bf16 and FP8), 6 at d = 64,
// where the MMAs are shorter and MUFU.EX2 (16/clk/SM) binds harder.
#ifndef FA2_FWD_EMU_PAIRS
#define FA2_FWD_EMU_PAIRS 4
#endif
#ifndef FA2_FWD_EMU_PAIRS_D64
#define FA2_FWD_EMU_PAIRS_D64 6
#endif
constexpr int kFwdEmuPairs = FA2_FWD_EMU_PAIRS;
template <int D, bool FP8> struct FwdCfg {
  static constexpr int SM_WARPS = 8;                   // softmax warps (both sub-tiles)
  static constexpr int THREADS = SM_WARPS * 32 + 128;  // + MMA, 2 TMA, 1 idle
  static constexpr int REG_SM = 224;                   // setmaxnreg: 224*256 + 56*128 == 168*384
  static constexpr int REG_OTHER = 56;
};
constexpr int kFwdEmuPairsD64 = FA2_FWD_EMU_PAIRS_D64;
// d = 64, causal square: ping-pong of the two softmax warpgroups' exponential phases through
// named barriers 1 / 2, as in the pair kernel (fa2_fwd2_sm100.cuh): S_{j+1} is issued as soon
// as S_j was read, so nothing else keeps the two sub-tiles out of phase, and the causal tiles
// (sub-tile 0 one block shorter) reset their phase every tile.  Causal N = 8k: 601-604 ->
// 667-691 TFLOP/s; non-causal measured 3-5% slower with it (725-739 -> 697-724), so it stays
// causal-only.
#ifndef FA2_FWD_PINGPONG64
#define FA2_FWD_PINGPONG64 1
#endif
#ifndef FA2_FWD_PP64_CH
#define FA2_FWD_PP64_CH 2   // signal after this many of the four 32-column chunks
#endif

struct FwdParams {
  void* o;             // fixed: [B, H, N_q, D]; packed: [T_q, H, D] (dtype)
  float* lse;          // fixed: [B, H, N_q]; packed: [H, T_q]
  int BH;              // B * H (query heads)
  int H, Hkv, group;   // query heads, key/value heads, H / Hkv (GQA; group == 1 for MHA)
  SeqGeom geom;        // sequence lengths / offsets (fa2_seq.cuh)
  long long o_bs, o_hs, o_rs;   // O strides in elements: batch, head, row
  long long l_bs, l_hs;         // L strides: batch, head (row stride 1)
  int num_m_blocks;    // ceil(N_q (max) / 256)
  int num_tiles;       // BH * num_m_blocks
  float scale_log2;    // softmax_scale * log2(e)  (FP8: times descale_q * descale_k)
  float o_descale;     // FP8: descale_v, applied with 1/l in the epilogue (unused otherwise)
  unsigned long long* trace;  // optional clock64 trace (CTA 0, first tile), nullptr in production
};

// Debug timeline: trace[(ev * 2 + who) * 64 + j] = clock64() for CTA 0's first
// work tile (j < 64).  who = sub-tile / MMA-side index.
// Every CTA's first work tile also lands at trace[65536 + ((cta * 8 + ev) * 2 + who) * 64 + j].
#define FA2_TRACE(ev, who, j)                                                          \
  do {                                                                                 \
    if (p.trace != nullptr && (j) < 64) {                                              \
      const unsigned long long c_ = clock64();                                         \
      if (blockIdx.x == 0) p.trace[((ev) * 2 + (who)) * 64 + (j)] = c_;                \
      p.trace[65536 + ((blockIdx.x * 8 + (ev)) * 2 + (who)) * 64 + (j)] = c_;          \
    }                                                                                  \
  } while (0)
// Debug tile timeline (same buffer, from element 4096): for each CTA's first 16 work tiles and
// each softmax warpgroup, {globaltimer, clock64} at the tile's start and after its epilogue,
// the tile index and its key-block count.
FA2_DEVICE void fa2_tile_trace(unsigned long long* tr, int n, int wg, int k, unsigned long long v) {
  if (tr != nullptr && n < 16) tr[4096 + ((blockIdx.x * 16 + n) * 2 + wg) * 8 + k] = v;
}
FA2_DEVICE unsigned fa2_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
FA2_DEVICE unsigned long long fa2_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Causal, square fixed-length path: host-computed balanced tile schedule (fa2_seq.cuh).
template <bool CAUSAL, bool GEN>
using FwdSchedT = SchedT<CAUSAL && !GEN>;

template <int D, int EB = 2>   // EB: bytes per Q/K/V element (2: bf16/fp16, 1: FP8)
struct FwdSmem {
  static constexpr int BM = 128, BN = 128;
  static constexpr int STAGES = (D == 64 || EB == 1) ? 3 : 2;
  static constexpr int TILE = 128 * D * EB;      // bytes of one 128 x D tile
  static constexpr int SUB = 128 * 128;          // one 128-row x 128-B swizzle box (16 KB)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * TILE;
  static constexpr int OFF_V = OFF_K + STAGES * TILE;
  // O staging for the TMA-store epilogue (FP8: bf16 O, 128 x 128 per softmax warpgroup).  At
  // d = 64 the same epilogue measured slower non-causal (792 -> 743 TFLOP/s, same box), so d = 64
  // keeps per-row stores.
  static constexpr bool HAS_OST = (EB == 1);
  static constexpr int O_TILE = 128 * D * 2;
  static constexpr int OFF_OST = OFF_V + STAGES * TILE;
  static constexpr int OFF_BAR = OFF_OST + (HAS_OST ? 2 * O_TILE : 0);
  // barriers: q_full[2] q_empty[2] k_full[S] k_empty[S] v_full[S] v_empty[S] s_full[2] p_full[2][2] o_done[2][2] o_empty[2]
  static constexpr int NBAR = 2 + 2 + 4 * STAGES + 2 + 4 + 4 + 2 + 2;   // + s_consumed[2]
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;   // slack for 1024-B alignment
};

// FP8: Q, K, V in E4M3 (kind::f8f6f4 MMAs, K = 32 per instruction),
// P~ quantized to E4M3 for the P~V MMA (P~ <= 2^8 under the lazy rescale, inside E4M3's
// 448), O written as bf16 (BF16 == true); d = 128 only (one 128-B swizzle atom per row).
template <int D, bool BF16, bool CAUSAL, bool GEN, bool FP8 = false>
__global__ void __launch_bounds__(FwdCfg<D, FP8>::THREADS, 1)
fa2_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o, const FwdParams p,
               const __grid_constant__ FwdSchedT<CAUSAL, GEN> sched) {
  static_assert(!FP8 || (D == 128 && BF16), "FP8 forward: d = 128, bf16 output");
  using L = FwdSmem<D, FP8 ? 1 : 2>;
  using CFG = FwdCfg<D, FP8>;
  constexpr int COLS = 128;   // S columns per softmax thread (one thread = one row)
  constexpr int W_MMA = CFG::SM_WARPS, W_TMA = CFG::SM_WARPS + 1;
  constexpr int STAGES = L::STAGES;
  constexpr int NSUB = D * (FP8 ? 1 : 2) / 128;   // 128-B swizzle boxes per tile row
  constexpr int BN = 128;                  // B_c: keys per block
  constexpr bool SEP_P = (D == 64);        // P~ in its own TMEM columns
  // TMEM columns of S_i, O_i and (SEP_P) P~_i
  constexpr uint32_t TS_STEP = BN, TO0 = 256, TP0 = 256 + 2 * D, TP_STEP = BN / 2;
  // p_full[i] / o_done[i] hand sub-tile i's P~ over (written / read by P~V number n)
  auto od_bar = [&](uint64_t* od, int i, uint32_t) { return &od[2 * i]; };
  auto od_par = [&](uint32_t n) -> uint32_t { return n & 1; };
  // FP8 (P~ over the first 32 columns of S_i): S_{j+1} in two N = 64 halves -- columns
  // 64-127 as soon as the softmax has read S_j (they are not under P~), columns 0-63 after
  // P~V_j -- so half of the next S overlaps the softmax instead of following P~V (+5-11%).
  // Not for bf16/fp16: each half re-reads the 32 KB Q tile, and S = Q K^T already runs at
  // the SMEM -> tensor-core rate (128 B/clk) with N = 128 (measured -15%).
#ifndef FA2_FWD_SPLIT_S
#define FA2_FWD_SPLIT_S 1
#endif
  constexpr bool SPLIT_S = !SEP_P && FP8 && FA2_FWD_SPLIT_S;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 2;
  uint64_t* k_full = bars + 4;
  uint64_t* k_empty = k_full + STAGES;
  uint64_t* v_full = k_empty + STAGES;
  uint64_t* v_empty = v_full + STAGES;
  uint64_t* s_full = v_empty + STAGES;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = p_full + 4;   // p_full / o_done: [sub-tile][P~ buffer], see od_bar
  uint64_t* o_empty = o_done + 4;
  uint64_t* s_consumed = o_empty + 2;   // [2] d=64 only: softmax has read S_i (4 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&p_full[2 * i], 4);
      ptx::mbar_init(&p_full[2 * i + 1], 4);
      ptx::mbar_init(&o_done[2 * i], 1);
      ptx::mbar_init(&o_done[2 * i + 1], 1);
      ptx::mbar_init(&o_empty[i], 4);
      ptx::mbar_init(&s_consumed[i], 4);
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 1);
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == W_TMA && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 0) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;


  // n-th work tile of this CTA (-1: done), shared by all roles
  auto tile_at = [&](int n) -> int { return sched_tile(sched, n, p.num_tiles); };
  // Work-tile decode, shared by all roles.  Heads are contiguous in the tile
  // order so that the CTAs running concurrently share K/V in L2; for causal the
  // heavy (late) row blocks of each head come first.  sq: the tile's sequence.
  auto decode = [&](int t, int& bh, int& mb, Seq& sq) {
    bh = t / p.num_m_blocks;
    int r = t % p.num_m_blocks;
    mb = CAUSAL ? (p.num_m_blocks - 1 - r) : r;
    sq = seq_of<GEN>(p.geom, bh / p.H);
  };
  // Number of KV blocks query sub-tile i of row block mb visits (0 when the sub-tile
  // is past the sequence end, or when no row of it sees a key: causal, N_q > N_k).
  auto n_blocks = [&](const Seq& sq, int mb, int i) -> int {
    const int r0 = mb * 256 + i * 128;
    if (r0 >= sq.nq) return 0;
    const int nkb = (sq.nk + BN - 1) / BN;
    if (!CAUSAL) return nkb;
    const int last_col = min(sq.nq - 1, r0 + 127) + sq.off;   // last key the sub-tile's last row sees
    return last_col < 0 ? 0 : min(nkb, last_col / BN + 1);
  };

  if (warp < CFG::SM_WARPS) {
    // ======================= softmax warpgroups =======================
    ptx::setmaxnreg_inc<CFG::REG_SM>();     // 224*256 + 56*128 == 168*384
    const int wg = warp / 4;                 // sub-tile index
    const int quad = warp % 4;               // TMEM lane quarter
    const int row = quad * 32 + lane;        // TMEM lane == row within sub-tile
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    const uint32_t tS = tmem + lane_base + wg * TS_STEP;
    // P~_i: over the first 64 columns of S_i (d = 128), or its own columns (d = 64: frees
    // S_i for S_{j+1} as soon as it has been read)
    const uint32_t tP0 = SEP_P ? (tmem + lane_base + TP0 + wg * TP_STEP) : (tmem + lane_base + wg * TS_STEP);
    const uint32_t tO = tmem + lane_base + TO0 + wg * D;
    uint32_t s_count = 0;   // completed waits on s_full[wg]
    uint32_t pv_count = 0;  // PV MMAs issued so far for this sub-tile (all tiles)
    constexpr bool PP = SEP_P && CAUSAL && !GEN && !FP8 && FA2_FWD_PINGPONG64;
    uint32_t gblk = 0;      // PP: key-block steps so far (incl. sub-tile 0's empty causal steps)
    const float sl2 = p.scale_log2;
    for (int n = 0, t; (t = tile_at(n)) >= 0; ++n) {
      int bh, mb;
      Seq sq;
      decode(t, bh, mb, sq);
      const int nb = n_blocks(sq, mb, wg);
      const int nkv = max(n_blocks(sq, mb, 0), n_blocks(sq, mb, 1));
      const bool last_tile = tile_at(n + 1) < 0;
      // PP: wait for the partner warpgroup before a block's exponentials, signal it half-way
      // (warpgroup 1 skips its very last signal: nobody waits for it)
      auto pp_wait = [&]() {
        if (PP && (wg == 1 || gblk > 0)) ptx::named_bar_sync(wg == 0 ? 2 : 1, 256);
      };
      auto pp_signal = [&](int j) {
        if (PP && !(wg == 1 && last_tile && j + 1 == nkv)) ptx::named_bar_arrive(wg == 0 ? 1 : 2, 256);
      };
      const int row0 = mb * 256 + wg * 128;
      const int grow = row0 + row;
      const bool ttr = threadIdx.x % 128 == 0;
      if (ttr) {
        fa2_tile_trace(p.trace, n, wg, 0, fa2_gtime());
        fa2_tile_trace(p.trace, n, wg, 1, clock64());
        fa2_tile_trace(p.trace, n, wg, 4, t);
        fa2_tile_trace(p.trace, n, wg, 5, nb);
        fa2_tile_trace(p.trace, n, wg, 6, fa2_smid());
      }
      if (nb == 0) {
        // PP: sub-tile 1 past the sequence end still steps through the ping-pong
        if constexpr (PP) {
          for (int j = 0; j < nkv; ++j) {
            pp_wait();
            pp_signal(j);
            ++gblk;
          }
        }
        // rows that see no key (R23): O = 0, L = -inf; no MMA work was scheduled
        if (grow < sq.nq) {
          uint4* dst = reinterpret_cast<uint4*>(
              reinterpret_cast<uint8_t*>(p.o) + (sq.bc * p.o_bs + (bh % p.H) * p.o_hs + (sq.q0 + grow) * p.o_rs) * 2);
#pragma unroll
          for (int e = 0; e < D / 8; ++e) dst[e] = make_uint4(0u, 0u, 0u, 0u);
          p.lse[sq.bc * p.l_bs + (bh % p.H) * p.l_hs + sq.q0 + grow] = -INFINITY;
        }
        continue;
      }
      float m_used = -INFINITY;   // running max in log2 units (may lag the true max by <= 8)
      float l_sum = 0.f;
      for (int j = 0; j < (PP ? nkv : nb); ++j) {
        if (PP && j >= nb) {   // causal: empty step of sub-tile 0 (one block fewer than sub-tile 1)
          pp_wait();
          pp_signal(j);
          ++gblk;
          continue;
        }
        ptx::mbar_wait(&s_full[wg], s_count & 1);
        ++s_count;
        if (threadIdx.x % 128 == 0 && n == 0) FA2_TRACE(0, wg, j);
        ptx::tc_fence_after();
        uint32_t su[COLS];
#pragma unroll
        for (int c = 0; c < COLS; c += 32) ptx::tmem_ld_x32(tS + c, su + c);
        ptx::tmem_wait_ld();
        if constexpr (SEP_P || SPLIT_S) {
          // S_i has been read: the MMA warp may compute (part of) S_i of the next block into it
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&s_consumed[wg]);
        }
        float s[COLS];
#pragma unroll
        for (int c = 0; c < COLS; ++c) s[c] = __uint_as_float(su[c]);
        const int c0 = j * BN;
        const bool need_mask = (c0 + BN > sq.nk) || (CAUSAL && (c0 + BN - 1 > row0 + sq.off));
        if (need_mask) {
          const int lim = CAUSAL ? min(sq.nk - 1, grow + sq.off) : (sq.nk - 1);
#pragma unroll
          for (int c = 0; c < COLS; ++c)
            if (c0 + c > lim) s[c] = -INFINITY;
        }
        // row max: a tree of 3-input maxima at d = 128 (+1.5% causal bf16, +3.5% FP8 on B200),
        // the serial FMNMX3 chain at d = 64 (the tree's temporaries cost it 10%)
        float mx;
        if constexpr (D == 128) {
          mx = ptx::tree_max<COLS>(s);
        } else {
          mx = s[0];
#pragma unroll
          for (int c = 1; c < COLS; ++c) mx = fmaxf(mx, s[c]);
        }
        if (threadIdx.x % 128 == 0 && n == 0) FA2_TRACE(1, wg, j);
        const float m_new = fmaxf(m_used, mx * sl2);
        const bool rescale = (m_new - m_used) > 8.0f;   // also true when m_used == -inf and m_new finite
        float alpha = 1.f;
        if (rescale) {
          alpha = ptx::ex2(m_used - m_new);             // 0 when m_used == -inf
          m_used = m_new;
        }
        const float base = (m_used == -INFINITY) ? 0.f : m_used;
        const float2 sl2x2 = make_float2(sl2, sl2), nb2 = make_float2(-base, -base);
        float2 rs2 = make_float2(0.f, 0.f);
        // exponent x = s * scale * log2(e) - m (FFMA2), P~ = 2^x.  On unmasked blocks
        // EMU of every 16 column pairs use the FMA-pipe polynomial, the rest MUFU.EX2.
        // SEP_P: the P buffer is free once the previous P~V MMA of this sub-tile completed.  The
        // exponentials do not need it: they are computed into registers first and the wait
        // comes right before the first TMEM store, so they overlap that P~V (d = 64: the exp
        // phase was 2270 cycles per block with the wait in front, ~MUFU-bound 1300 after)
        auto wait_p_free = [&]() {
          if constexpr (SEP_P) {
            if (pv_count >= 1) ptx::mbar_wait(od_bar(o_done, wg, pv_count - 1), od_par(pv_count - 1));
            ptx::tc_fence_after();
          }
        };
        const uint32_t tP = tP0;
        auto exp_block = [&](auto emu_tag) {
          constexpr int EMU = decltype(emu_tag)::value;
          uint32_t pk_all[COLS / 32][16];
#pragma unroll
          for (int ch = 0; ch < COLS / 32; ++ch) {
            if (ch == FA2_FWD_PP64_CH) pp_signal(j);
            uint32_t* pk = pk_all[ch];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float2 x = ptx::ffma2(make_float2(s[ch * 32 + 2 * e], s[ch * 32 + 2 * e + 1]), sl2x2, nb2);
              float2 pr;
              // d = 64: the emulated pairs spread over the 16 (Bresenham pattern), so the FMA-pipe
              // work sits between the MUFU ops instead of in one run (+5-8% at d = 64; the
              // contiguous run measured better at d = 128 and in the other kernels)
              if (D == 64 ? ((e % 16) * EMU) % 16 < EMU : e % 16 < EMU) {
                pr = ptx::exp2_poly2(x);
              } else {
                pr.x = ptx::ex2(x.x);
                pr.y = ptx::ex2(x.y);
              }
              rs2 = ptx::fadd2(rs2, pr);
              if constexpr (FP8) {   // 4 E4M3 values per TMEM column
                if (e % 2 == 0) pk[e / 2] = __float_as_uint(pr.x), pk[8 + e / 2] = __float_as_uint(pr.y);
                else pk[e / 2] = ptx::pack4_e4m3(__uint_as_float(pk[e / 2]), __uint_as_float(pk[8 + e / 2]), pr.x, pr.y);
              } else {
                pk[e] = ptx::pack2<BF16>(pr.x, pr.y);
              }
            }
            if constexpr (!SEP_P) {
              if constexpr (FP8) ptx::tmem_st_x8(tP + ch * 8, pk);
              else ptx::tmem_st_x16(tP + ch * 16, pk);
            }
          }
          if constexpr (SEP_P) {
            wait_p_free();
#pragma unroll
            for (int ch = 0; ch < COLS / 32; ++ch) ptx::tmem_st_x16(tP + ch * 16, pk_all[ch]);
          }
        };
        pp_wait();
        if (need_mask) exp_block(std::integral_constant<int, 0>{});
        else exp_block(std::integral_constant<int, D == 64 ? kFwdEmuPairsD64 : kFwdEmuPairs>{});
        l_sum = l_sum * alpha + (rs2.x + rs2.y);
        if (threadIdx.x % 128 == 0 && n == 0) FA2_TRACE(2, wg, j);
        // Rescale the un-normalised O accumulator before P~_j V_j is added
        // (needs PV_{j-1} finished; it was issued before S_j, so it usually is).
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
          ptx::mbar_wait(od_bar(o_done, wg, pv_count - 1), od_par(pv_count - 1));
          ptx::tc_fence_after();
#pragma unroll
          for (int ch = 0; ch < D / 32; ++ch) {
            uint32_t o[32];
            ptx::tmem_ld_x32(tO + ch * 32, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_x32(tO + ch * 32, o);
          }
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(od_bar(p_full, wg, pv_count));
        if (threadIdx.x % 128 == 0 && n == 0) FA2_TRACE(3, wg, j);
        ++pv_count;
        ++gblk;
      }
      // ---- epilogue: O = O / l, L = m + log l (natural log) ----
      ptx::mbar_wait(od_bar(o_done, wg, pv_count - 1), od_par(pv_count - 1));
      ptx::tc_fence_after();
      float inv_l = l_sum > 0.f ? 1.f / l_sum : 0.f;   // rows that saw no key: O = 0 (R23)
      if constexpr (FP8) inv_l *= p.o_descale;
      uint8_t* orow = reinterpret_cast<uint8_t*>(p.o) +
                      (GEN ? (sq.bc * p.o_bs + (bh % p.H) * p.o_hs + (sq.q0 + grow) * p.o_rs)
                           : (static_cast<size_t>(bh) * sq.nq + grow) * D) * 2;
      uint32_t pk[D / 32][16];
#pragma unroll
      for (int ch = 0; ch < D / 32; ++ch) {
        uint32_t o[32];
        ptx::tmem_ld_x32(tO + ch * 32, o);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          pk[ch][e] = ptx::pack2<BF16>(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
      }
      // O_i is out of TMEM: the next tile's first P~V may overwrite it
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&o_empty[wg]);
      if (grow < sq.nq)
        p.lse[GEN ? sq.bc * p.l_bs + (bh % p.H) * p.l_hs + sq.q0 + grow : static_cast<size_t>(bh) * sq.nq + grow] = l_sum > 0.f ? (m_used + ptx::lg2(l_sum)) * 0.69314718055994531f : -INFINITY;
      // TMA-store epilogue (FP8; same-box A/B 1442-1471 -> 1504-1529 TFLOP/s non-causal)
      constexpr bool OST = !GEN && L::HAS_OST;
      if constexpr (OST) {
        // staged in SW128 boxes of 64 columns and written by TMA tensor stores (rows past N
        // clipped by the tensor map)
        uint8_t* ost = smem + L::OFF_OST + wg * L::O_TILE;
        const uint32_t ost_row = ptx::smem_u32(ost) + row * 128;
#pragma unroll
        for (int c = 0; c < D / 8; ++c)
          ptx::sts_v4(ost_row + (c / 8) * (128 * 128) + (((c % 8) ^ (row % 8)) * 16), pk[c / 4][4 * (c % 4)],
                      pk[c / 4][4 * (c % 4) + 1], pk[c / 4][4 * (c % 4) + 2], pk[c / 4][4 * (c % 4) + 3]);
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(3 + wg, 128);
        if (row == 0) {
#pragma unroll
          for (int bx = 0; bx < D / 64; ++bx) ptx::tma_store_3d(&tm_o, ost + bx * 128 * 128, bx * 64, row0, bh);
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();   // the staging is read: the next tile's epilogue may reuse it
        }
        ptx::named_bar_sync(3 + wg, 128);
      } else if (grow < sq.nq) {
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint4* dst = reinterpret_cast<uint4*>(orow + ch * 64);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_uint4(pk[ch][4 * e], pk[ch][4 * e + 1], pk[ch][4 * e + 2], pk[ch][4 * e + 3]);
        }
      }
      if (ttr) {
        fa2_tile_trace(p.trace, n, wg, 2, fa2_gtime());
        fa2_tile_trace(p.trace, n, wg, 3, clock64());
      }
    }
    if (!GEN && L::HAS_OST && row == 0) ptx::bulk_wait<0>();   // the O tensor stores have completed
  } else {
    ptx::setmaxnreg_dec<CFG::REG_OTHER>();
    if (warp == W_MMA) {
      // ================== MMA issuer: whole warp, one elected lane issues ==================
      const int me = 0;
      // (E4M3 has format code 0 in the kind::f8f6f4 descriptor, as F16 in kind::f16)
      constexpr uint32_t IDESC_S = ptx::idesc_f16(FP8 ? false : BF16, 128, 128, false, false);
      constexpr uint32_t IDESC_O = ptx::idesc_f16(FP8 ? false : BF16, 128, D, false, true);
      // base descriptors; per-MMA descriptors add (byte offset >> 4) to the start-address field
      const uint64_t dQ = ptx::sw128_desc(ptx::smem_u32(sQ), 16, 1024);
      const uint64_t dK = ptx::sw128_desc(ptx::smem_u32(sK), 16, 1024);
      const uint64_t dV = ptx::sw128_desc(ptx::smem_u32(sV), L::SUB, 1024);
      int kslot = 0, vslot = 0;
      uint32_t kphase = 0, vphase = 0;
      uint32_t p_count0 = 0, p_count1 = 0, o_uses0 = 0, o_uses1 = 0;
      int it = 0;
      constexpr uint32_t IDESC_S64 = ptx::idesc_f16(FP8 ? false : BF16, 128, 64, false, false);
      auto mma_s = [&](int i, int slot) {
        // K steps of 32 bytes (16 bf16/fp16 or 32 E4M3 elements), 4 per 128-B swizzle box
#pragma unroll
        for (int k = 0; k < D * (FP8 ? 1 : 2) / 32; ++k) {
          const uint32_t off = (k / 4) * L::SUB + (k % 4) * 32;
          if constexpr (FP8)
            ptx::mma_ss_f8(tmem + i * 128, dQ + ((i * L::TILE + off) >> 4), dK + ((slot * L::TILE + off) >> 4),
                           IDESC_S, k > 0 ? 1u : 0u);
          else
            ptx::mma_ss(tmem + i * 128, dQ + ((i * L::TILE + off) >> 4), dK + ((slot * L::TILE + off) >> 4), IDESC_S,
                        k > 0 ? 1u : 0u);
        }
      };
      // one N = 64 half of S_i = Q_i K^T: key rows [64 h, 64 h + 64) -> S columns [64 h, 64 h + 64)
      auto mma_s_half = [&](int i, int slot, int h) {
#pragma unroll
        for (int k = 0; k < D * (FP8 ? 1 : 2) / 32; ++k) {
          const uint32_t off = (k / 4) * L::SUB + (k % 4) * 32;
          const uint32_t boff = slot * L::TILE + off + h * 64 * 128;   // 64 rows of 128 B further
          if constexpr (FP8)
            ptx::mma_ss_f8(tmem + i * 128 + h * 64, dQ + ((i * L::TILE + off) >> 4), dK + (boff >> 4), IDESC_S64,
                           k > 0 ? 1u : 0u);
          else
            ptx::mma_ss(tmem + i * 128 + h * 64, dQ + ((i * L::TILE + off) >> 4), dK + (boff >> 4), IDESC_S64,
                        k > 0 ? 1u : 0u);
        }
      };
      auto mma_pv = [&](int i, int slot, bool acc) {
        // K = 128 keys: 8 steps of 16 (P~ 16-bit: 8 TMEM columns, V rows 16 x 128 B) or
        // 4 steps of 32 (P~ E4M3: 8 TMEM columns, V rows 32 x 128 B)
        if constexpr (FP8) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            ptx::mma_ts_f8(tmem + TO0 + i * D, tmem + i * 128 + k * 8, dV + ((slot * L::TILE + k * 4096) >> 4), IDESC_O,
                           (acc || k > 0) ? 1u : 0u);
        } else {
#pragma unroll
          for (int k = 0; k < BN / 16; ++k)
            ptx::mma_ts(tmem + TO0 + i * D, tmem + (SEP_P ? TP0 + i * TP_STEP : i * 128) + k * 8,
                        dV + ((slot * L::TILE + k * 2048) >> 4), IDESC_O, (acc || k > 0) ? 1u : 0u);
        }
      };
      uint32_t s_iss01[2] = {0, 0};   // SEP_P: S MMAs issued per sub-tile (s_consumed phases)
      uint32_t p_cnt01[2] = {0, 0}, o_use01[2] = {0, 0};   // SEP_P: P~V MMAs / tiles per sub-tile
      uint32_t sc_count0 = 0, sc_count1 = 0;   // d = 128 SPLIT_S: s_consumed phases waited per sub-tile
      // d = 64: S_i into its buffer once softmax i has read the previous S_i
      auto issue_s_sep = [&](int i, uint32_t& s_iss) {
        if (s_iss > 0) ptx::mbar_wait(&s_consumed[i], (s_iss - 1) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) { mma_s(i, kslot); ptx::mma_commit(&s_full[i]); }
        __syncwarp();
        ++s_iss;
      };
      for (int n = 0, t; (t = tile_at(n)) >= 0; ++n, ++it) {
        int bh, mb;
        Seq sq;
        decode(t, bh, mb, sq);
        const int nb0 = n_blocks(sq, mb, 0), nb1 = n_blocks(sq, mb, 1);
        const int nkv = max(nb0, nb1);
        if constexpr (SEP_P) {
          const int i0 = 0, i1 = 1;
          uint32_t* s_iss = s_iss01;
          uint32_t* p_cnt = p_cnt01;
          uint32_t* o_use = o_use01;
          for (int i = i0; i <= i1; ++i) ptx::mbar_wait(&q_full[i], it & 1);
          // S_{j+1} is issued as soon as S_j has been read (P~ has its own buffer),
          // so the next block's scores are ready when the softmax finishes block j.
          for (int j = -1; j < nkv; ++j) {
            if (j + 1 < nkv) {
              const int jn = j + 1;
              ptx::mbar_wait(&k_full[kslot], kphase);
              if (it == 0) FA2_TRACE(4, me, jn);
              for (int i = i0; i <= i1; ++i) {
                const int nbi = i == 0 ? nb0 : nb1;
                if (jn < nbi) issue_s_sep(i, s_iss[i]);
                if (jn + 1 == nbi) {   // Q_i's last S: release Q_i for the next tile
                  if (ptx::elect_one()) ptx::mma_commit(&q_empty[i]);
                  __syncwarp();
                }
              }
              if (ptx::elect_one()) ptx::mma_commit(&k_empty[kslot]);
              __syncwarp();
              if (++kslot == STAGES) { kslot = 0; kphase ^= 1; }
            }
            if (j < 0) continue;
            ptx::mbar_wait(&v_full[vslot], vphase);
            auto pv = [&](int i, int nbi) {
              if (j >= nbi) return;
              if (j == 0) {
                if (o_use[i] > 0) ptx::mbar_wait(&o_empty[i], (o_use[i] - 1) & 1);
                ++o_use[i];
              }
              const uint32_t n = p_cnt[i]++;
              ptx::mbar_wait(od_bar(p_full, i, n), od_par(n));
              ptx::tc_fence_after();
              if (ptx::elect_one()) { mma_pv(i, vslot, j > 0); ptx::mma_commit(od_bar(o_done, i, n)); }
              __syncwarp();
            };
            for (int i = i0; i <= i1; ++i) pv(i, i == 0 ? nb0 : nb1);
            if (it == 0) FA2_TRACE(5, me, j);
            if (ptx::elect_one()) ptx::mma_commit(&v_empty[vslot]);
            __syncwarp();
            if (++vslot == STAGES) { vslot = 0; vphase ^= 1; }
          }
          if (ptx::elect_one())   // sub-tiles without key blocks release Q_i here
            for (int i = i0; i <= i1; ++i)
              if ((i == 0 ? nb0 : nb1) == 0) ptx::mma_commit(&q_empty[i]);
          __syncwarp();
          continue;
        }
        ptx::mbar_wait(&q_full[0], it & 1);
        ptx::mbar_wait(&q_full[1], it & 1);
        if (nkv > 0) {
          ptx::mbar_wait(&k_full[kslot], kphase);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            if (nb0 > 0) { mma_s(0, kslot); ptx::mma_commit(&s_full[0]); }
            if (nb0 <= 1) ptx::mma_commit(&q_empty[0]);   // Q_0's last S (see below)
            if (nb1 > 0) { mma_s(1, kslot); ptx::mma_commit(&s_full[1]); }
            if (nb1 <= 1) ptx::mma_commit(&q_empty[1]);
            ptx::mma_commit(&k_empty[kslot]);
          }
          __syncwarp();
          if (++kslot == STAGES) { kslot = 0; kphase ^= 1; }
        } else if (ptx::elect_one()) {
          ptx::mma_commit(&q_empty[0]);
          ptx::mma_commit(&q_empty[1]);
        }
        __syncwarp();
        for (int j = 0; j < nkv; ++j) {
          ptx::mbar_wait(&v_full[vslot], vphase);
          bool k_ready = false;
          // SPLIT_S: once softmax i has read S_i(j), S_i(j+1) columns 64-127
          auto step_b = [&](int i, int nbi, uint32_t& sc_count) {
            if (j >= nbi) return;
            ptx::mbar_wait(&s_consumed[i], sc_count & 1);   // every block's read is waited for (phases)
            ++sc_count;
            if (j + 1 >= nbi) return;
            if (!k_ready) {
              ptx::mbar_wait(&k_full[kslot], kphase);
              k_ready = true;
            }
            ptx::tc_fence_after();
            if (ptx::elect_one()) mma_s_half(i, kslot, 1);
            __syncwarp();
          };
          // sub-tile i: O_i += P_i V_j (after softmax i signals P_i), then S_i = Q_i K_{j+1}^T
          // (SPLIT_S: its columns 0-63, the rest was issued by step_b)
          auto step = [&](int i, int nbi, uint32_t& p_count, uint32_t& o_uses) {
            const bool do_pv = j < nbi, do_s = j + 1 < nbi;
            if (do_pv) {
              if (j == 0) {
                if (o_uses > 0) ptx::mbar_wait(&o_empty[i], (o_uses - 1) & 1);
                ++o_uses;
              }
              ptx::mbar_wait(od_bar(p_full, i, p_count), od_par(p_count));
              ++p_count;
              if (it == 0) FA2_TRACE(4, i, j);
            }
            if (do_s && !k_ready) {
              ptx::mbar_wait(&k_full[kslot], kphase);
              k_ready = true;
            }
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
              if (do_pv) { mma_pv(i, vslot, j > 0); ptx::mma_commit(od_bar(o_done, i, p_count - 1)); }
              if (do_s) {
                if constexpr (SPLIT_S) mma_s_half(i, kslot, 0);
                else mma_s(i, kslot);
                ptx::mma_commit(&s_full[i]);
                // Q_i is free once its last S completes: the producer loads the next
                // tile's Q_i while this tile's last softmax, P~V and epilogue run
                if (j + 2 == nbi) ptx::mma_commit(&q_empty[i]);
              }
            }
            __syncwarp();
            if (do_s && it == 0) FA2_TRACE(5, i, j);
          };
          if constexpr (SPLIT_S) step_b(0, nb0, sc_count0);
          step(0, nb0, p_count0, o_uses0);
          if constexpr (SPLIT_S) step_b(1, nb1, sc_count1);
          step(1, nb1, p_count1, o_uses1);
          if (ptx::elect_one()) {
            ptx::mma_commit(&v_empty[vslot]);
            if (k_ready) ptx::mma_commit(&k_empty[kslot]);
          }
          __syncwarp();
          if (++vslot == STAGES) { vslot = 0; vphase ^= 1; }
          if (k_ready && ++kslot == STAGES) { kslot = 0; kphase ^= 1; }
        }
      }
    } else if ((warp == W_TMA || warp == W_TMA + 1) && lane == 0) {
      // ===================== TMA producers: Q + K (warp W_TMA), V (W_TMA + 1) =====================
      // Two threads, so a K load never queues behind a V slot that the (later) P~V MMAs
      // still hold: S runs up to two key blocks ahead of P~V.
      const bool is_k = warp == W_TMA;
      int slot = 0;
      uint32_t phase = 0;
      int it = 0;
      const uint64_t pol_kv = ptx::l2_policy_evict_last();
      const uint64_t pol_q = ptx::l2_policy_evict_first();
      uint64_t* full = is_k ? k_full : v_full;
      uint64_t* empty = is_k ? k_empty : v_empty;
      uint8_t* buf = is_k ? sK : sV;
      const CUtensorMap* tm = is_k ? &tm_k : &tm_v;
      for (int n = 0, t; (t = tile_at(n)) >= 0; ++n, ++it) {
        int bh, mb;
        Seq sq;
        decode(t, bh, mb, sq);
        const int nblk = max(n_blocks(sq, mb, 0), n_blocks(sq, mb, 1));
        const int nkv = nblk;   // 128-row K/V stages
        // key/value head of this query head: implicit index manipulation
        const int h = bh % p.H, kvh = h / p.group;
        if (is_k) {
          for (int i = 0; i < 2; ++i) {
            if (it > 0) ptx::mbar_wait(&q_empty[i], (it - 1) & 1);
            ptx::mbar_arrive_expect_tx(&q_full[i], L::TILE);
            for (int s = 0; s < NSUB; ++s)
              tma_load_rows<GEN>(sQ + i * L::TILE + s * L::SUB, &tm_q, &q_full[i], p.geom, s * 64,
                                 sq.q0 + mb * 256 + i * 128, h, sq.bc, p.H, pol_q);
          }
        }
        for (int j = 0; j < nkv; ++j) {
          ptx::mbar_wait(&empty[slot], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[slot], L::TILE);
          for (int s = 0; s < NSUB; ++s)
            tma_load_rows<GEN>(buf + slot * L::TILE + s * L::SUB, tm, &full[slot], p.geom, s * 64, sq.k0 + j * 128,
                               kvh, sq.bc, p.Hkv, pol_kv);
          if (++slot == STAGES) { slot = 0; phase ^= 1; }
        }
      }
    }
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
