// FlashAttention-2 forward (Alg. 1) on a CTA pair (cta_group::2): the
// d = 128, bf16/fp16, fixed-layout path (the paper's benchmark shapes; also N_q != N_k, causal
// with N_q <= N_k).
//
// Why a pair: on one SM the chain softmax_i -> P~V_i -> S_i ->
// softmax_i bounds the forward, and breaking it needs P~ outside the S columns -- TMEM
// is full (S0 S1 O0 O1) and P~ in shared memory pushes one SM past its 128 B/clk
// SMEM -> tensor-core rate.  With cta_group::2 every MMA has M = 256 (128 rows per
// CTA) and each CTA holds only half of B (K: 64 of the block's 128 keys, V: 64 of the
// 128 head-dim columns), so S = Q K^T reads 96 B/clk per SM, K/V loads halve, and P~
// fits in shared memory as the A operand of P~V.  S_{j+1} is then issued as soon as
// the softmax has read S_j, so the softmax runs back to back.
//
// A work tile is (b*h, 512 query rows): CTA rank r of the pair owns rows
// [512 m + 256 r, +256) as two 128-row sub-tiles (TMEM lanes = rows).  Per key block j:
//   S_i  = Q_i K_j^T                    leader-issued M = 256 SS MMA -> S_i in both CTAs' TMEM
//   m, P~, l (online softmax)           softmax warpgroup i of each CTA; P~ -> SMEM (SW128)
//   O_i  = diag(e^{m_old-m_new}) O_i + P~ V_j    M = 256 SS MMA (A = P~ of both CTAs)
// The rescale is lazy as in fa2_fwd_sm100.cuh (threshold 2^8, exact).
//
// Barriers: "full"-type barriers the MMA warps wait on live in the leader (rank 0):
// TMA loads of both CTAs signal the leader's q_full/k_full/v_full (cta_group::2 TMA),
// the softmax warps of both CTAs arrive remotely on the leader's s_consumed/p_full/
// o_empty.  Barriers the MMAs release (s_full, o_done, q/k/v_empty) are signalled in
// both CTAs by multicast tcgen05.commit.
//
// Warp roles (384 threads per CTA): warps 0-3 / 4-7 softmax of sub-tile 0 / 1; warp 8
// (leader) MMA issuer of sub-tile 0, warp 11 (leader) of sub-tile 1; warp 9 TMA of Q
// and K, warp 10 TMA of V.
#pragma once
#include "fa2_fwd_sm100.cuh"
#include "sm100_pair.cuh"

namespace fa2 {

// FMA-pipe exponential pairs per 16 in the pair kernel, whose two sub-tiles' softmaxes run
// concurrently (two warps per SMSP): measured 1327 / 1394 / 1308 / 1250 TFLOP/s for
// 0 / 2 / 4 / 6 (d = 128, N = 8k, non-causal).
#ifndef FA2_FWD_PAIR_EMU
#define FA2_FWD_PAIR_EMU 2
#endif
constexpr int kFwdPairEmuPairs = FA2_FWD_PAIR_EMU;
// Ping-pong of the two sub-tiles' exponential phases (named barriers 1 / 2, 256 threads):
// softmax warpgroup 1 starts the exponentials of block g once warpgroup 0 has produced
// FA2_FWD_PP_C of its 16 P~ chunks of block g, and warpgroup 0 starts block g + 1 once
// warpgroup 1 is as far into block g.  Left free, the two warpgroups drift into phase (row
// max, S loads and P~V waits of both at once, MUFU idle) on most pairs: 2775-3250 cycles
// per key block depending on the pair, 2890-2930 on every pair with the ping-pong.
#ifndef FA2_FWD_PINGPONG
#define FA2_FWD_PINGPONG 1
#endif
#ifndef FA2_FWD_PP_C
#define FA2_FWD_PP_C 8
#endif


struct FwdPairSmem {
  static constexpr int D = 128;
  static constexpr int STAGES = 3;
  static constexpr int Q_TILE = 128 * D * 2;       // one 128-row sub-tile of Q (32 KB, 2 SW128 boxes)
  static constexpr int Q_BOX = 128 * 128;          // 128 rows x 128 B
  static constexpr int K_HALF = 64 * D * 2;        // 64 key rows x 128 d (16 KB, 2 boxes of 64 x 128 B)
  static constexpr int K_BOX = 64 * 128;
  static constexpr int V_HALF = 128 * 64 * 2;      // 128 key rows x 64 d columns (16 KB, 1 box)
  static constexpr int P_TILE = 128 * 128 * 2;     // P~ of one sub-tile: 128 rows x 128 keys (2 boxes)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + 2 * Q_TILE;
  static constexpr int OFF_V = OFF_K + STAGES * K_HALF;
  static constexpr int OFF_P = OFF_V + STAGES * V_HALF;
  static constexpr int OFF_BAR = OFF_P + 2 * P_TILE;
  // q_full[2] q_empty[2] k_full[S] k_empty[S] v_full[S] v_empty[S] s_full[2] s_consumed[2]
  // p_full[2] o_done[2] o_empty[2]
  static constexpr int NBAR = 4 + 4 * STAGES + 10;
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

// p: as for fa2_fwd_kernel with num_m_blocks = ceil(N / 512), num_tiles = BH * num_m_blocks.
// CAUSAL: CTA r's sub-tile i holds rows [512 m + 256 i + 128 r, +128), so every M = 256 MMA
// covers 256 consecutive rows and sub-tile i visits key blocks 0 .. 4 m + 2 i + 1 (the last
// two straddle or pass the diagonal of CTA 0's rows: masked).  Sub-tile 0 has two blocks
// fewer; its warpgroup runs them as empty ping-pong steps (no S, no exponentials, no P~V,
// its issuer only releases their K/V stages) so the two warpgroups keep alternating.  Tiles
// come heaviest first from the host's balanced pair schedule (fa2_seq.cuh TileSched).
// GEN: the packed variable-length layout (fa2_seq.cuh): every tile resolves its sequence (first
// rows, N_q, N_k, causal offset N_k - N_q); tiles past a sequence's rows are skipped by every
// role, sub-tiles whose rows see no key (N_k = 0, or causal N_q > N_k) write O = 0, L = -inf (R23)
// and step through the ping-pong empty.
template <bool BF16, bool CAUSAL, bool GEN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
fa2_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k64,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_o,
                    const FwdParams p,
                    const __grid_constant__ SchedT<CAUSAL && !GEN> sched) {
  using L = FwdPairSmem;
  constexpr int D = 128, STAGES = L::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 2;
  uint64_t* k_full = bars + 4;
  uint64_t* k_empty = k_full + STAGES;
  uint64_t* v_full = k_empty + STAGES;
  uint64_t* v_empty = v_full + STAGES;
  uint64_t* s_full = v_empty + STAGES;
  uint64_t* s_consumed = s_full + 2;
  uint64_t* p_full = s_consumed + 2;
  uint64_t* o_done = p_full + 2;
  uint64_t* o_empty = o_done + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = pair::cta_rank();
  const int pair_id = static_cast<int>(pair::cluster_id()), npairs = static_cast<int>(pair::num_clusters());

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_consumed[i], 8);   // 4 softmax warps x 2 CTAs (leader's copy)
      ptx::mbar_init(&p_full[i], 8);
      ptx::mbar_init(&o_done[i], 1);
      ptx::mbar_init(&o_empty[i], 8);
    }
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&k_full[s], 1);
      ptx::mbar_init(&k_empty[s], 2);      // one multicast commit per MMA-issuer warp
      ptx::mbar_init(&v_full[s], 1);
      ptx::mbar_init(&v_empty[s], 2);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 9 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q);
    ptx::tma_prefetch_desc(&tm_k64);
    ptx::tma_prefetch_desc(&tm_v);
  }
  if (warp == 0)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(ptx::smem_u32(tmem_slot)), "r"(512));
  ptx::tc_fence_before();
  pair::cluster_sync();   // barriers initialised and TMEM allocated in both CTAs
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // fixed layout: N_q query rows, N_k key rows, bottom-right causal offset N_k - N_q (R22)
  // work tiles (shared by all roles): n-th tile of this pair, its head and 512-row block
  auto tile_at = [&](int n) { return pair::sched_tile_pair(sched, n, p.num_tiles, pair_id, npairs); };
  // A work tile as every role sees it: head, 512-row block, its sequence's geometry
  struct PairFwdTile {
    int bh, mb, h, b;
    int q0, k0, nq, nk, off;   // first query / key row of the sequence in its tensor, lengths, offset
  };
  auto decode = [&](int t) {
    PairFwdTile w;
    w.bh = t / p.num_m_blocks;
    const int r = t % p.num_m_blocks;
    w.mb = CAUSAL ? p.num_m_blocks - 1 - r : r;   // causal: heavy row blocks first in the tile order
    w.h = w.bh % p.H;
    w.b = w.bh / p.H;
    if constexpr (GEN) {
      const Seq sq = seq_of<true>(p.geom, w.b);
      w.q0 = sq.q0; w.k0 = sq.k0; w.nq = sq.nq; w.nk = sq.nk;
    } else {
      w.q0 = 0; w.k0 = 0; w.nq = p.geom.Nq; w.nk = p.geom.Nk;
    }
    w.off = w.nk - w.nq;
    return w;
  };
  auto tile_empty = [&](const PairFwdTile& w) { return GEN && w.mb * 512 >= w.nq; };
  // first row of this CTA's sub-tile i, and the key blocks sub-tile i visits (both CTAs)
  auto row0_of = [&](int mb, int i) {
    return CAUSAL ? mb * 512 + i * 256 + static_cast<int>(rank) * 128 : mb * 512 + static_cast<int>(rank) * 256 + i * 128;
  };
  // key blocks sub-tile i visits (both CTAs): all of N_k, causal up to its last row's diagonal
  auto nblk = [&](const PairFwdTile& w, int i) -> int {
    const int nkb = (w.nk + 127) / 128;
    if (!CAUSAL) return nkb;
    const int last = min(w.nq - 1, w.mb * 512 + i * 256 + 255) + w.off;
    return last < 0 ? 0 : min(nkb, last / 128 + 1);
  };
  // the next tile of this pair that is not skipped (-1: none)
  auto next_tile = [&](int n) {
    int t;
    while ((t = tile_at(n)) >= 0 && tile_empty(decode(t))) ++n;
    return t;
  };

  if (warp < 8) {
    // ======================= softmax warpgroups =======================
    ptx::setmaxnreg_inc<224>();
    const int wg = warp / 4;
    const int row = threadIdx.x % 128;
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t tS = tmem + lane_base + wg * 128;
    const uint32_t tO = tmem + lane_base + 256 + wg * D;
    // P~ row `row` of sub-tile wg: SW128 K-major, box b = keys [64 b, 64 b + 64)
    const uint32_t sP_row = ptx::smem_u32(sP + wg * L::P_TILE) + row * 128;
    uint32_t s_count = 0, pv_count = 0, gblk = 0;   // gblk: key blocks stepped (incl. empty steps)
    const float sl2 = p.scale_log2;
    for (int tn = 0, t; (t = tile_at(tn)) >= 0; ++tn) {
      const PairFwdTile w = decode(t);
      if (tile_empty(w)) continue;
      const int mb = w.mb, nq = w.nq, nk = w.nk, off = w.off;
      const int r0 = row0_of(mb, wg), grow = r0 + row;
      const int nb = nblk(w, wg), nkv = nblk(w, 1);
      float m_used = -INFINITY, l_sum = 0.f;
      const bool tr = threadIdx.x % 128 == 0 && tn == 0;
      const bool last_tile = next_tile(tn + 1) < 0;
      // this row of O and L in the output tensors
      const long long o_off = static_cast<long long>(w.b) * p.o_bs + w.h * p.o_hs + static_cast<long long>(w.q0 + grow) * p.o_rs;
      const long long l_off = static_cast<long long>(w.b) * p.l_bs + w.h * p.l_hs + w.q0 + grow;
      // ping-pong: wait for the partner warpgroup before this block's exponentials, signal it
      // FA2_FWD_PP_C chunks in (warpgroup 1 skips its very last signal: nobody waits for it)
      auto pp_wait = [&]() {
        if (FA2_FWD_PINGPONG && (wg == 1 || gblk > 0)) ptx::named_bar_sync(wg == 0 ? 2 : 1, 256);
      };
      auto pp_signal = [&](int j) {
        if (FA2_FWD_PINGPONG && !(wg == 1 && last_tile && j + 1 == nkv)) ptx::named_bar_arrive(wg == 0 ? 1 : 2, 256);
      };
      if (threadIdx.x % 128 == 0) {
        fa2_tile_trace(p.trace, tn, wg, 0, fa2_gtime());
        fa2_tile_trace(p.trace, tn, wg, 1, clock64());
        fa2_tile_trace(p.trace, tn, wg, 4, t);
        fa2_tile_trace(p.trace, tn, wg, 5, nb);
        fa2_tile_trace(p.trace, tn, wg, 6, fa2_smid());
      }
      // ---- epilogue: O = O / l, L = m + log l ----
      auto epilogue = [&]() {
        if (threadIdx.x % 128 == 0) fa2_tile_trace(p.trace, tn, wg, 7, clock64());   // epilogue start
        ptx::mbar_wait(&o_done[wg], (pv_count - 1) & 1);
        ptx::tc_fence_after();
        const float inv_l = l_sum > 0.f ? 1.f / l_sum : 0.f;
        uint32_t q[4][16];
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t o[32];
          ptx::tmem_ld_x32(tO + ch * 32, o);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            q[ch][e] = ptx::pack2<BF16>(__uint_as_float(o[2 * e]) * inv_l, __uint_as_float(o[2 * e + 1]) * inv_l);
        }
        // O_i has been read out of TMEM: the next tile's first P~V may overwrite it
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair::arrive_remote(&o_empty[wg], 0);
        if (grow < nq) p.lse[l_off] = l_sum > 0.f ? (m_used + ptx::lg2(l_sum)) * 0.69314718055994531f : -INFINITY;
        if constexpr (!GEN) {
          // the sub-tile's P~ buffer (free: the last P~V has completed) stages O in the SW128
          // layout of two 64-column boxes, and one TMA store per box writes the 128 rows (rows
          // past N_q are clipped by the tensor map)
#pragma unroll
          for (int c = 0; c < 16; ++c)
            ptx::sts_v4(sP_row + (c / 8) * L::Q_BOX + (((c % 8) ^ (row % 8)) * 16), q[c / 4][4 * (c % 4)],
                        q[c / 4][4 * (c % 4) + 1], q[c / 4][4 * (c % 4) + 2], q[c / 4][4 * (c % 4) + 3]);
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(3 + wg, 128);
          if (threadIdx.x % 128 == 0) {
            ptx::tma_store_3d(&tm_o, sP + wg * L::P_TILE, 0, r0, w.bh);
            ptx::tma_store_3d(&tm_o, sP + wg * L::P_TILE + L::Q_BOX, 64, r0, w.bh);
            ptx::bulk_commit();
            ptx::bulk_wait_read<0>();   // the buffer is read: the next tile's P~ may go there
          }
          ptx::named_bar_sync(3 + wg, 128);
        } else {
          // packed layout: rows past this sequence belong to the next one, so per-row stores
          if (grow < nq) {
            uint8_t* orow = reinterpret_cast<uint8_t*>(p.o) + o_off * 2;
#pragma unroll
            for (int ch = 0; ch < D / 32; ++ch) {
              uint4* dst = reinterpret_cast<uint4*>(orow + ch * 64);
#pragma unroll
              for (int e = 0; e < 4; ++e) dst[e] = make_uint4(q[ch][4 * e], q[ch][4 * e + 1], q[ch][4 * e + 2], q[ch][4 * e + 3]);
            }
          }
        }
      };
      if (nb == 0) {   // no row of this sub-tile sees a key (R23): O = 0, L = -inf; no MMA work
        for (int j = 0; j < nkv; ++j) {
          pp_wait();
          pp_signal(j);
          ++gblk;
        }
        if (grow < nq) {
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(p.o) + o_off * 2);
#pragma unroll
          for (int e = 0; e < D / 8; ++e) dst[e] = make_uint4(0u, 0u, 0u, 0u);
          p.lse[l_off] = -INFINITY;
        }
        continue;
      }
      for (int j = 0; j < nkv; ++j) {
        if (j >= nb) {   // empty step of sub-tile 0 (its rows see none of these keys)
          pp_wait();
          pp_signal(j);
          ++gblk;
          continue;
        }
        ptx::mbar_wait(&s_full[wg], s_count & 1);
        ++s_count;
        if (tr) FA2_TRACE(0, wg, j);
        ptx::tc_fence_after();
        uint32_t su[128];
        ptx::tmem_ld_x32(tS + 0, su + 0);
        ptx::tmem_ld_x32(tS + 32, su + 32);
        ptx::tmem_ld_x32(tS + 64, su + 64);
        ptx::tmem_ld_x32(tS + 96, su + 96);
        ptx::tmem_wait_ld();
        // S_i has been read: the leader may compute S_i of the next block into it
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair::arrive_remote(&s_consumed[wg], 0);
        float s[128];
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = __uint_as_float(su[c]);
        const int c0 = j * 128;
        // ragged key tail; causal: blocks past the first row's diagonal (fully masked rows of
        // CTA 0 keep m: block 0 always holds a visible key, so m is finite by then)
        const bool need_mask = c0 + 128 > nk || (CAUSAL && c0 + 127 > r0 + off);
        if (need_mask) {
          const int lim = CAUSAL ? min(nk - 1, grow + off) : nk - 1;
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c0 + c > lim) s[c] = -INFINITY;
        }
        // row max: a tree of 3-input maxima for causal (+1-1.3%, same-box A/B), the serial chain
        // non-causal (the tree measured equal there, and 1.7% slower before the ping-pong)
        float mx;
        if constexpr (CAUSAL) {
          mx = ptx::tree_max<128>(s);
        } else {
          mx = s[0];
#pragma unroll
          for (int c = 1; c < 128; ++c) mx = fmaxf(mx, s[c]);
        }
        if (tr) FA2_TRACE(1, wg, j);
        const float m_new = fmaxf(m_used, mx * sl2);
        const bool rescale = (m_new - m_used) > 8.0f;
        float alpha = 1.f;
        if (rescale) {
          alpha = ptx::ex2(m_used - m_new);
          m_used = m_new;
        }
        const float base = (m_used == -INFINITY) ? 0.f : m_used;
        const float2 sl2x2 = make_float2(sl2, sl2), nb2 = make_float2(-base, -base);
        float2 rs2 = make_float2(0.f, 0.f);
        // P~ buffer and O: the previous P~V of this sub-tile must have completed (it was
        // issued a whole softmax ago, so this rarely waits); O is rescaled first, then P~
        // is stored chunk by chunk as the exponentials produce it, spreading the 32 KB of
        // SMEM writes over the MUFU-bound exponential phase instead of a burst at its end
        if (pv_count > 0) ptx::mbar_wait(&o_done[wg], (pv_count - 1) & 1);
        ptx::tc_fence_after();
        if (j > 0 && __any_sync(0xffffffffu, rescale)) {
#pragma unroll
          for (int ch = 0; ch < D / 32; ++ch) {
            uint32_t o[32];
            ptx::tmem_ld_x32(tO + ch * 32, o);
            ptx::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            ptx::tmem_st_x32(tO + ch * 32, o);
          }
          ptx::tmem_wait_st();
        }
        if (tr) FA2_TRACE(6, wg, j);
        pp_wait();
        if (tr) FA2_TRACE(7, wg, j);
        auto exp_block = [&](auto emu_tag) {
          constexpr int EMU = decltype(emu_tag)::value;
#pragma unroll
          for (int c = 0; c < 16; ++c) {   // chunk c: keys [8c, 8c + 8), 16 B of P~
            if (c == FA2_FWD_PP_C) pp_signal(j);
            uint32_t pk[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const int e = 4 * c + q;
              const float2 x = ptx::ffma2(make_float2(s[2 * e], s[2 * e + 1]), sl2x2, nb2);
              float2 pr;
              // emulated pairs spread among the MUFU ones (pairs 0 and 8 of 16 at EMU = 2: +0.3-0.7%
              // over a contiguous run, same-box A/B with the ping-pong)
              if (((e % 16) * EMU) % 16 < EMU) {
                pr = ptx::exp2_poly2(x);
              } else {
                pr.x = ptx::ex2(x.x);
                pr.y = ptx::ex2(x.y);
              }
              rs2 = ptx::fadd2(rs2, pr);
              pk[q] = ptx::pack2<BF16>(pr.x, pr.y);
            }
            // SW128 K-major: chunk c of box c / 8 at row * 128 + ((c ^ row) & 7) * 16
            ptx::sts_v4(sP_row + (c / 8) * L::Q_BOX + (((c % 8) ^ (row % 8)) * 16), pk[0], pk[1], pk[2], pk[3]);
          }
        };
        if (need_mask) exp_block(std::integral_constant<int, 0>{});
        else exp_block(std::integral_constant<int, kFwdPairEmuPairs>{});
        l_sum = l_sum * alpha + (rs2.x + rs2.y);
        if (tr) FA2_TRACE(2, wg, j);
        ptx::fence_proxy_async_smem();   // generic-proxy P~ writes -> visible to the tensor core
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) pair::arrive_remote(&p_full[wg], 0);
        if (tr) FA2_TRACE(3, wg, j);
        ++pv_count;
        ++gblk;
      }
      epilogue();   // (between sub-tile 0's empty steps instead: 1182 vs 1200 TFLOP/s causal N = 8k)
      if (threadIdx.x % 128 == 0) {
        fa2_tile_trace(p.trace, tn, wg, 2, fa2_gtime());
        fa2_tile_trace(p.trace, tn, wg, 3, clock64());
      }
    }
    if (!GEN && threadIdx.x % 128 == 0) ptx::bulk_wait<0>();   // the O stores have completed
  } else {
    ptx::setmaxnreg_dec<56>();
    if ((warp == 8 || warp == 11) && rank == 0) {
      // ============ MMA issuers (leader CTA): warp 8 -> sub-tile 0, warp 11 -> sub-tile 1 ============
      const int i = warp == 8 ? 0 : 1;
      constexpr uint32_t IDESC_S = ptx::idesc_f16(BF16, 256, 128, false, false);
      constexpr uint32_t IDESC_O = ptx::idesc_f16(BF16, 256, D, false, true);
      const uint64_t dQ = ptx::sw128_desc(ptx::smem_u32(sQ + i * L::Q_TILE), 16, 1024);
      const uint64_t dK = ptx::sw128_desc(ptx::smem_u32(sK), 16, 1024);
      const uint64_t dV = ptx::sw128_desc(ptx::smem_u32(sV), L::V_HALF, 1024);
      const uint64_t dP = ptx::sw128_desc(ptx::smem_u32(sP + i * L::P_TILE), 16, 1024);
      int kslot = 0, vslot = 0;
      uint32_t kphase = 0, vphase = 0, s_iss = 0, p_cnt = 0, o_use = 0;
      int it = 0;
      for (int n_ = 0, t; (t = tile_at(n_)) >= 0; ++n_) {
        const PairFwdTile w = decode(t);
        if (tile_empty(w)) continue;
        const int nb = nblk(w, i), nkv = nblk(w, 1);
        ptx::mbar_wait(&q_full[i], it & 1);
        ++it;
        if (nb == 0) {   // no row of sub-tile i sees a key: release Q_i now
          if (ptx::elect_one()) pair::commit_both(&q_empty[i]);
          __syncwarp();
        }
        for (int j = -1; j < nkv; ++j) {
          if (j + 1 >= nb && j + 1 < nkv) {   // sub-tile i skips this key block: release its K stage
            ptx::mbar_wait(&k_full[kslot], kphase);
            if (ptx::elect_one()) pair::commit_both(&k_empty[kslot]);
            __syncwarp();
            if (++kslot == STAGES) { kslot = 0; kphase ^= 1; }
          } else if (j + 1 < nkv) {   // S_i(j+1) = Q_i K_{j+1}^T once the softmax has read S_i(j)
            ptx::mbar_wait(&k_full[kslot], kphase);
            if (s_iss > 0) pair::wait_cluster(&s_consumed[i], (s_iss - 1) & 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < D * 2 / 32; ++k) {   // K = 16 per MMA: 4 per 128-B swizzle box
                const uint32_t offa = (k / 4) * L::Q_BOX + (k % 4) * 32;
                const uint32_t offb = kslot * L::K_HALF + (k / 4) * L::K_BOX + (k % 4) * 32;
                pair::mma_ss2(tmem + i * 128, dQ + (offa >> 4), dK + (offb >> 4), IDESC_S, k > 0 ? 1u : 0u);
              }
              pair::commit_both(&s_full[i]);
              if (j + 2 == nb) pair::commit_both(&q_empty[i]);   // Q_i's last S
              pair::commit_both(&k_empty[kslot]);
            }
            __syncwarp();
            if (it == 1) FA2_TRACE(5, i, j + 1);   // (it counts this pair's tiles, already incremented)
            ++s_iss;
            if (++kslot == STAGES) { kslot = 0; kphase ^= 1; }
          }
          if (j < 0) continue;
          // O_i += P~_i(j) V_j once both CTAs' softmax wrote P~_i(j)
          ptx::mbar_wait(&v_full[vslot], vphase);
          if (j >= nb) {   // skipped key block: release its V stage
            if (ptx::elect_one()) pair::commit_both(&v_empty[vslot]);
            __syncwarp();
            if (++vslot == STAGES) { vslot = 0; vphase ^= 1; }
            continue;
          }
          if (j == 0) {
            if (o_use > 0) pair::wait_cluster(&o_empty[i], (o_use - 1) & 1);
            ++o_use;
          }
          pair::wait_cluster(&p_full[i], p_cnt & 1);
          ++p_cnt;
          if (it == 1) FA2_TRACE(4, i, j);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {   // 16 keys per MMA
              const uint32_t offa = (k / 4) * L::Q_BOX + (k % 4) * 32;
              const uint32_t offb = vslot * L::V_HALF + k * 2048;
              pair::mma_ss2(tmem + 256 + i * D, dP + (offa >> 4), dV + (offb >> 4), IDESC_O, (j > 0 || k > 0) ? 1u : 0u);
            }
            pair::commit_both(&o_done[i]);
            pair::commit_both(&v_empty[vslot]);
          }
          __syncwarp();
          if (++vslot == STAGES) { vslot = 0; vphase ^= 1; }
        }
      }
    } else if ((warp == 9 || warp == 10) && lane == 0) {
      // ======= TMA producers: Q + K halves (warp 9), V halves (warp 10), into this CTA's SMEM =======
      const bool is_k = warp == 9;
      const uint64_t pol_kv = ptx::l2_policy_evict_last();
      const uint64_t pol_q = ptx::l2_policy_evict_first();
      int slot = 0;
      uint32_t phase = 0;
      int it = 0;
      // rows [row, row + box) of head `head` (of `heads`) at column c: fixed {d, N, B*heads},
      // packed {d, heads, T} (fa2_seq.cuh)
      auto load = [&](void* dst, const CUtensorMap* m, uint64_t* bar, int c, int row, int head, int heads, int b) {
        if constexpr (GEN) pair::tma_load_pair(dst, m, bar, c, head, row, m == &tm_q ? pol_q : pol_kv);
        else pair::tma_load_pair(dst, m, bar, c, row, b * heads + head, m == &tm_q ? pol_q : pol_kv);
      };
      for (int n_ = 0, t; (t = tile_at(n_)) >= 0; ++n_) {
        const PairFwdTile w = decode(t);
        if (tile_empty(w)) continue;
        const int mb = w.mb, nkv = nblk(w, 1);
        const int kvh = w.h / p.group, b = w.b;
        if (is_k) {
          for (int i = 0; i < 2; ++i) {
            if (it > 0) ptx::mbar_wait(&q_empty[i], (it - 1) & 1);
            if (rank == 0) ptx::mbar_arrive_expect_tx(&q_full[i], 2 * L::Q_TILE);
            for (int s = 0; s < 2; ++s)
              load(sQ + i * L::Q_TILE + s * L::Q_BOX, &tm_q, &q_full[i], s * 64, w.q0 + row0_of(mb, i), w.h, p.H, b);
          }
        }
        ++it;
        for (int j = 0; j < nkv; ++j) {
          ptx::mbar_wait(is_k ? &k_empty[slot] : &v_empty[slot], phase ^ 1);
          if (is_k) {   // key rows [128 j + 64 rank, +64), all d
            if (rank == 0) ptx::mbar_arrive_expect_tx(&k_full[slot], 2 * L::K_HALF);
            for (int s = 0; s < 2; ++s)
              load(sK + slot * L::K_HALF + s * L::K_BOX, &tm_k64, &k_full[slot], s * 64,
                   w.k0 + j * 128 + static_cast<int>(rank) * 64, kvh, p.Hkv, b);
          } else {      // key rows [128 j, +128), head-dim columns [64 rank, +64)
            if (rank == 0) ptx::mbar_arrive_expect_tx(&v_full[slot], 2 * L::V_HALF);
            load(sV + slot * L::V_HALF, &tm_v, &v_full[slot], static_cast<int>(rank) * 64, w.k0 + j * 128, kvh, p.Hkv, b);
          }
          if (++slot == STAGES) { slot = 0; phase ^= 1; }
        }
      }
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

}  // namespace fa2
