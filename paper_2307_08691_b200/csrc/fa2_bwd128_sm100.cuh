// FlashAttention-2 backward (Alg. 2), d = 128 kernel for
// sm_100a with 128-row query tiles (every MMA has N = 128).
//
// Orientation: key rows are TMEM lanes (M = 128).  A work tile is one key/value
// block K_j, V_j (128 rows; with GQA, every query head of the group).
// TMEM (512 columns):  S^T [0,128) | dP^T [128,256) | dV [256,384) | dK [384,512)
//   S^T_i  = K_j Q_i^T  -> P^T_i = exp(S^T - L_i) written in place (bf16 pairs)
//   dP^T_i = V_j dO_i^T -> dS^T_i = P^T o (dP^T - D_i) written in place, and to SMEM
//   dV += P^T dO_i (A from TMEM), dK += dS^T Q_i (A from TMEM)
//   dQ^T_i = K_j^T dS^T_i -> written over the dP^T columns, read out, scaled and
//                            reduce-added (fp32 bulk copies) into dQ_acc
// MMA issue order for query tile i:
//   dV(i) [P^T ready], dP^T(i) [dQ^T(i-1) read out], S^T(i+1), dK(i)+dQ^T(i) [dS^T ready]
// so the tensor core always has queued work: the compute warps derive dS^T(i)
// while S^T(i+1) runs and P^T(i+1) while dK(i)/dQ^T(i) run; the dQ^T(i-1) read-out
// hides behind dV(i).  MMAs complete in issue order, which orders every in-place
// reuse of the S^T and dP^T columns.
//
// Warp roles (512 threads): warps 0-7 two compute warpgroups (query columns
// [64w, 64w+64) each); warps 8-11 dQ read-out + fp32 bulk reduce-add (staged 16
// query rows at a time, two 8 KB buffers in flight); warp 12 MMA issuer; warp 13
// TMA producer; warps 14-15 idle.
//
// The dQ reduce-add is this kernel's co-bound: the chip's L2 fp32 reduction rate
// measured ~5.8 TB/s (~20 B/clk/SM; tools/micro/bulkred.cu, lsured.cu -- the same
// through TMA bulk reductions, LSU red.global, or both), and each 128x128 tile
// sends 64 KB of partials: >= ~3300 cycles/tile against a 2560-cycle MMA floor.
#pragma once
#include "fa2_bwd_sm100.cuh"

// dQ^T reduce-added straight from registers (red.global.add.v4.f32) into a chunked dQ_acc
// layout ([q/4][d][4] per 128-row tile) instead of SMEM staging + TMA bulk reduce-adds
#ifndef FA2_BWD_DQ_LSU
#define FA2_BWD_DQ_LSU 0
#endif
#ifndef FA2_BWD_RED_PACE
#define FA2_BWD_RED_PACE 0
#endif

// FMA-pipe exponential pairs per 16 in the P^T phase (unmasked tiles, square geometry)
#ifndef FA2_BWD_EMU
#define FA2_BWD_EMU 4
#endif

namespace fa2 {

constexpr bool kBwdDqLsu = FA2_BWD_DQ_LSU != 0;

struct Bwd128Smem {
  static constexpr int D = 128, BM = 128;
  static constexpr int TILE = 128 * D * 2;        // K_j, V_j, Q_i or dO_i (32 KB)
  static constexpr int SUB = 128 * 128;           // one 64-column swizzle box (16 KB)
  static constexpr int QSTAGES = 2;               // Q_i (+ L_i, D_i) ring
  static constexpr int DS_TILE = 128 * BM * 2;    // dS^T (bf16), B operand of the dQ MMA (32 KB)
  static constexpr int DQ_ROWS = 16;              // query rows per dQ reduce-add round (8 KB fp32)
  static constexpr int DQ_NBUF = 2;               // staging buffers (two reduce-adds in flight)
  static constexpr int DQ_BUF = DQ_ROWS * D * 4;
  static constexpr int DQ_STAGE = DQ_NBUF * DQ_BUF;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + TILE;
  static constexpr int OFF_Q = OFF_V + TILE;
  static constexpr int OFF_DO = OFF_Q + QSTAGES * TILE;
  static constexpr int OFF_DST = OFF_DO + TILE;
  static constexpr int OFF_DQ = OFF_DST + DS_TILE;
  static constexpr int OFF_VEC = OFF_DQ + DQ_STAGE;               // [QSTAGES][2][BM] floats: L2, D
  static constexpr int OFF_BAR = OFF_VEC + QSTAGES * 2 * BM * 4;
  // kv_full kv_empty q_full[2] q_empty[2] do_full do_empty s_full dp_full p_ready ds_ready
  // dq_full dq_empty dkv_full dkv_empty
  static constexpr int NBAR = 16;
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

template <bool BF16, bool CAUSAL, bool GEN>
__global__ void __launch_bounds__(kBwdThreads, 1)
fa2_bwd128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                  const __grid_constant__ CUtensorMap tm_dq, const BwdParams p,
               const __grid_constant__ SchedT<CAUSAL && !GEN> sched) {
  using L = Bwd128Smem;
  constexpr int D = 128, BM = 128, NSUB = 2;
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
  uint64_t* q_full = bars + 2;     // [2]
  uint64_t* q_empty = bars + 4;    // [2]
  uint64_t* do_full = bars + 6;
  uint64_t* do_empty = bars + 7;
  uint64_t* s_full = bars + 8;     // S^T(i) complete
  uint64_t* dp_full = bars + 9;    // dP^T(i) complete
  uint64_t* p_ready = bars + 10;   // P^T(i) written (8 warps)
  uint64_t* ds_ready = bars + 11;  // dS^T(i) written to TMEM and SMEM (8 warps)
  uint64_t* dq_full = bars + 12;   // dQ^T(i) complete
  uint64_t* dq_empty = bars + 13;  // dQ^T(i) read out of TMEM (4 warps)
  uint64_t* dkv_full = bars + 14;
  uint64_t* dkv_empty = bars + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(kv_empty, 1);
    for (int s = 0; s < 2; ++s) { ptx::mbar_init(&q_full[s], 1); ptx::mbar_init(&q_empty[s], 1); }
    ptx::mbar_init(do_full, 1);
    ptx::mbar_init(do_empty, 1);
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(dp_full, 1);
    ptx::mbar_init(p_ready, 8);
    ptx::mbar_init(ds_ready, 8);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(dq_empty, 4);
    ptx::mbar_init(dkv_full, 1);
    ptx::mbar_init(dkv_empty, 8);
    ptx::fence_mbar_init();
  }
  if (warp == 13 && lane == 0) {
    ptx::tma_prefetch_desc(&tm_q); ptx::tma_prefetch_desc(&tm_k); ptx::tma_prefetch_desc(&tm_v);
    ptx::tma_prefetch_desc(&tm_do);   // tm_dq unused: dQ goes out as contiguous 1D bulk reduce-adds
  }
  if (warp == 0) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t T_S = 0, T_DP = 128, T_DV = 256, T_DK = 384;

  const float* gD = p.dvec;
  const float* gL2 = p.dvec + p.acc_rows;

  if (warp < 8) {
    // ====================== compute warpgroups: P^T, dS^T ======================
    ptx::setmaxnreg_inc<152>();   // 152*256 + 152*128 + 48*128 == 128*512
    const int wg = warp / 4;
    const int r = threadIdx.x % 128;                   // key row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t sVec_a = ptx::smem_u32(sVec), sDST_a = ptx::smem_u32(sDST);
    const int c0 = wg * 64;                             // this warpgroup's 64 query columns
    uint32_t g = 0;
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
        const int i = bwd_q_tile(p, CAUSAL, w, x % nqt);
        const uint32_t slot = g & 1;
        const uint32_t vL2 = sVec_a + slot * 2 * BM * 4, vD = vL2 + BM * 4;
        // mask: causal tiles crossing the (bottom-right aligned, R22) diagonal and the ragged key tail;
        // query rows past N_q need none (their L*log2e is +inf in the workspace, so P = 0)
        const bool need_mask = (CAUSAL && nb * 128 + 127 > i * BM + off) || (nb * 128 + 128 > nk);
        // ---- P^T = exp2(S^T * scale*log2e - L*log2e), masked ----
        ptx::mbar_wait(&q_full[slot], (g >> 1) & 1);
        ptx::mbar_wait(s_full, g & 1);
        if (threadIdx.x == 0) FA2_BTRACE(0, g);
        ptx::tc_fence_after();
        // L, D of the warpgroup's 64 query columns come as float4 broadcasts; the exponent
        // argument as packed FFMA2; in unmasked tiles FA2_BWD_EMU of every 16 exponential
        // pairs run as the degree-3 polynomial on the FMA pipe (MUFU.EX2 is this phase's bound)
        float pf[64];
        const float2 sl2x2 = make_float2(p.scale_log2, p.scale_log2);
        auto p_block = [&](auto emu_tag) {
          constexpr int EMU = decltype(emu_tag)::value;
          // both 32-column chunks of S^T in one TMEM round trip (tcgen05.wait::ld waits for all)
          uint32_t sva[64];
          ptx::tmem_ld_x32(tmem + lane_base + T_S + c0, sva);
          ptx::tmem_ld_x32(tmem + lane_base + T_S + c0 + 32, sva + 32);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            const uint32_t* sv = sva + ch * 32;
#pragma unroll
            for (int e4 = 0; e4 < 8; ++e4) {
              const float4 l4 = ptx::lds_v4f(vL2 + (c0 + ch * 32 + e4 * 4) * 4);
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int e = e4 * 4 + 2 * h;   // column within this 32-column chunk
                const float2 x2 = ptx::ffma2(make_float2(__uint_as_float(sv[e]), __uint_as_float(sv[e + 1])), sl2x2,
                                             h == 0 ? make_float2(-l4.x, -l4.y) : make_float2(-l4.z, -l4.w));
                float2 pr;
                if ((ch * 16 + e / 2) % 16 < EMU) {
                  pr = ptx::exp2_poly2(x2);
                } else {
                  pr.x = ptx::ex2(x2.x);
                  pr.y = ptx::ex2(x2.y);
                }
                if (EMU == 0 && need_mask) {
                  const int q_row = i * BM + c0 + ch * 32 + e;
                  if ((CAUSAL && kv_row > q_row + off) || kv_row >= nk) pr.x = 0.f;
                  if ((CAUSAL && kv_row > q_row + 1 + off) || kv_row >= nk) pr.y = 0.f;
                }
                pf[ch * 32 + e] = pr.x;
                pf[ch * 32 + e + 1] = pr.y;
              }
            }
          }
        };
        // rows that see no key (R23) carry L*log2e = +inf: the polynomial would give 2^-125
        // instead of 0, so the general geometry keeps MUFU everywhere
        if (need_mask || GEN) p_block(std::integral_constant<int, 0>{});
        else p_block(std::integral_constant<int, FA2_BWD_EMU>{});
        if (threadIdx.x == 0) FA2_BTRACE(15, g);
        {
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) pk[e] = ptx::pack2<BF16>(pf[2 * e], pf[2 * e + 1]);
          // packed P^T over the first 32 of this warpgroup's own S^T columns
          ptx::tmem_st_x32(tmem + lane_base + T_S + c0, pk);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(p_ready);
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
            const float4 d4 = ptx::lds_v4f(vD + (c0 + ch * 32 + e4 * 4) * 4);
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
        ptx::tmem_st_x32(tmem + lane_base + T_DP + c0, dk);
        {
          // dS^T row r, query columns [c0, c0+64) -> SMEM region wg ([128 kv][64 q], 128-B swizzle)
          const uint32_t roff = wg * (128 * 128) + (r / 8) * 1024 + (r % 8) * 128;
#pragma unroll
          for (int q8 = 0; q8 < 8; ++q8)
            ptx::sts_v4(sDST_a + roff + ((q8 ^ (r % 8)) * 16), dk[4 * q8], dk[4 * q8 + 1], dk[4 * q8 + 2], dk[4 * q8 + 3]);
        }
        if (threadIdx.x == 0) FA2_BTRACE(12, g);
        ptx::tmem_wait_st();
        if (threadIdx.x == 0) FA2_BTRACE(13, g);
        ptx::fence_proxy_async_smem();
        if (threadIdx.x == 0) FA2_BTRACE(14, g);
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
      if (lane == 0) ptx::mbar_arrive(dkv_empty);
      ++it;
    }
  } else if (warp < 12) {
    // ====================== dQ read-out + fp32 reduce-add ======================
    ptx::setmaxnreg_inc<152>();
    const int r = threadIdx.x - 256;                    // 0..127 == TMEM lane == head-dim column d
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
        float* const dq_rows = p.dq_acc + (acc0 + i * BM) * D;                        // this tile's 128 rows
        ptx::mbar_wait(dq_full, g & 1);
        if (leader) FA2_BTRACE(9, g);
        ptx::tc_fence_after();
        uint32_t v[128];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) ptx::tmem_ld_x32(tmem + lane_base + T_DP + ch * 32, v + ch * 32);
        ptx::tmem_wait_ld();
        // dQ^T is in registers: the dP^T columns are free for the next tile
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(dq_empty);
        if (leader) FA2_BTRACE(10, g);
        if constexpr (kBwdDqLsu) {
          // straight from registers: the tile's dQ_acc block is laid out [q/4][d][4], so one
          // red.v4 of a warp (32 consecutive d, 4 query rows each) covers 512 contiguous bytes
          if (p.dq_sem != nullptr) {
            if (leader) dq_sem_wait(dq_sem_ptr(p, acc0, i), dq_rank(p, nb, x % nqt));
            ptx::named_bar_sync(1, 128);
          }
          float* const dst = dq_rows + r * 4;
          const long long t0 = clock64();
#pragma unroll
          for (int qc = 0; qc < BM / 4; ++qc) {
            if (FA2_BWD_RED_PACE > 0 && qc % 4 == 0 && qc > 0)
              while (clock64() - t0 < static_cast<long long>(qc / 4) * FA2_BWD_RED_PACE) {}
            ptx::red_add_v4_f32(dst + qc * (4 * D), __uint_as_float(v[4 * qc]) * p.scale,
                                __uint_as_float(v[4 * qc + 1]) * p.scale, __uint_as_float(v[4 * qc + 2]) * p.scale,
                                __uint_as_float(v[4 * qc + 3]) * p.scale);
          }
          if (p.dq_sem != nullptr) {   // the reductions are performed before the release is observed
            __threadfence();
            ptx::named_bar_sync(1, 128);
            if (leader) ptx::st_release_gpu(dq_sem_ptr(p, acc0, i), dq_rank(p, nb, x % nqt) + 1);
          }
          if (leader) FA2_BTRACE(16, g);
          continue;
        }
        // rounds of DQ_ROWS query rows, row-major [rows][128] fp32 staging (a warp's 32 lanes
        // write 128 contiguous bytes: conflict-free), each round one contiguous 8 KB bulk
        // reduce-add (dQ_acc rows are d*4 = 512 B apart, so DQ_ROWS rows are contiguous)
#pragma unroll
        for (int rd = 0; rd < BM / L::DQ_ROWS; ++rd) {
          const int buf = rd % L::DQ_NBUF;
          if (leader) {
            ptx::bulk_wait_read<L::DQ_NBUF - 1>();
            // deterministic mode: wait for this key block's turn on dQ tile (bhq, i)
            if (p.dq_sem != nullptr && rd == 0) dq_sem_wait(dq_sem_ptr(p, acc0, i), dq_rank(p, nb, x % nqt));
          }
          ptx::named_bar_sync(1, 128);
#pragma unroll
          for (int q = 0; q < L::DQ_ROWS; ++q)
            ptx::sts_f32(sDQ_a + buf * L::DQ_BUF + q * (D * 4) + r * 4, __uint_as_float(v[rd * L::DQ_ROWS + q]) * p.scale);
          ptx::fence_proxy_async_smem();
          ptx::named_bar_sync(1, 128);
          if (leader) {
            ptx::bulk_reduce_add_f32(dq_rows + rd * (L::DQ_ROWS * D),
                                     sDQ + buf * L::DQ_BUF, L::DQ_BUF);
            ptx::bulk_commit();
          }
        }
        if (leader && p.dq_sem != nullptr) dq_sem_release(dq_sem_ptr(p, acc0, i), dq_rank(p, nb, x % nqt));
        if (leader) FA2_BTRACE(16, g);
      }
    }
    if (!kBwdDqLsu && leader) ptx::bulk_wait<0>();
  } else if (warp == 12) {
    // ================== MMA issuer: whole warp, one elected lane issues ==================
    ptx::setmaxnreg_dec<48>();
    constexpr uint32_t IDESC = ptx::idesc_f16(BF16, 128, 128, false, false);     // S^T, dP^T
    constexpr uint32_t IDESC_G = ptx::idesc_f16(BF16, 128, D, false, true);     // dV, dK
    constexpr uint32_t IDESC_Q = ptx::idesc_f16(BF16, 128, 128, true, true);    // dQ^T
    const uint64_t dK_k = ptx::sw128_desc(ptx::smem_u32(sK), 16, 1024);
    const uint64_t dV_k = ptx::sw128_desc(ptx::smem_u32(sV), 16, 1024);
    const uint64_t dK_mn = ptx::sw128_desc(ptx::smem_u32(sK), L::SUB, 1024);
    const uint64_t dQ_k = ptx::sw128_desc(ptx::smem_u32(sQ), 16, 1024);
    const uint64_t dO_k = ptx::sw128_desc(ptx::smem_u32(sDO), 16, 1024);
    const uint64_t dQ_mn = ptx::sw128_desc(ptx::smem_u32(sQ), L::SUB, 1024);
    const uint64_t dO_mn = ptx::sw128_desc(ptx::smem_u32(sDO), L::SUB, 1024);
    const uint64_t dS_mn = ptx::sw128_desc(ptx::smem_u32(sDST), L::SUB, 1024);
    auto mma_s = [&](uint32_t slot) {   // S^T = K_j Q^T  (both K-major, K = d)
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t off = ((k / 4) * L::SUB + (k % 4) * 32) >> 4;
        ptx::mma_ss(tmem + T_S, dK_k + off, dQ_k + ((slot * L::TILE) >> 4) + off, IDESC, k > 0 ? 1u : 0u);
      }
    };
    auto mma_dp = [&]() {               // dP^T = V_j dO^T
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t off = ((k / 4) * L::SUB + (k % 4) * 32) >> 4;
        ptx::mma_ss(tmem + T_DP, dV_k + off, dO_k + off, IDESC, k > 0 ? 1u : 0u);
      }
    };
    uint32_t g = 0;
    int it = 0;
    uint32_t dkv_uses = 0;
    for (int n_ = 0, t; (t = sched_tile(sched, n_, p.num_tiles)) >= 0; ++n_) {
      BwdTile w;
      if (!bwd_tile<GEN>(p, CAUSAL, t, w) || w.nqt == 0) continue;
      const uint32_t n = static_cast<uint32_t>(w.nqt * w.nh);
      const uint32_t g0 = g;
      ptx::mbar_wait(kv_full, it & 1);
      // prologue: S^T of the first query tile (the S^T columns were last read by dV of the
      // previous work tile, issued earlier: in order)
      ptx::mbar_wait(&q_full[g0 & 1], (g0 >> 1) & 1);
      ptx::tc_fence_after();
      if (ptx::elect_one()) { mma_s(g0 & 1); ptx::mma_commit(s_full); }
      __syncwarp();
      if (dkv_uses > 0) ptx::mbar_wait(dkv_empty, (dkv_uses - 1) & 1);   // previous dK/dV drained
      for (uint32_t x = g0; x < g0 + n; ++x) {
        const uint32_t slot = x & 1;
        const bool first = (x == g0);
        // dV += P^T dO  (A: packed P^T of query columns [0,64) at cols 0-31, [64,128) at 64-95)
        ptx::mbar_wait(do_full, x & 1);
        ptx::mbar_wait(p_ready, x & 1);
        FA2_BTRACE(4, x);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BM / 16; ++k)
            ptx::mma_ts(tmem + T_DV, tmem + T_S + (k / 4) * 64 + (k % 4) * 8, dO_mn + ((k * 2048) >> 4), IDESC_G,
                        (!first || k > 0) ? 1u : 0u);
        }
        __syncwarp();
        // dP^T = V dO^T into the dP^T columns once dQ^T of the previous tile has been read out
        if (x > 0) ptx::mbar_wait(dq_empty, (x - 1) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          mma_dp();
          ptx::mma_commit(dp_full);
          ptx::mma_commit(do_empty);
        }
        __syncwarp();
        FA2_BTRACE(5, x);
        // S^T of the next query tile (its P^T columns were just consumed by dV, in order)
        if (x + 1 < g0 + n) {
          ptx::mbar_wait(&q_full[(x + 1) & 1], ((x + 1) >> 1) & 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) { mma_s((x + 1) & 1); ptx::mma_commit(s_full); }
          __syncwarp();
          FA2_BTRACE(6, x);
        }
        // dK += dS^T Q ; dQ^T = K^T dS^T (over the dP^T / dS^T columns, after dK read them)
        ptx::mbar_wait(ds_ready, x & 1);
        FA2_BTRACE(7, x);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BM / 16; ++k)
            ptx::mma_ts(tmem + T_DK, tmem + T_DP + (k / 4) * 64 + (k % 4) * 8,
                        dQ_mn + ((slot * L::TILE + k * 2048) >> 4), IDESC_G, (!first || k > 0) ? 1u : 0u);
          ptx::mma_commit(&q_empty[slot]);
#pragma unroll
          for (int k = 0; k < 128 / 16; ++k) {
            const uint32_t off = (k * 2048) >> 4;
            ptx::mma_ss(tmem + T_DP, dK_mn + off, dS_mn + off, IDESC_Q, k > 0 ? 1u : 0u);
          }
          ptx::mma_commit(dq_full);
        }
        __syncwarp();
        FA2_BTRACE(8, x);
      }
      g = g0 + n;
      ++dkv_uses;
      if (ptx::elect_one()) {
        ptx::mma_commit(dkv_full);
        ptx::mma_commit(kv_empty);
      }
      __syncwarp();
      ++it;
    }
  } else if (warp == 13) {
    // ============================ TMA producer ============================
    ptx::setmaxnreg_dec<48>();
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
        ptx::mbar_arrive_expect_tx(kv_full, 2 * L::TILE);
        for (int s = 0; s < NSUB; ++s) {
          tma_load_rows<GEN>(sK + s * L::SUB, &tm_k, kv_full, p.geom, s * 64, w.sq.k0 + nb * 128, w.kvh, w.sq.bc, p.Hkv, pol_kv);
          tma_load_rows<GEN>(sV + s * L::SUB, &tm_v, kv_full, p.geom, s * 64, w.sq.k0 + nb * 128, w.kvh, w.sq.bc, p.Hkv, pol_kv);
        }
        for (int x = 0; x < nqt * w.nh; ++x, ++g) {
          const int i = bwd_q_tile(p, CAUSAL, w, x % nqt), hq = w.kvh * p.group + w.h0 + x / nqt;
          const uint32_t slot = g & 1;
          // Q_i, L_i, D_i (2-stage ring; released after dK(i))
          if (g >= 2) ptx::mbar_wait(&q_empty[slot], ((g >> 1) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&q_full[slot], L::TILE + 2 * BM * 4);
          for (int s = 0; s < NSUB; ++s)
            tma_load_rows<GEN>(sQ + slot * L::TILE + s * L::SUB, &tm_q, &q_full[slot], p.geom, s * 64, w.sq.q0 + i * BM, hq,
                          w.sq.bc, p.H, pol_q);
          float* vdst = sVec + slot * 2 * BM;
          const long long voff = bwd_acc_row0<GEN>(p, w, hq) + static_cast<long long>(i) * BM;
          ptx::bulk_load_1d(vdst, gL2 + voff, BM * 4, &q_full[slot]);
          ptx::bulk_load_1d(vdst + BM, gD + voff, BM * 4, &q_full[slot]);
          // dO_i (single stage; released after dP^T(i))
          if (g >= 1) ptx::mbar_wait(do_empty, (g - 1) & 1);
          ptx::mbar_arrive_expect_tx(do_full, L::TILE);
          for (int s = 0; s < NSUB; ++s)
            tma_load_rows<GEN>(sDO + s * L::SUB, &tm_do, do_full, p.geom, s * 64, w.sq.q0 + i * BM, hq, w.sq.bc, p.H, pol_q);
        }
        ++it;
      }
    }
  } else {
    ptx::setmaxnreg_dec<48>();
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
