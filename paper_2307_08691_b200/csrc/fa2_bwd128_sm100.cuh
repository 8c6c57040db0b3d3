// FlashAttention-2 backward (Alg. 2), d = 128 kernel for
// sm_100a with a double-region TMEM pipeline.
//
// Same math and orientation as fa2_bwd_kernel (key rows = TMEM lanes, B_r = 64
// query rows per tile, dQ produced transposed), but the per-query-tile TMEM
// state alternates between two 128-column regions R_b (b = tile parity):
//
//   cols [0,64)   S^T_i   --(compute)-->  P^T_i  (bf16, written in place)
//   cols [64,128) dP^T_i  --(compute)-->  dS^T_i (bf16, written in place)
//                 then dQ^T_i = K^T dS^T_i overwrites cols [64,128)
//
// plus dV_j [256,384) and dK_j [384,512) accumulators.  The MMA issue order is
//   grads(i) = {dV += P^T dO_i, dK += dS^T Q_i, dQ^T_i = K^T dS^T_i},
//   S^T_{i+2} (region b cols 0-63), [dQ^T_i read out] dP^T_{i+2} (cols 64-127)
// so the compute warpgroups work on tile i+1 while the tensor core runs
// grads(i), and no stage waits for the previous tile's gradient MMAs: MMAs
// complete in issue order, so "S/dP of tile i+2 complete" already implies that
// every reader of region b and of dS^T SMEM buffer b for tile i is done.
//
// Warp roles (512 threads): warps 0-7 two compute warpgroups (query columns
// [32w, 32w+32) each); warps 8-11 dQ readout + fp32 TMA reduce-add; warp 12
// MMA issuer; warp 13 TMA producer; warps 14-15 idle.
#pragma once
#include "fa2_bwd_sm100.cuh"

namespace fa2 {

struct Bwd128Smem {
  static constexpr int D = 128, BM = 64;
  static constexpr int KV_TILE = 128 * D * 2;     // K_j or V_j (32 KB)
  static constexpr int Q_TILE = BM * D * 2;       // Q_i or dO_i (16 KB)
  static constexpr int Q_SUB = BM * 128;          // one 64-column swizzle box of a Q/dO tile
  static constexpr int DS_TILE = 128 * BM * 2;    // dS^T (bf16), B operand of the dQ MMA
  static constexpr int DQ_TILE = BM * D * 4;      // fp32 staging for the dQ reduce-add
  static constexpr int STAGES = 3;                // Q_i / dO_i / L_i / D_i ring
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KV_TILE;
  static constexpr int OFF_Q = OFF_V + KV_TILE;
  static constexpr int OFF_DO = OFF_Q + STAGES * Q_TILE;
  static constexpr int OFF_DST = OFF_DO + STAGES * Q_TILE;       // [2] double-buffered
  static constexpr int OFF_DQ = OFF_DST + 2 * DS_TILE;
  static constexpr int OFF_VEC = OFF_DQ + DQ_TILE;                // [STAGES][2][BM] floats: L2, D
  static constexpr int OFF_BAR = OFF_VEC + STAGES * 2 * BM * 4;
  // kv_full kv_empty q_full[S] q_empty[S] s_full[2] ds_ready[2] dq_full[2] dq_empty[2] dkv_full dkv_empty
  static constexpr int NBAR = 2 + 2 * STAGES + 8 + 2;
  static constexpr int OFF_TMEM = OFF_BAR + NBAR * 8;
  static constexpr int BYTES = OFF_TMEM + 16;
  static constexpr int ALLOC = BYTES + 1024;
  static_assert(ALLOC <= 232448, "shared memory budget");
};

template <bool BF16, bool CAUSAL>
__global__ void __launch_bounds__(kBwdThreads, 1)
fa2_bwd128_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                  const __grid_constant__ CUtensorMap tm_dq, const BwdParams p) {
  using L = Bwd128Smem;
  constexpr int D = 128, BM = 64, STAGES = L::STAGES, NSUB = 2, HALF = 32;
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
  uint64_t* s_full = q_empty + STAGES;      // [2] S^T and dP^T of region b complete
  uint64_t* ds_ready = s_full + 2;          // [2] P^T / dS^T of region b written (8 warps)
  uint64_t* dq_full = s_full + 4;           // [2] dQ^T of region b complete
  uint64_t* dq_empty = s_full + 6;          // [2] dQ^T of region b read out (4 warps)
  uint64_t* dkv_full = s_full + 8;
  uint64_t* dkv_empty = s_full + 9;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(kv_empty, 1);
    for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&q_full[s], 1); ptx::mbar_init(&q_empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&s_full[b], 1);
      ptx::mbar_init(&ds_ready[b], 8);
      ptx::mbar_init(&dq_full[b], 1);
      ptx::mbar_init(&dq_empty[b], 4);
    }
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
  constexpr uint32_t T_DV = 256, T_DK = 384;

  const int N = p.N;
  const int n_q_blocks = (N + BM - 1) / BM;
  const float* gD = p.dvec;
  const float* gL2 = p.dvec + static_cast<size_t>(p.BH) * p.npad;
  auto decode = [&](int t, int& bh, int& nb) { bh = t / p.num_n_blocks; nb = t % p.num_n_blocks; };
  auto q_begin = [&](int nb) -> int { return CAUSAL ? (nb * 128) / BM : 0; };

  if (warp < 8) {
    // ====================== compute warpgroups: P^T, dS^T ======================
    const int wg = warp / 4;
    const int r = threadIdx.x % 128;                   // key row within the block == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const uint32_t sVec_a = ptx::smem_u32(sVec), sDST_a = ptx::smem_u32(sDST);
    uint32_t g = 0;
    int it = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      int bh, nb;
      decode(t, bh, nb);
      const int kv_row = nb * 128 + r;
      const int i0 = q_begin(nb), nqt = n_q_blocks - i0;
      const int bq0 = (bh / p.Hkv) * p.H + (bh % p.Hkv) * p.group;   // first query head of this kv head
      for (int x = 0; x < nqt * p.group; ++x, ++g) {
        const int i = i0 + x % nqt, bhq = bq0 + x / nqt;            // query tile, query head
        const uint32_t slot = g % STAGES, b = g & 1;
        ptx::mbar_wait(&q_full[slot], (g / STAGES) & 1);
        ptx::mbar_wait(&s_full[b], (g >> 1) & 1);
        if (threadIdx.x == 0) FA2_BTRACE(0, g);
        ptx::tc_fence_after();
        const uint32_t vL2 = sVec_a + slot * 2 * BM * 4;     // L_i * log2(e) for the BM query rows
        const uint32_t vD = vL2 + BM * 4;                     // D_i
        const bool need_mask = (CAUSAL && (i * BM < nb * 128 + 128)) || (nb * 128 + 128 > N);
        const uint32_t tR = tmem + lane_base + b * 128;       // this tile's region
        const int c0 = wg * HALF;                             // first query column of this warpgroup
        uint32_t sv[32], dpv[32];
        ptx::tmem_ld_x32(tR + c0, sv);
        ptx::tmem_ld_x32(tR + 64 + c0, dpv);
        ptx::tmem_wait_ld();
        uint32_t pk[16], dk[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float pp[2], dd[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = c0 + 2 * e + h;
            float pv = ptx::ex2(fmaf(__uint_as_float(sv[2 * e + h]), p.scale_log2, -ptx::lds_f32(vL2 + c * 4)));
            if (need_mask) {
              const int q_row = i * BM + c;
              if ((CAUSAL && kv_row > q_row) || kv_row >= N) pv = 0.f;
            }
            pp[h] = pv;
            dd[h] = pv * (__uint_as_float(dpv[2 * e + h]) - ptx::lds_f32(vD + c * 4));
          }
          pk[e] = ptx::pack2<BF16>(pp[0], pp[1]);
          dk[e] = ptx::pack2<BF16>(dd[0], dd[1]);
        }
        // P^T / dS^T in place over this warpgroup's own S^T / dP^T columns (A operands
        // of the dV / dK MMAs) and dS^T into SMEM buffer b (B operand of the dQ MMA)
        ptx::tmem_st_x16(tR + c0, pk);
        ptx::tmem_st_x16(tR + 64 + c0, dk);
        {
          const uint32_t roff = b * L::DS_TILE + (r / 8) * 1024 + (r % 8) * 128;
          const int cc0 = c0 / 8;                               // first 16-B chunk within the 128-B row
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            ptx::sts_v4(sDST_a + roff + (((cc0 + q4) ^ (r % 8)) * 16), dk[4 * q4], dk[4 * q4 + 1], dk[4 * q4 + 2],
                        dk[4 * q4 + 3]);
        }
        ptx::tmem_wait_st();
        ptx::fence_proxy_async_smem();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&ds_ready[b]);
        if (threadIdx.x == 0) FA2_BTRACE(3, g);
      }
      // ---- epilogue: dV_j (warpgroup 0), dK_j * scale (warpgroup 1) ----
      ptx::mbar_wait(dkv_full, it & 1);
      ptx::tc_fence_after();
      {
        const uint32_t tsrc = tmem + lane_base + (wg == 0 ? T_DV : T_DK);
        const float mul = wg == 0 ? 1.f : p.scale;
        uint8_t* dst = reinterpret_cast<uint8_t*>(wg == 0 ? p.dv : p.dk) + (static_cast<size_t>(bh) * N + kv_row) * (D * 2);
#pragma unroll
        for (int ch = 0; ch < D / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld_x32(tsrc + ch * 32, v);
          ptx::tmem_wait_ld();
          uint32_t o16[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) o16[e] = ptx::pack2<BF16>(__uint_as_float(v[2 * e]) * mul, __uint_as_float(v[2 * e + 1]) * mul);
          if (kv_row < N) {
            uint4* o = reinterpret_cast<uint4*>(dst + ch * 64);
#pragma unroll
            for (int e = 0; e < 4; ++e) o[e] = make_uint4(o16[4 * e], o16[4 * e + 1], o16[4 * e + 2], o16[4 * e + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(dkv_empty);
    }
  } else if (warp < 12) {
    // ====================== dQ readout + fp32 reduce-add ======================
    const int r = threadIdx.x - 256;                    // 0..127 == TMEM lane == head-dim column
    const uint32_t lane_base = static_cast<uint32_t>((warp % 4) * 32) << 16;
    const bool leader = (r == 0);
    const uint32_t sDQ_a = ptx::smem_u32(sDQ);
    uint32_t g = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int bh, nb;
      decode(t, bh, nb);
      const int i0 = q_begin(nb), nqt = n_q_blocks - i0;
      const int bq0 = (bh / p.Hkv) * p.H + (bh % p.Hkv) * p.group;   // first query head of this kv head
      for (int x = 0; x < nqt * p.group; ++x, ++g) {
        const int i = i0 + x % nqt, bhq = bq0 + x / nqt;            // query tile, query head
        const uint32_t b = g & 1;
        ptx::mbar_wait(&dq_full[b], (g >> 1) & 1);
        if (leader) FA2_BTRACE(7, g);
        ptx::tc_fence_after();
        uint32_t v[64];
        ptx::tmem_ld_x32(tmem + lane_base + b * 128 + 64, v);
        ptx::tmem_ld_x32(tmem + lane_base + b * 128 + 96, v + 32);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&dq_empty[b]);
        // staging buffer free? (the previous reduce-add has finished reading it)
        if (leader) ptx::bulk_wait_read<0>();
        ptx::named_bar_sync(1, 128);
        // lane r = head-dim column d; 64 columns = the 64 query rows; 4 fp32 boxes of 32 columns
        const uint32_t box = sDQ_a + (r / 32) * (BM * 128) + (r % 4) * 4;
#pragma unroll
        for (int q = 0; q < 64; ++q)
          ptx::sts_f32(box + q * 128 + ((((r % 32) / 4) ^ (q % 8)) * 16), __uint_as_float(v[q]) * p.scale);
        ptx::fence_proxy_async_smem();
        ptx::named_bar_sync(1, 128);
        if (leader) {
#pragma unroll
          for (int bx = 0; bx < D / 32; ++bx) ptx::tma_reduce_add_3d(&tm_dq, sDQ + bx * (BM * 128), bx * 32, i * BM, bhq);
          ptx::bulk_commit();
          FA2_BTRACE(8, g);
        }
      }
    }
    if (leader) ptx::bulk_wait<0>();
  } else if (warp == 12) {
    // ================== MMA issuer: whole warp, one elected lane issues ==================
    constexpr uint32_t IDESC_S = ptx::idesc_f16(BF16, 128, BM, false, false);   // S^T, dP^T
    constexpr uint32_t IDESC_G = ptx::idesc_f16(BF16, 128, D, false, true);     // dV, dK
    constexpr uint32_t IDESC_Q = ptx::idesc_f16(BF16, 128, 64, true, true);     // dQ^T
    const uint64_t dK_k = ptx::sw128_desc(ptx::smem_u32(sK), 16, 1024);
    const uint64_t dV_k = ptx::sw128_desc(ptx::smem_u32(sV), 16, 1024);
    const uint64_t dK_mn = ptx::sw128_desc(ptx::smem_u32(sK), 128 * 128, 1024);
    const uint64_t dQ_k = ptx::sw128_desc(ptx::smem_u32(sQ), 16, 1024);
    const uint64_t dO_k = ptx::sw128_desc(ptx::smem_u32(sDO), 16, 1024);
    const uint64_t dQ_mn = ptx::sw128_desc(ptx::smem_u32(sQ), L::Q_SUB, 1024);
    const uint64_t dO_mn = ptx::sw128_desc(ptx::smem_u32(sDO), L::Q_SUB, 1024);
    const uint64_t dS_mn = ptx::sw128_desc(ptx::smem_u32(sDST), 128 * 128, 1024);
    // S^T (qk) or dP^T (vdo) of tile g into region g&1
    auto issue_s = [&](uint32_t g) {
      const uint32_t slot = g % STAGES, b = g & 1;
      if (ptx::elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t akv = ((k / 4) * (128 * 128) + (k % 4) * 32) >> 4;
          const uint32_t aq = (slot * L::Q_TILE + (k / 4) * L::Q_SUB + (k % 4) * 32) >> 4;
          ptx::mma_ss(tmem + b * 128, dK_k + akv, dQ_k + aq, IDESC_S, k > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
    };
    auto issue_dp = [&](uint32_t g) {
      const uint32_t slot = g % STAGES, b = g & 1;
      if (ptx::elect_one()) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t akv = ((k / 4) * (128 * 128) + (k % 4) * 32) >> 4;
          const uint32_t aq = (slot * L::Q_TILE + (k / 4) * L::Q_SUB + (k % 4) * 32) >> 4;
          ptx::mma_ss(tmem + b * 128 + 64, dV_k + akv, dO_k + aq, IDESC_S, k > 0 ? 1u : 0u);
        }
        ptx::mma_commit(&s_full[b]);
      }
      __syncwarp();
    };
    uint32_t g = 0;
    int it = 0;
    uint32_t dkv_uses = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
      int bh, nb;
      decode(t, bh, nb);
      const int i0 = q_begin(nb);
      // query tiles of every query head of this key/value head's group (GQA)
      const uint32_t g0 = g, n = static_cast<uint32_t>((n_q_blocks - i0) * p.group);
      ptx::mbar_wait(kv_full, it & 1);
      // prologue: S^T / dP^T of the first two query tiles
      for (uint32_t x = g0; x < g0 + 2 && x < g0 + n; ++x) {
        ptx::mbar_wait(&q_full[x % STAGES], (x / STAGES) & 1);
        if (x >= 2) ptx::mbar_wait(&dq_empty[x & 1], ((x >> 1) - 1) & 1);   // region's previous dQ^T read out
        ptx::tc_fence_after();
        issue_s(x);
        issue_dp(x);
      }
      if (dkv_uses > 0) ptx::mbar_wait(dkv_empty, (dkv_uses - 1) & 1);     // previous dK/dV drained
      for (uint32_t x = g0; x < g0 + n; ++x) {
        const uint32_t slot = x % STAGES, b = x & 1;
        const bool first = (x == g0);
        ptx::mbar_wait(&ds_ready[b], (x >> 1) & 1);
        FA2_BTRACE(5, x);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          // dV += P^T dO_i ; dK += dS^T Q_i   (A from TMEM region b: the 16 packed columns of
          // query columns [0,32) sit at cols 0-15, those of [32,64) at cols 32-47)
#pragma unroll
          for (int k = 0; k < BM / 16; ++k) {
            const uint32_t acol = (k / 2) * 32 + (k % 2) * 8;
            const uint32_t boff = (slot * L::Q_TILE + k * 2048) >> 4;
            const uint32_t acc = (!first || k > 0) ? 1u : 0u;
            ptx::mma_ts(tmem + T_DV, tmem + b * 128 + acol, dO_mn + boff, IDESC_G, acc);
            ptx::mma_ts(tmem + T_DK, tmem + b * 128 + 64 + acol, dQ_mn + boff, IDESC_G, acc);
          }
          ptx::mma_commit(&q_empty[slot]);
          // dQ^T = K^T dS^T -> region b cols [64,128)
#pragma unroll
          for (int k = 0; k < 128 / 16; ++k) {
            const uint32_t off = (k * 2048) >> 4;
            ptx::mma_ss(tmem + b * 128 + 64, dK_mn + off, dS_mn + ((b * L::DS_TILE) >> 4) + off, IDESC_Q,
                        k > 0 ? 1u : 0u);
          }
          ptx::mma_commit(&dq_full[b]);
        }
        __syncwarp();
        FA2_BTRACE(6, x);
        if (x + 2 < g0 + n) {
          const uint32_t y = x + 2;
          ptx::mbar_wait(&q_full[y % STAGES], (y / STAGES) & 1);
          ptx::tc_fence_after();
          issue_s(y);                                      // cols 0-63: free once dV(x) has read P^T (in order)
          ptx::mbar_wait(&dq_empty[b], (x >> 1) & 1);      // cols 64-127: dQ^T(x) read out
          ptx::tc_fence_after();
          issue_dp(y);
          FA2_BTRACE(4, y);
        }
      }
      g = g0 + n;
      ++dkv_uses;
      if (ptx::elect_one()) {
        ptx::mma_commit(dkv_full);
        ptx::mma_commit(kv_empty);
      }
      __syncwarp();
    }
  } else if (warp == 13) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      uint32_t g = 0;
      int it = 0;
      const uint64_t pol_q = ptx::l2_policy_evict_last();
      const uint64_t pol_kv = ptx::l2_policy_evict_first();
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++it) {
        int bh, nb;
        decode(t, bh, nb);
        if (it > 0) ptx::mbar_wait(kv_empty, (it - 1) & 1);
        ptx::mbar_arrive_expect_tx(kv_full, 2 * L::KV_TILE);
        for (int s = 0; s < NSUB; ++s) {
          ptx::tma_load_3d_hint(sK + s * 128 * 128, &tm_k, kv_full, s * 64, nb * 128, bh, pol_kv);
          ptx::tma_load_3d_hint(sV + s * 128 * 128, &tm_v, kv_full, s * 64, nb * 128, bh, pol_kv);
        }
        const int i0 = q_begin(nb), nqt = n_q_blocks - i0;
        const int bq0 = (bh / p.Hkv) * p.H + (bh % p.Hkv) * p.group;
        for (int x = 0; x < nqt * p.group; ++x, ++g) {
          const int i = i0 + x % nqt, bhq = bq0 + x / nqt;
          const int slot = g % STAGES;
          if (g >= STAGES) ptx::mbar_wait(&q_empty[slot], ((g / STAGES) - 1) & 1);
          ptx::mbar_arrive_expect_tx(&q_full[slot], 2 * L::Q_TILE + 2 * BM * 4);
          for (int s = 0; s < NSUB; ++s) {
            ptx::tma_load_3d_hint(sQ + slot * L::Q_TILE + s * L::Q_SUB, &tm_q, &q_full[slot], s * 64, i * BM, bhq, pol_q);
            ptx::tma_load_3d_hint(sDO + slot * L::Q_TILE + s * L::Q_SUB, &tm_do, &q_full[slot], s * 64, i * BM, bhq, pol_q);
          }
          float* vdst = sVec + slot * 2 * BM;
          const size_t voff = static_cast<size_t>(bhq) * p.npad + static_cast<size_t>(i) * BM;
          ptx::bulk_load_1d(vdst, gL2 + voff, BM * 4, &q_full[slot]);
          ptx::bulk_load_1d(vdst + BM, gD + voff, BM * 4, &q_full[slot]);
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
