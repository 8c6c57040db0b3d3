// Microbenchmark: tcgen05.mma issue-to-completion rate on sm_100a for the shapes the
// forward uses.  One CTA per SM, one thread issues R x 8 MMAs (K = 16 each, bf16, fp32
// accumulate) back to back into TMEM, commits, waits.  Reports cycles per K=16 MMA and
// the fraction of the 8192 flop/clk/SM floor.  SMEM operands hold zeros (timing only).
#include <cstdio>
#include <cstdint>
#include "../../paper_2307_08691_b200/csrc/sm100_ptx.cuh"
using namespace fa2;

template <int MODE, int SPIN = 0>
__global__ void __launch_bounds__(384, 1) k(unsigned long long* cyc, int reps) {
  __shared__ volatile int done;
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t bar2[8];
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (160 * 1024) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) { done = 0; ptx::mbar_init(&bar, 1); for (int i = 0; i < 8; ++i) ptx::mbar_init(&bar2[i], 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32) ptx::tmem_alloc(&slot, 512);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x < 32) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
    constexpr int N = MODE == 1 ? 256 : MODE == 4 ? 64 : 128;
    const uint64_t dA = ptx::sw128_desc(a, 16, 1024);
    const uint64_t dB = ptx::sw128_desc(b, 16, 1024);
    const uint64_t dBmn = ptx::sw128_desc(b, 16384, 1024);
    constexpr uint32_t ID = ptx::idesc_f16(true, 128, N, false, false);
    constexpr uint32_t IDmn = ptx::idesc_f16(true, 128, 128, false, true);
    const int BOX = N * 128;   // bytes of one 128-B-wide box of the B tile
    __syncwarp();
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32;
          const uint32_t offB = (kk / 4) * BOX + (kk % 4) * 32;
          if constexpr (MODE >= 5) break;
          if constexpr (MODE == 0 || MODE == 1 || MODE == 4)
            ptx::mma_ss(tmem, dA + (offA >> 4), dB + (offB >> 4), ID, 1u);
          else if constexpr (MODE == 2)   // A from TMEM (8 columns per K = 16), B K-major
            ptx::mma_ts(tmem, tmem + 384 + kk * 8, dB + (offB >> 4), ID, 1u);
          else if constexpr (MODE == 3)   // A from TMEM, B MN-major (the P~V shape)
            ptx::mma_ts(tmem + 128, tmem + 384 + kk * 8, dBmn + ((kk * 2048) >> 4), IDmn, 1u);
        }
        if constexpr (MODE == 9) {   // SS N128 with one commit per 8 MMAs
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32;
            const uint32_t offB = (kk / 4) * BOX + (kk % 4) * 32;
            ptx::mma_ss(tmem, dA + (offA >> 4), dB + (offB >> 4), ID, 1u);
          }
          ptx::mma_commit(&bar2[r & 3]);
        }
        if constexpr (MODE == 8 || MODE == 10) {   // HB block: S0, S1 (N = 64 SS, K = 128), P~V0, P~V1 (TS, K = 64, N = 128)
          constexpr uint32_t ID64 = ptx::idesc_f16(true, 128, 64, false, false);
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
              const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32;
              const uint32_t offB = (kk / 4) * 16384 + (kk % 4) * 32 + (r & 1) * 8192;
              ptx::mma_ss(tmem + 256 + i * 64, dA + (offA >> 4), dB + (offB >> 4), ID64, kk > 0 ? 1u : 0u);
            }
          if constexpr (MODE == 10) { ptx::mma_commit(&bar2[0]); ptx::mma_commit(&bar2[1]); ptx::mma_commit(&bar2[2]); }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::mma_ts(tmem + i * 128, tmem + 384 + i * 64 + (r & 1) * 32 + kk * 8,
                          dBmn + (((r & 1) * 8192 + kk * 2048) >> 4), IDmn, 1u);
          if constexpr (MODE == 10) { ptx::mma_commit(&bar2[3]); ptx::mma_commit(&bar2[4]); ptx::mma_commit(&bar2[5]); }
        }
        if constexpr (MODE >= 5 && MODE <= 7) {   // P~V (A = TMEM cols of S) then S into the same (5, 7) or other (6) columns
          const uint32_t sub = (MODE == 7) ? (r & 1) * 128u : 0u;
          const uint32_t sd = (MODE == 6 ? 128u : 0u) + sub;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            ptx::mma_ts(tmem + 256 + sub / 2, tmem + sub + kk * 8, dBmn + ((kk * 2048) >> 4), IDmn, 1u);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32;
            const uint32_t offB = (kk / 4) * BOX + (kk % 4) * 32;
            ptx::mma_ss(tmem + sd, dA + (offA >> 4), dB + (offB >> 4), ID, kk > 0 ? 1u : 0u);
          }
        }
      }
      ptx::mma_commit(&bar);
    }
    __syncwarp();
    ptx::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; done = 1; }
  } else if (SPIN && threadIdx.x < 32 * (1 + SPIN)) {   // SPIN warps polling an mbarrier that never completes
    const uint32_t a = ptx::smem_u32(&bar2[7]);
    while (!done) { (void)ptx::mbar_try_wait(a, 0); }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

template <int MODE, int SPIN = 0>
void run(const char* name, unsigned long long* cyc) {
  const int reps = 512;
  const int smem = 160 * 1024 + 1024;
  cudaFuncSetAttribute(k<MODE, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {1, 148}) {
    k<MODE, SPIN><<<grid, 384, smem>>>(cyc, reps);
    k<MODE, SPIN><<<grid, 384, smem>>>(cyc, reps);
    unsigned long long h[148];
    cudaMemcpy(h, cyc, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = mx > h[i] ? mx : h[i];
    const int N = MODE == 1 ? 256 : MODE == 4 ? 64 : 128;
    const double per = (MODE == 8 || MODE == 10) ? mx / reps : mx / (reps * 8.0 * (MODE >= 5 ? 2 : 1));
    const double floor_c = 128.0 * N / 256.0;
    printf("%-22s grid %3d: %.1f cycles per K=16 MMA (floor %.0f) -> %.1f%% of floor\n", name, grid, per, floor_c,
           100.0 * floor_c / per);
  }
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<0>("SS M128 N128 (S)", cyc);
  run<1>("SS M128 N256", cyc);
  run<4>("SS M128 N64", cyc);
  run<2>("TS M128 N128 Kmaj B", cyc);
  run<3>("TS M128 N128 MN B(PV)", cyc);
  run<5>("PV then S, aliased", cyc);
  run<6>("PV then S, separate", cyc);
  run<7>("2 subtiles PV,S aliased", cyc);
  run<8>("HB block (cyc/block, floor 1024)", cyc);
  run<10>("HB block + 6 commits (cyc/block)", cyc);
  run<8, 4>("HB block, 4 warps polling", cyc);
  run<8, 10>("HB block, 10 warps polling", cyc);
  run<0, 10>("SS N128, 10 warps polling", cyc);
  run<9>("SS N128 + commit per 8", cyc);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
