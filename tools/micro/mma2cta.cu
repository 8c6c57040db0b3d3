// Microbenchmark: tcgen05.mma with cta_group::2 (a CTA pair issues one M = 256 MMA,
// each CTA holding its 128 rows of A and half of B's N columns in its own shared
// memory) on sm_100a.  Validates the pair mechanics (cluster launch, 2-SM TMEM
// allocation, leader-issued MMA, multicast commit) and measures cycles per K = 16 step
// for the forward's S = Q K^T shape (N = 128 and N = 64), against the 1-SM rate
// (tools/micro/mma_rate.cu: 64 cycles at N = 128, 48 at N = 64, SMEM-bound).
#include <cstdio>
#include <cstdint>
#include "../../paper_2307_08691_b200/csrc/sm100_ptx.cuh"
using namespace fa2;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k(unsigned long long* cyc, int reps) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (96 * 1024) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(ptx::smem_u32(&slot)), "r"(512));
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  unsigned long long t0 = clock64();
  if (rank == 0 && threadIdx.x < 32) {
    // A: 128 rows x 128 B per swizzle box (this CTA's rows; the peer's at the same offset)
    // B: N / 2 rows per CTA (K-major, 128-B rows), boxes of (N / 2) x 128 B
    const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
    const uint64_t dA = ptx::sw128_desc(a, 16, 1024), dB = ptx::sw128_desc(b, 16, 1024);
    constexpr uint32_t ID = ptx::idesc_f16(true, 256, N, false, false);
    const int BOX = (N / 2) * 128;
    if (ptx::elect_one()) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t offA = (kk / 4) * 16384 + (kk % 4) * 32, offB = (kk / 4) * BOX + (kk % 4) * 32;
          const uint64_t da = dA + (offA >> 4), db = dB + (offB >> 4);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       :: "r"(tmem), "l"(da), "l"(db), "r"(ID), "r"(1u) : "memory");
        }
      }
      // arrive on `bar` in both CTAs of the pair when the MMAs complete
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(ptx::smem_u32(&bar)), "h"((uint16_t)0x3) : "memory");
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    ptx::mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  cluster_sync();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
  }
}

// The pair backward's dQ shape: M = 128 (64 query rows per CTA), N = d = 128 (64 per CTA),
// K = 256 keys in 16 steps; A (dS) and B (K) MN-major, 128-B swizzled boxes of 128 rows.
template <int M>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) kq(unsigned long long* cyc, int reps) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < (96 * 1024) / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t rank = cluster_rank();
  if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
  if (threadIdx.x < 32)
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(ptx::smem_u32(&slot)), "r"(512));
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  unsigned long long t0 = clock64();
  if (rank == 0 && threadIdx.x < 32) {
    const uint32_t a = ptx::smem_u32(smem), b = a + 32768;
    const uint64_t dA = ptx::sw128_desc(a, 16384, 1024), dB = ptx::sw128_desc(b, 16384, 1024);
    constexpr uint32_t ID = ptx::idesc_f16(true, M, 128, true, true);
    if (ptx::elect_one()) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const uint32_t off = ((kk / 8) * 16384 + (kk % 8) * 2048) >> 4;
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                       :: "r"(tmem), "l"(dA + off), "l"(dB + off), "r"(ID), "r"(1u) : "memory");
        }
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(ptx::smem_u32(&bar)), "h"((uint16_t)0x3) : "memory");
    }
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    ptx::mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  }
  ptx::tc_fence_before();
  cluster_sync();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::);
  }
}

template <int M>
void runq(unsigned long long* cyc) {
  const int reps = 512, smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(kq<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {2, 148}) {
    kq<M><<<grid, 128, smem>>>(cyc, reps);
    kq<M><<<grid, 128, smem>>>(cyc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("kq M=%d grid %d: %s\n", M, grid, cudaGetErrorString(e)); return; }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = mx > h[i] ? mx : h[i];
    const double per = mx / (reps * 16.0);
    printf("cta_group::2 M%d N128 MN-major A,B (dQ shape) grid %3d: %.1f cycles per K=16 MMA (full-rate floor %d)\n", M,
           grid, per, M * 128 / 256);
  }
}

template <int N>
void run(unsigned long long* cyc) {
  const int reps = 512, smem = 96 * 1024 + 1024;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int grid : {2, 148}) {
    k<N><<<grid, 128, smem>>>(cyc, reps);
    k<N><<<grid, 128, smem>>>(cyc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("N=%d grid %d: %s\n", N, grid, cudaGetErrorString(e)); return; }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = mx > h[i] ? mx : h[i];
    const double per = mx / (reps * 8.0);
    printf("cta_group::2 M256 N%-3d grid %3d: %.1f cycles per K=16 MMA (per-SM floor %d)\n", N, grid, per, 128 * N / 256);
  }
}

int main() {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  run<128>(cyc);
  run<64>(cyc);
  run<256>(cyc);
  runq<128>(cyc);
  runq<256>(cyc);
  return 0;
}
