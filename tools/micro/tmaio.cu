// Per-SM data-movement budget: bulk (TMA) loads L2 -> SMEM alone, bulk fp32 reduce-adds
// SMEM -> L2 alone, and both at once from the same CTA (one thread each), with every SM
// busy.  Answers whether inbound loads and outbound reductions share one per-SM limit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tmaio.cu -o tmaio
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// MODE bit 0: loads, bit 1: bulk reduce-adds, bit 2: LSU red.global.add.v4 (4 warps)
template <int MODE>
__global__ void k(const float* src, float* dst, size_t span_floats, int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  constexpr int LB = 16384, RB = 8192;   // load / reduce op sizes
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 32768 / 4; i += blockDim.x) reinterpret_cast<float*>(sm + 4 * LB)[i] = 1e-6f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const long long t0 = clock64();
  const size_t nl = span_floats / (LB / 4), nr = span_floats / (RB / 4);
  if ((MODE & 1) && threadIdx.x == 0) {
    size_t slot = (size_t)blockIdx.x * 37 % nl;
    for (int it = 0; it < iters; ++it) {
      const int s = it % 4;
      if (it >= 4) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                       : "=r"(ok) : "r"(su32(&bar[s])), "r"(((it / 4) - 1) & 1) : "memory");
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(&bar[s])), "r"(LB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(su32(sm + s * LB)), "l"(src + slot * (LB / 4)), "r"(LB), "r"(su32(&bar[s])) : "memory");
      slot += gridDim.x;
      if (slot >= nl) slot -= nl;
    }
    for (int s = 0; s < 4; ++s) {
      uint32_t ok = 0;
      const int last = iters - 4 + ((s - iters % 4 + 4) % 4);
      while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok) : "r"(su32(&bar[s])), "r"((last / 4) & 1) : "memory");
    }
  }
  if ((MODE & 2) && threadIdx.x == 32) {
    size_t slot = (size_t)blockIdx.x * 53 % nr;
    const int riters = iters * LB / RB;
    for (int it = 0; it < riters; ++it) {
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                   :: "l"(dst + slot * (RB / 4)), "r"(su32(sm + 4 * LB + (it % 4) * RB)), "r"(RB) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      slot += gridDim.x;
      if (slot >= nr) slot -= nr;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if ((MODE & 4) && threadIdx.x >= 64 && threadIdx.x < 192) {
    // 4 warps, each red.v4 of a warp covers 512 contiguous bytes; same byte count as the bulk reduces
    const int w = (threadIdx.x - 64) / 32, l = threadIdx.x % 32;
    size_t slot = (size_t)blockIdx.x * 53 % nr;
    const int riters = iters * LB / RB;
    for (int it = 0; it < riters; ++it) {
      float* d = dst + slot * (RB / 4) + w * 512 + l * 4;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" :: "l"(d + j * 128), "f"(1e-6f), "f"(1e-6f), "f"(1e-6f),
                     "f"(1e-6f) : "memory");
      slot += gridDim.x;
      if (slot >= nr) slot -= nr;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(cyc, (unsigned long long)(clock64() - t0));
}

template <int MODE>
void run(const float* src, float* dst, size_t span, int blocks, const char* name) {
  const int iters = 4000;
  const int smem = 4 * 16384 + 32768;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 8);
  k<MODE><<<blocks, 192, smem>>>(src, dst, span, 100, cyc);
  cudaMemset(cyc, 0, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<blocks, 192, smem>>>(src, dst, span, iters, cyc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_dir = double(iters) * 16384;   // bytes per SM per direction used
  const double dirs = ((MODE & 1) ? 1 : 0) + ((MODE & 6) ? 1 : 0);
  printf("%-28s blocks=%3d  %8.3f ms  %6.1f B/clk/SM total (%.1f per direction)  chip %7.1f GB/s\n", name, blocks, ms,
         dirs * per_dir / c, per_dir / c, dirs * per_dir * blocks / ms / 1e6);
  cudaFree(cyc);
}

int main() {
  const size_t span = 8ull << 20;   // 32 MB of floats: L2-resident
  float *src, *dst;
  cudaMalloc(&src, span * 4); cudaMalloc(&dst, span * 4);
  cudaMemset(src, 0, span * 4); cudaMemset(dst, 0, span * 4);
  for (int blocks : {1, 148}) {
    run<1>(src, dst, span, blocks, "bulk loads");
    run<2>(src, dst, span, blocks, "bulk reduce-adds");
    run<3>(src, dst, span, blocks, "loads + bulk reduce-adds");
    run<4>(src, dst, span, blocks, "LSU red.v4");
    run<5>(src, dst, span, blocks, "loads + LSU red.v4");
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
