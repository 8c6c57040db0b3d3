// DSMEM bulk copies inside a 2-CTA cluster (cp.async.bulk.shared::cluster.shared::cta):
// one-way latency of an S-byte copy (ping-pong: CTA 0 copies to CTA 1, which waits on its
// mbarrier and copies back), and streaming throughput, next to an optional stream of
// bulk fp32 reduce-adds to global memory (the pair backward's dQ traffic).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 dsmemcp.cu -o dsmemcp
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
  return r;
}
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
                 "selp.u32 %0,1,0,p;\n\t}" : "=r"(ok) : "r"(su32(bar)), "r"(ph) : "memory");
}
__device__ __forceinline__ void expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t rbar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "r"(su32(src)), "r"(bytes), "r"(rbar) : "memory");
}

// MODE 0: ping-pong latency; MODE 1: both CTAs stream copies to each other (depth 2)
template <int MODE, bool GRED>
__global__ void __cluster_dims__(2, 1, 1) k(float* g, size_t span, int bytes, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 98304);
  const uint32_t me = rank(), pe = me ^ 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1e-6f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (GRED && threadIdx.x == 32) {
    size_t slot = blockIdx.x;
    const size_t nslots = span / 2048;
    for (int it = 0; it < iters * (bytes / 8192 + 1); ++it) {
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                   :: "l"(g + slot * 2048), "r"(su32(sm + 65536 + (it & 1) * 8192)), "r"(8192) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      slot += gridDim.x; if (slot >= nslots) slot -= nslots;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    const uint32_t rbar0 = mapa(su32(&bar[0]), pe), rbar1 = mapa(su32(&bar[1]), pe);
    const uint32_t dst0 = mapa(su32(sm + 32768), pe);
    const long long t0 = clock64();
    if (MODE == 0) {
      for (int it = 0; it < iters; ++it) {
        if (me == 0) {
          copy(dst0, sm, bytes, rbar0);
          expect(&bar[0], bytes);
          wait(&bar[0], it & 1);
        } else {
          expect(&bar[0], bytes);
          wait(&bar[0], it & 1);
          copy(dst0, sm, bytes, rbar0);
        }
      }
    } else {
      for (int it = 0; it < iters; ++it) {
        const int s = it & 1;
        expect(&bar[s], bytes);
        copy(dst0 + s * 16384, sm + s * 16384, bytes, s ? rbar1 : rbar0);
        if (it >= 1) wait(&bar[s ^ 1], ((it - 1) >> 1) & 1);
      }
      wait(&bar[(iters - 1) & 1], ((iters - 1) >> 1) & 1);
    }
    const long long c = clock64() - t0;
    if (blockIdx.x == 0) out[0] = c;
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE, bool GRED>
void run(float* g, size_t span, int bytes, int clusters, unsigned long long* d) {
  const int iters = 2000, smem = 98304 + 64;
  cudaFuncSetAttribute(k<MODE, GRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE, GRED><<<2 * clusters, 64, smem>>>(g, span, bytes, 20, d);
  k<MODE, GRED><<<2 * clusters, 64, smem>>>(g, span, bytes, iters, d);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  if (MODE == 0)
    printf("ping-pong  bytes=%5d clusters=%2d gred=%d: one-way %6.0f cycles per copy (%5.1f B/clk)\n", bytes, clusters,
           GRED, c / (2.0 * iters), bytes * 2.0 * iters / c);
  else
    printf("stream     bytes=%5d clusters=%2d gred=%d: %6.0f cycles per copy, %5.1f B/clk per CTA\n", bytes, clusters,
           GRED, double(c) / iters, double(bytes) * iters / c);
}

int main() {
  const size_t span = 8ull << 20;
  float* g; cudaMalloc(&g, span * 4); cudaMemset(g, 0, span * 4);
  unsigned long long* d; cudaMalloc(&d, 16);
  for (int b : {1024, 4096, 16384}) run<0, false>(g, span, b, 1, d);
  run<0, false>(g, span, 16384, 74, d);
  run<0, true>(g, span, 16384, 74, d);
  for (int b : {4096, 16384}) run<1, false>(g, span, b, 74, d);
  run<1, true>(g, span, 16384, 74, d);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
