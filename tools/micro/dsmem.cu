// DSMEM (distributed shared memory) write bandwidth inside a 2-CTA cluster:
// LSU st.shared::cluster (scalar / v4) and bulk smem->peer-smem copies, alone and
// next to a stream of bulk fp32 reduce-adds to global memory.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t peer(uint32_t a) {
  uint32_t r, rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank ^ 1));
  return r;
}

// MODE 0: scalar LSU remote stores; 1: v4 LSU remote stores; 2: bulk copy 8 KB to peer (1 thread)
template <int MODE, bool GRED>
__global__ void __cluster_dims__(2, 1, 1) k(float* g, size_t span, int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1e-6f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  const int nw = blockDim.x / 32 - (GRED ? 1 : 0);
  unsigned long long bytes = 0;
  if (GRED && warp == nw) {
    if (lane == 0) {
      size_t slot = blockIdx.x;
      const size_t nslots = span / 2048;
      for (int it = 0; it < iters / 8; ++it) {
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                     :: "l"(g + slot * 2048), "r"(su32(sm + 32768 + (it & 1) * 8192)), "r"(8192) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        slot += gridDim.x; if (slot >= nslots) slot -= nslots;
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      atomicAdd(out + 1, (unsigned long long)(iters / 8) * 8192);
    }
  } else if (MODE == 0 || MODE == 1) {
    const uint32_t base = peer(su32(sm));
    for (int it = 0; it < iters; ++it) {
      if (MODE == 0) {
        const uint32_t a = base + ((it * nw + warp) % 256) * 128 + lane * 4;   // 32 KB window
        asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(a), "f"(1.f) : "memory");
        bytes += 128;
      } else {
        const uint32_t a = base + ((it * nw + warp) % 64) * 512 + lane * 16;
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %1, %1, %1};" :: "r"(a), "f"(1.f) : "memory");
        bytes += 512;
      }
    }
    if (lane == 0) atomicAdd(out, bytes);
  } else if (MODE == 2 && threadIdx.x == 0) {
    const uint32_t rb = peer(su32(bar));
    const uint32_t dst = peer(su32(sm + 16384));
    for (int it = 0; it < iters / 8; ++it) {
      // self-completing: count bytes on the PEER's barrier; nobody waits, we just drain at the end
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(dst), "r"(su32(sm)), "r"(8192), "r"(rb) : "memory");
      bytes += 8192;
    }
    atomicAdd(out, bytes);
  }
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE, bool GRED>
void run(float* g, size_t span, int warps, unsigned long long* d, int iters) {
  cudaFuncSetAttribute(k<MODE, GRED>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
  k<MODE, GRED><<<148, warps * 32, 65536 + 64>>>(g, span, 64, d);
  cudaMemset(d, 0, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, GRED><<<148, warps * 32, 65536 + 64>>>(g, span, iters, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long t[2]; cudaMemcpy(t, d, 16, cudaMemcpyDeviceToHost);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("mode=%d gred=%d warps=%d  dsmem %5.1f B/clk/SM   global-red %5.1f B/clk/SM  (%s)\n", MODE, GRED, warps,
         t[0] / cyc / 148, t[1] / cyc / 148, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const size_t span = 8ull << 20;
  float* g; cudaMalloc(&g, span * 4); cudaMemset(g, 0, span * 4);
  unsigned long long* d; cudaMalloc(&d, 16);
  run<0, false>(g, span, 4, d, 20000);
  run<1, false>(g, span, 4, d, 20000);
  run<0, false>(g, span, 8, d, 20000);
  run<1, false>(g, span, 8, d, 20000);

  run<0, true>(g, span, 5, d, 20000);
  run<1, true>(g, span, 5, d, 20000);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
