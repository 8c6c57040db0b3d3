// Throughput of LSU fp32 reductions (red.global.add scalar / v2 / v4, coalesced) and of
// LSU reductions running concurrently with TMA bulk reduce-add from another warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// VEC floats per lane; NW warps do LSU reds; if TMA, one extra warp does bulk reduces of 8 KB.
template <int VEC, bool TMA>
__global__ void k(float* g, size_t span, int iters, unsigned long long* bytes_out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  for (int i = threadIdx.x; i < 16384 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1e-6f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nw_lsu = blockDim.x / 32 - (TMA ? 1 : 0);
  if (TMA && warp == nw_lsu) {
    if (lane == 0) {
      size_t slot = blockIdx.x;
      const size_t nslots = span / 2048;
      for (int it = 0; it < iters / 4; ++it) {
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                     :: "l"(g + slot * 2048), "r"(su32(sm + (it & 1) * 8192)), "r"(8192) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        slot += gridDim.x; if (slot >= nslots) slot -= nslots;
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      atomicAdd(bytes_out, (unsigned long long)(iters / 4) * 8192);
    }
    return;
  }
  // each warp instruction covers 32*VEC*4 contiguous bytes
  const size_t per = 32 * VEC;
  const size_t nslots = span / per;
  size_t slot = (size_t)(blockIdx.x * nw_lsu + warp) * 7919 % nslots;
  const float a = 1e-7f;
  for (int it = 0; it < iters; ++it) {
    float* dst = g + slot * per + lane * VEC;
    if (VEC == 1) asm volatile("red.global.add.f32 [%0], %1;" :: "l"(dst), "f"(a) : "memory");
    if (VEC == 2) asm volatile("red.global.add.v2.f32 [%0], {%1, %1};" :: "l"(dst), "f"(a) : "memory");
    if (VEC == 4) asm volatile("red.global.add.v4.f32 [%0], {%1, %1, %1, %1};" :: "l"(dst), "f"(a) : "memory");
    slot += gridDim.x * nw_lsu; if (slot >= nslots) slot -= nslots;
  }
  if (lane == 0) atomicAdd(bytes_out, (unsigned long long)iters * per * 4);
}

template <int VEC, bool TMA>
void run(float* g, size_t span, int blocks, int warps, unsigned long long* d_bytes) {
  const int iters = 2000;
  cudaFuncSetAttribute(k<VEC, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  k<VEC, TMA><<<blocks, warps * 32, 16384>>>(g, span, 50, d_bytes);
  cudaMemset(d_bytes, 0, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<VEC, TMA><<<blocks, warps * 32, 16384>>>(g, span, iters, d_bytes);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long tot; cudaMemcpy(&tot, d_bytes, 8, cudaMemcpyDeviceToHost);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("vec=%d tma=%d blocks=%3d warps=%2d  %7.1f GB/s  %5.1f B/clk/SM\n", VEC, TMA, blocks, warps,
         tot / ms / 1e6, tot / (ms * 1e-3) / blocks / (clk * 1e3));
}

int main() {
  const size_t span = 8ull << 20;   // 32 MB, L2-resident
  float* g; cudaMalloc(&g, span * 4); cudaMemset(g, 0, span * 4);
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int w : {1, 4, 8}) { run<1, false>(g, span, 148, w, d); run<2, false>(g, span, 148, w, d); run<4, false>(g, span, 148, w, d); }
  run<4, false>(g, span, 1, 4, d);
  run<4, true>(g, span, 148, 5, d);
  run<4, true>(g, span, 148, 9, d);
  run<1, true>(g, span, 148, 5, d);
  run<4, true>(g, span, 148, 1, d);   // TMA warp only (nw_lsu = 0 -> no LSU work)
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
