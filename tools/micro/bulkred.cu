// Throughput of bulk smem->global fp32 reduce-add (and plain bulk store) vs CTA count,
// op size and in-flight depth.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 bulkred.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

template <int MODE, int DEPTH>   // MODE 0 reduce-add f32, 1 store, 2 reduce-add bf16
__global__ void k(float* g, size_t span_floats, int bytes, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1e-6f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t per = bytes / 4;
  const size_t nslots = span_floats / per;
  size_t slot = (size_t)blockIdx.x * 37 % nslots;
  for (int it = 0; it < iters; ++it) {
    float* dst = g + slot * per;
    const uint32_t src = su32(sm + (it % 4) * bytes % 65536);
    if (MODE == 0)
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" :: "l"(dst), "r"(src), "r"(bytes) : "memory");
    else if (MODE == 1)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst), "r"(src), "r"(bytes) : "memory");
    else
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.noftz.bf16 [%0], [%1], %2;" :: "l"(dst), "r"(src), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(DEPTH - 1) : "memory");
    slot += gridDim.x;
    if (slot >= nslots) slot -= nslots;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int MODE, int DEPTH>
void run(float* g, size_t span, int blocks, int bytes) {
  const int iters = 2000;
  cudaFuncSetAttribute(k<MODE, DEPTH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<MODE, DEPTH><<<blocks, 128, 65536>>>(g, span, bytes, 50);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, DEPTH><<<blocks, 128, 65536>>>(g, span, bytes, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double tot = double(blocks) * iters * bytes;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("mode=%d depth=%d blocks=%3d bytes=%5d  %7.1f GB/s  %5.1f B/clk/SM (at %d MHz)\n", MODE, DEPTH, blocks, bytes,
         tot / ms / 1e6, tot / (ms * 1e-3) / blocks / (clk * 1e3), clk / 1000);
}

int main() {
  const size_t span = 32ull << 20;   // 128 MB of floats? no: 32M floats = 128 MB; use 8M floats (32 MB, L2-resident)
  float* g; cudaMalloc(&g, span * 4); cudaMemset(g, 0, span * 4);
  const size_t l2span = 8ull << 20;
  for (int blocks : {1, 16, 74, 148}) {
    run<0, 2>(g, l2span, blocks, 8192);
    run<0, 4>(g, l2span, blocks, 8192);
  }
  for (int bytes : {2048, 4096, 16384, 32768}) run<0, 2>(g, l2span, 148, bytes);
  run<0, 8>(g, l2span, 148, 4096);
  run<1, 2>(g, l2span, 148, 8192);
  run<1, 4>(g, l2span, 148, 8192);
  run<1, 2>(g, l2span, 1, 8192);
  run<2, 2>(g, l2span, 148, 8192);
  run<0, 2>(g, span, 148, 8192);   // 128 MB span: beyond L2
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
}
