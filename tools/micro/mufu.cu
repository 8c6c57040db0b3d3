// Microbenchmark: can one warp per SMSP saturate MUFU.EX2?  Times the softmax-like
// inner loop (FFMA2 -> EX2 -> FADD2 + F2FP) for 128 values per thread.
#include <cstdio>
#include <cstdint>
#include "../../paper_2307_08691_b200/csrc/sm100_ptx.cuh"
using namespace fa2;

template <int EMU>
__global__ void k(float* out, unsigned long long* cyc, int iters) {
  float s[128];
  for (int c = 0; c < 128; ++c) s[c] = (threadIdx.x * 7 + c * 13) % 97 * 0.01f;
  float2 acc = make_float2(0.f, 0.f);
  uint32_t sink = 0;
  const float2 sc = make_float2(1.4427f, 1.4427f), nb = make_float2(-3.f, -3.f);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      const float2 x = ptx::ffma2(make_float2(s[2 * e], s[2 * e + 1]), sc, nb);
      float2 p;
      if (e % 16 < EMU) p = ptx::exp2_poly2(x);
      else { p.x = ptx::ex2(x.x); p.y = ptx::ex2(x.y); }
      acc = ptx::fadd2(acc, p);
      sink ^= ptx::pack2<true>(p.x, p.y);
    }
    s[it & 127] += acc.x * 1e-30f;
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 100;
  for (int warps : {4, 8, 16}) {
    for (int emu : {0, 4, 8}) {
      auto kern = emu == 0 ? k<0> : emu == 4 ? k<4> : k<8>;
      kern<<<148, warps * 32>>>(out, cyc, iters);
      kern<<<148, warps * 32>>>(out, cyc, iters);
      unsigned long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      // per warp: 128 exps per iter
      printf("warps/SM %2d (per SMSP %d) emu %d: %.1f cycles per 128-exp row per warp; MUFU-bound would be %d\n",
             warps, warps / 4, emu, double(h) / iters, (128 - 128 * emu / 16) * 8 * (warps / 4));
    }
  }
  return 0;
}
