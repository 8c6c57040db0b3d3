// Microbenchmark: throughput of the exponential variants a softmax row can use on
// sm_100a, one or two warps per SMSP: MUFU.EX2 f32, ex2.approx.f16x2 (two per lane-op),
// ex2.approx.ftz.bf16x2, and the FMA-pipe polynomial.  Cycles per 128 exps per warp.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "../../paper_2307_08691_b200/csrc/sm100_ptx.cuh"
using namespace fa2;

__device__ __forceinline__ uint32_t ex2_h2(uint32_t x) {
  uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y;
}
__device__ __forceinline__ uint32_t ex2_bf2(uint32_t x) {
  uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y;
}

template <int MODE>
__global__ void k(float* out, unsigned long long* cyc, int iters) {
  float s[128];
  for (int c = 0; c < 128; ++c) s[c] = -((threadIdx.x * 7 + c * 13) % 97) * 0.05f;
  float2 acc = make_float2(0.f, 0.f);
  uint32_t sink = 0;
  const float2 sc = make_float2(1.4427f, 1.4427f), nb = make_float2(-3.f, -3.f);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (MODE >= 22 && MODE <= 24) {   // 22: +F2FP, 23: +FADD2, 24: +FADD2 + integer RNE pack
      float2 accf = make_float2(0.f, 0.f);
      uint32_t acc_u = 0;
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 x = ptx::ffma2(make_float2(s[2 * e], s[2 * e + 1]), sc, nb);
        const float a = ptx::ex2(x.x), b = ptx::ex2(x.y);
        if constexpr (MODE == 22) acc_u ^= ptx::pack2<true>(a, b);
        if constexpr (MODE >= 23) accf = ptx::fadd2(accf, make_float2(a, b));
        if constexpr (MODE == 24) {
          const uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
          const uint32_t ra = ua + 0x7FFFu + ((ua >> 16) & 1u), rb = ub + 0x7FFFu + ((ub >> 16) & 1u);
          acc_u ^= __byte_perm(ra, rb, 0x7632);
        }
        if constexpr (MODE == 23) acc_u ^= __float_as_uint(a) ^ __float_as_uint(b);
      }
      sink ^= acc_u ^ __float_as_uint(accf.x + accf.y);
      s[it & 127] += accf.x * 1e-30f;
      continue;
    }
    if constexpr (MODE == 20 || MODE == 21) {   // pure MUFU.EX2 stream (20) / EX2 + FFMA2 per pair (21)
      uint32_t acc_u = 0;
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        float a = s[2 * e], b = s[2 * e + 1];
        if constexpr (MODE == 21) {
          const float2 x = ptx::ffma2(make_float2(a, b), sc, nb);
          a = x.x; b = x.y;
        }
        s[2 * e] = ptx::ex2(a);
        s[2 * e + 1] = ptx::ex2(b);
      }
#pragma unroll
      for (int e = 0; e < 128; ++e) acc_u ^= __float_as_uint(s[e]);
      sink ^= acc_u;
      s[it & 127] = -((it * 7) % 97) * 0.05f;
      continue;
    }
    if constexpr (MODE >= 4) {   // two passes: all exponentials first (in place), then sums and packs
      float p[128];
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        const float2 x = ptx::ffma2(make_float2(s[2 * e], s[2 * e + 1]), sc, nb);
        float2 r;
        if ((e % 16) < (MODE - 4)) r = ptx::exp2_poly2(x);
        else { r.x = ptx::ex2(x.x); r.y = ptx::ex2(x.y); }
        p[2 * e] = r.x; p[2 * e + 1] = r.y;
      }
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        acc = ptx::fadd2(acc, make_float2(p[2 * e], p[2 * e + 1]));
        sink ^= ptx::pack2<true>(p[2 * e], p[2 * e + 1]);
      }
      s[it & 127] += acc.x * 1e-30f;
      continue;
    }
#pragma unroll
    for (int e = 0; e < 64; ++e) {
      const float2 x = ptx::ffma2(make_float2(s[2 * e], s[2 * e + 1]), sc, nb);
      if constexpr (MODE == 0) {          // MUFU.EX2 f32
        float2 p; p.x = ptx::ex2(x.x); p.y = ptx::ex2(x.y);
        acc = ptx::fadd2(acc, p);
        sink ^= ptx::pack2<true>(p.x, p.y);
      } else if constexpr (MODE == 1) {   // f16x2 exp, sum in f32
        const uint32_t h = ptx::pack2<false>(x.x, x.y);
        const uint32_t ph = ex2_h2(h);
        const float2 p = __half22float2(*reinterpret_cast<const __half2*>(&ph));
        acc = ptx::fadd2(acc, p);
        sink ^= ph;
      } else if constexpr (MODE == 2) {   // bf16x2 exp, sum in f32
        const uint32_t h = ptx::pack2<true>(x.x, x.y);
        const uint32_t ph = ex2_bf2(h);
        const float2 p = make_float2(__uint_as_float(ph << 16), __uint_as_float(ph & 0xffff0000u));
        acc = ptx::fadd2(acc, p);
        sink ^= ph;
      } else {                            // FMA-pipe polynomial
        const float2 p = ptx::exp2_poly2(x);
        acc = ptx::fadd2(acc, p);
        sink ^= ptx::pack2<true>(p.x, p.y);
      }
    }
    s[it & 127] += acc.x * 1e-30f;
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + __uint_as_float(sink);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, float* out, unsigned long long* cyc) {
  const int iters = 100;
  for (int warps : {4, 8}) {
    k<MODE><<<148, warps * 32>>>(out, cyc, iters);
    k<MODE><<<148, warps * 32>>>(out, cyc, iters);
    unsigned long long h;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-10s warps/SMSP %d: %.1f cycles per 128-exp row per warp\n", name, warps / 4, double(h) / iters);
  }
}

int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  run<0>("ex2.f32", out, cyc);
  run<1>("ex2.f16x2", out, cyc);
  run<2>("ex2.bf16x2", out, cyc);
  run<3>("poly", out, cyc);
  run<20>("pure EX2", out, cyc);
  run<22>("EX2+FFMA2+F2FP", out, cyc);
  run<23>("EX2+FFMA2+FADD2", out, cyc);
  run<24>("EX2+FFMA2+FADD2+intRNE", out, cyc);
  run<21>("EX2 + FFMA2", out, cyc);
  run<4>("2pass emu0", out, cyc);
  run<8>("2pass emu4", out, cyc);
  run<10>("2pass emu6", out, cyc);
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
