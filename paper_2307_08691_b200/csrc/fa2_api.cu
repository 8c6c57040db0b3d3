// C-ABI host side of the B200 FlashAttention-2 library (include/fa2.h).
// Argument validation, TMA descriptor encoding, workspace carving and launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <mutex>

#include "../../include/fa2.h"
#include "fa2_fwd_sm100.cuh"
#include "fa2_bwd_sm100.cuh"
#include "fa2_bwd128_sm100.cuh"

namespace {

thread_local std::string g_detail;
thread_local int g_launches = 0;
thread_local cudaEvent_t const* g_events = nullptr;   // benchmark timing hook (fa2_set_timing_events)
thread_local unsigned long long* g_trace = nullptr;     // debug timeline buffer (fa2_debug_set_trace)

inline void mark(int i, cudaStream_t st) {
  if (g_events != nullptr) cudaEventRecord(g_events[i], st);
}

fa2_status_t fail(fa2_status_t s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
fa2_status_t fail(fa2_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_detail = buf;
  return s;
}

#define FA2_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(FA2_ERR_CUDA, "%s failed: %s", #call, cudaGetErrorString(e_));          \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

fa2_status_t check_common(int B, int H, int N, int d, float scale, fa2_dtype_t dtype, bool need_scale) {
  if (B < 1 || H < 1 || N < 1) return fail(FA2_ERR_INVALID_ARG, "B, H, N must be >= 1 (got %d, %d, %d)", B, H, N);
  if (static_cast<long long>(B) * H > 0x7fffffffLL) return fail(FA2_ERR_INVALID_ARG, "B*H too large");
  if (d != 64 && d != 128) return fail(FA2_ERR_UNSUPPORTED, "head dim d=%d unsupported (64 or 128)", d);
  if (dtype != FA2_BF16 && dtype != FA2_FP16) return fail(FA2_ERR_UNSUPPORTED, "unknown dtype %d", (int)dtype);
  if (need_scale && !(std::isfinite(scale) && scale > 0.f))
    return fail(FA2_ERR_INVALID_ARG, "softmax_scale must be finite and > 0");
  return FA2_OK;
}

fa2_status_t check_ptrs(std::initializer_list<const void*> ps) {
  int i = 0;
  for (const void* p : ps) {
    if (p == nullptr) return fail(FA2_ERR_INVALID_ARG, "pointer argument #%d is NULL", i);
    if (!aligned16(p)) return fail(FA2_ERR_INVALID_ARG, "pointer argument #%d is not 16-byte aligned", i);
    ++i;
  }
  return FA2_OK;
}

struct DeviceInfo {
  int sms = 0;
  int major = 0;
};

fa2_status_t device_info(DeviceInfo& di) {
  int dev = 0;
  FA2_CUDA(cudaGetDevice(&dev));
  FA2_CUDA(cudaDeviceGetAttribute(&di.sms, cudaDevAttrMultiProcessorCount, dev));
  FA2_CUDA(cudaDeviceGetAttribute(&di.major, cudaDevAttrComputeCapabilityMajor, dev));
  if (di.major != 10) return fail(FA2_ERR_UNSUPPORTED, "device compute capability %d.x is not sm_100", di.major);
  return FA2_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// 3-D map over a [BH, rows, cols] tensor with box {box_cols, box_rows, 1}.
fa2_status_t make_map_3d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, int cols,
                         int rows, int bh, int box_cols, int box_rows, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FA2_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(bh)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * elem_bytes,
                           static_cast<cuuint64_t>(cols) * elem_bytes * static_cast<cuuint64_t>(rows)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FA2_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return FA2_OK;
}

CUtensorMapDataType tma_dtype(fa2_dtype_t dt) {
  return dt == FA2_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
}

template <typename K>
fa2_status_t set_smem(K kernel, int bytes) {
  FA2_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  return FA2_OK;
}

// ----------------------------------------------------------------------------
// Forward
// ----------------------------------------------------------------------------
template <int D, bool BF16, bool CAUSAL>
fa2_status_t launch_fwd(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const fa2::FwdParams& p,
                        int sms, cudaStream_t st) {
  auto kern = fa2::fa2_fwd_kernel<D, BF16, CAUSAL>;
  constexpr int smem = fa2::FwdSmem<D>::ALLOC;
  fa2_status_t s = set_smem(kern, smem);
  if (s != FA2_OK) return s;
  const int grid = p.num_tiles < sms ? p.num_tiles : sms;
  mark(0, st);
  kern<<<grid, 384, smem, st>>>(mq, mk, mv, p);
  mark(1, st);
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

template <int D, bool BF16>
fa2_status_t dispatch_fwd_causal(bool causal, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                                 const fa2::FwdParams& p, int sms, cudaStream_t st) {
  return causal ? launch_fwd<D, BF16, true>(mq, mk, mv, p, sms, st) : launch_fwd<D, BF16, false>(mq, mk, mv, p, sms, st);
}

fa2_status_t forward_impl(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H, int Hkv,
                          int N, int d, int causal, float scale, fa2_dtype_t dtype, cudaStream_t st, int sms) {
  const int BH = B * H;
  CUtensorMap mq, mk, mv;
  const CUtensorMapDataType dt = tma_dtype(dtype);
  fa2_status_t s;
  if ((s = make_map_3d(&mq, q, dt, 2, d, N, BH, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  if ((s = make_map_3d(&mk, k, dt, 2, d, N, B * Hkv, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  if ((s = make_map_3d(&mv, v, dt, 2, d, N, B * Hkv, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  fa2::FwdParams p;
  p.o = o;
  p.lse = lse;
  p.BH = BH;
  p.H = H;
  p.Hkv = Hkv;
  p.group = H / Hkv;
  p.N = N;
  p.num_m_blocks = (N + 255) / 256;
  p.num_tiles = BH * p.num_m_blocks;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = g_trace;
  const bool bf16 = dtype == FA2_BF16;
  if (d == 64)
    s = bf16 ? dispatch_fwd_causal<64, true>(causal, mq, mk, mv, p, sms, st)
             : dispatch_fwd_causal<64, false>(causal, mq, mk, mv, p, sms, st);
  else
    s = bf16 ? dispatch_fwd_causal<128, true>(causal, mq, mk, mv, p, sms, st)
             : dispatch_fwd_causal<128, false>(causal, mq, mk, mv, p, sms, st);
  return s;
}

// ----------------------------------------------------------------------------
// Backward
// ----------------------------------------------------------------------------
size_t pad128(int N) { return static_cast<size_t>((N + 127) / 128) * 128; }

size_t ws_dq_bytes(int B, int H, int N, int d) { return static_cast<size_t>(B) * H * pad128(N) * d * 4; }
// D and L*log2(e), each [B,H,N_pad] fp32
size_t ws_d_bytes(int B, int H, int N) { return 2 * static_cast<size_t>(B) * H * pad128(N) * 4; }
// deterministic-mode dQ tile counters, [B,H,N_pad/128] int32 (16-byte rounded)
size_t ws_sem_bytes(int B, int H, int N) { return (static_cast<size_t>(B) * H * (pad128(N) / 128) * 4 + 15) / 16 * 16; }

fa2_status_t preprocess_impl(const void* o, const void* dout, const float* lse, float* dvec, float* lse2,
                             float* dq_acc, int BH, int N, int npad, int d, fa2_dtype_t dtype, cudaStream_t st,
                             int* dq_sem = nullptr) {
  // one warp per row of the padded [BH, npad] grid; 8 rows per 256-thread block
  const long long rows = static_cast<long long>(BH) * npad;
  const int grid = static_cast<int>((rows + 7) / 8);
  const bool bf16 = dtype == FA2_BF16;
  if (d == 64) {
    if (bf16) fa2::fa2_bwd_preprocess<64, true><<<grid, 256, 0, st>>>(o, dout, dvec, dq_acc, BH, N, npad, lse, lse2, dq_sem);
    else fa2::fa2_bwd_preprocess<64, false><<<grid, 256, 0, st>>>(o, dout, dvec, dq_acc, BH, N, npad, lse, lse2, dq_sem);
  } else {
    if (bf16) fa2::fa2_bwd_preprocess<128, true><<<grid, 256, 0, st>>>(o, dout, dvec, dq_acc, BH, N, npad, lse, lse2, dq_sem);
    else fa2::fa2_bwd_preprocess<128, false><<<grid, 256, 0, st>>>(o, dout, dvec, dq_acc, BH, N, npad, lse, lse2, dq_sem);
  }
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

template <typename Kern>
fa2_status_t launch_bwd_kernel(Kern kern, int smem, const fa2::BwdMaps& maps, const fa2::BwdParams& p, int sms,
                               cudaStream_t st) {
  fa2_status_t s = set_smem(kern, smem);
  if (s != FA2_OK) return s;
  int grid = p.num_tiles < sms ? p.num_tiles : sms;
  // deterministic cyclic schedule: whole heads per wave (see bwd_q_tile in fa2_bwd_sm100.cuh)
  if (p.dq_sem != nullptr && p.det_cyclic) grid = (grid / p.num_n_blocks) * p.num_n_blocks;
  mark(3, st);
  kern<<<grid, fa2::kBwdThreads, smem, st>>>(maps.q, maps.k, maps.v, maps.dout, maps.dq_acc, p);
  mark(4, st);
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

template <int D, bool BF16, bool CAUSAL>
fa2_status_t launch_bwd(const fa2::BwdMaps& maps, const fa2::BwdParams& p, int sms, cudaStream_t st) {
  // d = 128: fa2_bwd128_sm100.cuh; d = 64: fa2_bwd_kernel
  if constexpr (D == 128)
    return launch_bwd_kernel(fa2::fa2_bwd128_kernel<BF16, CAUSAL>, fa2::Bwd128Smem::ALLOC, maps, p, sms, st);
  else
    return launch_bwd_kernel(fa2::fa2_bwd_kernel<D, BF16, CAUSAL>, fa2::BwdSmem<D>::ALLOC, maps, p, sms, st);
}

template <int D, bool BF16>
fa2_status_t dispatch_bwd_causal(bool causal, const fa2::BwdMaps& maps, const fa2::BwdParams& p, int sms,
                                 cudaStream_t st) {
  return causal ? launch_bwd<D, BF16, true>(maps, p, sms, st) : launch_bwd<D, BF16, false>(maps, p, sms, st);
}

fa2_status_t backward_impl(const void* q, const void* k, const void* v, const void* o, const float* lse,
                           const void* dout, void* dq, void* dk, void* dv, void* ws, int B, int H, int Hkv, int N,
                           int d, int causal, float scale, fa2_dtype_t dtype, cudaStream_t st, int sms,
                           bool deterministic = false) {
  const int BH = B * H;
  const size_t npad = pad128(N);
  float* dq_acc = reinterpret_cast<float*>(ws);
  float* dvec = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + ws_dq_bytes(B, H, N, d));
  float* lse2 = dvec + static_cast<size_t>(BH) * npad;
  int* dq_sem = deterministic ? reinterpret_cast<int*>(lse2 + static_cast<size_t>(BH) * npad) : nullptr;
  mark(2, st);
  fa2_status_t s = preprocess_impl(o, dout, lse, dvec, lse2, dq_acc, BH, N, static_cast<int>(npad), d, dtype, st, dq_sem);
  if (s != FA2_OK) return s;
  fa2::BwdMaps maps;
  const CUtensorMapDataType dt = tma_dtype(dtype);
  const int bm = 128;   // query rows per backward tile (both kernels)
  if ((s = make_map_3d(&maps.q, q, dt, 2, d, N, BH, 64, bm, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  if ((s = make_map_3d(&maps.dout, dout, dt, 2, d, N, BH, 64, bm, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  if ((s = make_map_3d(&maps.k, k, dt, 2, d, N, B * Hkv, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  if ((s = make_map_3d(&maps.v, v, dt, 2, d, N, B * Hkv, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK) return s;
  // fp32 dQ accumulator [BH, npad, d]; reduce-add boxes of 32 columns x BM rows (128-B swizzle rows;
  // the d=128 kernel uses contiguous 1D bulk reductions instead)
  if ((s = make_map_3d(&maps.dq_acc, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, static_cast<int>(npad), BH, 32,
                       bm, CU_TENSOR_MAP_SWIZZLE_128B)) != FA2_OK)
    return s;
  fa2::BwdParams p;
  p.lse = lse;
  p.dvec = dvec;
  p.dk = dk;
  p.dv = dv;
  p.dq_acc = dq_acc;
  p.BH = BH;
  p.H = H;
  p.Hkv = Hkv;
  p.group = H / Hkv;
  p.N = N;
  p.npad = static_cast<int>(npad);
  p.num_n_blocks = (N + 127) / 128;
  p.num_tiles = B * Hkv * p.num_n_blocks;   // one work tile per (key/value head, key block)
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = g_trace;
  p.dq_sem = dq_sem;
  p.det_cyclic = p.num_n_blocks <= sms ? 1 : 0;
  const bool bf16 = dtype == FA2_BF16;
  if (d == 64)
    s = bf16 ? dispatch_bwd_causal<64, true>(causal, maps, p, sms, st) : dispatch_bwd_causal<64, false>(causal, maps, p, sms, st);
  else
    s = bf16 ? dispatch_bwd_causal<128, true>(causal, maps, p, sms, st)
             : dispatch_bwd_causal<128, false>(causal, maps, p, sms, st);
  if (s != FA2_OK) return s;
  // dQ = cast(dq_acc) (the softmax scale is already applied to dS), rows < N only
  {
    const long long elems = static_cast<long long>(BH) * N * d;
    const int grid = static_cast<int>((elems / 8 + 255) / 256);
    if (bf16) fa2::fa2_dq_convert<true><<<grid, 256, 0, st>>>(dq_acc, dq, BH, N, static_cast<int>(npad), d);
    else fa2::fa2_dq_convert<false><<<grid, 256, 0, st>>>(dq_acc, dq, BH, N, static_cast<int>(npad), d);
    FA2_CUDA(cudaGetLastError());
    mark(5, st);
  }
  return FA2_OK;
}

fa2_status_t backward_entry(const void* q, const void* k, const void* v, const void* o, const float* lse,
                            const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                            int B, int H, int H_kv, int N, int d, int causal, float softmax_scale, fa2_dtype_t dtype,
                            void* stream, bool deterministic);

}  // namespace

extern "C" {

const char* fa2_status_string(fa2_status_t s) {
  switch (s) {
    case FA2_OK: return "FA2_OK";
    case FA2_ERR_INVALID_ARG: return "FA2_ERR_INVALID_ARG";
    case FA2_ERR_UNSUPPORTED: return "FA2_ERR_UNSUPPORTED";
    case FA2_ERR_WORKSPACE: return "FA2_ERR_WORKSPACE";
    case FA2_ERR_CUDA: return "FA2_ERR_CUDA";
  }
  return "FA2_UNKNOWN_STATUS";
}

const char* fa2_last_error_detail(void) { return g_detail.c_str(); }
void fa2_debug_set_trace(void* dev_buf) { g_trace = reinterpret_cast<unsigned long long*>(dev_buf); }
void fa2_set_timing_events(void* const* events) { g_events = reinterpret_cast<cudaEvent_t const*>(events); }
int fa2_last_launch_count(void) { return g_launches; }

fa2_status_t fa2_kv_block_range(int N, int Br, int Bc, int i, int causal, int* n_blocks, int* first_masked) {
  if (N < 1 || Br < 1 || Bc < 1 || i < 0 || n_blocks == nullptr || first_masked == nullptr)
    return fail(FA2_ERR_INVALID_ARG, "fa2_kv_block_range: bad arguments");
  const int tr = (N + Br - 1) / Br;
  if (i >= tr) return fail(FA2_ERR_INVALID_ARG, "row block %d out of range (T_r=%d)", i, tr);
  const int tc = (N + Bc - 1) / Bc;
  const int r0 = i * Br;
  const int r1 = (r0 + Br < N ? r0 + Br : N) - 1;   // last valid row
  int nb = causal ? (r1 / Bc + 1) : tc;
  if (nb > tc) nb = tc;
  // first block needing a mask: causal -> first block with a column > r0; ragged -> block containing column N
  // block j needs the causal mask iff its last column j*Bc+Bc-1 exceeds the first row r0,
  // i.e. j >= (r0+1)/Bc; the ragged tail needs a mask in the last block when Bc does not divide N.
  int fm = nb;
  if (causal && (r0 + 1) / Bc < fm) fm = (r0 + 1) / Bc;
  if (N % Bc != 0 && tc - 1 < fm) fm = tc - 1;
  *n_blocks = nb;
  *first_masked = fm;
  return FA2_OK;
}

fa2_status_t fa2_forward_gqa(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H, int H_kv,
                             int N, int d, int causal, float softmax_scale, fa2_dtype_t dtype, void* stream) {
  g_detail.clear();
  fa2_status_t s = check_common(B, H, N, d, softmax_scale, dtype, true);
  if (s != FA2_OK) return s;
  if (H_kv < 1 || H % H_kv != 0) return fail(FA2_ERR_INVALID_ARG, "H=%d must be a positive multiple of H_kv=%d", H, H_kv);
  if ((s = check_ptrs({q, k, v, o, lse})) != FA2_OK) return s;
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  s = forward_impl(q, k, v, o, lse, B, H, H_kv, N, d, causal, softmax_scale, dtype, static_cast<cudaStream_t>(stream),
                   di.sms);
  if (s == FA2_OK) g_launches = 1;
  return s;
}

fa2_status_t fa2_forward(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H, int N, int d,
                         int causal, float softmax_scale, fa2_dtype_t dtype, void* stream) {
  return fa2_forward_gqa(q, k, v, o, lse, B, H, H, N, d, causal, softmax_scale, dtype, stream);
}

size_t fa2_backward_workspace_size(int B, int H, int N, int d) {
  if (B < 1 || H < 1 || N < 1 || (d != 64 && d != 128)) return 0;
  return ws_dq_bytes(B, H, N, d) + ws_d_bytes(B, H, N) + ws_sem_bytes(B, H, N);
}

fa2_status_t fa2_backward(const void* q, const void* k, const void* v, const void* o, const float* lse,
                          const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                          int B, int H, int N, int d, int causal, float softmax_scale, fa2_dtype_t dtype,
                          void* stream) {
  return fa2_backward_gqa(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes, B, H, H, N, d, causal,
                          softmax_scale, dtype, stream);
}

fa2_status_t fa2_backward_gqa(const void* q, const void* k, const void* v, const void* o, const float* lse,
                              const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                              int B, int H, int H_kv, int N, int d, int causal, float softmax_scale, fa2_dtype_t dtype,
                              void* stream) {
  return backward_entry(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes, B, H, H_kv, N, d, causal,
                        softmax_scale, dtype, stream, false);
}

fa2_status_t fa2_backward_deterministic(const void* q, const void* k, const void* v, const void* o, const float* lse,
                                        const void* dout, void* dq, void* dk, void* dv, void* workspace,
                                        size_t workspace_bytes, int B, int H, int H_kv, int N, int d, int causal,
                                        float softmax_scale, fa2_dtype_t dtype, void* stream) {
  return backward_entry(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes, B, H, H_kv, N, d, causal,
                        softmax_scale, dtype, stream, true);
}

}  // extern "C"

namespace {
fa2_status_t backward_entry(const void* q, const void* k, const void* v, const void* o, const float* lse,
                            const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                            int B, int H, int H_kv, int N, int d, int causal, float softmax_scale, fa2_dtype_t dtype,
                            void* stream, bool deterministic) {
  g_detail.clear();
  fa2_status_t s = check_common(B, H, N, d, softmax_scale, dtype, true);
  if (s != FA2_OK) return s;
  if (H_kv < 1 || H % H_kv != 0) return fail(FA2_ERR_INVALID_ARG, "H=%d must be a positive multiple of H_kv=%d", H, H_kv);
  if ((s = check_ptrs({q, k, v, o, lse, dout, dq, dk, dv})) != FA2_OK) return s;
  if (workspace == nullptr || !aligned16(workspace))
    return fail(FA2_ERR_WORKSPACE, "workspace is NULL or not 16-byte aligned");
  if (workspace_bytes < fa2_backward_workspace_size(B, H, N, d))
    return fail(FA2_ERR_WORKSPACE, "workspace too small: %zu < %zu", workspace_bytes,
                fa2_backward_workspace_size(B, H, N, d));
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  s = backward_impl(q, k, v, o, lse, dout, dq, dk, dv, workspace, B, H, H_kv, N, d, causal, softmax_scale, dtype,
                    static_cast<cudaStream_t>(stream), di.sms, deterministic);
  if (s == FA2_OK) g_launches = 3;
  return s;
}
}  // namespace

extern "C" {

fa2_status_t fa2_backward_preprocess(const void* o, const void* dout, float* d_out, int B, int H, int N, int d,
                                     fa2_dtype_t dtype, void* stream) {
  g_detail.clear();
  fa2_status_t s = check_common(B, H, N, d, 1.f, dtype, false);
  if (s != FA2_OK) return s;
  if ((s = check_ptrs({o, dout, d_out})) != FA2_OK) return s;
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  // d_out has N entries per head (no padding); write D via a padded-stride-free variant: npad == N here.
  const int BH = B * H;
  const long long rows = static_cast<long long>(BH) * N;
  const int grid = static_cast<int>((rows + 7) / 8);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool bf16 = dtype == FA2_BF16;
  if (d == 64) {
    if (bf16) fa2::fa2_bwd_preprocess<64, true><<<grid, 256, 0, st>>>(o, dout, d_out, nullptr, BH, N, N);
    else fa2::fa2_bwd_preprocess<64, false><<<grid, 256, 0, st>>>(o, dout, d_out, nullptr, BH, N, N);
  } else {
    if (bf16) fa2::fa2_bwd_preprocess<128, true><<<grid, 256, 0, st>>>(o, dout, d_out, nullptr, BH, N, N);
    else fa2::fa2_bwd_preprocess<128, false><<<grid, 256, 0, st>>>(o, dout, d_out, nullptr, BH, N, N);
  }
  FA2_CUDA(cudaGetLastError());
  g_launches = 1;
  return FA2_OK;
}

size_t fa2_step_arena_size(int B, int H, int N, int d) {
  if (B < 1 || H < 1 || N < 1 || (d != 64 && d != 128)) return 0;
  const size_t t = static_cast<size_t>(B) * H * N * d * 2;
  const size_t t16 = (t + 255) & ~size_t(255);
  const size_t l = (static_cast<size_t>(B) * H * N * 4 + 255) & ~size_t(255);
  return 9 * t16 + l + fa2_backward_workspace_size(B, H, N, d);
}

fa2_status_t fa2_attention_step_host(const void* q_h, const void* k_h, const void* v_h, const void* dout_h, void* o_h,
                                     float* lse_h, void* dq_h, void* dk_h, void* dv_h, void* arena,
                                     size_t arena_bytes, int B, int H, int N, int d, int causal, float softmax_scale,
                                     fa2_dtype_t dtype, void* stream) {
  g_detail.clear();
  fa2_status_t s = check_common(B, H, N, d, softmax_scale, dtype, true);
  if (s != FA2_OK) return s;
  if (q_h == nullptr || k_h == nullptr || v_h == nullptr || dout_h == nullptr)
    return fail(FA2_ERR_INVALID_ARG, "host input pointer is NULL");
  if (arena == nullptr || !aligned16(arena)) return fail(FA2_ERR_WORKSPACE, "arena is NULL or not 16-byte aligned");
  if (arena_bytes < fa2_step_arena_size(B, H, N, d))
    return fail(FA2_ERR_WORKSPACE, "arena too small: %zu < %zu", arena_bytes, fa2_step_arena_size(B, H, N, d));
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t t = static_cast<size_t>(B) * H * N * d * 2;
  const size_t t16 = (t + 255) & ~size_t(255);
  const size_t lbytes = static_cast<size_t>(B) * H * N * 4;
  uint8_t* a = reinterpret_cast<uint8_t*>(arena);
  void *q = a, *k = a + t16, *v = a + 2 * t16, *dout = a + 3 * t16, *o = a + 4 * t16, *dq = a + 5 * t16,
       *dk = a + 6 * t16, *dv = a + 7 * t16;
  float* lse = reinterpret_cast<float*>(a + 9 * t16);
  void* ws = a + 9 * t16 + ((lbytes + 255) & ~size_t(255));
  FA2_CUDA(cudaMemcpyAsync(q, q_h, t, cudaMemcpyHostToDevice, st));
  FA2_CUDA(cudaMemcpyAsync(k, k_h, t, cudaMemcpyHostToDevice, st));
  FA2_CUDA(cudaMemcpyAsync(v, v_h, t, cudaMemcpyHostToDevice, st));
  FA2_CUDA(cudaMemcpyAsync(dout, dout_h, t, cudaMemcpyHostToDevice, st));
  if ((s = forward_impl(q, k, v, o, lse, B, H, H, N, d, causal, softmax_scale, dtype, st, di.sms)) != FA2_OK) return s;
  if ((s = backward_impl(q, k, v, o, lse, dout, dq, dk, dv, ws, B, H, H, N, d, causal, softmax_scale, dtype, st,
                         di.sms)) != FA2_OK)
    return s;
  if (o_h) FA2_CUDA(cudaMemcpyAsync(o_h, o, t, cudaMemcpyDeviceToHost, st));
  if (lse_h) FA2_CUDA(cudaMemcpyAsync(lse_h, lse, lbytes, cudaMemcpyDeviceToHost, st));
  if (dq_h) FA2_CUDA(cudaMemcpyAsync(dq_h, dq, t, cudaMemcpyDeviceToHost, st));
  if (dk_h) FA2_CUDA(cudaMemcpyAsync(dk_h, dk, t, cudaMemcpyDeviceToHost, st));
  if (dv_h) FA2_CUDA(cudaMemcpyAsync(dv_h, dv, t, cudaMemcpyDeviceToHost, st));
  FA2_CUDA(cudaStreamSynchronize(st));
  g_launches = 4;
  return FA2_OK;
}

}  // extern "C"
