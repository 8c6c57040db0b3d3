// C-ABI host side of the B200 FlashAttention-2 library (include/fa2.h).
// Argument validation, TMA descriptor encoding, workspace carving and launches.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <mutex>
#include <algorithm>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "../../include/fa2.h"
#include "fa2_fwd_sm100.cuh"
#include "fa2_bwd_sm100.cuh"
#include "fa2_bwd128_sm100.cuh"
#include "fa2_fwd2_sm100.cuh"
#include "fa2_bwd2_sm100.cuh"

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

// Geometry of one call: fixed lengths ([B,H,N_q,d] / [B,H_kv,N_k,d]) or packed
// variable-length ([T_q,H,d] / [T_k,H_kv,d] with device cu_seqlens).
struct Geom {
  int B = 0, H = 0, Hkv = 0, d = 0;
  int Nq = 0, Nk = 0;                          // fixed lengths, or the packed maxima
  bool packed = false;
  const int* cu_q = nullptr;
  const int* cu_k = nullptr;
  int Tq = 0, Tk = 0;                          // packed totals
};

Geom fixed_geom(int B, int H, int Hkv, int Nq, int Nk, int d) {
  Geom g;
  g.B = B; g.H = H; g.Hkv = Hkv; g.d = d; g.Nq = Nq; g.Nk = Nk;
  return g;
}

// 3-D row-tile map in memory order (fa2_seq.cuh): fixed {d, N, B*heads}, packed
// {d, heads, T}; box = 64 columns x 128 rows of one head.
fa2_status_t make_rows_map(CUtensorMap* m, const void* base, CUtensorMapDataType dt, const Geom& g, int heads,
                           bool is_q, int elem_bytes = 2, int box_rows = 128) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FA2_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const cuuint64_t d = static_cast<cuuint64_t>(g.d), eb = static_cast<cuuint64_t>(elem_bytes);
  const cuuint32_t box_cols = static_cast<cuuint32_t>(128 / elem_bytes);   // one 128-B swizzle row
  cuuint64_t dims[3], strides[2];
  cuuint32_t box[3];
  if (!g.packed) {
    const cuuint64_t n = static_cast<cuuint64_t>(is_q ? g.Nq : g.Nk);
    dims[0] = d; dims[1] = n; dims[2] = static_cast<cuuint64_t>(heads) * static_cast<cuuint64_t>(g.B);
    strides[0] = d * eb; strides[1] = n * d * eb;
    box[0] = box_cols; box[1] = static_cast<cuuint32_t>(box_rows); box[2] = 1;
  } else {
    const cuuint64_t t = static_cast<cuuint64_t>(std::max(1, is_q ? g.Tq : g.Tk));
    dims[0] = d; dims[1] = static_cast<cuuint64_t>(heads); dims[2] = t;
    strides[0] = d * eb; strides[1] = static_cast<cuuint64_t>(heads) * d * eb;
    box[0] = box_cols; box[1] = 1; box[2] = static_cast<cuuint32_t>(box_rows);
  }
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, dt, 3, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FA2_ERR_CUDA, "cuTensorMapEncodeTiled (rows) failed (%d)", static_cast<int>(r));
  return FA2_OK;
}

// Validation shared by the packed variable-length entry points.
fa2_status_t varlen_geom(const int* cu_q, const int* cu_k, int B, int H, int Hkv, int total_q, int total_k, int max_q,
                         int max_k, int d, float scale, fa2_dtype_t dtype, Geom& g) {
  fa2_status_t s = check_common(B, H, 1, d, scale, dtype, true);
  if (s != FA2_OK) return s;
  if (Hkv < 1 || H % Hkv != 0) return fail(FA2_ERR_INVALID_ARG, "H=%d must be a positive multiple of H_kv=%d", H, Hkv);
  if (total_q < 1 || total_k < 1) return fail(FA2_ERR_INVALID_ARG, "total_q, total_k must be >= 1 (got %d, %d)", total_q, total_k);
  if (max_q < 1 || max_k < 1 || max_q > total_q || max_k > total_k)
    return fail(FA2_ERR_INVALID_ARG, "max_seqlen_q/k must be in [1, total] (got %d, %d)", max_q, max_k);
  if (cu_q == nullptr || cu_k == nullptr || (reinterpret_cast<uintptr_t>(cu_q) & 3u) || (reinterpret_cast<uintptr_t>(cu_k) & 3u))
    return fail(FA2_ERR_INVALID_ARG, "cu_seqlens_q / cu_seqlens_k must be non-NULL, 4-byte aligned int32 arrays");
  g.B = B; g.H = H; g.Hkv = Hkv; g.d = d;
  g.Nq = max_q; g.Nk = max_k;
  g.packed = true; g.cu_q = cu_q; g.cu_k = cu_k; g.Tq = total_q; g.Tk = total_k;
  return FA2_OK;
}

fa2::SeqGeom seq_geom(const Geom& g) {
  fa2::SeqGeom s;
  s.cu_q = g.packed ? g.cu_q : nullptr;
  s.cu_k = g.packed ? g.cu_k : nullptr;
  s.Nq = g.Nq;
  s.Nk = g.Nk;
  return s;
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
#ifndef FA2_SCHED
#define FA2_SCHED 1   // 0: static stride schedule everywhere (A/B builds)
#endif
// Balanced schedules (fa2::TileSched): tiles in windows of heads (window = `win` tiles
// of consecutive heads, ~64k rows of K/V or Q/dO, which stays in L2), heaviest first
// inside a window, each assigned to the least-loaded CTA.  Memoised per shape.
void build_sched(fa2::TileSched& sc, const std::vector<int>& work, int tiles_per_head, int heads_per_win, int grid) {
  const int T = static_cast<int>(work.size());
  std::vector<int> ord(T);
  for (int t = 0; t < T; ++t) ord[t] = t;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
    const int wa = (a / tiles_per_head) / heads_per_win, wb = (b / tiles_per_head) / heads_per_win;
    return wa != wb ? wa < wb : work[a] > work[b];
  });
  std::vector<std::vector<uint16_t>> lists(grid);
  std::vector<std::pair<long long, int>> heap;   // (load, cta), min-heap
  for (int c = 0; c < grid; ++c) heap.emplace_back(0LL, c);
  auto cmp = [](const std::pair<long long, int>& x, const std::pair<long long, int>& y) { return x > y; };
  std::make_heap(heap.begin(), heap.end(), cmp);
  for (int t : ord) {
    std::pop_heap(heap.begin(), heap.end(), cmp);
    heap.back().first += work[t];
    lists[heap.back().second].push_back(static_cast<uint16_t>(t));
    std::push_heap(heap.begin(), heap.end(), cmp);
  }
  int pos = 0;
  for (int c = 0; c < grid; ++c) {
    sc.start[c] = static_cast<uint16_t>(pos);
    for (uint16_t t : lists[c]) sc.order[pos++] = t;
  }
  sc.start[grid] = static_cast<uint16_t>(pos);
  sc.n = T;
}

// key: (device, kind, tiles, tiles per head, rows, heads per tile, grid); make_work(work) fills the
// tile works.  Entries are shared_ptr so a caller's schedule outlives a concurrent eviction.
using SchedPtr = std::shared_ptr<const fa2::TileSched>;
template <typename F>
SchedPtr cached_sched(int kind, int T, int tiles_per_head, int N, int nh, int grid, F make_work) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int, int>, SchedPtr> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(dev, kind, T, tiles_per_head, N, nh, grid);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  auto sc = std::make_shared<fa2::TileSched>();
  std::vector<int> work(T);
  make_work(work);
  build_sched(*sc, work, tiles_per_head, std::max(1, 65536 / std::max(1, N)), grid);
  std::lock_guard<std::mutex> lock(mu);
  if (cache.size() > 256) cache.clear();   // live schedules stay alive through their shared_ptr
  return cache.emplace(key, std::move(sc)).first->second;
}

// Co-resident clusters of 2 for a kernel (the persistent pair kernels' grid cap), per device.
template <typename K>
int max_active_pairs(K kern, int smem, int threads, int sms) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(dev, reinterpret_cast<const void*>(kern));
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2; attr.val.clusterDim.y = 1; attr.val.clusterDim.z = 1;
  cfg.gridDim = dim3(static_cast<unsigned>(sms & ~1));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  int n = 0;
  const int v = cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0 ? n : sms / 2;
  cache.emplace(key, v);
  return v;
}

// Forward (causal, square): tile t = (head, row block mb = nmb - 1 - t % nmb), work = key
// blocks of its two 128-row sub-tiles + 1 (prologue / epilogue).
SchedPtr fwd_sched(const fa2::FwdParams& p, int grid) {
  const int nmb = p.num_m_blocks, N = p.geom.Nq;
  return cached_sched(0, p.num_tiles, nmb, N, 1, grid, [&](std::vector<int>& work) {
    const int nkb = (N + 127) / 128;
    for (int t = 0; t < p.num_tiles; ++t) {
      const int mb = nmb - 1 - t % nmb;
      int w = 1;
      for (int i = 0; i < 2; ++i) {
        const int r0 = mb * 256 + i * 128;
        if (r0 < N) w += std::min(nkb, std::min(N - 1, r0 + 127) / 128 + 1);
      }
      work[t] = w;
    }
  });
}

// Backward (causal, square, arrival-order dQ): tile t = (head split, key block nb = t % nnb),
// work = query tiles i >= nb times the query heads of the tile, + 1.
SchedPtr bwd_sched(const fa2::BwdParams& p, int grid) {
  const int nnb = p.num_n_blocks, N = p.geom.Nq, nh = p.group / p.hsplit;
  return cached_sched(1, p.num_tiles, nnb, N, nh, grid, [&](std::vector<int>& work) {
    const int nqb = (N + 127) / 128;
    for (int t = 0; t < p.num_tiles; ++t) work[t] = (nqb - t % nnb) * nh + 1;
  });
}

template <int D, bool BF16, bool CAUSAL, bool GEN, bool FP8 = false>
fa2_status_t launch_fwd(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv, const CUtensorMap& mo,
                        const fa2::FwdParams& p, int sms, cudaStream_t st) {
  auto kern = fa2::fa2_fwd_kernel<D, BF16, CAUSAL, GEN, FP8>;
  constexpr int smem = fa2::FwdSmem<D, FP8 ? 1 : 2>::ALLOC;
  fa2_status_t s = set_smem(kern, smem);
  if (s != FA2_OK) return s;
  const int grid = p.num_tiles < sms ? p.num_tiles : sms;
  fa2::FwdSchedT<CAUSAL, GEN> sched;
  sched.n = 0;
  if constexpr (CAUSAL && !GEN) {
    if (FA2_SCHED && p.num_tiles <= fa2::kSchedMaxTiles && grid <= fa2::kSchedMaxCtas) {
      const SchedPtr sc = fwd_sched(p, grid);
      mark(0, st);
      kern<<<grid, fa2::FwdCfg<D, FP8>::THREADS, smem, st>>>(mq, mk, mv, mo, p, *sc);
      mark(1, st);
      FA2_CUDA(cudaGetLastError());
      return FA2_OK;
    }
  }
  mark(0, st);
  kern<<<grid, fa2::FwdCfg<D, FP8>::THREADS, smem, st>>>(mq, mk, mv, mo, p, sched);
  mark(1, st);
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

template <int D, bool BF16>
fa2_status_t dispatch_fwd_causal(bool causal, const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
                                 const CUtensorMap& mo,
                                 const fa2::FwdParams& p, int sms, cudaStream_t st) {
  // general geometry (packed varlen or N_q != N_k) vs the square fixed-length path
  if (p.geom.cu_q != nullptr || p.geom.Nq != p.geom.Nk)
    return causal ? launch_fwd<D, BF16, true, true>(mq, mk, mv, mo, p, sms, st)
                  : launch_fwd<D, BF16, false, true>(mq, mk, mv, mo, p, sms, st);
  return causal ? launch_fwd<D, BF16, true, false>(mq, mk, mv, mo, p, sms, st)
                : launch_fwd<D, BF16, false, false>(mq, mk, mv, mo, p, sms, st);
}

#ifndef FA2_FWD_PAIR
#define FA2_FWD_PAIR 1   // 0: the one-SM forward kernel for every shape (A/B builds)
#endif
#ifndef FA2_FWD_PAIR_CAUSAL
#define FA2_FWD_PAIR_CAUSAL 1   // 0: causal square d = 128 on the one-SM kernel (A/B builds)
#endif
// Pair forward (causal, fixed layout, N_q <= N_k): tile t = (head, 512-row block mb = nmb - 1 -
// t % nmb), work = key blocks of its two sub-tiles (sub-tile i: the blocks up to its last row +
// N_k - N_q, at most T_c) + 2 (prologue / epilogue); one list per CTA pair.
SchedPtr fwd_pair_sched(const fa2::FwdParams& p, int npairs) {
  const int nmb = p.num_m_blocks, N = p.geom.Nq, Nk = p.geom.Nk;
  // (N_k rides in the cache key's heads-per-tile slot, which the forward schedules leave at 1)
  return cached_sched(3, p.num_tiles, nmb, N, Nk, npairs, [&](std::vector<int>& work) {
    const int nkb = (Nk + 127) / 128, off = Nk - N;
    for (int t = 0; t < p.num_tiles; ++t) {
      const int mb = nmb - 1 - t % nmb;
      work[t] = 2;
      for (int i = 0; i < 2; ++i) {
        const int last = std::min(N - 1, mb * 512 + i * 256 + 255) + off;
        work[t] += last < 0 ? 0 : std::min(nkb, last / 128 + 1);
      }
    }
  });
}

// CTA-pair forward (fa2_fwd2_sm100.cuh): square fixed-length, d = 128, bf16/fp16
template <bool BF16, bool CAUSAL, bool GEN>
fa2_status_t launch_fwd_pair(const CUtensorMap& mq, const CUtensorMap& mk64, const CUtensorMap& mv,
                             const CUtensorMap& mo, fa2::FwdParams p, int sms, cudaStream_t st) {
  auto kern = fa2::fa2_fwd_pair_kernel<BF16, CAUSAL, GEN>;
  constexpr int smem = fa2::FwdPairSmem::ALLOC;
  fa2_status_t s = set_smem(kern, smem);
  if (s != FA2_OK) return s;
  p.num_m_blocks = (p.geom.Nq + 511) / 512;
  p.num_tiles = p.BH * p.num_m_blocks;
  // persistent grid of co-resident pairs: no more clusters than can be active at once
  // (the static pair-tile list would otherwise wait for a second wave)
  const int max_clusters = max_active_pairs(kern, smem, 384, sms);
  int grid = 2 * p.num_tiles < sms ? 2 * p.num_tiles : sms;
  grid &= ~1;
  if (grid > 2 * max_clusters) grid = 2 * max_clusters;
  if constexpr (CAUSAL && !GEN) {
    if (FA2_SCHED && p.num_tiles <= fa2::kSchedMaxTiles && grid / 2 <= fa2::kSchedMaxCtas) {
      const SchedPtr sc = fwd_pair_sched(p, grid / 2);
      mark(0, st);
      kern<<<grid, 384, smem, st>>>(mq, mk64, mv, mo, p, *sc);
      mark(1, st);
      FA2_CUDA(cudaGetLastError());
      return FA2_OK;
    }
  }
  fa2::SchedT<CAUSAL && !GEN> sched;
  sched.n = 0;
  mark(0, st);
  kern<<<grid, 384, smem, st>>>(mq, mk64, mv, mo, p, sched);
  mark(1, st);
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

fa2_status_t forward_impl(const void* q, const void* k, const void* v, void* o, float* lse, const Geom& g,
                          int causal, float scale, fa2_dtype_t dtype, cudaStream_t st, int sms) {
  CUtensorMap mq, mk, mv;
  const CUtensorMapDataType dt = tma_dtype(dtype);
  fa2_status_t s;
  if ((s = make_rows_map(&mq, q, dt, g, g.H, true)) != FA2_OK) return s;
  // CTA pair: every d = 128 bf16/fp16 forward (fixed layout incl. N_q != N_k, and packed varlen)
  const bool pair = FA2_FWD_PAIR && (!causal || FA2_FWD_PAIR_CAUSAL) && g.d == 128;
  if ((s = make_rows_map(&mk, k, dt, g, g.Hkv, false, 2, pair ? 64 : 128)) != FA2_OK) return s;
  if ((s = make_rows_map(&mv, v, dt, g, g.Hkv, false)) != FA2_OK) return s;
  fa2::FwdParams p;
  p.o = o;
  p.lse = lse;
  p.BH = g.B * g.H;
  p.H = g.H;
  p.Hkv = g.Hkv;
  p.group = g.H / g.Hkv;
  p.geom = seq_geom(g);
  const long long d = g.d;
  if (!g.packed) {
    p.o_rs = d; p.o_hs = static_cast<long long>(g.Nq) * d; p.o_bs = p.o_hs * g.H;
    p.l_hs = g.Nq; p.l_bs = static_cast<long long>(g.Nq) * g.H;
  } else {
    p.o_rs = d * g.H; p.o_hs = d; p.o_bs = 0;
    p.l_hs = g.Tq; p.l_bs = 0;
  }
  p.num_m_blocks = (g.Nq + 255) / 256;
  p.num_tiles = p.BH * p.num_m_blocks;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = g_trace;
  const bool bf16 = dtype == FA2_BF16;
  // O as a TMA store target (fixed layout; the packed layout stores rows one by one)
  CUtensorMap mo = mq;
  if (!g.packed && (s = make_rows_map(&mo, o, dt, g, g.H, true)) != FA2_OK) return s;
  if (pair) {
    if (g.packed) {
      if (causal) return bf16 ? launch_fwd_pair<true, true, true>(mq, mk, mv, mo, p, sms, st) : launch_fwd_pair<false, true, true>(mq, mk, mv, mo, p, sms, st);
      return bf16 ? launch_fwd_pair<true, false, true>(mq, mk, mv, mo, p, sms, st) : launch_fwd_pair<false, false, true>(mq, mk, mv, mo, p, sms, st);
    }
    if (causal) return bf16 ? launch_fwd_pair<true, true, false>(mq, mk, mv, mo, p, sms, st) : launch_fwd_pair<false, true, false>(mq, mk, mv, mo, p, sms, st);
    return bf16 ? launch_fwd_pair<true, false, false>(mq, mk, mv, mo, p, sms, st) : launch_fwd_pair<false, false, false>(mq, mk, mv, mo, p, sms, st);
  }
  if (g.d == 64)
    s = bf16 ? dispatch_fwd_causal<64, true>(causal, mq, mk, mv, mo, p, sms, st)
             : dispatch_fwd_causal<64, false>(causal, mq, mk, mv, mo, p, sms, st);
  else
#if !FA2_FWD_PAIR || !FA2_FWD_PAIR_CAUSAL
    // (d = 128 on the one-SM kernel: A/B builds without the pair forward only; the product
    // build instantiates it for FP8 alone)
    s = bf16 ? dispatch_fwd_causal<128, true>(causal, mq, mk, mv, mo, p, sms, st)
             : dispatch_fwd_causal<128, false>(causal, mq, mk, mv, mo, p, sms, st);
#else
    s = fail(FA2_ERR_UNSUPPORTED, "internal: d = 128 forward not routed to the pair kernel");
#endif
  return s;
}

// FP8 forward: E4M3 q, k, v with per-tensor descales, bf16 O.
fa2_status_t forward_fp8_impl(const void* q, const void* k, const void* v, void* o, float* lse, const Geom& g,
                              int causal, float scale, float dq, float dk, float dv, cudaStream_t st, int sms) {
  CUtensorMap mq, mk, mv;
  fa2_status_t s;
  if ((s = make_rows_map(&mq, q, CU_TENSOR_MAP_DATA_TYPE_UINT8, g, g.H, true, 1)) != FA2_OK) return s;
  if ((s = make_rows_map(&mk, k, CU_TENSOR_MAP_DATA_TYPE_UINT8, g, g.Hkv, false, 1)) != FA2_OK) return s;
  if ((s = make_rows_map(&mv, v, CU_TENSOR_MAP_DATA_TYPE_UINT8, g, g.Hkv, false, 1)) != FA2_OK) return s;
  fa2::FwdParams p;
  p.o = o;
  p.lse = lse;
  p.BH = g.B * g.H;
  p.H = g.H;
  p.Hkv = g.Hkv;
  p.group = g.H / g.Hkv;
  p.geom = seq_geom(g);
  const long long d = g.d;
  p.o_rs = d; p.o_hs = static_cast<long long>(g.Nq) * d; p.o_bs = p.o_hs * g.H;
  p.l_hs = g.Nq; p.l_bs = static_cast<long long>(g.Nq) * g.H;
  p.num_m_blocks = (g.Nq + 255) / 256;
  p.num_tiles = p.BH * p.num_m_blocks;
  // S = scale * (descale_q q8) . (descale_k k8): fold the descales into the exponent scale
  p.scale_log2 = static_cast<float>(static_cast<double>(scale) * dq * dk * 1.4426950408889634);
  p.o_descale = dv;
  p.trace = g_trace;
  CUtensorMap mo;   // O (bf16) as the TMA store target
  if ((s = make_rows_map(&mo, o, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, g, g.H, true)) != FA2_OK) return s;
  return causal ? launch_fwd<128, true, true, false, true>(mq, mk, mv, mo, p, sms, st)
                : launch_fwd<128, true, false, false, true>(mq, mk, mv, mo, p, sms, st);
}

// Copy streams and events of fa2_attention_step_host, created once per host thread and
// device (streams and events belong to the device that was current when they were made).
struct StepStreams {
  static constexpr int kChunks = 16;
  cudaStream_t in = nullptr, out = nullptr;
  cudaEvent_t start = nullptr, in_done[kChunks] = {}, comp_done[kChunks] = {};
};
StepStreams& step_streams() {
  thread_local std::map<int, StepStreams> per_dev;
  int dev = 0;
  cudaGetDevice(&dev);
  StepStreams& ss = per_dev[dev];
  if (ss.in == nullptr) {
    StepStreams t;
    bool ok = cudaStreamCreateWithFlags(&t.in, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&t.out, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&t.start, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < StepStreams::kChunks; ++i)
      ok = cudaEventCreateWithFlags(&t.in_done[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&t.comp_done[i], cudaEventDisableTiming) == cudaSuccess;
    if (ok) ss = t;
  }
  return ss;
}

// ----------------------------------------------------------------------------
// Backward
// ----------------------------------------------------------------------------
size_t pad128(long long N) { return static_cast<size_t>((N + 127) / 128) * 128; }
size_t round16(size_t b) { return (b + 15) / 16 * 16; }

// Backward workspace (both layouts), in this order:
//   dq_acc [rows, d] fp32 | D [rows] fp32 | L*log2e [rows] fp32 | counters [rows/32] int32 |
//   tile_off [B+1] int32 (packed only)
// rows = padded query rows: fixed B*H*N_pad; packed H * pad128(T_q + 127 B) (every sequence is
// padded to whole 128-row tiles, fa2_bwd_sm100.cuh RowParams).
struct WsLayout {
  long long rows = 0, rows_per_head = 0;
  size_t dq = 0, dvec = 0, lse2 = 0, sem = 0, tile = 0, total = 0;
};
WsLayout ws_layout(const Geom& g) {
  WsLayout w;
  if (!g.packed) {
    w.rows_per_head = static_cast<long long>(pad128(g.Nq));
    w.rows = static_cast<long long>(g.B) * g.H * w.rows_per_head;
  } else {
    w.rows_per_head = static_cast<long long>(pad128(static_cast<long long>(g.Tq) + 127LL * g.B));
    w.rows = static_cast<long long>(g.H) * w.rows_per_head;
  }
  w.dq = 0;
  w.dvec = w.dq + static_cast<size_t>(w.rows) * g.d * 4;
  w.lse2 = w.dvec + static_cast<size_t>(w.rows) * 4;
  w.sem = w.lse2 + static_cast<size_t>(w.rows) * 4;
  w.tile = w.sem + round16(static_cast<size_t>(w.rows / 32) * 4);   // 4 counters per 128-row tile
  w.total = w.tile + (g.packed ? round16(static_cast<size_t>(g.B + 1) * 4) : 0);
  return w;
}

fa2::RowParams row_params(const Geom& g, const WsLayout& w, const void* o, const void* dout, void* dq,
                          const float* lse, void* ws) {
  fa2::RowParams r;
  uint8_t* base = reinterpret_cast<uint8_t*>(ws);
  r.o = o;
  r.dout = dout;
  r.dq = dq;
  r.lse = lse;
  r.dq_acc = reinterpret_cast<float*>(base + w.dq);
  r.dvec = reinterpret_cast<float*>(base + w.dvec);
  r.lse2 = reinterpret_cast<float*>(base + w.lse2);
  r.dq_sem = nullptr;
  r.B = g.B;
  r.H = g.H;
  r.Nq = g.Nq;
  r.cu_q = g.packed ? g.cu_q : nullptr;
  r.tile_off = g.packed ? reinterpret_cast<const int*>(base + w.tile) : nullptr;
  r.acc_hs = w.rows_per_head;
  r.acc_rows = w.rows;
  const long long d = g.d;
  if (!g.packed) {
    r.o_rs = d; r.o_hs = static_cast<long long>(g.Nq) * d; r.o_bs = r.o_hs * g.H;
    r.l_hs = g.Nq; r.l_bs = static_cast<long long>(g.Nq) * g.H;
  } else {
    r.o_rs = d * g.H; r.o_hs = d; r.o_bs = 0;
    r.l_hs = g.Tq; r.l_bs = 0;
  }
  return r;
}

fa2_status_t preprocess_impl(const fa2::RowParams& rp, int d, fa2_dtype_t dtype, cudaStream_t st) {
  // d / 8 threads per padded workspace row, 256-thread blocks
  if (rp.acc_rows >= (1LL << 31)) return fail(FA2_ERR_INVALID_ARG, "problem too large: %lld padded query rows", rp.acc_rows);
  const long long grid = (rp.acc_rows * (d / 8) + 255) / 256;
  if (grid >= (1LL << 31)) return fail(FA2_ERR_INVALID_ARG, "problem too large: %lld padded query rows", rp.acc_rows);
  const bool bf16 = dtype == FA2_BF16;
  if (d == 64) {
    if (bf16) fa2::fa2_bwd_preprocess<64, true><<<static_cast<int>(grid), 256, 0, st>>>(rp);
    else fa2::fa2_bwd_preprocess<64, false><<<static_cast<int>(grid), 256, 0, st>>>(rp);
  } else {
    if (bf16) fa2::fa2_bwd_preprocess<128, true><<<static_cast<int>(grid), 256, 0, st>>>(rp);
    else fa2::fa2_bwd_preprocess<128, false><<<static_cast<int>(grid), 256, 0, st>>>(rp);
  }
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

// 2-D fp32 view {d, rows} of dq_acc with box {32, 128} (d = 64 kernel's tensor reduce-adds).
fa2_status_t make_acc_map(CUtensorMap* m, float* dq_acc, int d, long long rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(FA2_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 4};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq_acc, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FA2_ERR_CUDA, "cuTensorMapEncodeTiled (dq_acc) failed (%d)", static_cast<int>(r));
  return FA2_OK;
}

template <bool SCHED, typename Kern>
fa2_status_t launch_bwd_kernel(Kern kern, int smem, const fa2::BwdMaps& maps, const fa2::BwdParams& p, int sms,
                               cudaStream_t st) {
  fa2_status_t s = set_smem(kern, smem);
  if (s != FA2_OK) return s;
  int grid = p.num_tiles < sms ? p.num_tiles : sms;
  // deterministic cyclic schedule: whole heads per wave (see bwd_q_tile in fa2_bwd_sm100.cuh)
  if (p.dq_sem != nullptr && p.det_cyclic) grid = (grid / p.num_n_blocks) * p.num_n_blocks;
  fa2::SchedT<SCHED> sched;
  sched.n = 0;
  if constexpr (SCHED) {   // causal square arrival-order backward: balanced tile lists
    if (FA2_SCHED && p.dq_sem == nullptr && p.num_tiles <= fa2::kSchedMaxTiles && grid <= fa2::kSchedMaxCtas) {
      const SchedPtr sc = bwd_sched(p, grid);
      mark(3, st);
      kern<<<grid, fa2::kBwdThreads, smem, st>>>(maps.q, maps.k, maps.v, maps.dout, maps.dq_acc, p, *sc);
      mark(4, st);
      FA2_CUDA(cudaGetLastError());
      return FA2_OK;
    }
  }
  mark(3, st);
  kern<<<grid, fa2::kBwdThreads, smem, st>>>(maps.q, maps.k, maps.v, maps.dout, maps.dq_acc, p, sched);
  mark(4, st);
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

template <int D, bool BF16, bool CAUSAL, bool GEN>
fa2_status_t launch_bwd(const fa2::BwdMaps& maps, const fa2::BwdParams& p, int sms, cudaStream_t st) {
  // d = 128: fa2_bwd128_sm100.cuh; d = 64: fa2_bwd_kernel
  if constexpr (D == 128)
    return launch_bwd_kernel<CAUSAL && !GEN>(fa2::fa2_bwd128_kernel<BF16, CAUSAL, GEN>, fa2::Bwd128Smem::ALLOC, maps, p,
                                             sms, st);
  else
    return launch_bwd_kernel<CAUSAL && !GEN>(fa2::fa2_bwd_kernel<D, BF16, CAUSAL, GEN>, fa2::BwdSmem<D>::ALLOC, maps, p,
                                             sms, st);
}

template <int D, bool BF16>
fa2_status_t dispatch_bwd_causal(bool causal, const fa2::BwdMaps& maps, const fa2::BwdParams& p, int sms,
                                 cudaStream_t st) {
  if (p.geom.cu_q != nullptr || p.geom.Nq != p.geom.Nk)   // general geometry
    return causal ? launch_bwd<D, BF16, true, true>(maps, p, sms, st) : launch_bwd<D, BF16, false, true>(maps, p, sms, st);
  return causal ? launch_bwd<D, BF16, true, false>(maps, p, sms, st) : launch_bwd<D, BF16, false, false>(maps, p, sms, st);
}

#ifndef FA2_BWD_PAIR
#define FA2_BWD_PAIR 1   // 0: the one-SM d = 128 backward kernel for every shape (A/B builds)
#endif
// CTA-pair backward (fa2_bwd2_sm100.cuh): d = 128, every geometry (GEN: N_q != N_k and/or
// packed variable-length), arrival-order or deterministic dQ.  p arrives with the 128-row
// tiling; the pair kernel tiles keys by 256.
template <bool BF16, bool CAUSAL, bool GEN>
fa2_status_t launch_bwd_pair(const fa2::BwdMaps& maps, const CUtensorMap& mq64, const CUtensorMap& mdo64,
                             const CUtensorMap& mdk, const CUtensorMap& mdv, fa2::BwdParams p, int sms, cudaStream_t st) {
  auto kern = fa2::fa2_bwd_pair_kernel<BF16, CAUSAL, GEN>;
  constexpr int smem = fa2::BwdPairSmem::ALLOC;
  fa2_status_t s = set_smem(kern, smem);
  if (s != FA2_OK) return s;
  const int N = p.geom.Nq;
  p.num_n_blocks = (p.geom.Nk + 255) / 256;
  p.num_tiles = (p.BH / p.group) * p.hsplit * p.num_n_blocks;
  int npairs = std::min(p.num_tiles, std::min(sms / 2, max_active_pairs(kern, smem, fa2::kBwdThreads, sms)));
  if (p.dq_sem != nullptr) {
    // deterministic mode (fa2_bwd2_sm100.cuh pair_q_tile / pair_rank): the cyclic order needs an
    // even number of query tiles and a head's key blocks side by side, i.e. a pair grid that is
    // a multiple of them
#ifndef FA2_DET_CYCLIC_PAIR
#define FA2_DET_CYCLIC_PAIR 1
#endif
    p.det_cyclic = (!GEN && FA2_DET_CYCLIC_PAIR && p.num_n_blocks <= npairs && ((N + 127) / 128) % 2 == 0) ? 1 : 0;
    if (p.det_cyclic) npairs = (npairs / p.num_n_blocks) * p.num_n_blocks;
  }
  fa2::SchedT<CAUSAL && !GEN> sched;
  sched.n = 0;
  if constexpr (CAUSAL && !GEN) {   // balanced pair-tile lists: key block nb2 sees nqb - 2 nb2 query tiles per head
    if (FA2_SCHED && p.dq_sem == nullptr && p.num_tiles <= fa2::kSchedMaxTiles && npairs <= fa2::kSchedMaxCtas) {
      const int nnb2 = p.num_n_blocks, nh = p.group / p.hsplit, nt = p.num_tiles;
      const SchedPtr sc = cached_sched(2, nt, nnb2, N, nh, npairs, [&](std::vector<int>& work) {
        const int nqb = (N + 127) / 128;
        for (int t = 0; t < nt; ++t) work[t] = (nqb - 2 * (t % nnb2)) * nh + 1;
      });
      mark(3, st);
      kern<<<2 * npairs, fa2::kBwdThreads, smem, st>>>(mq64, maps.q, maps.k, maps.v, mdo64, maps.dout, mdk, mdv, p, *sc);
      mark(4, st);
      FA2_CUDA(cudaGetLastError());
      return FA2_OK;
    }
  }
  mark(3, st);
  kern<<<2 * npairs, fa2::kBwdThreads, smem, st>>>(mq64, maps.q, maps.k, maps.v, mdo64, maps.dout, mdk, mdv, p, sched);
  mark(4, st);
  FA2_CUDA(cudaGetLastError());
  return FA2_OK;
}

// GQA load balance (BwdParams::hsplit): the query heads of a key/value group are split
// over `hsplit` work tiles when the unsplit tile count would leave SMs idle (< 2 waves) or,
// causal, when the heaviest tile exceeds a quarter of an SM's average share.  Needs fp32 dK/dV
// accumulators (2 * numel(dk) * 4 bytes) after the base workspace; not used in the
// deterministic mode (the fp32 reduce-adds would make dK/dV order-dependent).
int choose_hsplit(const Geom& g, bool causal, bool deterministic, int sms, size_t ws_bytes, size_t base,
                  size_t& acc_off, long long& dk_numel) {
  const int group = g.H / g.Hkv;
  dk_numel = (g.packed ? static_cast<long long>(g.Tk) : static_cast<long long>(g.B) * g.Nk) * g.Hkv * g.d;
  acc_off = (base + 255) / 256 * 256;
  if (group == 1 || deterministic || ws_bytes < acc_off + static_cast<size_t>(dk_numel) * 8) return 1;
  // the CTA-pair kernel (square fixed-length d = 128) tiles keys by 256 on pairs of SMs
  const bool pair_path = g.d == 128;
  const long long kb = pair_path ? 256 : 128, units = pair_path ? sms / 2 : sms;
  const long long nkb = (g.Nk + kb - 1) / kb, nqb = (g.Nq + 127) / 128;
  const long long tiles1 = static_cast<long long>(g.B) * g.Hkv * nkb;
  long long need = (2LL * units + tiles1 - 1) / tiles1;
  if (causal) {   // heaviest tile (key block 0: nqb query tiles x group/split heads) <= 1/4 of an SM's share
    const long long den = (nqb + 1) * g.B * g.Hkv;
    need = std::max(need, (8LL * units * (pair_path ? 2 : 1) + den - 1) / den);
  }
  for (int sp = 1; sp <= group; ++sp)
    if (group % sp == 0 && sp >= need) return sp;
  return group;
}

fa2_status_t backward_impl(const void* q, const void* k, const void* v, const void* o, const float* lse,
                           const void* dout, void* dq, void* dk, void* dv, void* ws, const Geom& g, int causal,
                           float scale, fa2_dtype_t dtype, cudaStream_t st, int sms, bool deterministic,
                           size_t ws_bytes) {
  const WsLayout wl = ws_layout(g);
  size_t acc_off = 0;
  long long dk_numel = 0;
  const int hsplit = choose_hsplit(g, causal != 0, deterministic, sms, ws_bytes, wl.total, acc_off, dk_numel);
  float* dk_acc = hsplit > 1 ? reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) + acc_off) : nullptr;
  float* dv_acc = hsplit > 1 ? dk_acc + dk_numel : nullptr;
  fa2::RowParams rp = row_params(g, wl, o, dout, dq, lse, ws);
  int* dq_sem = deterministic ? reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ws) + wl.sem) : nullptr;
  rp.dq_sem = dq_sem;
  mark(2, st);
  if (g.packed) {
    fa2::fa2_tile_prefix<<<1, 1024, 0, st>>>(g.cu_q, g.B, const_cast<int*>(rp.tile_off));
    FA2_CUDA(cudaGetLastError());
  }
  fa2_status_t s = preprocess_impl(rp, g.d, dtype, st);
  if (s != FA2_OK) return s;
  if (hsplit > 1) FA2_CUDA(cudaMemsetAsync(dk_acc, 0, static_cast<size_t>(dk_numel) * 8, st));
  fa2::BwdMaps maps;
  const CUtensorMapDataType dt = tma_dtype(dtype);
  if ((s = make_rows_map(&maps.q, q, dt, g, g.H, true)) != FA2_OK) return s;
  if ((s = make_rows_map(&maps.dout, dout, dt, g, g.H, true)) != FA2_OK) return s;
  if ((s = make_rows_map(&maps.k, k, dt, g, g.Hkv, false)) != FA2_OK) return s;
  if ((s = make_rows_map(&maps.v, v, dt, g, g.Hkv, false)) != FA2_OK) return s;
  if ((s = make_acc_map(&maps.dq_acc, rp.dq_acc, g.d, wl.rows)) != FA2_OK) return s;
  fa2::BwdParams p;
  p.lse = lse;
  p.dvec = rp.dvec;
  p.dk = dk;
  p.dv = dv;
  p.dq_acc = rp.dq_acc;
  p.BH = g.B * g.H;
  p.H = g.H;
  p.Hkv = g.Hkv;
  p.group = g.H / g.Hkv;
  p.num_n_blocks = (g.Nk + 127) / 128;
  p.hsplit = hsplit;
  p.dk_acc = dk_acc;
  p.dv_acc = dv_acc;
  // one work tile per (sequence, key/value head, query-head split, key block)
  p.num_tiles = g.B * g.Hkv * hsplit * p.num_n_blocks;
  p.scale = scale;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.trace = g_trace;
  p.dq_sem = dq_sem;
  // the cyclic deterministic schedule needs one square query/key tile grid per head
  p.det_cyclic = (!g.packed && g.Nq == g.Nk && p.num_n_blocks <= sms) ? 1 : 0;
  p.geom = seq_geom(g);
  const long long d = g.d;
  if (!g.packed) {
    p.k_rs = d; p.k_hs = static_cast<long long>(g.Nk) * d; p.k_bs = p.k_hs * g.Hkv;
    p.acc_hs = wl.rows_per_head; p.acc_bs = wl.rows_per_head * g.H;
  } else {
    p.k_rs = d * g.Hkv; p.k_hs = d; p.k_bs = 0;
    p.acc_hs = wl.rows_per_head; p.acc_bs = 0;
  }
  p.acc_rows = wl.rows;
  p.tile_off = rp.tile_off;
  const bool bf16 = dtype == FA2_BF16;
  // the CTA-pair kernel serves the square fixed-length arrival-order d = 128
  // path; FA2_BWD_PAIR=0 in the environment selects the one-SM kernel instead (A/B runs and
  // the one-SM kernel's parity test)
  static const bool pair_env = [] { const char* e = std::getenv("FA2_BWD_PAIR"); return !(e && e[0] == '0'); }();
  const bool pair = FA2_BWD_PAIR && pair_env && g.d == 128;
  if (pair) {
    CUtensorMap mq64, mdo64;
    if ((s = make_rows_map(&mq64, q, dt, g, g.H, true, 2, 64)) != FA2_OK) return s;
    if ((s = make_rows_map(&mdo64, dout, dt, g, g.H, true, 2, 64)) != FA2_OK) return s;
    // dK / dV as TMA store targets (fixed layout; the packed one stores rows one by one)
    CUtensorMap mdk = maps.k, mdv = maps.v;
    if (!g.packed && hsplit == 1) {
      if ((s = make_rows_map(&mdk, dk, dt, g, g.Hkv, false)) != FA2_OK) return s;
      if ((s = make_rows_map(&mdv, dv, dt, g, g.Hkv, false)) != FA2_OK) return s;
    }
    const bool gen = g.packed || g.Nq != g.Nk;
#define FA2_PAIR_LAUNCH(B16, C, G) launch_bwd_pair<B16, C, G>(maps, mq64, mdo64, mdk, mdv, p, sms, st)
    if (gen)
      s = bf16 ? (causal ? FA2_PAIR_LAUNCH(true, true, true) : FA2_PAIR_LAUNCH(true, false, true))
               : (causal ? FA2_PAIR_LAUNCH(false, true, true) : FA2_PAIR_LAUNCH(false, false, true));
    else
      s = bf16 ? (causal ? FA2_PAIR_LAUNCH(true, true, false) : FA2_PAIR_LAUNCH(true, false, false))
               : (causal ? FA2_PAIR_LAUNCH(false, true, false) : FA2_PAIR_LAUNCH(false, false, false));
#undef FA2_PAIR_LAUNCH
  } else if (g.d == 64)
    s = bf16 ? dispatch_bwd_causal<64, true>(causal, maps, p, sms, st) : dispatch_bwd_causal<64, false>(causal, maps, p, sms, st);
  else
    s = bf16 ? dispatch_bwd_causal<128, true>(causal, maps, p, sms, st)
             : dispatch_bwd_causal<128, false>(causal, maps, p, sms, st);
  if (s != FA2_OK) return s;
  if (hsplit > 1) {   // dK, dV = cast(fp32 sums over the group's query-head splits)
    const long long n8 = dk_numel / 8;
    const long long grid = (2 * n8 + 255) / 256;
    if (bf16) fa2::fa2_dkv_convert<true><<<static_cast<int>(grid), 256, 0, st>>>(dk_acc, dv_acc, dk, dv, n8);
    else fa2::fa2_dkv_convert<false><<<static_cast<int>(grid), 256, 0, st>>>(dk_acc, dv_acc, dk, dv, n8);
    FA2_CUDA(cudaGetLastError());
  }
  // dQ = cast(dq_acc) (the softmax scale is already applied to dS), real rows only
  {
    const long long rows_out = g.packed ? static_cast<long long>(g.Tq) * g.H : static_cast<long long>(g.B) * g.H * g.Nq;
    if (rows_out >= (1LL << 31)) return fail(FA2_ERR_INVALID_ARG, "problem too large: %lld query rows", rows_out);
    const long long grid = (rows_out * (g.d / 8) + 255) / 256;
    if (g.d == 64) {
      if (bf16) fa2::fa2_dq_convert<64, true><<<static_cast<int>(grid), 256, 0, st>>>(rp, rows_out);
      else fa2::fa2_dq_convert<64, false><<<static_cast<int>(grid), 256, 0, st>>>(rp, rows_out);
    } else if (pair) {   // the pair kernel's chunked accumulator layout, one thread per (padded row, 8 columns)
      const long long pgrid = (wl.rows * (g.d / 8) + 255) / 256;
      if (bf16) fa2::fa2_dq_convert_pair<true><<<static_cast<int>(pgrid), 256, 0, st>>>(rp);
      else fa2::fa2_dq_convert_pair<false><<<static_cast<int>(pgrid), 256, 0, st>>>(rp);
    } else if (fa2::kBwdDqLsu) {   // fa2_bwd128_kernel's chunked accumulator layout
      const long long cgrid = (wl.rows / 4 * (g.d / 8) + 255) / 256;
      if (bf16) fa2::fa2_dq_convert_chunked<true><<<static_cast<int>(cgrid), 256, 0, st>>>(rp);
      else fa2::fa2_dq_convert_chunked<false><<<static_cast<int>(cgrid), 256, 0, st>>>(rp);
    } else {
      if (bf16) fa2::fa2_dq_convert<128, true><<<static_cast<int>(grid), 256, 0, st>>>(rp, rows_out);
      else fa2::fa2_dq_convert<128, false><<<static_cast<int>(grid), 256, 0, st>>>(rp, rows_out);
    }
    FA2_CUDA(cudaGetLastError());
    mark(5, st);
  }
  return FA2_OK;
}

fa2_status_t backward_entry(const void* q, const void* k, const void* v, const void* o, const float* lse,
                            const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                            const Geom& g, float softmax_scale, fa2_dtype_t dtype, void* stream, int causal,
                            bool deterministic);

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

fa2_status_t fa2_tile_schedule(int pass, int heads, int N, int heads_per_tile, int grid, unsigned short* order,
                               unsigned short* start, int capacity, int* n_tiles) {
  if ((pass != 0 && pass != 1) || heads < 1 || N < 1 || heads_per_tile < 1 || grid < 1 ||
      grid > fa2::kSchedMaxCtas || order == nullptr || start == nullptr || n_tiles == nullptr)
    return fail(FA2_ERR_INVALID_ARG, "fa2_tile_schedule: bad arguments");
  const long long per_head = pass == 0 ? (N + 255) / 256 : (N + 127) / 128;
  const long long T = per_head * heads;
  if (T > fa2::kSchedMaxTiles || T > capacity)
    return fail(FA2_ERR_INVALID_ARG, "fa2_tile_schedule: %lld tiles (max %d, capacity %d)", T, fa2::kSchedMaxTiles,
                capacity);
  SchedPtr sc;
  if (pass == 0) {
    fa2::FwdParams p{};
    p.num_m_blocks = static_cast<int>(per_head);
    p.num_tiles = static_cast<int>(T);
    p.geom.Nq = p.geom.Nk = N;
    sc = fwd_sched(p, grid);
  } else {
    fa2::BwdParams p{};
    p.num_n_blocks = static_cast<int>(per_head);
    p.num_tiles = static_cast<int>(T);
    p.geom.Nq = p.geom.Nk = N;
    p.group = heads_per_tile;
    p.hsplit = 1;
    sc = bwd_sched(p, grid);
  }
  for (int c = 0; c <= grid; ++c) start[c] = sc->start[c];
  for (long long t = 0; t < T; ++t) order[t] = sc->order[t];
  *n_tiles = static_cast<int>(T);
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
  s = forward_impl(q, k, v, o, lse, fixed_geom(B, H, H_kv, N, N, d), causal, softmax_scale, dtype,
                   static_cast<cudaStream_t>(stream), di.sms);
  if (s == FA2_OK) g_launches = 1;
  return s;
}

fa2_status_t fa2_forward_ex(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H, int H_kv,
                            int N_q, int N_k, int d, int causal, float softmax_scale, fa2_dtype_t dtype, void* stream) {
  g_detail.clear();
  fa2_status_t s = check_common(B, H, N_q, d, softmax_scale, dtype, true);
  if (s != FA2_OK) return s;
  if (N_k < 1) return fail(FA2_ERR_INVALID_ARG, "N_k must be >= 1 (got %d)", N_k);
  if (H_kv < 1 || H % H_kv != 0) return fail(FA2_ERR_INVALID_ARG, "H=%d must be a positive multiple of H_kv=%d", H, H_kv);
  if ((s = check_ptrs({q, k, v, o, lse})) != FA2_OK) return s;
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  s = forward_impl(q, k, v, o, lse, fixed_geom(B, H, H_kv, N_q, N_k, d), causal, softmax_scale, dtype,
                   static_cast<cudaStream_t>(stream), di.sms);
  if (s == FA2_OK) g_launches = 1;
  return s;
}

fa2_status_t fa2_forward_varlen(const void* q, const void* k, const void* v, void* o, float* lse,
                                const int* cu_seqlens_q, const int* cu_seqlens_k, int B, int H, int H_kv,
                                int total_q, int total_k, int max_seqlen_q, int max_seqlen_k, int d, int causal,
                                float softmax_scale, fa2_dtype_t dtype, void* stream) {
  g_detail.clear();
  fa2_status_t s;
  Geom g;
  if ((s = varlen_geom(cu_seqlens_q, cu_seqlens_k, B, H, H_kv, total_q, total_k, max_seqlen_q, max_seqlen_k, d,
                       softmax_scale, dtype, g)) != FA2_OK)
    return s;
  if ((s = check_ptrs({q, k, v, o, lse})) != FA2_OK) return s;
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  s = forward_impl(q, k, v, o, lse, g, causal, softmax_scale, dtype, static_cast<cudaStream_t>(stream), di.sms);
  if (s == FA2_OK) g_launches = 1;
  return s;
}

fa2_status_t fa2_forward_fp8(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H, int H_kv,
                             int N, int d, int causal, float softmax_scale, float descale_q, float descale_k,
                             float descale_v, void* stream) {
  g_detail.clear();
  fa2_status_t s = check_common(B, H, N, d, softmax_scale, FA2_BF16, true);
  if (s != FA2_OK) return s;
  if (d != 128) return fail(FA2_ERR_UNSUPPORTED, "FP8 forward supports d = 128 (got %d)", d);
  if (H_kv < 1 || H % H_kv != 0) return fail(FA2_ERR_INVALID_ARG, "H=%d must be a positive multiple of H_kv=%d", H, H_kv);
  for (float x : {descale_q, descale_k, descale_v})
    if (!(std::isfinite(x) && x > 0.f)) return fail(FA2_ERR_INVALID_ARG, "descale factors must be finite and > 0");
  if ((s = check_ptrs({q, k, v, o, lse})) != FA2_OK) return s;
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  s = forward_fp8_impl(q, k, v, o, lse, fixed_geom(B, H, H_kv, N, N, d), causal, softmax_scale, descale_q, descale_k,
                       descale_v, static_cast<cudaStream_t>(stream), di.sms);
  if (s == FA2_OK) g_launches = 1;
  return s;
}

fa2_status_t fa2_forward(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H, int N, int d,
                         int causal, float softmax_scale, fa2_dtype_t dtype, void* stream) {
  return fa2_forward_gqa(q, k, v, o, lse, B, H, H, N, d, causal, softmax_scale, dtype, stream);
}

size_t fa2_backward_workspace_size(int B, int H, int N, int d) {
  if (B < 1 || H < 1 || N < 1 || (d != 64 && d != 128)) return 0;
  // base layout + room for the GQA split's fp32 dK/dV accumulators (H_kv <= H, N_k = N)
  return (ws_layout(fixed_geom(B, H, H, N, N, d)).total + 255) / 256 * 256 + static_cast<size_t>(B) * H * N * d * 8;
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
  return backward_entry(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes, fixed_geom(B, H, H_kv, N, N, d),
                        softmax_scale, dtype, stream, causal, false);
}

fa2_status_t fa2_backward_deterministic(const void* q, const void* k, const void* v, const void* o, const float* lse,
                                        const void* dout, void* dq, void* dk, void* dv, void* workspace,
                                        size_t workspace_bytes, int B, int H, int H_kv, int N, int d, int causal,
                                        float softmax_scale, fa2_dtype_t dtype, void* stream) {
  return backward_entry(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes, fixed_geom(B, H, H_kv, N, N, d),
                        softmax_scale, dtype, stream, causal, true);
}

fa2_status_t fa2_backward_ex(const void* q, const void* k, const void* v, const void* o, const float* lse,
                             const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                             int B, int H, int H_kv, int N_q, int N_k, int d, int causal, float softmax_scale,
                             int deterministic, fa2_dtype_t dtype, void* stream) {
  if (N_k < 1) {
    g_detail.clear();
    return fail(FA2_ERR_INVALID_ARG, "N_k must be >= 1 (got %d)", N_k);
  }
  return backward_entry(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes,
                        fixed_geom(B, H, H_kv, N_q, N_k, d), softmax_scale, dtype, stream, causal, deterministic != 0);
}

size_t fa2_backward_varlen_workspace_size(int B, int H, int total_q, int d) {
  if (B < 1 || H < 1 || total_q < 1 || (d != 64 && d != 128)) return 0;
  Geom g;
  g.B = B; g.H = H; g.Hkv = H; g.d = d; g.packed = true; g.Tq = total_q;
  // base layout + room for the GQA split's fp32 dK/dV accumulators when total_k <= total_q
  return (ws_layout(g).total + 255) / 256 * 256 + static_cast<size_t>(total_q) * H * d * 8;
}

fa2_status_t fa2_backward_varlen(const void* q, const void* k, const void* v, const void* o, const float* lse,
                                 const void* dout, void* dq, void* dk, void* dv, const int* cu_seqlens_q,
                                 const int* cu_seqlens_k, void* workspace, size_t workspace_bytes, int B, int H,
                                 int H_kv, int total_q, int total_k, int max_seqlen_q, int max_seqlen_k, int d,
                                 int causal, float softmax_scale, int deterministic, fa2_dtype_t dtype, void* stream) {
  g_detail.clear();
  Geom g;
  fa2_status_t s = varlen_geom(cu_seqlens_q, cu_seqlens_k, B, H, H_kv, total_q, total_k, max_seqlen_q, max_seqlen_k,
                               d, softmax_scale, dtype, g);
  if (s != FA2_OK) return s;
  return backward_entry(q, k, v, o, lse, dout, dq, dk, dv, workspace, workspace_bytes, g, softmax_scale, dtype, stream,
                        causal, deterministic != 0);
}

}  // extern "C"

namespace {
fa2_status_t backward_entry(const void* q, const void* k, const void* v, const void* o, const float* lse,
                            const void* dout, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes,
                            const Geom& g, float softmax_scale, fa2_dtype_t dtype, void* stream, int causal,
                            bool deterministic) {
  g_detail.clear();
  fa2_status_t s = check_common(g.B, g.H, g.packed ? 1 : g.Nq, g.d, softmax_scale, dtype, true);
  if (s != FA2_OK) return s;
  if (g.Hkv < 1 || g.H % g.Hkv != 0)
    return fail(FA2_ERR_INVALID_ARG, "H=%d must be a positive multiple of H_kv=%d", g.H, g.Hkv);
  if ((s = check_ptrs({q, k, v, o, lse, dout, dq, dk, dv})) != FA2_OK) return s;
  if (workspace == nullptr || !aligned16(workspace))
    return fail(FA2_ERR_WORKSPACE, "workspace is NULL or not 16-byte aligned");
  const size_t need = ws_layout(g).total;
  if (workspace_bytes < need) return fail(FA2_ERR_WORKSPACE, "workspace too small: %zu < %zu", workspace_bytes, need);
  DeviceInfo di;
  if ((s = device_info(di)) != FA2_OK) return s;
  s = backward_impl(q, k, v, o, lse, dout, dq, dk, dv, workspace, g, causal, softmax_scale, dtype,
                    static_cast<cudaStream_t>(stream), di.sms, deterministic, workspace_bytes);
  if (s == FA2_OK) {
    size_t acc_off = 0;
    long long dk_numel = 0;
    const bool split = choose_hsplit(g, causal != 0, deterministic, di.sms, workspace_bytes, need, acc_off, dk_numel) > 1;
    g_launches = (g.packed ? 4 : 3) + (split ? 1 : 0);
  }
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
  // d_out has N entries per head (no padding): the fixed row geometry with N_pad = N
  fa2::RowParams rp{};
  rp.o = o;
  rp.dout = dout;
  rp.dvec = d_out;
  rp.B = B;
  rp.H = H;
  rp.Nq = N;
  rp.acc_hs = N;
  rp.acc_rows = static_cast<long long>(B) * H * N;
  rp.o_rs = d;
  rp.o_hs = static_cast<long long>(N) * d;
  rp.o_bs = rp.o_hs * H;
  if ((s = preprocess_impl(rp, d, dtype, static_cast<cudaStream_t>(stream))) != FA2_OK) return s;
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
  // The (b, h) units are independent and contiguous in every tensor, so the
  // step runs as a pipeline over chunks of units: chunk c's inputs are copied in on one
  // stream while chunk c-1 computes on `stream` and chunk c-2's results are copied out
  // on a third -- the copies in both directions overlap each other and the kernels.
  StepStreams& ss = step_streams();
  if (ss.in == nullptr) return fail(FA2_ERR_CUDA, "could not create the copy streams");
  const int units = B * H;
  const int nchunks = units < StepStreams::kChunks ? units : StepStreams::kChunks;
  const int per = (units + nchunks - 1) / nchunks;
  const size_t urow = static_cast<size_t>(N) * d * 2;   // bytes of one unit of q/k/v/o/...
  FA2_CUDA(cudaEventRecord(ss.start, st));              // order after the caller's prior work
  FA2_CUDA(cudaStreamWaitEvent(ss.in, ss.start, 0));
  FA2_CUDA(cudaStreamWaitEvent(ss.out, ss.start, 0));
  const uint8_t* hin[4] = {static_cast<const uint8_t*>(q_h), static_cast<const uint8_t*>(k_h),
                           static_cast<const uint8_t*>(v_h), static_cast<const uint8_t*>(dout_h)};
  uint8_t* din[4] = {static_cast<uint8_t*>(q), static_cast<uint8_t*>(k), static_cast<uint8_t*>(v),
                     static_cast<uint8_t*>(dout)};
  uint8_t* hout[4] = {static_cast<uint8_t*>(o_h), static_cast<uint8_t*>(dq_h), static_cast<uint8_t*>(dk_h),
                      static_cast<uint8_t*>(dv_h)};
  const uint8_t* dout_[4] = {static_cast<const uint8_t*>(o), static_cast<const uint8_t*>(dq),
                             static_cast<const uint8_t*>(dk), static_cast<const uint8_t*>(dv)};
  int launches = 0;
  for (int c = 0, u0 = 0; u0 < units; ++c, u0 += per) {
    const int nu = units - u0 < per ? units - u0 : per;
    const size_t off = static_cast<size_t>(u0) * urow, bytes = static_cast<size_t>(nu) * urow;
    for (int i = 0; i < 4; ++i) FA2_CUDA(cudaMemcpyAsync(din[i] + off, hin[i] + off, bytes, cudaMemcpyHostToDevice, ss.in));
    FA2_CUDA(cudaEventRecord(ss.in_done[c], ss.in));
    FA2_CUDA(cudaStreamWaitEvent(st, ss.in_done[c], 0));
    auto at = [&](void* p) { return static_cast<void*>(static_cast<uint8_t*>(p) + off); };
    float* lse_c = lse + static_cast<size_t>(u0) * N;
    const Geom gc = fixed_geom(1, nu, nu, N, N, d);   // this chunk: nu independent heads
    if ((s = forward_impl(at(q), at(k), at(v), at(o), lse_c, gc, causal, softmax_scale, dtype, st, di.sms)) != FA2_OK)
      return s;
    if ((s = backward_impl(at(q), at(k), at(v), at(o), lse_c, at(dout), at(dq), at(dk), at(dv), ws, gc, causal,
                           softmax_scale, dtype, st, di.sms, false, 0)) != FA2_OK)
      return s;
    launches += 4;
    FA2_CUDA(cudaEventRecord(ss.comp_done[c], st));
    FA2_CUDA(cudaStreamWaitEvent(ss.out, ss.comp_done[c], 0));
    for (int i = 0; i < 4; ++i)
      if (hout[i]) FA2_CUDA(cudaMemcpyAsync(hout[i] + off, dout_[i] + off, bytes, cudaMemcpyDeviceToHost, ss.out));
    if (lse_h)
      FA2_CUDA(cudaMemcpyAsync(lse_h + static_cast<size_t>(u0) * N, lse_c, static_cast<size_t>(nu) * N * 4,
                               cudaMemcpyDeviceToHost, ss.out));
  }
  FA2_CUDA(cudaStreamSynchronize(ss.out));
  FA2_CUDA(cudaStreamSynchronize(st));
  g_launches = launches;
  (void)lbytes;
  return FA2_OK;
}

}  // extern "C"
