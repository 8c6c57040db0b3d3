/*
 * fa2.h — C ABI of the B200 (sm_100a) FlashAttention-2 hot path.
 *
 * The operation (PAPER.md = /root/reference/PAPER.md, cited P:<line>):
 *   For every batch b < B and head h < H (computed independently),
 *   with Q, K, V in R^{N x d}:
 *     S = softmax_scale * Q K^T   (scale per footnote P:160-162)
 *     causal: S_ij = -inf for j > i, top-left aligned, N_q = N_k
 *     P = rowwise softmax(S), O = P V
 *     L_i = m_i + log(l_i) = log sum_j exp(S_ij)  (natural log)
 *   Backward (Alg. 2):
 *     D_i = rowsum(dO o O)_i
 *     P_ij = exp(S_ij - L_i)
 *     dV = P^T dO, dP = dO V^T, dS = P o (dP - D_i)
 *     dQ = softmax_scale * dS K,  dK = softmax_scale * dS^T Q
 *
 * Layout: q, k, v, o, dout, dq, dk, dv are DEVICE pointers to contiguous
 *   row-major [B, H, N, d] tensors of `dtype` (each head's N x d matrix is
 *   contiguous).  lse is a DEVICE pointer to [B, H, N] float32.
 * Alignment: every tensor pointer must be 16-byte aligned (TMA).
 * Supported: d in {64, 128}; dtype FA2_BF16 or FA2_FP16; N >= 1 (any N, ragged
 *   tails are masked); B, H >= 1; B*H <= 2^31-1; softmax_scale finite and > 0.
 * Ownership: the caller owns every buffer; the library never allocates device
 *   memory.  Inputs are read-only.  o and lse written by fa2_forward are inputs
 *   of fa2_backward and must not be modified in between.
 * Streams: `stream` is a cudaStream_t (0 = legacy default stream).  Calls are
 *   asynchronous with respect to the host; no host synchronisation happens
 *   inside the device-pointer entry points.  Host-side state: a per-thread
 *   error-detail string, launch count and timing/trace hooks; per-device caches
 *   (co-resident cluster counts) and a shape-keyed cache of the balanced causal
 *   schedules, both mutex-guarded and immutable once published (schedules are
 *   shared_ptr-owned, so eviction never frees one in use); the copy/compute
 *   streams of fa2_attention_step_host are per thread and per device.  No device
 *   memory is allocated and no device-side state persists between calls, so
 *   calls are reentrant and may run concurrently on different streams.
 * Errors: argument errors are detected before anything is launched and are
 *   returned synchronously (nothing is launched).  Launch failures return
 *   FA2_ERR_CUDA; fa2_last_error_detail() describes the last failure of the
 *   calling thread.  Asynchronous kernel faults surface at the caller's next
 *   synchronisation, as with any CUDA library.
 */
#ifndef FA2_H_
#define FA2_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FA2_API __attribute__((visibility("default")))
#else
#define FA2_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { FA2_BF16 = 0, FA2_FP16 = 1 } fa2_dtype_t;

typedef enum {
  FA2_OK = 0,
  FA2_ERR_INVALID_ARG = 1, /* null pointer, B/H/N < 1, scale not finite or <= 0, misaligned pointer */
  FA2_ERR_UNSUPPORTED = 2, /* d not in {64,128}, dtype unknown, device is not sm_100 */
  FA2_ERR_WORKSPACE = 3,   /* workspace null or smaller than fa2_backward_workspace_size() */
  FA2_ERR_CUDA = 4         /* CUDA runtime/driver error; see fa2_last_error_detail() */
} fa2_status_t;

/* Forward pass, Alg. 1.  Writes o [B,H,N,d] (dtype) and lse [B,H,N]
 * (fp32, natural log of the scaled logits). */
FA2_API fa2_status_t fa2_forward(const void* q, const void* k, const void* v, void* o, float* lse,
                         int B, int H, int N, int d, int causal, float softmax_scale,
                         fa2_dtype_t dtype, void* stream);

/* Bytes of device scratch fa2_backward needs: the fp32 dQ accumulator
 * [B,H,N_pad,d], D [B,H,N_pad] and L*log2(e) [B,H,N_pad] (fp32), where N_pad is
 * N rounded up to a multiple of 128, plus [B,H,N_pad/32] int32 dQ-tile
 * counters (4 per 128-row tile, used by fa2_backward_deterministic), rounded up
 * to 16 bytes -- the
 * minimum -- plus, 256-byte aligned, 2*B*H*N*d fp32 for the GQA load-balance
 * split (fp32 dK, dV partial sums when the query heads of a key/value group are
 * spread over several CTAs; used only when H_kv < H, not deterministic, and the
 * caller's workspace has the room). */
FA2_API size_t fa2_backward_workspace_size(int B, int H, int N, int d);

/* Backward pass, Alg. 2: writes dq, dk, dv ([B,H,N,d], dtype).
 * `workspace` is caller-owned device memory of at least
 * fa2_backward_workspace_size(B,H,N,d) bytes, 16-byte aligned; its contents on
 * entry are ignored (the library zeroes what it uses). */
FA2_API fa2_status_t fa2_backward(const void* q, const void* k, const void* v, const void* o,
                          const float* lse, const void* dout, void* dq, void* dk, void* dv,
                          void* workspace, size_t workspace_bytes,
                          int B, int H, int N, int d, int causal, float softmax_scale,
                          fa2_dtype_t dtype, void* stream);

/* Multi-query / grouped-query attention: q, o, dout, dq are
 * [B,H,N,d]; k, v, dk, dv are [B,H_kv,N,d] with H a multiple of H_kv.  Query
 * head h attends with key/value head h / (H/H_kv) ("implicitly manipulate the
 * indices into the head"); dk, dv are the sums over the H/H_kv query heads of
 * each group (computed inside one work tile, no atomics).  H_kv == H is
 * exactly fa2_forward / fa2_backward.  Workspace: fa2_backward_workspace_size(B,H,N,d). */
FA2_API fa2_status_t fa2_forward_gqa(const void* q, const void* k, const void* v, void* o, float* lse,
                                     int B, int H, int H_kv, int N, int d, int causal, float softmax_scale,
                                     fa2_dtype_t dtype, void* stream);
FA2_API fa2_status_t fa2_backward_gqa(const void* q, const void* k, const void* v, const void* o,
                                      const float* lse, const void* dout, void* dq, void* dk, void* dv,
                                      void* workspace, size_t workspace_bytes,
                                      int B, int H, int H_kv, int N, int d, int causal, float softmax_scale,
                                      fa2_dtype_t dtype, void* stream);

/* General fixed-length attention: q, o [B,H,N_q,d]; k, v
 * [B,H_kv,N_k,d]; lse [B,H,N_q].  N_q may differ from N_k.  The paper defines the
 * causal mask only for N_q == N_k; here it is aligned to the
 * bottom-right corner: query row i sees key j iff j <= i + (N_k - N_q)
 * (R22), which is the paper's mask when N_q == N_k.  A row that sees no
 * key (causal with N_q > N_k) gets O = 0 and lse = -inf (R23).  fa2_forward and
 * fa2_forward_gqa are the special cases N_q == N_k.  Errors as fa2_forward_gqa,
 * plus FA2_ERR_INVALID_ARG for N_k < 1. */
FA2_API fa2_status_t fa2_forward_ex(const void* q, const void* k, const void* v, void* o, float* lse,
                                    int B, int H, int H_kv, int N_q, int N_k, int d, int causal,
                                    float softmax_scale, fa2_dtype_t dtype, void* stream);

/* Variable-length batch in the packed layout: sequence b is rows
 * [cu_seqlens_q[b], cu_seqlens_q[b+1]) of q, o ([total_q, H, d], contiguous) and
 * rows [cu_seqlens_k[b], cu_seqlens_k[b+1]) of k, v ([total_k, H_kv, d]); lse is
 * [H, total_q] fp32.  cu_seqlens_q / cu_seqlens_k are DEVICE int32 arrays of
 * B+1 entries, non-decreasing, starting at 0 and ending at total_q / total_k
 * (not validated on the host: that would need a device sync; a violation gives
 * undefined results).  max_seqlen_q / _k must be >= every sequence's length
 * (they size the tile grid; rows past max_seqlen_q are not computed).  Empty
 * sequences are allowed.  Masking per sequence as fa2_forward_ex (R22, R23).
 * Errors: FA2_ERR_INVALID_ARG for NULL / misaligned pointers, B, H < 1, H not
 * a multiple of H_kv, total_q or total_k < 1, max_seqlen outside [1, total];
 * FA2_ERR_UNSUPPORTED as fa2_forward. */
FA2_API fa2_status_t fa2_forward_varlen(const void* q, const void* k, const void* v, void* o, float* lse,
                                        const int* cu_seqlens_q, const int* cu_seqlens_k, int B, int H, int H_kv,
                                        int total_q, int total_k, int max_seqlen_q, int max_seqlen_k, int d,
                                        int causal, float softmax_scale, fa2_dtype_t dtype, void* stream);

/* FP8 forward (the paper lists FP8 as future work).
 * q [B,H,N,d], k, v [B,H_kv,N,d] are float8 E4M3 (1 byte per element, the same
 * contiguous layouts as fa2_forward_gqa); the represented values are
 * descale_q * q, descale_k * k, descale_v * v (per-tensor fp32 factors, finite
 * and > 0).  Computes the same O and lse as fa2_forward_gqa on those values:
 * S = softmax_scale * (descale_q q)(descale_k k)^T is accumulated exactly in fp32
 * (E4M3 products are exact), the online softmax runs in fp32, and P~ is rounded
 * to E4M3 for the P~V product (R25: relative error <= 2^-4 per P~
 * entry); l sums the fp32 P~.  o is written as bf16 [B,H,N,d], lse fp32
 * [B,H,N].  d = 128 only (FA2_ERR_UNSUPPORTED otherwise).  There is no FP8
 * backward. */
FA2_API fa2_status_t fa2_forward_fp8(const void* q, const void* k, const void* v, void* o, float* lse,
                                     int B, int H, int H_kv, int N, int d, int causal, float softmax_scale,
                                     float descale_q, float descale_k, float descale_v, void* stream);

/* Deterministic backward.  Same arguments, layouts, workspace and
 * errors as fa2_backward_gqa (H_kv == H for plain multi-head attention); the
 * result is bitwise reproducible from run to run on the same device and
 * arguments.  Alg. 2 accumulates dQ_i += dS_ij K_j into HBM from every key block
 * j with atomic adds, so the fp32 summation order -- and
 * the last bits of dQ -- follow arrival order.  Here every dQ tile (query head,
 * 128-row query tile; in the CTA-pair d = 128 kernel each query half and d half
 * of it) takes its key blocks' contributions in one fixed order, serialised by
 * counters in the workspace; the arithmetic is otherwise
 * identical (dK, dV are accumulated on chip in a fixed order in both modes).
 * Slower than fa2_backward_gqa by the waits on those counters. */
FA2_API fa2_status_t fa2_backward_deterministic(const void* q, const void* k, const void* v, const void* o,
                                                const float* lse, const void* dout, void* dq, void* dk, void* dv,
                                                void* workspace, size_t workspace_bytes,
                                                int B, int H, int H_kv, int N, int d, int causal,
                                                float softmax_scale, fa2_dtype_t dtype, void* stream);

/* Backward of fa2_forward_ex (N_q may differ from N_k; causal bottom-right
 * aligned, R22; rows that saw no key contribute nothing, R23): q, o, dout, dq
 * [B,H,N_q,d]; k, v, dk, dv [B,H_kv,N_k,d]; lse [B,H,N_q] as fa2_forward_ex wrote
 * it.  Workspace: fa2_backward_workspace_size(B, H, N_q, d) bytes.
 * deterministic != 0 gives the fixed dQ summation order of
 * fa2_backward_deterministic.  Errors as fa2_backward_gqa, plus
 * FA2_ERR_INVALID_ARG for N_k < 1. */
FA2_API fa2_status_t fa2_backward_ex(const void* q, const void* k, const void* v, const void* o,
                                     const float* lse, const void* dout, void* dq, void* dk, void* dv,
                                     void* workspace, size_t workspace_bytes,
                                     int B, int H, int H_kv, int N_q, int N_k, int d, int causal,
                                     float softmax_scale, int deterministic, fa2_dtype_t dtype, void* stream);

/* Bytes of device scratch fa2_backward_varlen needs for B sequences with total_q
 * query rows: the same buffers as fa2_backward_workspace_size over padded query
 * rows (every sequence padded to a multiple of 128 rows; at most
 * H * (total_q + 127 B) rounded up to 128), plus [B+1] int32 tile offsets. */
FA2_API size_t fa2_backward_varlen_workspace_size(int B, int H, int total_q, int d);

/* Backward of fa2_forward_varlen (packed layout, same arguments and layouts;
 * dq [total_q, H, d], dk, dv [total_k, H_kv, d]).  Key rows of a sequence with
 * no query row get dK = dV = 0.  deterministic != 0: fixed dQ summation order.
 * Workspace: fa2_backward_varlen_workspace_size(B, H, total_q, d).  Errors as
 * fa2_forward_varlen plus FA2_ERR_WORKSPACE. */
FA2_API fa2_status_t fa2_backward_varlen(const void* q, const void* k, const void* v, const void* o,
                                         const float* lse, const void* dout, void* dq, void* dk, void* dv,
                                         const int* cu_seqlens_q, const int* cu_seqlens_k,
                                         void* workspace, size_t workspace_bytes, int B, int H, int H_kv,
                                         int total_q, int total_k, int max_seqlen_q, int max_seqlen_k, int d,
                                         int causal, float softmax_scale, int deterministic, fa2_dtype_t dtype,
                                         void* stream);

/* D = rowsum(dO o O) alone, into d_out [B,H,N] fp32 (device).  Exposed
 * so the preprocessing step can be checked on its own; fa2_backward runs it
 * internally. */
FA2_API fa2_status_t fa2_backward_preprocess(const void* o, const void* dout, float* d_out,
                                     int B, int H, int N, int d, fa2_dtype_t dtype, void* stream);

/* End-to-end step through HOST buffers: copies q,k,v,dout (pinned host memory
 * recommended) to the device arena, runs fa2_forward then fa2_backward, and
 * copies o, lse, dq, dk, dv back to host; returns after all of it completed.
 * The (b, h) units are independent, so the step is pipelined over up
 * to 8 chunks of units: chunk c's inputs are copied in on an internal stream
 * while chunk c-1 computes on `stream` and chunk c-2's results are copied out on
 * another internal stream (ordered after the caller's prior work on `stream`).
 * `arena` is caller-owned device memory of at least fa2_step_arena_size(B,H,N,d)
 * bytes.  Host output pointers may be NULL to skip that copy. */
FA2_API size_t fa2_step_arena_size(int B, int H, int N, int d);
FA2_API fa2_status_t fa2_attention_step_host(const void* q_h, const void* k_h, const void* v_h, const void* dout_h,
                                     void* o_h, float* lse_h, void* dq_h, void* dk_h, void* dv_h,
                                     void* arena, size_t arena_bytes,
                                     int B, int H, int N, int d, int causal, float softmax_scale,
                                     fa2_dtype_t dtype, void* stream);

/* Host-side tile map (no GPU needed), the grid logic of P:345-351, P:378-386:
 * for query row block `i` of size Br, the number of key/value blocks of size Bc
 * that are computed (n_blocks) and the first block index that needs the causal
 * or ragged mask (first_masked; == n_blocks when none).  Returns FA2_OK or
 * FA2_ERR_INVALID_ARG. */
FA2_API fa2_status_t fa2_kv_block_range(int N, int Br, int Bc, int i, int causal, int* n_blocks, int* first_masked);

/* Host-side balanced tile schedule (no GPU needed) that the causal square-length
 * one-SM forward (`pass` = 0) and arrival-order backward (`pass` = 1) launches (d = 64)
 * pass to their kernels; the d = 128 CTA-pair kernels use per-pair lists built by the same
 * greedy assignment over 512-row / 256-key-row pair tiles (the row-block loops of Alg. 1/2, P:345-351,
 * P:421-436, with the causal skip of P:378-386 making tiles unequal).
 *   heads: B * H query heads (forward) or B * H_kv * hsplit work heads (backward)
 *   N: sequence length; heads_per_tile: query heads one backward tile visits
 *   (H / H_kv / hsplit; 1 for MHA; ignored by the forward); grid: CTAs (<= 160).
 * Tiles are numbered as the kernels decode them (forward: head * ceil(N/256) + r,
 * row block ceil(N/256)-1-r; backward: head * ceil(N/128) + key block).  On
 * success CTA c runs order[start[c] .. start[c+1]) and *n_tiles is the tile count;
 * `order` holds `capacity` entries (>= tiles), `start` grid + 1.  Returns
 * FA2_ERR_INVALID_ARG for bad sizes or more than 8192 tiles (the kernels then
 * use the stride schedule).  Caller owns both arrays; nothing is allocated. */
FA2_API fa2_status_t fa2_tile_schedule(int pass, int heads, int N, int heads_per_tile, int grid, unsigned short* order,
                                       unsigned short* start, int capacity, int* n_tiles);

/* Optional benchmark timing hook (per calling thread).  `events` points to 6
 * cudaEvent_t created by the caller (or is NULL to disable).  While set,
 * fa2_forward records events[0] / events[1] on `stream` immediately before /
 * after its kernel, and fa2_backward records events[2] before the D
 * preprocessing kernel, events[3] before the main backward kernel, events[4]
 * after it and events[5] after the dQ conversion kernel.  The array must stay
 * valid until the calls that use it have been issued. */
FA2_API void fa2_set_timing_events(void* const* events);

/* Debug only: when `dev_buf` (device memory, >= 16384 x uint64) is non-NULL,
 * the calling thread's fa2_forward launches record clock64() timestamps of the
 * first work tile of CTA 0 into it (layout documented in fa2_fwd_sm100.cuh). */
FA2_API void fa2_debug_set_trace(void* dev_buf);

FA2_API const char* fa2_status_string(fa2_status_t s);
FA2_API const char* fa2_last_error_detail(void);
/* Number of kernels the last successful fa2_forward / fa2_backward call launched. */
FA2_API int fa2_last_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FA2_H_ */
