// CTA-pair (cluster of 2, tcgen05 cta_group::2) building blocks shared by the pair
// forward (fa2_fwd2_sm100.cuh) and the pair backward (fa2_bwd2_sm100.cuh): cluster
// ids, remote mbarrier arrivals and shared-memory stores (mapa), multicast
// tcgen05.commit, the cta_group::2 MMAs and the pair TMA load whose completion
// bytes land on the leader CTA's mbarrier.
#pragma once
#include "fa2_seq.cuh"

namespace fa2 {

namespace pair {

FA2_DEVICE uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
FA2_DEVICE uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
FA2_DEVICE uint32_t num_clusters() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
FA2_DEVICE void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// arrive on the mbarrier at the same shared-memory offset in CTA `cta` of the cluster
FA2_DEVICE void arrive_remote(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}"
      :: "r"(ptx::smem_u32(bar)), "r"(cta) : "memory");
}
// wait on a local mbarrier whose arrivals come from the whole cluster
FA2_DEVICE void wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  }
}
// arrive (once) on `bar` in both CTAs of the pair when this thread's tcgen05 ops complete
FA2_DEVICE void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
      :: "r"(ptx::smem_u32(bar)), "h"(static_cast<uint16_t>(0x3)) : "memory");
}
FA2_DEVICE void mma_ss2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
      :: "r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
// TMA 3-D load into this CTA's SMEM whose completion bytes land on the leader's mbarrier
// at the same offset (peer bit of the shared::cluster address cleared)
FA2_DEVICE void tma_load_pair(void* smem_dst, const CUtensorMap* d, uint64_t* bar, int c0, int c1, int c2,
                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      :: "r"(ptx::smem_u32(smem_dst)), "l"(reinterpret_cast<uint64_t>(d)), "r"(c0), "r"(c1), "r"(c2),
         "r"(ptx::smem_u32(bar) & 0xFEFFFFFFu), "l"(policy)
      : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem desc], cta_group::2: each CTA's TMEM holds its M/2 rows of A
FA2_DEVICE void mma_ts2(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
      :: "r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate) : "memory");
}
// shared::cluster address of `local` (a shared::cta address) in CTA `cta` of the cluster
FA2_DEVICE uint32_t map_cta(uint32_t local, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
  return r;
}
FA2_DEVICE void st_cluster_v4(uint32_t cluster_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared::cluster.v4.b32 [%0], {%1, %2, %3, %4};" :: "r"(cluster_addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
// generic-proxy shared-memory writes of this thread (local or remote) -> visible to the async proxy
FA2_DEVICE void fence_proxy_async_cluster() { asm volatile("fence.proxy.async.shared::cluster;" ::: "memory"); }
// release at cluster scope: orders this thread's prior (remote) shared-memory writes before the arrival
FA2_DEVICE void arrive_remote_release(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}"
      :: "r"(ptx::smem_u32(bar)), "r"(cta) : "memory");
}
FA2_DEVICE void wait_cluster_acquire(uint64_t* bar, uint32_t parity) {
  const uint32_t a = ptx::smem_u32(bar);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(a), "r"(parity) : "memory");
  }
}
// Bulk copy of `bytes` (multiple of 16) from this CTA's shared memory to the shared memory of
// another CTA of the cluster (DSMEM, async proxy); completion bytes land on the mbarrier
// `remote_bar` (a shared::cluster address in the destination CTA).
FA2_DEVICE void bulk_copy_to_cta(uint32_t remote_dst, const void* src, uint32_t bytes, uint32_t remote_bar) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(remote_dst), "r"(ptx::smem_u32(src)), "r"(bytes), "r"(remote_bar) : "memory");
}
// Asynchronous 16-byte store into another CTA's shared memory (DSMEM) whose completion bytes
// land on that CTA's mbarrier `remote_bar` (both shared::cluster addresses of the destination).
FA2_DEVICE void st_async_v4(uint32_t remote_addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];"
               :: "r"(remote_addr), "r"(a), "r"(b), "r"(c), "r"(d), "r"(remote_bar) : "memory");
}
// n-th work tile of this CTA pair (-1: none left): balanced table indexed by the pair,
// else the static stride schedule over pairs
template <class S>
FA2_DEVICE int sched_tile_pair(const S& sc, int n, int num_tiles, int pid, int npairs) {
  if constexpr (std::is_same<S, TileSched>::value) {
    if (sc.n > 0) {
      const int i = sc.start[pid] + n;
      return i < sc.start[pid + 1] ? sc.order[i] : -1;
    }
  }
  const int t = pid + n * npairs;
  return t < num_tiles ? t : -1;
}

}  // namespace pair

}  // namespace fa2
