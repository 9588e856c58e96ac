// mas_ptx.cuh -- thin inline-PTX wrappers for sm_100a: mbarrier, TMA
// (cp.async.bulk.tensor), cluster / DSMEM, release/acquire flags.
#pragma once
#include <cstdio>

#include <cuda.h>
#include <cstdint>

namespace mas {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
// Non-blocking probe of a phase (acquire on success); issued early, its
// result is consumed later, so the barrier latency overlaps other work.
__device__ __forceinline__ bool mbar_test_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Warp-uniform variants for warps that shuffle right after: every lane
// leaves with the same answer, so the warp stays converged (a lane that
// left a spin loop alone would push every later SHFL onto the divergent
// WARPSYNC path).
__device__ __forceinline__ bool mbar_test_wait_all(uint32_t bar, uint32_t parity) {
  return __all_sync(0xffffffffu, mbar_test_wait(bar, parity));
}
__device__ __forceinline__ void mbar_wait_all(uint32_t bar, uint32_t parity) {
  while (!__all_sync(0xffffffffu, mbar_try_wait(bar, parity))) {
  }
}
// mbar_wait_all unless `skip` (warp-uniform: a vote result or a
// warp-invariant flag), as ONE asm block: the compiler sees no branch, so
// the hot loop carries no convergence barrier (BSSY/BSYNC) around the
// rarely taken wait.
__device__ __forceinline__ void mbar_wait_all_unless(bool skip, uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p, s;\n\t"
      "setp.ne.b32 s, %2, 0;\n\t"
      "@s bra.uni MAS_WAIT_DONE;\n\t"
      "MAS_WAIT_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "vote.sync.all.pred p, p, 0xffffffff;\n\t"
      "@!p bra.uni MAS_WAIT_LOOP;\n\t"
      "MAS_WAIT_DONE:\n\t}" ::"r"(bar),
      "r"(parity), "r"(static_cast<int>(skip))
      : "memory");
}

// Predicated forms (one guarded instruction instead of a branch around it:
// the per-quad bookkeeping otherwise costs BSSY/ISETP/BRA per operation).
__device__ __forceinline__ void mbar_arrive_expect_tx_if(bool c, uint32_t bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(bar),
      "r"(bytes), "r"(static_cast<int>(c))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_local_if(bool c, uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %1, 0;\n\t"
      "@p mbarrier.arrive.shared::cta.b64 _, [%0];\n\t}" ::"r"(bar),
      "r"(static_cast<int>(c))
      : "memory");
}

// ---- TMA ------------------------------------------------------------------
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_unchanged() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// 2-D tile load global -> shared (this CTA), completion on `bar`, L2 hint.
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}
// 2-D tile store shared -> global (bulk-group completion), no L2 hint.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// 4-D tile store shared -> global (bulk-group completion).
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// Wait until every bulk store of this thread has been performed.
__device__ __forceinline__ void bulk_store_complete() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// Wait until every bulk store of this thread has finished reading shared
// memory (the CTA may not exit before that).
__device__ __forceinline__ void bulk_store_drain() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// TMA L2 prefetch of one box (no shared-memory destination).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int c0, int c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---- cluster / DSMEM ------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n\t"
      "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void st_cluster_v4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}
// Asynchronous 16-byte store into a (possibly remote) CTA's shared memory
// that completes 16 bytes of transaction count on that CTA's mbarrier --
// the boundary-row FIFO's data path (SASS: STAS.128).
__device__ __forceinline__ void st_async_v4(uint32_t addr, float a, float b, float c, float d,
                                            uint32_t remote_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(addr),
      "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(c)),
      "r"(__float_as_uint(d)), "r"(remote_bar)
      : "memory");
}
__device__ __forceinline__ void st_async_v4_if(bool c, uint32_t addr, float a, float b, float d0,
                                               float d1, uint32_t remote_bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
      "@p st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n\t}" ::"r"(addr),
      "r"(__float_as_uint(a)), "r"(__float_as_uint(b)), "r"(__float_as_uint(d0)),
      "r"(__float_as_uint(d1)), "r"(remote_bar), "r"(static_cast<int>(c))
      : "memory");
}
__device__ __forceinline__ void st_async_b32_if(bool c, uint32_t addr, uint32_t v,
                                                uint32_t remote_bar) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\t"
      "@p st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n\t}" ::"r"(addr),
      "r"(v), "r"(remote_bar), "r"(static_cast<int>(c))
      : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t addr, uint32_t v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                   addr),
               "r"(v), "r"(remote_bar)
               : "memory");
}
// Relaxed arrive on a (possibly remote) mbarrier: no membar is emitted
// (a .release.cluster arrive costs MEMBAR.ALL.GPU).  Callers issue it only
// after every value read from the released buffer has been consumed.
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}

// ---- misc -----------------------------------------------------------------
// a > b as an all-ones / zero mask (FSET), so a bit can be merged into a
// word with a single LOP3.
__device__ __forceinline__ uint32_t gt_mask(float a, float b) {
  uint32_t d;
  asm("set.gt.u32.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b));
  return d;
}
// if (a > b) w += (1 << BIT), as a predicated IMAD so the bit packing runs on
// the FMA pipe (the ALU pipe is the DP's bottleneck: FMNMX + FSETP).  `one`
// must be an opaque register holding 1 (else ptxas turns it into IADD3).
template <int BIT>
__device__ __forceinline__ void set_bit_if_gt(uint32_t& w, float a, float b, uint32_t one) {
  asm("{\n\t.reg .pred q;\n\tsetp.gt.f32 q, %1, %2;\n\t@q mad.lo.u32 %0, %3, %4, %0;\n\t}"
      : "+r"(w)
      : "f"(a), "f"(b), "r"(one), "n"(1u << BIT));
}
// acc = q * zero + acc on the FMA pipe (`zero` an opaque 0.0f): acc turns
// NaN as soon as a folded q is inf or NaN (inf * 0 = NaN).
__device__ __forceinline__ void fold_nonfinite(float& acc, float q, float zero) {
  asm("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc) : "f"(q), "f"(zero));
}
// max.NaN over |a|, |b| folded into acc: acc turns NaN / +inf as soon as any
// folded value is non-finite (one FMNMX3.NAN per two values on sm_100a).
__device__ __forceinline__ void fold_abs_max_nan(float& acc, float a, float b) {
  asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(acc) : "f"(fabsf(a)), "f"(fabsf(b)));
}

__device__ __forceinline__ void st_global_v2_evict_last(uint32_t* p, uint32_t a, uint32_t b,
                                                        uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(a), "r"(b),
               "l"(pol)
               : "memory");
}

}  // namespace mas
