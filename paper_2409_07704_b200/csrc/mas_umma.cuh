// mas_umma.cuh -- the tcgen05 (5th-generation tensor core) pieces of the
// fused log-likelihood path (DESIGN.md 3 K4/K1g):
// TMEM allocation, tcgen05.st / tcgen05.ld, the shared-memory operand
// descriptor of a K-major, 128-byte-swizzled bf16 operand as TMA writes it,
// the instruction descriptor of a BF16 x BF16 -> FP32 MMA, the MMA with its
// A operand in TMEM, and the commit to an mbarrier.  sm_100a only.
//
// Operand shapes used here: D[128 rows x 64 columns] fp32 in TMEM (lane =
// row, column = speech frame), A[128 rows x K] bf16 in TMEM (lane = row, two
// bf16 per 32-bit column, element k in column k/2, even k in the low half),
// B[K x 64 columns] bf16 in shared memory, K-major (each column's K values
// contiguous) in 64-element (128-byte) swizzle atoms of 64 rows.  (N = 32
// measured 2x slower on the issue side: ~120 cycles per tcgen05.mma
// regardless of N at these sizes, r12.)
#pragma once

#include <cstdint>

namespace mas {
namespace umma {

constexpr int kM = 128;         // rows per MMA (TMEM lanes)
constexpr int kN = 64;          // columns (frames) per MMA: two K1 stages
constexpr int kStageN = 32;     // columns per K1 stage / TMEM load
constexpr int kKStep = 16;      // K per kind::f16 MMA
constexpr int kAtomK = 64;      // bf16 elements per 128-byte swizzle row
constexpr int kAtomBytes = kN * 128;  // one B atom: 64 columns x 128 bytes

// ---- instruction descriptor (kind::f16): BF16 A/B, FP32 D, both K-major ----
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4)                                  // D format: F32
         | (1u << 7)                                // A format: BF16
         | (1u << 10)                               // B format: BF16
         | (0u << 15) | (0u << 16)                  // A, B K-major
         | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

// ---- shared-memory descriptor: K-major, SWIZZLE_128B ----------------------
// start address >> 4 (bits 0-13), leading byte offset (ignored for swizzled
// K-major, 16 B) >> 4 (bits 16-29), stride byte offset = 8 rows x 128 B
// (bits 32-45), version 1 (bits 46-47, sm_100), base offset 0 (atoms are
// 1024-byte aligned), layout SWIZZLE_128B = 2 (bits 61-63).  Stepping K by
// 16 elements inside an atom adds 32 bytes to the start address.
__device__ __forceinline__ uint64_t sdesc_kmajor_sw128(uint32_t smem_byte_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_byte_addr >> 4) & 0x3fffu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// ---- TMEM allocation (one warp) -------------------------------------------
// `cols` a power of two >= 32.
__device__ __forceinline__ void tmem_alloc(uint32_t smem_slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_slot),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols)
               : "memory");
}
__host__ __device__ constexpr uint32_t tmem_cols_pow2(uint32_t n) {
  return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512;
}
__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- TMEM <-> registers (32 lanes x 32-bit, 8 / 32 columns) ----------------
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* u = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, "
      "%30, %31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
        "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
        "=r"(u[14]), "=r"(u[15]), "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]),
        "=r"(u[21]), "=r"(u[22]), "=r"(u[23]), "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]),
        "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- the MMA: D[tmem] (+)= A[tmem] . B[smem] ------------------------------
__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                       uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate ? 1u : 0u)
      : "memory");
}
// Arrives (once) on `bar` when every MMA this thread issued before has
// completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}

// D[128 x 64] = A[128 x Kp] . B[Kp x 64] for one tile: Kp / 16 MMAs, the
// B stage being Kp / 64 atoms of 64 columns x 128 bytes at `b_smem`.
// (mma_tiles interleaves the K steps of several tiles: consecutive MMAs then
// accumulate into different TMEM tiles instead of waiting on each other.)
__device__ __forceinline__ void mma_tile(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_smem, int Kp,
                                         uint32_t idesc) {
  for (int ks = 0; ks < Kp / kKStep; ++ks) {
    const uint32_t b_addr = b_smem + static_cast<uint32_t>((ks / 4) * kAtomBytes + (ks % 4) * 32);
    mma_ts(d_tmem, a_tmem + static_cast<uint32_t>(ks * (kKStep / 2)), sdesc_kmajor_sw128(b_addr),
           idesc, ks > 0);
  }
}

// `ntiles` tiles sharing B: D_t = A_t . B, tile t's D at d_tmem + t * d_step
// and A at a_tmem + t * a_step (TMEM columns), K steps interleaved.
__device__ __forceinline__ void mma_tiles(uint32_t d_tmem, uint32_t d_step, uint32_t a_tmem,
                                          uint32_t a_step, int ntiles, uint32_t b_smem, int Kp,
                                          uint32_t idesc, uint32_t atom_bytes = kAtomBytes) {
  for (int ks = 0; ks < Kp / kKStep; ++ks) {
    const uint64_t bd =
        sdesc_kmajor_sw128(b_smem + static_cast<uint32_t>(ks / 4) * atom_bytes + (ks % 4) * 32);
    for (int t = 0; t < ntiles; ++t)
      mma_ts(d_tmem + static_cast<uint32_t>(t) * d_step,
             a_tmem + static_cast<uint32_t>(t) * a_step + static_cast<uint32_t>(ks * (kKStep / 2)),
             bd, idesc, ks > 0);
  }
}

}  // namespace umma
}  // namespace mas
