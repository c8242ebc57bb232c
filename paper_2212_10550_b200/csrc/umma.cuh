// umma.cuh -- hand-written tcgen05 (5th-gen tensor core) helpers for sm_100a: canonical
// no-swizzle K-major operand layout in shared memory, smem matrix descriptors, the kind::f16
// instruction descriptor, split-bf16 MMAs (x = hi + lo; hi*hi + hi*lo + lo*hi with f32
// accumulation in TMEM), commit / mbarrier waits, TMEM loads. Used by the tcgen05 render
// decoder (field_tc.cu) and the tcgen05 training backward (train_tc.cu).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace arfx {
namespace umma {

// K-major, no-swizzle canonical layout (cute "INTERLEAVE"): element (r, k) of an R x K bf16
// operand at byte (k/8)*(R*16) + (r/8)*128 + (r%8)*16 + (k%8)*2 = (k/8)*(R*16) + r*16 + (k%8)*2.
// Core matrices are 8 rows x 16 B; LBO (next 16-B K chunk) = R*16, SBO (next 8 rows) = 128.
__device__ __forceinline__ int kmaj_off(int r, int k, int R) { return (k >> 3) * (R * 16) + r * 16 + (k & 7) * 2; }

__device__ __forceinline__ void split_bf16(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;  // descriptor version for sm_100
  return d;         // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// D (+)= sum over K-steps of Ahi*Bhi + Ahi*Blo + Alo*Bhi; operand planes: hi at off, lo at
// off + plane bytes. K per MMA = 16 (two 16-byte chunks).
// acc_in: accumulate onto D's current contents from the first MMA on (else overwrite).
__device__ __forceinline__ void mma_split(uint32_t tmem_d, uint32_t a_hi, uint32_t a_plane, int a_rows,
                                          uint32_t b_hi, uint32_t b_plane, int b_rows, int K, uint32_t idesc,
                                          bool acc_in = false) {
  for (int ks = 0; ks < K / 16; ++ks) {
    const uint32_t ao = a_hi + ks * 2 * (a_rows * 16), bo = b_hi + ks * 2 * (b_rows * 16);
    const uint64_t ah = smem_desc(ao, a_rows * 16, 128), al = smem_desc(ao + a_plane, a_rows * 16, 128);
    const uint64_t bh = smem_desc(bo, b_rows * 16, 128), bl = smem_desc(bo + b_plane, b_rows * 16, 128);
    mma_bf16(tmem_d, ah, bh, idesc, (ks > 0 || acc_in) ? 1u : 0u);
    mma_bf16(tmem_d, ah, bl, idesc, 1u);
    mma_bf16(tmem_d, al, bh, idesc, 1u);
  }
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// A from tensor memory (".kind::f16 [d], [a], b_desc"): the A operand is M rows x K bf16 in
// TMEM, row m in lane m, two consecutive K elements packed per 32-bit column (element 2c in
// the low half) -- K = 16 per MMA = 8 columns.
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t idesc,
                                            uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(idesc), "r"(acc));
}

// split-bf16 product with A (hi plane at column a_hi, lo plane at a_lo) in TMEM, B in smem
__device__ __forceinline__ void mma_split_ts(uint32_t tmem_d, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                             uint32_t b_plane, int b_rows, int K, uint32_t idesc) {
  for (int ks = 0; ks < K / 16; ++ks) {
    const uint32_t bo = b_hi + ks * 2 * (b_rows * 16);
    const uint64_t bh = smem_desc(bo, b_rows * 16, 128), bl = smem_desc(bo + b_plane, b_rows * 16, 128);
    mma_bf16_ts(tmem_d, a_hi + 8 * ks, bh, idesc, ks > 0 ? 1u : 0u);
    mma_bf16_ts(tmem_d, a_hi + 8 * ks, bl, idesc, 1u);
    mma_bf16_ts(tmem_d, a_lo + 8 * ks, bh, idesc, 1u);
  }
}

// 8 consecutive 32-bit TMEM columns of this thread's lane (caller waits with tmem_st_wait)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

}  // namespace umma
}  // namespace arfx
