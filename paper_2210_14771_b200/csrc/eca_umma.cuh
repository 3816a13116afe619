// tcgen05 helpers shared by the tensor-core kernels (eca_cnn.cu inference
// CNN, eca_train.cu training convs): 3xTF32 MMAs (hi*hi + hi*lo + lo*hi, FP32
// accumulators in TMEM) on K-major, no-swizzle shared-memory operands made
// of 8-row x 16-byte core matrices.
#pragma once

#include "eca_common.cuh"

namespace eca {

ECA_DEV float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// byte offset of (row, k) in a K-major no-swizzle operand with row-group stride sbo
ECA_DEV int kmaj_off(int row, int k, int sbo) {
  return (row >> 3) * sbo + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4;
}
ECA_DEV uint64_t umma_desc(uint32_t saddr, int sbo) {
  return uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (uint64_t(1) << 46);   // version 1, no swizzle
}
// kind::tf32, D F32, A/B TF32 K-major, M = 128
constexpr uint32_t idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}
ECA_DEV void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
// 3xTF32 product accumulated into tmem: hi*hi, hi*lo, lo*hi
ECA_DEV void mma3(uint32_t tmem, uint32_t a_hi, uint32_t a_lo, int sboa, uint32_t b_hi, uint32_t b_lo,
                  int sbob, uint32_t idesc, bool first) {
  mma_tf32(tmem, umma_desc(a_hi, sboa), umma_desc(b_hi, sbob), idesc, first ? 0u : 1u);
#ifndef ECA_EXPERIMENT_MMA1   // timing experiment only: wrong numerics
  mma_tf32(tmem, umma_desc(a_hi, sboa), umma_desc(b_lo, sbob), idesc, 1u);
  mma_tf32(tmem, umma_desc(a_lo, sboa), umma_desc(b_hi, sbob), idesc, 1u);
#endif
}
ECA_DEV void st_hilo(uint8_t* hi, uint8_t* lo, int off, float4 v) {
  float4 h, l;
  h.x = tf32_rna(v.x); l.x = tf32_rna(v.x - h.x);
  h.y = tf32_rna(v.y); l.y = tf32_rna(v.y - h.y);
  h.z = tf32_rna(v.z); l.z = tf32_rna(v.z - h.z);
  h.w = tf32_rna(v.w); l.w = tf32_rna(v.w - h.w);
  *reinterpret_cast<float4*>(hi + off) = h;
  *reinterpret_cast<float4*>(lo + off) = l;
}
template <int N>
ECA_DEV void tmem_ld(uint32_t addr, float* v);
template <>
ECA_DEV void tmem_ld<2>(uint32_t addr, float* v) {
  uint32_t r[2];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
  v[0] = __uint_as_float(r[0]);
  v[1] = __uint_as_float(r[1]);
}
template <>
ECA_DEV void tmem_ld<4>(uint32_t addr, float* v) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
#pragma unroll
  for (int i = 0; i < 4; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
ECA_DEV void tmem_ld<8>(uint32_t addr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(addr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
template <>
ECA_DEV void tmem_ld<16>(uint32_t addr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
ECA_DEV void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nECA_MW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra ECA_MW;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
// st.shared by all threads -> visible to the tensor core; all threads past the barrier
ECA_DEV void publish_operands() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

}  // namespace eca
