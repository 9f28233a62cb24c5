// rfr_tcgen05.cuh -- the tcgen05 (5th-generation tensor core) building blocks shared by the
// tensor-core kernels of librfr: shared-memory matrix descriptors (K-major, SWIZZLE_NONE canonical
// layout), the fp16 hi / lo split of the "3xFP16" scheme, TMEM loads / stores of 16 columns, the
// tcgen05 fences and one kind::f16 MMA with A in tensor memory.  Inline PTX for sm_100a.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace rfr {
namespace {

// shared-memory matrix descriptor: K-major, SWIZZLE_NONE canonical layout, Blackwell version 1
__device__ __forceinline__ uint64_t umma_sdesc(unsigned saddr, unsigned lbo, unsigned sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// two floats -> f16x2, `lo_elem` in bits 0..15 (the even K element of an A column)
__device__ __forceinline__ unsigned pack_h2(float lo_elem, float hi_elem) {
  unsigned r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi_elem), "f"(lo_elem));
  return r;
}

// hi part of the 3-term split: x with the 13 low mantissa bits cleared (one LOP3).  It has 11
// significant bits, so it is exact in fp16 for |x| >= 2^-14 (below that the fp16 conversion
// leaves an absolute error < 2^-25 of the row scale); lo = x - hi is exact in fp32.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ void tmem_st16(unsigned addr, const unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};" ::"r"(addr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(unsigned addr, unsigned (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[tmem] . B[smem]^T, one K step of 16 fp16 columns (8 TMEM columns of A)
__device__ __forceinline__ void umma_f16_ts(unsigned d_tmem, unsigned a_tmem, uint64_t b_desc,
                                            unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred pa;\n setp.ne.b32 pa, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, pa;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate));
}

}  // namespace
}  // namespace rfr
