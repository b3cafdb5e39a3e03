// tc.cuh — tcgen05 (5th-generation tensor core) + TMEM + tensor-TMA wrappers
// for sm_100a, written as inline PTX (no CUTLASS).
//
// Operand layout used by the kernels of this library: K-major tiles with the
// 128-byte swizzle, i.e. 8-row x 128-byte atoms (1024 B, 1024-aligned), rows
// at 128 B inside an atom, consecutive 8-row groups `sbo` bytes apart.  The
// MMA reads A (M x K) and B (N x K) from shared memory and accumulates f32 in
// tensor memory; one elected thread issues, tcgen05.commit signals mbarriers.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace chess {
namespace tc {

// Shared-memory matrix descriptor (tcgen05 "smem descriptor"):
//   [0,14)  start address >> 4        [16,30) leading byte offset >> 4
//   [32,46) stride byte offset >> 4   [46,48) version (1 on sm_100)
//   [49,52) base offset (0: atoms 1024-aligned)   [61,64) layout (2 = SWIZZLE_128B)
// For swizzled K-major operands the leading offset is unused (1 by convention);
// the stride offset is the distance between 8-row groups.  Advancing K by 16
// half-precision elements inside an atom adds 32 B to the start address.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t smem_addr, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3fffu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)2u << 61;
  return d;
}

// Instruction descriptor of kind::f16: D f32, A/B f16 (fmt 0) or bf16 (fmt 1),
// both K-major, M x N.
//   [4,6) c_format (1 = F32)  [7,10) a_format  [10,13) b_format
//   [15] a_major  [16] b_major  [17,23) N >> 3  [24,29) M >> 4
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int ab_fmt) {
  return (1u << 4) | ((uint32_t)ab_fmt << 7) | ((uint32_t)ab_fmt << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// General shared-memory descriptor: layout 2 = SWIZZLE_128B, 0 = no swizzle
// ("interleave": 8 x 16-byte core matrices).  K-major SW128: lbo unused,
// sbo = 8-row group stride.  MN-major SW128: lbo = stride between 64-element
// MN blocks, sbo = 8-row K group stride.  MN-major no-swizzle: 8 MN elements
// contiguous (16 B), K rows 16 B apart, lbo = stride between 8-row K groups.
// (Verified on B200 by tools/tc_attn_probe.cu.)
__device__ __forceinline__ uint64_t smem_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3fffu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3fffu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3fffu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// kind::f16 instruction descriptor with operand majors (0 = K-major, 1 = MN-major)
__host__ __device__ constexpr uint32_t idesc_f16_major(int M, int N, int ab_fmt, int a_mn, int b_mn) {
  return idesc_f16(M, N, ab_fmt) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16);
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread for the CTA.
__device__ __forceinline__ void mma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive (once) on an mbarrier when every tcgen05.mma issued so far by this
// thread has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// TMEM allocation: one full warp, power-of-two columns >= 32; the base
// address lands in shared memory.
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(smem_dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// Two consecutive f32 columns of this thread's TMEM lane (warp w reads lanes
// 32*(w%4) .. +31; taddr = base + ((32*(w%4)) << 16) + column).
__device__ __forceinline__ void tmem_ld_x2(uint32_t taddr, float& c0, float& c1) {
  uint32_t r0, r1;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr) : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  c0 = __uint_as_float(r0);
  c1 = __uint_as_float(r1);
}

// Eight consecutive f32 columns of this thread's TMEM lane (then wait::ld).
__device__ __forceinline__ void tmem_ld_x8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 3-D tensor TMA load completing on an mbarrier (SASS: UTMALDG).
__device__ __forceinline__ void tma_load_3d(void* dst_smem, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"((uint32_t)__cvta_generic_to_shared(dst_smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2),
      "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}

}  // namespace tc
}  // namespace chess
