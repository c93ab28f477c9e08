// mma.cuh -- warp-level bf16 MMA (m16n8k16) + ldmatrix + cp.async helpers used by the
// attention kernels (the GEMMs use tcgen05; see gemm.cu).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

namespace cs {

CS_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

CS_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// D = A(16x16, row) * B(16x8, col) + C ; bf16 inputs, fp32 accumulate
CS_DEV void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 16-byte async copy global->shared; src_bytes 0 zero-fills the destination.
CS_DEV void cp_async16(uint32_t dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
CS_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
CS_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// byte offset of 16B chunk `c` of row `r` in a [rows][D] bf16 tile with XOR swizzle
template <int D>
CS_DEV uint32_t swz(int r, int c) {
  constexpr int CH = D / 8;  // 16B chunks per row
  return (uint32_t)(r * (D * 2) + ((c ^ (r & 7)) & (CH - 1)) * 16 + ((c & ~(CH - 1)) * 16));
}

}  // namespace cs
