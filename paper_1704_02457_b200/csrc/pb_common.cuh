// Shared device helpers for the panel-major FP64 kernels (sm_100a).
//
// Panel-major addressing (ps = 4, matstore.py:37-45): element (i, j) of a
// matrix with panel length cn lives at (i & ~3)*cn + 4*j + (i & 3).  An
// 8-row x 4-column block at a panel-aligned row is therefore two
// contiguous 128-byte runs, which is exactly one m8n8k4 f64 A (or B)
// fragment: lane t holds element (row t>>2, col t&3) and lanes 0-15 /
// 16-31 each read one 128-byte run -> conflict-free in shared memory and
// fully coalesced in global memory.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/pb_b200.h"

namespace pb {

typedef int64_t ix;

// Warp index as a value the compiler can prove warp-uniform (a shuffle from
// lane 0).  Derived straight from threadIdx it is not, so every shuffle / MMA
// inside a warp-dependent branch got WARPSYNC + collective fix-up code (the
// n = 128 potrf team kernel: 1622 -> 854 IMAD, 123 WARPSYNC -> 0).
__device__ __forceinline__ int warp_uniform() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

__host__ __device__ __forceinline__ ix eo(ix i, ix j, ix cn) { return (i & ~(ix)3) * cn + 4 * j + (i & 3); }

// Per-launch view of one operand: item base pointer + stride + panel length.
struct Mat {
  double *p;
  ix stride;  // doubles between items (0 = broadcast)
  ix cn;      // panel length
  double *d;  // diag_inv of item 0
  ix dstride;
  __device__ __forceinline__ double *item(ix b) const { return p + b * stride; }
  __device__ __forceinline__ double *ditem(ix b) const { return d + b * dstride; }
};

// m8n8k4 f64 MMA, D = A*B + C (SASS: DMMA.8x8x4).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// cp.async helpers (LDGSTS).  src_bytes < size zero-fills the remainder.
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double ldg_nc(const double *p) { return __ldg(p); }
__device__ __forceinline__ double2 ldg_nc2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

// ---- mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) ----
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 1-D bulk copy shared -> global (bulk-group completion), bytes % 16 == 0.
__device__ __forceinline__ void tma_store_1d(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// wait until every committed bulk store has finished READING shared memory
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Named barrier for a team of `nthreads` (multiple of 32) with id 1..15.
__device__ __forceinline__ void team_sync(int id, int nthreads) {
  if (nthreads == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
  }
}

}  // namespace pb
