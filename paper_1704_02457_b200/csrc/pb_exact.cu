// Reference-order pass for the items the register-tile potrf kernel marked
// PB_INFO_EXACT (non-finite write set); see pb_exact.cuh.  One warp per
// marked item; unmarked items cost one coalesced 4-byte read of info.
#include "pb_exact.cuh"
#include "pb_gemm.cuh"

namespace pb {

__global__ void __launch_bounds__(128) potrf_exact_kernel(PotrfArgs g) {
  const int lane = threadIdx.x & 31;
  const ix w0 = ((ix)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((ix)gridDim.x * blockDim.x) >> 5;
  // each warp scans 32 consecutive statuses per pass (one coalesced load),
  // then redoes the marked ones together
  for (ix b0 = w0 * 32; b0 < g.batch; b0 += nw * 32) {
    const ix bl = b0 + lane;
    unsigned marked = __ballot_sync(0xffffffffu, bl < g.batch && g.info[bl] == PB_INFO_EXACT);
    while (marked) {
      const int k = __ffs(marked) - 1;
      marked &= marked - 1;
      const ix b = b0 + k;
      const int f = potrf_exact_warp(g.C.p + b * g.C.stride, g.ci, g.cj, g.C.cn, g.D.p + b * g.D.stride, g.di, g.dj,
                                     g.D.cn, g.D.d + b * g.D.dstride + g.dj, (int)g.n);
      if (lane == 0) g.info[b] = f >= 0 ? f + g.info_offset : -1;
    }
  }
}

cudaError_t run_potrf_exact_fixup(const PotrfArgs &g, cudaStream_t st) {
  ix blocks = (g.batch + 127) / 128;  // 4 warps per block, 32 statuses per warp per pass
  const ix cap = (ix)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  potrf_exact_kernel<<<(unsigned)blocks, 128, 0, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
