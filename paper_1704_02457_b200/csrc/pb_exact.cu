// Reference-order pass for the items the register-tile potrf kernel marked
// PB_INFO_EXACT (non-finite write set); see pb_exact.cuh.  One warp per
// marked item; unmarked items cost one 4-byte read of info.
#include "pb_exact.cuh"
#include "pb_gemm.cuh"

namespace pb {

__global__ void __launch_bounds__(128) potrf_exact_kernel(PotrfArgs g) {
  const int lane = threadIdx.x & 31;
  const ix w0 = ((ix)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((ix)gridDim.x * blockDim.x) >> 5;
  for (ix b = w0; b < g.batch; b += nw) {
    if (g.info[b] != PB_INFO_EXACT) continue;  // warp-uniform
    const int f = potrf_exact_warp(g.C.p + b * g.C.stride, g.ci, g.cj, g.C.cn, g.D.p + b * g.D.stride, g.di, g.dj,
                                   g.D.cn, g.D.d + b * g.D.dstride + g.dj, (int)g.n);
    if (lane == 0) g.info[b] = f >= 0 ? f + g.info_offset : -1;
  }
}

cudaError_t run_potrf_exact_fixup(const PotrfArgs &g, cudaStream_t st) {
  ix blocks = (g.batch + 3) / 4;  // 4 warps per block, one item per warp per pass
  const ix cap = (ix)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  potrf_exact_kernel<<<(unsigned)blocks, 128, 0, st>>>(g);
  note_launch();
  return cudaGetLastError();
}

}  // namespace pb
