// Internal launch-argument structs shared by the kernels and the C ABI.
#pragma once
#include <mutex>

#include "pb_common.cuh"

namespace pb {

struct GemmArgs {
  ix m, n, k;
  double alpha, beta;
  Mat A, B, C, D;
  ix ai, aj, bi, bj, ci, cj, di, dj;
  ix batch;
  bool vecA, vecB;      // 16-byte cp.async legal for the A / B stream
  bool tma;             // bulk copies legal for A and B (16-byte aligned items)
  bool tmaC;            // ... and for C
  const int32_t *skip;  // optional: item b is left untouched if skip[b] >= 0
};

struct TrsmArgs {
  ix m, n;
  double alpha;
  Mat A, B, D;
  ix ai, aj, bi, bj, di, dj;
  int use_dA;
  int32_t *info;
  ix batch;
  const int32_t *skip;  // optional: item b is left untouched if skip[b] >= 0
};

struct PotrfArgs {
  ix m, n;
  Mat C, D;
  ix ci, cj, di, dj;
  int32_t *info;
  ix batch;
  // merge mode (blocked driver): items with info[b] >= 0 on entry are
  // skipped; a new failure is stored as info_offset + local index.
  int merge;
  int info_offset;
  // fused syrk_potrf (syrk_potrf_drv ccore.pyx:908-941): factor
  // lower(C + A*B^T), A m x k, B n x k; B may be A's own window (ab_same)
  int syrk = 0;
  int ab_same = 0;
  Mat A{}, B{};
  ix ai = 0, aj = 0, bi = 0, bj = 0, k = 0;
  // fused commit (blocked driver, chain kernel only): after item b's factorization, rows [0, rmax) x
  // [0, c_cols) of the aligned panel matrix cS (the solved rows below the previous panel) are copied to
  // D at (c_di, c_dj); rmax = c_rows for a healthy item, (f & ~3) + 4 for one failing at local pivot f
  // (the reference's row-panel write set, ccore.pyx:877-905); skipped items commit nothing
  int commit = 0;
  Mat cS{};
  ix c_rows = 0, c_cols = 0, c_di = 0, c_dj = 0;
};

struct CopyArgs {
  ix m, n;
  // strided (dense) side
  const double *X;
  double *Xw;
  ix x_row, x_col, x_stride;
  // panel sides
  Mat S, D;
  ix si, sj, di, dj;
  ix batch;
};

void note_launch();
int num_sms();  // of the current device (cached per device)

// Launch attributes of one kernel instantiation whose dynamic shared memory
// depends on the call's shape: the max-dynamic-smem attribute is raised once
// per device to the largest size seen and the occupancy is queried once per
// (device, smem, threads) -- no per-call driver queries on the launch path.
struct LaunchCache {
  std::mutex mu;
  int smem_set[16] = {0};
  int64_t keys[64];
  int vals[64];
  int n = 0;
  int occupancy(const void *kern, int threads, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (dev >= 0 && dev < 16 && (int)smem > smem_set[dev]) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      smem_set[dev] = (int)smem;
    }
    const int64_t key = ((int64_t)dev << 48) | ((int64_t)smem << 12) | threads;
    for (int i = 0; i < n; ++i)
      if (keys[i] == key) return vals[i];
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    if (occ < 1) occ = 1;
    if (n < 64) keys[n] = key, vals[n++] = occ;
    return occ;
  }
};

cudaError_t run_gemm_nt(const GemmArgs &g, cudaStream_t st);
cudaError_t run_syrk_ln(const GemmArgs &g, cudaStream_t st);
cudaError_t run_gemm_nn(const GemmArgs &g, cudaStream_t st);
cudaError_t run_trmm_rlnn(const GemmArgs &g, cudaStream_t st);
cudaError_t run_trsm_rltn(const TrsmArgs &g, cudaStream_t st);
cudaError_t run_potrf_l(const PotrfArgs &g, cudaStream_t st);
cudaError_t run_pack(const CopyArgs &g, cudaStream_t st);
cudaError_t run_unpack(const CopyArgs &g, cudaStream_t st);
cudaError_t run_gecp(const CopyArgs &g, cudaStream_t st);
cudaError_t run_diag_check(const Mat &A, ix ai, ix aj, ix n, ix batch, int32_t *info, cudaStream_t st);
bool potrf_fits(ix m, ix n);
bool syrk_potrf_fits(ix m, ix n, ix k, bool ab_same);
cudaError_t run_syrk_potrf(const PotrfArgs &g, cudaStream_t st);
bool potrf_small_ok(const PotrfArgs &g);
bool potrf_reg_ok(const PotrfArgs &g);
cudaError_t run_potrf_reg(const PotrfArgs &g, cudaStream_t st);
cudaError_t run_potrf_small(const PotrfArgs &g, cudaStream_t st);
bool potrf_chain_ok(const PotrfArgs &g);
cudaError_t run_potrf_chain(const PotrfArgs &g, cudaStream_t st);
cudaError_t run_potrf_exact_fixup(const PotrfArgs &g, cudaStream_t st);
bool trsm_fits(ix m, ix n);
bool trsm_wide_ok(const TrsmArgs &g);
cudaError_t run_trsm_wide(const TrsmArgs &g, cudaStream_t st);
size_t getrf_smem(int m, int n);
cudaError_t run_getrf(int m, int n, int pivot, const Mat &C, ix ci, ix cj, const Mat &D, ix di, ix dj, int64_t *ipiv,
                      ix ipiv_stride, int32_t *info, ix batch, cudaStream_t st);

}  // namespace pb
