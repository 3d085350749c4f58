// K4: batched symmetric eigendecomposition (reference numerics.sym_eig,
// numerics.py:75-97): symmetrize (M + M^T)/2, decompose, eigenvalues in
// DESCENDING order with eigenvectors as the columns of q.
//
// n <= 128: one CTA per matrix, one-sided (Hestenes) Jacobi in shared memory
// (jacobi1s.cuh): the n/2 column-pair rotations of a tournament round are
// independent, one warp each; sweeps stop once every column pair is orthogonal
// to rel_tol.  (Round 1 used a two-sided Jacobi with a row and a column phase per
// round on 256 threads: ~10 ms for 24 matrices of n=128, now ~0.1-0.3 ms.)
// n > 128: the tensor-core block Jacobi of syevj.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "dpk_internal.h"
#include "jacobi1s.cuh"

#include <vector>

namespace dpk {
namespace {

constexpr int JAC_N = 128;  // largest n handled on chip
constexpr int JAC_MAX = 256;

struct EigBatch {
  int n;
  float rel_tol, abs_tol;  // rotation thresholds (jac_tolerances)
  dpk_eig_job j[JAC_MAX];
};

// One CTA (1024 threads) per matrix: one-sided Jacobi in shared memory
// (jacobi1s.cuh), then eigenvalues ranked descending (ties by index) and the
// eigenvector columns scattered to their ranks.
__global__ void __launch_bounds__(J1_THREADS) jacobi_kernel(const __grid_constant__ EigBatch b) {
  extern __shared__ float sm[];
  __shared__ float lam[JAC_N + 2];
  __shared__ int rank_of[JAC_N];
  const dpk_eig_job& J = b.j[blockIdx.x];
  const int n = J.n;
  const int m = n + (n & 1);  // padded to even; the padding column is inert
  const int ld = m;
  float* U = sm;
  float* V = sm + m * ld;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int c = e / m, r = e - (e / m) * m;  // column-major: element (r, c) at c*ld + r
    float a = 0.f;
    if (r < n && c < n) a = 0.5f * (J.src[r * n + c] + J.src[c * n + r]);
    U[c * ld + r] = a;
    V[c * ld + r] = (r == c) ? 1.0f : 0.0f;
  }
  __syncthreads();
  onesided_jacobi(U, V, ld, n, m, b.rel_tol, lam);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float wi = lam[i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const float wj = lam[j];
      r += (wj > wi) || (wj == wi && j < i);
    }
    rank_of[i] = r;
    if (!isfinite(wi) && J.info) *J.info = DPK_INFO_NONFINITE;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) J.w[rank_of[i]] = lam[i];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e - (e / n) * n;
    J.q[r * n + rank_of[c]] = V[c * ld + r];
  }
}

}  // namespace

// Jacobi rotation threshold: rotate the column pair (p, q) only if
// |u_p . u_q| > rel |u_p| |u_q| -- below it the columns are orthogonal to the
// rounding level of the fp32 dot products (~sqrt(n) eps) and further rotations
// only re-inject noise.  DPK_JAC_REL overrides (default 2e-6); abs is unused by
// the one-sided kernels and kept for the ABI of the batch structs.
void jac_tolerances(float& rel, float& abs_) {
  static float r = -1.f;
  if (r < 0.f) {
    const char* e = getenv("DPK_JAC_REL");
    r = e ? static_cast<float>(atof(e)) : 2e-6f;
  }
  rel = r;
  abs_ = 0.f;
}
}  // namespace dpk

extern "C" {

size_t dpk_syevd_workspace_bytes(const dpk_eig_job* jobs, int n_jobs) {
  if (n_jobs <= 0 || jobs == nullptr) return 0;
  return dpk::syevj_workspace_bytes(jobs, n_jobs);
}

int dpk_syevd_batched(const dpk_eig_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_syevd_batched: bad job list");
    return DPK_EARG;
  }
  int maxm = 2;
  for (int i = 0; i < n_jobs; ++i) {
    if (jobs[i].n < 1 || !jobs[i].src || !jobs[i].q || !jobs[i].w) {
      dpk::set_error("dpk_syevd_batched: invalid job");
      return DPK_EARG;
    }
    if (jobs[i].n <= dpk::JAC_N) maxm = std::max(maxm, jobs[i].n + (jobs[i].n & 1));
  }
  cudaStream_t st0 = static_cast<cudaStream_t>(stream);
  // n > 128: block Jacobi on the tensor cores (syevj.cu)
  int rc0 = dpk::syevj_run(jobs, n_jobs, workspace, ws_bytes, st0);
  if (rc0) return rc0;
  std::vector<dpk_eig_job> small;
  for (int i = 0; i < n_jobs; ++i)
    if (jobs[i].n <= dpk::JAC_N) small.push_back(jobs[i]);
  if (small.empty()) return DPK_OK;
  jobs = small.data();
  n_jobs = static_cast<int>(small.size());
  const int smem = 2 * maxm * maxm * 4;
  static std::atomic<uint64_t> configured_on{0};
  if (dpk::first_on_device(configured_on)) {
    cudaError_t e = cudaFuncSetAttribute(dpk::jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * dpk::JAC_N * dpk::JAC_N * 4);
    if (e != cudaSuccess) return dpk::cuda_status(e, "cudaFuncSetAttribute(jacobi_kernel)");
  }
  thread_local dpk::EigBatch b;
  dpk::jac_tolerances(b.rel_tol, b.abs_tol);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int first = 0; first < n_jobs; first += dpk::JAC_MAX) {
    const int cnt = std::min(dpk::JAC_MAX, n_jobs - first);
    b.n = cnt;
    for (int i = 0; i < cnt; ++i) b.j[i] = jobs[first + i];
    dpk::jacobi_kernel<<<cnt, dpk::J1_THREADS, smem, st>>>(b);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "jacobi_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

}  // extern "C"
