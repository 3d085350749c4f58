// K4: batched symmetric eigendecomposition (reference numerics.sym_eig,
// numerics.py:75-97): symmetrize (M + M^T)/2, decompose, eigenvalues in
// DESCENDING order with eigenvectors as the columns of q.
//
// n <= 128: one CTA per matrix, A and V staged in shared memory, cyclic
// two-sided Jacobi with the round-robin (tournament) ordering so the n/2
// rotations of a round are independent and applied in parallel; sweeps stop
// once every off-diagonal entry is negligible against its diagonal pair.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "dpk_internal.h"

#include <vector>

namespace dpk {
namespace {

constexpr int JAC_N = 128;  // largest n handled on chip
constexpr int JAC_THREADS = 256;
constexpr int JAC_MAX = 256;
constexpr int MAX_SWEEPS = 15;

struct EigBatch {
  int n;
  dpk_eig_job j[JAC_MAX];
};

// tournament pairing: players 0..m-1 (m even), player m-1 fixed, others rotate
__device__ __forceinline__ void pair_of(int round, int slot, int m, int& p, int& q) {
  int a, b;
  if (slot == 0) {
    a = m - 1;
    b = round;
  } else {
    a = (round + slot) % (m - 1);
    b = (round - slot + (m - 1)) % (m - 1);
  }
  p = min(a, b);
  q = max(a, b);
}

__global__ void __launch_bounds__(JAC_THREADS) jacobi_kernel(const __grid_constant__ EigBatch b) {
  extern __shared__ float sm[];
  __shared__ float cs[JAC_N / 2 + 1], sn[JAC_N / 2 + 1];
  __shared__ float dp_new[JAC_N / 2 + 1], dq_new[JAC_N / 2 + 1];
  __shared__ int pp[JAC_N / 2 + 1], qq[JAC_N / 2 + 1];
  __shared__ int rot_count;
  __shared__ float fro2;
  __shared__ int rank_of[JAC_N];
  const dpk_eig_job& J = b.j[blockIdx.x];
  const int n = J.n;
  const int m = n + (n & 1);  // padded to even; padded index is inert
  const int ld = m + 1;
  float* A = sm;
  float* V = sm + m * ld;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e / m, c = e - (e / m) * m;
    float a = 0.f;
    if (i < n && c < n) a = 0.5f * (J.src[i * n + c] + J.src[c * n + i]);
    A[i * ld + c] = a;
    V[i * ld + c] = (i == c) ? 1.0f : 0.0f;
  }
  if (threadIdx.x == 0) fro2 = 0.0f;
  __syncthreads();
  {
    float acc = 0.0f;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const float a = A[(e / m) * ld + (e % m)];
      acc += a * a;
    }
    atomicAdd(&fro2, acc);
  }
  __syncthreads();
  // off-diagonal entries below ~eps*||A||_F are rounding noise of the other
  // rotations; rotating them only re-injects noise (and never terminates)
  const float abs_tol = 3e-8f * sqrtf(fro2);
  const int half = m / 2;
  for (int sweep = 0; sweep < MAX_SWEEPS && m > 1; ++sweep) {
    if (threadIdx.x == 0) rot_count = 0;
    __syncthreads();
    for (int round = 0; round < m - 1; ++round) {
      // 1. rotation angles, one thread per pair
      for (int s = threadIdx.x; s < half; s += blockDim.x) {
        int p, q;
        pair_of(round, s, m, p, q);
        pp[s] = p;
        qq[s] = q;
        const float apq = A[p * ld + q];
        const float app = A[p * ld + p], aqq = A[q * ld + q];
        float c = 1.f, si = 0.f;
        if (fabsf(apq) > 2e-7f * sqrtf(fabsf(app * aqq)) && fabsf(apq) > abs_tol && fabsf(apq) > 1e-36f) {
          // IEEE-rounded sqrt / division: c^2 + s^2 = 1 to 1/2 ulp with no bias
          // (rsqrtf's bias compounds over thousands of rotations into a visible
          // shrink of the spectrum)
          const float tau = (aqq - app) / (2.0f * apq);
          const float t = copysignf(1.0f, tau) / (fabsf(tau) + __fsqrt_rn(1.0f + tau * tau));
          c = __fdiv_rn(1.0f, __fsqrt_rn(1.0f + t * t));
          si = t * c;
          atomicAdd(&rot_count, 1);
          // the rotated 2x2 block is known in closed form (NR 11.1.14-15); writing it
          // exactly after the generic row/column updates keeps the diagonal clean
          dp_new[s] = app - t * apq;
          dq_new[s] = aqq + t * apq;
        } else {
          dp_new[s] = app;
          dq_new[s] = aqq;
        }
        cs[s] = c;
        sn[s] = si;
      }
      __syncthreads();
      // 2. rows p, q  (A <- J^T A)
      for (int e = threadIdx.x; e < half * m; e += blockDim.x) {
        const int s = e / m, c = e - s * m;
        const int p = pp[s], q = qq[s];
        const float co = cs[s], si = sn[s];
        const float ap = A[p * ld + c], aq = A[q * ld + c];
        A[p * ld + c] = co * ap - si * aq;
        A[q * ld + c] = si * ap + co * aq;
      }
      __syncthreads();
      // 3. columns p, q (A <- A J) and V <- V J
      for (int e = threadIdx.x; e < half * m; e += blockDim.x) {
        const int s = e / m, r = e - s * m;
        const int p = pp[s], q = qq[s];
        const float co = cs[s], si = sn[s];
        const float ap = A[r * ld + p], aq = A[r * ld + q];
        A[r * ld + p] = co * ap - si * aq;
        A[r * ld + q] = si * ap + co * aq;
        const float vp = V[r * ld + p], vq = V[r * ld + q];
        V[r * ld + p] = co * vp - si * vq;
        V[r * ld + q] = si * vp + co * vq;
      }
      __syncthreads();
      for (int s = threadIdx.x; s < half; s += blockDim.x) {
        if (sn[s] != 0.0f) {
          const int p = pp[s], q = qq[s];
          A[p * ld + p] = dp_new[s];
          A[q * ld + q] = dq_new[s];
          A[p * ld + q] = 0.0f;
          A[q * ld + p] = 0.0f;
        }
      }
      __syncthreads();
    }
    if (rot_count == 0) break;
    __syncthreads();
  }
  // re-normalize V's columns: thousands of rotations with c^2 + s^2 = 1 only to
  // 1/2 ulp drift the column norms by ~1e-5; orthogonality between columns is
  // already at the 1e-7 level, so a rescale restores an orthonormal basis.
  // (8 warps; warp w owns columns w, w+8, ...; lanes stride the rows.)
  {
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = wid; c < n; c += JAC_THREADS / 32) {
      float ss = 0.f;
      for (int r = lane; r < n; r += 32) ss = fmaf(V[r * ld + c], V[r * ld + c], ss);
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const float inv = ss > 0.f ? rsqrtf(ss) : 1.f;
      const float fix = inv * (1.5f - 0.5f * ss * inv * inv);  // one Newton step: rsqrt to ~1 ulp
      for (int r = lane; r < n; r += 32) V[r * ld + c] *= fix;
    }
  }
  __syncthreads();
  // rank eigenvalues descending (ties by index) and scatter
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float wi = A[i * ld + i];
    int r = 0;
    for (int j = 0; j < n; ++j) {
      const float wj = A[j * ld + j];
      r += (wj > wi) || (wj == wi && j < i);
    }
    rank_of[i] = r;
    if (!isfinite(wi) && J.info) *J.info = DPK_INFO_NONFINITE;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) J.w[rank_of[i]] = A[i * ld + i];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int r = e / n, c = e - (e / n) * n;
    J.q[r * n + rank_of[c]] = V[r * ld + c];
  }
}

}  // namespace
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
  const int smem = 2 * maxm * (maxm + 1) * 4;
  static std::atomic<uint64_t> configured_on{0};
  if (dpk::first_on_device(configured_on)) {
    cudaError_t e = cudaFuncSetAttribute(dpk::jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * dpk::JAC_N * (dpk::JAC_N + 1) * 4);
    if (e != cudaSuccess) return dpk::cuda_status(e, "cudaFuncSetAttribute(jacobi_kernel)");
  }
  thread_local dpk::EigBatch b;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int first = 0; first < n_jobs; first += dpk::JAC_MAX) {
    const int cnt = std::min(dpk::JAC_MAX, n_jobs - first);
    b.n = cnt;
    for (int i = 0; i < cnt; ++i) b.j[i] = jobs[first + i];
    dpk::jacobi_kernel<<<cnt, dpk::JAC_THREADS, smem, st>>>(b);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "jacobi_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

}  // extern "C"
