// K3: batched damped SPD inverse  dst = (src + shift I)^-1   (reference
// numerics.sym_inverse numerics.py:100-114 through kfac.damped_inverses
// kfac.py:140-155).
//
// Small matrices (n <= 128) are inverted by one CTA each, fully staged in
// shared memory, with the symmetric sweep: pivot k has value p_k = L_kk^2 (the
// squared Cholesky diagonal of the leading block), so "p_k <= 0" is exactly the
// condition under which the reference's cho_factor raises -- reported through
// the info word.  Every update is applied symmetrically, so the result is
// exactly symmetric like the reference's (inv + inv^T)/2.
//
// Larger matrices use the recursive 2x2 block (Schur complement) form of the
// same elimination, whose work is four tcgen05 3xTF32 GEMMs per level:
//   X11 = A11^-1 (recurse)          Z = X11 A12
//   S = A22 - A21 Z (symmetric)     X22 = S^-1 (recurse)
//   X12 = -Z X22, X21 = X12^T       X11 = X11 - X12 Z^T (symmetric)
// n^3 flops in total, like potrf+potri; the leaves are the shared-memory kernel.
// All matrices of a call advance in lock-step rounds (<= 2 launches per round).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "dpk_internal.h"

namespace dpk {
namespace {

constexpr int LEAF_N = 128;
constexpr int LEAF_THREADS = 256;
constexpr int LEAF_MAX = 256;

struct LeafJob {
  float* mat;
  int64_t ld;
  int32_t n;
  int32_t fail_code;
  int32_t* info;
};
struct LeafBatch {
  int n;
  LeafJob j[LEAF_MAX];
};

// In-place symmetric sweep on an n x n block (n <= 128) staged in smem;
// writes +inverse back.  Full storage, 2 barriers per pivot.
__global__ void __launch_bounds__(LEAF_THREADS) spd_leaf_kernel(const __grid_constant__ LeafBatch b) {
  extern __shared__ float S[];
  __shared__ float v[LEAF_N];
  const LeafJob& J = b.j[blockIdx.x];
  const int n = J.n;
  const int lds = n + 1;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < n; i += LEAF_THREADS / 32)
    for (int j = tx; j < n; j += 32) S[i * lds + j] = J.mat[static_cast<int64_t>(i) * J.ld + j];
  __syncthreads();
  bool failed = false;
  for (int k = 0; k < n; ++k) {
    for (int j = threadIdx.x; j < n; j += LEAF_THREADS) v[j] = S[k * lds + j];
    __syncthreads();
    const float p = v[k];
    if (!(p > 0.0f) || !isfinite(p)) {  // uniform across the block
      failed = true;
      break;
    }
    const float r = 1.0f / p;
    for (int i = ty; i < n; i += LEAF_THREADS / 32) {
      const float vi = v[i];
      for (int j = tx; j < n; j += 32) {
        float* s = &S[i * lds + j];
        if (i == k) {
          *s = (j == k) ? -r : v[j] * r;
        } else if (j == k) {
          *s = vi * r;
        } else {
          *s -= (vi * v[j]) * r;
        }
      }
    }
    __syncthreads();
  }
  if (failed) {
    if (threadIdx.x == 0 && J.info) *J.info = J.fail_code;
    return;
  }
  for (int i = ty; i < n; i += LEAF_THREADS / 32)
    for (int j = tx; j < n; j += 32) J.mat[static_cast<int64_t>(i) * J.ld + j] = -S[i * lds + j];
}

// dst = src + shift * I (copy, then the recursion works in place on dst)
constexpr int PREP_MAX = 256;
struct PrepBatch {
  int n;
  dpk_spd_job j[PREP_MAX];
};
__global__ void prep_kernel(const __grid_constant__ PrepBatch b) {
  const dpk_spd_job& J = b.j[blockIdx.y];
  const int64_t total = static_cast<int64_t>(J.n) * J.n;
  const float sh = J.shift ? *J.shift : 0.0f;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / J.n;
    const int64_t c = e - i * J.n;
    float x = J.src[e];
    if (i == c) x += sh;
    J.dst[e] = x;
  }
}

struct Op {
  bool leaf;
  LeafJob lj;
  GemmSpec g;
};

int split_point(int n) {
  int n1 = ((n / 2 + 63) / 64) * 64;
  return std::min(n1, n - 1);
}

size_t recursion_ws_floats(int n) {
  if (n <= LEAF_N) return 0;
  const int n1 = split_point(n), n2 = n - n1;
  return static_cast<size_t>(n1) * n2 + std::max(recursion_ws_floats(n1), recursion_ws_floats(n2));
}

GemmSpec spec(const dpk_operand& a, const dpk_operand& b, float* out, int64_t ldo, float alpha, float beta,
              int symmetric, float* out_t = nullptr, int64_t ldt = 0) {
  GemmSpec s{};
  s.job.a = a;
  s.job.b = b;
  s.job.out = out;
  s.job.ldo = ldo;
  s.job.cin = beta != 0.0f ? out : nullptr;
  s.job.ldc = ldo;
  s.job.alpha = alpha;
  s.job.beta = beta;
  s.job.symmetric = symmetric;
  s.epi = EPI_LINEAR;
  s.out_t = out_t;
  s.ldt = ldt;
  return s;
}

void build_ops(float* A, int64_t ld, int n, float* ws, int fail_code, int32_t* info, std::vector<Op>& ops) {
  if (n <= LEAF_N) {
    Op op{};
    op.leaf = true;
    op.lj = LeafJob{A, ld, n, fail_code, info};
    ops.push_back(op);
    return;
  }
  const int n1 = split_point(n), n2 = n - n1;
  float* A11 = A;
  float* A12 = A + n1;
  float* A21 = A + static_cast<int64_t>(n1) * ld;
  float* A22 = A21 + n1;
  float* Z = ws;  // n1 x n2
  float* child = ws + static_cast<size_t>(n1) * n2;
  build_ops(A11, ld, n1, child, fail_code, info, ops);
  Op op{};
  op.leaf = false;
  // Z = X11 A12
  op.g = spec(rows_k(A11, n1, n1, ld), rows_mn(A12, n2, n1, ld), Z, n2, 1.0f, 0.0f, 0);
  ops.push_back(op);
  // A22 <- A22 - A21 Z   (Schur complement, symmetric)
  op.g = spec(rows_k(A21, n2, n1, ld), rows_mn(Z, n2, n1, n2), A22, ld, -1.0f, 1.0f, 1);
  ops.push_back(op);
  build_ops(A22, ld, n2, child, fail_code, info, ops);
  // X12 = -Z X22 ; X21 = X12^T
  op.g = spec(rows_k(Z, n1, n2, n2), rows_k(A22, n2, n2, ld), A12, ld, -1.0f, 0.0f, 0, A21, ld);
  ops.push_back(op);
  // X11 <- X11 - X12 Z^T  (= X11 + Z X22 Z^T, symmetric)
  op.g = spec(rows_k(A12, n1, n2, ld), rows_k(Z, n1, n2, n2), A11, ld, -1.0f, 1.0f, 1);
  ops.push_back(op);
}

struct SpdPlan {
  std::vector<std::vector<Op>> lists;
  size_t rec_bytes = 0;
  size_t gemm_bytes = 0;
};

// float* base == nullptr: dry run for sizing (pointers are fake but sizes exact)
void make_spd_plan(const dpk_spd_job* jobs, int n, char* base, SpdPlan& plan) {
  plan.lists.assign(n, {});
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const size_t fl = recursion_ws_floats(jobs[i].n);
    float* ws = reinterpret_cast<float*>((base ? base : reinterpret_cast<char*>(0x100000)) + off);
    build_ops(jobs[i].dst, jobs[i].n, jobs[i].n, ws, jobs[i].fail_code, jobs[i].info, plan.lists[i]);
    off += align_up(fl * sizeof(float), 256);
  }
  plan.rec_bytes = off;
  // largest GEMM round
  std::vector<size_t> idx(n, 0);
  size_t worst = 0;
  for (;;) {
    std::vector<GemmSpec> g;
    bool any = false;
    for (int i = 0; i < n; ++i) {
      if (idx[i] >= plan.lists[i].size()) continue;
      any = true;
      const Op& op = plan.lists[i][idx[i]];
      if (!op.leaf) g.push_back(op.g);
      ++idx[i];
    }
    if (!any) break;
    if (!g.empty()) worst = std::max(worst, gemm_workspace_bytes(g.data(), static_cast<int>(g.size())));
  }
  plan.gemm_bytes = worst;
}

int launch_leaves(std::vector<LeafJob>& leaves, cudaStream_t st) {
  static bool configured = false;
  const int smem = LEAF_N * (LEAF_N + 1) * 4;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(spd_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(spd_leaf_kernel)");
    configured = true;
  }
  thread_local LeafBatch b;
  for (size_t first = 0; first < leaves.size(); first += LEAF_MAX) {
    const int cnt = static_cast<int>(std::min<size_t>(LEAF_MAX, leaves.size() - first));
    b.n = cnt;
    int maxn = 1;
    for (int i = 0; i < cnt; ++i) {
      b.j[i] = leaves[first + i];
      maxn = std::max(maxn, b.j[i].n);
    }
    spd_leaf_kernel<<<cnt, LEAF_THREADS, maxn * (maxn + 1) * 4, st>>>(b);
    note_launch();
    int rc = cuda_status(cudaGetLastError(), "spd_leaf_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

}  // namespace
}  // namespace dpk

extern "C" {

size_t dpk_chol_inv_workspace_bytes(const dpk_spd_job* jobs, int n_jobs) {
  if (n_jobs <= 0 || jobs == nullptr) return 0;
  dpk::SpdPlan plan;
  dpk::make_spd_plan(jobs, n_jobs, nullptr, plan);
  return dpk::align_up(plan.rec_bytes, 1024) + plan.gemm_bytes;
}

int dpk_chol_inv_damped_batched(const dpk_spd_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                                dpk_stream_t stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_chol_inv_damped_batched: bad job list");
    return DPK_EARG;
  }
  for (int i = 0; i < n_jobs; ++i) {
    if (jobs[i].n < 1 || jobs[i].src == nullptr || jobs[i].dst == nullptr || jobs[i].src == jobs[i].dst) {
      dpk::set_error("dpk_chol_inv_damped_batched: invalid job (n >= 1, distinct src/dst required)");
      return DPK_EARG;
    }
  }
  const size_t need = dpk_chol_inv_workspace_bytes(jobs, n_jobs);
  if (need > ws_bytes || (need > 0 && workspace == nullptr)) {
    dpk::set_error("dpk_chol_inv_damped_batched: workspace too small");
    return DPK_ENOSPACE;
  }
  // dst = src + shift I
  thread_local dpk::PrepBatch pb;
  for (int first = 0; first < n_jobs; first += dpk::PREP_MAX) {
    const int cnt = std::min(dpk::PREP_MAX, n_jobs - first);
    pb.n = cnt;
    int64_t maxe = 0;
    for (int i = 0; i < cnt; ++i) {
      pb.j[i] = jobs[first + i];
      maxe = std::max<int64_t>(maxe, static_cast<int64_t>(pb.j[i].n) * pb.j[i].n);
    }
    const int gx = static_cast<int>(std::min<int64_t>((maxe + 255) / 256, 2048));
    dpk::prep_kernel<<<dim3(gx, cnt), 256, 0, st>>>(pb);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "prep_kernel launch");
    if (rc) return rc;
  }
  dpk::SpdPlan plan;
  char* base = static_cast<char*>(workspace);
  dpk::make_spd_plan(jobs, n_jobs, base, plan);
  char* gemm_ws = base + dpk::align_up(plan.rec_bytes, 1024);
  std::vector<size_t> idx(n_jobs, 0);
  for (;;) {
    std::vector<dpk::LeafJob> leaves;
    std::vector<dpk::GemmSpec> g;
    bool any = false;
    for (int i = 0; i < n_jobs; ++i) {
      if (idx[i] >= plan.lists[i].size()) continue;
      any = true;
      const dpk::Op& op = plan.lists[i][idx[i]];
      if (op.leaf)
        leaves.push_back(op.lj);
      else
        g.push_back(op.g);
      ++idx[i];
    }
    if (!any) break;
    if (!leaves.empty()) {
      int rc = dpk::launch_leaves(leaves, st);
      if (rc) return rc;
    }
    if (!g.empty()) {
      int rc = dpk::gemm_launch(g.data(), static_cast<int>(g.size()), gemm_ws, plan.gemm_bytes, DPK_PREC_3XTF32, st);
      if (rc) return rc;
    }
  }
  return DPK_OK;
}

}  // extern "C"
