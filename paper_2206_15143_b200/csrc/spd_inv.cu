// K3: batched damped SPD inverse  dst = (src + shift I)^-1   (reference
// numerics.sym_inverse numerics.py:100-114 -- cho_factor(lower) + cho_solve(I),
// symmetrized -- through kfac.damped_inverses kfac.py:140-155).
//
// Same method as the reference: Cholesky factor, then the inverse from the
// factor (potrf -> trtri -> L^-T L^-1, LAPACK potri's route).
//
// n <= 128: one CTA per matrix, everything in shared memory: right-looking
//   Cholesky (a non-positive pivot is exactly where cho_factor raises ->
//   info word), right-looking triangular inverse X = L^-1, then X^T X written
//   as lower tiles + mirror, so the result is exactly symmetric.
// n > 128: recursive 2x2 blocking whose off-diagonal work is tcgen05 3xTF32
//   GEMMs (fp32-grade):
//      L11, X11 = chol/trtri(A11)            (recurse; leaves = the smem kernel)
//      L21 = A21 X11^T                       (TRSM via the triangular inverse)
//      A22 <- A22 - L21 L21^T                (symmetric, lower tiles + mirror)
//      L22, X22 = chol/trtri(A22)            (recurse)
//      X21 = -X22 (L21 X11)
//   and finally dst = X^T X (symmetric).  Leaves only need X = L^-1 of their
//   diagonal block.  All matrices of a call advance in lock-step rounds of at
//   most one leaf launch + one grouped GEMM launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "dpk_internal.h"

namespace dpk {
namespace {

constexpr int LEAF_N = 128;
constexpr int LEAF_THREADS = 256;  // 16 x 16 thread grid
constexpr int LEAF_MAX = 256;

struct LeafJob {
  const float* src;    // input block (row stride lds)
  float* dst;          // TRI: X = L^-1 block (lower, zeros above); FULL: the inverse
  const float* shift;  // FULL mode: damping added to the diagonal (may be null)
  int64_t lds;
  int64_t ldd;
  int32_t n;
  int32_t full;        // 1: whole matrix -> inverse; 0: diagonal block -> L^-1
  int32_t fail_code;
  int32_t _pad;
  int32_t* info;
};
struct LeafBatch {
  int n;
  LeafJob j[LEAF_MAX];
};

// Register-resident leaf.  The (padded) N x N block, N = 16*NB, is spread over a
// 16 x 16 thread grid with a stride-16 interleave: thread (ty, tx) owns rows
// ty + 16r and columns tx + 16c (r, c < NB), so every broadcast vector read
// below is bank-conflict free and the work stays balanced as the active
// trailing block shrinks.  One fused sweep over k does both
//   right-looking Cholesky      A[i][j] -= L[i][k] L[j][k]        (i, j > k)
//   right-looking L^-1 (trtri)  X[i][:] -= L[i][k] X[k][:] / L[k][k]  (i > k)
// with one __syncthreads per column (double-buffered column / row vectors).
// Blocks that provably stay zero / untouched are skipped at compile time
// (kb, r, c are all unrolled).  Padding rows/columns are the identity, so
// pivots past n are 1 and the real n x n result is unaffected.
template <int NB>
__global__ void __launch_bounds__(LEAF_THREADS, 1) spd_leaf_kernel(const __grid_constant__ LeafBatch b) {
  constexpr int N = 16 * NB;
  constexpr int LDX = N + 1;
  extern __shared__ float smem[];
  float* colb = smem;          // [2][N]  column k of the partially factored A
  float* rowb = smem + 2 * N;  // [2][N]  row k of the partially solved X
  float* Xs = smem + 4 * N;    // [N][N+1] X for the FULL-mode X^T X
  const LeafJob& J = b.j[blockIdx.x];
  const int n = J.n;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const float sh = (J.full && J.shift) ? *J.shift : 0.0f;
  const float* src = J.src;
  const int64_t lds = J.lds;
  float a[NB][NB], x[NB][NB];
#pragma unroll
  for (int r = 0; r < NB; ++r)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int i = ty + 16 * r, j = tx + 16 * c;
      float v = (i == j) ? 1.0f : 0.0f;
      if (i < n && j < n) v = src[static_cast<int64_t>(i) * lds + j] + ((i == j) ? sh : 0.0f);
      a[r][c] = v;
      x[r][c] = (i == j) ? 1.0f : 0.0f;
    }
#pragma unroll
  for (int kb = 0; kb < NB; ++kb) {
#pragma unroll 1
    for (int kk = 0; kk < 16; ++kk) {
      const int k = 16 * kb + kk;
      float* cb = colb + (k & 1) * N;
      float* rb = rowb + (k & 1) * N;
      if (tx == kk) {
#pragma unroll
        for (int r = kb; r < NB; ++r) cb[ty + 16 * r] = a[r][kb];
      }
      if (ty == kk) {
#pragma unroll
        for (int c = 0; c <= kb; ++c) rb[tx + 16 * c] = x[kb][c];
      }
      __syncthreads();
      const float p = cb[k];
      if (!(p > 0.0f) || !isfinite(p)) {  // uniform: every thread read the same pivot
        if (tid == 0 && J.info) *J.info = J.fail_code;
        return;
      }
      const float inv = 1.0f / sqrtf(p);
      float lr[NB], lc[NB], xc[NB];
#pragma unroll
      for (int r = kb; r < NB; ++r) {
        const int i = ty + 16 * r;
        lr[r] = (i > k) ? cb[i] * inv : 0.0f;
      }
#pragma unroll
      for (int c = kb; c < NB; ++c) {
        const int j = tx + 16 * c;
        lc[c] = (j > k) ? cb[j] * inv : 0.0f;
      }
#pragma unroll
      for (int c = 0; c <= kb; ++c) xc[c] = rb[tx + 16 * c] * inv;
#pragma unroll
      for (int r = kb; r < NB; ++r) {
#pragma unroll
        for (int c = kb; c < NB; ++c) a[r][c] = fmaf(-lr[r], lc[c], a[r][c]);
#pragma unroll
        for (int c = 0; c <= kb; ++c) x[r][c] = fmaf(-lr[r], xc[c], x[r][c]);
      }
      if (ty == kk) {
#pragma unroll
        for (int c = 0; c <= kb; ++c) x[kb][c] = xc[c];
      }
    }
  }
  float* dst = J.dst;
  const int64_t ldd = J.ldd;
  if (!J.full) {  // X = L^-1: exactly zero above the diagonal by construction
#pragma unroll
    for (int r = 0; r < NB; ++r)
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int i = ty + 16 * r, j = tx + 16 * c;
        if (i < n && j < n) dst[static_cast<int64_t>(i) * ldd + j] = x[r][c];
      }
    return;
  }
  // ---- inverse = X^T X  (X[k][i] == 0 for k < i: block kb only meets r, c <= kb)
#pragma unroll
  for (int r = 0; r < NB; ++r)
#pragma unroll
    for (int c = 0; c < NB; ++c) Xs[(ty + 16 * r) * LDX + tx + 16 * c] = x[r][c];
  __syncthreads();
  float acc[NB][NB];
#pragma unroll
  for (int r = 0; r < NB; ++r)
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[r][c] = 0.0f;
#pragma unroll
  for (int kb = 0; kb < NB; ++kb) {
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      const float* row = Xs + (16 * kb + kk) * LDX;
      float xi[NB], xj[NB];
#pragma unroll
      for (int r = 0; r <= kb; ++r) xi[r] = row[ty + 16 * r];
#pragma unroll
      for (int c = 0; c <= kb; ++c) xj[c] = row[tx + 16 * c];
#pragma unroll
      for (int r = 0; r <= kb; ++r)
#pragma unroll
        for (int c = 0; c <= kb; ++c) acc[r][c] = fmaf(xi[r], xj[c], acc[r][c]);
    }
  }
#pragma unroll
  for (int r = 0; r < NB; ++r)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int i = ty + 16 * r, j = tx + 16 * c;
      if (i < n && j < n) dst[static_cast<int64_t>(i) * ldd + j] = acc[r][c];
    }
}

template <int NB>
constexpr int leaf_smem_bytes() {
  return (4 * 16 * NB + 16 * NB * (16 * NB + 1)) * 4;
}

// Aw = src + shift I for the blocked path; Aw rows are padded to ldw (a multiple
// of 4 floats) so every recursion operand is a 16-byte aligned TMA view.
constexpr int PREP_MAX = 256;
struct PrepJob {
  const float* src;
  float* dst;
  const float* shift;
  int64_t n;
  int64_t ldw;
};
struct PrepBatch {
  int n;
  PrepJob j[PREP_MAX];
};
__global__ void prep_kernel(const __grid_constant__ PrepBatch b) {
  const PrepJob& J = b.j[blockIdx.y];
  const int64_t total = J.n * J.n;
  const float sh = J.shift ? *J.shift : 0.0f;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e / J.n;
    const int64_t c = e - i * J.n;
    float x = J.src[e];
    if (i == c) x += sh;
    J.dst[i * J.ldw + c] = x;
  }
}

inline int64_t padded_ld(int n) { return (static_cast<int64_t>(n) + 3) / 4 * 4; }

struct Op {
  bool leaf;
  LeafJob lj;
  GemmSpec g;
};

int split_point(int n) {
  const int n1 = ((n / 2 + 63) / 64) * 64;
  return std::min(n1, n - 1);
}

size_t t_floats(int n) {  // largest n2 x n1 scratch over the recursion
  if (n <= LEAF_N) return 0;
  const int n1 = split_point(n), n2 = n - n1;
  return std::max<size_t>(static_cast<size_t>(n1) * n2, std::max(t_floats(n1), t_floats(n2)));
}

size_t matrix_ws_floats(int n) {
  if (n <= LEAF_N) return 0;
  // working copy Aw, L21 blocks, X = L^-1 (all n x padded_ld), T scratch (+4 for alignment)
  return 3 * static_cast<size_t>(n) * padded_ld(n) + t_floats(n) + 4;
}

GemmSpec spec(const dpk_operand& a, const dpk_operand& b, float* out, int64_t ldo, float alpha, float beta,
              int symmetric) {
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
  return s;
}

// Aw, Lb, Xb share the row stride ld; T has room for n2 x n1 floats.
void build_ops(float* Aw, float* Lb, float* Xb, int64_t ld, int n, float* T, int fail_code, int32_t* info,
               std::vector<Op>& ops) {
  if (n <= LEAF_N) {
    Op op{};
    op.leaf = true;
    op.lj = LeafJob{Aw, Xb, nullptr, ld, ld, n, 0, fail_code, 0, info};
    ops.push_back(op);
    return;
  }
  const int n1 = split_point(n), n2 = n - n1;
  const int64_t o21 = static_cast<int64_t>(n1) * ld, o22 = o21 + n1;
  build_ops(Aw, Lb, Xb, ld, n1, T, fail_code, info, ops);
  Op op{};
  op.leaf = false;
  // L21 = A21 X11^T
  op.g = spec(rows_k(Aw + o21, n2, n1, ld), rows_k(Xb, n1, n1, ld), Lb + o21, ld, 1.0f, 0.0f, 0);
  ops.push_back(op);
  // A22 <- A22 - L21 L21^T
  op.g = spec(rows_k(Lb + o21, n2, n1, ld), rows_k(Lb + o21, n2, n1, ld), Aw + o22, ld, -1.0f, 1.0f, 1);
  ops.push_back(op);
  build_ops(Aw + o22, Lb + o22, Xb + o22, ld, n2, T, fail_code, info, ops);
  // T = L21 X11
  op.g = spec(rows_k(Lb + o21, n2, n1, ld), rows_mn(Xb, n1, n1, ld), T, n1, 1.0f, 0.0f, 0);
  ops.push_back(op);
  // X21 = -X22 T
  op.g = spec(rows_k(Xb + o22, n2, n2, ld), rows_mn(T, n1, n2, n1), Xb + o21, ld, -1.0f, 0.0f, 0);
  ops.push_back(op);
}

struct SpdPlan {
  std::vector<std::vector<Op>> lists;
  std::vector<PrepJob> preps;
  std::vector<float*> zero_x;
  std::vector<size_t> zero_bytes;
  size_t rec_bytes = 0;
  size_t gemm_bytes = 0;
};

void make_spd_plan(const dpk_spd_job* jobs, int n, char* base, SpdPlan& plan) {
  plan.lists.assign(n, {});
  char* b = base ? base : reinterpret_cast<char*>(0x100000);
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int m = jobs[i].n;
    std::vector<Op>& ops = plan.lists[i];
    if (m <= LEAF_N) {
      Op op{};
      op.leaf = true;
      op.lj = LeafJob{jobs[i].src, jobs[i].dst, jobs[i].shift, m, m, m, 1, jobs[i].fail_code, 0, jobs[i].info};
      ops.push_back(op);
      continue;
    }
    const int64_t ldw = padded_ld(m);  // 16-byte rows -> TMA-addressable operands
    const size_t blk = static_cast<size_t>(m) * ldw;
    float* Aw = reinterpret_cast<float*>(b + off);
    float* Lb = Aw + blk;
    float* Xb = Lb + blk;
    float* T = Xb + blk;
    off += align_up(matrix_ws_floats(m) * sizeof(float), 256);
    plan.preps.push_back(PrepJob{jobs[i].src, Aw, jobs[i].shift, m, ldw});
    plan.zero_x.push_back(Xb);
    plan.zero_bytes.push_back(blk * sizeof(float));
    build_ops(Aw, Lb, Xb, ldw, m, T, jobs[i].fail_code, jobs[i].info, ops);
    Op op{};
    op.leaf = false;
    // dst = X^T X  (X lower triangular; symmetric output, written with the caller's ld = n)
    op.g = spec(rows_mn(Xb, m, m, ldw), rows_mn(Xb, m, m, ldw), jobs[i].dst, m, 1.0f, 0.0f, 1);
    ops.push_back(op);
  }
  plan.rec_bytes = off;
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

template <int NB>
int launch_leaf_nb(const LeafBatch& b, int cnt, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(spd_leaf_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         leaf_smem_bytes<NB>());
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(spd_leaf_kernel)");
    configured = true;
  }
  spd_leaf_kernel<NB><<<cnt, LEAF_THREADS, leaf_smem_bytes<NB>(), st>>>(b);
  note_launch();
  return cuda_status(cudaGetLastError(), "spd_leaf_kernel launch");
}

int launch_leaves(std::vector<LeafJob>& leaves, cudaStream_t st) {
  thread_local LeafBatch b;
  for (size_t first = 0; first < leaves.size(); first += LEAF_MAX) {
    const int cnt = static_cast<int>(std::min<size_t>(LEAF_MAX, leaves.size() - first));
    b.n = cnt;
    int maxn = 1;
    for (int i = 0; i < cnt; ++i) {
      b.j[i] = leaves[first + i];
      maxn = std::max(maxn, b.j[i].n);
    }
    int rc;
    if (maxn <= 16)
      rc = launch_leaf_nb<1>(b, cnt, st);
    else if (maxn <= 32)
      rc = launch_leaf_nb<2>(b, cnt, st);
    else if (maxn <= 64)
      rc = launch_leaf_nb<4>(b, cnt, st);
    else
      rc = launch_leaf_nb<8>(b, cnt, st);
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
  dpk::SpdPlan plan;
  char* base = static_cast<char*>(workspace);
  dpk::make_spd_plan(jobs, n_jobs, base, plan);
  char* gemm_ws = base + dpk::align_up(plan.rec_bytes, 1024);
  // blocked path set-up: working copy with the damping, X = 0
  thread_local dpk::PrepBatch pb;
  for (size_t first = 0; first < plan.preps.size(); first += dpk::PREP_MAX) {
    const int cnt = static_cast<int>(std::min<size_t>(dpk::PREP_MAX, plan.preps.size() - first));
    pb.n = cnt;
    int64_t maxe = 0;
    for (int i = 0; i < cnt; ++i) {
      pb.j[i] = plan.preps[first + i];
      maxe = std::max<int64_t>(maxe, pb.j[i].n * pb.j[i].n);
    }
    const int gx = static_cast<int>(std::min<int64_t>((maxe + 255) / 256, 2048));
    dpk::prep_kernel<<<dim3(gx, cnt), 256, 0, st>>>(pb);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "prep_kernel launch");
    if (rc) return rc;
  }
  for (size_t i = 0; i < plan.zero_x.size(); ++i) {
    int rc = dpk::cuda_status(cudaMemsetAsync(plan.zero_x[i], 0, plan.zero_bytes[i], st), "cudaMemsetAsync");
    if (rc) return rc;
  }
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
