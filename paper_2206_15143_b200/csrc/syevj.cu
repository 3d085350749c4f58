// K4 for n > 128: symmetric eigendecomposition by parallel two-sided BLOCK
// Jacobi (reference numerics.sym_eig, numerics.py:75-97: symmetrize, decompose,
// eigenvalues DESCENDING, eigenvectors as the columns of q).
//
// The matrix (zero-padded to N = 64 * nb, nb even) is split into nb blocks of 64
// rows/columns.  A round pairs the blocks (2p, 2p+1) of the CURRENT layout:
//   1. bj_pair_kernel (one CTA per pair): the 128 x 128 diagonal block of the pair
//      is diagonalised on chip (the same cyclic Jacobi as the n <= 128 kernel), its
//      eigenvectors ordered so the rotation keeps "uniformly bounded cosines" (the
//      64 columns with the largest weight in the first half are the first block's
//      continuation) and the two halves swapped: V_p lands on the p-th diagonal
//      128-block of Vbig (the off-diagonal blocks stay zero);
//   2. three tcgen05 3xTF32 GEMMs with block-diagonal K clipping (TRI_BLOCK: a
//      tile only reads the 128 (or 256) rows of Vbig of its own block):
//         Bt = A Vbig,   Q' = Q Vbig,   A' = Vbig^T Bt
//      each written with a cyclic shift of one block (+64 rows / columns, the
//      last 64 wrap to the front: two problems per product).
// The shift makes the next round's pairs -- the odd pairs (2p+1, 2p+2) of the
// odd-even transposition network -- aligned at (2p, 2p+1) again, and the swap
// moves each block one slot along the network, so every pair of blocks meets
// exactly once per nb rounds (one sweep); at odd rounds the pair holding the two
// ends of the line is the identity (no rotation, no swap).  A' = Q'^T A0 Q'
// throughout; after the sweeps diag(A') are the eigenvalues and the columns of
// Q' the eigenvectors.  Padding rows / columns are exactly zero (their rotations
// have zero angle, GEMMs multiply them by exact 0/1 entries), so padded
// eigenvectors stay unit vectors on the padding coordinates and are dropped.
//
// Costs ~12 N^3 flops per sweep on the tensor cores (3 passes each) and converges
// quadratically (5-8 sweeps for fp32 on K-FAC factors); every launch of a call is
// captured once into a CUDA graph keyed by the job list and replayed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "dpk_internal.h"
#include "jacobi1s.cuh"

namespace dpk {
namespace {

constexpr int BJ_B = 64;          // block edge; a pair is one 128 x 128 on-chip problem
constexpr int BJ_P = 2 * BJ_B;
constexpr int BJ_MAXJ = 128;      // pair-kernel jobs per launch

struct PairJob {
  float* A;      // current layout, N x N, row stride N
  float* Vbig;   // N x N; only the diagonal 128-blocks are written
  int32_t N;
  int32_t pair0;  // first global pair index of this job in the launch
  int32_t npairs;
  int32_t ident;  // pair index that is the identity this round, or -1
};
struct PairBatch {
  int n;
  float rel_tol, abs_tol;
  PairJob j[BJ_MAXJ];
};


// One CTA per pair: one-sided Jacobi (jacobi1s.cuh) of the 128 x 128 diagonal
// block, then the UBC column order + half swap, written into Vbig.
__global__ void __launch_bounds__(J1_THREADS) bj_pair_kernel(const __grid_constant__ PairBatch b) {
  extern __shared__ float sm[];
  constexpr int m = BJ_P, ld = BJ_P;
  float* U = sm;
  float* V = sm + m * ld;
  __shared__ float lam[BJ_P];
  __shared__ float wgt[BJ_P];
  __shared__ int dest[BJ_P];
  int q = 0;
  while (q + 1 < b.n && b.j[q + 1].pair0 <= static_cast<int>(blockIdx.x)) ++q;
  const PairJob& J = b.j[q];
  const int p = blockIdx.x - J.pair0;
  const int64_t N = J.N;
  const int64_t base = static_cast<int64_t>(p) * BJ_P * (N + 1);  // diagonal block (p, p)
  float* vout = J.Vbig + base;
  if (p == J.ident) {  // the two ends of the line: identity, no swap
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = e / m, c = e - (e / m) * m;
      vout[i * N + c] = (i == c) ? 1.0f : 0.0f;
    }
    return;
  }
  const float* src = J.A + base;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int c = e / m, r = e - (e / m) * m;
    U[c * ld + r] = 0.5f * (src[r * N + c] + src[c * N + r]);
    V[c * ld + r] = (r == c) ? 1.0f : 0.0f;
  }
  __syncthreads();
  onesided_jacobi(U, V, ld, m, m, b.rel_tol, lam);
  // UBC order: weight of each eigenvector column in the first block (rows 0..63);
  // the 64 heaviest continue block 1 and move to slot 2 (the swap), the rest go to
  // slot 1; original column order within each half
  {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int c = warp; c < m; c += (J1_THREADS >> 5)) {
      float s1 = 0.f;
      for (int r = lane; r < BJ_B; r += 32) s1 = fmaf(V[c * ld + r], V[c * ld + r], s1);
      s1 = j1_warp_sum(s1);
      if (lane == 0) wgt[c] = s1;
    }
  }
  __syncthreads();
  if (threadIdx.x < m) {
    const int c = threadIdx.x;
    const float w = wgt[c];
    int rank = 0;
    for (int c2 = 0; c2 < m; ++c2) {
      const float w2 = wgt[c2];
      rank += (w2 > w) || (w2 == w && c2 < c);
    }
    dest[c] = rank < BJ_B ? 1 : 0;  // 1: first set (goes to slot 2)
  }
  __syncthreads();
  if (threadIdx.x < m) {
    const int c = threadIdx.x;
    const int mine = dest[c];
    int pos = 0;
    for (int c2 = 0; c2 < c; ++c2) pos += dest[c2] == mine;
    wgt[c] = __int_as_float(mine ? BJ_B + pos : pos);  // reuse: output column of c
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int r = e / m, c = e - (e / m) * m;
    vout[r * N + __float_as_int(wgt[c])] = V[c * ld + r];
  }
}

// A = pad(sym(src)), Q = I, Vbig = 0 (N x N each).  grid (blocks over rows, jobs)
struct InitJob {
  const float* src;
  float* A;
  float* Q;
  float* Vbig;
  int32_t n, N;
};
struct InitBatch {
  int n;
  InitJob j[BJ_MAXJ];
};
__global__ void __launch_bounds__(256) bj_init_kernel(const __grid_constant__ InitBatch b) {
  const InitJob& J = b.j[blockIdx.y];
  const int n = J.n, N = J.N;
  for (int r = blockIdx.x; r < N; r += gridDim.x) {
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      const int64_t e = static_cast<int64_t>(r) * N + c;
      float a = 0.0f;
      if (r < n && c < n)
        a = 0.5f * (__ldg(J.src + static_cast<int64_t>(r) * n + c) + __ldg(J.src + static_cast<int64_t>(c) * n + r));
      J.A[e] = a;
      J.Q[e] = (r == c) ? 1.0f : 0.0f;
      J.Vbig[e] = 0.0f;
    }
  }
}

// Eigenvalues = diag(A), eigenvectors = columns of Q (current layout).  Columns
// whose mass lies on the padding coordinates are dropped; the rest are ranked by
// eigenvalue, descending (ties by column).  Two kernels: rank, then scatter.
struct ExtractJob {
  const float* A;
  const float* Q;
  float* q;       // n x n output
  float* w;       // n output
  int32_t* slot;  // N: output column of each current column, -1 = padding
  int32_t* pad;   // N scratch: 1 = padding column
  int32_t* info;
  int32_t n, N;
};
struct ExtractBatch {
  int n;
  ExtractJob j[BJ_MAXJ];
};
// padding columns are (exactly) unit vectors on the padding rows n..N-1
__global__ void __launch_bounds__(256) bj_padflag_kernel(const __grid_constant__ ExtractBatch b) {
  const ExtractJob& J = b.j[blockIdx.y];
  const int n = J.n, N = J.N;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  float pm = 0.0f;
  for (int r = n; r < N; ++r) {
    const float v = J.Q[static_cast<int64_t>(r) * N + c];
    pm = fmaf(v, v, pm);
  }
  J.pad[c] = pm > 0.5f ? 1 : 0;
}
__global__ void __launch_bounds__(256) bj_rank_kernel(const __grid_constant__ ExtractBatch b) {
  const ExtractJob& J = b.j[blockIdx.y];
  const int N = J.N;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  const int64_t NN = N;
  if (J.pad[c]) {
    J.slot[c] = -1;
    return;
  }
  const float wc = J.A[c * NN + c];
  int rank = 0;
  for (int c2 = 0; c2 < N; ++c2) {
    if (J.pad[c2]) continue;
    const float w2 = J.A[static_cast<int64_t>(c2) * NN + c2];
    rank += (w2 > wc) || (w2 == wc && c2 < c);
  }
  J.w[rank] = wc;
  if (!isfinite(wc) && J.info) *J.info = DPK_INFO_NONFINITE;
  J.slot[c] = rank;
}
__global__ void __launch_bounds__(256) bj_scatter_kernel(const __grid_constant__ ExtractBatch b) {
  const ExtractJob& J = b.j[blockIdx.y];
  const int n = J.n, N = J.N;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    const float* qrow = J.Q + static_cast<int64_t>(r) * N;
    float* out = J.q + static_cast<int64_t>(r) * n;
    for (int c = threadIdx.x; c < N; c += blockDim.x) {
      const int s = J.slot[c];
      if (s >= 0) {
        const float v = qrow[c];
        out[s] = v;
        if (!isfinite(v) && J.info) *J.info = DPK_INFO_NONFINITE;
      }
    }
  }
}

int eig_sweeps() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_EIG_SWEEPS");
    v = e ? std::max(1, atoi(e)) : 8;
  }
  return v;
}

inline int bj_blocks(int n) {
  int nb = (n + BJ_B - 1) / BJ_B;
  return nb + (nb & 1);
}

struct BjMat {
  const dpk_eig_job* job;
  int n, N, nb, rounds;
  float *A, *Bt, *Q[2], *Vbig;
  int32_t* slot;
};

size_t bj_matrix_bytes(int n) {
  const int N = bj_blocks(n) * BJ_B;
  return align_up(5 * static_cast<size_t>(N) * N * sizeof(float) + N * sizeof(int32_t) + 1024, 1024);
}

GemmSpec bj_spec(const dpk_operand& a, const dpk_operand& b, float* out, int64_t ldo) {
  GemmSpec s{};
  s.job.a = a;
  s.job.b = b;
  s.job.out = out;
  s.job.ldo = ldo;
  s.job.ldc = ldo;
  s.job.alpha = 1.0f;
  s.job.beta = 0.0f;
  s.epi = EPI_LINEAR;
  return s;
}

// out[:, (c + 64) mod N] = X[:, c] * (Vbig block column c): the +1 block shift of a
// column update, as (main, wrap) problems
void shifted_col_update(const float* X, const float* Vbig, float* out, int N, std::vector<GemmSpec>& g) {
  GemmSpec m = bj_spec(rows_k(X, N, N, N), rows_mn(Vbig, N - BJ_B, N, N), out + BJ_B, N);
  m.tri_b = TRI_BLOCK;
  g.push_back(m);
  const int64_t o = static_cast<int64_t>(N - BJ_P);
  g.push_back(bj_spec(rows_k(X + o, N, BJ_P, N), rows_mn(Vbig + o * N + (N - BJ_B), BJ_B, BJ_P, N), out, N));
}
// out[(r + 64) mod N, :] = (Vbig^T Bt)[r, :]
void shifted_row_update(const float* Bt, const float* Vbig, float* out, int N, std::vector<GemmSpec>& g) {
  GemmSpec m = bj_spec(rows_mn(Vbig, N - BJ_B, N, N), rows_mn(Bt, N, N, N), out + static_cast<int64_t>(BJ_B) * N, N);
  m.tri_a = TRI_BLOCK;
  g.push_back(m);
  const int64_t o = static_cast<int64_t>(N - BJ_P);
  g.push_back(bj_spec(rows_mn(Vbig + o * N + (N - BJ_B), BJ_B, BJ_P, N), rows_mn(Bt + o * N, N, BJ_P, N), out, N));
}

void plan_mats(const dpk_eig_job* jobs, const std::vector<int>& big, char* base, std::vector<BjMat>& mats) {
  size_t off = 0;
  for (int i : big) {
    BjMat M{};
    M.job = &jobs[i];
    M.n = jobs[i].n;
    M.nb = bj_blocks(M.n);
    M.N = M.nb * BJ_B;
    M.rounds = eig_sweeps() * M.nb;
    const size_t NN = static_cast<size_t>(M.N) * M.N;
    float* f = reinterpret_cast<float*>(base + off);
    M.A = f;
    M.Bt = f + NN;
    M.Q[0] = f + 2 * NN;
    M.Q[1] = f + 3 * NN;
    M.Vbig = f + 4 * NN;
    M.slot = reinterpret_cast<int32_t*>(f + 5 * NN);
    off += bj_matrix_bytes(M.n);
    mats.push_back(M);
  }
}

size_t bj_workspace_bytes(const dpk_eig_job* jobs, int n_jobs) {
  size_t mb = 0;
  for (int i = 0; i < n_jobs; ++i)
    if (jobs[i].n > 128) mb += bj_matrix_bytes(jobs[i].n);
  if (mb == 0) return 0;
  // GEMM workspace: scheduler counters only (block-diagonal problems never split K)
  return mb + 64 * 1024;
}

int bj_run(const dpk_eig_job* jobs, const std::vector<int>& big, void* workspace, size_t ws_bytes,
           cudaStream_t st) {
  std::vector<BjMat> mats;
  plan_mats(jobs, big, static_cast<char*>(workspace), mats);
  size_t used = 0;
  for (auto& M : mats) used += bj_matrix_bytes(M.n);
  char* gemm_ws = static_cast<char*>(workspace) + used;
  const size_t gemm_bytes = ws_bytes - used;
  static std::atomic<uint64_t> attr_on{0};
  const int pair_smem = 2 * BJ_P * BJ_P * 4;
  if (first_on_device(attr_on)) {
    cudaError_t e = cudaFuncSetAttribute(bj_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pair_smem);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(bj_pair_kernel)");
  }
  // init
  thread_local InitBatch ib;
  for (size_t first = 0; first < mats.size(); first += BJ_MAXJ) {
    const int cnt = static_cast<int>(std::min<size_t>(BJ_MAXJ, mats.size() - first));
    ib.n = cnt;
    int maxN = 0;
    for (int i = 0; i < cnt; ++i) {
      const BjMat& M = mats[first + i];
      ib.j[i] = InitJob{M.job->src, M.A, M.Q[0], M.Vbig, M.n, M.N};
      maxN = std::max(maxN, M.N);
    }
    bj_init_kernel<<<dim3(std::min(maxN, 1024), cnt), 256, 0, st>>>(ib);
    note_launch();
    int rc = cuda_status(cudaGetLastError(), "bj_init_kernel launch");
    if (rc) return rc;
  }
  int rc = cuda_status(cudaMemsetAsync(gemm_ws, 0, GEMM_SCHED_BYTES, st), "cudaMemsetAsync(counters)");
  if (rc) return rc;
  int max_rounds = 0;
  for (auto& M : mats) max_rounds = std::max(max_rounds, M.rounds);
  thread_local PairBatch pb;
  jac_tolerances(pb.rel_tol, pb.abs_tol);
  for (int r = 0; r < max_rounds; ++r) {
    // 1. pair eigenproblems of every active matrix
    pb.n = 0;
    int total_pairs = 0;
    auto flush_pairs = [&]() -> int {
      if (pb.n == 0) return DPK_OK;
      bj_pair_kernel<<<total_pairs, J1_THREADS, pair_smem, st>>>(pb);
      note_launch();
      pb.n = 0;
      total_pairs = 0;
      return cuda_status(cudaGetLastError(), "bj_pair_kernel launch");
    };
    for (auto& M : mats) {
      if (r >= M.rounds) continue;
      if (pb.n == BJ_MAXJ) {
        rc = flush_pairs();
        if (rc) return rc;
      }
      const int ident = (r & 1) ? ((r - 1) % M.nb) / 2 : -1;
      pb.j[pb.n++] = PairJob{M.A, M.Vbig, M.N, total_pairs, M.nb / 2, ident};
      total_pairs += M.nb / 2;
    }
    rc = flush_pairs();
    if (rc) return rc;
    // 2. column updates of A and Q (independent), then the row update of A
    std::vector<GemmSpec> g1, g2;
    for (auto& M : mats) {
      if (r >= M.rounds) continue;
      const int cur = r & 1;
      shifted_col_update(M.A, M.Vbig, M.Bt, M.N, g1);
      shifted_col_update(M.Q[cur], M.Vbig, M.Q[cur ^ 1], M.N, g1);
      shifted_row_update(M.Bt, M.Vbig, M.A, M.N, g2);
    }
    rc = gemm_launch(g1.data(), static_cast<int>(g1.size()), gemm_ws, gemm_bytes, DPK_PREC_3XTF32, st, false);
    if (rc) return rc;
    rc = gemm_launch(g2.data(), static_cast<int>(g2.size()), gemm_ws, gemm_bytes, DPK_PREC_3XTF32, st, false);
    if (rc) return rc;
  }
  // extract (Q lives in Q[rounds & 1])
  thread_local ExtractBatch eb;
  for (size_t first = 0; first < mats.size(); first += BJ_MAXJ) {
    const int cnt = static_cast<int>(std::min<size_t>(BJ_MAXJ, mats.size() - first));
    eb.n = cnt;
    int maxN = 0, maxn = 0;
    for (int i = 0; i < cnt; ++i) {
      const BjMat& M = mats[first + i];
      eb.j[i] = ExtractJob{M.A, M.Q[M.rounds & 1], M.job->q, M.job->w, M.slot,
                           reinterpret_cast<int32_t*>(M.Bt), M.job->info, M.n, M.N};
      maxN = std::max(maxN, M.N);
      maxn = std::max(maxn, M.n);
    }
    bj_padflag_kernel<<<dim3((maxN + 255) / 256, cnt), 256, 0, st>>>(eb);
    note_launch();
    rc = cuda_status(cudaGetLastError(), "bj_padflag_kernel launch");
    if (rc) return rc;
    bj_rank_kernel<<<dim3((maxN + 255) / 256, cnt), 256, 0, st>>>(eb);
    note_launch();
    rc = cuda_status(cudaGetLastError(), "bj_rank_kernel launch");
    if (rc) return rc;
    bj_scatter_kernel<<<dim3(std::min(maxn, 1024), cnt), 256, 0, st>>>(eb);
    note_launch();
    rc = cuda_status(cudaGetLastError(), "bj_scatter_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

// The whole call is replayed from a CUDA graph keyed by the job list, workspace
// and device (the rounds are ~3 launches each, thousands per call).
struct BjGraph {
  std::vector<char> key;
  cudaGraphExec_t exec;
  unsigned long long launches;
  unsigned long long last_use;
};

int bj_run_cached(const dpk_eig_job* jobs, const std::vector<int>& big, void* workspace, size_t ws_bytes,
                  cudaStream_t st) {
  static std::mutex mu;
  static std::vector<BjGraph> cache;
  static unsigned long long tick = 0;
  static std::vector<cudaStream_t> cap_streams;
  constexpr size_t CACHE_MAX = 8;
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  rc = cuda_status(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
  if (rc) return rc;
  if (cs != cudaStreamCaptureStatusNone) return bj_run(jobs, big, workspace, ws_bytes, st);
  std::vector<char> key;
  auto put = [&](const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    key.insert(key.end(), c, c + n);
  };
  for (int i : big) put(&jobs[i], sizeof(dpk_eig_job));
  put(&workspace, sizeof(void*));
  put(&ws_bytes, sizeof(size_t));
  put(&dev, sizeof(int));
  const int sw = eig_sweeps();
  put(&sw, sizeof(int));
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache) {
    if (e.key == key) {
      e.last_use = ++tick;
      rc = cuda_status(cudaGraphLaunch(e.exec, st), "cudaGraphLaunch(block Jacobi)");
      if (!rc) note_launches(e.launches);
      return rc;
    }
  }
  if (static_cast<int>(cap_streams.size()) <= dev) cap_streams.resize(dev + 1, nullptr);
  if (!cap_streams[dev]) {
    rc = cuda_status(cudaStreamCreateWithFlags(&cap_streams[dev], cudaStreamNonBlocking), "cudaStreamCreate");
    if (rc) return rc;
  }
  cudaStream_t cap = cap_streams[dev];
  const unsigned long long before = launch_counter();
  rc = cuda_status(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
  if (rc) return rc;
  rc = bj_run(jobs, big, workspace, ws_bytes, cap);
  cudaGraph_t graph = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(cap, &graph);
  const unsigned long long captured = launch_counter() - before;
  set_launch_counter(before);
  if (rc || ee != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    return rc ? rc : cuda_status(ee, "cudaStreamEndCapture");
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  rc = cuda_status(ie, "cudaGraphInstantiate(block Jacobi)");
  if (rc) return rc;
  if (cache.size() >= CACHE_MAX) {
    auto old = std::min_element(cache.begin(), cache.end(),
                                [](const BjGraph& a, const BjGraph& b) { return a.last_use < b.last_use; });
    cudaGraphExecDestroy(old->exec);
    cache.erase(old);
  }
  cache.push_back(BjGraph{std::move(key), exec, captured, ++tick});
  rc = cuda_status(cudaGraphLaunch(exec, st), "cudaGraphLaunch(block Jacobi)");
  if (!rc) note_launches(captured);
  return rc;
}

}  // namespace

// entry points used by syevd.cu
size_t syevj_workspace_bytes(const dpk_eig_job* jobs, int n_jobs) { return bj_workspace_bytes(jobs, n_jobs); }

int syevj_run(const dpk_eig_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, cudaStream_t st) {
  std::vector<int> big;
  for (int i = 0; i < n_jobs; ++i)
    if (jobs[i].n > 128) big.push_back(i);
  if (big.empty()) return DPK_OK;
  const size_t need = bj_workspace_bytes(jobs, n_jobs);
  if (workspace == nullptr || ws_bytes < need) {
    set_error("dpk_syevd_batched: workspace too small for n > 128 (see dpk_syevd_workspace_bytes)");
    return DPK_ENOSPACE;
  }
  const char* g = getenv("DPK_EIG_GRAPH");
  if (g && g[0] == '0') return bj_run(jobs, big, workspace, ws_bytes, st);
  return bj_run_cached(jobs, big, workspace, ws_bytes, st);
}

}  // namespace dpk
