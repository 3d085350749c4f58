// K5 / K6: preconditioning of the (aggregated) layer gradient on tcgen05.
//   inverse mode (kfac.py:251-254):  out = G_inv @ grad @ A_inv             2 GEMM phases
//   eigen mode   (kfac.py:174-191):  out = Q_G ((Q_G^T grad Q_A) / D) Q_A^T  4 GEMM phases,
//        D = max(v_G,0) max(v_A,0)^T + gamma divided out in the epilogue of phase 2.
// Every phase is ONE grouped launch over all owned layers.
#include <cuda_runtime.h>

#include <vector>

#include "dpk_internal.h"

namespace dpk {
namespace {

using Specs = std::vector<GemmSpec>;

GemmSpec lin(const dpk_operand& a, const dpk_operand& b, float* out, int64_t ldo) {
  GemmSpec s{};
  s.job.a = a;
  s.job.b = b;
  s.job.out = out;
  s.job.ldo = ldo;
  s.job.alpha = 1.0f;
  s.epi = EPI_LINEAR;
  return s;
}

bool check_jobs(const dpk_precond_job* jobs, int n, bool eigen) {
  if (n < 0 || (n > 0 && jobs == nullptr)) return false;
  for (int i = 0; i < n; ++i) {
    const dpk_precond_job& j = jobs[i];
    if (j.d_out < 1 || j.d_in < 1 || !j.grad || !j.a_mat || !j.g_mat || !j.out || !j.tmp) return false;
    if (eigen && (!j.a_vals || !j.g_vals)) return false;
    if (j.out == j.grad || j.tmp == j.grad) return false;
  }
  return true;
}

void inverse_phases(const dpk_precond_job* J, int n, Specs& p1, Specs& p2) {
  for (int i = 0; i < n; ++i) {
    const int o = J[i].d_out, d = J[i].d_in;
    // tmp = grad @ A_inv   (A_inv symmetric: B[n][k] = A_inv[n][k])
    p1.push_back(lin(rows_k(J[i].grad, o, d, d), rows_k(J[i].a_mat, d, d, d), J[i].tmp, d));
    // out = G_inv @ tmp    (B[n][k] = tmp[k][n])
    p2.push_back(lin(rows_k(J[i].g_mat, o, o, o), rows_mn(J[i].tmp, d, o, d), J[i].out, d));
  }
}

void eigen_phases(const dpk_precond_job* J, int n, float gamma, Specs (&p)[4]) {
  for (int i = 0; i < n; ++i) {
    const int o = J[i].d_out, d = J[i].d_in;
    // T1 = grad Q_A -> tmp
    p[0].push_back(lin(rows_k(J[i].grad, o, d, d), rows_mn(J[i].a_mat, d, d, d), J[i].tmp, d));
    // R = (Q_G^T T1) / D -> out
    GemmSpec s = lin(rows_mn(J[i].g_mat, o, o, o), rows_mn(J[i].tmp, d, o, d), J[i].out, d);
    s.epi = EPI_EIGDIV;
    s.vrow = J[i].g_vals;
    s.vcol = J[i].a_vals;
    s.gamma = gamma;
    p[1].push_back(s);
    // T2 = R Q_A^T -> tmp
    p[2].push_back(lin(rows_k(J[i].out, o, d, d), rows_k(J[i].a_mat, d, d, d), J[i].tmp, d));
    // out = Q_G T2
    p[3].push_back(lin(rows_k(J[i].g_mat, o, o, o), rows_mn(J[i].tmp, d, o, d), J[i].out, d));
  }
}

// out = X_G^T (X_G (grad X_A^T) X_A), phases alternating between tmp and out
void factored_phases(const dpk_precond_factor_job* J, int n, Specs (&p)[4]) {
  for (int i = 0; i < n; ++i) {
    const int o = J[i].d_out, d = J[i].d_in;
    // P1 = grad X_A^T -> tmp:  B[j][k] = X_A[j][k], zero for k > j
    GemmSpec s = lin(rows_k(J[i].grad, o, d, d), rows_k(J[i].xa, d, d, J[i].ldxa), J[i].tmp, d);
    s.tri_b = TRI_LOWER;
    p[0].push_back(s);
    // P2 = P1 X_A -> out:  B[j][k] = X_A[k][j], zero for k < j
    s = lin(rows_k(J[i].tmp, o, d, d), rows_mn(J[i].xa, d, d, J[i].ldxa), J[i].out, d);
    s.tri_b = TRI_UPPER;
    p[1].push_back(s);
    // P3 = X_G P2 -> tmp:  A = X_G (zero for k > i), B[j][k] = P2[k][j]
    s = lin(rows_k(J[i].xg, o, o, J[i].ldxg), rows_mn(J[i].out, d, o, d), J[i].tmp, d);
    s.tri_a = TRI_LOWER;
    p[2].push_back(s);
    // out = X_G^T P3:  A[i][k] = X_G[k][i] (zero for k < i), B[j][k] = P3[k][j]
    s = lin(rows_mn(J[i].xg, o, o, J[i].ldxg), rows_mn(J[i].tmp, d, o, d), J[i].out, d);
    s.tri_a = TRI_UPPER;
    p[3].push_back(s);
  }
}

bool check_factor_jobs(const dpk_precond_factor_job* jobs, int n) {
  if (n < 0 || (n > 0 && jobs == nullptr)) return false;
  for (int i = 0; i < n; ++i) {
    const dpk_precond_factor_job& j = jobs[i];
    if (j.d_out < 1 || j.d_in < 1 || !j.grad || !j.xa || !j.xg || !j.out || !j.tmp) return false;
    if (j.ldxa < j.d_in || j.ldxg < j.d_out || j.out == j.grad || j.tmp == j.grad || j.out == j.tmp) return false;
  }
  return true;
}

// min over the clamped outer product + gamma = max(min v_G,0) * max(min v_A,0) + gamma
// (values are descending, so the minimum is the last entry).
constexpr int DEN_MAX = 512;
struct DenBatch {
  int n;
  float gamma;
  const float* va[DEN_MAX];
  const float* vg[DEN_MAX];
  int da[DEN_MAX];
  int dg[DEN_MAX];
  int32_t* info[DEN_MAX];
};
__global__ void eig_denom_check(const __grid_constant__ DenBatch b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.n) return;
  const float ma = fmaxf(b.va[i][b.da[i] - 1], 0.0f);
  const float mg = fmaxf(b.vg[i][b.dg[i] - 1], 0.0f);
  if (!(ma * mg + b.gamma > 0.0f) && b.info[i]) *b.info[i] = DPK_INFO_EIG_DENOM;
}

}  // namespace
}  // namespace dpk

extern "C" {

size_t dpk_precond_workspace_bytes(const dpk_precond_job* jobs, int n_jobs) {
  if (!dpk::check_jobs(jobs, n_jobs, false) || n_jobs == 0) return 0;
  dpk::Specs p[4];
  dpk::eigen_phases(jobs, n_jobs, 0.0f, p);
  size_t w = 0;
  for (auto& s : p) w = std::max(w, dpk::gemm_workspace_bytes(s.data(), static_cast<int>(s.size())));
  return w;
}

int dpk_precond_inverse(const dpk_precond_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, int precision,
                        dpk_stream_t stream) {
  if (!dpk::check_jobs(jobs, n_jobs, false)) {
    dpk::set_error("dpk_precond_inverse: invalid job list");
    return DPK_EARG;
  }
  if (n_jobs == 0) return DPK_OK;
  dpk::Specs p1, p2;
  dpk::inverse_phases(jobs, n_jobs, p1, p2);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = dpk::gemm_launch(p1.data(), n_jobs, workspace, ws_bytes, precision, st);
  if (rc) return rc;
  return dpk::gemm_launch(p2.data(), n_jobs, workspace, ws_bytes, precision, st, false);
}

size_t dpk_precond_factor_workspace_bytes(const dpk_precond_factor_job* jobs, int n_jobs) {
  if (!dpk::check_factor_jobs(jobs, n_jobs) || n_jobs == 0) return 0;
  dpk::Specs p[4];
  dpk::factored_phases(jobs, n_jobs, p);
  size_t w = 0;
  for (auto& s : p) w = std::max(w, dpk::gemm_workspace_bytes(s.data(), static_cast<int>(s.size())));
  return w;
}

int dpk_precond_factored(const dpk_precond_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                         int precision, dpk_stream_t stream) {
  if (!dpk::check_factor_jobs(jobs, n_jobs)) {
    dpk::set_error("dpk_precond_factored: invalid job list");
    return DPK_EARG;
  }
  if (n_jobs == 0) return DPK_OK;
  dpk::Specs p[4];
  dpk::factored_phases(jobs, n_jobs, p);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  bool first = true;
  for (auto& s : p) {
    int rc = dpk::gemm_launch(s.data(), n_jobs, workspace, ws_bytes, precision, st, first);
    if (rc) return rc;
    first = false;
  }
  return DPK_OK;
}

int dpk_precond_eigen(const dpk_precond_job* jobs, int n_jobs, float gamma, void* workspace, size_t ws_bytes,
                      int precision, dpk_stream_t stream) {
  if (!dpk::check_jobs(jobs, n_jobs, true) || !(gamma >= 0.0f)) {
    dpk::set_error("dpk_precond_eigen: invalid job list");
    return DPK_EARG;
  }
  if (n_jobs == 0) return DPK_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  thread_local dpk::DenBatch db;
  for (int first = 0; first < n_jobs; first += dpk::DEN_MAX) {
    const int cnt = std::min(dpk::DEN_MAX, n_jobs - first);
    db.n = cnt;
    db.gamma = gamma;
    for (int i = 0; i < cnt; ++i) {
      db.va[i] = jobs[first + i].a_vals;
      db.vg[i] = jobs[first + i].g_vals;
      db.da[i] = jobs[first + i].d_in;
      db.dg[i] = jobs[first + i].d_out;
      db.info[i] = jobs[first + i].info;
    }
    dpk::eig_denom_check<<<(cnt + 127) / 128, 128, 0, st>>>(db);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "eig_denom_check launch");
    if (rc) return rc;
  }
  dpk::Specs p[4];
  dpk::eigen_phases(jobs, n_jobs, gamma, p);
  bool first = true;
  for (auto& s : p) {
    int rc = dpk::gemm_launch(s.data(), n_jobs, workspace, ws_bytes, precision, st, first);
    if (rc) return rc;
    first = false;
  }
  return DPK_OK;
}

}  // extern "C"
