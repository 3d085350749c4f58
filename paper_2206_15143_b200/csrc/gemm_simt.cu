// Latency path of the GEMM engine: batched FP32 (CUDA-core) GEMM for groups of
// small problems -- the deep rounds of the SPD recursion (blocks of 64..576),
// where a tcgen05 launch is dominated by its fixed costs (TMA descriptor fetch,
// stage hand-offs, TMEM round trip) rather than by math.  Same job semantics
// as the tensor-core engine (GemmSpec: alpha/beta/cin, symmetric lower tiles
// with or without the mirror, triangular K clipping); exact fp32 products, so
// it is at least as accurate as the 3xTF32 path it stands in for.
//
// One CTA per (problem, 64 x 64 or 32 x 32 output tile), 256 threads in a 16 x 16
// grid, 4 x 4 (2 x 2) outputs per thread; K in chunks of 32 staged through shared
// memory (k-major, so the inner loop reads two float4 per 16 FMAs) by cp.async in a
// SNS-stage ring: the loads of up to SNS-1 chunks ahead are in flight together, so
// a K <= 96 problem costs one global-load latency instead of one per chunk (these
// launches are latency-bound: 2M FMA spread over 16+ SMs).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <vector>

#include "dpk_internal.h"
#include "dpk_ptx.cuh"

namespace dpk {
namespace {

constexpr int SK = 32;       // K chunk
constexpr int SNS = 4;       // cp.async ring stages
constexpr int SMAXP = 192;

struct SimtProb {
  const float* a;
  const float* b;
  float* out;
  const float* cin;
  int64_t lda, ldb, ldo, ldc;
  float alpha, beta;
  int M, N, K;
  int a_mn, b_mn;  // 1: operand is ROWS_MN (element (r, k) at data[k * ld + r])
  int sym;         // 0 general, 1 lower tiles + mirror, 2 lower tiles only
  int tri_a, tri_b;
  int tiles_n;
  int tile_begin;
};
struct SimtBatch {
  int n;
  int total;
  SimtProb p[SMAXP];
};

__device__ __forceinline__ void tile_of(const SimtProb& P, int t, int& tm, int& tn) {
  if (P.sym) {
    int r = static_cast<int>((sqrtf(8.0f * t + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= t) ++r;
    while (r * (r + 1) / 2 > t) --r;
    tm = r;
    tn = t - r * (r + 1) / 2;
  } else {
    tm = t / P.tiles_n;
    tn = t - tm * P.tiles_n;
  }
}

// T/8 elements per thread of one T x 32 operand chunk (rows r0.., k k0..) copied to
// shared memory k-major (s[k][r]) by 4-byte cp.async; out-of-range elements are
// zero-filled (src-size 0, nothing read)
template <int T>
__device__ __forceinline__ void copy_chunk(float* s, const float* p, int64_t ld, int mn, int rows, int r0, int k0,
                                           int klo, int khi, int tid) {
  constexpr int SP = T + 4;
#pragma unroll
  for (int i = 0; i < T / 8; ++i) {
    const int idx = tid + 256 * i;
    const int r = mn ? idx % T : idx / SK;  // mn: coalesced along r, else along k
    const int k = mn ? idx / T : idx % SK;
    const int gr = r0 + r, gk = k0 + k;
    const bool ok = gr < rows && gk >= klo && gk < khi;
    const float* src = ok ? p + (mn ? static_cast<int64_t>(gk) * ld + gr : static_cast<int64_t>(gr) * ld + gk) : p;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(s + k * SP + r));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(ok ? 4 : 0) : "memory");
  }
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int T>
constexpr int simt_smem_bytes() {
  return 2 * SNS * SK * (T + 4) * 4;
}

// T x T output tile per CTA (T = 32 or 64), R x R outputs per thread
template <int T>
__global__ void __launch_bounds__(256, 1) simt_gemm_kernel(const __grid_constant__ SimtBatch bt) {
  constexpr int R = T / 16;
  constexpr int SP = T + 4;  // smem row stride: 16-byte aligned rows
  extern __shared__ __align__(16) float simt_smem[];
  float* As = simt_smem;                 // [SNS][SK * SP]
  float* Bs = simt_smem + SNS * SK * SP;  // [SNS][SK * SP]
  pdl_wait();
  pdl_trigger();
  int pi = 0;
  while (pi + 1 < bt.n && bt.p[pi + 1].tile_begin <= static_cast<int>(blockIdx.x)) ++pi;
  const SimtProb& P = bt.p[pi];
  int tm, tn;
  tile_of(P, blockIdx.x - P.tile_begin, tm, tn);
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = tm * T, n0 = tn * T;
  // K range where both operands can be nonzero (triangular structure)
  int klo = 0, khi = P.K;
  if (P.tri_a == TRI_UPPER) klo = max(klo, m0);
  if (P.tri_b == TRI_UPPER) klo = max(klo, n0);
  if (P.tri_a == TRI_LOWER) khi = min(khi, m0 + T);
  if (P.tri_b == TRI_LOWER) khi = min(khi, n0 + T);
  if (P.tri_a == TRI_BLOCK || P.tri_b == TRI_BLOCK) return;  // never planned here (simt_eligible)
  const int kstart = (klo / SK) * SK;
  const int nch = khi > kstart ? (khi - kstart + SK - 1) / SK : 0;
  float acc[R][R] = {};
  auto issue = [&](int c) {  // chunk c into stage c % SNS (an empty group past the end)
    if (c < nch) {
      const int st = c % SNS;
      copy_chunk<T>(As + st * SK * SP, P.a, P.lda, P.a_mn, P.M, m0, kstart + c * SK, klo, khi, tid);
      copy_chunk<T>(Bs + st * SK * SP, P.b, P.ldb, P.b_mn, P.N, n0, kstart + c * SK, klo, khi, tid);
    }
    cp_async_commit();
  };
#pragma unroll
  for (int c = 0; c < SNS - 1; ++c) issue(c);
  for (int c = 0; c < nch; ++c) {
    cp_async_wait<SNS - 2>();  // this thread's copies of chunk c have landed
    __syncthreads();           // everyone's have; stage (c - 1) % SNS is free again
    issue(c + SNS - 1);
    const float* as = As + (c % SNS) * SK * SP;
    const float* bs = Bs + (c % SNS) * SK * SP;
#pragma unroll 8
    for (int kk = 0; kk < SK; ++kk) {
      float ar[R], br[R];
      if constexpr (R == 4) {
        const float4 a4 = *reinterpret_cast<const float4*>(as + kk * SP + ty * 4);
        const float4 b4 = *reinterpret_cast<const float4*>(bs + kk * SP + tx * 4);
        ar[0] = a4.x; ar[1] = a4.y; ar[2] = a4.z; ar[3] = a4.w;
        br[0] = b4.x; br[1] = b4.y; br[2] = b4.z; br[3] = b4.w;
      } else {
        const float2 a2 = *reinterpret_cast<const float2*>(as + kk * SP + ty * 2);
        const float2 b2 = *reinterpret_cast<const float2*>(bs + kk * SP + tx * 2);
        ar[0] = a2.x; ar[1] = a2.y;
        br[0] = b2.x; br[1] = b2.y;
      }
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) acc[i][j] = fmaf(ar[i], br[j], acc[i][j]);
    }
  }
  cp_async_wait<0>();  // no copy may outlive the CTA
  // epilogue: alpha * acc + beta * cin; symmetric diagonal tiles keep gn <= gm
  const bool diag = P.sym == 1 && tm == tn;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int gm = m0 + ty * R + i;
    if (gm >= P.M) continue;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int gn = n0 + tx * R + j;
      if (gn >= P.N || (diag && gn > gm)) continue;
      float v = P.alpha * acc[i][j];
      if (P.beta != 0.0f) v = fmaf(P.beta, P.cin[static_cast<int64_t>(gm) * P.ldc + gn], v);
      P.out[static_cast<int64_t>(gm) * P.ldo + gn] = v;
      if (P.sym == 1 && gn != gm) P.out[static_cast<int64_t>(gn) * P.ldo + gm] = v;
    }
  }
}

int tiles_for(const GemmSpec& g, int T) {
  const int tmn = (g.job.a.rows + T - 1) / T;
  const int tn = (g.job.b.rows + T - 1) / T;
  return g.job.symmetric ? tmn * (tmn + 1) / 2 : tmn * tn;
}

}  // namespace

// Whole-group eligibility: every problem a plain 2-D view (rows_k / rows_mn,
// no bias row), linear epilogue, no transposed copy, and small enough that the
// group's math stays in the few-microsecond range.
bool simt_eligible(const GemmSpec* specs, int n, int precision) {
  if (precision != DPK_PREC_3XTF32 || n <= 0 || n > SMAXP) return false;
  double fma = 0.0;
  for (int i = 0; i < n; ++i) {
    const GemmSpec& g = specs[i];
    const dpk_operand& a = g.job.a;
    const dpk_operand& b = g.job.b;
    if (g.epi != EPI_LINEAR || g.out_t || g.alpha_amax || g.tri_a == TRI_BLOCK || g.tri_b == TRI_BLOCK) return false;
    for (const dpk_operand* o : {&a, &b})
      if ((o->kind != DPK_OPND_ROWS_K && o->kind != DPK_OPND_ROWS_MN) || o->bias_row) return false;
    if (a.rows > 640 || b.rows > 640 || a.cols > 640) return false;
    double f = static_cast<double>(a.rows) * b.rows * a.cols;
    if (g.job.symmetric) f *= 0.5;
    fma += f;
  }
  return fma <= simt_fma_limit();
}

double simt_fma_limit() {
  static double v = -1.0;
  if (v < 0.0) {
    const char* e = getenv("DPK_SIMT_FMA");
    v = e ? atof(e) : 5e7;  // re-tuned after the 3-pass producer fix (ResNet-50 N=1 6.75 -> 6.62 ms)
  }
  return v;
}

int simt_gemm_launch(const GemmSpec* specs, int n, cudaStream_t st) {
  // 64-wide tiles when they already give most SMs a CTA, else 32-wide (4x the CTAs)
  int t64 = 0;
  for (int i = 0; i < n; ++i) t64 += tiles_for(specs[i], 64);
  const int T = t64 >= num_sms() * 3 / 4 ? 64 : 32;
  thread_local SimtBatch bt;
  bt.n = n;
  int tiles = 0;
  for (int i = 0; i < n; ++i) {
    const GemmSpec& g = specs[i];
    SimtProb& P = bt.p[i];
    P.a = g.job.a.data;
    P.b = g.job.b.data;
    P.lda = g.job.a.ld;
    P.ldb = g.job.b.ld;
    P.a_mn = g.job.a.kind == DPK_OPND_ROWS_MN;
    P.b_mn = g.job.b.kind == DPK_OPND_ROWS_MN;
    P.out = g.job.out;
    P.cin = g.job.cin;
    P.ldo = g.job.ldo;
    P.ldc = g.job.ldc;
    P.alpha = g.job.alpha;
    P.beta = g.job.beta;
    P.M = g.job.a.rows;
    P.N = g.job.b.rows;
    P.K = static_cast<int>(g.job.a.cols);
    P.sym = g.job.symmetric ? (g.lower_only ? 2 : 1) : 0;
    P.tri_a = g.tri_a;
    P.tri_b = g.tri_b;
    P.tiles_n = (P.N + T - 1) / T;
    P.tile_begin = tiles;
    tiles += tiles_for(g, T);
    if (P.beta != 0.0f && P.cin == nullptr) {
      set_error("dpk_gemm: beta != 0 needs cin");
      return DPK_EARG;
    }
  }
  bt.total = tiles;
  if (tiles == 0) return DPK_OK;
  static std::atomic<uint64_t> configured_on{0};
  if (first_on_device(configured_on)) {
    cudaError_t e = cudaFuncSetAttribute(simt_gemm_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         simt_smem_bytes<64>());
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(simt_gemm_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               simt_smem_bytes<32>());
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(simt_gemm_kernel)");
  }
  const cudaError_t e = T == 64 ? launch_k(simt_gemm_kernel<64>, dim3(tiles), dim3(256), simt_smem_bytes<64>(), st, 1, bt)
                                : launch_k(simt_gemm_kernel<32>, dim3(tiles), dim3(256), simt_smem_bytes<32>(), st, 1, bt);
  note_launch();
  return cuda_status(e, "simt_gemm_kernel launch");
}

}  // namespace dpk
