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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "dpk_internal.h"
#include "dpk_ptx.cuh"

namespace dpk {
namespace {

constexpr int LEAF_N = 128;
constexpr int LEAF_THREADS = 512;  // 16 x 32 thread grid
constexpr int LEAF_MAX = 256;

struct LeafJob {
  const float* src;    // input block (row stride lds)
  float* dst;          // TRI: X = L^-1 block (lower, zeros above); FULL: the inverse
  const float* shift;  // FULL mode: damping added to the diagonal (may be null)
  int64_t lds;
  int64_t ldd;
  int32_t n;
  int32_t full;        // 1: whole matrix -> inverse; 0: diagonal block -> L^-1; 2: whole matrix -> L^-1
  int32_t fail_code;
  int32_t _pad;
  int32_t* info;
};
struct LeafBatch {
  int n;
  int skip_done;  // phase 3 skips the finished rows of the current row block
  LeafJob j[LEAF_MAX];
};

// Register-resident leaf.  The (padded) N x N block, N = 16*RB, is spread over a
// 16 x 32 grid of 512 threads with strided ownership: thread (ty, tx) owns rows
// ty + 16r (r < RB) and columns tx + 32c (c < RB/2).  A warp is one ty and 32
// consecutive tx, so column-vector reads are conflict-free and row-vector
// reads are broadcasts; the work stays balanced as the trailing block shrinks.
// One fused sweep does both
//   right-looking Cholesky      A[i][j] -= L[i][k] L[j][k]            (i, j > k)
//   right-looking L^-1 (trtri)  X[i][:] -= L[i][k] X[k][:] / L[k][k]  (i > k)
// four columns k..k+3 per step, in three phases separated by two barriers:
//   1. the owners publish the raw columns k..k+3 of A and rows k..k+3 of X;
//   2. thread i < N turns row i of the column panel into L[i][k..k+3] (forward
//      substitution with the 4x4 pivot block, which each of these threads
//      factors itself), thread N + j turns column j of the X rows into the
//      finished X[k..k+3][j]; both are published (zero where they do not apply);
//   3. every thread applies the rank-4 updates to its registers, reading the
//      published L / X values as float4 broadcasts.
// Only lower-triangle blocks of A are updated (blocks entirely above the
// diagonal are skipped at compile time; the 16-row block index kr is
// unrolled), so the upper triangle of the input is never read.  Padding
// rows/columns are the identity, so pivots past n are 1 and the real n x n
// result is unaffected.
#ifdef DPK_LEAF_PROF
__device__ unsigned long long g_leaf_prof[12];
#endif
template <int RB, int W>
__global__ void __launch_bounds__(LEAF_THREADS, 1) spd_leaf_kernel(const __grid_constant__ LeafBatch b) {
  constexpr int N = 16 * RB;
  constexpr int CB = RB / 2 > 0 ? RB / 2 : 1;
  constexpr int LDX = N + 1;
  constexpr int W4 = W / 4;  // float4s per published panel row
  extern __shared__ float smem[];
  float4* colb = reinterpret_cast<float4*>(smem);  // [N][W/4] raw A[i][k..k+W)
  float4* rowb = colb + N * W4;                    // [N][W/4] raw X[k..k+W)[j]
  float4* lpan = rowb + N * W4;                    // [N][W/4] L[i][k..k+W) (0 for i < k+W)
  float4* xrow = lpan + N * W4;                    // [N][W/4] finished X[k..k+W)[j] (0 for j >= k+W)
  float* Xs = smem + 4 * N * W;                    // [N][N+1] X for the FULL-mode X^T X
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  pdl_wait();
  pdl_trigger();
  const LeafJob& J = b.j[blockIdx.x];
  const int n = J.n;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const float sh = (J.full && J.shift) ? *J.shift : 0.0f;
  const float* src = J.src;
  const int64_t lds = J.lds;
  float a[RB][CB], x[RB][CB];
  // unconditional loads (padding reads element 0 and is replaced afterwards):
  // all RB*CB loads are in flight together instead of one branch-guarded
  // round trip each
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int i = ty + 16 * r, j = tx + 32 * c;
      const bool in = i < n && j < n;
      a[r][c] = __ldg(src + (in ? static_cast<int64_t>(i) * lds + j : 0));
    }
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int i = ty + 16 * r, j = tx + 32 * c;
      const bool in = i < n && j < n;
      a[r][c] = in ? a[r][c] + ((i == j) ? sh : 0.0f) : ((i == j) ? 1.0f : 0.0f);
      x[r][c] = (i == j) ? 1.0f : 0.0f;
    }
#pragma unroll
  for (int kr = 0; kr < RB; ++kr) {
    const int kc = kr / 2;  // column block holding k (compile-time after unrolling)
#pragma unroll 1
    for (int kq = 0; kq < 16 / W; ++kq) {
      const int k = 16 * kr + W * kq;
#ifdef DPK_LEAF_PROF
      long long c0 = clock64();
#endif
      // ---- phase 1: publish raw columns k..k+W-1 (rows >= 16 kr) and X rows k..k+W-1
      const int tcol = tx - (k & 31), trow = ty - (k & 15);
      if (tcol >= 0 && tcol < W) {
        float* cf = reinterpret_cast<float*>(colb);
#pragma unroll
        for (int r = kr; r < RB; ++r) cf[(ty + 16 * r) * W + tcol] = a[r][kc];
      }
      if (trow >= 0 && trow < W) {
        float* rf = reinterpret_cast<float*>(rowb);
#pragma unroll
        for (int c = 0; c <= kc; ++c) rf[(tx + 32 * c) * W + trow] = x[kr][c];
      }
#ifdef DPK_LEAF_PROF
      long long c1 = clock64();
#endif
      __syncthreads();
#ifdef DPK_LEAF_PROF
      long long c2 = clock64();
#endif
      // ---- phase 2: pivot block (each worker factors it itself), L panel rows,
      // finished X rows
      if (tid < 2 * N) {
        const float* cf = reinterpret_cast<const float*>(colb);
        float L[W][W], inv[W];
        bool ok = true;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          float d = cf[(k + j) * W + j];
#pragma unroll
          for (int t = 0; t < j; ++t) d = fmaf(-L[j][t], L[j][t], d);
          inv[j] = rsqrtf(d);
          ok = ok && d > 0.0f && isfinite(inv[j]);
#pragma unroll
          for (int m = j + 1; m < W; ++m) {
            float v = cf[(k + m) * W + j];
#pragma unroll
            for (int t = 0; t < j; ++t) v = fmaf(-L[m][t], L[j][t], v);
            L[m][j] = v * inv[j];
          }
        }
        if (!ok && tid == 0) s_fail = 1;  // uniform: every phase-2 thread factored the same block
        const int row = tid < N ? tid : tid - N;
        float v[W];
        const float4* srcp = (tid < N ? colb : rowb) + row * W4;
#pragma unroll
        for (int q = 0; q < W4; ++q) {
          const float4 t4 = srcp[q];
          v[4 * q] = t4.x;
          v[4 * q + 1] = t4.y;
          v[4 * q + 2] = t4.z;
          v[4 * q + 3] = t4.w;
        }
        float o[W];
        // row i of the panel (i >= k+W): forward substitution against L^T;
        // column j of the X rows (j < k+W): forward substitution against L
        const bool live = tid < N ? row >= k + W : row < k + W;
#pragma unroll
        for (int t = 0; t < W; ++t) {
          float y = v[t];
#pragma unroll
          for (int u = 0; u < t; ++u) y = fmaf(-o[u], L[t][u], y);
          o[t] = y * inv[t];
        }
        float4* dstp = (tid < N ? lpan : xrow) + row * W4;
#pragma unroll
        for (int q = 0; q < W4; ++q)
          dstp[q] = live ? make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3])
                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#ifdef DPK_LEAF_PROF
      long long c3 = clock64();
#endif
      __syncthreads();
#ifdef DPK_LEAF_PROF
      long long c4 = clock64();
#endif
      if (s_fail) {  // a non-positive pivot: exactly where cho_factor raises
        if (tid == 0 && J.info) *J.info = J.fail_code;
        return;
      }
      const bool skip_done = b.skip_done;
      // ---- phase 3: rank-W updates (lower-triangle blocks of A; X columns < k+W).
      // Column-outer: each thread's column vectors (lane-distinct, 4 smem wavefronts
      // per float4) are loaded once per step; the row vectors are warp-uniform
      // broadcasts (1 wavefront) and are re-read per column block.
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        const bool acol = c >= kc;   // A columns >= k (compile-time per kr, c)
        const bool xcol = c <= kc;   // X columns <= k+W-1
        float cv[W];
#pragma unroll
        for (int q = 0; q < W4; ++q) {
          const float4 t4 = acol && !xcol ? lpan[(tx + 32 * c) * W4 + q] : xcol && !acol ? xrow[(tx + 32 * c) * W4 + q]
                                                                                         : lpan[(tx + 32 * c) * W4 + q];
          cv[4 * q] = t4.x;
          cv[4 * q + 1] = t4.y;
          cv[4 * q + 2] = t4.z;
          cv[4 * q + 3] = t4.w;
        }
        float xv[W];
        if (acol && xcol) {  // c == kc: both an A and an X column block
#pragma unroll
          for (int q = 0; q < W4; ++q) {
            const float4 t4 = xrow[(tx + 32 * c) * W4 + q];
            xv[4 * q] = t4.x;
            xv[4 * q + 1] = t4.y;
            xv[4 * q + 2] = t4.z;
            xv[4 * q + 3] = t4.w;
          }
        }
#pragma unroll
        for (int r = kr; r < RB; ++r) {
          if (RB > 2 && r <= 2 * c - 1) continue;  // block entirely above the diagonal
          // this warp's row of block kr is finished (L[i][k..k+W) = 0: the updates are
          // exact no-ops): skip it (warp-uniform; DPK_LEAF_SKIP=0 keeps the FMAs)
          if (r == kr && skip_done && ty < W * kq + W) continue;
          float lr[W];
#pragma unroll
          for (int q = 0; q < W4; ++q) {
            const float4 t4 = lpan[(ty + 16 * r) * W4 + q];
            lr[4 * q] = t4.x;
            lr[4 * q + 1] = t4.y;
            lr[4 * q + 2] = t4.z;
            lr[4 * q + 3] = t4.w;
          }
          if (acol) {
            float v = a[r][c];
#pragma unroll
            for (int t = 0; t < W; ++t) v = fmaf(-lr[t], cv[t], v);
            a[r][c] = v;
          }
          if (xcol) {
            const float* xs = acol ? xv : cv;
            float v = x[r][c];
#pragma unroll
            for (int t = 0; t < W; ++t) v = fmaf(-lr[t], xs[t], v);
            x[r][c] = v;
          }
        }
      }
#ifdef DPK_LEAF_PROF
      long long c5 = clock64();
      if (blockIdx.x == 0 && (tid == 0 || tid == 511)) {
        unsigned long long* g = g_leaf_prof + (tid ? 6 : 0);
        atomicAdd(g + 0, c1 - c0); atomicAdd(g + 1, c2 - c1); atomicAdd(g + 2, c3 - c2);
        atomicAdd(g + 3, c4 - c3); atomicAdd(g + 4, c5 - c4); atomicAdd(g + 5, 1ull);
      }
#endif
      if (trow >= 0 && trow < W) {  // rows k..k+W-1 of X are final
        const float* xf = reinterpret_cast<const float*>(xrow);
#pragma unroll
        for (int c = 0; c <= kc; ++c) x[kr][c] = xf[(tx + 32 * c) * W + trow];
      }
    }
  }
  float* dst = J.dst;
  const int64_t ldd = J.ldd;
  if (J.full != 1) {  // X = L^-1: exactly zero above the diagonal by construction
#pragma unroll
    for (int r = 0; r < RB; ++r)
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        const int i = ty + 16 * r, j = tx + 32 * c;
        if (i < n && j < n) dst[static_cast<int64_t>(i) * ldd + j] = x[r][c];
      }
    return;
  }
  // ---- inverse = X^T X  (X[k][i] == 0 for k < i: 16-row block kr meets r <= kr, c <= kr/2)
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int c = 0; c < CB; ++c) Xs[(ty + 16 * r) * LDX + tx + 32 * c] = x[r][c];
  __syncthreads();
  float acc[RB][CB];
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int c = 0; c < CB; ++c) acc[r][c] = 0.0f;
#pragma unroll
  for (int kr = 0; kr < RB; ++kr) {
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      const float* row = Xs + (16 * kr + kk) * LDX;
      float xi[RB], xj[CB];
#pragma unroll
      for (int r = 0; r <= kr; ++r) xi[r] = row[ty + 16 * r];
#pragma unroll
      for (int c = 0; c <= kr / 2; ++c) xj[c] = row[tx + 32 * c];
#pragma unroll
      for (int r = 0; r <= kr; ++r)
#pragma unroll
        for (int c = 0; c <= kr / 2; ++c) acc[r][c] = fmaf(xi[r], xj[c], acc[r][c]);
    }
  }
#pragma unroll
  for (int r = 0; r < RB; ++r)
#pragma unroll
    for (int c = 0; c < CB; ++c) {
      const int i = ty + 16 * r, j = tx + 32 * c;
      if (i < n && j < n) dst[static_cast<int64_t>(i) * ldd + j] = acc[r][c];
    }
}

// ---- tensor-core leaf (TRI mode, n <= 128): the same fused right-looking Cholesky +
// L^-1 sweep, 8 columns per step, with the rank-8 updates of the trailing A block and
// of the X rows below the panel as mma.sync m16n8k8 TF32 products in 3xTF32 form
// (hi*hi + hi*lo + lo*hi: fp32-grade).  A and X live in registers as 16x8 accumulator
// tiles (lower tiles only: 72 + 72, nine per warp, tile w + 16j of warp w); per step
//   1. owners publish A's column block k..k+7 (Pan) and X's rows k..k+7 (XR);
//   2. threads 0-127 / 128-255 each factor the 8x8 pivot block themselves and form a
//      panel row L[i][k..k+7] = A[i][k..k+7] L_kk^-T (LP) / a column of the finished
//      X rows L_kk^-1 XR (XRn);
//   3. every warp updates its active tiles: A -= LP LP^T, X -= LP XRn, and copies
//      the finished X rows.
// 16 steps x 2 barriers; the SIMT leaf needs 32 x 2 and ~4x the instructions.
constexpr int LM_THREADS = 512;
constexpr int LM_PS = 12;    // Pan / LP row stride (floats): conflict-free fragment loads
constexpr int LM_XS = 136;   // XR / XRn row stride
__device__ __forceinline__ uint32_t lm_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void lm_split(float x, uint32_t& hi, uint32_t& lo) {
  hi = lm_tf32(x);
  lo = lm_tf32(x - __uint_as_float(hi));
}
__device__ __forceinline__ void lm_mma(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                       uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// lower tile index -> (tile row tr: 16 rows, tile column tc: 8 columns), tc <= 2 tr + 1
__device__ __forceinline__ void lm_tile(int i, int& tr, int& tc) {
  int r = static_cast<int>((sqrtf(4.0f * i + 1.0f) - 1.0f) * 0.5f);
  while ((r + 1) * (r + 2) <= i) ++r;
  while (r * (r + 1) > i) --r;
  tr = r;
  tc = i - r * (r + 1);
}

__global__ void __launch_bounds__(LM_THREADS, 1) spd_leaf_mma_kernel(const __grid_constant__ LeafBatch b) {
  __shared__ float Pan[128 * LM_PS];
  __shared__ uint32_t LPh[128 * LM_PS], LPl[128 * LM_PS];     // panel rows, TF32 hi / lo
  __shared__ float XR[8 * LM_XS];
  __shared__ float XRn[8 * LM_XS];                            // finished X rows
  __shared__ uint32_t XNh[8 * LM_XS], XNl[8 * LM_XS];         // -XRn, TF32 hi / lo
  __shared__ int s_fail;
  if (threadIdx.x == 0) s_fail = 0;
  pdl_wait();
  pdl_trigger();
  const LeafJob& J = b.j[blockIdx.x];
  const int n = J.n;
  const float* src = J.src;
  const int64_t lds = J.lds;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  // tiles j = 0..8 of this warp: global index w + 16 j; < 72 an A tile, else an X tile
  float acc[9][4];
  int ttr[9], ttc[9];
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    const int id = warp + 16 * j;
    const bool isa = id < 72;
    lm_tile(isa ? id : id - 72, ttr[j], ttc[j]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = 16 * ttr[j] + g + 8 * (e >> 1), c = 8 * ttc[j] + 2 * t4 + (e & 1);
      float v = (r == c) ? 1.0f : 0.0f;
      if (isa && r < n && c < n) v = __ldg(src + static_cast<int64_t>(r) * lds + c);
      acc[j][e] = v;
    }
  }
  for (int k = 0; k < 128; k += 8) {
    const int kc = k >> 3;
#ifdef DPK_LEAF_PROF
    long long c0 = clock64();
#endif
    // ---- 1. publish column block kc of A (rows >= k) and X rows k..k+7
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const bool isa = warp + 16 * j < 72;
      const int r0 = 16 * ttr[j];
      if (isa && ttc[j] == kc && r0 + 15 >= k) {
#pragma unroll
        for (int e = 0; e < 4; ++e) Pan[(r0 + g + 8 * (e >> 1)) * LM_PS + 2 * t4 + (e & 1)] = acc[j][e];
      }
      if (!isa && r0 == (k & ~15) && ttc[j] <= kc) {
        const bool h = (k >> 3) & 1;  // which 8-row half of the tile holds rows k..k+7
        XR[g * LM_XS + 8 * ttc[j] + 2 * t4] = h ? acc[j][2] : acc[j][0];  // (no dynamic register index)
        XR[g * LM_XS + 8 * ttc[j] + 2 * t4 + 1] = h ? acc[j][3] : acc[j][1];
      }
    }
#ifdef DPK_LEAF_PROF
    long long c1 = clock64();
#endif
    __syncthreads();
#ifdef DPK_LEAF_PROF
    long long c2 = clock64();
#endif
    // ---- 2. pivot block, panel rows, finished X rows
    if (tid < 256) {
      float L[8][8], inv[8];
      bool ok = true;
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        float d = Pan[(k + jj) * LM_PS + jj];
#pragma unroll
        for (int q = 0; q < jj; ++q) d = fmaf(-L[jj][q], L[jj][q], d);
        inv[jj] = rsqrtf(d);
        ok = ok && d > 0.0f && isfinite(inv[jj]);
#pragma unroll
        for (int m = jj + 1; m < 8; ++m) {
          float v = Pan[(k + m) * LM_PS + jj];
#pragma unroll
          for (int q = 0; q < jj; ++q) v = fmaf(-L[m][q], L[jj][q], v);
          L[m][jj] = v * inv[jj];
        }
      }
      if (!ok && tid == 0) s_fail = 1;
      // Linv = L^-1 (lower): column c by forward substitution
      float Li[8][8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r < c) {
            Li[r][c] = 0.0f;
          } else if (r == c) {
            Li[r][c] = inv[r];
          } else {
            float v = 0.0f;
#pragma unroll
            for (int q = c; q < r; ++q) v = fmaf(L[r][q], Li[q][c], v);
            Li[r][c] = -v * inv[r];
          }
        }
      }
      if (tid < 128) {  // panel row i: L[i][k..k+7] = A[i][k..k+7] L_kk^-T (zero above the panel)
        const int i = tid;
        float a[8], o[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = Pan[i * LM_PS + q];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float v = 0.0f;
#pragma unroll
          for (int m = 0; m <= q; ++m) v = fmaf(a[m], Li[q][m], v);
          o[q] = v;
        }
        const bool live = i >= k + 8;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          uint32_t hi, lo;
          lm_split(live ? o[q] : 0.0f, hi, lo);
          LPh[i * LM_PS + q] = hi;
          LPl[i * LM_PS + q] = lo;
        }
      } else {  // finished X rows, column jc: XRn[a][jc] = sum_m Linv[a][m] XR[m][jc]
        const int jc = tid - 128;
        if (jc < k + 8) {
          float xr[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) xr[q] = XR[q * LM_XS + jc];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            float v = 0.0f;
#pragma unroll
            for (int m = 0; m <= a; ++m) v = fmaf(Li[a][m], xr[m], v);
            XRn[a * LM_XS + jc] = v;
            uint32_t hi, lo;
            lm_split(-v, hi, lo);
            XNh[a * LM_XS + jc] = hi;
            XNl[a * LM_XS + jc] = lo;
          }
        }
      }
    }
#ifdef DPK_LEAF_PROF
    long long c3 = clock64();
#endif
    __syncthreads();
#ifdef DPK_LEAF_PROF
    long long c4 = clock64();
#endif
    if (s_fail) {  // a non-positive pivot: exactly where cho_factor raises
      if (tid == 0 && J.info) *J.info = J.fail_code;
      return;
    }
    // ---- 3. rank-8 updates on the tensor cores
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      const bool isa = warp + 16 * j < 72;
      const int r0 = 16 * ttr[j], c0 = 8 * ttc[j];
      if (r0 + 15 < k + 8) continue;  // no row below the panel
      if (isa ? (c0 + 7 < k + 8) : (ttc[j] > kc)) continue;  // finished A columns / X columns >= k+8
      // A fragment: LP rows r0+g / r0+g+8, k-columns t4 / t4+4 (pre-split TF32 hi / lo)
      const int ia = (r0 + g) * LM_PS + t4, ib = ia + 8 * LM_PS;
      const uint32_t ah0 = LPh[ia], ah1 = LPh[ib], ah2 = LPh[ia + 4], ah3 = LPh[ib + 4];
      const uint32_t al0 = LPl[ia], al1 = LPl[ib], al2 = LPl[ia + 4], al3 = LPl[ib + 4];
      uint32_t bh0, bh1, bl0, bl1;  // B fragment: -LP^T (A update) or -XRn (X update)
      if (isa) {
        const int ic = (c0 + g) * LM_PS + t4;
        bh0 = LPh[ic] ^ 0x80000000u;
        bh1 = LPh[ic + 4] ^ 0x80000000u;
        bl0 = LPl[ic] ^ 0x80000000u;
        bl1 = LPl[ic + 4] ^ 0x80000000u;
      } else {
        const int ic = t4 * LM_XS + c0 + g;
        bh0 = XNh[ic];
        bh1 = XNh[ic + 4 * LM_XS];
        bl0 = XNl[ic];
        bl1 = XNl[ic + 4 * LM_XS];
      }
      lm_mma(acc[j], ah0, ah1, ah2, ah3, bh0, bh1);
      lm_mma(acc[j], ah0, ah1, ah2, ah3, bl0, bl1);
      lm_mma(acc[j], al0, al1, al2, al3, bh0, bh1);
    }
    // finished X rows k..k+7 into their tiles (their LP rows are zero: the mma left them)
#pragma unroll
    for (int j = 0; j < 9; ++j) {
      if (warp + 16 * j < 72 || 16 * ttr[j] != (k & ~15) || ttc[j] > kc) continue;
      const bool h = (k >> 3) & 1;
      const float v0 = XRn[g * LM_XS + 8 * ttc[j] + 2 * t4], v1 = XRn[g * LM_XS + 8 * ttc[j] + 2 * t4 + 1];
      acc[j][0] = h ? acc[j][0] : v0;
      acc[j][1] = h ? acc[j][1] : v1;
      acc[j][2] = h ? v0 : acc[j][2];
      acc[j][3] = h ? v1 : acc[j][3];
    }
#ifdef DPK_LEAF_PROF
    long long c5 = clock64();
    if (blockIdx.x == 0 && (tid == 0 || tid == 511)) {
      unsigned long long* gp = g_leaf_prof + (tid ? 6 : 0);
      atomicAdd(gp + 0, c1 - c0); atomicAdd(gp + 1, c2 - c1); atomicAdd(gp + 2, c3 - c2);
      atomicAdd(gp + 3, c4 - c3); atomicAdd(gp + 4, c5 - c4); atomicAdd(gp + 5, 1ull);
    }
#endif
  }
  // X = L^-1 (zero above the diagonal): the lower tiles; the rest of the block is zeroed
  float* dst = J.dst;
  const int64_t ldd = J.ldd;
#pragma unroll
  for (int j = 0; j < 9; ++j) {
    if (warp + 16 * j < 72) continue;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = 16 * ttr[j] + g + 8 * (e >> 1), c = 8 * ttc[j] + 2 * t4 + (e & 1);
      if (r < n && c < n) dst[static_cast<int64_t>(r) * ldd + c] = acc[j][e];
    }
  }
  for (int e = tid; e < 128 * 128; e += LM_THREADS) {
    const int r = e >> 7, c = e & 127;
    if (r < n && c < n && (c >> 3) > 2 * (r >> 4) + 1) dst[static_cast<int64_t>(r) * ldd + c] = 0.0f;
  }
}

// DPK_LEAF_MMA=1: the tensor-core leaf for TRI-mode leaves.  Parity-green but measured
// slower than the SIMT leaf (~36 vs 27 us per 128 leaf): per step the redundant 8x8
// pivot factor + inverse costs ~1600 cycles and the 432 legacy mma.sync TF32
// instructions (3 per tile) ~1300-2400 cycles, against ~1200 cycles for a 4-column
// SIMT step -- so it is off by default.
bool leaf_mma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_LEAF_MMA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <int RB, int W>
constexpr int leaf_smem_bytes() {
  return (4 * 16 * RB * W + 16 * RB * (16 * RB + 1)) * 4;  // 4 panels of N x W + the X^T X copy
}
int leaf_width() {  // columns per sweep step (DPK_LEAF_W=4 default, or 8)
  static int w = -1;
  if (w < 0) {
    const char* e = getenv("DPK_LEAF_W");
    w = (e && e[0] == '8') ? 8 : 4;
  }
  return w;
}

// Blocked-path set-up, one warp per row i:  Aw[i][0..i] = src[i][0..i] (+ shift
// on the diagonal) and X[i][i+1..n) = 0.  The recursion only ever reads the
// lower triangle of Aw (A21 blocks, lower-only Schur updates, leaves factor
// from the lower part), and every lower block of X is overwritten by a leaf or
// an X21 product, so nothing else needs initialising.  Aw / X rows are padded to
// ldw (a multiple of 4 floats) so every recursion operand is a 16-byte aligned
// TMA view.
constexpr int PREP_MAX = 256;
constexpr int PREP_WARPS = 8;
struct PrepJob {
  const float* src;
  float* dst;
  float* x;
  const float* shift;
  int64_t n;
  int64_t ldw;
};
struct PrepBatch {
  int n;
  PrepJob j[PREP_MAX];
};
__global__ void __launch_bounds__(PREP_WARPS * 32) prep_kernel(const __grid_constant__ PrepBatch b) {
  pdl_wait();
  pdl_trigger();
  const PrepJob& J = b.j[blockIdx.y];
  const int n = static_cast<int>(J.n);
  const int64_t ldw = J.ldw;
  const float sh = J.shift ? *J.shift : 0.0f;
  const int lane = threadIdx.x & 31;
  // float4 path: every row of src / Aw / X starts 16-byte aligned
  const bool vec = (n % 4) == 0 && (ldw % 4) == 0 &&
                   ((reinterpret_cast<uintptr_t>(J.src) | reinterpret_cast<uintptr_t>(J.dst) |
                     reinterpret_cast<uintptr_t>(J.x)) & 15) == 0;
  for (int i = blockIdx.x * PREP_WARPS + (threadIdx.x >> 5); i < n; i += gridDim.x * PREP_WARPS) {
    const float* srow = J.src + static_cast<int64_t>(i) * n;
    float* arow = J.dst + static_cast<int64_t>(i) * ldw;
    float* xrow = J.x + static_cast<int64_t>(i) * ldw;
    if (vec) {
      // lower part [0, i] in whole float4s (the entries past i in the last vector are
      // upper-triangle values of Aw the recursion never reads), the damping on the diagonal
      const int q_end = i / 4;  // last vector touching column i
      for (int q = lane; q <= q_end; q += 32) {
        float4 v = __ldg(reinterpret_cast<const float4*>(srow) + q);
        if (q == q_end) {
          const int e = i - 4 * q;
          if (e == 0) v.x += sh;
          else if (e == 1) v.y += sh;
          else if (e == 2) v.z += sh;
          else v.w += sh;
        }
        reinterpret_cast<float4*>(arow)[q] = v;
      }
      // X[i][i+1..n) = 0: the partial vector scalar, then float4s
      const int z0 = i + 1, zq = (z0 + 3) / 4;
      if (lane < 4 * zq - z0 && z0 + lane < n) xrow[z0 + lane] = 0.0f;
      for (int q = zq + lane; q < n / 4; q += 32) reinterpret_cast<float4*>(xrow)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int c = lane; c <= i; c += 32) {
        const float v = __ldg(srow + c);
        arow[c] = c == i ? v + sh : v;
      }
      for (int c = i + 1 + lane; c < n; c += 32) xrow[c] = 0.0f;
    }
  }
}

inline int64_t padded_ld(int n) { return (static_cast<int64_t>(n) + 3) / 4 * 4; }

// One lock-step round of one matrix: a leaf, or one or two independent GEMMs.
struct Op {
  bool leaf;
  LeafJob lj;
  int ng;
  GemmSpec g[2];
};

// Split so that every block of a multiple-of-128 size stays a multiple of 128
// (4608 -> 36 leaves of 128 instead of 32 of 128 + 8 of 64, and 4 fewer
// internal nodes of 3 rounds each); DPK_SPLIT64=1 restores the half-rounded-to-64
// split.
int split_point(int n) {
  static int s64 = -1;
  if (s64 < 0) {
    const char* e = getenv("DPK_SPLIT64");
    s64 = (e && e[0] == '1') ? 1 : 0;
  }
  int n1;
  if (s64 || n <= 2 * LEAF_N) {
    n1 = ((n / 2 + 63) / 64) * 64;
  } else {
    n1 = ((n / 2 + 64) / 128) * 128;  // nearest multiple of 128 to n/2 (ties up)
    n1 = std::max(n1, LEAF_N);
  }
  return std::min(n1, n - 1);
}

size_t matrix_ws_floats(int n, bool factor) {
  if (n <= LEAF_N) return 0;
  // working copy Aw, L blocks, X = L^-1 (all n x padded_ld; +4 for alignment);
  // factor mode writes X straight into the caller's dst
  return (factor ? 2 : 3) * static_cast<size_t>(n) * padded_ld(n) + 4;
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

// Aw, Lb, Xb share the row stride ld.  Three GEMM rounds per recursion node:
//   (a) L21 = A21 X11^T
//   (b) A22 -= L21 L21^T (lower tiles only)   and   T^T = X11^T L21^T
//   (c) X21 = -X22 T                               (after the A22 recursion)
// T^T (n1 x n2) lives in the node's upper-right block of Lb: L is lower
// triangular, and no descendant of either child touches that block.
void build_ops(float* Aw, float* Lb, float* Xb, int64_t ld, int n, int fail_code, int32_t* info,
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
  float* Tt = Lb + n1;  // n1 x n2, row stride ld
  build_ops(Aw, Lb, Xb, ld, n1, fail_code, info, ops);
  Op op{};
  op.leaf = false;
  op.ng = 1;
  op.g[0] = spec(rows_k(Aw + o21, n2, n1, ld), rows_k(Xb, n1, n1, ld), Lb + o21, ld, 1.0f, 0.0f, 0);
  op.g[0].tri_b = TRI_LOWER;  // X11 lower: output column block j only needs k <= j
  ops.push_back(op);
  op.ng = 2;
  op.g[0] = spec(rows_k(Lb + o21, n2, n1, ld), rows_k(Lb + o21, n2, n1, ld), Aw + o22, ld, -1.0f, 1.0f, 1);
  op.g[0].lower_only = 1;  // the recursion reads only the lower triangle of A22
  // T^T[j][i] = sum_k X11[k][j] L21[i][k]: A = X11^T (rows_mn view), B = L21
  op.g[1] = spec(rows_mn(Xb, n1, n1, ld), rows_k(Lb + o21, n2, n1, ld), Tt, ld, 1.0f, 0.0f, 0);
  op.g[1].tri_a = TRI_UPPER;  // op view of X11 is X11^T: k >= j
  ops.push_back(op);
  build_ops(Aw + o22, Lb + o22, Xb + o22, ld, n2, fail_code, info, ops);
  op.ng = 1;
  op.g[1] = GemmSpec{};
  // X21 = -X22 T:  B[j][k] = T[k][j] = T^T[j][k]
  op.g[0] = spec(rows_k(Xb + o22, n2, n2, ld), rows_k(Tt, n1, n2, ld), Xb + o21, ld, -1.0f, 0.0f, 0);
  op.g[0].tri_a = TRI_LOWER;  // X22 lower: k <= i
  ops.push_back(op);
}

// Matrices advance in lock-step rounds inside a group; groups are independent
// chains on their own streams (forked from / joined to the caller's stream), so
// the long recursion of the largest factors is not paced by -- and its rounds
// are not split into several launches by -- the many mid-sized ones.
constexpr int MAX_GROUPS = 6;
// One factor of a batched call, either public job kind:
//   factor == 0: dst (ldd = n) = (src + shift I)^-1          (dpk_chol_inv_damped_batched)
//   factor == 1: dst (ldd = round_up(n, 4)) = L^-1, L L^T = src + shift I
//                (dpk_chol_factor_inv_batched: the recursion's X, written in place)
struct SpdReq {
  const float* src;
  float* dst;
  int64_t ldd;
  int32_t n;
  int32_t fail_code;
  const float* shift;
  int32_t* info;
  int32_t factor;
  int32_t _pad;
};
// Right-looking blocked Cholesky with look-ahead (the largest size class): the
// matrix's working buffers, kept per job so the schedule can be generated.
struct RlMat {
  float* Aw;
  float* Lb;
  float* Xb;
  int64_t ld;
  int n;
  int fail_code;
  int32_t* info;
};
struct SpdPlan {
  std::vector<std::vector<Op>> lists;
  std::vector<PrepJob> preps;
  std::vector<std::vector<int>> groups;   // job indices; groups[0] = the largest factors
  std::vector<size_t> group_ws;           // split-K workspace offset of each group
  std::vector<int> group_rl;              // 1: the group runs the right-looking schedule
  std::vector<size_t> group_ws_side;      // RL groups: workspace offset of the side (T2) stream
  std::vector<RlMat> mats;                // per job (blocked path only)
  size_t rec_bytes = 0;
  size_t gemm_bytes = 0;                  // sum over groups
};

// groups: distinct sizes in descending order, a new group whenever the size
// drops below 0.6x the group's largest (ResNet-50: 4608 | 2304..2048 |
// 1152..1000 | 576, 512 | 256 | 147, 128 and below); at most MAX_GROUPS.
void make_groups(const SpdReq* jobs, int n, SpdPlan& plan) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return jobs[a].n > jobs[b].n; });
  plan.groups.clear();
  int gmax = 0;
  for (int i : order) {
    const int m = jobs[i].n;
    if (plan.groups.empty() || (m * 10 < gmax * 6 && static_cast<int>(plan.groups.size()) < MAX_GROUPS)) {
      plan.groups.emplace_back();
      gmax = m;
    }
    plan.groups.back().push_back(i);
  }
  for (auto& g : plan.groups) std::sort(g.begin(), g.end());  // ascending layer order inside a group
}

// ---------------------------------------------------------------- right-looking schedule
// Blocks of 128 (the last may be smaller).  Step k, all matrices of the group in
// lock-step:
//   LEAF(k)   X_kk = L_kk^-1 of the (fully updated) diagonal block     [critical]
//   PANEL(k)  L_ik = A_ik X_kk^T, i > k                                 [critical]
//   T1(k)     A_{i,k+1} -= L_ik L_{k+1,k}^T, i >= k+1  (next column)     [critical,
//             after T2(k-1)]
//   T2(k)     A_ij -= L_ik L_jk^T, i >= j >= k+2 (lower tiles)           [side stream,
//             after PANEL(k); capped to leave SMs to the critical stream]
// so the bulk trailing update of step k runs under LEAF(k+1) / PANEL(k+1) instead
// of on the critical path.  Then X = L^-1 from the leaf inverses, level-batched
// recursion over block ranges (X21 = -X22 (L21 X11)): 2 rounds per level.
struct RlStep {
  int stream;          // 0 critical, 1 side (T2)
  int wait;            // 0 none, 1 wait ev_panel (side), 2 wait ev_t2 (critical)
  int record;          // 0 none, 1 record ev_panel (critical), 2 record ev_t2 (side)
  std::vector<LeafJob> leaves;
  std::vector<GemmSpec> g;
};

inline int rl_blocks(int n) { return (n + LEAF_N - 1) / LEAF_N; }

void rl_schedule(const std::vector<const RlMat*>& mats, std::vector<RlStep>& out) {
  out.clear();
  int maxb = 0;
  for (auto* M : mats) maxb = std::max(maxb, rl_blocks(M->n));
  for (int k = 0; k < maxb; ++k) {
    RlStep leaf{0, 0, 0, {}, {}}, panel{0, 0, 1, {}, {}}, t1{0, k > 0 ? 2 : 0, 0, {}, {}}, t2{1, 1, 2, {}, {}};
    for (auto* M : mats) {
      const int B = rl_blocks(M->n);
      if (k >= B) continue;
      const int64_t ld = M->ld;
      const int r0 = k * LEAF_N, bk = std::min(LEAF_N, M->n - r0);
      const int r1 = r0 + bk, rest = M->n - r1;
      leaf.leaves.push_back(LeafJob{M->Aw + r0 * ld + r0, M->Xb + r0 * ld + r0, nullptr, ld, ld, bk, 0,
                                    M->fail_code, 0, M->info});
      if (rest <= 0) continue;
      // PANEL: L[r1:, r0:r1] = A[r1:, r0:r1] X_kk^T   (X_kk lower: column block j needs k <= j)
      GemmSpec pg = spec(rows_k(M->Aw + r1 * ld + r0, rest, bk, ld), rows_k(M->Xb + r0 * ld + r0, bk, bk, ld),
                         M->Lb + r1 * ld + r0, ld, 1.0f, 0.0f, 0);
      pg.tri_b = TRI_LOWER;
      panel.g.push_back(pg);
      // T1: A[r1:, r1:r1+b1] -= L[r1:, k] L[r1:r1+b1, k]^T
      const int b1 = std::min(LEAF_N, rest);
      t1.g.push_back(spec(rows_k(M->Lb + r1 * ld + r0, rest, bk, ld), rows_k(M->Lb + r1 * ld + r0, b1, bk, ld),
                          M->Aw + r1 * ld + r1, ld, -1.0f, 1.0f, 0));
      // T2: A[r2:, r2:] -= L[r2:, k] L[r2:, k]^T (lower tiles)
      const int r2 = r1 + b1, rest2 = M->n - r2;
      if (rest2 > 0) {
        GemmSpec g2 = spec(rows_k(M->Lb + r2 * ld + r0, rest2, bk, ld), rows_k(M->Lb + r2 * ld + r0, rest2, bk, ld),
                           M->Aw + r2 * ld + r2, ld, -1.0f, 1.0f, 1);
        g2.lower_only = 1;
        t2.g.push_back(g2);
      }
    }
    out.push_back(std::move(leaf));
    if (!panel.g.empty()) out.push_back(std::move(panel));
    else out.push_back(RlStep{0, 0, 1, {}, {}});  // keep the event sequence uniform
    if (!t1.g.empty() || k > 0) out.push_back(std::move(t1));
    out.push_back(std::move(t2));
  }
  // join: the critical stream waits for the last trailing update
  out.push_back(RlStep{0, 2, 0, {}, {}});
  // X = L^-1, level-batched over block ranges [s, e) of each matrix
  struct Rng {
    const RlMat* M;
    int s, e;  // block indices
  };
  std::vector<std::vector<Rng>> levels;  // levels[0] = the whole ranges
  {
    std::vector<Rng> cur;
    for (auto* M : mats) cur.push_back(Rng{M, 0, rl_blocks(M->n)});
    while (!cur.empty()) {
      levels.push_back(cur);
      std::vector<Rng> nxt;
      for (auto& r : cur)
        if (r.e - r.s > 1) {
          const int mid = r.s + (r.e - r.s + 1) / 2;
          nxt.push_back(Rng{r.M, r.s, mid});
          nxt.push_back(Rng{r.M, mid, r.e});
        }
      cur.swap(nxt);
    }
  }
  for (int lv = static_cast<int>(levels.size()) - 1; lv >= 0; --lv) {  // bottom-up
    RlStep ra{0, 0, 0, {}, {}}, rb{0, 0, 0, {}, {}};
    for (auto& r : levels[lv]) {
      if (r.e - r.s < 2) continue;
      const RlMat* M = r.M;
      const int64_t ld = M->ld;
      const int mid = r.s + (r.e - r.s + 1) / 2;
      const int c0 = r.s * LEAF_N, c1 = mid * LEAF_N, c2 = std::min(M->n, r.e * LEAF_N);
      const int n1 = c1 - c0, n2 = c2 - c1;
      // T = L21 X11 into the (consumed) working block A[c1:c2, c0:c1]
      GemmSpec ta = spec(rows_k(M->Lb + c1 * ld + c0, n2, n1, ld), rows_mn(M->Xb + c0 * ld + c0, n1, n1, ld),
                         M->Aw + c1 * ld + c0, ld, 1.0f, 0.0f, 0);
      ta.tri_b = TRI_UPPER;  // op view of X11 is X11^T: k >= j
      ra.g.push_back(ta);
      // X21 = -X22 T
      GemmSpec tb = spec(rows_k(M->Xb + c1 * ld + c1, n2, n2, ld), rows_mn(M->Aw + c1 * ld + c0, n1, n2, ld),
                         M->Xb + c1 * ld + c0, ld, -1.0f, 0.0f, 0);
      tb.tri_a = TRI_LOWER;  // X22 lower: k <= i
      rb.g.push_back(tb);
    }
    if (!ra.g.empty()) {
      out.push_back(std::move(ra));
      out.push_back(std::move(rb));
    }
  }
}

// DPK_SPD_RL=<n>: groups whose largest factor is >= n use the right-looking schedule.
// Off by default: measured slower than the recursion on B200 (three 4608 factors
// 3.90 vs 3.66 ms, the ResNet-50 set 5.75 vs 4.82 ms): the chain is ~65% bound by
// the 3xTF32 flops, and the rank-128 trailing updates stream the whole trailing
// matrix per block column (n^3 / 3b floats of traffic) where the recursion's
// large-K products reuse operands on chip; the side lane also contends for SMs.
int rl_min_n() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_SPD_RL");
    v = e ? atoi(e) : 0;
    if (v <= 0) v = 1 << 30;
  }
  return v;
}

void make_spd_plan(const SpdReq* jobs, int n, char* base, SpdPlan& plan) {
  plan.lists.assign(n, {});
  char* b = base ? base : reinterpret_cast<char*>(0x100000);
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int m = jobs[i].n;
    std::vector<Op>& ops = plan.lists[i];
    if (m <= LEAF_N) {
      Op op{};
      op.leaf = true;
      op.lj = LeafJob{jobs[i].src, jobs[i].dst,     jobs[i].shift, m,
                      jobs[i].ldd, m,            jobs[i].factor ? 2 : 1, jobs[i].fail_code,
                      0,           jobs[i].info};
      ops.push_back(op);
      continue;
    }
    const int64_t ldw = padded_ld(m);  // 16-byte rows -> TMA-addressable operands
    const size_t blk = static_cast<size_t>(m) * ldw;
    const bool factor = jobs[i].factor != 0;
    float* Aw = reinterpret_cast<float*>(b + off);
    float* Lb = Aw + blk;
    float* Xb = factor ? jobs[i].dst : Lb + blk;
    off += align_up(matrix_ws_floats(m, factor) * sizeof(float), 256);
    plan.preps.push_back(PrepJob{jobs[i].src, Aw, Xb, jobs[i].shift, m, ldw});
    if (static_cast<int>(plan.mats.size()) < n) plan.mats.resize(n);
    plan.mats[i] = RlMat{Aw, Lb, Xb, ldw, m, jobs[i].fail_code, jobs[i].info};
    build_ops(Aw, Lb, Xb, ldw, m, jobs[i].fail_code, jobs[i].info, ops);
    if (factor) continue;  // X is the result
    Op op{};
    op.leaf = false;
    op.ng = 1;
    // dst = X^T X  (X lower triangular; symmetric output, written with the caller's ld = n)
    op.g[0] = spec(rows_mn(Xb, m, m, ldw), rows_mn(Xb, m, m, ldw), jobs[i].dst, m, 1.0f, 0.0f, 1);
    op.g[0].tri_a = op.g[0].tri_b = TRI_UPPER;  // (X^T X)[i][j] = sum over k >= max(i, j)
    ops.push_back(op);
  }
  plan.rec_bytes = off;
  plan.mats.resize(n);
  make_groups(jobs, n, plan);
  plan.gemm_bytes = 0;
  plan.group_ws.clear();
  plan.group_rl.clear();
  plan.group_ws_side.clear();
  for (const auto& grp : plan.groups) {
    // right-looking schedule: factored-mode groups of large factors (explicit
    // inverses keep the recursion, whose X^T X round follows the same lists)
    bool rl = true;
    int gmax = 0;
    for (int q : grp) {
      rl = rl && jobs[q].factor && jobs[q].n > LEAF_N;
      gmax = std::max(gmax, jobs[q].n);
    }
    rl = rl && gmax >= rl_min_n();
    plan.group_rl.push_back(rl ? 1 : 0);
    if (rl) {
      std::vector<const RlMat*> ms;
      for (int q : grp) ms.push_back(&plan.mats[q]);
      std::vector<RlStep> steps;
      rl_schedule(ms, steps);
      size_t wc = 0, wsd = 0;
      for (auto& stp : steps)
        if (!stp.g.empty()) {
          const size_t w = gemm_workspace_bytes(stp.g.data(), static_cast<int>(stp.g.size()));
          (stp.stream ? wsd : wc) = std::max(stp.stream ? wsd : wc, w);
        }
      plan.group_ws.push_back(plan.gemm_bytes);
      plan.gemm_bytes += align_up(std::max<size_t>(wc, GEMM_SCHED_BYTES), 1024);
      plan.group_ws_side.push_back(plan.gemm_bytes);
      plan.gemm_bytes += align_up(std::max<size_t>(wsd, GEMM_SCHED_BYTES), 1024);
      continue;
    }
    plan.group_ws_side.push_back(0);
    std::vector<size_t> idx(grp.size(), 0);
    size_t worst = 0;
    for (;;) {
      std::vector<GemmSpec> g;
      bool any = false;
      for (size_t q = 0; q < grp.size(); ++q) {
        const auto& list = plan.lists[grp[q]];
        if (idx[q] >= list.size()) continue;
        any = true;
        const Op& op = list[idx[q]];
        if (!op.leaf)
          for (int t = 0; t < op.ng; ++t) g.push_back(op.g[t]);
        ++idx[q];
      }
      if (!any) break;
      if (!g.empty()) worst = std::max(worst, gemm_workspace_bytes(g.data(), static_cast<int>(g.size())));
    }
    plan.group_ws.push_back(plan.gemm_bytes);
    plan.gemm_bytes += align_up(worst, 1024);
  }
}

template <int NB, int W>
int launch_leaf_nb(const LeafBatch& b, int cnt, cudaStream_t st) {
  static std::atomic<uint64_t> configured_on{0};
  if (first_on_device(configured_on)) {
    cudaError_t e = cudaFuncSetAttribute(spd_leaf_kernel<NB, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         leaf_smem_bytes<NB, W>());
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(spd_leaf_kernel)");
  }
  const cudaError_t e = launch_k(spd_leaf_kernel<NB, W>, dim3(cnt), dim3(LEAF_THREADS), leaf_smem_bytes<NB, W>(),
                                 st, 1, b);
  note_launch();
  return cuda_status(e, "spd_leaf_kernel launch");
}

template <int NB>
int launch_leaf_w(const LeafBatch& b, int cnt, cudaStream_t st) {
  return leaf_width() == 4 ? launch_leaf_nb<NB, 4>(b, cnt, st) : launch_leaf_nb<NB, 8>(b, cnt, st);
}

bool leaf_skip_done() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_LEAF_SKIP");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int launch_leaves(std::vector<LeafJob>& leaves, cudaStream_t st) {
  thread_local LeafBatch b;
  b.skip_done = leaf_skip_done() ? 1 : 0;
  for (size_t first = 0; first < leaves.size(); first += LEAF_MAX) {
    const int cnt = static_cast<int>(std::min<size_t>(LEAF_MAX, leaves.size() - first));
    b.n = cnt;
    int maxn = 1;
    for (int i = 0; i < cnt; ++i) {
      b.j[i] = leaves[first + i];
      maxn = std::max(maxn, b.j[i].n);
    }
    bool tri = true;
    for (int i = 0; i < cnt; ++i) tri = tri && b.j[i].full == 0;
    int rc;
    if (tri && maxn > 64 && leaf_mma_enabled()) {
      rc = cuda_status(launch_k(spd_leaf_mma_kernel, dim3(cnt), dim3(LM_THREADS), 0, st, 1, b),
                       "spd_leaf_mma_kernel launch");
      note_launch();
    } else if (maxn <= 32)
      rc = launch_leaf_w<2>(b, cnt, st);
    else if (maxn <= 64)
      rc = launch_leaf_w<4>(b, cnt, st);
    else
      rc = launch_leaf_w<8>(b, cnt, st);
    if (rc) return rc;
  }
  return DPK_OK;
}

// DPK_SPD_TRACE=1: time every lock-step round with events and print a table
// (diagnostics only; synchronises the stream at the end of the call).
bool spd_trace() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("DPK_SPD_TRACE");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

// Rounds of at least this many useful FMAs run as 3xF16 (fp16 hi / lo parts on
// kind::f16 MMAs, twice the 3xTF32 rate; one extra amax launch): DPK_SPD_F16_MIN,
// 0 = every tensor-core round, negative = never.
double spd_f16_min_fma() {
  static double v = -2.0;
  if (v == -2.0) {
    const char* e = getenv("DPK_SPD_F16_MIN");
    v = e ? atof(e) : -1.0;
    if (v < 0.0) v = 1e300;
  }
  return v;
}

double spec_fma(const GemmSpec& g) {
  const double M = g.job.a.rows, N = g.job.b.rows, K = static_cast<double>(g.job.a.cols);
  double f = M * N * K;
  if (g.job.symmetric) f *= 0.5;
  if (g.tri_a) f *= 0.5;
  if (g.tri_b) f *= (g.tri_a ? 2.0 / 3.0 : 0.5);
  return f;
}

bool spd_graphs_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("DPK_SPD_GRAPH");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}
int run_inverse(const SpdReq* jobs, int n_jobs, void* workspace, cudaStream_t st, bool trace);
int run_lockstep(const SpdPlan& plan, const std::vector<int>& grp, char* gemm_ws, size_t gemm_bytes,
                 cudaStream_t st, bool trace);

// per-device side streams (priority: group 0 -- the critical chain -- stays on
// the caller's stream; side streams get lower priority) and fork/join events
struct SideStreams {
  cudaStream_t s[MAX_GROUPS] = {};
  cudaEvent_t fork = nullptr;
  cudaEvent_t join[MAX_GROUPS] = {};
  int n = 0;
};
SideStreams& side_streams() {
  static std::mutex mu;
  static std::vector<SideStreams> per_dev;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (static_cast<int>(per_dev.size()) <= dev) per_dev.resize(dev + 1);
  return per_dev[dev];
}
int ensure_side_streams(int n) {
  SideStreams& ss = side_streams();
  if (!ss.fork) {
    int rc = cuda_status(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming), "cudaEventCreate");
    if (rc) return rc;
  }
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  while (ss.n < n) {
    int rc = cuda_status(cudaStreamCreateWithPriority(&ss.s[ss.n], cudaStreamNonBlocking, least),
                         "cudaStreamCreateWithPriority");
    if (rc) return rc;
    rc = cuda_status(cudaEventCreateWithFlags(&ss.join[ss.n], cudaEventDisableTiming), "cudaEventCreate");
    if (rc) return rc;
    ++ss.n;
  }
  return DPK_OK;
}
int run_cached_graph(const SpdReq* jobs, int n_jobs, void* workspace, size_t ws_bytes, cudaStream_t st);

// per-device streams and events of the right-looking schedule's side (T2) lane
struct RlLanes {
  cudaStream_t side[MAX_GROUPS] = {};
  cudaEvent_t ev_panel[MAX_GROUPS] = {};
  cudaEvent_t ev_t2[MAX_GROUPS] = {};
};
int rl_lane(int g, cudaStream_t& side, cudaEvent_t& ev_panel, cudaEvent_t& ev_t2) {
  static std::mutex mu;
  static std::vector<RlLanes> per_dev;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  if (static_cast<int>(per_dev.size()) <= dev) per_dev.resize(dev + 1);
  RlLanes& L = per_dev[dev];
  if (!L.side[g]) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    int rc = cuda_status(cudaStreamCreateWithPriority(&L.side[g], cudaStreamNonBlocking, least), "cudaStreamCreate(rl)");
    if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&L.ev_panel[g], cudaEventDisableTiming), "cudaEventCreate(rl)");
    if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&L.ev_t2[g], cudaEventDisableTiming), "cudaEventCreate(rl)");
    if (rc) return rc;
  }
  side = L.side[g];
  ev_panel = L.ev_panel[g];
  ev_t2 = L.ev_t2[g];
  return DPK_OK;
}

int rl_side_cap() {  // SMs the trailing updates may use (DPK_RL_CAP, default num_sms - 32)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_RL_CAP");
    v = e ? atoi(e) : std::max(16, num_sms() - 32);
  }
  return v;
}

int run_rl(const SpdPlan& plan, int g, char* ws_crit, size_t bytes_crit, char* ws_side, size_t bytes_side,
           cudaStream_t st) {
  std::vector<const RlMat*> ms;
  for (int q : plan.groups[g]) ms.push_back(&plan.mats[q]);
  std::vector<RlStep> steps;
  rl_schedule(ms, steps);
  cudaStream_t side;
  cudaEvent_t ev_panel, ev_t2;
  int rc = rl_lane(g, side, ev_panel, ev_t2);
  if (rc) return rc;
  // the side lane starts after everything already on the critical stream (prep)
  rc = cuda_status(cudaEventRecord(ev_panel, st), "cudaEventRecord(rl fork)");
  if (!rc) rc = cuda_status(cudaStreamWaitEvent(side, ev_panel, 0), "cudaStreamWaitEvent(rl fork)");
  if (!rc) rc = cuda_status(cudaMemsetAsync(ws_crit, 0, GEMM_SCHED_BYTES, st), "cudaMemsetAsync(rl counters)");
  if (!rc) rc = cuda_status(cudaMemsetAsync(ws_side, 0, GEMM_SCHED_BYTES, side), "cudaMemsetAsync(rl counters)");
  if (!rc) rc = cuda_status(cudaEventRecord(ev_t2, side), "cudaEventRecord(rl)");
  if (rc) return rc;
  for (const RlStep& stp : steps) {
    cudaStream_t s = stp.stream ? side : st;
    if (stp.wait == 1) rc = cuda_status(cudaStreamWaitEvent(s, ev_panel, 0), "cudaStreamWaitEvent(rl panel)");
    if (stp.wait == 2) rc = cuda_status(cudaStreamWaitEvent(s, ev_t2, 0), "cudaStreamWaitEvent(rl t2)");
    if (rc) return rc;
    if (!stp.leaves.empty()) {
      std::vector<LeafJob> lv = stp.leaves;
      rc = launch_leaves(lv, s);
      if (rc) return rc;
    }
    if (!stp.g.empty()) {
      if (stp.stream) set_grid_cap_override(rl_side_cap());
      rc = gemm_launch(stp.g.data(), static_cast<int>(stp.g.size()), stp.stream ? ws_side : ws_crit,
                       stp.stream ? bytes_side : bytes_crit, DPK_PREC_3XTF32, s, false);
      set_grid_cap_override(0);
      if (rc) return rc;
    }
    if (stp.record == 1) rc = cuda_status(cudaEventRecord(ev_panel, s), "cudaEventRecord(rl panel)");
    if (stp.record == 2) rc = cuda_status(cudaEventRecord(ev_t2, s), "cudaEventRecord(rl t2)");
    if (rc) return rc;
  }
  return DPK_OK;
}

}  // namespace
}  // namespace dpk


namespace dpk {
namespace {

size_t spd_workspace_bytes(const std::vector<SpdReq>& r) {
  const int n_jobs = static_cast<int>(r.size());
  if (n_jobs <= 0) return 0;
  UnitsPerSm units(1);  // latency-bound rounds: no split-K reduce launches on the chain
  // depends only on the sizes and modes (the plan is built against a dummy base)
  static LruCache<size_t> cache;
  std::string key;
  int dev = 0;
  cudaGetDevice(&dev);
  key_put(key, dev);
  for (const auto& q : r) {
    key_put(key, q.n);
    key_put(key, q.factor);
  }
  {
    std::lock_guard<std::mutex> lock(cache.mu);
    if (size_t* v = cache.find(key)) return *v;
  }
  SpdPlan plan;
  make_spd_plan(r.data(), n_jobs, nullptr, plan);
  const size_t need = align_up(plan.rec_bytes, 1024) + plan.gemm_bytes;
  std::lock_guard<std::mutex> lock(cache.mu);
  cache.put(key, need);
  return need;
}

int spd_run(const std::vector<SpdReq>& r, void* workspace, size_t ws_bytes, cudaStream_t st, const char* who) {
  const int n_jobs = static_cast<int>(r.size());
  if (n_jobs == 0) return DPK_OK;
  UnitsPerSm units(1);  // same split-K depth as spd_workspace_bytes
  for (const auto& q : r) {
    if (q.n < 1 || q.src == nullptr || q.dst == nullptr || q.src == q.dst) {
      set_error(std::string(who) + ": invalid job (n >= 1, distinct src/dst required)");
      return DPK_EARG;
    }
    if (q.factor && (q.ldd != padded_ld(q.n) || (reinterpret_cast<uintptr_t>(q.dst) & 15) != 0)) {
      set_error(std::string(who) + ": dst must be 16-byte aligned with row stride round_up(n, 4)");
      return DPK_EARG;
    }
  }
  const size_t need = spd_workspace_bytes(r);
  if (need > ws_bytes || (need > 0 && workspace == nullptr)) {
    set_error(std::string(who) + ": workspace too small");
    return DPK_ENOSPACE;
  }
  const bool trace = spd_trace();
  if (!trace && spd_graphs_enabled()) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    int rc = cuda_status(cudaStreamIsCapturing(st, &cs), "cudaStreamIsCapturing");
    if (rc) return rc;
    // inside a caller's capture the launches simply join that graph
    if (cs == cudaStreamCaptureStatusNone) return run_cached_graph(r.data(), n_jobs, workspace, ws_bytes, st);
  }
  return run_inverse(r.data(), n_jobs, workspace, st, trace);
}

std::vector<SpdReq> reqs_of(const dpk_spd_job* jobs, int n) {
  std::vector<SpdReq> r(std::max(n, 0));
  for (int i = 0; i < n; ++i)
    r[i] = SpdReq{jobs[i].src, jobs[i].dst, jobs[i].n, jobs[i].n, jobs[i].fail_code, jobs[i].shift, jobs[i].info, 0, 0};
  return r;
}
std::vector<SpdReq> reqs_of(const dpk_spd_factor_job* jobs, int n) {
  std::vector<SpdReq> r(std::max(n, 0));
  for (int i = 0; i < n; ++i)
    r[i] = SpdReq{jobs[i].src, jobs[i].dst, jobs[i].ldd, jobs[i].n, jobs[i].fail_code, jobs[i].shift, jobs[i].info, 1, 0};
  return r;
}

}  // namespace
}  // namespace dpk

extern "C" {

size_t dpk_chol_inv_workspace_bytes(const dpk_spd_job* jobs, int n_jobs) {
  if (n_jobs <= 0 || jobs == nullptr) return 0;
  return dpk::spd_workspace_bytes(dpk::reqs_of(jobs, n_jobs));
}

int dpk_chol_inv_damped_batched(const dpk_spd_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                                dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_chol_inv_damped_batched: bad job list");
    return DPK_EARG;
  }
  return dpk::spd_run(dpk::reqs_of(jobs, n_jobs), workspace, ws_bytes, static_cast<cudaStream_t>(stream),
                      "dpk_chol_inv_damped_batched");
}

size_t dpk_chol_factor_inv_workspace_bytes(const dpk_spd_factor_job* jobs, int n_jobs) {
  if (n_jobs <= 0 || jobs == nullptr) return 0;
  return dpk::spd_workspace_bytes(dpk::reqs_of(jobs, n_jobs));
}

int dpk_chol_factor_inv_batched(const dpk_spd_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                                dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_chol_factor_inv_batched: bad job list");
    return DPK_EARG;
  }
  return dpk::spd_run(dpk::reqs_of(jobs, n_jobs), workspace, ws_bytes, static_cast<cudaStream_t>(stream),
                      "dpk_chol_factor_inv_batched");
}

#ifdef DPK_LEAF_PROF
int dpk_leaf_prof(unsigned long long* out12) {
  return dpk::cuda_status(cudaMemcpyFromSymbol(out12, dpk::g_leaf_prof, 12 * 8), "leaf prof");
}
#endif
}  // extern "C"

namespace dpk {
namespace {

int run_inverse(const SpdReq* jobs, int n_jobs, void* workspace, cudaStream_t st, bool trace) {
  dpk::SpdPlan plan;
  char* base = static_cast<char*>(workspace);
  dpk::make_spd_plan(jobs, n_jobs, base, plan);
  char* gemm_ws = base + dpk::align_up(plan.rec_bytes, 1024);
  // blocked path set-up: working copy with the damping, X = 0
  thread_local dpk::PrepBatch pb;
  for (size_t first = 0; first < plan.preps.size(); first += dpk::PREP_MAX) {
    const int cnt = static_cast<int>(std::min<size_t>(dpk::PREP_MAX, plan.preps.size() - first));
    pb.n = cnt;
    int64_t maxn = 0;
    for (int i = 0; i < cnt; ++i) {
      pb.j[i] = plan.preps[first + i];
      maxn = std::max<int64_t>(maxn, pb.j[i].n);
    }
    const int gx = static_cast<int>(std::min<int64_t>((maxn + dpk::PREP_WARPS - 1) / dpk::PREP_WARPS, 64));
    const cudaError_t e = dpk::launch_k(dpk::prep_kernel, dim3(gx, cnt), dim3(dpk::PREP_WARPS * 32), 0, st, 1, pb);
    dpk::note_launch();
    int rc = dpk::cuda_status(e, "prep_kernel launch");
    if (rc) return rc;
  }
  if (trace) {  // diagnostics: one lock-step chain over all matrices, rounds timed
    std::vector<int> all(n_jobs);
    for (int i = 0; i < n_jobs; ++i) all[i] = i;
    return run_lockstep(plan, all, gemm_ws, plan.gemm_bytes, st, true);
  }
  const int ng = static_cast<int>(plan.groups.size());
  auto run_group = [&](int g, cudaStream_t s) -> int {
    const size_t off = plan.group_ws[g];
    if (plan.group_rl[g]) {
      const size_t side = plan.group_ws_side[g];
      const size_t end = g + 1 < ng ? plan.group_ws[g + 1] : plan.gemm_bytes;
      return run_rl(plan, g, gemm_ws + off, side - off, gemm_ws + side, end - side, s);
    }
    const size_t bytes = (g + 1 < ng ? plan.group_ws[g + 1] : plan.gemm_bytes) - off;
    return run_lockstep(plan, plan.groups[g], gemm_ws + off, bytes, s, false);
  };
  if (ng == 1) return run_group(0, st);
  int rc = ensure_side_streams(ng - 1);
  if (rc) return rc;
  SideStreams& ss = side_streams();
  rc = cuda_status(cudaEventRecord(ss.fork, st), "cudaEventRecord(fork)");
  if (rc) return rc;
  for (int g = 1; g < ng; ++g) {
    rc = cuda_status(cudaStreamWaitEvent(ss.s[g - 1], ss.fork, 0), "cudaStreamWaitEvent(fork)");
    if (rc) return rc;
  }
  for (int g = 0; g < ng; ++g) {
    rc = run_group(g, g == 0 ? st : ss.s[g - 1]);
    if (rc) return rc;
  }
  for (int g = 1; g < ng; ++g) {
    rc = cuda_status(cudaEventRecord(ss.join[g - 1], ss.s[g - 1]), "cudaEventRecord(join)");
    if (rc) return rc;
    rc = cuda_status(cudaStreamWaitEvent(st, ss.join[g - 1], 0), "cudaStreamWaitEvent(join)");
    if (rc) return rc;
  }
  return DPK_OK;
}

int run_lockstep(const SpdPlan& plan, const std::vector<int>& grp, char* gemm_ws, size_t gemm_bytes,
                 cudaStream_t st, bool trace) {
  std::vector<size_t> idx(grp.size(), 0);
  bool counters_zeroed = false;
  struct RoundRec {
    cudaEvent_t e0, e1, e2;
    int nleaf, maxn, ngemm;
    double fma;
    int bm, bn, bk;
  };
  std::vector<RoundRec> recs;
  for (;;) {
    std::vector<dpk::LeafJob> leaves;
    std::vector<dpk::GemmSpec> g;
    bool any = false;
    for (size_t q = 0; q < grp.size(); ++q) {
      const auto& list = plan.lists[grp[q]];
      if (idx[q] >= list.size()) continue;
      any = true;
      const dpk::Op& op = list[idx[q]];
      if (op.leaf)
        leaves.push_back(op.lj);
      else
        for (int t = 0; t < op.ng; ++t) g.push_back(op.g[t]);
      ++idx[q];
    }
    if (!any) break;
    RoundRec rr{};
    if (trace) {
      cudaEventCreate(&rr.e0);
      cudaEventCreate(&rr.e1);
      cudaEventCreate(&rr.e2);
      cudaEventRecord(rr.e0, st);
      rr.nleaf = static_cast<int>(leaves.size());
      for (auto& l : leaves) rr.maxn = std::max(rr.maxn, l.n);
      rr.ngemm = static_cast<int>(g.size());
      double best = -1;
      for (auto& x : g) {
        const double f = dpk::spec_fma(x);
        rr.fma += f;
        if (f > best) {
          best = f;
          rr.bm = x.job.a.rows;
          rr.bn = x.job.b.rows;
          rr.bk = static_cast<int>(x.job.a.cols);
        }
      }
    }
    if (!leaves.empty()) {
      int rc = dpk::launch_leaves(leaves, st);
      if (rc) return rc;
    }
    if (trace) cudaEventRecord(rr.e1, st);
    if (!g.empty()) {
      if (!counters_zeroed) {  // once per chain: the GEMM kernels leave the counters zero
        int rc = cuda_status(cudaMemsetAsync(gemm_ws, 0, GEMM_SCHED_BYTES, st), "cudaMemsetAsync(counters)");
        if (rc) return rc;
        counters_zeroed = true;
      }
      double fma = 0.0;
      for (auto& x : g) fma += dpk::spec_fma(x);
      int rc = dpk::gemm_launch(g.data(), static_cast<int>(g.size()), gemm_ws, gemm_bytes,
                                fma >= dpk::spd_f16_min_fma() ? DPK_PREC_3XF16 : DPK_PREC_3XTF32, st, false);
      if (rc) return rc;
    }
    if (trace) {
      cudaEventRecord(rr.e2, st);
      recs.push_back(rr);
    }
  }
  if (trace) {
    cudaStreamSynchronize(st);
    double tl = 0, tg = 0, tf = 0;
    fprintf(stderr, "round  leaves(maxn)  leaf_us  gemms  gemm_us  GFMA  TF/s(useful)  largest MxNxK\n");
    for (size_t i = 0; i < recs.size(); ++i) {
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, recs[i].e0, recs[i].e1);
      cudaEventElapsedTime(&b, recs[i].e1, recs[i].e2);
      tl += a;
      tg += b;
      tf += recs[i].fma;
      fprintf(stderr, "%5zu  %4d(%4d)  %8.1f  %5d  %8.1f  %7.3f  %6.1f  %dx%dx%d\n", i, recs[i].nleaf, recs[i].maxn,
              a * 1e3, recs[i].ngemm, b * 1e3, recs[i].fma / 1e9, b > 0 ? 2 * recs[i].fma / (b * 1e9) : 0.0,
              recs[i].bm, recs[i].bn, recs[i].bk);
      cudaEventDestroy(recs[i].e0);
      cudaEventDestroy(recs[i].e1);
      cudaEventDestroy(recs[i].e2);
    }
    fprintf(stderr, "total: leaves %.3f ms, gemms %.3f ms, %.1f GFMA -> %.1f TF/s useful\n", tl, tg, tf / 1e9,
            tg > 0 ? 2 * tf / (tg * 1e9) : 0.0);
  }
  return DPK_OK;
}

// Every training step inverts the same factor buffers with the same workspace,
// so the ~200 launches of the lock-step recursion are captured once into a
// CUDA graph (on a private stream) and replayed: host launch cost per round
// disappears and the GPU runs the rounds back to back.  Keyed by the exact job
// list + workspace + device; a small LRU bounds the cache.
struct GraphEntry {
  std::vector<char> key;
  cudaGraphExec_t exec;
  unsigned long long launches;
  unsigned long long last_use;
};

int run_cached_graph(const SpdReq* jobs, int n_jobs, void* workspace, size_t ws_bytes, cudaStream_t st) {
  static std::mutex mu;
  static std::vector<GraphEntry> cache;
  static unsigned long long tick = 0;
  static std::vector<cudaStream_t> cap_streams;
  constexpr size_t CACHE_MAX = 8;
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  std::vector<char> key(sizeof(SpdReq) * n_jobs + sizeof(void*) + sizeof(size_t) + 2 * sizeof(int));
  char* k = key.data();
  const int capv = grid_cap_override();  // the captured launches bake the grid size in
  std::memcpy(k, &capv, sizeof(int));
  k += sizeof(int);
  std::memcpy(k, jobs, sizeof(SpdReq) * n_jobs);
  k += sizeof(SpdReq) * n_jobs;
  std::memcpy(k, &workspace, sizeof(void*));
  k += sizeof(void*);
  std::memcpy(k, &ws_bytes, sizeof(size_t));
  k += sizeof(size_t);
  std::memcpy(k, &dev, sizeof(int));
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache) {
    if (e.key == key) {
      e.last_use = ++tick;
      rc = cuda_status(cudaGraphLaunch(e.exec, st), "cudaGraphLaunch(spd inverse)");
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
  rc = run_inverse(jobs, n_jobs, workspace, cap, false);
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
  rc = cuda_status(ie, "cudaGraphInstantiate(spd inverse)");
  if (rc) return rc;
  if (cache.size() >= CACHE_MAX) {
    auto old = std::min_element(cache.begin(), cache.end(),
                                [](const GraphEntry& a, const GraphEntry& b) { return a.last_use < b.last_use; });
    cudaGraphExecDestroy(old->exec);
    cache.erase(old);
  }
  cache.push_back(GraphEntry{std::move(key), exec, captured, ++tick});
  rc = cuda_status(cudaGraphLaunch(exec, st), "cudaGraphLaunch(spd inverse)");
  if (!rc) note_launches(captured);
  return rc;
}

}  // namespace
}  // namespace dpk
