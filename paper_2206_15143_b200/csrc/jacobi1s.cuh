// One-sided (Hestenes) Jacobi for a symmetric n x n block (n <= 128) held in
// shared memory, shared by the on-chip eigensolver (syevd.cu, n <= 128) and the
// pair problems of the block Jacobi (syevj.cu).
//
// U starts as the symmetrized matrix, V as the identity (both COLUMN-major, row
// stride ld, so a warp walks a column with consecutive lanes: conflict-free).  A
// round rotates the m/2 disjoint column pairs of the tournament ordering, one
// warp per pair: the three dot products |u_p|^2, |u_q|^2, u_p.u_q by a warp
// reduction (a half-warp per pair), then the plane rotation that makes u_p, u_q
// orthogonal, applied to U
// and V.  No rotation touches another pair's columns, so a round needs one
// barrier (the two-sided method needs a row phase and a column phase).  At
// convergence U = A V has orthogonal columns: V holds the eigenvectors and
// lam_i = u_i . v_i = v_i^T A v_i the eigenvalues (with sign).
#pragma once

namespace dpk {

constexpr int J1_THREADS = 1024;  // 32 warps
constexpr int J1_MAX_SWEEPS = 30;

__device__ __forceinline__ void j1_pair(int round, int slot, int m, int& p, int& q) {
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

__device__ __forceinline__ float j1_warp_sum(float v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float j1_half_sum(float v) {  // within each 16-lane half
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// U, V: m x m column-major (ld >= m), n <= m <= 128, m even, columns >= n zero in U.
// A half-warp per column pair (two pairs per warp in flight).  Rotate (p, q) only if
//   |g| > rel_tol |u_p||u_q|      (not yet orthogonal),
//   |g| > 1e-6 max(a, b)          (above the rounding floor of a rotation: with graded
//                                  columns the relative cosine cannot drop below
//                                  eps sqrt(a/b), and chasing it never terminates),
//   max(a, b) > 1e-12 ||A||_F^2    (not both numerically zero columns: their mutual
//                                  orientation is rounding noise; measured in an fp32
//                                  model: 23-40 -> 8-11 sweeps, same accuracy),
// with a = |u_p|^2, b = |u_q|^2, g = u_p.u_q.  Fast reciprocal / sqrt are fine here:
// a rotation's rounding only scales u_i and v_i together (U = A V), and lam_i =
// u_i.v_i / |v_i|^2 and the final column re-normalisation remove it.
// Writes lam[0..m).
__device__ __forceinline__ void onesided_jacobi(float* U, float* V, int ld, int n, int m, float rel_tol, float* lam) {
  __shared__ float j1_f2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hl = lane & 15;
  const int nhalf = blockDim.x >> 4;
  const int half = m / 2;
  if (threadIdx.x == 0) j1_f2 = 0.f;
  __syncthreads();
  {
    float acc = 0.f;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const float x = U[(e / m) * ld + (e % m)];
      acc = fmaf(x, x, acc);
    }
    acc = j1_warp_sum(acc);
    if (lane == 0) atomicAdd(&j1_f2, acc);
  }
  __syncthreads();
  const float floor2 = 1e-12f * j1_f2;
  for (int sweep = 0; sweep < J1_MAX_SWEEPS; ++sweep) {
    int rotated = 0;
    for (int round = 0; round < m - 1; ++round) {
      for (int s = 2 * warp + (lane >> 4); s < half + ((half & 1) ? 1 : 0); s += nhalf) {
        // (both halves of a warp iterate together; a half without a pair idles)
        const bool live = s < half;
        int p = 0, q = 1;
        if (live) j1_pair(round, s, m, p, q);
        float* up = U + p * ld;
        float* uq = U + q * ld;
        float a = 0.f, b = 0.f, g = 0.f;
        if (live)
          for (int r = hl; r < n; r += 16) {
            const float x = up[r], y = uq[r];
            a = fmaf(x, x, a);
            b = fmaf(y, y, b);
            g = fmaf(x, y, g);
          }
        a = j1_half_sum(a);
        b = j1_half_sum(b);
        g = j1_half_sum(g);
        const float mx = fmaxf(a, b);
        if (live && fabsf(g) > rel_tol * sqrtf(a * b) && fabsf(g) > 1e-6f * mx && mx > floor2) {
          const float zeta = __fdividef(b - a, 2.0f * g);
          const float t = copysignf(1.0f, zeta) / (fabsf(zeta) + sqrtf(1.0f + zeta * zeta));
          const float c = rsqrtf(1.0f + t * t);
          const float sn = t * c;
          float* vp = V + p * ld;
          float* vq = V + q * ld;
          for (int r = hl; r < m; r += 16) {
            if (r < n) {
              const float x = up[r], y = uq[r];
              up[r] = c * x - sn * y;
              uq[r] = sn * x + c * y;
            }
            const float x = vp[r], y = vq[r];
            vp[r] = c * x - sn * y;
            vq[r] = sn * x + c * y;
          }
          rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  for (int c = warp; c < m; c += (blockDim.x >> 5)) {
    float l = 0.f, ss = 0.f;
    for (int r = lane; r < m; r += 32) {
      const float v = V[c * ld + r];
      if (r < n) l = fmaf(U[c * ld + r], v, l);
      ss = fmaf(v, v, ss);
    }
    l = j1_warp_sum(l);
    ss = j1_warp_sum(ss);
    const float inv = ss > 0.f ? rsqrtf(ss) : 1.f;
    const float fix = inv * (1.5f - 0.5f * ss * inv * inv);
    for (int r = lane; r < m; r += 32) V[c * ld + r] *= fix;
    if (lane == 0) lam[c] = l * fix * fix;
  }
  __syncthreads();
}

}  // namespace dpk
