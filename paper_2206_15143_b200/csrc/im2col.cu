// Sample-major patch matrix for conv A factors:  out[k*ld + r] = X[r, k].
//
// X is the implicit-im2col linear form (reference conv convention, SURVEY
// section 8(a) A3): rows (c,i,j) [DPK_OPND_IM2COL] or (i,j,c)
// [DPK_OPND_IM2COL_TAPMAJOR], columns k = (n, oh, ow); zero padding outside
// the image; the bias ones row last.  HBM-bound copy: with a channels-last
// input and tap-major rows, each (pixel, tap) is one contiguous run of C floats
// moved as float4s (coalesced reads and writes).  The SYRK then streams the
// result through 2-D TMA as an MN-major operand.
#include <cuda_runtime.h>

#include <algorithm>

#include "dpk_internal.h"

namespace dpk {
namespace {

constexpr int I2C_MAX = 128;
struct I2cBatch {
  int n;
  dpk_im2col_job j[I2C_MAX];
};

// One warp per output pixel k (patch row): (n, oh, ow) is decomposed once, then
// the lanes stream the row's (tap, channel) entries.  32-bit index math only:
// every per-tensor offset below is < 2^31 elements except the sample offset,
// which is taken in 64 bits.
constexpr int I2C_WARPS = 8;

// vectorised: tap-major rows, channels contiguous, C % 4 == 0, 16-byte aligned rows
__global__ void __launch_bounds__(I2C_WARPS * 32) im2col_vec_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const int c4n = o.C / 4;
  const int taps = o.kh * o.kw;
  const int per_pixel = taps * c4n;
  const int lane = threadIdx.x & 31;
  const int ohw = o.OH * o.OW;
  const int64_t npix = o.cols;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * I2C_WARPS + (threadIdx.x >> 5); k < npix;
       k += static_cast<int64_t>(gridDim.x) * I2C_WARPS) {
    const int n = static_cast<int>(k / ohw);
    const int rem = static_cast<int>(k - static_cast<int64_t>(n) * ohw);
    const int oh = rem / o.OW, ow = rem - (rem / o.OW) * o.OW;
    const int ih0 = oh * o.sh - o.ph, iw0 = ow * o.sw - o.pw;
    const float* base = o.data + static_cast<int64_t>(n) * o.sn;
    float4* out = reinterpret_cast<float4*>(J.out + k * J.ld);
    for (int e = lane; e < per_pixel; e += 32) {
      const int tap = e / c4n;
      const int c4 = e - tap * c4n;
      const int i = tap / o.kw, j = tap - (tap / o.kw) * o.kw;
      const int ih = ih0 + i * o.dh, iw = iw0 + j * o.dw;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) && static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
        v = __ldg(reinterpret_cast<const float4*>(base + static_cast<int64_t>(ih) * o.shs +
                                                  static_cast<int64_t>(iw) * o.sws) + c4);
      out[e] = v;  // tap * C + 4 * c4 == 4 * e
    }
    if (o.bias_row && lane == 0) J.out[k * J.ld + o.rows] = 1.0f;
  }
}

// generic: any strides, either row order
__global__ void __launch_bounds__(I2C_WARPS * 32) im2col_scalar_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const int d = o.rows + (o.bias_row ? 1 : 0);
  const int kk = o.kh * o.kw;
  const int lane = threadIdx.x & 31;
  const int ohw = o.OH * o.OW;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * I2C_WARPS + (threadIdx.x >> 5); k < o.cols;
       k += static_cast<int64_t>(gridDim.x) * I2C_WARPS) {
    const int n = static_cast<int>(k / ohw);
    const int rem = static_cast<int>(k - static_cast<int64_t>(n) * ohw);
    const int oh = rem / o.OW, ow = rem - (rem / o.OW) * o.OW;
    const int ih0 = oh * o.sh - o.ph, iw0 = ow * o.sw - o.pw;
    const float* base = o.data + static_cast<int64_t>(n) * o.sn;
    float* out = J.out + k * J.ld;
    for (int r = lane; r < d; r += 32) {
      float v = 1.0f;  // the bias row
      if (r < o.rows) {
        int c, i, j;
        if (o.kind == DPK_OPND_IM2COL) {
          c = r / kk;
          const int t = r - c * kk;
          i = t / o.kw;
          j = t - i * o.kw;
        } else {
          const int t = r / o.C;
          c = r - t * o.C;
          i = t / o.kw;
          j = t - i * o.kw;
        }
        const int ih = ih0 + i * o.dh, iw = iw0 + j * o.dw;
        v = 0.0f;
        if (static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) &&
            static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
          v = __ldg(base + static_cast<int64_t>(c) * o.sc + static_cast<int64_t>(ih) * o.shs +
                    static_cast<int64_t>(iw) * o.sws);
      }
      out[r] = v;
    }
  }
}

// row-staged: one CTA per output row (n, oh) at a time.  The kh input rows the
// row's patches touch are staged zero-padded in shared memory as [i][w][c]
// (any input strides: coalesced global reads), then the OW x ld patch block --
// contiguous in the output -- is written as float4s, each entry found through a
// per-job table off[r] = i*rowlen + j*dw*C + c (-1: zero pad, -2: bias ones).
// For small-C convs (the 3-channel stem) where a warp per pixel would move
// 4-byte scalars through divisions.
constexpr int ROWS_THREADS = 256;
constexpr int ROWS_SMEM_MAX = 160 * 1024;

struct RowsGeom {
  int padl, wp, rowlen;
};
__host__ __device__ inline RowsGeom rows_geom(const dpk_operand& o) {
  RowsGeom g;
  g.padl = o.pw;
  const int right = (o.OW - 1) * o.sw - o.pw + (o.kw - 1) * o.dw;  // last input column touched
  g.wp = o.pw + max(o.W, right + 1);
  g.rowlen = g.wp * o.C;
  return g;
}
__host__ inline size_t rows_smem(const dpk_im2col_job& j) {
  const RowsGeom g = rows_geom(j.x);
  return (static_cast<size_t>(j.x.kh) * g.rowlen + static_cast<size_t>(j.ld)) * 4;
}

__global__ void __launch_bounds__(ROWS_THREADS) im2col_rows_kernel(const __grid_constant__ I2cBatch b) {
  extern __shared__ float sm[];
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const RowsGeom g = rows_geom(o);
  const int ld = static_cast<int>(J.ld);
  float* stage = sm;
  int* off = reinterpret_cast<int*>(sm + o.kh * g.rowlen);
  for (int r = threadIdx.x; r < ld; r += ROWS_THREADS) {
    int v = -1;
    if (r < o.rows) {
      int c, i, j;
      if (o.kind == DPK_OPND_IM2COL) {
        const int kk = o.kh * o.kw;
        c = r / kk;
        const int t = r - c * kk;
        i = t / o.kw;
        j = t - i * o.kw;
      } else {
        const int t = r / o.C;
        c = r - t * o.C;
        i = t / o.kw;
        j = t - i * o.kw;
      }
      v = i * g.rowlen + j * o.dw * o.C + c;
    } else if (r == o.rows && o.bias_row) {
      v = -2;
    }
    off[r] = v;
  }
  const int ohw = o.OH * o.OW;
  const int64_t nrows = o.cols / o.OW;
  const int ld4 = ld / 4;
  const int shift = o.sw * o.C;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int n = static_cast<int>(row / o.OH);
    const int oh = static_cast<int>(row - static_cast<int64_t>(n) * o.OH);
    const float* base = o.data + static_cast<int64_t>(n) * o.sn;
    __syncthreads();  // previous row's readers are done (and the table is written)
    for (int e = threadIdx.x; e < o.kh * g.rowlen; e += ROWS_THREADS) {
      const int i = e / g.rowlen;
      const int q = e - i * g.rowlen;
      const int wq = q / o.C;
      const int c = q - wq * o.C;
      const int ih = oh * o.sh - o.ph + i * o.dh, iw = wq - g.padl;
      float v = 0.0f;
      if (static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) && static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
        v = __ldg(base + static_cast<int64_t>(c) * o.sc + static_cast<int64_t>(ih) * o.shs +
                  static_cast<int64_t>(iw) * o.sws);
      stage[e] = v;
    }
    __syncthreads();
    float4* out = reinterpret_cast<float4*>(J.out + (static_cast<int64_t>(n) * ohw + static_cast<int64_t>(oh) * o.OW) * ld);
    for (int e = threadIdx.x; e < o.OW * ld4; e += ROWS_THREADS) {
      const int ow = e / ld4;
      const int r0 = (e - ow * ld4) * 4;
      const int sh = ow * shift;
      float v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = off[r0 + q];
        v[q] = t >= 0 ? stage[t + sh] : (t == -2 ? 1.0f : 0.0f);
      }
      __stcs(out + e, make_float4(v[0], v[1], v[2], v[3]));
    }
  }
}

bool rows_ok(const dpk_im2col_job& j) {
  const dpk_operand& o = j.x;
  return j.ld % 4 == 0 && (reinterpret_cast<uintptr_t>(j.out) & 15) == 0 && o.cols % o.OW == 0 &&
         rows_smem(j) <= static_cast<size_t>(ROWS_SMEM_MAX);
}

bool vec_ok(const dpk_im2col_job& j) {
  const dpk_operand& o = j.x;
  return o.kind == DPK_OPND_IM2COL_TAPMAJOR && o.sc == 1 && o.C % 4 == 0 &&
         (reinterpret_cast<uintptr_t>(o.data) & 15) == 0 && (reinterpret_cast<uintptr_t>(j.out) & 15) == 0 &&
         o.sn % 4 == 0 && o.shs % 4 == 0 && o.sws % 4 == 0 && j.ld % 4 == 0;
}

}  // namespace
}  // namespace dpk

extern "C" int dpk_im2col_materialize(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_im2col_materialize: bad job list");
    return DPK_EARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  thread_local dpk::I2cBatch vb, sb, rb;
  vb.n = sb.n = rb.n = 0;
  int64_t vmax = 0, smax = 0;
  size_t rsmem = 0;
  auto flush_rows = [&]() -> int {
    if (rb.n == 0) return DPK_OK;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(dpk::im2col_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dpk::ROWS_SMEM_MAX);
      attr = true;
    }
    int64_t rows = 0;
    for (int i = 0; i < rb.n; ++i) rows = std::max<int64_t>(rows, rb.j[i].x.cols / rb.j[i].x.OW);
    const int gx = static_cast<int>(std::min<int64_t>(rows, 4 * 148));
    dpk::im2col_rows_kernel<<<dim3(gx, rb.n), dpk::ROWS_THREADS, rsmem, st>>>(rb);
    dpk::note_launch();
    rb.n = 0;
    rsmem = 0;
    return dpk::cuda_status(cudaGetLastError(), "im2col rows kernel launch");
  };
  auto flush = [&](dpk::I2cBatch& b, int64_t maxe, bool vec) -> int {
    if (b.n == 0) return DPK_OK;
    // maxe = the largest job's pixel count: one warp per pixel, grid-strided
    const int gx = static_cast<int>(std::min<int64_t>((maxe + dpk::I2C_WARPS - 1) / dpk::I2C_WARPS, 2048));
    if (vec)
      dpk::im2col_vec_kernel<<<dim3(gx, b.n), dpk::I2C_WARPS * 32, 0, st>>>(b);
    else
      dpk::im2col_scalar_kernel<<<dim3(gx, b.n), dpk::I2C_WARPS * 32, 0, st>>>(b);
    dpk::note_launch();
    b.n = 0;
    return dpk::cuda_status(cudaGetLastError(), "im2col kernel launch");
  };
  for (int i = 0; i < n_jobs; ++i) {
    const dpk_im2col_job& j = jobs[i];
    const dpk_operand& o = j.x;
    if ((o.kind != DPK_OPND_IM2COL && o.kind != DPK_OPND_IM2COL_TAPMAJOR) || j.out == nullptr || o.data == nullptr ||
        o.cols < 1 || o.rows != o.C * o.kh * o.kw || j.ld < o.rows + (o.bias_row ? 1 : 0)) {
      dpk::set_error("dpk_im2col_materialize: invalid job " + std::to_string(i));
      return DPK_EARG;
    }
    if (!dpk::vec_ok(j) && dpk::rows_ok(j)) {
      if (rb.n == dpk::I2C_MAX) {
        int rc = flush_rows();
        if (rc) return rc;
      }
      rb.j[rb.n++] = j;
      rsmem = std::max(rsmem, dpk::rows_smem(j));
      continue;
    }
    if (dpk::vec_ok(j)) {
      if (vb.n == dpk::I2C_MAX) {
        int rc = flush(vb, vmax, true);
        if (rc) return rc;
        vmax = 0;
      }
      vb.j[vb.n++] = j;
      vmax = std::max<int64_t>(vmax, o.cols);
    } else {
      if (sb.n == dpk::I2C_MAX) {
        int rc = flush(sb, smax, false);
        if (rc) return rc;
        smax = 0;
      }
      sb.j[sb.n++] = j;
      smax = std::max<int64_t>(smax, o.cols);
    }
  }
  int rc = flush(vb, vmax, true);
  if (rc) return rc;
  rc = flush_rows();
  if (rc) return rc;
  return flush(sb, smax, false);
}
