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

__device__ __forceinline__ void pixel_of(const dpk_operand& o, int64_t k, int& n, int& oh, int& ow) {
  const int64_t ohw = static_cast<int64_t>(o.OH) * o.OW;
  n = static_cast<int>(k / ohw);
  const int rem = static_cast<int>(k - n * ohw);
  oh = rem / o.OW;
  ow = rem - oh * o.OW;
}

// vectorised: tap-major rows, channels contiguous, C % 4 == 0, 16-byte aligned rows
__global__ void im2col_vec_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const int c4n = o.C / 4;
  const int taps = o.kh * o.kw;
  const int64_t per_pixel = static_cast<int64_t>(taps) * c4n;
  const int64_t total = o.cols * per_pixel;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = e / per_pixel;
    const int rem = static_cast<int>(e - k * per_pixel);
    const int tap = rem / c4n;
    const int c4 = rem - tap * c4n;
    int n, oh, ow;
    pixel_of(o, k, n, oh, ow);
    const int i = tap / o.kw, j = tap - (tap / o.kw) * o.kw;
    const int ih = oh * o.sh - o.ph + i * o.dh;
    const int iw = ow * o.sw - o.pw + j * o.dw;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) && static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
      v = __ldg(reinterpret_cast<const float4*>(o.data + n * o.sn + static_cast<int64_t>(ih) * o.shs +
                                                static_cast<int64_t>(iw) * o.sws) + c4);
    *reinterpret_cast<float4*>(J.out + k * J.ld + static_cast<int64_t>(tap) * o.C + 4 * c4) = v;
    if (o.bias_row && rem == 0) J.out[k * J.ld + o.rows] = 1.0f;
  }
}

// generic: any strides, either row order
__global__ void im2col_scalar_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const int d = o.rows + (o.bias_row ? 1 : 0);
  const int64_t total = o.cols * d;
  const int kk = o.kh * o.kw;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = e / d;
    const int r = static_cast<int>(e - k * d);
    float v;
    if (r == o.rows) {
      v = 1.0f;
    } else {
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
      int n, oh, ow;
      pixel_of(o, k, n, oh, ow);
      const int ih = oh * o.sh - o.ph + i * o.dh;
      const int iw = ow * o.sw - o.pw + j * o.dw;
      v = 0.0f;
      if (static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) && static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
        v = __ldg(o.data + n * o.sn + static_cast<int64_t>(c) * o.sc + static_cast<int64_t>(ih) * o.shs +
                  static_cast<int64_t>(iw) * o.sws);
    }
    J.out[k * J.ld + r] = v;
  }
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
  thread_local dpk::I2cBatch vb, sb;
  vb.n = sb.n = 0;
  int64_t vmax = 0, smax = 0;
  auto flush = [&](dpk::I2cBatch& b, int64_t maxe, bool vec) -> int {
    if (b.n == 0) return DPK_OK;
    const int gx = static_cast<int>(std::min<int64_t>((maxe + 255) / 256, 4096));
    if (vec)
      dpk::im2col_vec_kernel<<<dim3(gx, b.n), 256, 0, st>>>(b);
    else
      dpk::im2col_scalar_kernel<<<dim3(gx, b.n), 256, 0, st>>>(b);
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
    if (dpk::vec_ok(j)) {
      if (vb.n == dpk::I2C_MAX) {
        int rc = flush(vb, vmax, true);
        if (rc) return rc;
        vmax = 0;
      }
      vb.j[vb.n++] = j;
      vmax = std::max<int64_t>(vmax, o.cols * o.kh * o.kw * (o.C / 4));
    } else {
      if (sb.n == dpk::I2C_MAX) {
        int rc = flush(sb, smax, false);
        if (rc) return rc;
        smax = 0;
      }
      sb.j[sb.n++] = j;
      smax = std::max<int64_t>(smax, o.cols * (o.rows + (o.bias_row ? 1 : 0)));
    }
  }
  int rc = flush(vb, vmax, true);
  if (rc) return rc;
  return flush(sb, smax, false);
}
