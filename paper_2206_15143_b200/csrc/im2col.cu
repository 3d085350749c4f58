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
  return flush(sb, smax, false);
}
