// Sample-major patch matrix for conv A factors:  out[k*ld + r] = X[r, k].
//
// X is the implicit-im2col linear form (reference conv convention, SURVEY
// section 8(a) A3): rows (c,i,j) [DPK_OPND_IM2COL] or (i,j,c)
// [DPK_OPND_IM2COL_TAPMAJOR], columns k = (n, oh, ow); zero padding outside
// the image; the bias ones row last.  HBM-bound copy: with a channels-last
// input and tap-major rows, each (pixel, tap) is one contiguous run of C floats
// moved as float4s (coalesced reads and writes).  The SYRK then streams the
// result through 2-D TMA as an MN-major operand.
#include <cuda_fp16.h>
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

// ---------------------------------------------------------------- fp16, feature-major
// out[r*ld + k] = half(X[r, k]).  Tiled: NHWC tap-major, C % 8 == 0 -- a block
// gathers 64 output pixels x 32 feature rows (32 channels of one tap, or C-channel runs of several) (coalesced 128-B rows of the
// input, zero outside the image), transposes through shared memory and writes
// 32 rows x 64 halves (128 B each).  Generic: one element per thread, k fastest.
constexpr int K16_PIX = 64;
// A flat 1-D grid: job q owns blocks [first[q], first[q+1]) = its (pixel block,
// 32-row group) pairs, pixel blocks fastest -- no empty blocks for small jobs.
struct K16Batch {
  int n;
  int first[I2C_MAX + 1];
  dpk_im2col_job j[I2C_MAX];
};
constexpr int K16_GROUPS = 16;  // 32-row groups per block (the pixel decode is shared)
__global__ void __launch_bounds__(256) im2col_k16_tiled_kernel(const __grid_constant__ K16Batch b) {
  // Each group: 64 pixels x 32 channels of one tap.  Thread t loads the 4 channels
  // 4*(t&7).. of the two adjacent pixels 2*(t>>3), 2*(t>>3)+1 (8 threads cover one
  // pixel's 128-B row: coalesced), packs them as half2 (pixel pair) per channel into a
  // [32 rows][32 words] fp16 tile whose word column is XOR-swizzled by 4*(row/4) --
  // conflict-free for these stores and for the 16-B row reads -- then every thread
  // writes 8 halves (16 B) of one channel row.  ~3 instructions per element.
  __shared__ __align__(16) uint32_t T[2][32 * 32];
  int q = 0;
  while (q + 1 < b.n && b.first[q + 1] <= static_cast<int>(blockIdx.x)) ++q;
  const dpk_im2col_job& J = b.j[q];
  const dpk_operand& o = J.x;
  const int local = static_cast<int>(blockIdx.x) - b.first[q];
  const int kblocks = static_cast<int>((o.cols + K16_PIX - 1) / K16_PIX);
  const int gb = local / kblocks;  // block of K16_GROUPS row groups
  const int64_t k0 = static_cast<int64_t>(local - gb * kblocks) * K16_PIX;
  // job parameters into registers once (a dynamically indexed __grid_constant__
  // struct is otherwise re-read from the constant bank at every use)
  const int OW = o.OW, ohw = o.OH * OW, C = o.C, H = o.H, W = o.W, kw = o.kw;
  const int sh = o.sh, sw = o.sw, dh = o.dh, dw = o.dw;
  const int shs = static_cast<int>(o.shs), sws = static_cast<int>(o.sws);  // within one image
  const int64_t cols = o.cols, ld = J.ld;
  const int tid = threadIdx.x;
  const int pp = tid >> 3, qq = tid & 7;
  // the thread's two pixels, decoded once: image base pointer and tap-0 input coordinates
  const float* base[2];
  int ih0[2], iw0[2];
  bool pin[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t k = k0 + 2 * pp + h;
    pin[h] = k < cols;
    const uint32_t kk = pin[h] ? static_cast<uint32_t>(k) : 0u;  // cols < 2^31 (k16_tiled_ok)
    const uint32_t n = kk / static_cast<uint32_t>(ohw);
    const int rem = static_cast<int>(kk - n * static_cast<uint32_t>(ohw));
    const int oh = rem / OW, ow = rem - (rem / OW) * OW;
    base[h] = o.data + static_cast<int64_t>(n) * o.sn;
    ih0[h] = oh * sh - o.ph;
    iw0[h] = ow * sw - o.pw;
  }
  const float sc = J.amax ? ldexpf(1.0f, -prescale_exponent(__ldg(J.amax))) : 1.0f;  // exact 2^-e
  const int rows = o.rows, nrg = (rows + 31) / 32, kh = o.kh;
  int rg = gb * K16_GROUPS;
  // this thread's load row r = 32 rg + 4 qq: its tap (ti, tj) and channel c, walked
  // incrementally (+32 rows per group; a tap boundary falls on a multiple of 4 rows
  // since C % 4 == 0, so the thread's 4 channels never straddle one).  C % 32 == 0
  // keeps the whole warp on one tap; C = 16 puts two taps in one row group.
  int c = 32 * rg + 4 * qq, ti, tj;
  {
    const int tap = c / C;
    c -= tap * C;
    ti = tap / kw;
    tj = tap - ti * kw;
  }
  // store-phase coordinates: row = tid >> 3 (channel), segment = tid & 7 (8 pixels)
  const int srow = tid >> 3, sseg = tid & 7;
  const int64_t kk0 = k0 + sseg * 8;
  __half* out = reinterpret_cast<__half*>(J.out) + static_cast<int64_t>(32 * rg + srow) * ld + kk0;
  const int rsw = (4 * sseg) ^ (4 * (srow >> 2));  // swizzled word of the store-phase read
  const int wcol = pp ^ (4 * qq);                  // rows 4qq..4qq+3 share the swizzle 4*qq
  for (int g = 0; g < K16_GROUPS; ++g, ++rg) {
    if (rg >= nrg) break;
    uint32_t* Tb = T[g & 1];
    float4 v[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      v[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      const int ih = ih0[h] + ti * dh, iw = iw0[h] + tj * dw;
      if (pin[h] && ti < kh && static_cast<unsigned>(ih) < static_cast<unsigned>(H) &&
          static_cast<unsigned>(iw) < static_cast<unsigned>(W))
        v[h] = __ldg(reinterpret_cast<const float4*>(base[h] + (ih * shs + iw * sws + c)));
    }
    const __half2 h0 = __floats2half2_rn(v[0].x * sc, v[1].x * sc);
    const __half2 h1 = __floats2half2_rn(v[0].y * sc, v[1].y * sc);
    const __half2 h2 = __floats2half2_rn(v[0].z * sc, v[1].z * sc);
    const __half2 h3 = __floats2half2_rn(v[0].w * sc, v[1].w * sc);
    uint32_t* tw = Tb + 4 * qq * 32 + wcol;
    tw[0] = *reinterpret_cast<const uint32_t*>(&h0);
    tw[32] = *reinterpret_cast<const uint32_t*>(&h1);
    tw[64] = *reinterpret_cast<const uint32_t*>(&h2);
    tw[96] = *reinterpret_cast<const uint32_t*>(&h3);
    __syncthreads();  // (double-buffered T: one barrier per group)
    const uint4 w = *reinterpret_cast<const uint4*>(Tb + srow * 32 + rsw);
    if (32 * rg + srow < rows) {  // the last group of d % 32 != 0 (C = 16 with an odd tap count)
      if (kk0 + 8 <= cols) {
        __stcs(reinterpret_cast<uint4*>(out), w);
      } else {
        const __half* hv = reinterpret_cast<const __half*>(&w);
        for (int e = 0; e < 8 && kk0 + e < cols; ++e) out[e] = hv[e];
      }
    }
    out += 32 * ld;
    c += 32;
    while (c >= C) {
      c -= C;
      if (++tj == kw) {
        tj = 0;
        ++ti;
      }
    }
  }
}

__global__ void __launch_bounds__(256) im2col_k16_generic_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const int d = o.rows + (o.bias_row ? 1 : 0);
  const int kk = o.kh * o.kw;
  const int ohw = o.OH * o.OW;
  const int64_t total = static_cast<int64_t>(d) * o.cols;
  __half* out = reinterpret_cast<__half*>(J.out);
  const float sc = J.amax ? ldexpf(1.0f, -prescale_exponent(__ldg(J.amax))) : 1.0f;  // exact 2^-e
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(e / o.cols);
    const int64_t k = e - static_cast<int64_t>(r) * o.cols;
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
      const int n = static_cast<int>(k / ohw);
      const int rem = static_cast<int>(k - static_cast<int64_t>(n) * ohw);
      const int oh = rem / o.OW, ow = rem - (rem / o.OW) * o.OW;
      const int ih = oh * o.sh - o.ph + i * o.dh, iw = ow * o.sw - o.pw + j * o.dw;
      v = 0.0f;
      if (static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) && static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
        v = __ldg(o.data + static_cast<int64_t>(n) * o.sn + static_cast<int64_t>(c) * o.sc +
                  static_cast<int64_t>(ih) * o.shs + static_cast<int64_t>(iw) * o.sws);
    }
    out[static_cast<int64_t>(r) * J.ld + k] = __float2half_rn(v * sc);
  }
}

// fp16 feature-major from the row-staged layout (small-C stems, any input strides):
// one CTA per output row (n, oh) stages the kh input rows in smem exactly like
// im2col_rows_kernel, expands them into a [d][OW] fp16 tile in smem -- lanes walk
// the feature rows r (consecutive staged words: conflict-free reads; the tile's
// odd word stride makes the transposed half2 writes conflict-free) -- and writes
// the tile's rows to global memory as 16-byte stores (OW % 8 == 0).
constexpr int K16R_TILE_WORDS_MAX = 12 * 1024;  // d * (OW/2 + 1) words of the fp16 tile
__global__ void __launch_bounds__(ROWS_THREADS) im2col_k16_rows_kernel(const __grid_constant__ I2cBatch b) {
  extern __shared__ float sm[];
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const RowsGeom g = rows_geom(o);
  const int d = o.rows + (o.bias_row ? 1 : 0);
  const int C = o.C, OW = o.OW, OH = o.OH, kh = o.kh, rowlen = g.rowlen;
  const int half_ow = OW >> 1;
  const int tw = half_ow + 1;  // tile word stride (odd when OW/2 is even)
  const int64_t ld = J.ld, nrows = o.cols / OW;
  float* stage = sm;
  int* off = reinterpret_cast<int*>(sm + kh * rowlen);
  uint32_t* tile = reinterpret_cast<uint32_t*>(off + d);
  const float sc = J.amax ? ldexpf(1.0f, -prescale_exponent(__ldg(J.amax))) : 1.0f;  // exact 2^-e
  for (int r = threadIdx.x; r < d; r += ROWS_THREADS) {
    int v = -2;  // the bias row
    if (r < o.rows) {
      int c, i, j;
      if (o.kind == DPK_OPND_IM2COL) {
        const int kk = o.kh * o.kw;
        c = r / kk;
        const int t = r - c * kk;
        i = t / o.kw;
        j = t - i * o.kw;
      } else {
        const int t = r / C;
        c = r - t * C;
        i = t / o.kw;
        j = t - i * o.kw;
      }
      v = i * rowlen + j * o.dw * C + c;
    }
    off[r] = v;
  }
  const int shift = o.sw * C;
  for (int64_t row = blockIdx.x; row < nrows; row += gridDim.x) {
    const int n = static_cast<int>(row / OH);
    const int oh = static_cast<int>(row - static_cast<int64_t>(n) * OH);
    const float* base = o.data + static_cast<int64_t>(n) * o.sn;
    __syncthreads();
    // stage: input rows oh*sh - ph + i*dh (i < kh), padded columns, channel-interleaved
    // (thread over padded input columns, channels inner: no division per element)
    for (int i = 0; i < kh; ++i) {
      const int ih = oh * o.sh - o.ph + i * o.dh;
      const bool rin = static_cast<unsigned>(ih) < static_cast<unsigned>(o.H);
      for (int wq = threadIdx.x; wq < g.wp; wq += ROWS_THREADS) {
        const int iw = wq - g.padl;
        const bool in = rin && static_cast<unsigned>(iw) < static_cast<unsigned>(o.W);
        const float* src = base + static_cast<int64_t>(ih) * o.shs + static_cast<int64_t>(iw) * o.sws;
        for (int c = 0; c < C; ++c)
          stage[i * rowlen + wq * C + c] = in ? __ldg(src + static_cast<int64_t>(c) * o.sc) * sc : 0.0f;
      }
    }
    __syncthreads();
    // expand into the fp16 tile: warp w takes pixel pairs p = w, w+8, ...; lanes walk the
    // feature rows r (consecutive staged words: conflict-free; odd tile stride)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int p = warp; p < half_ow; p += ROWS_THREADS / 32) {
      const int s0 = 2 * p * shift;
      for (int r = lane; r < d; r += 32) {
        const int t = off[r];
        float a, c2;
        if (t >= 0) {
          a = stage[t + s0];
          c2 = stage[t + s0 + shift];
        } else {
          a = c2 = (t == -2 ? sc : 0.0f);  // the bias row holds 1 (prescaled)
        }
        const __half2 hv = __floats2half2_rn(a, c2);
        tile[r * tw + p] = *reinterpret_cast<const uint32_t*>(&hv);
      }
    }
    __syncthreads();
    // rows out as 16-byte stores: half-warp h of warp w takes rows r = 2(w + 8j) + h,
    // its lanes the row's 8-half segments
    __half* out = reinterpret_cast<__half*>(J.out) + row * OW;
    const int segs = OW >> 3;
    const int hh = lane >> 4, sq = lane & 15;
    for (int r = 2 * warp + hh; r < d; r += 2 * (ROWS_THREADS / 32)) {
      for (int q = sq; q < segs; q += 16) {
        const uint32_t* tr = tile + r * tw + 4 * q;
        uint4 w;
        w.x = tr[0];
        w.y = tr[1];
        w.z = tr[2];
        w.w = tr[3];
        __stcs(reinterpret_cast<uint4*>(out + r * ld + 8 * q), w);
      }
    }
  }
}

// ---------------------------------------------------------------- amax for the fp16 prescale
// grid (x: blocks striding over the input, y: job).  Dense inputs (the four strides
// a permutation of a packed layout, any memory format) are read as one flat range
// (float4 when aligned); others element by element through the strides.  |x| as
// int bits is order-preserving for non-negative floats (NaN bits sort above inf).
__global__ void amax_zero_kernel(const __grid_constant__ I2cBatch b) {
  for (int i = threadIdx.x; i < b.n; i += blockDim.x)
    if (b.j[i].amax) *b.j[i].amax = b.j[i].x.bias_row ? __float_as_int(1.0f) : 0;
}

__device__ __forceinline__ int abs_bits(float v) { return __float_as_int(v) & 0x7fffffff; }

__global__ void __launch_bounds__(256) amax_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  if (!J.amax) return;
  const dpk_operand& o = J.x;
  const int64_t numel = static_cast<int64_t>(o.cols / (static_cast<int64_t>(o.OH) * o.OW)) * o.C * o.H * o.W;
  const int64_t nb = o.cols / (static_cast<int64_t>(o.OH) * o.OW);
  int m = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t first = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // dense: max offset + 1 == numel (strides a permutation of a packed layout)
  const int64_t span = (nb - 1) * o.sn + (o.C - 1) * o.sc + (o.H - 1) * o.shs + (o.W - 1) * o.sws + 1;
  if (span == numel) {
    if ((reinterpret_cast<uintptr_t>(o.data) & 15) == 0) {
      const float4* p4 = reinterpret_cast<const float4*>(o.data);
      for (int64_t e = first; e < numel / 4; e += stride) {
        const float4 v = __ldg(p4 + e);
        m = max(m, max(max(abs_bits(v.x), abs_bits(v.y)), max(abs_bits(v.z), abs_bits(v.w))));
      }
      for (int64_t e = (numel / 4) * 4 + first; e < numel; e += stride) m = max(m, abs_bits(__ldg(o.data + e)));
    } else {
      for (int64_t e = first; e < numel; e += stride) m = max(m, abs_bits(__ldg(o.data + e)));
    }
  } else {
    const int64_t hw = static_cast<int64_t>(o.H) * o.W, chw = o.C * hw;
    for (int64_t e = first; e < numel; e += stride) {
      const int64_t n = e / chw;
      int64_t r = e - n * chw;
      const int64_t c = r / hw;
      r -= c * hw;
      const int64_t h = r / o.W, w = r - (r / o.W) * o.W;
      m = max(m, abs_bits(__ldg(o.data + n * o.sn + c * o.sc + h * o.shs + w * o.sws)));
    }
  }
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(J.amax, m);
}

// ---------------------------------------------------------------- fp16 NHWC copy for the implicit SYRK
// out = half(x * 2^-e), the dense channels-last input itself (N*H*W*C halves, the
// same element order): the operand DPK_OPND_IM2COL_TAPMAJOR_F16 then gathers the
// patches by TMA im2col loads inside the SYRK, so no patch matrix is ever written.
// 8 elements per thread: two float4 loads, one 16-byte store.
bool convert_ok(const dpk_im2col_job& j) {
  const dpk_operand& o = j.x;
  const int64_t hw = static_cast<int64_t>(o.H) * o.W;
  return o.kind == DPK_OPND_IM2COL_TAPMAJOR && o.data != nullptr && j.out != nullptr && o.C % 8 == 0 &&
         o.sc == 1 && o.sws == o.C && o.shs == static_cast<int64_t>(o.W) * o.C && o.sn == hw * o.C && o.OH > 0 &&
         o.OW > 0 && o.cols % (static_cast<int64_t>(o.OH) * o.OW) == 0 &&
         (reinterpret_cast<uintptr_t>(o.data) & 15) == 0 && (reinterpret_cast<uintptr_t>(j.out) & 15) == 0;
}

__global__ void __launch_bounds__(256) convert_f16_kernel(const __grid_constant__ I2cBatch b) {
  const dpk_im2col_job& J = b.j[blockIdx.y];
  const dpk_operand& o = J.x;
  const int64_t n8 = (o.cols / (static_cast<int64_t>(o.OH) * o.OW)) * o.sn / 8;
  const float sc = J.amax ? ldexpf(1.0f, -prescale_exponent(__ldg(J.amax))) : 1.0f;  // exact 2^-e
  const float4* src = reinterpret_cast<const float4*>(o.data);
  uint4* dst = reinterpret_cast<uint4*>(J.out);
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n8;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float4 a = __ldcs(src + 2 * e), c = __ldcs(src + 2 * e + 1);
    const __half2 h0 = __floats2half2_rn(a.x * sc, a.y * sc), h1 = __floats2half2_rn(a.z * sc, a.w * sc);
    const __half2 h2 = __floats2half2_rn(c.x * sc, c.y * sc), h3 = __floats2half2_rn(c.z * sc, c.w * sc);
    uint4 w;
    w.x = *reinterpret_cast<const uint32_t*>(&h0);
    w.y = *reinterpret_cast<const uint32_t*>(&h1);
    w.z = *reinterpret_cast<const uint32_t*>(&h2);
    w.w = *reinterpret_cast<const uint32_t*>(&h3);
    dst[e] = w;  // default store: the SYRK reads it next, from L2 where it still fits
  }
}

bool k16_rows_ok(const dpk_im2col_job& j) {
  const dpk_operand& o = j.x;
  const RowsGeom g = rows_geom(o);
  const int d = o.rows + (o.bias_row ? 1 : 0);
  const size_t smem = (static_cast<size_t>(o.kh) * g.rowlen + d) * 4 + static_cast<size_t>(d) * (o.OW / 2 + 1) * 4;
  return o.OW % 8 == 0 && o.cols % o.OW == 0 && smem <= static_cast<size_t>(ROWS_SMEM_MAX) &&
         static_cast<int64_t>(d) * (o.OW / 2 + 1) <= K16R_TILE_WORDS_MAX;
}

bool k16_tiled_ok(const dpk_im2col_job& j) {
  const dpk_operand& o = j.x;
  return o.kind == DPK_OPND_IM2COL_TAPMAJOR && o.sc == 1 && o.C % 8 == 0 && !o.bias_row &&
         (reinterpret_cast<uintptr_t>(o.data) & 15) == 0 && o.sn % 4 == 0 && o.shs % 4 == 0 && o.sws % 4 == 0 &&
         static_cast<int64_t>(o.H) * o.shs + static_cast<int64_t>(o.W) * o.sws + o.C < (int64_t{1} << 31) &&
         o.cols < (int64_t{1} << 31);
}

}  // namespace
}  // namespace dpk

extern "C" int dpk_im2col_materialize_f16(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_im2col_materialize_f16: bad job list");
    return DPK_EARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  thread_local dpk::K16Batch tb;
  thread_local dpk::I2cBatch gb, rbf;
  tb.n = gb.n = rbf.n = 0;
  size_t rsm = 0;
  auto flush_r = [&]() -> int {
    if (rbf.n == 0) return DPK_OK;
    static std::atomic<uint64_t> attr_on{0};
    if (dpk::first_on_device(attr_on)) {
      cudaFuncSetAttribute(dpk::im2col_k16_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           dpk::ROWS_SMEM_MAX);
    }
    int64_t rows = 0;
    for (int i = 0; i < rbf.n; ++i) rows = std::max<int64_t>(rows, rbf.j[i].x.cols / rbf.j[i].x.OW);
    const int gx = static_cast<int>(std::min<int64_t>(rows, 4 * 148));
    dpk::im2col_k16_rows_kernel<<<dim3(gx, rbf.n), dpk::ROWS_THREADS, rsm, st>>>(rbf);
    dpk::note_launch();
    rbf.n = 0;
    rsm = 0;
    return dpk::cuda_status(cudaGetLastError(), "im2col_k16_rows_kernel launch");
  };
  tb.first[0] = 0;
  int64_t gmax = 0;
  auto flush_t = [&]() -> int {
    if (tb.n == 0) return DPK_OK;
    dpk::im2col_k16_tiled_kernel<<<tb.first[tb.n], 256, 0, st>>>(tb);
    dpk::note_launch();
    tb.n = 0;
    return dpk::cuda_status(cudaGetLastError(), "im2col_k16_tiled_kernel launch");
  };
  auto flush_g = [&]() -> int {
    if (gb.n == 0) return DPK_OK;
    const int gx = static_cast<int>(std::min<int64_t>((gmax + 255) / 256, 4 * 148 * 8));
    dpk::im2col_k16_generic_kernel<<<dim3(gx, gb.n), 256, 0, st>>>(gb);
    dpk::note_launch();
    gb.n = 0;
    gmax = 0;
    return dpk::cuda_status(cudaGetLastError(), "im2col_k16_generic_kernel launch");
  };
  for (int i = 0; i < n_jobs; ++i) {
    const dpk_im2col_job& j = jobs[i];
    const dpk_operand& o = j.x;
    if ((o.kind != DPK_OPND_IM2COL && o.kind != DPK_OPND_IM2COL_TAPMAJOR) || j.out == nullptr || o.data == nullptr ||
        o.cols < 1 || o.rows != o.C * o.kh * o.kw || j.ld < o.cols || j.ld % 8 != 0 ||
        (reinterpret_cast<uintptr_t>(j.out) & 15) != 0 || o.OH * static_cast<int64_t>(o.OW) < 1) {
      dpk::set_error("dpk_im2col_materialize_f16: invalid job " + std::to_string(i));
      return DPK_EARG;
    }
    const int64_t nblk = ((o.cols + dpk::K16_PIX - 1) / dpk::K16_PIX) *
                         ((((o.rows + 31) / 32) + dpk::K16_GROUPS - 1) / dpk::K16_GROUPS);
    if (dpk::k16_tiled_ok(j) && nblk < (int64_t{1} << 30)) {
      if (tb.n == dpk::I2C_MAX || tb.first[tb.n] + nblk >= (int64_t{1} << 31)) {
        int rc = flush_t();
        if (rc) return rc;
        tb.first[0] = 0;
      }
      tb.j[tb.n] = j;
      tb.first[tb.n + 1] = tb.first[tb.n] + static_cast<int>(nblk);
      ++tb.n;
    } else if (dpk::k16_rows_ok(j)) {
      if (rbf.n == dpk::I2C_MAX) {
        int rc = flush_r();
        if (rc) return rc;
      }
      rbf.j[rbf.n++] = j;
      const dpk::RowsGeom g = dpk::rows_geom(o);
      const int d = o.rows + (o.bias_row ? 1 : 0);
      rsm = std::max(rsm, (static_cast<size_t>(o.kh) * g.rowlen + d) * 4 + static_cast<size_t>(d) * (o.OW / 2 + 1) * 4);
    } else {
      if (gb.n == dpk::I2C_MAX) {
        int rc = flush_g();
        if (rc) return rc;
      }
      gb.j[gb.n++] = j;
      gmax = std::max<int64_t>(gmax, static_cast<int64_t>(o.rows + (o.bias_row ? 1 : 0)) * o.cols);
    }
  }
  int rc = flush_t();
  if (rc) return rc;
  rc = flush_r();
  if (rc) return rc;
  return flush_g();
}

extern "C" int dpk_im2col_amax(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_im2col_amax: bad job list");
    return DPK_EARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  thread_local dpk::I2cBatch ab;
  for (int first = 0; first < n_jobs; first += dpk::I2C_MAX) {
    const int cnt = std::min(dpk::I2C_MAX, n_jobs - first);
    ab.n = cnt;
    int64_t most = 0;
    for (int i = 0; i < cnt; ++i) {
      const dpk_im2col_job& j = jobs[first + i];
      const dpk_operand& o = j.x;
      if ((o.kind != DPK_OPND_IM2COL && o.kind != DPK_OPND_IM2COL_TAPMAJOR) || o.data == nullptr || o.cols < 1 ||
          o.OH < 1 || o.OW < 1 ||
          o.cols % (static_cast<int64_t>(o.OH) * o.OW) != 0) {
        dpk::set_error("dpk_im2col_amax: invalid job " + std::to_string(first + i));
        return DPK_EARG;
      }
      ab.j[i] = j;
      most = std::max<int64_t>(most, (o.cols / (static_cast<int64_t>(o.OH) * o.OW)) * o.C * o.H * o.W);
    }
    dpk::amax_zero_kernel<<<1, 128, 0, st>>>(ab);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "amax_zero_kernel launch");
    if (rc) return rc;
    const int gx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((most / 4 + 255) / 256, 2 * 148)));
    dpk::amax_kernel<<<dim3(gx, cnt), 256, 0, st>>>(ab);
    dpk::note_launch();
    rc = dpk::cuda_status(cudaGetLastError(), "amax_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

extern "C" int dpk_im2col_convert_f16(const dpk_im2col_job* jobs, int n_jobs, dpk_stream_t stream) {
  if (n_jobs == 0) return DPK_OK;
  if (n_jobs < 0 || jobs == nullptr) {
    dpk::set_error("dpk_im2col_convert_f16: bad job list");
    return DPK_EARG;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  thread_local dpk::I2cBatch cb;
  for (int first = 0; first < n_jobs; first += dpk::I2C_MAX) {
    const int cnt = std::min(dpk::I2C_MAX, n_jobs - first);
    cb.n = cnt;
    int64_t most = 0;
    for (int i = 0; i < cnt; ++i) {
      const dpk_im2col_job& j = jobs[first + i];
      if (!dpk::convert_ok(j)) {
        dpk::set_error("dpk_im2col_convert_f16: job " + std::to_string(first + i) +
                       " needs a dense channels-last fp32 input (DPK_OPND_IM2COL_TAPMAJOR), C % 8 == 0, "
                       "16-byte aligned input and output");
        return DPK_EARG;
      }
      cb.j[i] = j;
      const dpk_operand& o = j.x;
      most = std::max<int64_t>(most, (o.cols / (static_cast<int64_t>(o.OH) * o.OW)) * o.sn / 8);
    }
    const int gx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((most + 255) / 256, 4 * 148)));
    dpk::convert_f16_kernel<<<dim3(gx, cnt), 256, 0, st>>>(cb);
    dpk::note_launch();
    const int rc = dpk::cuda_status(cudaGetLastError(), "convert_f16_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

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
    static std::atomic<uint64_t> attr_on{0};
    if (dpk::first_on_device(attr_on)) {
      cudaFuncSetAttribute(dpk::im2col_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dpk::ROWS_SMEM_MAX);
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
