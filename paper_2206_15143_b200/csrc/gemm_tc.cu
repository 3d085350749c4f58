// Grouped tcgen05 (kind::tf32) GEMM / SYRK engine for sm_100a.
//
//   out[m,n] = alpha * sum_k A[m,k] B[n,k] + beta * cin[m,n]     (EPI_LINEAR)
//   out[m,n] = alpha * sum_k A[m,k] B[n,k] / (max(vr[m],0) max(vc[n],0) + gamma)   (EPI_EIGDIV)
//
// One persistent launch serves a whole group of problems (e.g. all Kronecker
// factors of all owned layers).  Work units are (problem, 128x128 output tile,
// K split).  Warp roles per CTA (12 warps, one CTA per SM):
//   warps 0-3  epilogue: tcgen05.ld the TMEM accumulator (lane = tile row),
//              apply alpha/beta (the fused running average) or the eigen
//              divide, store, mirror lower tiles for symmetric outputs, and
//              run the deterministic split-K fix-up (last split sums partials);
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer;
//   warp 5     TMA issuer: operands that TMA can address (row-major K-major,
//              column-major MN-major, NCHW 1x1 "slab" captures as a 3-D map)
//              are fetched with cp.async.bulk.tensor into 128B-swizzled
//              stages, running ahead through the whole stage ring;
//   warps 6-11 gather / convert: round TMA-landed tiles to TF32 in place (RN
//              mode) or derive the 3xTF32 low parts; everything else -- implicit im2col
//              of NCHW conv inputs (patches never touch HBM), bias rows,
//              unaligned views -- is gathered by the warps with a one-chunk
//              software pipeline and stored in the same canonical K-major
//              SW128 layout.
// Pipelines: smem stages (full / tma / empty barriers), two TMEM accumulators
// full/empty (MMA <-> epilogue) so tile i's epilogue overlaps tile i+1's MMAs.
//
// Reference semantics reproduced (kfaclab 0.1.0): compute_factors
// kfac.py:85-104 (symmetric A = X X^T / M), update_running_average
// kfac.py:107-125 (alpha/beta epilogue), precondition_inverse / _eigen
// kfac.py:165-191 (plain and eigen-divide epilogues).
#include <cuda.h>  // CUtensorMap / enums only; the encoder is fetched through the runtime
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "dpk_internal.h"
#include "dpk_ptx.cuh"

namespace dpk {
bool debug_ts_enabled();
struct ForkLane;
int fork_lane(cudaStream_t st, ForkLane*& out, int purpose);
int fork_begin(ForkLane* L, cudaStream_t st);
int fork_end(ForkLane* L, cudaStream_t st);
cudaStream_t fork_side(ForkLane* L);
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 32;                       // fp32 elements per row of a stage = 128 B
constexpr int TILE_BYTES = BM * BK * 4;      // 16 KB
constexpr int EPI_WARPS = 4;                 // warps 0..3 (one per TMEM lane quadrant)
constexpr int MMA_WARP = 4;
constexpr int TMA_WARP = 5;                               // one elected thread issues all TMA loads
constexpr int PROD_WARP0 = 6;
constexpr int PROD_WARPS = 6;                             // 12 warps total -> up to 168 regs/thread
constexpr int NPROD = PROD_WARPS * 32;                    // 192 gather / convert threads
constexpr int TILE_TASKS = BM * (BK / 4);                 // (row, 16B chunk) tasks per operand tile
constexpr int NTASK = (TILE_TASKS + NPROD - 1) / NPROD;   // 5 tasks per producer thread
constexpr int NTHREADS = (PROD_WARP0 + PROD_WARPS) * 32;  // 384
constexpr int MAXP = 40;                                  // problems per launch (kernel params)
constexpr size_t SCHED_BYTES = GEMM_SCHED_BYTES;          // scheduler counters at the workspace start
static_assert(NPROD % 8 == 0, "im2col chunk sharing needs NPROD % 8 == 0");

// TMA_ROWS_MN3: MN-major operand whose row count is a multiple of 32, fetched as
// ONE 3-D box {32 rows, 32 k, 4 row blocks} per 128-row tile instead of four
// 2-D boxes (same shared-memory image)
// TMA_TAPS: implicit im2col of an NHWC conv input through plain TILED boxes:
// a 5-D map {c32, w, h, n, c-block} over the input itself, one box per (tap,
// channel block) group of 32/64/128 factor rows at the tap-shifted pixel
// coordinates; out-of-image taps are TMA zero fill.  A K chunk is 32 output
// pixels (wb x hb of one image block x nb samples), the same pixel set for every
// row group, so patches never exist in HBM (SYRK only: both operands share the
// map and the K order).  Measured TMA-issue bound.
// TMA_ROWS_K16: K-major fp16 operand (DPK_OPND_ROWS_K_F16), 64 elements per 128-B
// stage row, consumed by kind::f16 MMAs; a K chunk of such a problem covers 64 columns.
// TMA_IM2COL16: implicit im2col of an fp16 NHWC input (DPK_OPND_IM2COL_TAPMAJOR_F16):
// a K chunk is 64 output pixels; per 64-row group (one tap, 64 channels) one TMA
// im2col box of 64 pixels x 128 B lands as the MN-major SWIZZLE_128B kind::f16
// operand (8 KB, two per 128-row tile).
// TMA_ROWS_MN_PLAIN (3xF16 only): an MN-major fp32 tile without swizzle, k rows of
// 128 floats (512 B) -- read by the producer warps, never by the MMA.
enum { TMA_NONE = 0, TMA_ROWS_K = 1, TMA_ROWS_MN = 2, TMA_SLAB = 3, TMA_IM2COL = 4, TMA_ROWS_MN3 = 5, TMA_TAPS = 6,
       TMA_ROWS_K16 = 7, TMA_IM2COL16 = 8, TMA_ROWS_MN_PLAIN = 9 };
__host__ __device__ __forceinline__ bool tma_mn(int kind) {
  return kind == TMA_ROWS_MN || kind == TMA_IM2COL || kind == TMA_ROWS_MN3 || kind == TMA_TAPS ||
         kind == TMA_IM2COL16;
}
__host__ __device__ __forceinline__ bool tma_f16(int kind) { return kind == TMA_ROWS_K16 || kind == TMA_IM2COL16; }

__host__ __device__ __forceinline__ bool is_im2col(int kind) {
  return kind == DPK_OPND_IM2COL || kind == DPK_OPND_IM2COL_TAPMAJOR;
}

struct alignas(64) Problem {
  CUtensorMap tmap_a;  // valid iff tma_a != TMA_NONE
  CUtensorMap tmap_b;
  dpk_operand a;
  dpk_operand b;
  float* out;
  const float* cin;
  const float* vrow;
  const float* vcol;
  float* partials;  // split-K partial slots (ntiles * splits * BM * BN), splits > 1
  float* out_t;
  int64_t ldt;
  int64_t ldo;
  int64_t ldc;
  const int32_t* alpha_amax;  // optional: prescaled fp16 operands, alpha *= 2^(2e)
  const int32_t* amax_a;      // 3xF16: operand amax bits (scales 2^-e_a, 2^-e_b; alpha *= 2^(e_a+e_b))
  const int32_t* amax_b;
  float alpha, beta, gamma;
  int M, N;
  int symmetric, same_ab, epi;  // symmetric: 1 lower tiles + mirror, 2 lower tiles only
  int tiles_n, ntiles, splits;
  int chunks, cps;  // K chunks of 32, chunks per split
  int unit_begin;
  int tma_a, tma_b;
  int slab_cpn;     // TMA_SLAB: chunks per sample (K index = (sample, 32-pixel chunk));
                    // TMA_TAPS: wb | hb << 6 | group boxes << 12 | sample blocks << 16
  int tri_a, tri_b; // TRI_*: per-tile K clipping for triangular operands
  int order;        // tile visiting order (non-symmetric): 0 row-major, 1 row-major reversed,
                    // 2 column-major, 3 column-major reversed -- heaviest K ranges first
};

struct Batch {
  int nprob;
  int total_units;
  int debug_ts;   // record %globaltimer checkpoints of CTA 0 (dpk_debug_timestamps)
  int producers;  // 0: every operand tile arrives by TMA ready for the MMA (no gather /
                  // conversion anywhere in the launch) -> warps 6-11 sit the launch out
  int dynamic;    // 1: units handed out by an atomic counter (sched[0]); 0: static round robin
  int* sched;     // [0] next unit, [1] finished workers (the last one resets both)
  Problem p[MAXP];
};
static_assert(sizeof(Batch) <= 32764, "kernel parameter space is 32764 bytes");

__device__ unsigned long long g_dbg_ts[16];
// per-unit checkpoints of CTA 0 (DPK_DEBUG_TS=1): [it][0] MMA start (accumulator free),
// [1] first chunk's data ready, [2] last MMA issued, [3] epilogue start (accumulator
// full), [4] epilogue end
constexpr int DBG_UNITS = 64;
__device__ unsigned long long g_dbg_unit[DBG_UNITS][5];
__device__ __forceinline__ void dbg_unit(const Batch& bt, int it, int slot) {
  if (bt.debug_ts && blockIdx.x == 0 && it < DBG_UNITS) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dbg_unit[it][slot] = t;
  }
}

__device__ __forceinline__ void dbg_ts(const Batch& bt, int slot) {
  if (bt.debug_ts && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dbg_ts[slot] = t;
  }
}

// Every tcgen05 launch asks for the whole opt-in shared memory of an SM (227 KB),
// so none of its CTAs ever shares an SM with another kernel's CTA.  Otherwise a
// concurrently running library kernel (cuDNN/cuBLAS sm_100 kernels hold TMEM
// too) could sit on the same SM holding TMEM while it waits for peer CTAs that
// cannot be scheduled because our persistent CTAs occupy every SM, and our CTA
// would block in tcgen05.alloc behind it: a deadlock observed when the factor
// pipeline runs under the backward pass (early=True).
constexpr int SMEM_SM_EXCL = 232448;

template <int NPASS>
struct Cfg {
  static constexpr int STAGES = NPASS == 1 ? 6 : 3;
  static constexpr int OPS = NPASS == 1 ? 2 : 4;  // A, B (+ A_lo, B_lo)
  static constexpr int STAGE_BYTES = OPS * TILE_BYTES;
  static constexpr int NSLOT = 4;  // unit-id ring between the scheduler thread and the roles
  static constexpr int BAR_BYTES = 8 * (3 * STAGES + 4) + 16 + 8 * 2 * NSLOT + 4 * NSLOT;
  static constexpr int EPI_BYTES = EPI_WARPS * 32 * 33 * 4;  // per-warp 32x32 (+1 pad) staging
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + BAR_BYTES + EPI_BYTES;
  static_assert(SMEM <= SMEM_SM_EXCL, "stage ring exceeds the SM's shared memory");
};

__device__ __forceinline__ void decode_unit(const Batch& bt, int u, int& pi, int& tm, int& tn, int& tile,
                                            int& split) {
  int p = 0;
  while (p + 1 < bt.nprob && bt.p[p + 1].unit_begin <= u) ++p;
  const Problem& P = bt.p[p];
  int local = u - P.unit_begin;
  // split-major: CTAs of one wave take different tiles of the same K range, so
  // each K slab of the operands is fetched from DRAM once and shared through L2
  split = local / P.ntiles;
  const int v = local - split * P.ntiles;  // visiting position -> canonical (row-major) tile index
  if (P.order == 0 || P.symmetric) {
    tile = v;
  } else if (P.order == 1) {
    tile = P.ntiles - 1 - v;
  } else {
    const int tiles_m = P.ntiles / P.tiles_n;
    const int w = P.order == 3 ? P.ntiles - 1 - v : v;
    const int cn = w / tiles_m;
    tile = (w - cn * tiles_m) * P.tiles_n + cn;
  }
  if (P.symmetric) {
    int r = static_cast<int>((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= tile) ++r;
    while (r * (r + 1) / 2 > tile) --r;
    tm = r;
    tn = tile - r * (r + 1) / 2;
  } else {
    tm = tile / P.tiles_n;
    tn = tile - tm * P.tiles_n;
  }
  pi = p;
}

// K chunks [kc0, kc1) of one unit: the tile's structural range (triangular
// operands) split into cps-chunk pieces.  May be empty for trailing splits.
template <int CG>
__device__ __forceinline__ void chunk_range(const Problem& P, int tm, int tn, int split, int& kc0, int& kc1) {
  constexpr int TC = 128 * CG / BK;  // K chunks per unit tile edge
  int lo = 0, hi = P.chunks;
  if (P.tri_a == TRI_UPPER) lo = max(lo, tm * TC);
  if (P.tri_b == TRI_UPPER) lo = max(lo, tn * TC);
  if (P.tri_a == TRI_LOWER) hi = min(hi, (tm + 1) * TC);
  if (P.tri_b == TRI_LOWER) hi = min(hi, (tn + 1) * TC);
  if (P.tri_a == TRI_BLOCK) {
    lo = max(lo, tm * TC);
    hi = min(hi, (tm + 1) * TC);
  }
  if (P.tri_b == TRI_BLOCK) {
    lo = max(lo, tn * TC);
    hi = min(hi, (tn + 1) * TC);
  }
  kc0 = lo + split * P.cps;
  kc1 = min(hi, kc0 + P.cps);
}

// ------------------------------------------------------------------ manual producer
// A row task: one (row, 16-byte chunk) of a 128 x 32 stage tile.
struct RowTask {
  int64_t off;  // element offset of the row inside the operand
  int packed;   // bits 0-1 flag (0 zero row, 1 data row, 2 ones/bias row),
                // bits 2-16 im2col column offset j*dw, bits 17-31 row offset i*dh
  __device__ __forceinline__ int flag() const { return packed & 3; }
  __device__ __forceinline__ int iw() const { return (packed >> 2) & 0x7FFF; }
  __device__ __forceinline__ int ih() const { return packed >> 17; }
};

__device__ __forceinline__ bool kfast(const dpk_operand& o) { return o.kind != DPK_OPND_ROWS_MN; }

// task q = ptid + NPROD*j (q < TILE_TASKS).  k-fast: 8 lanes cover one 128 B row
// segment; row-fast: consecutive lanes take consecutive rows (column-major sources).
__device__ __forceinline__ bool task_row_chunk(bool kf, int ptid, int j, int& row, int& chunk) {
  const int q = ptid + NPROD * j;
  if (kf) {
    row = q >> 3;
    chunk = q & 7;
  } else {
    row = q & (BM - 1);
    chunk = q >> 7;
  }
  return q < TILE_TASKS;
}

__device__ __forceinline__ void setup_tasks(const dpk_operand& o, int row0, int ptid, RowTask (&t)[NTASK]) {
  const bool kf = kfast(o);
#pragma unroll
  for (int j = 0; j < NTASK; ++j) {
    int row, chunk;
    const bool valid = task_row_chunk(kf, ptid, j, row, chunk);
    const int r = row0 + row;
    t[j].off = 0;
    t[j].packed = 0;
    if (!valid) continue;
    if (r < o.rows) {
      t[j].packed = 1;
      if (o.kind == DPK_OPND_ROWS_K) {
        t[j].off = static_cast<int64_t>(r) * o.ld;
      } else if (o.kind == DPK_OPND_ROWS_MN) {
        t[j].off = r;
      } else {
        int c, i, jj;
        if (o.kind == DPK_OPND_IM2COL) {  // rows (c, i, j): F.unfold / weight.view order
          const int kk = o.kh * o.kw;
          c = r / kk;
          const int rem = r - c * kk;
          i = rem / o.kw;
          jj = rem - i * o.kw;
        } else {  // TAPMAJOR rows (i, j, c): channels-last weight order
          const int tap = r / o.C;
          c = r - tap * o.C;
          i = tap / o.kw;
          jj = tap - i * o.kw;
        }
        const int ihd = i * o.dh, iwd = jj * o.dw;
        t[j].packed = 1 | (iwd << 2) | (ihd << 17);
        t[j].off = static_cast<int64_t>(c) * o.sc + static_cast<int64_t>(ihd) * o.shs +
                   static_cast<int64_t>(iwd) * o.sws;
      }
    } else {
      t[j].packed = (o.bias_row && r == o.rows) ? 2 : 0;
    }
  }
}

// Gather this thread's tasks of one operand for the k-chunk starting at k_base.
__device__ __forceinline__ void fetch_tasks(const dpk_operand& o, const RowTask (&t)[NTASK], int ptid, int64_t k_base,
                                            float4 (&v)[NTASK]) {
  const bool kf = kfast(o);
  if (is_im2col(o.kind)) {
    // all tasks of this thread share one chunk (NPROD % 8 == 0) -> decompose its 4 sample columns once
    const int64_t k0 = k_base + 4 * (ptid & 7);
    const int ohw = o.OH * o.OW;
    int64_t kb[4];
    int ih0[4], iw0[4];
    bool kv[4];
    {
      int64_t n = k0 / ohw;
      int rem = static_cast<int>(k0 - n * ohw);
      int oh = rem / o.OW;
      int ow = rem - oh * o.OW;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        kv[e] = (k0 + e) < o.cols;
        ih0[e] = oh * o.sh - o.ph;
        iw0[e] = ow * o.sw - o.pw;
        kb[e] = n * o.sn + static_cast<int64_t>(ih0[e]) * o.shs + static_cast<int64_t>(iw0[e]) * o.sws;
        if (++ow == o.OW) {
          ow = 0;
          if (++oh == o.OH) {
            oh = 0;
            ++n;
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NTASK; ++j) {
      float x[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float val = 0.0f;
        if (t[j].flag() == 1) {
          const int ih = ih0[e] + t[j].ih();
          const int iw = iw0[e] + t[j].iw();
          if (kv[e] && static_cast<unsigned>(ih) < static_cast<unsigned>(o.H) &&
              static_cast<unsigned>(iw) < static_cast<unsigned>(o.W))
            val = __ldg(o.data + kb[e] + t[j].off);
        } else if (t[j].flag() == 2) {
          val = kv[e] ? 1.0f : 0.0f;
        }
        x[e] = val;
      }
      v[j] = make_float4(x[0], x[1], x[2], x[3]);
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < NTASK; ++j) {
    int row, chunk;
    task_row_chunk(kf, ptid, j, row, chunk);  // invalid tasks carry flag 0 -> zeros
    const int64_t k0 = k_base + 4 * chunk;
    float x[4] = {0.f, 0.f, 0.f, 0.f};
    if (t[j].flag() == 1) {
      if (o.kind == DPK_OPND_ROWS_K) {
        const float* p = o.data + t[j].off + k0;
        if (k0 + 3 < o.cols && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(p));
          x[0] = q.x;
          x[1] = q.y;
          x[2] = q.z;
          x[3] = q.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (k0 + e < o.cols) x[e] = __ldg(p + e);
        }
      } else {  // ROWS_MN: consecutive lanes read consecutive rows (coalesced)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (k0 + e < o.cols) x[e] = __ldg(o.data + (k0 + e) * o.ld + t[j].off);
      }
    } else if (t[j].flag() == 2) {
#pragma unroll
      for (int e = 0; e < 4; ++e) x[e] = (k0 + e < o.cols) ? 1.0f : 0.0f;
    }
    v[j] = make_float4(x[0], x[1], x[2], x[3]);
  }
}

// Canonical K-major SWIZZLE_128B position of (row, 16B chunk) in a 128 x 32 fp32 tile.
__device__ __forceinline__ uint32_t sw128_offset(int row, int chunk) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}

__device__ __forceinline__ uint32_t tf32_trunc_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

template <int NPASS, bool RN>
__device__ __forceinline__ void store_tasks(const dpk_operand& o, int ptid, uint8_t* tile, uint8_t* tile_lo,
                                            const float4 (&v)[NTASK]) {
  const bool kf = kfast(o);
#pragma unroll
  for (int j = 0; j < NTASK; ++j) {
    int row, chunk;
    if (!task_row_chunk(kf, ptid, j, row, chunk)) continue;
    const uint32_t off = sw128_offset(row, chunk);
    const float x[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (NPASS == 3) {  // hi = what the tensor core reads (truncation), lo = exact remainder
        hi[e] = __float_as_uint(x[e]);
        lo[e] = __float_as_uint(x[e] - __uint_as_float(tf32_trunc_bits(x[e])));
      } else {
        hi[e] = RN ? to_tf32(x[e]) : __float_as_uint(x[e]);
      }
    }
    *reinterpret_cast<uint4*>(tile + off) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    if (NPASS == 3) *reinterpret_cast<uint4*>(tile_lo + off) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// In-place pass over a TMA-filled tile (layout-agnostic, elementwise).
template <int NPASS>
__device__ __forceinline__ void convert_tile(uint8_t* tile, uint8_t* tile_lo, int ptid) {
  uint4* t = reinterpret_cast<uint4*>(tile);
  uint4* l = reinterpret_cast<uint4*>(tile_lo);
  for (int i = ptid; i < TILE_BYTES / 16; i += NPROD) {
    const uint4 v = t[i];
    const float x[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
    uint32_t r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e)
      r[e] = (NPASS == 3) ? __float_as_uint(x[e] - __uint_as_float(tf32_trunc_bits(x[e]))) : to_tf32(x[e]);
    if (NPASS == 3)
      l[i] = make_uint4(r[0], r[1], r[2], r[3]);
    else
      t[i] = make_uint4(r[0], r[1], r[2], r[3]);
  }
}

// ---- 3xF16: fp32 -> (hi, lo) fp16 parts of x * sc in K-major SWIZZLE_64B tiles
// (128 rows x 32 k halves = 64 B rows, 8 KB each; hi at dst, lo at dst + 8 KB).
// Element (r, k) of such a tile sits at byte (r>>3)*512 + (r&7)*64 + (((k>>3) ^ ((r>>1)&3)) << 4) + (k&7)*2.
__device__ __forceinline__ uint32_t sw64_chunk_offset(int row, int c) {
  return static_cast<uint32_t>((row >> 3) * 512 + (row & 7) * 64 + ((c ^ ((row >> 1) & 3)) << 4));
}
__device__ __forceinline__ void split_f16(float x, float sc, __half& hi, __half& lo) {
  const float v = x * sc;
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}
constexpr uint32_t F16_TILE = 8192;  // one 128 x 32 fp16 tile

// manual (gathered) operand tasks straight into the fp16 tiles: task (row, fp32 chunk q)
// = k 4q..4q+3 = halves 0-3 or 4-7 of 16-byte chunk q/2
__device__ __forceinline__ void store_tasks_f16x3(const dpk_operand& o, int ptid, uint8_t* dst, float sc,
                                                  const float4 (&v)[NTASK]) {
  const bool kf = kfast(o);
#pragma unroll
  for (int j = 0; j < NTASK; ++j) {
    int row, chunk;
    if (!task_row_chunk(kf, ptid, j, row, chunk)) continue;
    const uint32_t off = sw64_chunk_offset(row, chunk >> 1) + (chunk & 1) * 8;
    const float x[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
    __half h[4], l[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) split_f16(x[e], sc, h[e], l[e]);
    __half2 h01 = __halves2half2(h[0], h[1]), h23 = __halves2half2(h[2], h[3]);
    __half2 l01 = __halves2half2(l[0], l[1]), l23 = __halves2half2(l[2], l[3]);
    *reinterpret_cast<uint2*>(dst + off) =
        make_uint2(*reinterpret_cast<uint32_t*>(&h01), *reinterpret_cast<uint32_t*>(&h23));
    *reinterpret_cast<uint2*>(dst + F16_TILE + off) =
        make_uint2(*reinterpret_cast<uint32_t*>(&l01), *reinterpret_cast<uint32_t*>(&l23));
  }
}

// 8 scaled values -> the 16-byte hi chunk and the 16-byte lo chunk (packed
// conversions: cvt.rn.f16x2.f32 twice and f16x2 -> f32 once per pair)
__device__ __forceinline__ void split8_f16(const float (&x)[8], float sc, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 v = make_float2(x[2 * e] * sc, x[2 * e + 1] * sc);
    const __half2 hh = __float22half2_rn(v);
    const float2 back = __half22float2(hh);
    const __half2 ll = __float22half2_rn(make_float2(v.x - back.x, v.y - back.y));
    h[e] = *reinterpret_cast<const uint32_t*>(&hh);
    l[e] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// a TMA-landed fp32 tile (K-major SW128, or TMA_ROWS_MN_PLAIN) -> hi / lo fp16 tiles.
// K-major: thread -> (row r = idx & 127, 16-byte chunk c = idx >> 7), two 16-byte
// loads (consecutive lanes take consecutive rows: conflict-free with the SW128
// swizzle).  MN plain: thread -> (row pair 2p, 2p+1, chunk c), eight 8-byte loads of
// the pair (a warp reads 256 contiguous bytes per k).  All loads are issued before
// the conversions.
__device__ __forceinline__ void convert_tile_f16x3(const uint8_t* src, bool mn_plain, uint8_t* dst, float sc,
                                                   int ptid) {
  if (mn_plain) {
    for (int idx = ptid; idx < 64 * 4; idx += NPROD) {
      const int p = idx & 63, c = idx >> 6;
      const float2* f = reinterpret_cast<const float2*>(src) + p + (8 * c) * 64;  // k row = 128 floats = 64 float2
      float2 y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = f[e * 64];
      float x0[8], x1[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        x0[e] = y[e].x;
        x1[e] = y[e].y;
      }
      uint4 h, l;
      split8_f16(x0, sc, h, l);
      uint32_t off = sw64_chunk_offset(2 * p, c);
      *reinterpret_cast<uint4*>(dst + off) = h;
      *reinterpret_cast<uint4*>(dst + F16_TILE + off) = l;
      split8_f16(x1, sc, h, l);
      off = sw64_chunk_offset(2 * p + 1, c);
      *reinterpret_cast<uint4*>(dst + off) = h;
      *reinterpret_cast<uint4*>(dst + F16_TILE + off) = l;
    }
    return;
  }
  for (int idx = ptid; idx < 128 * 4; idx += NPROD) {
    const int r = idx & 127, c = idx >> 7;
    const float4 a = *reinterpret_cast<const float4*>(src + sw128_offset(r, 2 * c));
    const float4 b = *reinterpret_cast<const float4*>(src + sw128_offset(r, 2 * c + 1));
    const float x[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    uint4 h, l;
    split8_f16(x, sc, h, l);
    const uint32_t off = sw64_chunk_offset(r, c);
    *reinterpret_cast<uint4*>(dst + off) = h;
    *reinterpret_cast<uint4*>(dst + F16_TILE + off) = l;
  }
}

// 3xTF32 low parts of both TMA-landed tiles of a stage (A at st, B at st + TILE_BYTES,
// lows 2 tiles further): every load of the thread's 16-byte chunks is issued before
// any is converted -- with six producer warps the pass is otherwise bound by the
// shared-memory load latency (measured ~1150 cycles per chunk, more than the
// single-CTA chunk's 12 MMAs).
template <int J0, int NJ>
__device__ __forceinline__ void convert_lo_part(uint8_t* st, bool cA, bool cB, int ptid) {
  const uint4* ta = reinterpret_cast<const uint4*>(st);
  const uint4* tb = reinterpret_cast<const uint4*>(st + TILE_BYTES);
  uint4 va[NJ], vb[NJ];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int i = ptid + NPROD * (J0 + j);
    if (i < TILE_BYTES / 16) {
      if (cA) va[j] = ta[i];
      if (cB) vb[j] = tb[i];
    }
  }
  auto lo4 = [](const uint4 v) {
    const float x[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
    uint32_t r[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) r[e] = __float_as_uint(x[e] - __uint_as_float(tf32_trunc_bits(x[e])));
    return make_uint4(r[0], r[1], r[2], r[3]);
  };
  uint4* la = reinterpret_cast<uint4*>(st + 2 * TILE_BYTES);
  uint4* lb = reinterpret_cast<uint4*>(st + 3 * TILE_BYTES);
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    const int i = ptid + NPROD * (J0 + j);
    if (i < TILE_BYTES / 16) {
      if (cA) la[i] = lo4(va[j]);
      if (cB) lb[i] = lo4(vb[j]);
    }
  }
}
__device__ __forceinline__ void convert_lo_pair(uint8_t* st, bool cA, bool cB, int ptid) {
  constexpr int PER = (TILE_BYTES / 16 + NPROD - 1) / NPROD;  // chunks per thread per tile (6)
  static_assert(PER == 6, "two batches of three");
  convert_lo_part<0, 3>(st, cA, cB, ptid);
  convert_lo_part<3, 3>(st, cA, cB, ptid);
}

// 3xF16, TMA-only launches: both operands' fp32 tiles -> hi / lo fp16 tiles, items
// (16-byte output chunks; MN plain: row pairs) in two batches of three per thread,
// every load of a batch issued before its conversions.
template <int Q0>
__device__ __forceinline__ void convert_f16x3_batch(uint8_t* st, bool cA, bool mnA, float scA, bool cB, bool mnB,
                                                    float scB, int ptid) {
  constexpr int NB = 3;
  float x[NB][8], y[NB][8];
#pragma unroll
  for (int qq = 0; qq < NB; ++qq) {
    const int u = ptid + NPROD * (Q0 + qq);
    const int op = u >> 9, v = u & 511;
    const bool mn = op == 0 ? mnA : mnB;
    if (u >= 1024 || !(op == 0 ? cA : cB) || (mn && v >= 256)) continue;
    const uint8_t* src = st + op * TILE_BYTES;
    if (mn) {
      const int p = v & 63, c = v >> 6;
      const float2* f = reinterpret_cast<const float2*>(src) + p + (8 * c) * 64;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float2 t = f[e * 64];
        x[qq][e] = t.x;
        y[qq][e] = t.y;
      }
    } else {
      const int r = v & 127, c = v >> 7;
      const float4 a = *reinterpret_cast<const float4*>(src + sw128_offset(r, 2 * c));
      const float4 b = *reinterpret_cast<const float4*>(src + sw128_offset(r, 2 * c + 1));
      x[qq][0] = a.x; x[qq][1] = a.y; x[qq][2] = a.z; x[qq][3] = a.w;
      x[qq][4] = b.x; x[qq][5] = b.y; x[qq][6] = b.z; x[qq][7] = b.w;
    }
  }
#pragma unroll
  for (int qq = 0; qq < NB; ++qq) {
    const int u = ptid + NPROD * (Q0 + qq);
    const int op = u >> 9, v = u & 511;
    const bool mn = op == 0 ? mnA : mnB;
    if (u >= 1024 || !(op == 0 ? cA : cB) || (mn && v >= 256)) continue;
    const float sc = op == 0 ? scA : scB;
    uint8_t* dst = st + (2 + op) * TILE_BYTES;
    const int r = mn ? 2 * (v & 63) : (v & 127), c = mn ? (v >> 6) : (v >> 7);
    uint4 h, l;
    split8_f16(x[qq], sc, h, l);
    uint32_t off = sw64_chunk_offset(r, c);
    *reinterpret_cast<uint4*>(dst + off) = h;
    *reinterpret_cast<uint4*>(dst + F16_TILE + off) = l;
    if (mn) {
      split8_f16(y[qq], sc, h, l);
      off = sw64_chunk_offset(r + 1, c);
      *reinterpret_cast<uint4*>(dst + off) = h;
      *reinterpret_cast<uint4*>(dst + F16_TILE + off) = l;
    }
  }
}

// Bytes one TMA'd operand tile delivers.  Box loads always count their full
// (zero-filled) size; im2col tiles skip 32-row groups past the operand's rows
// (those smem rows only feed accumulator rows the epilogue never stores).
__device__ __forceinline__ uint32_t tma_tile_bytes(int kind, const dpk_operand& o, int row0) {
  if (kind == TMA_IM2COL16) {
    const int groups = min(BM / 64, (o.rows - row0 + 63) / 64);
    return static_cast<uint32_t>(max(groups, 0)) * 8192u;
  }
  if (kind != TMA_IM2COL && kind != TMA_TAPS) return TILE_BYTES;
  const int groups = min(BM / 32, (o.rows - row0 + 31) / 32);
  return static_cast<uint32_t>(max(groups, 0)) * 4096u;
}

// PAIR: signal `bar` (possibly the peer CTA's, a shared::cluster address)
template <bool PAIR = false>
__device__ __forceinline__ void issue_tma(int kind, const CUtensorMap* map, const dpk_operand& o, uint32_t dst,
                                          uint32_t bar, int row0, int kc, int cpn) {
  auto ld2 = [&](uint32_t d, int c0, int c1) {
    if (PAIR)
      tma_load_2d_pair(d, map, bar, c0, c1);
    else
      tma_load_2d(d, map, bar, c0, c1);
  };
  if (kind == TMA_ROWS_K) {
    ld2(dst, kc * BK, row0);
  } else if (kind == TMA_ROWS_K16) {
    ld2(dst, kc * 2 * BK, row0);
  } else if (kind == TMA_ROWS_MN_PLAIN) {  // one {128 rows, 32 k} box, k rows of 512 B
    ld2(dst, row0, kc * BK);
  } else if (kind == TMA_ROWS_MN) {
#pragma unroll
    for (int b = 0; b < BM / 32; ++b) ld2(dst + b * 4096, row0 + 32 * b, kc * BK);
  } else if (kind == TMA_ROWS_MN3) {  // dims {32, K, rows / 32}
    if (PAIR)
      tma_load_3d_pair(dst, map, bar, 0, kc * BK, row0 / 32);
    else
      tma_load_3d(dst, map, bar, 0, kc * BK, row0 / 32);
  } else if (kind == TMA_SLAB) {  // dims {HW, C, N}
    const int n = kc / cpn;
    if (PAIR)
      tma_load_3d_pair(dst, map, bar, (kc - n * cpn) * BK, row0, n);
    else
      tma_load_3d(dst, map, bar, (kc - n * cpn) * BK, row0, n);
  } else if (kind == TMA_TAPS) {
    // K chunk kc = (sample block, output-row block, output-column block); rows (i, j, c)
    const int wb = cpn & 0x3F, hb = (cpn >> 6) & 0x3F, g = (cpn >> 12) & 0xF, nbs = 32 / (wb * hb);
    const int owbs = o.OW / wb, ohbs = o.OH / hb;
    const int q = kc / owbs;
    const int owb = kc - q * owbs;
    const int nbk = q / ohbs;
    const int ohb = q - nbk * ohbs;
    const int w0 = owb * wb * o.sw - o.pw, h0 = ohb * hb * o.sh - o.ph, n0 = nbk * nbs;
    for (int b = 0; b < BM / 32; b += (g == 0 ? 1 : g)) {
      const int r = row0 + 32 * b;
      if (r >= o.rows) break;
      const int tap = r / o.C;
      const int c0 = r - tap * o.C;
      const int i = tap / o.kw, j = tap - (tap / o.kw) * o.kw;
      if (g == 0) {  // 4-D map {C, W, H, N}: one 32-channel box per row group
        if (PAIR)
          tma_load_4d_pair(dst + b * 4096, map, bar, c0, w0 + j * o.dw, h0 + i * o.dh, n0);
        else
          tma_load_4d(dst + b * 4096, map, bar, c0, w0 + j * o.dw, h0 + i * o.dh, n0);
        continue;
      }
      if (PAIR)
        tma_load_5d_pair(dst + b * 4096, map, bar, 0, w0 + j * o.dw, h0 + i * o.dh, n0, c0 >> 5);
      else
        tma_load_5d(dst + b * 4096, map, bar, 0, w0 + j * o.dw, h0 + i * o.dh, n0, c0 >> 5);
    }
  } else if (kind == TMA_IM2COL16) {  // fp16 NHWC input; a box = 64 output pixels x 64 channels
    const int64_t k0 = static_cast<int64_t>(kc) * 2 * BK;
    const int ohw = o.OH * o.OW;
    const int n = static_cast<int>(k0 / ohw);
    const int rem = static_cast<int>(k0 - static_cast<int64_t>(n) * ohw);
    const int oh = rem / o.OW;
    const int ow = rem - oh * o.OW;
    const int w0 = ow * o.sw - o.pw, h0 = oh * o.sh - o.ph;
    for (int b = 0; b < BM / 64; ++b) {
      const int r = row0 + 64 * b;
      if (r >= o.rows) break;
      const int tap = r / o.C;
      const int c0 = r - tap * o.C;
      const int i = tap / o.kw, j = tap - (tap / o.kw) * o.kw;
      if (PAIR)
        tma_load_im2col_4d_pair(dst + b * 8192, map, bar, c0, w0, h0, n, static_cast<uint16_t>(j * o.dw),
                                static_cast<uint16_t>(i * o.dh));
      else
        tma_load_im2col_4d(dst + b * 8192, map, bar, c0, w0, h0, n, static_cast<uint16_t>(j * o.dw),
                           static_cast<uint16_t>(i * o.dh));
    }
  } else {  // TMA_IM2COL: NHWC input, rows (i, j, c); a box = 32 output pixels x 32 channels
    const int64_t k0 = static_cast<int64_t>(kc) * BK;
    const int ohw = o.OH * o.OW;
    const int n = static_cast<int>(k0 / ohw);
    const int rem = static_cast<int>(k0 - static_cast<int64_t>(n) * ohw);
    const int oh = rem / o.OW;
    const int ow = rem - oh * o.OW;
    const int w0 = ow * o.sw - o.pw, h0 = oh * o.sh - o.ph;
    for (int b = 0; b < BM / 32; ++b) {
      const int r = row0 + 32 * b;
      if (r >= o.rows) break;
      const int tap = r / o.C;
      const int c0 = r - tap * o.C;
      const int i = tap / o.kw, j = tap - (tap / o.kw) * o.kw;
      if (PAIR)
        tma_load_im2col_4d_pair(dst + b * 4096, map, bar, c0, w0, h0, n, static_cast<uint16_t>(j * o.dw),
                                static_cast<uint16_t>(i * o.dh));
      else
        tma_load_im2col_4d(dst + b * 4096, map, bar, c0, w0, h0, n, static_cast<uint16_t>(j * o.dw),
                           static_cast<uint16_t>(i * o.dh));
    }
  }
}

// ------------------------------------------------------------------ epilogue
// Problem fields live in the kernel parameter bank and are indexed by the
// problem id, so every use is an indexed LDC; ptxas happily re-issues those in
// the row loop (a constant-cache round trip per row).  Pin them in registers.
__device__ __forceinline__ int pin(int v) {
  asm volatile("mov.b32 %0, %0;" : "+r"(v));
  return v;
}
__device__ __forceinline__ float pin(float v) {
  asm volatile("mov.b32 %0, %0;" : "+f"(v));
  return v;
}
template <class T>
__device__ __forceinline__ T* pin(T* v) {
  uint64_t x = reinterpret_cast<uint64_t>(v);
  asm volatile("mov.b64 %0, %0;" : "+l"(x));
  return reinterpret_cast<T*>(x);
}
__device__ __forceinline__ int64_t pin(int64_t v) {
  asm volatile("mov.b64 %0, %0;" : "+l"(v));
  return v;
}

// plain weak global store (st.global.f32): no cache-scope strength, so the LSU
// never has to order consecutive epilogue stores
__device__ __forceinline__ void st_out(float* p, float v) {
  asm volatile("st.global.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// predicated store: no branch / reconvergence point per element
__device__ __forceinline__ void st_out_if(bool pred, float* p, float v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.f32 [%0], %1;\n\t}\n" ::"l"(p), "f"(v),
      "r"(static_cast<int>(pred))
      : "memory");
}
__device__ __forceinline__ float ld_cg_if(bool pred, const float* p) {
  float v = 0.0f;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cg.f32 %0, [%1];\n\t}\n"
      : "+f"(v)
      : "l"(p), "r"(static_cast<int>(pred)));
  return v;
}

struct Epi {
  float* out;
  const float* cin;
  const float* vrow;
  const float* vcol;
  float* part;  // this unit's partial slot (split-K) or nullptr
  float* out_t;
  int64_t ldo, ldc, ldt;
  float alpha, beta, gamma;
  int M, N, symmetric, eigdiv;
};

// unit tiles are (128*CG) x (128*CG); each CTA of a pair owns 128 of its rows
template <int CG>
__device__ __forceinline__ Epi load_epi(const Problem& P, int tile, int split) {
  constexpr int64_t UNIT = static_cast<int64_t>(128 * CG) * (128 * CG);
  Epi e;
  e.out = pin(P.out);
  e.cin = pin(P.cin);
  e.vrow = pin(P.vrow);
  e.vcol = pin(P.vcol);
  e.part = P.splits > 1 ? pin(P.partials + static_cast<int64_t>(tile * P.splits + split) * UNIT) : nullptr;
  e.out_t = pin(P.out_t);
  e.ldo = pin(P.ldo);
  e.ldc = pin(P.ldc);
  e.ldt = pin(P.ldt);
  e.alpha = pin(P.alpha);
  if (P.alpha_amax) e.alpha = ldexpf(e.alpha, 2 * prescale_exponent(__ldg(P.alpha_amax)));
  if (P.amax_a)
    e.alpha = ldexpf(e.alpha, prescale_exponent(__ldg(P.amax_a)) + prescale_exponent(__ldg(P.amax_b)));
  e.beta = pin(P.beta);
  e.gamma = pin(P.gamma);
  e.M = pin(P.M);
  e.N = pin(P.N);
  e.symmetric = pin(P.symmetric);
  e.eigdiv = pin(P.epi == EPI_EIGDIV ? 1 : 0);
  return e;
}

// One warp's 32x32 accumulator block (rows warp*32.., columns c*32..) goes
// through a padded smem transpose buffer so that every global access is a
// 128 B coalesced row segment: the direct pass walks rows with lane = column,
// the mirror / out_t pass walks columns with lane = row.  Every phase first
// pulls all 32 of its smem (and cin) values into registers, then issues the
// 32 stores back to back -- no load waits behind a store.
__device__ __forceinline__ void dbg_raw(bool on, int slot) {
  if (on) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dbg_ts[slot] = t;
  }
}

// gm0: global row of this warp's first row; gnc: global column of the chunk's
// first column; part: the chunk's split-K partial (row 0, column 0) with row
// stride pstride; diag: symmetric diagonal unit (store gn <= gm, mirror gn < gm).
__device__ __forceinline__ void store_chunk(const Epi& e, bool diag, int gm0, int gnc, float* part, int pstride,
                                            int lane, const uint32_t (&r)[32], float* T, bool dbg = false) {
#pragma unroll
  for (int j = 0; j < 32; ++j) T[lane * 33 + j] = __uint_as_float(r[j]);
  __syncwarp();
  dbg_raw(dbg, 13);
  float v[32];
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) v[rr] = T[rr * 33 + lane];
  dbg_raw(dbg, 14);
  if (part) {
    float* pp = part + lane;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) st_out(pp + rr * pstride, v[rr]);
    __syncwarp();
    return;
  }
  const int gn = gnc + lane;
  const int nrows = min(32, e.M - gm0);
  // row rr is written by this lane iff rr < nrows, gn < N and (not diag or gn <= gm)
  const int rlo = diag ? max(0, gn - gm0) : 0;
  const bool col_ok = gn < e.N;
  if (e.eigdiv) {
    const float vc = col_ok ? fmaxf(__ldg(e.vcol + gn), 0.0f) : 0.0f;
    // lane rr holds row rr's eigenvalue (one coalesced load), broadcast by shuffle
    const float vr_lane = lane < nrows ? fmaxf(__ldg(e.vrow + gm0 + lane), 0.0f) : 0.0f;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) v[rr] = e.alpha * v[rr] / (__shfl_sync(0xffffffffu, vr_lane, rr) * vc + e.gamma);
  } else if (e.beta != 0.0f) {
    const float* cp = e.cin + static_cast<int64_t>(gm0) * e.ldc + gn;
    float cv[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) {
      cv[rr] = ld_cg_if(col_ok && rr >= rlo && rr < nrows, cp);
      cp += e.ldc;
    }
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) v[rr] = fmaf(e.beta, cv[rr], e.alpha * v[rr]);
  } else {
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) v[rr] *= e.alpha;
  }
  float* op = e.out + static_cast<int64_t>(gm0) * e.ldo + gn;
  dbg_raw(dbg, 15);
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) {
    st_out_if(col_ok && rr >= rlo && rr < nrows, op, v[rr]);
    op += e.ldo;
  }
  dbg_raw(dbg, 12);
  if (e.symmetric == 1 || e.out_t) {
    __syncwarp();  // every lane has read its column of T
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) T[rr * 33 + lane] = v[rr];
    __syncwarp();
    float w[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) w[j] = T[lane * 33 + j];
    const int gm = gm0 + lane;
    const int gn0 = gnc;
    // columns written in the direct pass for this row: g < N and (not diag or g <= gm)
    const int jend = lane < nrows ? min(32, min(e.N, diag ? gm + 1 : e.N) - gn0) : 0;
    if (e.symmetric == 1) {
      float* mp = e.out + static_cast<int64_t>(gn0) * e.ldo + gm;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        st_out_if(j < jend && gn0 + j != gm, mp, w[j]);
        mp += e.ldo;
      }
    }
    if (e.out_t) {
      float* tp = e.out_t + static_cast<int64_t>(gn0) * e.ldt + gm;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        st_out_if(j < jend, tp, w[j]);
        tp += e.ldt;
      }
    }
  }
  __syncwarp();
}

// CG = 1: one CTA per 128x128 unit tile, cta_group::1 MMAs (M=128, N=128).
// CG = 2: a CTA pair (cluster of 2) per 256x256 unit tile, cta_group::2 MMAs
// (M=256, N=256) issued by the leader: CTA r stages rows [128r, 128r+128) of
// the tile's A rows and of its B rows (the pair's two B halves form N=256), so
// each SM moves half the operand bytes per flop of the CG=1 tile and reads half
// the shared memory per MMA -- the 1-SM tf32 MMA is otherwise shared-memory
// bound (MMA operand reads + TMA writes > 128 B/clk).  Each CTA's TMEM holds its
// 128 rows x 256 columns.  Producers of both CTAs arrive on the leader's full
// barrier, both epilogues arrive on the leader's TMEM-empty barrier, and the
// leader's commits multicast to both CTAs' stage-empty / TMEM-full barriers.
// GATHER=false: every operand of the launch is TMA-planned -- the producers' gather
// path is compiled out (3xTF32 single-CTA launches then keep their conversion loop
// free of the gather arrays' registers)
template <int NPASS, bool RN, int CG, bool GATHER = true>
__global__ void __launch_bounds__(NTHREADS, 1) tc_gemm_kernel(const __grid_constant__ Batch bt) {
  using C = Cfg<NPASS>;
  constexpr int UT = 128 * CG;                  // unit tile edge (rows and columns)
  constexpr uint32_t ACC_COLS = UT;             // TMEM columns per accumulator
  constexpr uint32_t TMEM_N = 2 * ACC_COLS;     // two accumulators
  // TMA'd tiles need a pass before the MMA only for the 3xTF32 low parts: in RN
  // mode the tensor map's TFLOAT32 data type rounds during the copy itself.
  constexpr bool CONVERT = (NPASS == 3);
  // NPASS == 3 with RN set: 3xF16 (fp16 hi / lo parts of the scaled operands, kind::f16)
  constexpr bool F16X3 = (NPASS == 3 && RN);
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bars = base + C::STAGES * C::STAGE_BYTES;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (C::STAGES + s); };
  auto tma_bar = [&](int s) { return bars + 8u * (2 * C::STAGES + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (3 * C::STAGES + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (3 * C::STAGES + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (3 * C::STAGES + 4);
  // unit ring: the scheduler (CG=1 / leader TMA thread) publishes unit ids, every
  // looping role reads them in order; -1 ends the launch
  const uint32_t rbase = tmem_slot + 16u;
  auto rfull_bar = [&](int q) { return rbase + 8u * q; };
  auto rempty_bar = [&](int q) { return rbase + 8u * (C::NSLOT + q); };
  const uint32_t ring_ids = rbase + 16u * C::NSLOT;
  volatile int* ring = reinterpret_cast<volatile int*>(gbase + (ring_ids - base));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = (CG == 2) ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int half = static_cast<int>(rank) * 128;  // this CTA's row offset inside a unit tile
  const int unit0 = (CG == 2) ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
  const int ustep = (CG == 2) ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
  const bool prods_ = bt.producers != 0;
  // ring consumers per CTA: MMA thread (CG=1 / leader) or the peer's TMA thread,
  // 4 epilogue warps, the producer warps when they run
  const int consumers = 1 + EPI_WARPS + (prods_ ? PROD_WARPS : 0);
  if (threadIdx.x == 0) dbg_ts(bt, 0);

  // full-barrier arrivals per stage use: every producer warp of the CTA (CG=2:
  // of both CTAs) or, in producer-free launches, the TMA thread alone (CG=2: the
  // leader's, whose expect_tx covers both CTAs' loads)
  const bool prods = bt.producers != 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(full_bar(s), prods ? CG * PROD_WARPS : 1);
      mbar_init(empty_bar(s), 1);
      mbar_init(tma_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull_bar(a), 1);
      mbar_init(tempty_bar(a), EPI_WARPS * 32 * CG);
    }
    for (int q = 0; q < C::NSLOT; ++q) {
      mbar_init(rfull_bar(q), 1);
      mbar_init(rempty_bar(q), consumers * CG);  // CG=2: both CTAs' consumers, on the leader
    }
    mbar_fence_init();
  }
  if (warp == MMA_WARP) {
    if (CG == 2)
      tmem_alloc2(tmem_slot, TMEM_N);
    else
      tmem_alloc(tmem_slot, TMEM_N);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // peer barriers initialised before any remote arrive / multicast
  tc_fence_after();
  // everything above overlaps the previous kernel's tail (PDL); from here on we
  // read operands / cin and write outputs
  pdl_wait();
  pdl_trigger();
  const uint32_t tmem_base = *reinterpret_cast<volatile uint32_t*>(gbase + (tmem_slot - base));
  if (threadIdx.x == 0) dbg_ts(bt, 1);
  // scheduler side (CG=1, or the leader's TMA thread): next unit id, -1 when done
  auto sched_next = [&](int it) -> int {
    int u = bt.dynamic ? atomicAdd(bt.sched, 1) : unit0 + it * ustep;
    return u < bt.total_units ? u : -1;
  };
  auto ring_publish = [&](int it, int u) {
    const int q = it % C::NSLOT;
    const uint32_t par = static_cast<uint32_t>((it / C::NSLOT) & 1);
    if (CG == 2)
      mbar_wait_cluster(rempty_bar(q), par ^ 1);
    else
      mbar_wait(rempty_bar(q), par ^ 1);
    ring[q] = u;
    if (CG == 2) {
      st_shared_cluster_s32(mapa_shared(ring_ids + 4u * q, 1), u);
      mbar_arrive(rfull_bar(q));
      mbar_arrive_remote(mapa_shared(rfull_bar(q), 1));
    } else {
      mbar_arrive(rfull_bar(q));
    }
  };
  // consumer side: every thread of the calling warp reads; `arrive` = this
  // thread releases the slot for its role (one per warp / role)
  auto ring_take = [&](int it, bool arrive) -> int {
    const int q = it % C::NSLOT;
    const uint32_t par = static_cast<uint32_t>((it / C::NSLOT) & 1);
    if (CG == 2 && !leader)
      mbar_wait_cluster(rfull_bar(q), par);
    else
      mbar_wait(rfull_bar(q), par);
    const int u = ring[q];
    if (arrive) {
      if (CG == 2 && !leader)
        mbar_arrive_remote(mapa_shared(rempty_bar(q), 0));
      else
        mbar_arrive(rempty_bar(q));
    }
    return u;
  };

  if (warp == TMA_WARP) {
    // =============================== TMA issuer: runs ahead through the stage ring
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // the next unit id is drawn one unit ahead, so the atomic's round trip
      // overlaps this unit's load issue
      int u_next = (CG == 1 || leader) ? sched_next(0) : 0;
      for (int it = 0;; ++it) {
        int u;
        if (CG == 1 || leader) {
          u = u_next;
          ring_publish(it, u);
          if (u >= 0) u_next = sched_next(it + 1);
        } else {
          u = ring_take(it, true);
        }
        if (u < 0) break;
        int pi, tm, tn, tile, split;
        decode_unit(bt, u, pi, tm, tn, tile, split);
        const Problem& P = bt.p[pi];
        const bool skip_b = P.same_ab && tm == tn;
        const bool tA = P.tma_a != TMA_NONE;
        const bool tB = !skip_b && P.tma_b != TMA_NONE;
        if (tA) tma_prefetch_desc(&P.tmap_a);
        if (tB) tma_prefetch_desc(&P.tmap_b);
        int kc0, kc1;
        chunk_range<CG>(P, tm, tn, split, kc0, kc1);
        const int ra = tm * UT + half, rb = tn * UT + half;
        auto tile_bytes = [&](int a_row, int b_row) -> uint32_t {
          return (tA ? tma_tile_bytes(P.tma_a, P.a, a_row) : 0u) + (tB ? tma_tile_bytes(P.tma_b, P.b, b_row) : 0u);
        };
        const uint32_t bytes = tile_bytes(ra, rb);
        // CG=2 without an smem conversion: both CTAs' loads complete directly on
        // the leader's full barrier (cta_group::2 TMA), no producer hand-off
        // CG=2 without producers: both CTAs' loads complete on the leader's full barrier
        const bool direct = CG == 2 && !prods;
        const uint32_t pair_bytes = direct ? bytes + tile_bytes(tm * UT + (128 - half), tn * UT + (128 - half)) : 0u;
        for (int kc = kc0; kc < kc1; ++kc) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          const uint32_t sst = base + stage * C::STAGE_BYTES;
          if (direct) {
            const uint32_t fb = leader ? full_bar(stage) : mapa_shared(full_bar(stage), 0);
            if (leader) mbar_arrive_expect_tx(full_bar(stage), pair_bytes);
            if (tA) issue_tma<true>(P.tma_a, &P.tmap_a, P.a, sst, fb, ra, kc, P.slab_cpn);
            if (tB) issue_tma<true>(P.tma_b, &P.tmap_b, P.b, sst + TILE_BYTES, fb, rb, kc, P.slab_cpn);
          } else {
            // exactly one arrival per stage use; tx bytes only for TMA'd tiles
            mbar_arrive_expect_tx(tma_bar(stage), bytes);
            if (!prods) mbar_arrive(full_bar(stage));  // CG=1 producer-free: stands in for the producers
            if (tA) issue_tma(P.tma_a, &P.tmap_a, P.a, sst, tma_bar(stage), ra, kc, P.slab_cpn);
            if (tB) issue_tma(P.tma_b, &P.tmap_b, P.b, sst + TILE_BYTES, tma_bar(stage), rb, kc, P.slab_cpn);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      dbg_ts(bt, 2);
    }
  } else if (warp >= PROD_WARP0 && prods) {
    // =============================== gather / convert warps
    const int ptid = threadIdx.x - PROD_WARP0 * 32;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0;; ++it) {
      const int u = ring_take(it, lane == 0);
      __syncwarp();
      if (u < 0) break;
      int pi, tm, tn, tile, split;
      decode_unit(bt, u, pi, tm, tn, tile, split);
      const Problem& P = bt.p[pi];
      const bool skip_b = P.same_ab && tm == tn;
      const bool tA = P.tma_a != TMA_NONE;
      const bool tB = !skip_b && P.tma_b != TMA_NONE;
      const bool mA = GATHER && CG == 1 && !tA;  // CG=2 problems are planned TMA-only
      const bool mB = GATHER && CG == 1 && !skip_b && !tB;
      const bool cA = tA;  // 3-pass: TMA'd tiles get their low part computed here
      const bool cB = tB;
      // 3xF16: the operands' exact power-of-two scales
      const float sc_a = F16X3 ? ldexpf(1.0f, -prescale_exponent(__ldg(P.amax_a))) : 1.0f;
      const float sc_b = F16X3 ? ldexpf(1.0f, -prescale_exponent(__ldg(P.amax_b))) : 1.0f;
      int kc0, kc1;
      chunk_range<CG>(P, tm, tn, split, kc0, kc1);
      if (!GATHER) {
        // every operand of the launch arrives by TMA: the loop only derives the 3xTF32
        // low parts (or the 3xF16 hi / lo tiles), a stage's loads in flight at once
        const bool mnA = P.tma_a == TMA_ROWS_MN_PLAIN, mnB = P.tma_b == TMA_ROWS_MN_PLAIN;
        for (int kc = kc0; kc < kc1; ++kc) {
          mbar_wait(empty_bar(stage), phase ^ 1);
          uint8_t* st = gbase + stage * C::STAGE_BYTES;
          if (CONVERT && (cA || cB)) {
            mbar_wait(tma_bar(stage), phase);
            if (F16X3) {
              convert_f16x3_batch<0>(st, cA, mnA, sc_a, cB, mnB, sc_b, ptid);
              convert_f16x3_batch<3>(st, cA, mnA, sc_a, cB, mnB, sc_b, ptid);
            } else {
              convert_lo_pair(st, cA, cB, ptid);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2 && !leader)
              mbar_arrive_remote(mapa_shared(full_bar(stage), 0));
            else
              mbar_arrive(full_bar(stage));
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        continue;
      }
      RowTask ta[NTASK], tb[NTASK];
      if (mA) setup_tasks(P.a, tm * UT, ptid, ta);
      if (mB) setup_tasks(P.b, tn * UT, ptid, tb);
      // manual operands: chunk kc+1's gathers are in flight while chunk kc is stored
      float4 va[NTASK], vb[NTASK], na[NTASK], nb[NTASK];
      if (mA) fetch_tasks(P.a, ta, ptid, static_cast<int64_t>(kc0) * BK, va);
      if (mB) fetch_tasks(P.b, tb, ptid, static_cast<int64_t>(kc0) * BK, vb);
      for (int kc = kc0; kc < kc1; ++kc) {
        if (kc + 1 < kc1) {
          const int64_t knext = static_cast<int64_t>(kc + 1) * BK;
          if (mA) fetch_tasks(P.a, ta, ptid, knext, na);
          if (mB) fetch_tasks(P.b, tb, ptid, knext, nb);
        }
        const bool pdbg = bt.debug_ts && blockIdx.x == 0 && ptid == 0;
        long long q0 = pdbg ? clock64() : 0;
        mbar_wait(empty_bar(stage), phase ^ 1);
        long long q1 = pdbg ? clock64() : 0, q2 = q1;
        uint8_t* st = gbase + stage * C::STAGE_BYTES;
        if (F16X3) {  // hi / lo fp16 tiles of A in slot 2, of B in slot 3
          if (mA) store_tasks_f16x3(P.a, ptid, st + 2 * TILE_BYTES, sc_a, va);
          if (mB) store_tasks_f16x3(P.b, ptid, st + 3 * TILE_BYTES, sc_b, vb);
        } else {
          if (mA) store_tasks<NPASS, RN>(P.a, ptid, st, st + 2 * TILE_BYTES, va);
          if (mB) store_tasks<NPASS, RN>(P.b, ptid, st + TILE_BYTES, st + 3 * TILE_BYTES, vb);
        }
        // CG=2 with a conversion: the leader's MMA cannot see this CTA's TMA
        // barrier, so the producers forward its completion with their arrival
        // (without one, the loads signal the leader's full barrier directly)
        if (CONVERT && (cA || cB)) {
          mbar_wait(tma_bar(stage), phase);
          q2 = pdbg ? clock64() : 0;
          if (F16X3) {
            if (cA) convert_tile_f16x3(st, P.tma_a == TMA_ROWS_MN_PLAIN, st + 2 * TILE_BYTES, sc_a, ptid);
            if (cB) convert_tile_f16x3(st + TILE_BYTES, P.tma_b == TMA_ROWS_MN_PLAIN, st + 3 * TILE_BYTES, sc_b, ptid);
          } else {
            if (cA) convert_tile<NPASS>(st, st + 2 * TILE_BYTES, ptid);
            if (cB) convert_tile<NPASS>(st + TILE_BYTES, st + 3 * TILE_BYTES, ptid);
          }
        }
        if (pdbg) {  // debug timeline: producer cycles waiting for a free stage / for the TMA data / converting
          const long long q3 = clock64();
          atomicAdd(&g_dbg_unit[DBG_UNITS - 1][0], static_cast<unsigned long long>(q1 - q0));
          atomicAdd(&g_dbg_unit[DBG_UNITS - 1][1], static_cast<unsigned long long>(q2 - q1));
          atomicAdd(&g_dbg_unit[DBG_UNITS - 1][2], static_cast<unsigned long long>(q3 - q2));
          atomicAdd(&g_dbg_unit[DBG_UNITS - 1][3], 1ull);
        }
        // one arrival per producer warp (measured faster than a named barrier +
        // a single elected arrival: the warps' cluster-scope releases overlap)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2 && !leader)
            mbar_arrive_remote(mapa_shared(full_bar(stage), 0));
          else
            mbar_arrive(full_bar(stage));
        }
        if (++stage == C::STAGES) {
          stage = 0;
          phase ^= 1;
        }
#pragma unroll
        for (int j = 0; j < NTASK; ++j) {
          va[j] = na[j];
          vb[j] = nb[j];
        }
      }
    }
    if (ptid == 0) dbg_ts(bt, 3);
  } else if (warp == MMA_WARP) {
    // =============================== MMA issuer (CG=2: the leader CTA only)
    // The whole warp runs the loop (every value warp-uniform, so descriptors live in
    // uniform registers); each tcgen05.mma / commit is issued by one elected lane.
    if (leader) {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0;; ++it) {
        const int u = ring_take(it, lane == 0);
        if (u < 0) break;
        int pi, tm, tn, tile, split;
        decode_unit(bt, u, pi, tm, tn, tile, split);
        const Problem& P = bt.p[pi];
        const bool skip_b = P.same_ab && tm == tn;
        const int a_mn = tma_mn(P.tma_a);
        const int b_mn = skip_b ? a_mn : tma_mn(P.tma_b);
        const bool f16 = tma_f16(P.tma_a);  // SYRK on fp16 operands (both sides)
        const uint32_t idesc = F16X3 ? idesc_f16(UT, UT)  // K-major fp16 hi / lo tiles
                               : f16 ? idesc_f16(UT, UT, a_mn, b_mn) : idesc_tf32(UT, UT, a_mn, b_mn);
        const int acc = it & 1;
        if (CG == 2)
          mbar_wait_cluster(tempty_bar(acc), ((it >> 1) & 1) ^ 1);
        else
          mbar_wait(tempty_bar(acc), ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        dbg_unit(bt, it, 0);
        const uint32_t d = tmem_base + acc * ACC_COLS;
        int kc0, kc1;
        chunk_range<CG>(P, tm, tn, split, kc0, kc1);
        // stage-0 descriptors of the A / B tiles and the per-UMMA_K step (16-byte units):
        // K-major +32 B along the 128 B row; MN-major the next 8-row k group (+1024 B),
        // two groups for a 16-deep f16 step (+2048 B, 64-wide M/N blocks 8 KB apart)
        const uint32_t sa0 = base, sb0 = skip_b ? base : base + TILE_BYTES;
        const uint64_t da0 = a_mn ? (f16 ? sdesc_mnmajor_sw128_16b(sa0, 8192) : sdesc_mnmajor_sw128(sa0, 4096))
                                  : sdesc_kmajor_sw128(sa0);
        const uint64_t db0 = b_mn ? (f16 ? sdesc_mnmajor_sw128_16b(sb0, 8192) : sdesc_mnmajor_sw128(sb0, 4096))
                                  : sdesc_kmajor_sw128(sb0);
        const uint32_t astep = a_mn ? (f16 ? 128u : 64u) : 2u;
        const uint32_t bstep = b_mn ? (f16 ? 128u : 64u) : 2u;
        for (int kc = kc0; kc < kc1; ++kc) {
          if (CG == 2) {
            // producers of both CTAs (TMA forwarded) arrive with release.cluster: acquire at
            // cluster scope (emits an L1 invalidate per chunk).  Producer-free launches only
            // see TMA complete_tx (async proxy, like the MMA) and the leader's own
            // expect_tx: the CTA-scope wait suffices and keeps the MMA issue loop short.
            if (prods)
              mbar_wait_cluster(full_bar(stage), phase);
            else
              mbar_wait(full_bar(stage), phase);
          } else {
            mbar_wait(full_bar(stage), phase);
            mbar_wait(tma_bar(stage), phase);
          }
          if (kc == kc0) dbg_unit(bt, it, 1);
          tc_fence_after();
          // descriptors: the unit's stage-0 descriptors plus the address-field offset
          // (16-byte units; the field never carries: every operand lies below 256 KB)
          const uint64_t so = static_cast<uint64_t>(stage) * (C::STAGE_BYTES >> 4);
          const uint64_t da = da0 + so, db = db0 + so;
          const uint32_t accum0 = kc > kc0 ? 1u : 0u;
          if (F16X3) {  // hi*hi + hi*lo + lo*hi on the SW64 fp16 tiles: 2 x (K = 16) per chunk
            const uint32_t s0 = base + stage * C::STAGE_BYTES;
            const uint64_t ah = sdesc_kmajor_sw64(s0 + 2 * TILE_BYTES), al = ah + (F16_TILE >> 4);
            const uint64_t bh = skip_b ? ah : sdesc_kmajor_sw64(s0 + 3 * TILE_BYTES), bl = bh + (F16_TILE >> 4);
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const uint32_t o = 2u * s;  // +32 B along the 64 B row
              if (CG == 2) {
                mma_f16_pair(d, ah + o, bh + o, idesc, s > 0 ? 1u : accum0);
                mma_f16_pair(d, ah + o, bl + o, idesc, 1u);
                mma_f16_pair(d, al + o, bh + o, idesc, 1u);
              } else {
                mma_f16(d, ah + o, bh + o, idesc, s > 0 ? 1u : accum0);
                mma_f16(d, ah + o, bl + o, idesc, 1u);
                mma_f16(d, al + o, bh + o, idesc, 1u);
              }
            }
          } else if (NPASS == 1 && f16) {  // UMMA_K = 16 fp16 = the same 32 B step
#pragma unroll
            for (int s = 0; s < BK / 8; ++s) {
              if (CG == 2)
                mma_f16_pair(d, da + s * astep, db + s * bstep, idesc, s > 0 ? 1u : accum0);
              else
                mma_f16(d, da + s * astep, db + s * bstep, idesc, s > 0 ? 1u : accum0);
            }
          } else {
#pragma unroll
            for (int s = 0; s < BK / 8; ++s) {  // UMMA_K = 8 for tf32
              const uint64_t das = da + s * astep, dbs = db + s * bstep;
              if (CG == 2)
                mma_tf32_pair(d, das, dbs, idesc, s > 0 ? 1u : accum0);
              else
                mma_tf32(d, das, dbs, idesc, s > 0 ? 1u : accum0);
              if (NPASS == 3) {  // + hi*lo + lo*hi (the low parts sit 2 / 3 tiles further)
                const uint64_t dal = das + 2 * (TILE_BYTES >> 4);
                const uint64_t dbl = skip_b ? dal : dbs + 2 * (TILE_BYTES >> 4);
                if (CG == 2) {
                  mma_tf32_pair(d, das, dbl, idesc, 1u);
                  mma_tf32_pair(d, dal, dbs, idesc, 1u);
                } else {
                  mma_tf32(d, das, dbl, idesc, 1u);
                  mma_tf32(d, dal, dbs, idesc, 1u);
                }
              }
            }
          }
          if (CG == 2)
            mma_commit_pair(empty_bar(stage), 0x3);
          else
            mma_commit(empty_bar(stage));
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        dbg_unit(bt, it, 2);
        if (CG == 2)
          mma_commit_pair(tfull_bar(acc), 0x3);
        else
          mma_commit(tfull_bar(acc));
      }
      if (lane == 0) dbg_ts(bt, 4);
    }
  } else if (warp < EPI_WARPS) {
    // =============================== epilogue (warps 0-3, thread = tile row)
    const int m = warp * 32 + lane;
    float* T = reinterpret_cast<float*>(gbase + (bars - base) + C::BAR_BYTES) + warp * 32 * 33;
    for (int it = 0;; ++it) {
      const int u = ring_take(it, lane == 0);
      __syncwarp();
      if (u < 0) break;
      int pi, tm, tn, tile, split;
      decode_unit(bt, u, pi, tm, tn, tile, split);
      const Problem& P = bt.p[pi];
      const int acc = it & 1;
      mbar_wait(tfull_bar(acc), (it >> 1) & 1);
      if (threadIdx.x == 0) dbg_unit(bt, it, 3);
      if (it == 0 && threadIdx.x == 0) dbg_ts(bt, 9);
      tc_fence_after();
      const uint32_t taddr = tmem_base + acc * ACC_COLS + (static_cast<uint32_t>(warp * 32) << 16);
      const Epi e = load_epi<CG>(P, tile, split);
      int kc0, kc1;
      chunk_range<CG>(P, tm, tn, split, kc0, kc1);
      const bool empty = kc1 <= kc0;  // nothing accumulated: the tile's product is zero
      const bool diag = e.symmetric == 1 && tm == tn;
      const int gm0 = tm * UT + half + warp * 32;
#pragma unroll 1
      for (int c = 0; c < static_cast<int>(ACC_COLS) / 32; ++c) {
        uint32_t r[32];
        if (empty) {
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = 0u;
        } else {
          tmem_ld32(taddr + c * 32, r);
          tmem_ld_wait();
        }
        if (it == 0 && c == 0 && threadIdx.x == 0) dbg_ts(bt, 10);
        float* part = e.part ? e.part + static_cast<int64_t>(half + warp * 32) * UT + c * 32 : nullptr;
        store_chunk(e, diag, gm0, tn * UT + c * 32, part, UT, lane, r, T,
                    bt.debug_ts && blockIdx.x == 0 && it == 0 && c == 0 && threadIdx.x == 0);
        if (it == 0 && c == 0 && threadIdx.x == 0) dbg_ts(bt, 11);
      }
      tc_fence_before();
      if (threadIdx.x == 0) dbg_unit(bt, it, 4);
      if (CG == 2 && !leader)
        mbar_arrive_remote(mapa_shared(tempty_bar(acc), 0));
      else
        mbar_arrive(tempty_bar(acc));
      // split-K partials are summed (in split order, deterministic) and finished
      // by splitk_reduce_kernel, spread over the whole GPU
      if (m == 0) dbg_ts(bt, 5 + (it > 0));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // no CTA leaves while its pair may still signal it
  if (threadIdx.x == 0) dbg_ts(bt, 7);
  // dynamic schedule: the last worker to finish resets the counters for the next
  // launch on this stream (every worker has drawn its final, out-of-range id)
  if (bt.dynamic && threadIdx.x == 0 && (CG == 1 || leader)) {
    __threadfence();
    if (atomicAdd(bt.sched + 1, 1) == static_cast<int>(gridDim.x) / CG - 1) {
      bt.sched[0] = 0;
      bt.sched[1] = 0;
      __threadfence();
    }
  }
  if (warp == MMA_WARP) {
    __syncwarp();
    tc_fence_after();
    if (CG == 2)
      tmem_dealloc2(tmem_base, TMEM_N);
    else
      tmem_dealloc(tmem_base, TMEM_N);
    if (lane == 0) dbg_ts(bt, 8);
  }
}

// ------------------------------------------------------------------ 3xF16 operand scales
// amax|op| of every operand view of a 3xF16 call (the float bits, int-compared:
// order-preserving for non-negative floats; NaN sorts above inf and propagates).
// Elements a triangular operand never contributes (TRI_LOWER / TRI_UPPER) are
// skipped -- they may hold anything -- and a bias row counts as 1.
constexpr int AMAX_MAXV = 256;
struct AmaxView {
  const float* data;
  int64_t ld, cols;
  int rows, mn, tri, bias;
  int32_t* out;
};
struct AmaxBatch {
  int n;
  AmaxView v[AMAX_MAXV];
};
__global__ void __launch_bounds__(256) operand_amax_kernel(const __grid_constant__ AmaxBatch b) {
  const AmaxView& V = b.v[blockIdx.y];
  const int64_t R = V.mn ? V.cols : V.rows, C = V.mn ? V.rows : V.cols;  // memory rows / columns
  int m = (V.bias && blockIdx.x == 0 && threadIdx.x == 0) ? __float_as_int(1.0f) : 0;
  for (int64_t i = blockIdx.x; i < R; i += gridDim.x) {
    const float* row = V.data + i * V.ld;
    for (int64_t j = threadIdx.x; j < C; j += blockDim.x) {
      const int64_t r = V.mn ? j : i, k = V.mn ? i : j;  // operand (row, k)
      if ((V.tri == TRI_LOWER && k > r) || (V.tri == TRI_UPPER && k < r)) continue;
      m = max(m, __float_as_int(__ldg(row + j)) & 0x7fffffff);
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0) atomicMax(V.out, m);
}

// ------------------------------------------------------------------ split-K reduction
// One CTA per (split tile, 8-row slab): 256 threads, each owns 4 consecutive
// columns of one row, sums the partials in split order (deterministic) and
// applies the same epilogue as the single-split path.
constexpr int RED_MAX = 96;
struct RedJob {
  float* out;
  const float* cin;
  const float* vrow;
  const float* vcol;
  const float* partials;
  float* out_t;
  int64_t ldo, ldc, ldt;
  const int32_t* alpha_amax;
  const int32_t* amax_a;
  const int32_t* amax_b;
  float alpha, beta, gamma;
  int M, N, symmetric, epi, tiles_n, splits;
  int ut;          // unit tile edge (128 or 256)
  int slab_begin;  // prefix over (tiles x (ut/32)^2) 32x32 blocks
};
struct RedBatch {
  int n;
  int total;
  RedJob j[RED_MAX];
};

// One CTA per 32 x 32 block of a split unit tile: 256 threads, thread (ty, tx)
// owns rows ty + 8q (q < 4) of column tx.  Partials are summed in split order
// (deterministic), the single-split epilogue is applied, and every global
// access is a 128-byte row segment: direct stores walk rows, the mirror /
// transposed copies go through a padded shared-memory transpose.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const __grid_constant__ RedBatch b) {
  pdl_wait();
  pdl_trigger();
  __shared__ float T[32][33];
  const int blk = blockIdx.x;
  int p = 0;
  while (p + 1 < b.n && b.j[p + 1].slab_begin <= blk) ++p;
  const RedJob& J = b.j[p];
  const int ut = J.ut;
  const int nb = ut / 32;  // 32-blocks per tile edge
  const int local = blk - J.slab_begin;
  const int tile = local / (nb * nb);
  const int bi = (local - tile * nb * nb) / nb, bj = local % nb;
  int tm, tn;
  if (J.symmetric) {
    int r = static_cast<int>((sqrtf(8.0f * tile + 1.0f) - 1.0f) * 0.5f);
    while ((r + 1) * (r + 2) / 2 <= tile) ++r;
    while (r * (r + 1) / 2 > tile) --r;
    tm = r;
    tn = tile - r * (r + 1) / 2;
  } else {
    tm = tile / J.tiles_n;
    tn = tile - tm * J.tiles_n;
  }
  const bool diag = J.symmetric == 1 && tm == tn;
  if (diag && bj > bi) return;  // block entirely above the diagonal: the mirror writes it
  const int gm0 = tm * ut + bi * 32, gn0 = tn * ut + bj * 32;
  if (gm0 >= J.M || gn0 >= J.N) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t unit = static_cast<int64_t>(ut) * ut;
  const float* src = J.partials + static_cast<int64_t>(tile) * J.splits * unit +
                     static_cast<int64_t>(bi * 32) * ut + bj * 32 + tx;
  // 4 interleaved partial sums per element (splits s = 4t + u), so 16 loads are in
  // flight per thread; combined in a fixed order (deterministic)
  float acc4[4][4] = {};
  int s = 0;
  for (; s + 4 <= J.splits; s += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc4[u][q] += __ldcg(src + (s + u) * unit + static_cast<int64_t>(ty + 8 * q) * ut);
  }
  for (; s < J.splits; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) acc4[0][q] += __ldcg(src + s * unit + static_cast<int64_t>(ty + 8 * q) * ut);
  }
  float acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = (acc4[0][q] + acc4[1][q]) + (acc4[2][q] + acc4[3][q]);
  const int gn = gn0 + tx;
  const float vc = (J.epi == EPI_EIGDIV && gn < J.N) ? fmaxf(J.vcol[gn], 0.0f) : 0.0f;
  float alpha = J.alpha_amax ? ldexpf(J.alpha, 2 * prescale_exponent(__ldg(J.alpha_amax))) : J.alpha;
  if (J.amax_a) alpha = ldexpf(alpha, prescale_exponent(__ldg(J.amax_a)) + prescale_exponent(__ldg(J.amax_b)));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty + 8 * q;
    const int gm = gm0 + r;
    float val = alpha * acc[q];
    const bool in = gm < J.M && gn < J.N;
    if (J.epi == EPI_EIGDIV) {
      val = in ? val / (fmaxf(J.vrow[gm], 0.0f) * vc + J.gamma) : 0.0f;
    } else if (J.beta != 0.0f && in && !(diag && gn > gm)) {
      val += J.beta * J.cin[static_cast<int64_t>(gm) * J.ldc + gn];
    }
    if (in && !(diag && gn > gm)) J.out[static_cast<int64_t>(gm) * J.ldo + gn] = val;
    T[r][tx] = val;
  }
  if (J.symmetric != 1 && !J.out_t) return;
  __syncthreads();
  // transposed pass: element (row gm0 + tx, column gn0 + r) of the block goes to
  // out[gn0 + r][gm0 + tx] (mirror, strictly lower elements) and out_t likewise
  const int gmt = gm0 + tx;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int r = ty + 8 * q;
    const int gnt = gn0 + r;
    const float val = T[tx][r];
    const bool in = gmt < J.M && gnt < J.N && !(diag && gnt > gmt);
    if (J.symmetric == 1 && in && gnt != gmt) J.out[static_cast<int64_t>(gnt) * J.ldo + gmt] = val;
    if (J.out_t && in) J.out_t[static_cast<int64_t>(gnt) * J.ldt + gmt] = val;
  }
}

// ------------------------------------------------------------------ host: tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool tma_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_DISABLE_TMA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool mn3_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_MN3");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

bool dynamic_schedule() {  // DPK_DYN=0: static round-robin units
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_DYN");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

thread_local int g_cap_override = 0;
thread_local int g_units_override = 0;
}  // namespace
void set_grid_cap_override(int cap) { g_cap_override = cap; }
int grid_cap_override() { return g_cap_override; }
int units_per_sm_override() { return g_units_override; }
void set_units_per_sm_override(int u) { g_units_override = u; }
// split-K target: about this many units per worker.  Callers set it per context
// (UnitsPerSm guards: factor SYRKs 2, the latency-bound SPD rounds 1, everything else
// 3); DPK_UNITS_PER_SM overrides all of them (tuning).
int split_min_chunks() {  // no split-K piece below this many K chunks (DPK_SPLIT_MIN, default 64: measured)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_SPLIT_MIN");
    v = e ? std::max(1, atoi(e)) : 64;
  }
  return v;
}
int units_per_sm() {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("DPK_UNITS_PER_SM");
    env = e ? std::max(1, atoi(e)) : 0;
  }
  if (env > 0) return env;
  return g_units_override > 0 ? g_units_override : 3;
}
namespace {
int grid_cap() {
  if (g_cap_override > 0) return g_cap_override;
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("DPK_GRID_CAP");
    v = e ? atoi(e) : 0;
  }
  return v;
}

int units_per_cta() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("DPK_UNITS_PER_CTA");
    v = e ? atoi(e) : 0;
  }
  return v;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// tf32_rn: TMA rounds fp32 -> TF32 (nearest) in flight (TFLOAT32 data type);
// otherwise raw fp32 bits land in shared memory (tensor core truncates).
bool encode(CUtensorMap* m, int rank, const void* data, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box, bool tf32_rn, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  EncodeTiledFn fn = encoder();
  if (!fn) return false;
  const cuuint32_t es[3] = {1, 1, 1};
  return fn(m, tf32_rn ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(data), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D maps for row-major (K-major) / column-major (MN-major) operands.
int plan_tma_2d(const dpk_operand& o, CUtensorMap* m, bool rn) {
  if (o.kind == DPK_OPND_ROWS_K_F16) {
    if (tma_disabled() || o.bias_row || o.rows < 1 || !aligned16(o.data) || (o.ld * 2) % 16 != 0) return TMA_NONE;
    EncodeTiledFn fn = encoder();
    if (!fn) return TMA_NONE;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(o.cols), static_cast<cuuint64_t>(o.rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(o.ld) * 2};
    const cuuint32_t box[2] = {2 * BK, BM};
    const cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<float*>(o.data), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS
               ? TMA_ROWS_K16
               : TMA_NONE;
  }
  if (tma_disabled() || o.bias_row || o.rows < 1 || !aligned16(o.data) || (o.ld * 4) % 16 != 0) return TMA_NONE;
  if (o.kind == DPK_OPND_ROWS_K) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(o.cols), static_cast<cuuint64_t>(o.rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(o.ld) * 4};
    const cuuint32_t box[2] = {BK, BM};
    return encode(m, 2, o.data, dims, strides, box, rn) ? TMA_ROWS_K : TMA_NONE;
  }
  if (o.kind == DPK_OPND_ROWS_MN && o.rows % 32 == 0 && !mn3_disabled()) {
    const cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(o.cols), static_cast<cuuint64_t>(o.rows / 32)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(o.ld) * 4, 128};
    const cuuint32_t box[3] = {32, BK, BM / 32};
    if (encode(m, 3, o.data, dims, strides, box, rn, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) return TMA_ROWS_MN3;
  }
  if (o.kind == DPK_OPND_ROWS_MN) {
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(o.rows), static_cast<cuuint64_t>(o.cols)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(o.ld) * 4};
    const cuuint32_t box[2] = {32, BK};
    // MN-major tf32 must use the 32-byte-atom 128B swizzle (matches SWIZZLE_128B_BASE32B)
    return encode(m, 2, o.data, dims, strides, box, rn, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ? TMA_ROWS_MN : TMA_NONE;
  }
  return TMA_NONE;
}

// 3xF16 MN-major operand for the producers: one {128 rows, 32 k} box, no swizzle.
int plan_tma_mn_plain(const dpk_operand& o, CUtensorMap* m) {
  if (tma_disabled() || o.bias_row || o.rows < 1 || !aligned16(o.data) || (o.ld * 4) % 16 != 0) return TMA_NONE;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(o.rows), static_cast<cuuint64_t>(o.cols)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(o.ld) * 4};
  const cuuint32_t box[2] = {BM, BK};
  return encode(m, 2, o.data, dims, strides, box, false, CU_TENSOR_MAP_SWIZZLE_NONE) ? TMA_ROWS_MN_PLAIN : TMA_NONE;
}

// NCHW 1x1/s1 capture (or any conv grad_output): per sample a contiguous C x HW
// slab -> 3-D map {HW, C, N}; K is re-indexed as (sample, 32-pixel chunk).
bool slab_eligible(const dpk_operand& o) {
  return o.kind == DPK_OPND_IM2COL && !o.bias_row && o.kh == 1 && o.kw == 1 && o.sh == 1 && o.sw == 1 &&
         o.ph == 0 && o.pw == 0 && o.OH == o.H && o.OW == o.W && o.sws == 1 && o.shs == o.W &&
         aligned16(o.data) && (o.sc * 4) % 16 == 0 && (o.sn * 4) % 16 == 0 && !tma_disabled();
}

bool plan_tma_slab(const dpk_operand& o, CUtensorMap* m, bool rn) {
  const int64_t hw = static_cast<int64_t>(o.H) * o.W;
  const int64_t n = o.cols / hw;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(hw), static_cast<cuuint64_t>(o.C), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(o.sc) * 4, static_cast<cuuint64_t>(o.sn) * 4};
  const cuuint32_t box[3] = {BK, BM, 1};
  return encode(m, 3, o.data, dims, strides, box, rn);
}

// im2col-mode map over an NHWC conv input: dims {C, W, H, N}; the bounding box
// (lower corner -pad, upper corner pad - dilation*(k-1)) spans exactly the
// output pixels, traversed with the conv stride; a box is 32 output pixels x
// 32 channels (one 128 B row per pixel), written in the MN-major tf32 layout.
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn im2col_encoder() {
  static EncodeIm2colFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
  }
  return fn;
}

bool im2col_eligible(const dpk_operand& o) {
  return o.kind == DPK_OPND_IM2COL_TAPMAJOR && !o.bias_row && !tma_disabled() && o.C % 32 == 0 && o.sc == 1 &&
         aligned16(o.data) && (o.sws * 4) % 16 == 0 && (o.shs * 4) % 16 == 0 && (o.sn * 4) % 16 == 0 &&
         o.pw <= 127 && o.ph <= 127 && o.pw - o.dw * (o.kw - 1) >= -128 && o.ph - o.dh * (o.kh - 1) >= -128 &&
         o.sw <= 8 && o.sh <= 8 && o.dw * (o.kw - 1) < 65536 && o.dh * (o.kh - 1) < 65536;
}

bool plan_tma_im2col(const dpk_operand& o, CUtensorMap* m, bool rn) {
  EncodeIm2colFn fn = im2col_encoder();
  if (!fn) return false;
  const int64_t n = o.cols / (static_cast<int64_t>(o.OH) * o.OW);
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(o.C), static_cast<cuuint64_t>(o.W),
                              static_cast<cuuint64_t>(o.H), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(o.sws) * 4, static_cast<cuuint64_t>(o.shs) * 4,
                                 static_cast<cuuint64_t>(o.sn) * 4};
  const int lower[2] = {-o.pw, -o.ph};
  const int upper[2] = {o.pw - o.dw * (o.kw - 1), o.ph - o.dh * (o.kh - 1)};
  const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(o.sw), static_cast<cuuint32_t>(o.sh), 1};
  const CUresult r =
      fn(m, rn ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(o.data),
         dims, strides, lower, upper, 32, 32, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// DPK_OPND_IM2COL_TAPMAJOR_F16: the same im2col-mode map over the fp16 NHWC copy;
// a box is 64 output pixels x 64 channels (128 B per pixel), SWIZZLE_128B -- the
// MN-major kind::f16 operand image.  A 64-row group never crosses a tap (C % 64).
bool im2col16_eligible(const dpk_operand& o) {
  return o.kind == DPK_OPND_IM2COL_TAPMAJOR_F16 && !o.bias_row && !tma_disabled() && o.C % 64 == 0 &&
         o.sc == 1 && aligned16(o.data) && (o.sws * 2) % 16 == 0 && (o.shs * 2) % 16 == 0 &&
         (o.sn * 2) % 16 == 0 && o.pw <= 127 && o.ph <= 127 && o.pw - o.dw * (o.kw - 1) >= -128 &&
         o.ph - o.dh * (o.kh - 1) >= -128 && o.sw <= 8 && o.sh <= 8 && o.dw * (o.kw - 1) < 65536 &&
         o.dh * (o.kh - 1) < 65536 && o.cols % (static_cast<int64_t>(o.OH) * o.OW) == 0;
}

bool plan_tma_im2col16(const dpk_operand& o, CUtensorMap* m) {
  EncodeIm2colFn fn = im2col_encoder();
  if (!fn) return false;
  const int64_t n = o.cols / (static_cast<int64_t>(o.OH) * o.OW);
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(o.C), static_cast<cuuint64_t>(o.W),
                              static_cast<cuuint64_t>(o.H), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(o.sws) * 2, static_cast<cuuint64_t>(o.shs) * 2,
                                 static_cast<cuuint64_t>(o.sn) * 2};
  const int lower[2] = {-o.pw, -o.ph};
  const int upper[2] = {o.pw - o.dw * (o.kw - 1), o.ph - o.dh * (o.kh - 1)};
  const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(o.sw), static_cast<cuuint32_t>(o.sh), 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<float*>(o.data), dims, strides, lower, upper, 64, 64,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA_TAPS geometry: a K chunk is 32 output pixels = wb columns x hb rows of one
// output image block x nb samples (wb | OW, hb | OH exactly -- an invented pixel
// past the image edge could still read real input at a shifted tap; the sample
// tail is safe: samples >= N are TMA zero fill for every tap).  The widest
// spatial block wins (consecutive pixels are contiguous NHWC rows, so a box is a
// few dense DRAM runs); group boxes of 4/2/1 x 32 channels never cross a tap.
struct TapsGeom {
  int wb, hb, nb, nblk, g;
  int64_t chunks;
};

bool taps_disabled() {  // DPK_TAPS=0: keep TMA im2col mode / the gather path
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_TAPS");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

bool taps_4d();
bool taps_eligible(const dpk_operand& o, TapsGeom* tg = nullptr) {
  if (o.kind != DPK_OPND_IM2COL_TAPMAJOR || o.bias_row || tma_disabled() || taps_disabled()) return false;
  if (o.C % 32 != 0 || o.sc != 1 || !aligned16(o.data)) return false;
  if ((o.sws * 4) % 16 != 0 || (o.shs * 4) % 16 != 0 || (o.sn * 4) % 16 != 0) return false;
  if (o.sw > 8 || o.sh > 8 || o.OW < 1 || o.OH < 1) return false;
  const int64_t hw = static_cast<int64_t>(o.OH) * o.OW;
  if (o.cols % hw != 0) return false;
  const int64_t n = o.cols / hw;
  int bw = 1, bh = 1;
  for (int wb = 32; wb >= 1; wb /= 2) {
    if (o.OW % wb != 0 || wb * o.sw > 256) continue;
    for (int hb = 32 / wb; hb >= 1; hb /= 2) {
      if (o.OH % hb != 0 || hb * o.sh > 256) continue;
      if (wb * hb > bw * bh) {
        bw = wb;
        bh = hb;
      }
      break;
    }
  }
  if (tg) {
    tg->wb = bw;
    tg->hb = bh;
    tg->nb = 32 / (bw * bh);
    tg->nblk = static_cast<int>((n + tg->nb - 1) / tg->nb);
    tg->g = taps_4d() ? 0 : o.C % 128 == 0 ? 4 : o.C % 64 == 0 ? 2 : 1;
    tg->chunks = static_cast<int64_t>(o.OH / bh) * (o.OW / bw) * tg->nblk;
  }
  return tg == nullptr || tg->nblk < 65536;
}

bool taps_4d() {  // DPK_TAPS4D=1: 4-D maps {C, W, H, N}, one box per 32-row group
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_TAPS4D");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

bool plan_tma_taps(const dpk_operand& o, const TapsGeom& tg, CUtensorMap* m, bool rn) {
  EncodeTiledFn fn = encoder();
  if (!fn) return false;
  const int64_t n = o.cols / (static_cast<int64_t>(o.OH) * o.OW);
  if (tg.g == 0) {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(o.C), static_cast<cuuint64_t>(o.W),
                                static_cast<cuuint64_t>(o.H), static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(o.sws) * 4, static_cast<cuuint64_t>(o.shs) * 4,
                                   static_cast<cuuint64_t>(o.sn) * 4};
    const cuuint32_t box[4] = {32, static_cast<cuuint32_t>(tg.wb * o.sw), static_cast<cuuint32_t>(tg.hb * o.sh),
                               static_cast<cuuint32_t>(tg.nb)};
    const cuuint32_t es[4] = {1, static_cast<cuuint32_t>(o.sw), static_cast<cuuint32_t>(o.sh), 1};
    return fn(m, rn ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
              const_cast<float*>(o.data), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const cuuint64_t dims[5] = {32, static_cast<cuuint64_t>(o.W), static_cast<cuuint64_t>(o.H),
                              static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(o.C / 32)};
  const cuuint64_t strides[4] = {static_cast<cuuint64_t>(o.sws) * 4, static_cast<cuuint64_t>(o.shs) * 4,
                                 static_cast<cuuint64_t>(o.sn) * 4, 128};
  const cuuint32_t box[5] = {32, static_cast<cuuint32_t>(tg.wb * o.sw), static_cast<cuuint32_t>(tg.hb * o.sh),
                             static_cast<cuuint32_t>(tg.nb), static_cast<cuuint32_t>(tg.g)};
  const cuuint32_t es[5] = {1, static_cast<cuuint32_t>(o.sw), static_cast<cuuint32_t>(o.sh), 1, 1};
  return fn(m, rn ? CU_TENSOR_MAP_DATA_TYPE_TFLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(o.data),
            dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ------------------------------------------------------------------ host planning
struct Plan {
  std::vector<Problem> probs;
  size_t ws_bytes = 0;
  int cg = 1;
};

int operand_rows(const dpk_operand& o) { return o.rows + (o.bias_row ? 1 : 0); }

bool valid_operand(const dpk_operand& o) {
  if (o.data == nullptr && o.rows > 0) return false;
  if (o.rows < 0 || o.cols < 1) return false;
  if (is_im2col(o.kind) || o.kind == DPK_OPND_IM2COL_TAPMAJOR_F16) {
    if (o.kh < 1 || o.kw < 1 || o.sh < 1 || o.sw < 1 || o.dh < 1 || o.dw < 1 || o.OH < 1 || o.OW < 1) return false;
    if (o.rows != o.C * o.kh * o.kw) return false;
  } else if (o.kind != DPK_OPND_ROWS_K && o.kind != DPK_OPND_ROWS_MN && o.kind != DPK_OPND_ROWS_K_F16) {
    return false;
  }
  return true;
}


int make_plan(const GemmSpec* specs, int n, Plan& plan, bool with_maps, int precision = DPK_PREC_TF32, int cg = 1) {
  const bool rn = precision == DPK_PREC_TF32;
  const int UT = 128 * cg;
  plan.cg = cg;
  plan.probs.clear();
  plan.probs.resize(n);
  int64_t total_work = 0;
  for (int i = 0; i < n; ++i) {
    const dpk_gemm_job& j = specs[i].job;
    if (!valid_operand(j.a) || !valid_operand(j.b)) {
      set_error("dpk_gemm: invalid operand view (job " + std::to_string(i) + ")");
      return DPK_EARG;
    }
    if (j.a.cols != j.b.cols) {
      set_error("dpk_gemm: operand column (sample) counts differ (job " + std::to_string(i) + ")");
      return DPK_ESHAPE;
    }
    Problem& P = plan.probs[i];
    std::memset(static_cast<void*>(&P), 0, sizeof(P));
    P.a = j.a;
    P.b = j.b;
    P.out = j.out;
    P.cin = j.cin;
    P.ldo = j.ldo;
    P.ldc = j.ldc;
    P.alpha = j.alpha;
    P.alpha_amax = specs[i].alpha_amax;
    P.amax_a = specs[i].amax_a;
    P.amax_b = specs[i].amax_b;
    if (precision == DPK_PREC_3XF16) {
      auto plain = [](const dpk_operand& o) { return o.kind == DPK_OPND_ROWS_K || o.kind == DPK_OPND_ROWS_MN; };
      if (!P.amax_a || !P.amax_b || !plain(j.a) || !plain(j.b) || specs[i].alpha_amax) {
        set_error("dpk_gemm: 3xF16 needs amax slots for both operands and plain row / column views");
        return DPK_EARG;
      }
    } else if (P.amax_a || P.amax_b) {
      set_error("dpk_gemm: operand amax slots are a 3xF16 feature");
      return DPK_EARG;
    }
    P.beta = j.beta;
    P.M = operand_rows(j.a);
    P.N = operand_rows(j.b);
    P.symmetric = j.symmetric ? (specs[i].lower_only ? 2 : 1) : 0;
    if (P.symmetric && P.M != P.N) {
      set_error("dpk_gemm: symmetric output needs M == N");
      return DPK_ESHAPE;
    }
    P.same_ab = std::memcmp(&j.a, &j.b, sizeof(dpk_operand)) == 0 ? 1 : 0;
    P.epi = specs[i].epi;
    P.vrow = specs[i].vrow;
    P.vcol = specs[i].vcol;
    P.gamma = specs[i].gamma;
    P.out_t = specs[i].out_t;
    P.ldt = specs[i].ldt;
    P.tri_a = specs[i].tri_a;
    P.tri_b = specs[i].tri_b;
    // K clipping makes tile cost grow along one tile index: visit the heavy
    // tiles first so the static round-robin schedule ends on light ones
    P.order = P.tri_a == TRI_LOWER ? 1 : P.tri_b == TRI_LOWER ? 3 : P.tri_b == TRI_UPPER ? 2 : 0;
    if (P.beta != 0.0f && P.cin == nullptr) {
      set_error("dpk_gemm: beta != 0 needs cin");
      return DPK_EARG;
    }
    const int tmn = (P.M + UT - 1) / UT;
    P.tiles_n = (P.N + UT - 1) / UT;
    P.ntiles = P.symmetric ? tmn * (tmn + 1) / 2 : tmn * P.tiles_n;
    P.chunks = static_cast<int>((j.a.cols + BK - 1) / BK);
    const bool f16a = j.a.kind == DPK_OPND_ROWS_K_F16 || j.a.kind == DPK_OPND_IM2COL_TAPMAJOR_F16;
    const bool f16b = j.b.kind == DPK_OPND_ROWS_K_F16 || j.b.kind == DPK_OPND_IM2COL_TAPMAJOR_F16;
    if (f16a || f16b) {
      if (!(f16a && f16b) || precision != DPK_PREC_TF32 || P.tri_a || P.tri_b) {
        set_error("dpk_gemm: fp16 operands need fp16 on both sides, 1-pass precision, no triangular clipping");
        return DPK_EARG;
      }
      if (j.a.kind == DPK_OPND_IM2COL_TAPMAJOR_F16 && (!P.same_ab || !im2col16_eligible(j.a))) {
        set_error("dpk_gemm: DPK_OPND_IM2COL_TAPMAJOR_F16 is a SYRK-only, TMA-only view (C % 64 == 0, c "
                  "contiguous, 16-byte aligned strides, no bias row, padding within the TMA im2col limits)");
        return DPK_EARG;
      }
      P.chunks = static_cast<int>((j.a.cols + 2 * BK - 1) / (2 * BK));
    }
    TapsGeom tg;
    if (P.same_ab && taps_eligible(j.a, &tg)) {
      P.chunks = static_cast<int>(tg.chunks);
      P.slab_cpn = tg.wb | (tg.hb << 6) | (tg.g << 12) | (tg.nblk << 16);
      if (with_maps) {
        if (!plan_tma_taps(j.a, tg, &P.tmap_a, rn)) {
          set_error("dpk_gemm: cuTensorMapEncodeTiled rejected the implicit-im2col (taps) map");
          return DPK_ECUDA;
        }
        P.tmap_b = P.tmap_a;
        P.tma_a = P.tma_b = TMA_TAPS;
      }
    } else if (P.same_ab && slab_eligible(j.a)) {
      // SYRK over an NCHW slab: both operands through one 3-D map, K = (sample, chunk)
      const int64_t hw = static_cast<int64_t>(j.a.H) * j.a.W;
      P.slab_cpn = static_cast<int>((hw + BK - 1) / BK);
      P.chunks = static_cast<int>((j.a.cols / hw) * P.slab_cpn);
      if (with_maps) {
        if (plan_tma_slab(j.a, &P.tmap_a, rn)) {
          P.tmap_b = P.tmap_a;
          P.tma_a = P.tma_b = TMA_SLAB;
        } else {  // cannot happen for eligible views; fall back to the flat gather
          P.slab_cpn = 0;
          P.chunks = static_cast<int>((j.a.cols + BK - 1) / BK);
        }
      }
    } else if (with_maps) {
      auto plan_one = [&](const dpk_operand& o, CUtensorMap* m) -> int {
        if (o.kind == DPK_OPND_IM2COL_TAPMAJOR_F16) return plan_tma_im2col16(o, m) ? TMA_IM2COL16 : TMA_NONE;
        if (o.kind == DPK_OPND_IM2COL_TAPMAJOR)
          return (im2col_eligible(o) && plan_tma_im2col(o, m, rn)) ? TMA_IM2COL : TMA_NONE;
        if (precision == DPK_PREC_3XF16 && o.kind == DPK_OPND_ROWS_MN) return plan_tma_mn_plain(o, m);
        return plan_tma_2d(o, m, rn);
      };
      P.tma_a = plan_one(j.a, &P.tmap_a);
      if (j.a.kind == DPK_OPND_IM2COL_TAPMAJOR_F16 && P.tma_a == TMA_NONE) {
        set_error("dpk_gemm: cuTensorMapEncodeIm2col rejected the fp16 implicit-im2col map");
        return DPK_ECUDA;
      }
      if (P.same_ab) {
        P.tma_b = P.tma_a;
        P.tmap_b = P.tmap_a;
      } else {
        P.tma_b = plan_one(j.b, &P.tmap_b);
      }
    }
    // block-diagonal operands: every tile reads one tile edge of K (no split-K)
    const bool blockdiag = P.tri_a == TRI_BLOCK || P.tri_b == TRI_BLOCK;
    total_work += static_cast<int64_t>(P.ntiles) * (blockdiag ? std::min(P.chunks, UT / BK) : P.chunks);
  }
  // Split K so that the group yields ~3 units per SM, but never below 32 chunks
  // (1024 samples) per unit so tile set-up and the partial round trip stay amortised.
  const int64_t sms = num_sms() / cg;  // workers: CTAs or CTA pairs
  const int64_t per = units_per_sm();
  const int64_t target = std::max<int64_t>(split_min_chunks(), (total_work + per * sms - 1) / (per * sms));
  size_t partial_tiles = 0;
  for (auto& P : plan.probs) {
    P.splits = static_cast<int>(std::max<int64_t>(1, (P.chunks + target - 1) / target));
    if (P.tri_a == TRI_BLOCK || P.tri_b == TRI_BLOCK) P.splits = 1;
    P.cps = (P.chunks + P.splits - 1) / P.splits;
    P.splits = (P.chunks + P.cps - 1) / P.cps;
    if (P.splits > 1) partial_tiles += static_cast<size_t>(P.ntiles) * P.splits;
  }
  plan.ws_bytes = SCHED_BYTES + partial_tiles * UT * UT * sizeof(float);
  return DPK_OK;
}

// CTA-pair (256x256 unit) eligibility, decided without encoding tensor maps so
// the workspace query and the launch partition identically: every operand must
// be TMA-addressable (CG=2 has no manual gather path) and both output edges
// must exceed one 128 tile (smaller problems waste the 256-wide unit).
bool tma_possible_2d(const dpk_operand& o) {
  if (o.kind == DPK_OPND_ROWS_K_F16)
    return !tma_disabled() && !o.bias_row && o.rows >= 1 && aligned16(o.data) && (o.ld * 2) % 16 == 0;
  return !tma_disabled() && !o.bias_row && o.rows >= 1 && aligned16(o.data) && (o.ld * 4) % 16 == 0 &&
         (o.kind == DPK_OPND_ROWS_K || o.kind == DPK_OPND_ROWS_MN);
}

bool cg2_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_CG2");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

bool wants_cg2(const GemmSpec& g) {
  if (!cg2_enabled()) return false;
  const dpk_gemm_job& j = g.job;
  if (operand_rows(j.a) <= 128 || operand_rows(j.b) <= 128) return false;
  const bool same = std::memcmp(&j.a, &j.b, sizeof(dpk_operand)) == 0;
  auto ok = [&](const dpk_operand& o) {
    if (tma_possible_2d(o)) return true;
    if (o.kind == DPK_OPND_IM2COL_TAPMAJOR_F16) return im2col16_eligible(o);
    if (o.kind == DPK_OPND_IM2COL_TAPMAJOR) return im2col_eligible(o);
    return false;
  };
  if (same && (slab_eligible(j.a) || taps_eligible(j.a))) return true;
  return ok(j.a) && (same || ok(j.b));
}

// Pairs only pay when the eligible problems give every pair work: a group whose
// 256x256 units -- counting the split-K pieces of at least 32 chunks that long-K
// problems can be cut into -- cannot fill the GPU runs as single CTAs, where
// twice the CTAs share the same output (measured: the 2048/2304 Schur rounds of
// the SPD recursion lose 30% as pairs, the 4608 products gain 30%; a 576 x 100352
// factor SYRK gains as pairs despite the 256-row padding).
void partition_cg(const GemmSpec* specs, int n, std::vector<GemmSpec>& g1, std::vector<GemmSpec>& g2) {
  g1.clear();
  g2.clear();
  int64_t units2 = 0;
  for (int i = 0; i < n; ++i) {
    if (!wants_cg2(specs[i])) continue;
    const int64_t tm = (operand_rows(specs[i].job.a) + 255) / 256, tn = (operand_rows(specs[i].job.b) + 255) / 256;
    const int64_t pieces = std::max<int64_t>(1, specs[i].job.a.cols / (32 * BK));
    units2 += (specs[i].job.symmetric ? tm * (tm + 1) / 2 : tm * tn) * pieces;
  }
  const bool pairs = units2 >= num_sms();
  for (int i = 0; i < n; ++i) (pairs && wants_cg2(specs[i]) ? g2 : g1).push_back(specs[i]);
}

int launch_reduce(const std::vector<Problem>& probs, int ut, cudaStream_t st) {
  thread_local RedBatch rb;
  rb.n = 0;
  rb.total = 0;
  auto flush = [&]() -> int {
    if (rb.n == 0) return DPK_OK;
    const cudaError_t e = launch_k(splitk_reduce_kernel, dim3(rb.total), dim3(256), 0, st, 1, rb);
    note_launch();
    rb.n = 0;
    rb.total = 0;
    return cuda_status(e, "splitk_reduce_kernel launch");
  };
  for (const auto& P : probs) {
    if (P.splits <= 1) continue;
    if (rb.n == RED_MAX) {
      int rc = flush();
      if (rc) return rc;
    }
    RedJob& J = rb.j[rb.n++];
    J.out = P.out;
    J.cin = P.cin;
    J.vrow = P.vrow;
    J.vcol = P.vcol;
    J.partials = P.partials;
    J.out_t = P.out_t;
    J.ldo = P.ldo;
    J.ldc = P.ldc;
    J.ldt = P.ldt;
    J.alpha = P.alpha;
    J.alpha_amax = P.alpha_amax;
    J.amax_a = P.amax_a;
    J.amax_b = P.amax_b;
    J.beta = P.beta;
    J.gamma = P.gamma;
    J.M = P.M;
    J.N = P.N;
    J.symmetric = P.symmetric;
    J.epi = P.epi;
    J.tiles_n = P.tiles_n;
    J.splits = P.splits;
    J.ut = ut;
    J.slab_begin = rb.total;
    rb.total += P.ntiles * (ut * ut / 1024);
  }
  return flush();
}

template <int NPASS, bool RN, int CG, bool GATHER = true>
int launch_batch(const Batch& bt, cudaStream_t st) {
  using C = Cfg<NPASS>;
  static std::atomic<uint64_t> configured_on{0};
  static int max_pairs = 0;
  if (first_on_device(configured_on)) {
    cudaError_t e =
        cudaFuncSetAttribute(tc_gemm_kernel<NPASS, RN, CG, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             SMEM_SM_EXCL);
    if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(tc_gemm_kernel)");
    if (CG == 2) {
      cudaLaunchConfig_t q = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.gridDim = dim3(2 * (num_sms() / 2), 1, 1);
      q.blockDim = dim3(NTHREADS, 1, 1);
      q.dynamicSmemBytes = SMEM_SM_EXCL;
      q.attrs = at;
      q.numAttrs = 1;
      int clusters = 0;
      e = cudaOccupancyMaxActiveClusters(&clusters, tc_gemm_kernel<NPASS, RN, CG, GATHER>, &q);
      if (e != cudaSuccess) return cuda_status(e, "cudaOccupancyMaxActiveClusters(tc_gemm_kernel)");
      max_pairs = std::max(clusters, 1);
    }
  }
  // persistent CTAs (CTA pairs) walk the units round-robin; DPK_UNITS_PER_CTA
  // caps how many units one CTA takes, so long launches hand SMs back to the
  // block scheduler (and to higher-priority streams) between units
  const int cap = grid_cap();  // experiment: leave SMs to concurrent streams
  const int workers = cap > 0 ? std::max(1, std::min(CG == 1 ? num_sms() : max_pairs, cap / CG))
                              : (CG == 1 ? num_sms() : max_pairs);
  const int upc = units_per_cta();
  const int want = upc > 0 ? std::max(workers, (bt.total_units + upc - 1) / upc) : workers;
  const int grid = CG == 1 ? std::min(bt.total_units, want) : 2 * std::min(bt.total_units, want);
  const cudaError_t e =
      launch_k(tc_gemm_kernel<NPASS, RN, CG, GATHER>, dim3(grid), dim3(NTHREADS), SMEM_SM_EXCL, st, CG, bt);
  note_launch();
  return cuda_status(e, "tc_gemm_kernel launch");
}

template <int CG>
int launch_group(const Batch& bt, int precision, cudaStream_t st) {
  bool tma_only = true;
  for (int i = 0; i < bt.nprob; ++i) tma_only = tma_only && bt.p[i].tma_a != TMA_NONE && bt.p[i].tma_b != TMA_NONE;
  if (precision == DPK_PREC_3XTF32)
    return tma_only ? launch_batch<3, false, CG, false>(bt, st) : launch_batch<3, false, CG>(bt, st);
  if (precision == DPK_PREC_3XF16)  // (RN slot = the fp16 split)
    return tma_only ? launch_batch<3, true, CG, false>(bt, st) : launch_batch<3, true, CG>(bt, st);
  if (precision == DPK_PREC_TF32_TRUNC) return launch_batch<1, false, CG>(bt, st);
  return launch_batch<1, true, CG>(bt, st);
}

bool chunk_fork_enabled() {  // DPK_CHUNK_FORK=0: a plan's MAXP-problem launches back to back on one stream
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_CHUNK_FORK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// One plan (all problems share the unit-tile size) -> grouped launches of up to
// MAXP problems, then the split-K reduction.  A plan of more problems than one
// launch holds alternates its launches between the caller's stream and a forked
// lane (each with its own scheduler counters), so a launch's tail overlaps the
// next launch's start; the reduction joins both.
int run_plan(Plan& plan, void* ws, size_t ws_bytes, int precision, cudaStream_t st) {
  if (plan.ws_bytes > ws_bytes || ws == nullptr) {
    set_error("dpk_gemm: workspace too small (" + std::to_string(ws_bytes) + " < " +
              std::to_string(plan.ws_bytes) + ")");
    return DPK_ENOSPACE;
  }
  const int ut = 128 * plan.cg;
  size_t partial_tiles = 0;
  // workspace: [scheduler counters | split-K partials]
  int* sched = static_cast<int*>(ws);
  float* partials = reinterpret_cast<float*>(static_cast<char*>(ws) + SCHED_BYTES);
  for (auto& P : plan.probs) {
    if (P.splits > 1) {
      P.partials = partials + partial_tiles * ut * ut;
      partial_tiles += static_cast<size_t>(P.ntiles) * P.splits;
    }
  }
  const int n = static_cast<int>(plan.probs.size());
  ForkLane* lane = nullptr;
  // not under an SM cap: two concurrent capped launches would hold twice the cap
  // (and halving the cap per lane measured slower: ResNet-50 6.65 -> 6.90 ms)
  if (n > MAXP && chunk_fork_enabled() && grid_cap() == 0) {
    int rc = fork_lane(st, lane, 1);
    if (!rc) rc = fork_begin(lane, st);
    if (rc) return rc;
  }
  thread_local Batch bt;  // host-side staging only (kernel params are copied at launch)
  for (int first = 0; first < n; first += MAXP) {
    const int cnt = std::min(MAXP, n - first);
    const bool odd = lane != nullptr && ((first / MAXP) & 1);
    cudaStream_t s = odd ? fork_side(lane) : st;
    bt.nprob = cnt;
    int units = 0;
    for (int i = 0; i < cnt; ++i) {
      bt.p[i] = plan.probs[first + i];
      bt.p[i].unit_begin = units;
      units += bt.p[i].ntiles * bt.p[i].splits;
    }
    bt.total_units = units;
    bt.debug_ts = debug_ts_enabled() ? 1 : 0;
    bt.sched = sched + (odd ? 2 : 0);  // a counter pair per lane (every launch leaves its pair zero)
    bt.dynamic = dynamic_schedule() ? 1 : 0;
    // producer warps are needed for 3xTF32 low parts and for operands TMA cannot address
    bt.producers = (precision == DPK_PREC_3XTF32 || precision == DPK_PREC_3XF16) ? 1 : 0;
    for (int i = 0; i < cnt; ++i)
      if (bt.p[i].tma_a == TMA_NONE || bt.p[i].tma_b == TMA_NONE) bt.producers = 1;
    if (units == 0) continue;
    const int rc = plan.cg == 2 ? launch_group<2>(bt, precision, s) : launch_group<1>(bt, precision, s);
    if (rc != DPK_OK) return rc;
  }
  if (lane) {
    const int rc = fork_end(lane, st);
    if (rc) return rc;
  }
  return launch_reduce(plan.probs, ut, st);
}

}  // namespace

bool debug_ts_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_DEBUG_TS");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

std::string specs_key(const GemmSpec* specs, int n, int precision) {
  std::string k;
  k.reserve(static_cast<size_t>(n) * (sizeof(GemmSpec) + 8) + 16);
  int dev = 0;
  cudaGetDevice(&dev);
  key_put(k, dev);
  key_put(k, precision);
  key_put(k, units_per_sm());  // the split-K plan depends on it
  for (int i = 0; i < n; ++i) key_spec(k, specs[i]);
  return k;
}

size_t gemm_workspace_bytes_uncached(const GemmSpec* specs, int n);

// DPK_GEMM_FORK=0: run the CTA-pair and the single-CTA plans of one call back to back
bool concurrent_plans() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("DPK_GEMM_FORK");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// One forked stream per caller stream (same priority), with its fork/join events:
// the single-CTA plan of a call runs there beside the pair plan, so the small
// problems of a group (precondition phases, SPD rounds with mixed sizes) fill the
// SMs the pair launch's tail leaves idle instead of queueing behind it.
struct ForkLane {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
int fork_lane(cudaStream_t st, ForkLane*& out, int purpose) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<cudaStream_t, int>, ForkLane*>> lanes;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : lanes)
    if (e.first.first == st && e.first.second == purpose) {
      out = e.second;
      return DPK_OK;
    }
  ForkLane* L = new ForkLane();
  int prio = 0;
  cudaStreamGetPriority(st, &prio);
  int rc = cuda_status(cudaStreamCreateWithPriority(&L->side, cudaStreamNonBlocking, prio), "cudaStreamCreate(fork)");
  if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&L->fork, cudaEventDisableTiming), "cudaEventCreate(fork)");
  if (!rc) rc = cuda_status(cudaEventCreateWithFlags(&L->join, cudaEventDisableTiming), "cudaEventCreate(join)");
  if (rc) return rc;
  lanes.emplace_back(std::make_pair(st, purpose), L);
  out = L;
  return DPK_OK;
}
int fork_begin(ForkLane* L, cudaStream_t st) {
  int rc = cuda_status(cudaEventRecord(L->fork, st), "cudaEventRecord(fork)");
  if (!rc) rc = cuda_status(cudaStreamWaitEvent(L->side, L->fork, 0), "cudaStreamWaitEvent(fork)");
  return rc;
}
int fork_end(ForkLane* L, cudaStream_t st) {
  int rc = cuda_status(cudaEventRecord(L->join, L->side), "cudaEventRecord(join)");
  if (!rc) rc = cuda_status(cudaStreamWaitEvent(st, L->join, 0), "cudaStreamWaitEvent(join)");
  return rc;
}
cudaStream_t fork_side(ForkLane* L) { return L->side; }

size_t gemm_workspace_bytes(const GemmSpec* specs, int n) {
  if (n <= 0) return 0;
  static LruCache<size_t> cache;
  const std::string k = specs_key(specs, n, 0);
  {
    std::lock_guard<std::mutex> lock(cache.mu);
    if (size_t* v = cache.find(k)) return *v;
  }
  const size_t ws = gemm_workspace_bytes_uncached(specs, n);
  std::lock_guard<std::mutex> lock(cache.mu);
  cache.put(k, ws);
  return ws;
}

// 3xF16: two amax slots per job at the END of the caller's workspace
size_t amax_region(int n) { return align_up(static_cast<size_t>(n) * 8, 1024); }

int launch_operand_amax(const GemmSpec* specs, int n, int32_t* slots, cudaStream_t st) {
  int rc = cuda_status(cudaMemsetAsync(slots, 0, static_cast<size_t>(n) * 8, st), "cudaMemsetAsync(amax slots)");
  if (rc) return rc;
  thread_local AmaxBatch ab;
  ab.n = 0;
  int64_t most = 1;
  auto flush = [&]() -> int {
    if (ab.n == 0) return DPK_OK;
    const int gx = static_cast<int>(std::min<int64_t>(most, 2 * num_sms()));
    operand_amax_kernel<<<dim3(gx, ab.n), 256, 0, st>>>(ab);
    note_launch();
    ab.n = 0;
    most = 1;
    return cuda_status(cudaGetLastError(), "operand_amax_kernel launch");
  };
  for (int i = 0; i < n; ++i) {
    for (int side = 0; side < 2; ++side) {
      const dpk_operand& o = side ? specs[i].job.b : specs[i].job.a;
      AmaxView& v = ab.v[ab.n++];
      v.data = o.data;
      v.ld = o.ld;
      v.cols = o.cols;
      v.rows = o.rows;
      v.mn = o.kind == DPK_OPND_ROWS_MN;
      v.tri = side ? specs[i].tri_b : specs[i].tri_a;
      v.bias = o.bias_row;
      v.out = slots + 2 * i + side;
      most = std::max<int64_t>(most, v.mn ? o.cols : o.rows);
      if (ab.n == AMAX_MAXV && (rc = flush())) return rc;
    }
  }
  return flush();
}

size_t gemm_workspace_bytes_uncached(const GemmSpec* specs, int n) {
  std::vector<GemmSpec> g1, g2;
  partition_cg(specs, n, g1, g2);
  size_t w1 = 0, w2 = 0;
  Plan plan;
  if (!g1.empty() && make_plan(g1.data(), static_cast<int>(g1.size()), plan, false, DPK_PREC_TF32, 1) == DPK_OK)
    w1 = plan.ws_bytes;
  if (!g2.empty() && make_plan(g2.data(), static_cast<int>(g2.size()), plan, false, DPK_PREC_TF32, 2) == DPK_OK)
    w2 = plan.ws_bytes;
  // both unit shapes present: the single-CTA plan runs concurrently with the pair
  // plan in its own workspace region behind the pair plan's; the 3xF16 operand
  // scales take the last bytes
  if (w1 && w2 && concurrent_plans()) return align_up(w2, 1024) + w1 + amax_region(n);
  return std::max(w1, w2) + amax_region(n);
}

int gemm_launch(const GemmSpec* specs, int n, void* ws, size_t ws_bytes, int precision, cudaStream_t st,
                bool zero_counters) {
  if (n == 0) return DPK_OK;
  if (n < 0 || specs == nullptr) {
    set_error("dpk_gemm: bad job list");
    return DPK_EARG;
  }
  if (precision != DPK_PREC_TF32 && precision != DPK_PREC_TF32_TRUNC && precision != DPK_PREC_3XTF32 &&
      precision != DPK_PREC_3XF16) {
    set_error("dpk_gemm: precision must be DPK_PREC_TF32, DPK_PREC_TF32_TRUNC, DPK_PREC_3XTF32 or DPK_PREC_3XF16");
    return DPK_EARG;
  }
  // small 3xTF32 groups (deep SPD-recursion rounds): latency path on CUDA cores
  if (simt_eligible(specs, n, precision)) return simt_gemm_launch(specs, n, st);
  // 3xF16: every operand's amax into the slots at the end of the workspace (one launch)
  thread_local std::vector<GemmSpec> scaled;
  if (precision == DPK_PREC_3XF16 && !specs[0].amax_a) {
    const size_t reg = amax_region(n);
    if (ws == nullptr || ws_bytes < reg + SCHED_BYTES) {
      set_error("dpk_gemm: workspace too small for the 3xF16 operand scales");
      return DPK_ENOSPACE;
    }
    ws_bytes -= reg;
    int32_t* slots = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + ws_bytes);
    scaled.assign(specs, specs + n);
    for (int i = 0; i < n; ++i) {
      scaled[i].amax_a = slots + 2 * i;
      scaled[i].amax_b = slots + 2 * i + 1;
    }
    const int rc = launch_operand_amax(scaled.data(), n, slots, st);
    if (rc) return rc;
    specs = scaled.data();
  }
  if (zero_counters && ws != nullptr && ws_bytes >= SCHED_BYTES) {
    const int rc = cuda_status(cudaMemsetAsync(ws, 0, SCHED_BYTES, st), "cudaMemsetAsync(scheduler counters)");
    if (rc) return rc;
  }
  // big problems run on CTA pairs, the rest on single CTAs (two launches, same
  // stream: the split-K workspace is reused in order).  The plans (tensor maps
  // included) of a job list seen before come from the cache.
  static LruCache<std::vector<Plan>> cache;
  const std::string key = specs_key(specs, n, precision);
  std::vector<Plan> plans;
  {
    std::lock_guard<std::mutex> lock(cache.mu);
    if (std::vector<Plan>* v = cache.find(key)) plans = *v;
  }
  if (plans.empty()) {
    std::vector<GemmSpec> g1, g2;
    partition_cg(specs, n, g1, g2);
    for (int cg = 2; cg >= 1; --cg) {
      std::vector<GemmSpec>& g = cg == 2 ? g2 : g1;
      if (g.empty()) continue;
      Plan plan;
      int rc = make_plan(g.data(), static_cast<int>(g.size()), plan, true, precision, cg);
      if (rc != DPK_OK) return rc;
      if (cg == 2) {
        // a view the predicate accepted must have been TMA-planned; anything else
        // (encode failure) is an internal inconsistency, not a silent fallback
        for (const auto& P : plan.probs) {
          if (P.tma_a == TMA_NONE || (!P.same_ab && P.tma_b == TMA_NONE)) {
            set_error("dpk_gemm: CTA-pair problem without a TMA plan (tensor map encode failed)");
            return DPK_ECUDA;
          }
        }
      }
      plans.push_back(std::move(plan));
    }
    std::lock_guard<std::mutex> lock(cache.mu);
    cache.put(key, plans);
  }
  if (plans.size() == 2 && concurrent_plans() && ws != nullptr) {
    // plans[0]: CTA pairs on the caller's stream; plans[1]: single CTAs on the fork lane
    const size_t off = align_up(plans[0].ws_bytes, 1024);
    if (ws_bytes >= off + plans[1].ws_bytes) {
      ForkLane* L = nullptr;
      int rc = fork_lane(st, L, 0);
      if (rc) return rc;
      char* ws2 = static_cast<char*>(ws) + off;
      rc = cuda_status(cudaEventRecord(L->fork, st), "cudaEventRecord(fork)");
      if (!rc) rc = cuda_status(cudaStreamWaitEvent(L->side, L->fork, 0), "cudaStreamWaitEvent(fork)");
      // the region's scheduler counters: offsets move with the job list, so they are
      // cleared on every fork (callers that skip the clear own only the first region)
      if (!rc) rc = cuda_status(cudaMemsetAsync(ws2, 0, SCHED_BYTES, L->side), "cudaMemsetAsync(fork counters)");
      if (!rc) rc = run_plan(plans[1], ws2, ws_bytes - off, precision, L->side);
      if (!rc) rc = run_plan(plans[0], ws, off, precision, st);
      if (!rc) rc = cuda_status(cudaEventRecord(L->join, L->side), "cudaEventRecord(join)");
      if (!rc) rc = cuda_status(cudaStreamWaitEvent(st, L->join, 0), "cudaStreamWaitEvent(join)");
      return rc;
    }
  }
  for (Plan& plan : plans) {
    const int rc = run_plan(plan, ws, ws_bytes, precision, st);
    if (rc != DPK_OK) return rc;
  }
  return DPK_OK;
}

}  // namespace dpk

// ===================================================================== C ABI
extern "C" {

size_t dpk_gemm_workspace_bytes(const dpk_gemm_job* jobs, int n_jobs) {
  std::vector<dpk::GemmSpec> specs(std::max(n_jobs, 0));
  for (int i = 0; i < n_jobs; ++i) specs[i] = dpk::GemmSpec{jobs[i], dpk::EPI_LINEAR, nullptr, nullptr, 0.f, nullptr, 0, 0, 0};
  return dpk::gemm_workspace_bytes(specs.data(), n_jobs);
}

int dpk_gemm(const dpk_gemm_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, int precision,
             dpk_stream_t stream) {
  if (n_jobs < 0 || (n_jobs > 0 && jobs == nullptr)) {
    dpk::set_error("dpk_gemm: bad job list");
    return DPK_EARG;
  }
  std::vector<dpk::GemmSpec> specs(n_jobs);
  for (int i = 0; i < n_jobs; ++i) specs[i] = dpk::GemmSpec{jobs[i], dpk::EPI_LINEAR, nullptr, nullptr, 0.f, nullptr, 0, 0, 0};
  return dpk::gemm_launch(specs.data(), n_jobs, workspace, ws_bytes, precision,
                          static_cast<cudaStream_t>(stream));
}

static std::vector<dpk::GemmSpec> factor_specs(const dpk_factor_job* jobs, int n) {
  std::vector<dpk::GemmSpec> specs(std::max(n, 0));
  for (int i = 0; i < n; ++i) {
    dpk_gemm_job g{};
    g.a = jobs[i].x;
    g.b = jobs[i].x;
    const int d = jobs[i].x.rows + (jobs[i].x.bias_row ? 1 : 0);
    g.out = jobs[i].factor;
    g.ldo = d;
    g.cin = jobs[i].factor;
    g.ldc = d;
    g.alpha = jobs[i].alpha;
    g.beta = jobs[i].beta;
    g.symmetric = 1;
    specs[i] = dpk::GemmSpec{g, dpk::EPI_LINEAR, nullptr, nullptr, 0.f, nullptr, 0, 0, 0};
    specs[i].alpha_amax = jobs[i].x_amax;
  }
  return specs;
}

size_t dpk_factor_workspace_bytes(const dpk_factor_job* jobs, int n_jobs) {
  dpk::UnitsPerSm units(2);  // factor SYRKs: measured best split-K depth
  auto specs = factor_specs(jobs, n_jobs);
  return dpk::gemm_workspace_bytes(specs.data(), n_jobs);
}

int dpk_syrk_ema(const dpk_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, int precision,
                 dpk_stream_t stream) {
  if (n_jobs < 0 || (n_jobs > 0 && jobs == nullptr)) {
    dpk::set_error("dpk_syrk_ema: bad job list");
    return DPK_EARG;
  }
  for (int i = 0; i < n_jobs; ++i) {
    if (jobs[i].factor == nullptr) {
      dpk::set_error("dpk_syrk_ema: null factor pointer");
      return DPK_EARG;
    }
    if (jobs[i].x.cols < 1) {
      dpk::set_error("captured inputs must be a nonempty d x B matrix");
      return DPK_EARG;
    }
  }
  dpk::UnitsPerSm units(2);
  auto specs = factor_specs(jobs, n_jobs);
  return dpk::gemm_launch(specs.data(), n_jobs, workspace, ws_bytes, precision, static_cast<cudaStream_t>(stream));
}

int dpk_conv_im2col_syrk_ema(const dpk_factor_job* jobs, int n_jobs, void* workspace, size_t ws_bytes,
                             int precision, dpk_stream_t stream) {
  for (int i = 0; i < n_jobs; ++i) {
    if (!dpk::is_im2col(jobs[i].x.kind) && jobs[i].x.kind != DPK_OPND_IM2COL_TAPMAJOR_F16) {
      dpk::set_error("dpk_conv_im2col_syrk_ema: operand must be DPK_OPND_IM2COL, DPK_OPND_IM2COL_TAPMAJOR or "
                     "DPK_OPND_IM2COL_TAPMAJOR_F16");
      return DPK_EARG;
    }
  }
  return dpk_syrk_ema(jobs, n_jobs, workspace, ws_bytes, precision, stream);
}

}  // extern "C"

// Debug: %globaltimer checkpoints (ns) of CTA 0 of the last GEMM launch made with
// DPK_DEBUG_TS=1: start, set-up done, TMA done, gathers done, MMA done,
// epilogue unit 0 / last unit done, final barrier, TMEM released.
extern "C" int dpk_set_launch_cap(int sms) {
  if (sms < 0) {
    dpk::set_error("dpk_set_launch_cap: sms must be >= 0");
    return DPK_EARG;
  }
  dpk::set_grid_cap_override(sms);
  return DPK_OK;
}

extern "C" int dpk_debug_unit_timestamps(unsigned long long* host320) {
  if (!host320) return DPK_EARG;
  return dpk::cuda_status(cudaMemcpyFromSymbol(host320, dpk::g_dbg_unit, sizeof(unsigned long long) * 320),
                          "cudaMemcpyFromSymbol");
}

extern "C" int dpk_debug_timestamps(unsigned long long* host16) {
  if (!host16) return DPK_EARG;
  return dpk::cuda_status(cudaMemcpyFromSymbol(host16, dpk::g_dbg_ts, sizeof(unsigned long long) * 16),
                          "cudaMemcpyFromSymbol");
}
