// Library plumbing plus the HBM-bound helper kernels of the DP-KFAC update:
//   * A6  dpk_trace_pi          -- traces, pi and the split damping shifts on device
//   * K7  dpk_pack/unpack_owner_major -- gradient [W | b] <-> flat owner-major buffer
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <string>

#include "dpk_internal.h"

namespace dpk {

namespace {
thread_local std::string g_last_error;
std::atomic<unsigned long long> g_launches{0};
}

void set_error(const std::string& msg) { g_last_error = msg; }
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void note_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
unsigned long long launch_counter() { return g_launches.load(std::memory_order_relaxed); }
void set_launch_counter(unsigned long long v) { g_launches.store(v, std::memory_order_relaxed); }

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return DPK_OK;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return DPK_ECUDA;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    // off by default: measured slower on the SPD graph (early-launched CTAs hold
    // SMs that concurrent streams' kernels could use); DPK_PDL=1 enables
    const char* e = getenv("DPK_PDL");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

int num_sms() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      cached = n;
    else
      cached = 148;
  }
  return cached;
}

namespace {

// ---------------------------------------------------------------- A6: traces and pi
constexpr int PI_MAX = 256;
struct PiBatch {
  int n;
  double root_gamma;
  dpk_pi_job j[PI_MAX];
};

__device__ double block_sum(double v) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  v = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
  if (w == 0)
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  return v;
}

// One block per layer: tr A, tr G accumulated in double (the diagonal is short:
// d fp64 adds), then pi = sqrt((trA/dA)/(trG/dG)) in double on the RAW averaged
// factors (kfac.py:128-137, 145); the shifts are rounded to fp32 once at the end.
__global__ void trace_pi_kernel(const __grid_constant__ PiBatch b) {
  const dpk_pi_job& J = b.j[blockIdx.x];
  double sa = 0.0, sg = 0.0;
  for (int i = threadIdx.x; i < J.da; i += blockDim.x) sa += J.a[static_cast<int64_t>(i) * (J.da + 1)];
  for (int i = threadIdx.x; i < J.dg; i += blockDim.x) sg += J.g[static_cast<int64_t>(i) * (J.dg + 1)];
  sa = block_sum(sa);
  sg = block_sum(sg);
  if (threadIdx.x == 0) {
    double pi = 1.0;
    if (!(sa > 0.0) || !(sg > 0.0)) {
      if (J.info) *J.info = DPK_INFO_TRACE;
    } else {
      pi = sqrt((sa / J.da) / (sg / J.dg));
    }
    const double rg = static_cast<double>(b.root_gamma);
    J.shifts[0] = static_cast<float>(pi * rg);
    J.shifts[1] = static_cast<float>(rg / pi);
    if (J.pi) *J.pi = static_cast<float>(pi);
  }
}

// ---------------------------------------------------------------- K7: pack / unpack
constexpr int SEG_MAX = 128;
struct SegBatch {
  int n;
  float scale;
  // unpack only, optional: KL-clip scale nu = min(1, sqrt(kl_clip / (lr^2 |sum_r slot_r|)))
  // from the per-rank partial <preconditioned, gradient> dots (kl_n slots, kl_stride apart)
  const float* kl_slots;
  int64_t kl_stride;
  int kl_n;
  float kl_clip, lr2;
  dpk_segment s[SEG_MAX];
};

__device__ __forceinline__ float kl_scale(const SegBatch& b) {
  if (!b.kl_slots) return 1.0f;
  double vg = 0.0;
  for (int r = 0; r < b.kl_n; ++r) vg += static_cast<double>(__ldg(b.kl_slots + r * b.kl_stride));
  vg = fabs(vg) * static_cast<double>(b.lr2);
  if (!(vg > 0.0)) return 1.0f;
  return static_cast<float>(fmin(1.0, sqrt(static_cast<double>(b.kl_clip) / vg)));
}

// grid.y = segment; grid.x strides over the segment's rows*(cols_w+has_bias) elements.
// A plain segment (no bias column, no tap permutation, dense rows, 16-byte aligned
// ends) is one contiguous run on both sides: float4 copies.  Everything else maps
// flat element e -> (row, column) with 32-bit arithmetic (segments < 2^31 elements).
template <bool PACK>
__global__ void segment_kernel(const __grid_constant__ SegBatch b, float* flat) {
  const dpk_segment& S = b.s[blockIdx.y];
  const int cols = S.cols_w + (S.bias ? 1 : 0);
  const int total = S.rows * cols;
  float* dst = flat + S.offset;
  const float sc = PACK ? b.scale : b.scale * kl_scale(b);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const bool plain = S.perm_khw == 0 && S.bias == nullptr && S.ldw == S.cols_w &&
                     ((reinterpret_cast<uintptr_t>(S.weight) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  if (plain) {
    float4* w4 = reinterpret_cast<float4*>(S.weight);
    float4* d4 = reinterpret_cast<float4*>(dst);
    const int n4 = total >> 2;
    for (int e = tid; e < n4; e += nth) {
      if (PACK) {
        const float4 v = __ldcs(w4 + e);
        __stcs(d4 + e, make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w));
      } else {
        const float4 v = __ldcs(d4 + e);
        __stcs(w4 + e, make_float4(sc * v.x, sc * v.y, sc * v.z, sc * v.w));
      }
    }
    for (int e = (n4 << 2) + tid; e < total; e += nth) {
      if (PACK)
        dst[e] = sc * S.weight[e];
      else
        S.weight[e] = sc * dst[e];
    }
    return;
  }
  const int cin = S.perm_khw > 0 ? S.cols_w / S.perm_khw : 1;
  for (int e = tid; e < total; e += nth) {
    const int r = e / cols;
    const int c = e - r * cols;
    int cw = c;
    if (S.perm_khw > 0 && c < S.cols_w) {  // flat (kh, kw, ci) <- weight (ci, kh, kw)
      const int tap = c / cin;
      cw = (c - tap * cin) * S.perm_khw + tap;
    }
    float* src = (c < S.cols_w) ? S.weight + static_cast<int64_t>(r) * S.ldw + cw : S.bias + r;
    if (PACK)
      dst[e] = sc * *src;
    else
      *src = sc * dst[e];
  }
}

template <bool PACK>
int run_segments(const dpk_segment* segs, int n, float* flat, float scale, cudaStream_t st,
                 const float* kl_slots = nullptr, int kl_n = 0, int64_t kl_stride = 0, float kl_clip = 0.f,
                 float lr2 = 0.f) {
  if (n < 0 || (n > 0 && (segs == nullptr || flat == nullptr))) {
    set_error("dpk_pack/unpack: bad arguments");
    return DPK_EARG;
  }
  thread_local SegBatch b;
  for (int first = 0; first < n; first += SEG_MAX) {
    const int cnt = std::min(SEG_MAX, n - first);
    b.n = cnt;
    b.scale = scale;
    b.kl_slots = kl_slots;
    b.kl_n = kl_n;
    b.kl_stride = kl_stride;
    b.kl_clip = kl_clip;
    b.lr2 = lr2;
    int64_t maxe = 0;
    for (int i = 0; i < cnt; ++i) {
      b.s[i] = segs[first + i];
      if (b.s[i].rows < 0 || b.s[i].cols_w < 0 || b.s[i].weight == nullptr ||
          static_cast<int64_t>(b.s[i].rows) * (b.s[i].cols_w + 1) >= (int64_t{1} << 31)) {
        set_error("dpk_pack/unpack: invalid segment");
        return DPK_EARG;
      }
      maxe = std::max<int64_t>(maxe, static_cast<int64_t>(b.s[i].rows) * (b.s[i].cols_w + (b.s[i].bias ? 1 : 0)));
    }
    const int threads = 256;
    const int gx = static_cast<int>(std::min<int64_t>((maxe + 4 * threads - 1) / (4 * threads), 592));
    if (gx == 0) continue;
    segment_kernel<PACK><<<dim3(gx, cnt), threads, 0, st>>>(b, flat);
    note_launch();
    int rc = cuda_status(cudaGetLastError(), "segment_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

// <a, b> over n floats, deterministic: every block writes its fp64 partial, the
// last block to finish (ticket) sums them in block order and stores the result.
constexpr int DOT_BLOCKS = 148;
__global__ void __launch_bounds__(256) kl_dot_kernel(const float* a, const float* b, int64_t n, float* out,
                                                     double* partials, unsigned int* ticket) {
  double acc = 0.0;
  const int64_t nth = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  for (int64_t e = tid; e < n4; e += nth) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(a) + e), y = __ldg(reinterpret_cast<const float4*>(b) + e);
    acc += static_cast<double>(x.x) * y.x + static_cast<double>(x.y) * y.y + static_cast<double>(x.z) * y.z +
           static_cast<double>(x.w) * y.w;
  }
  for (int64_t e = 4 * n4 + tid; e < n; e += nth) acc += static_cast<double>(__ldg(a + e)) * __ldg(b + e);
  acc = block_sum(acc);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = acc;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) s += static_cast<volatile double*>(partials)[i];
    *out = static_cast<float>(s);
    *ticket = 0u;  // ready for the next call
  }
}

// Peer all-gather (DPKFAC peer_gather): one launch copies every rank's owner-major
// chunk -- read in place from the other GPUs' memory over NVLink (IPC-mapped) -- into
// the local gathered buffer; blockIdx.y = source rank, 4 independent 16-byte loads in
// flight per thread.
constexpr int PEER_MAX = 8;
struct PeerSrcs {
  const float4* src[PEER_MAX];
};
__global__ void __launch_bounds__(256) peer_gather_kernel(float4* __restrict__ dst, const __grid_constant__ PeerSrcs s,
                                                          int64_t n4) {
  const float4* __restrict__ src = s.src[blockIdx.y];
  float4* __restrict__ d = dst + static_cast<int64_t>(blockIdx.y) * n4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; k + 3 * stride < n4; k += 4 * stride) {
    const float4 v0 = src[k], v1 = src[k + stride], v2 = src[k + 2 * stride], v3 = src[k + 3 * stride];
    d[k] = v0;
    d[k + stride] = v1;
    d[k + 2 * stride] = v2;
    d[k + 3 * stride] = v3;
  }
  for (; k < n4; k += stride) d[k] = src[k];
}

}  // namespace
}  // namespace dpk

extern "C" {

size_t dpk_kl_dot_workspace_bytes(void) { return dpk::DOT_BLOCKS * sizeof(double) + 256; }

int dpk_kl_dot(const float* pre, const float* grad, int64_t n, float* out, void* workspace, size_t ws_bytes,
               dpk_stream_t stream) {
  if (n < 0 || out == nullptr || (n > 0 && (pre == nullptr || grad == nullptr)) || workspace == nullptr ||
      ws_bytes < dpk_kl_dot_workspace_bytes() || (reinterpret_cast<uintptr_t>(workspace) & 7) != 0) {
    dpk::set_error("dpk_kl_dot: bad arguments (workspace: dpk_kl_dot_workspace_bytes(), zeroed once, 8-aligned)");
    return DPK_EARG;
  }
  double* partials = static_cast<double*>(workspace);
  unsigned int* ticket = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + dpk::DOT_BLOCKS * sizeof(double));
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(dpk::DOT_BLOCKS, (n + 1023) / 1024)));
  dpk::kl_dot_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(pre, grad, n, out, partials, ticket);
  dpk::note_launch();
  return dpk::cuda_status(cudaGetLastError(), "kl_dot_kernel launch");
}

int dpk_unpack_owner_major_klclip(const dpk_segment* segs, int n_segs, const float* flat, float scale,
                                  const float* kl_slots, int n_slots, int64_t slot_stride, float kl_clip, float lr,
                                  dpk_stream_t stream) {
  if (kl_slots == nullptr || n_slots < 1 || !(kl_clip > 0.0f)) {
    dpk::set_error("dpk_unpack_owner_major_klclip: need kl_slots, n_slots >= 1 and kl_clip > 0");
    return DPK_EARG;
  }
  return dpk::run_segments<false>(segs, n_segs, const_cast<float*>(flat), scale, static_cast<cudaStream_t>(stream),
                                  kl_slots, n_slots, slot_stride, kl_clip, lr * lr);
}

int dpk_ipc_export(const void* ptr, int device, void* handle, int64_t* offset) {
  if (ptr == nullptr || handle == nullptr || offset == nullptr || device < 0) {
    dpk::set_error("dpk_ipc_export: bad arguments");
    return DPK_EARG;
  }
  int rc = dpk::cuda_status(cudaSetDevice(device), "cudaSetDevice");
  if (rc) return rc;
  // the allocation holding ptr (a caching allocator's block lives inside a larger
  // cudaMalloc segment): its IPC handle plus ptr's offset from the segment base
  using AddrRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static AddrRangeFn range = nullptr;
  if (range == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range = reinterpret_cast<AddrRangeFn>(p);
  }
  if (range == nullptr) {
    dpk::set_error("dpk_ipc_export: cuMemGetAddressRange unavailable");
    return DPK_ECUDA;
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0) {
    dpk::set_error("dpk_ipc_export: cuMemGetAddressRange failed");
    return DPK_ECUDA;
  }
  cudaIpcMemHandle_t h;
  rc = dpk::cuda_status(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
  if (rc) return rc;
  std::memcpy(handle, &h, sizeof(h));
  *offset = static_cast<int64_t>(reinterpret_cast<unsigned long long>(ptr) - base);
  return DPK_OK;
}

int dpk_ipc_open(const void* handle, int device, void** base) {
  if (handle == nullptr || base == nullptr || device < 0) {
    dpk::set_error("dpk_ipc_open: bad arguments");
    return DPK_EARG;
  }
  int rc = dpk::cuda_status(cudaSetDevice(device), "cudaSetDevice");
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return dpk::cuda_status(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

int dpk_ipc_close(void* base) { return dpk::cuda_status(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle"); }

int dpk_peer_gather(float* dst, const float* const* srcs, int n_src, int64_t count, dpk_stream_t stream) {
  if (dst == nullptr || srcs == nullptr || n_src < 1 || n_src > dpk::PEER_MAX || count < 0 || count % 4 != 0 ||
      (reinterpret_cast<uintptr_t>(dst) & 15) != 0) {
    dpk::set_error("dpk_peer_gather: bad arguments (1..8 sources, count % 4 == 0, 16-byte aligned)");
    return DPK_EARG;
  }
  dpk::PeerSrcs s{};
  for (int i = 0; i < n_src; ++i) {
    if (srcs[i] == nullptr || (reinterpret_cast<uintptr_t>(srcs[i]) & 15) != 0) {
      dpk::set_error("dpk_peer_gather: null or unaligned source");
      return DPK_EARG;
    }
    s.src[i] = reinterpret_cast<const float4*>(srcs[i]);
  }
  if (count == 0) return DPK_OK;
  const int64_t n4 = count / 4;
  const int bx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(2 * dpk::num_sms() / n_src, (n4 + 1023) / 1024)));
  dpk::peer_gather_kernel<<<dim3(bx, n_src), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<float4*>(dst), s, n4);
  dpk::note_launch();
  return dpk::cuda_status(cudaGetLastError(), "peer_gather_kernel launch");
}

const char* dpk_version(void) { return "dpkfac-b200 0.1.0 (sm_100a, tcgen05 tf32/3xtf32)"; }

const char* dpk_last_error(void) { return dpk::g_last_error.c_str(); }

unsigned long long dpk_launch_count(void) { return dpk::g_launches.load(std::memory_order_relaxed); }

int dpk_trace_pi(const dpk_pi_job* jobs, int n_jobs, float gamma, dpk_stream_t stream) {
  if (n_jobs < 0 || (n_jobs > 0 && jobs == nullptr) || !(gamma >= 0.0f)) {
    dpk::set_error("dpk_trace_pi: bad arguments");
    return DPK_EARG;
  }
  thread_local dpk::PiBatch b;
  for (int first = 0; first < n_jobs; first += dpk::PI_MAX) {
    const int cnt = std::min(dpk::PI_MAX, n_jobs - first);
    b.n = cnt;
    b.root_gamma = std::sqrt(static_cast<double>(gamma));
    for (int i = 0; i < cnt; ++i) {
      b.j[i] = jobs[first + i];
      if (b.j[i].a == nullptr || b.j[i].g == nullptr || b.j[i].shifts == nullptr || b.j[i].da < 1 ||
          b.j[i].dg < 1) {
        dpk::set_error("dpk_trace_pi: invalid job");
        return DPK_EARG;
      }
    }
    dpk::trace_pi_kernel<<<cnt, 256, 0, static_cast<cudaStream_t>(stream)>>>(b);
    dpk::note_launch();
    int rc = dpk::cuda_status(cudaGetLastError(), "trace_pi_kernel launch");
    if (rc) return rc;
  }
  return DPK_OK;
}

int dpk_pack_owner_major(const dpk_segment* segs, int n_segs, float* flat, float scale, dpk_stream_t stream) {
  return dpk::run_segments<true>(segs, n_segs, flat, scale, static_cast<cudaStream_t>(stream));
}

int dpk_unpack_owner_major(const dpk_segment* segs, int n_segs, const float* flat, float scale,
                           dpk_stream_t stream) {
  return dpk::run_segments<false>(segs, n_segs, const_cast<float*>(flat), scale, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
