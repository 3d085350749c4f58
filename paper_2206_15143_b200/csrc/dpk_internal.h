// Internal (C++) interfaces shared by the translation units of libdpkfac.so.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/dpkfac.h"

namespace dpk {

void set_error(const std::string& msg);
void note_launch();  // counts every kernel this library launches (dpk_launch_count)
void note_launches(unsigned long long n);  // graph replays: the kernels the graph holds
unsigned long long launch_counter();
void set_launch_counter(unsigned long long v);  // captures launch nothing: undo their counts
int cuda_status(cudaError_t e, const char* what);
int num_sms();

// Function attributes (cudaFuncSetAttribute) apply to the CURRENT device only:
// true the first time it is called for a given flag word on the current device.
// Usage: static std::atomic<uint64_t> done{0}; if (first_on_device(done)) {...}
inline bool first_on_device(std::atomic<uint64_t>& done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
  const uint64_t bit = 1ull << dev;
  return (done.fetch_or(bit, std::memory_order_relaxed) & bit) == 0;
}

// -------------------------------------------------------------- GEMM engine
enum { EPI_LINEAR = 0, EPI_EIGDIV = 1 };

struct GemmSpec {
  dpk_gemm_job job;
  int epi;              // EPI_LINEAR or EPI_EIGDIV
  const float* vrow;    // EIGDIV: per-row eigenvalues (G side)
  const float* vcol;    // EIGDIV: per-column eigenvalues (A side)
  float gamma;          // EIGDIV damping
  float* out_t;         // optional: also write out_t[n*ldt + m] = value (transposed copy)
  int64_t ldt;
  // operand structure (TRI_*): a tile's K range is clipped to the chunks where
  // both operands can be nonzero (triangular factors in the SPD recursion)
  int tri_a = 0;
  int tri_b = 0;
  // symmetric jobs only: compute and store the lower tiles, no mirror (the
  // upper triangle of the output is left as it was, or -- on diagonal tiles --
  // receives the full product)
  int lower_only = 0;
  // optional: device float bits of amax|operand| -- the operands hold X * 2^-e
  // (fp16 prescaled patches), the epilogue multiplies alpha by 2^(2e)
  const int32_t* alpha_amax = nullptr;
  // DPK_PREC_3XF16: device float bits of amax|A| and amax|B| (required); the
  // operands are split as x * 2^-e = hi + lo in fp16 and alpha gets 2^(e_a + e_b)
  const int32_t* amax_a = nullptr;
  const int32_t* amax_b = nullptr;
};

// Power-of-two prescale of fp16 patch operands (dpk_im2col_job.amax): the largest
// magnitude lands in [2^14, 2^15).  Shared by the patch writers and the SYRK epilogue.
__host__ __device__ inline int prescale_exponent(int32_t amax_bits) {
  const uint32_t u = static_cast<uint32_t>(amax_bits) & 0x7fffffffu;
  const int be = static_cast<int>(u >> 23);
  if (be == 0 || be == 255) return 0;  // zero/subnormal amax, or inf/nan: no scaling
  return (be - 127) - 14;
}
constexpr int TRI_NONE = 0;
constexpr int TRI_LOWER = 1;  // op[r][k] == 0 for k > r
constexpr int TRI_UPPER = 2;  // op[r][k] == 0 for k < r
// block diagonal: op[r][k] == 0 unless r and k lie in the same unit-tile-sized
// block (128 or 256, the engine's tile edge; zeros must be stored inside a
// 256 block) -- the rotation sets of the block-Jacobi eigensolver (syevj.cu)
constexpr int TRI_BLOCK = 3;

size_t gemm_workspace_bytes(const GemmSpec* specs, int n);
// tcgen05 launches made by this thread use at most `cap` SMs (0 = all): a
// concurrent stream keeps the rest (spd_inv.cu's right-looking trailing updates)
void set_grid_cap_override(int cap);
int grid_cap_override();
// split-K depth of the tcgen05 plans made by this thread (units per SM; 0 = default 3)
int units_per_sm();
int split_min_chunks();
int units_per_sm_override();
void set_units_per_sm_override(int u);
struct UnitsPerSm {  // scoped override
  int prev;
  explicit UnitsPerSm(int u) : prev(units_per_sm_override()) { set_units_per_sm_override(u); }
  ~UnitsPerSm() { set_units_per_sm_override(prev); }
};
// K4 Jacobi rotation thresholds (syevd.cu), shared by the on-chip and block kernels
void jac_tolerances(float& rel, float& abs_);
// K4 n > 128: block Jacobi (syevj.cu); jobs with n <= 128 are ignored
size_t syevj_workspace_bytes(const dpk_eig_job* jobs, int n_jobs);
int syevj_run(const dpk_eig_job* jobs, int n_jobs, void* workspace, size_t ws_bytes, cudaStream_t st);
// CUDA-core latency path for groups of small problems (gemm_simt.cu)
bool simt_eligible(const GemmSpec* specs, int n, int precision);
double simt_fma_limit();
int simt_gemm_launch(const GemmSpec* specs, int n, cudaStream_t st);
// zero_counters: clear the scheduler counters at the workspace start first (callers
// that issue several launches on one workspace/stream clear once; every kernel
// leaves them zero)
int gemm_launch(const GemmSpec* specs, int n, void* ws, size_t ws_bytes, int precision, cudaStream_t st,
                bool zero_counters = true);
constexpr size_t GEMM_SCHED_BYTES = 256;

inline dpk_operand rows_k(const float* p, int rows, int64_t cols, int64_t ld) {
  dpk_operand o{};
  o.data = p;
  o.kind = DPK_OPND_ROWS_K;
  o.rows = rows;
  o.cols = cols;
  o.ld = ld;
  return o;
}
inline dpk_operand rows_mn(const float* p, int rows, int64_t cols, int64_t ld) {
  dpk_operand o{};
  o.data = p;
  o.kind = DPK_OPND_ROWS_MN;
  o.rows = rows;
  o.cols = cols;
  o.ld = ld;
  return o;
}

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Small LRU keyed by raw bytes: host-side plans (tensor maps, unit layouts,
// workspace sizes) of launches that repeat every training step with the same
// buffers are built once.  Not thread-safe by itself; callers hold `mu`.
template <class V>
struct LruCache {
  struct Entry {
    std::string key;
    V value;
    unsigned long long last;
  };
  std::mutex mu;
  std::vector<Entry> entries;
  unsigned long long tick = 0;
  size_t cap = 64;
  V* find(const std::string& k) {
    for (auto& e : entries)
      if (e.key == k) {
        e.last = ++tick;
        return &e.value;
      }
    return nullptr;
  }
  V* put(const std::string& k, V v) {
    if (entries.size() >= cap) {
      size_t old = 0;
      for (size_t i = 1; i < entries.size(); ++i)
        if (entries[i].last < entries[old].last) old = i;
      entries.erase(entries.begin() + old);
    }
    entries.push_back(Entry{k, std::move(v), ++tick});
    return &entries.back().value;
  }
};
template <class T>
inline void key_put(std::string& k, const T& v) {
  k.append(reinterpret_cast<const char*>(&v), sizeof(T));
}
// every field of a GemmSpec (not its padding) -> cache key bytes
inline void key_spec(std::string& k, const GemmSpec& g) {
  key_put(k, g.job);
  key_put(k, g.epi);
  key_put(k, g.vrow);
  key_put(k, g.vcol);
  key_put(k, g.gamma);
  key_put(k, g.out_t);
  key_put(k, g.ldt);
  key_put(k, g.tri_a);
  key_put(k, g.tri_b);
  key_put(k, g.lower_only);
  key_put(k, g.alpha_amax);
  key_put(k, g.amax_a);
  key_put(k, g.amax_b);
}

// Kernel launch with optional programmatic dependent launch (DPK_PDL=1) and an
// optional cluster dimension.  Kernels launched this way must call pdl_wait()
// before touching global memory.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster_x,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cluster_x > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster_x;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace dpk
