// Store-rate microbenchmark: 4 warps x 32 coalesced 128 B row stores, under
// (a) no smem, (b) ~215 KB dynamic smem (L1 carve-out squeezed), (c) + 8 extra
// warps spinning on an mbarrier try_wait like the GEMM's idle roles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(float* out, int ld, long long* t, int spin) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t bar = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(1));
  __syncthreads();
  if (warp >= 4) {
    if (spin) {
      asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}\n" ::"r"(bar), "r"(0) : "memory");
    }
    return;
  }
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = lane * 1.0f + i;
  long long t0 = clock64();
  float* p = out + (warp * 32) * ld + lane;
#pragma unroll
  for (int rr = 0; rr < 32; ++rr) asm volatile("st.global.f32 [%0], %1;" ::"l"(p + rr * ld), "f"(v[rr]) : "memory");
  long long t1 = clock64();
  if (lane == 0) t[warp] = t1 - t0;
  asm volatile("bar.sync 1, 128;");
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
int main() {
  float* out; long long* t; long long h[4];
  cudaMalloc(&out, 1 << 26); cudaMalloc(&t, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int cfg = 0; cfg < 4; ++cfg) {
    const int smem = (cfg & 1) ? 215 * 1024 : 64;
    const int spin = cfg >= 2;
    for (int rep = 0; rep < 3; ++rep) k<<<1, 384, smem>>>(out, 4608, t, spin);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
    printf("smem %6d spin %d: cycles per warp %lld %lld %lld %lld (%s)\n", smem, spin, h[0], h[1], h[2], h[3], cudaGetErrorString(e));
  }
  return 0;
}
