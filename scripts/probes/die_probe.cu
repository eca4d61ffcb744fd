// Probe (not product code): where do the logprob kernel's clusters land, and which SMs share a die?
// Launch 148 CTAs as 74 clusters of 2 with ~200 KB of shared memory each (one CTA per SM, as the
// forward kernel); every CTA records %smid / %clusterid / %cluster_ctarank and the latency of
// dependent L2 loads (ld.global.cg) of one fixed 128-B line, first touch and warm.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smid() { uint32_t r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t clusterid() { uint32_t r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

__global__ void __cluster_dims__(2, 1, 1) probe(const uint64_t* __restrict__ line, uint32_t* out, int reps) {
  extern __shared__ uint8_t sm[];
  if (threadIdx.x != 0) return;
  sm[0] = 1;
  const uint32_t b = blockIdx.x;
  out[b * 8 + 0] = smid();
  out[b * 8 + 1] = clusterid();
  out[b * 8 + 2] = ctarank();
  // serialize the CTAs' timing windows roughly: each CTA spins until its turn by globaltimer would
  // be complex; instead every CTA times its own dependent chain (contention is light: 148 threads)
  uint64_t p = 0;  // the line holds zeros: a true dependent chain on the same address
  for (int i = 0; i < 4; ++i) {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(line + p));
    p += v;
  }
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    uint64_t v;
    asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(line + p));
    p += v;
  }
  long long t1 = clock64();
  out[b * 8 + 3] = static_cast<uint32_t>((t1 - t0) / reps);
  out[b * 8 + 4] = static_cast<uint32_t>(p);
}

int main() {
  uint64_t* buf;
  uint32_t* out;
  cudaMalloc(&buf, 1 << 26);
  cudaMemset(buf, 0, 1 << 26);
  cudaMalloc(&out, 148 * 8 * 4);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint32_t h[148 * 8];
  for (int li = 0; li < 4; ++li) {
    const uint64_t* line = buf + li * 4096 * 16;  // four lines 512 KB apart
    probe<<<148, 192, smem>>>(line, out, 256);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("line %d\n", li);
    for (int b = 0; b < 148; ++b) printf("cta %3d smid %3u cluster %3u rank %u lat %u\n", b, h[b * 8], h[b * 8 + 1], h[b * 8 + 2], h[b * 8 + 3]);
  }
  return 0;
}
