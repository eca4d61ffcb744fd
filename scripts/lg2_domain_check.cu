// Exhaustive check of the sampling twin's Gumbel arithmetic domain: for all 2^23 uniforms
// u = ((x >> 9) + 1/2) 2^-23 (as gumbel_chunk forms them), L = -lg2.approx(u) > 0 and lg2.approx(L) is
// finite, so no column can get a +inf / NaN score.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/c lg2_domain_check.cu
// Result on B200 (round 1): "bad count 0".
#include <cstdio>
#include <cstdint>
__device__ float lg2a(float x) { float y; asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void k(float* out) {
  // u for mantissa m = (x >> 9), over all 2^23 values
  uint32_t m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= (1u << 23)) return;
  float u = __uint_as_float(0x3f800000u | m) - 0x1.fffffep-1f;
  float L = -lg2a(u);
  float g = lg2a(L);
  if (!(L > 0.f) || !isfinite(g)) { int i = atomicAdd((int*)out, 1); if (i < 8) { out[2 + 3*i] = u; out[3 + 3*i] = L; out[4 + 3*i] = g; } }
}
int main() {
  float* d; cudaMalloc(&d, 4096); cudaMemset(d, 0, 4096);
  k<<<(1u << 23) / 256, 256>>>(d);
  float h[40]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("bad count %d\n", *(int*)h);
  for (int i = 0; i < 8 && i < *(int*)h; ++i) printf("u=%.10g (%a) L=%g g=%g\n", h[2+3*i], h[2+3*i], h[3+3*i], h[4+3*i]);
  return 0;
}
