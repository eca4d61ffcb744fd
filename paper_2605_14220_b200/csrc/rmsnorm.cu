// rmsnorm.cu -- NEXT-4: batch-invariant RMSNorm prologue of the lm_head.
//
// The final norm in front of the head (§3.1 P:207 "vExact additionally implements
// RMSNorm ... batch invariant"), with the Hugging Face Qwen3 semantics the paper's model uses:
//   x1  = bf16( h * (1 / sqrt(mean_k h_k^2 + eps)) )     (fp32 arithmetic)
//   out = bf16( gamma * x1 )
// One warp per row; every lane reads 16-B vectors at a fixed stride and the row's sum of squares
// is reduced in a fixed order (lane-sequential, then a fixed shuffle-down tree) that depends only
// on d -- the same bits for a row whatever batch it is in.  HBM-bound: 4 d bytes per row.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tim_internal.h"

namespace tim {

__global__ void __launch_bounds__(256) rmsnorm_kernel(RmsNormParams p) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (row >= p.n) return;
  const int nvec = p.d / 8;  // 8 bf16 per 16-B vector
  const uint4* src = reinterpret_cast<const uint4*>(p.h + row * p.ld);
  float ss = 0.f;
  for (int v = lane; v < nvec; v += 32) {
    const uint4 q = __ldg(src + v);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(b[k]);
      ss = fmaf(f.x, f.x, ss);
      ss = fmaf(f.y, f.y, ss);
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, off);
  ss = __shfl_sync(0xffffffffu, ss, 0);  // lane 0's fixed tree, one value for the whole row
  const float var = __fdiv_rn(ss, static_cast<float>(p.d));
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, p.eps)));
  uint4* dst = reinterpret_cast<uint4*>(p.out + row * p.d);
  const uint4* gam = reinterpret_cast<const uint4*>(p.gamma);
  for (int v = lane; v < nvec; v += 32) {
    const uint4 q = __ldg(src + v);
    const uint4 g = __ldg(gam + v);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
    const __nv_bfloat162* gb = reinterpret_cast<const __nv_bfloat162*>(&g);
    uint4 o;
    __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(b[k]);
      const float2 gf = __bfloat1622float2(gb[k]);
      const float2 x1 = __bfloat1622float2(__floats2bfloat162_rn(__fmul_rn(f.x, inv), __fmul_rn(f.y, inv)));
      ob[k] = __floats2bfloat162_rn(__fmul_rn(gf.x, x1.x), __fmul_rn(gf.y, x1.y));
    }
    dst[v] = o;
  }
}

cudaError_t launch_rmsnorm(const RmsNormParams& p, cudaStream_t stream) {
  const int64_t warps = p.n;
  const int blocks = static_cast<int>((warps * 32 + 255) / 256);
  rmsnorm_kernel<<<blocks, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace tim
