// epilogue.cuh -- IQ envelope + log compression over RF lines resident in
// shared memory.
#pragma once
#include "internal.h"

namespace supra {

// ---------------------------------------------------------------------------
// Epilogue over FB RF lines resident in shared memory (rf[b][P + k]).
// env[k] = 2 |sum_j g_j RF[k - j]|, g_j = h_j e^{+i w j} (reading #18).
template <int FB>
__device__ __forceinline__ void fused_epilogue(const float* rfs, const float2* fir, int T, int S, int L,
                                               int line, int f0, int F, int ref_fixed, float k1,
                                               float k0, float* env_out, void* y_out, int y_type,
                                               unsigned* frame_max, unsigned* smax) {
  const int P = (T - 1) / 2;
  const int stride = S + 2 * P;
  float bmax[FB];
#pragma unroll
  for (int b = 0; b < FB; b++) bmax[b] = 0.f;
  for (int i = threadIdx.x; i < FB * S; i += blockDim.x) {
    const int b = i / S, k = i - b * S;
    const int f = f0 + b;
    if (f >= F) continue;
    const float* x = rfs + b * stride + P + k;  // x[-j] = RF[k - j]
    float re = 0.f, im = 0.f;
#pragma unroll 5
    for (int j = 0; j < T; j++) {
      float v = x[P - j];
      float2 g = fir[j];
      re = fmaf(g.x, v, re);
      im = fmaf(g.y, v, im);
    }
    const float env = 2.f * sqrtf(re * re + im * im);
    const size_t o = ((size_t)f * L + line) * S + k;
    if (ref_fixed) {
      float y = env > 0.f ? fminf(fmaxf(fmaf(k1, log2f(env), k0), 0.f), 1.f) : 0.f;
      if (y_type == SUPRA_T_U8) ((uint8_t*)y_out)[o] = (uint8_t)floorf(255.f * y + 0.5f);
      else ((float*)y_out)[o] = y;
    } else {
      env_out[o] = env;
#pragma unroll
      for (int bb = 0; bb < FB; bb++)
        if (bb == b) bmax[bb] = fmaxf(bmax[bb], env);
    }
  }
  if (!ref_fixed) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int b = 0; b < FB; b++) {
      float m = bmax[b];
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) atomicMax(&smax[b], __float_as_uint(m));
    }
    __syncthreads();
    if (threadIdx.x < FB && f0 + (int)threadIdx.x < F)
      atomicMax(&frame_max[f0 + threadIdx.x], smax[threadIdx.x]);
  }
}

}  // namespace supra
