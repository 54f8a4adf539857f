// epilogue.cuh -- IQ envelope of one RF sample (S:195,
// S:227-229), in exactly the arithmetic order of the fused DAS epilogue
// (das.cu fir_output), so the standalone and fused paths agree bitwise.
#pragma once
#include "internal.h"

namespace supra {

// x points at RF[k] inside a zero-padded line (x[-P .. P] readable).
// b = c0 x[k] + sum_{j>=1} c_j (x[k-j] + x[k+j]) + i s_j (x[k-j] - x[k+j]);
// env = 2 |b|  (reading #18: g_j = h_j e^{+i w j}, h symmetric).
__device__ __forceinline__ float envelope_at(const float* x, const float* c, const float* s, int P) {
  float re = c[0] * x[0], im = 0.f;
  for (int j = 1; j <= P; j++) {
    const float xm = x[-j], xp = x[j];
    re = fmaf(c[j], xm + xp, re);
    im = fmaf(s[j], xm - xp, im);
  }
  return 2.f * sqrtf(fmaf(re, re, im * im));
}

}  // namespace supra
