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

// Band bank (frequency compounding): env = sum_b w_b env_b,
// bands in order; cs holds [band][c 0..P | s 0..P] with row kCsRow.
constexpr int kCsRow = 2 * (kMaxHalfTaps + 1);
__device__ __forceinline__ float compound_at(const float* x, const float* cs, const float* w, int nb, int P) {
  float env = w[0] * envelope_at(x, cs, cs + kMaxHalfTaps + 1, P);
  for (int b = 1; b < nb; b++) env = fmaf(w[b], envelope_at(x, cs + b * kCsRow, cs + b * kCsRow + kMaxHalfTaps + 1, P), env);
  return env;
}

}  // namespace supra
