// epilogue.cu -- standalone IQ envelope + log compression on an RF buffer
// (supra_bf_envelope_log) and the frame-max finalisation shared with the
// fused path.
#include <algorithm>

#include "epilogue.cuh"

namespace supra {

// One CTA per (line, frame): the RF line is staged in shared memory with
// zeroed FIR halos; each thread produces env (or y) for strided samples.
__global__ void __launch_bounds__(256) envlog_kernel(const EnvArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = a.S, P = (a.fir_taps - 1) / 2;
  float* cs = (float*)smem_raw;                  // per band: c[0..P], s[0..P]
  float* rfs = cs + a.nbands * kCsRow;
  __shared__ unsigned smax;
  const int line = blockIdx.x, f = blockIdx.y;
  const float* src = a.rf + ((size_t)f * a.L + line) * S;
  for (int i = threadIdx.x; i < a.nbands * (P + 1); i += blockDim.x) {
    const int b = i / (P + 1), j = i - b * (P + 1);
    cs[b * kCsRow + j] = a.fir[b * a.fir_taps + j + P].x;
    cs[b * kCsRow + kMaxHalfTaps + 1 + j] = a.fir[b * a.fir_taps + j + P].y;
  }
  for (int i = threadIdx.x; i < S + 2 * P; i += blockDim.x) {
    int k = i - P;
    rfs[i] = (k >= 0 && k < S) ? src[k] : 0.f;
  }
  if (threadIdx.x == 0) smax = 0u;
  __syncthreads();
  float m = 0.f;
  for (int q = threadIdx.x; q < a.Sd; q += blockDim.x) {  // decimation keeps k = dec q
    const int k = q * a.dec;
    const float env = compound_at(rfs + P + k, cs, a.band_w, a.nbands, P);
    const size_t o = ((size_t)f * a.L + line) * a.Sd + q;
    if (a.ref_fixed) {
      const float y = env > 0.f ? fminf(fmaxf(fmaf(a.log_k1, lg2_approx(env), a.log_k0), 0.f), 1.f) : 0.f;
      if (a.y_type == SUPRA_T_U8) ((uint8_t*)a.y_out)[o] = (uint8_t)floorf(255.f * y + 0.5f);
      else ((float*)a.y_out)[o] = y;
    } else {
      a.env_out[o] = env;
      m = fmaxf(m, env);
    }
  }
  if (!a.ref_fixed) {
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(&smax, __float_as_uint(m));
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&a.frame_max[f], smax);
  }
}

// y = 1 + (20 log10 2 / DR) (log2 env - log2 ref), clamped to [0,1]; env = 0
// or an all-zero frame -> 0.  Grid-stride, 4 samples/thread.
// Element e0 of the converted set lives at f * frame_stride + offset + (e0 - f * per)
// in both env and y (a contiguous line range of each frame).
__global__ void __launch_bounds__(256) finalize_kernel(const FinalizeArgs a) {
  const long long per = a.per_frame;
  const long long total = per * a.F;
  const long long n4 = total >> 2;
  const bool vec = ((per | a.frame_stride | a.offset) & 3) == 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < (vec ? n4 : total); i += stride) {
    const long long e0 = vec ? i * 4 : i;
    const int f = (int)(e0 / per);
    const long long ad = e0 + (long long)f * (a.frame_stride - per) + a.offset;
    const float ref = a.frame_max ? __uint_as_float(a.frame_max[f]) : a.fixed_ref;
    const float lref = ref > 0.f ? lg2_approx(ref) : 0.f;
    float v[4];
    int n = vec ? 4 : 1;
    if (vec) {
      float4 x = *reinterpret_cast<const float4*>(a.env + ad);
      v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
    } else {
      v[0] = a.env[ad];
    }
    float y[4];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      if (j < n) {
        float e = v[j];
        y[j] = (e > 0.f && ref > 0.f) ? fminf(fmaxf(fmaf(a.DR_k, lg2_approx(e) - lref, 1.f), 0.f), 1.f) : 0.f;
      }
    }
    if (a.y_type == SUPRA_T_U8) {
      uint8_t* o = (uint8_t*)a.y_out;
      if (vec) {
        uchar4 q;
        q.x = (uint8_t)floorf(255.f * y[0] + 0.5f);
        q.y = (uint8_t)floorf(255.f * y[1] + 0.5f);
        q.z = (uint8_t)floorf(255.f * y[2] + 0.5f);
        q.w = (uint8_t)floorf(255.f * y[3] + 0.5f);
        *reinterpret_cast<uchar4*>(o + ad) = q;
      } else {
        o[ad] = (uint8_t)floorf(255.f * y[0] + 0.5f);
      }
    } else {
      float* o = (float*)a.y_out;
      if (vec) *reinterpret_cast<float4*>(o + ad) = make_float4(y[0], y[1], y[2], y[3]);
      else o[ad] = y[0];
    }
  }
}

cudaError_t launch_envlog(const EnvArgs& a, cudaStream_t st) {
  const int P = (a.fir_taps - 1) / 2;
  size_t smem = sizeof(float) * (a.nbands * kCsRow + a.S + 2 * P);
  cudaError_t e = cudaFuncSetAttribute(envlog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.L, a.F);
  envlog_kernel<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st) {
  long long total = a.per_frame * a.F;
  long long work = ((a.per_frame | a.frame_stride | a.offset) & 3) == 0 ? total / 4 : total;
  int blocks = (int)std::min<long long>((work + 255) / 256, 148LL * 16);
  if (blocks < 1) blocks = 1;
  finalize_kernel<<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace supra
