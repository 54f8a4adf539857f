// dev aid: throughput of int16 -> f32 conversion forms on sm_100a (per SM per clock)
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(uint32_t seed, float* out, long long* cyc) {
  uint32_t w[8];
#pragma unroll
  for (int i = 0; i < 8; i++) w[i] = seed * (threadIdx.x + 1) + i * 0x10001u;
  float acc[8] = {0};
  long long t0 = clock64();
  for (int it = 0; it < 2048; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      float a, b;
      if (MODE == 0) {  // I2F.S16 lo / .H1
        short2 s = *reinterpret_cast<short2*>(&w[i]);
        asm volatile("cvt.rn.f32.s16 %0, %1;" : "=f"(a) : "h"(s.x));
        asm volatile("cvt.rn.f32.s16 %0, %1;" : "=f"(b) : "h"(s.y));
      } else if (MODE == 1) {  // I2FP.F32.S32 of two sign-extended words
        int lo = (int)(short)(w[i] & 0xffff), hi = ((int)w[i]) >> 16;
        asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(a) : "r"(lo));
        asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(b) : "r"(hi));
      } else {  // magic: xor, 2 prmt, packed fadd
        uint32_t x = w[i] ^ 0x80008000u, l, h;
        asm volatile("prmt.b32 %0, %1, %2, 0x7610;" : "=r"(l) : "r"(x), "r"(0x4B000000u));
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(h) : "r"(x), "r"(0x4B000000u));
        asm volatile("{.reg .b64 r, k, d; mov.b64 r, {%2, %3}; mov.b64 k, {%4, %4}; add.rn.f32x2 d, r, k; mov.b64 {%0, %1}, d;}"
                     : "=f"(a), "=f"(b) : "r"(l), "r"(h), "f"(-8421376.f));
      }
      acc[i] += a * b;
      w[i] += 0x00030007u;
    }
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 148 * 4 * 1024 * 4); cudaMalloc(&c, 148 * 4 * 8);
  for (int mode = 0; mode < 3; mode++) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148 * 4, 512>>>(12345, o, c);
      if (mode == 1) k<1><<<148 * 4, 512>>>(12345, o, c);
      if (mode == 2) k<2><<<148 * 4, 512>>>(12345, o, c);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
      double conv = 148.0 * 4 * 512 * 2048 * 16;  // conversions (2 per word)
      printf("mode %d: %.3f ms, %.2f conversions/clk/SM (at 1.965 GHz), block cycles %lld\n", mode, ms,
             conv / (ms * 1e-3) / 148 / 1.965e9, hc);
    }
  }
  return 0;
}
