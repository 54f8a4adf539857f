// das_common.cuh -- device helpers shared by the DAS kernels (das.cu,
// das_warp.cu): PTX wrappers (mbarrier, TMA, MUFU, packed f32x2), the split
// delay (reading #30), int16 staging loads and the fused FIR/envelope/log
// epilogue block (reading #18).  Internal; not part of the ABI.
#pragma once
#include "internal.h"

namespace supra {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// mbarrier.try_wait blocks for a hardware-defined window, then the loop
// retries.  (Measured: a suspend-time hint, or __nanosleep back-off of
// 32-500 ns between tries, is no faster -- the retries' issue slots are not
// what bounds the DAS kernels.)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// acq_rel: orders this warp's reads of the slot (after __syncwarp) before the
// count, and lets the last arriver see every other warp's release.
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v)
               : "memory");
  return old;
}

// 5-D TMA tile load: box {16 pairs, rows, 1 channel, 1 event, FB frames}.
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_ftz(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

__device__ __forceinline__ float2 add_rm2(float2 a, float2 b) {
  float2 r;
  asm("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rm.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}

// delta = |q + h d| - h (samples), cancellation-free (reading #30).  With
// hn = (|q|^2 + 2h d.q)/2:  r2 = h^2 + 2 hn,  y ~ 1/sqrt(r2) (MUFU.RSQ),
// d0 = r2 y - h, and one Newton step on delta(delta + 2h) = 2 hn:
//   delta = d0 + y (hn - d0 (d0/2 + h)).
__device__ __forceinline__ float split_delay(float Ah, float B, float h, float h2) {
  const float hn = fmaf(h, B, Ah);
  const float r2 = fmaf(hn, 2.0f, h2);
  const float y = rsqrt_ftz(r2);
  const float d0 = fmaf(r2, y, -h);
  const float s = fmaf(d0, -0.5f, -h);
  const float R = fmaf(d0, s, hn);
  return fmaf(y, R, d0);
}

// The same for two output samples at once (packed f32x2: FFMA2 per step,
// two MUFU.RSQ); per lane the operations and their order are those of
// split_delay, so the results are identical.
__device__ __forceinline__ float2 split_delay2(float Ah, float B, float2 h, float2 h2) {
  const float2 hn = __ffma2_rn(h, make_float2(B, B), make_float2(Ah, Ah));
  const float2 r2 = __ffma2_rn(hn, make_float2(2.0f, 2.0f), h2);
  const float2 y = make_float2(rsqrt_ftz(r2.x), rsqrt_ftz(r2.y));
  const float2 nh = make_float2(-h.x, -h.y);
  const float2 d0 = __ffma2_rn(r2, y, nh);
  const float2 s = __ffma2_rn(d0, make_float2(-0.5f, -0.5f), nh);
  const float2 R = __ffma2_rn(d0, s, hn);
  return __ffma2_rn(y, R, d0);
}

// int16 sample -> float: sign-extending shared load (LDS.S16) + I2FP.F32.S32
// (the full-rate conversion; the compiler's own choice is LDS.U16 + the
// quarter-rate I2F.S16).  `off` is a compile-time byte offset.
__device__ __forceinline__ float lds_s16f(uint32_t addr, int off) {
  int v;
  asm volatile("ld.shared.s16 %0, [%1];" : "=r"(v) : "r"(addr + (uint32_t)off) : "memory");
  float f;
  asm("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(v));
  return f;
}
constexpr float kFloorMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kFloorMagicBits = 0x4B400000;

__host__ __device__ constexpr size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

// Trace stage: FB frames x rows x 32 samples (int16), 128-byte aligned.
__host__ __device__ inline size_t stage_bytes(int FB, int rows) {
  return align128((size_t)FB * rows * kRowSamples * 2);
}
// FIR line buffer of one pass: RF at k in [k0 - 2P, k0 + PL + P + 4) for
// ngroups = ceil(FB/4) frame groups, float4 = 4 frames, with a 16-byte pad
// after every 4 samples (conflict-free sliding LDS.128).
__host__ __device__ inline int fir_pad(int b) { return b + (b >> 2); }
__host__ __device__ inline int fir_span(int PL, int P) { return fir_pad(PL + 3 * P + 4); }
__host__ __device__ inline int fir_groups(int FB) { return (FB + 3) / 4; }

// ---------------------------------------------------------------------------
// Epilogue: envelope of 4 consecutive outputs o0..o0+3 (< o_end) for the 4
// frames of one frame group, sliding over the pass's line buffer (buffer
// position b = k - kbase; RF outside [0, S) is zero in the buffer), then log
// compression or env + running max.
// b[k] = c0 x[k] + sum_{j>=1} c_j (x[k-j] + x[k+j]) + i s_j (x[k-j] - x[k+j])
// (reading #18: g_j = h_j e^{+i w j}, h symmetric), env = 2 |b|; with a band
// bank (frequency compounding) env = sum_b w_b env_b, bands in
// order (the arithmetic of epilogue.cuh envelope_at, so fused and standalone
// results agree bitwise).
// PC > 0: the half-length P = PC is a compile-time constant with PC % 4 == 0
// (the 65-tap default, P = 32) and o0 - kbase is a multiple of 4, so every
// buffer read is a load at a compile-time offset from one base address:
// fir_pad(b0 + d) = b0 + b0/4 + d + floor(d/4) for b0 % 4 == 0.  PC = 0: P
// at run time.  Same operations in the same order either way.
template <int B, int PC = 0>
__device__ __forceinline__ void band_env(const DasArgs& a, const float4* lineg, int kbase, int o0, int P,
                                         float (&env)[4][4]) {
  const int b0 = o0 - kbase;
  const float4* p0 = lineg + b0 + (b0 >> 2);  // X(o0 + d) = p0[d + (d >> 2)] (PC > 0)
  auto X = [&](int k) {
    if constexpr (PC > 0) {
      const int d = k - o0;
      return p0[d + (d >> 2)];
    } else {
      return lineg[fir_pad(k - kbase)];
    }
  };
  if constexpr (PC > 0) P = PC;
  float4 Lw[4], Rw[4];
#pragma unroll
  for (int o = 0; o < 4; o++) Lw[o] = Rw[o] = X(o0 + o);
  float2 re[4][2], im[4][2];
  const float c0 = a.fir_c[B][0];
#pragma unroll
  for (int o = 0; o < 4; o++) {
    re[o][0] = __fmul2_rn(make_float2(c0, c0), make_float2(Lw[o].x, Lw[o].y));
    re[o][1] = __fmul2_rn(make_float2(c0, c0), make_float2(Lw[o].z, Lw[o].w));
    im[o][0] = im[o][1] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int j = 1; j <= kMaxHalfTaps; j++) {
    if (j > P) break;
    // shift: Lw[o] = x[o0 + o - j], Rw[o] = x[o0 + o + j]
    Lw[3] = Lw[2]; Lw[2] = Lw[1]; Lw[1] = Lw[0]; Lw[0] = X(o0 - j);
    Rw[0] = Rw[1]; Rw[1] = Rw[2]; Rw[2] = Rw[3]; Rw[3] = X(o0 + 3 + j);
    const float2 cj = make_float2(a.fir_c[B][j], a.fir_c[B][j]), sj = make_float2(a.fir_s[B][j], a.fir_s[B][j]);
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const float2 l0 = make_float2(Lw[o].x, Lw[o].y), l1 = make_float2(Lw[o].z, Lw[o].w);
      const float2 r0 = make_float2(Rw[o].x, Rw[o].y), r1 = make_float2(Rw[o].z, Rw[o].w);
      re[o][0] = __ffma2_rn(cj, __fadd2_rn(l0, r0), re[o][0]);
      re[o][1] = __ffma2_rn(cj, __fadd2_rn(l1, r1), re[o][1]);
      im[o][0] = __ffma2_rn(sj, sub2(l0, r0), im[o][0]);
      im[o][1] = __ffma2_rn(sj, sub2(l1, r1), im[o][1]);
    }
    // keeps each step's two loads in place: with compile-time offsets the
    // compiler would otherwise hoist all 2P of them (and spill)
    if constexpr (PC > 0) asm volatile("" ::: "memory");
  }
  const float w = a.band_w[B];
#pragma unroll
  for (int o = 0; o < 4; o++) {
    const float2 e0 = __ffma2_rn(re[o][0], re[o][0], __fmul2_rn(im[o][0], im[o][0]));
    const float2 e1 = __ffma2_rn(re[o][1], re[o][1], __fmul2_rn(im[o][1], im[o][1]));
    const float eb[4] = {2.f * sqrtf(e0.x), 2.f * sqrtf(e0.y), 2.f * sqrtf(e1.x), 2.f * sqrtf(e1.y)};
#pragma unroll
    for (int q = 0; q < 4; q++) env[o][q] = B == 0 ? w * eb[q] : fmaf(w, eb[q], env[o][q]);
  }
}

// vout[q] = (line, frame) of the group's q-th (virtual) frame, frame < 0:
// nothing to store (past the call's frames).
// PC: compile-time half-length (see band_env), 0 = run time; the caller
// picks PC = 32 when fir_taps == 65 and (o0 - kbase) % 4 == 0.
template <int FB, int PC = 0>
__device__ __forceinline__ void fir_block(const DasArgs& a, const float4* lineg, int kbase, int o0, int o_end,
                                          const int2* vout, float* bmax) {
  const int P = (a.fir_taps - 1) / 2;
  float env[4][4];
  band_env<0, PC>(a, lineg, kbase, o0, P, env);
  if (a.nbands > 1) band_env<1, PC>(a, lineg, kbase, o0, P, env);
  if (a.nbands > 2) band_env<2, PC>(a, lineg, kbase, o0, P, env);
  if (a.nbands > 3) band_env<3, PC>(a, lineg, kbase, o0, P, env);
  static_assert(kMaxBands == 4, "band unrolling");
  if (a.vec_out && a.dec == 1 && o0 + 3 < o_end) {
    // the 4 outputs are consecutive samples of each frame's line: one
    // 16-byte (f32) or 4-byte (u8) store per frame (o0 % 4 == 0, S % 32 == 0)
#pragma unroll
    for (int q = 0; q < 4; q++) {
      if (q >= FB) break;
      const int2 lf = vout[q];
      if (lf.y < 0) continue;
      const size_t base = ((size_t)lf.y * a.L + lf.x) * a.Sd + o0;
      if (a.ref_fixed) {
        float y[4];
#pragma unroll
        for (int o = 0; o < 4; o++) {
          const float e = env[o][q];
          y[o] = e > 0.f ? fminf(fmaxf(fmaf(a.log_k1, lg2_approx(e), a.log_k0), 0.f), 1.f) : 0.f;
        }
        if (a.y_type == SUPRA_T_U8) {
          uint32_t w = 0u;
#pragma unroll
          for (int o = 0; o < 4; o++) w |= (uint32_t)(uint8_t)floorf(255.f * y[o] + 0.5f) << (8 * o);
          *reinterpret_cast<uint32_t*>((uint8_t*)a.y_out + base) = w;
        } else {
          *reinterpret_cast<float4*>((float*)a.y_out + base) = make_float4(y[0], y[1], y[2], y[3]);
        }
      } else {
        *reinterpret_cast<float4*>(a.env_out + base) = make_float4(env[0][q], env[1][q], env[2][q], env[3][q]);
        bmax[q] = fmaxf(bmax[q], fmaxf(fmaxf(env[0][q], env[1][q]), fmaxf(env[2][q], env[3][q])));
      }
    }
    return;
  }
#pragma unroll
  for (int o = 0; o < 4; o++) {
    const int k = o0 + o;
    if (k >= o_end) break;
    // decimation: only k = dec q is kept, at line-image index q
    int kq = k;
    if (a.dec > 1) {
      kq = k / a.dec;
      if (kq * a.dec != k || kq >= a.Sd) continue;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      if (q >= FB) break;
      const int2 lf = vout[q];
      if (lf.y < 0) continue;
      const size_t out = ((size_t)lf.y * a.L + lf.x) * a.Sd + kq;
      const float e = env[o][q];
      if (a.ref_fixed) {
        const float y = e > 0.f ? fminf(fmaxf(fmaf(a.log_k1, lg2_approx(e), a.log_k0), 0.f), 1.f) : 0.f;
        if (a.y_type == SUPRA_T_U8) ((uint8_t*)a.y_out)[out] = (uint8_t)floorf(255.f * y + 0.5f);
        else ((float*)a.y_out)[out] = y;
      } else {
        a.env_out[out] = e;
        bmax[q] = fmaxf(bmax[q], e);
      }
    }
  }
}

}  // namespace
}  // namespace supra
