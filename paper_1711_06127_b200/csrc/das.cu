// das.cu -- sm_100a delay-and-sum receive beamforming with the fused
// IQ-envelope / log-compression epilogue (
// S:133).
//
// One CTA = one scanline x FB frames.  The loop runs over the line's receive
// aperture entries (channels, pre-sorted by aperture entry depth k_enter in
// binary64, reading #6); every consumer thread keeps the RF of its NT output
// samples k = kt + 256 m for all FB frames in registers.  Warp-specialised:
//   warp 8 (producer): per entry ONE 5-D TMA (cp.async.bulk.tensor -> SASS
//     UTMALDG) fetches the entry's whole referenced trace [ws, S) for the FB
//     frames into a 3-stage shared-memory ring -- each referenced sample is
//     read from HBM once, the start is 32-sample aligned, samples < 0 or
//     >= S come back as zeros (the TMA out-of-bounds fill = the zero
//     padding of reading #10).  It also publishes the entry record
//     {|q|^2/2, d.q, pi cu, k_enter} so consumers do no dot products.
//   warps 0-7 (consumers): per entry and output tile, the closed-form split
//     delay tau = k + delta, delta = |q + h d| - h (h = k/2 in sample units)
//     with one MUFU.RSQ + Newton correction (reading #30), magic-number
//     floor, Hann weight (MUFU.COS), then for each frame pair the int16->f32
//     magic conversion, linear interpolation and accumulation in packed
//     f32x2 (FADD2/FFMA2): geometry is amortised over the FB frames.
// After the last entry RF = sum / N (N from a binary64-derived count table)
// is written to shared memory (reusing the trace ring) in a padded,
// bank-conflict-free layout and the epilogue runs the 65-tap complex FIR as
// a sliding window (4 outputs x 4 frames per thread, taps in the constant
// bank), |.|, then 20 log10 against a fixed reference, or env + per-frame
// max for the frame-max reference (finalised by finalize_kernel).
#include "internal.h"

namespace supra {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// try_wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes (or ~the hint elapses) instead of spinning on issue slots.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(1000000u)
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

// Named barrier over the 256 consumer threads (warps 0-7) only.
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

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

// int16 -> float via the 2^23 + 2^15 magic: bits (u ^ 0x4B008000) of the
// zero-extended 16-bit value u are the float 2^23 + 2^15 + v.
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
constexpr int kHalo = 64;                   // FIR halo (>= kMaxHalfTaps), each side

__host__ __device__ constexpr size_t align128(size_t x) { return (x + 127) & ~size_t(127); }

// Trace stage: FB frames x rows x 32 samples (int16), 128-byte aligned.
__host__ __device__ inline size_t stage_bytes(int FB, int rows) {
  return align128((size_t)FB * rows * kRowSamples * 2);
}
// FIR line buffer: ngroups x padded(S + 2 halo + 4) float4 (4 frames), with
// a 16-byte pad after every 4 samples (conflict-free sliding LDS.128).
__host__ __device__ inline int fir_pad(int kp) { return kp + (kp >> 2); }
__host__ __device__ inline int fir_span(int S) { return fir_pad(S + 2 * kHalo + 4); }
__host__ __device__ inline size_t fir_bytes(int FB, int S) {
  return align128((size_t)((FB + 3) / 4) * fir_span(S) * 16);
}

// Stages in the trace ring: as many as fit a ~100 KB budget (2 CTAs/SM), 3..8.
__host__ __device__ inline int das_stages(int FB, int S) {
  const int n = (int)((100 * 1024) / stage_bytes(FB, das_rows(S)));
  return n < 3 ? 3 : (n > kMaxStages ? kMaxStages : n);
}

struct SmemLayout {
  int16_t* stage;   // [NS][stage_bytes]
  float4* rec;      // [nent] {|q|^2/2, d.q, pi*cu, k_enter bits}
  int2* wse;        // [nent] {window start ws, channel}
  uint64_t* full;   // [NS]
  unsigned* rel;    // [NS] warps done with the slot (last one refills it)
  unsigned* smax;   // [8]
  float4* line;     // FIR buffer, aliases the stage ring after the DAS loop
};

__host__ __device__ inline size_t layout_bytes(int FB, int S, int nent_max, size_t* off) {
  const int rows = das_rows(S);
  const size_t ring = (size_t)das_stages(FB, S) * stage_bytes(FB, rows);
  const size_t fb = fir_bytes(FB, S);
  size_t o = 0;
  off[0] = o; o = align128(o + (ring > fb ? ring : fb));
  off[1] = o; o = align128(o + sizeof(float4) * nent_max);
  off[2] = o; o = align128(o + sizeof(int2) * nent_max);
  off[3] = o; o = align128(o + sizeof(uint64_t) * kMaxStages);
  off[4] = o; o = align128(o + sizeof(unsigned) * kMaxStages);
  off[5] = o; o = align128(o + sizeof(unsigned) * 8);
  return o;
}

__device__ __forceinline__ SmemLayout carve(unsigned char* base, int FB, int S, int nent_max) {
  size_t off[6];
  layout_bytes(FB, S, nent_max, off);
  SmemLayout L;
  L.stage = (int16_t*)(base + off[0]);
  L.line = (float4*)(base + off[0]);
  L.rec = (float4*)(base + off[1]);
  L.wse = (int2*)(base + off[2]);
  L.full = (uint64_t*)(base + off[3]);
  L.rel = (unsigned*)(base + off[4]);
  L.smax = (unsigned*)(base + off[5]);
  return L;
}

// ---------------------------------------------------------------------------
// Epilogue: envelope of 4 consecutive outputs k0..k0+3 for the 4 frames of
// one frame group (sliding window over the padded line buffer; x(k) = 0
// outside [0, S)), then log compression or env + running max.
// b[k] = c0 x[k] + sum_{j>=1} c_j (x[k-j] + x[k+j]) + i s_j (x[k-j] - x[k+j])
// (reading #18: g_j = h_j e^{+i w j}, h symmetric), env = 2 |b|.
template <int FB>
__device__ __forceinline__ void fir_block(const DasArgs& a, const float4* lineg, int k0, int line, int fg0,
                                          float* bmax) {
  const int P = (a.fir_taps - 1) / 2;
  auto X = [&](int k) { return lineg[fir_pad(k + kHalo)]; };
  float4 Lw[4], Rw[4];
#pragma unroll
  for (int o = 0; o < 4; o++) Lw[o] = Rw[o] = X(k0 + o);
  float2 re[4][2], im[4][2];
  const float c0 = a.fir_c[0];
#pragma unroll
  for (int o = 0; o < 4; o++) {
    re[o][0] = __fmul2_rn(make_float2(c0, c0), make_float2(Lw[o].x, Lw[o].y));
    re[o][1] = __fmul2_rn(make_float2(c0, c0), make_float2(Lw[o].z, Lw[o].w));
    im[o][0] = im[o][1] = make_float2(0.f, 0.f);
  }
#pragma unroll
  for (int j = 1; j <= kMaxHalfTaps; j++) {
    if (j > P) break;
    // shift: Lw[o] = x[k0 + o - j], Rw[o] = x[k0 + o + j]
    Lw[3] = Lw[2]; Lw[2] = Lw[1]; Lw[1] = Lw[0]; Lw[0] = X(k0 - j);
    Rw[0] = Rw[1]; Rw[1] = Rw[2]; Rw[2] = Rw[3]; Rw[3] = X(k0 + 3 + j);
    const float2 cj = make_float2(a.fir_c[j], a.fir_c[j]), sj = make_float2(a.fir_s[j], a.fir_s[j]);
#pragma unroll
    for (int o = 0; o < 4; o++) {
      const float2 l0 = make_float2(Lw[o].x, Lw[o].y), l1 = make_float2(Lw[o].z, Lw[o].w);
      const float2 r0 = make_float2(Rw[o].x, Rw[o].y), r1 = make_float2(Rw[o].z, Rw[o].w);
      re[o][0] = __ffma2_rn(cj, __fadd2_rn(l0, r0), re[o][0]);
      re[o][1] = __ffma2_rn(cj, __fadd2_rn(l1, r1), re[o][1]);
      im[o][0] = __ffma2_rn(sj, sub2(l0, r0), im[o][0]);
      im[o][1] = __ffma2_rn(sj, sub2(l1, r1), im[o][1]);
    }
  }
#pragma unroll
  for (int o = 0; o < 4; o++) {
    const int k = k0 + o;
    if (k >= a.S) break;
    const float2 e0 = __ffma2_rn(re[o][0], re[o][0], __fmul2_rn(im[o][0], im[o][0]));
    const float2 e1 = __ffma2_rn(re[o][1], re[o][1], __fmul2_rn(im[o][1], im[o][1]));
    const float env[4] = {2.f * sqrtf(e0.x), 2.f * sqrtf(e0.y), 2.f * sqrtf(e1.x), 2.f * sqrtf(e1.y)};
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int f = fg0 + q;
      if (q >= FB || f >= a.F) break;
      const size_t out = ((size_t)f * a.L + line) * a.S + k;
      if (a.ref_fixed) {
        const float e = env[q];
        const float y = e > 0.f ? fminf(fmaxf(fmaf(a.log_k1, lg2_approx(e), a.log_k0), 0.f), 1.f) : 0.f;
        if (a.y_type == SUPRA_T_U8) ((uint8_t*)a.y_out)[out] = (uint8_t)floorf(255.f * y + 0.5f);
        else ((float*)a.y_out)[out] = y;
      } else {
        a.env_out[out] = env[q];
        bmax[q] = fmaxf(bmax[q], env[q]);
      }
    }
  }
}

}  // namespace

// Accumulators of one thread: NT output samples x FB frames.
template <int FB, int NT>
struct Acc {
  float s[FB == 1 ? NT : 1];
  float2 p[FB >= 2 ? NT : 1][FB >= 2 ? FB / 2 : 1];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int m = 0; m < NT; m++) {
      if constexpr (FB == 1) {
        s[m] = 0.f;
      } else {
#pragma unroll
        for (int q = 0; q < FB / 2; q++) p[m][q] = make_float2(0.f, 0.f);
      }
    }
  }
};

// Specialisation granularity of the first active tile (code size).
__host__ __device__ constexpr int tile_gran(int NT) { return NT <= 8 ? 1 : 2; }

// One aperture entry, output tiles M0 .. NT-1 (straight-line).
template <int FB, int NT, int M0, bool T0>
__device__ __forceinline__ void entry_tiles(const DasArgs& a, const float4& r, int kenter, int wsm,
                                            const unsigned short* st, int kt, float ktf, int S,
                                            Acc<FB, NT>& acc) {
  constexpr int FR = (NT * 8 + 2) * kRowSamples;
#pragma unroll
  for (int m = M0; m < NT; m++) {
    const int k = m * kTileK + kt;
    // k_enter < (M0 + gran) * 256, so only the first gran tiles can hold
    // non-members.  Outputs k >= S (when S < 256 NT) are computed but never
    // stored, and their taps stay inside the staged window.
    const bool first = m < M0 + tile_gran(NT);
    const bool mem = !first || k >= kenter;
    const float kf = ktf + (float)(m * kTileK);
    const float h = 0.5f * kf;
    const float h2 = (m == 0 && kt == 0) ? 1e-20f : h * h;  // r2 > 0 even at k = 0, q = 0
    float delta = split_delay(r.x, r.y, h, h2);
    if (T0) delta += a.t0fs;
    const float tf = __fadd_rd(delta, kFloorMagic);
    int idx = __float_as_int(tf) - wsm + m * kTileK;  // i0 - ws  (wsm = ws + magic - kt)
    const float fr = delta - (tf - kFloorMagic);
    idx = mem ? idx : 0;
    // opaque copy: keeps one materialised index so the 2 FB loads below use
    // immediate offsets instead of one address add each
    asm("mov.b32 %0, %0;" : "+r"(idx));
    float w = fmaf(__cosf(r.z * rcp_ftz(fmaxf(kf, 1.f))), a.win_b, a.win_a);
    w = mem ? w : 0.f;
    // linear interpolation as two weights: w (1-f) x[i0] + w f x[i0+1]
    const float w1 = w * fr, w0 = w - w1;
    const uint32_t pa = smem_u32(st) + 2u * (uint32_t)idx;
    if constexpr (FB == 1) {
      acc.s[m] = fmaf(w0, lds_s16f(pa, 0), acc.s[m]);
      acc.s[m] = fmaf(w1, lds_s16f(pa, 2), acc.s[m]);
    } else {
#pragma unroll
      for (int q = 0; q < FB / 2; q++) {
        // sign-extending 16-bit loads + int->float (I2FP), packed over a frame pair
        const float2 x0 = make_float2(lds_s16f(pa, 2 * (2 * q) * FR), lds_s16f(pa, 2 * (2 * q + 1) * FR));
        const float2 x1 = make_float2(lds_s16f(pa, 2 * (2 * q) * FR + 2), lds_s16f(pa, 2 * (2 * q + 1) * FR + 2));
        acc.p[m][q] = __ffma2_rn(make_float2(w0, w0), x0, acc.p[m][q]);
        acc.p[m][q] = __ffma2_rn(make_float2(w1, w1), x1, acc.p[m][q]);
      }
    }
  }
}

template <int FB, int NT, bool T0, int G = 0>
__device__ __forceinline__ void dispatch_tiles(int g, const DasArgs& a, const float4& r, int kenter, int wsm,
                                               const unsigned short* st, int kt, float ktf, int S,
                                               Acc<FB, NT>& acc) {
  constexpr int M0 = G * tile_gran(NT);
  if constexpr (M0 < NT) {
    if (g == G) entry_tiles<FB, NT, M0, T0>(a, r, kenter, wsm, st, kt, ktf, S, acc);
    else dispatch_tiles<FB, NT, T0, G + 1>(g, a, r, kenter, wsm, st, kt, ktf, S, acc);
  }
}

template <int FB, int NT, bool T0>
__global__ void __launch_bounds__(256, 2) das_fused_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const DasArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = a.S;
  constexpr int FR = (NT * 8 + 2) * kRowSamples;  // int16 elements per frame in a stage
  const size_t SB = stage_bytes(FB, NT * 8 + 2);
  SmemLayout sm = carve(smem_raw, FB, S, a.entries_per_group);
  const int line = a.line0 + blockIdx.x;
  const int f0 = blockIdx.y * FB;
  const int g = a.line_group[line];
  const DasEntry* __restrict__ ents = a.entries + (size_t)g * a.entries_per_group;
  const int nent = a.nentries[g];
  const int lane = threadIdx.x & 31;
  const int ev = a.line_event[line];

  const int NS = das_stages(FB, S);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; i++) {
      mbar_init(&sm.full[i], 1);
      sm.rel[i] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (threadIdx.x < 8) sm.smax[threadIdx.x] = 0u;
  // Entry records for this line, computed once in parallel:
  // window [ws, ws + rows*32), rows = 8 NT + 2 >= S/32 + 2,
  // ws <= floor(tau(k_enter)) - 2 and 32-aligned: d tau/dk in [0, 1] gives
  // i0(k) + 1 <= ws + S + 34 for every member k < S, inside the window;
  // reads past the record (>= S) or before it (< 0) come back as TMA zeros.
  {
    const float4 dir = a.line_dir[line];
    for (int i = threadIdx.x; i < nent; i += blockDim.x) {
      const DasEntry e = ents[i];
      const float B = fmaf(dir.z, e.qz, fmaf(dir.y, e.qy, dir.x * e.qx));
      const float Ah = 0.5f * e.A;
      const int kb = e.kenter;
      const float hb = 0.5f * (float)kb;
      const float tb = (float)kb + split_delay(Ah, B, hb, kb > 0 ? hb * hb : 1e-20f) + a.t0fs;
      const int ws = ((int)floorf(tb) - 2) & ~(kRowSamples - 1);
      sm.rec[i] = make_float4(Ah, B, 3.14159265358979f * e.cu, __int_as_float(kb));
      sm.wse[i] = make_int2(ws, e.elem);
    }
  }
  __syncthreads();

  // Producer step: TMA of entry jj's trace (all FB frames) into slot buf.
  auto produce = [&](int jj, int buf) {
    const int2 we = sm.wse[jj];
    mbar_arrive_tx(&sm.full[buf], (unsigned)(FB * FR * 2));
    tma_load_5d((unsigned char*)sm.stage + buf * SB, &tmap, 0, we.x / kRowSamples, we.y, ev, f0, &sm.full[buf]);
  };
  if (threadIdx.x == 0 && a.debug_skip != 2)
    for (int jj = 0; jj < NS && jj < nent; jj++) produce(jj, jj);

  {
    // ------------------------------ consumers -----------------------------
    const int kt = threadIdx.x;
    const float ktf = (float)kt;
    Acc<FB, NT> acc;
    acc.zero();
    int buf = 0;
    unsigned phase = 0;
    for (int j = 0; j < nent; j++) {
      if (a.debug_skip != 2) mbar_wait(&sm.full[buf], phase);
      const float4 r = sm.rec[j];
      const int kenter = __float_as_int(r.w);
      const int wsm = sm.wse[j].x + kFloorMagicBits - kt;
      const unsigned short* st = (const unsigned short*)((const unsigned char*)sm.stage + buf * SB);
      // straight-line code for the tiles at or after the entry's first
      // active tile (no per-tile branches: the chains of consecutive tiles
      // interleave)
      if (a.debug_skip != 1)
        dispatch_tiles<FB, NT, T0>(min(kenter / kTileK, NT - 1) / tile_gran(NT), a, r, kenter, wsm, st, kt, ktf, S,
                                   acc);
      // release the slot; the last warp to release it refills it (no warp
      // ever waits for another to issue a copy)
      __syncwarp();
      if (lane == 0) {
        const unsigned prev = atom_add_acqrel(&sm.rel[buf], 1u);
        if (prev == (blockDim.x / 32) - 1) {
          sm.rel[buf] = 0u;
          if (j + NS < nent && a.debug_skip != 2) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            produce(j + NS, buf);
          }
        }
      }
      if (++buf == NS) {
        buf = 0;
        phase ^= 1u;
      }
    }
    // ---- RF = sum / N (reading #7; 0 when N = 0) ----
    const uint16_t* ncount = a.ncount + (size_t)g * S;
    __syncthreads();  // every warp is done with the trace ring (aliased below)
    const int span = fir_span(S);
#pragma unroll
    for (int m = 0; m < NT; m++) {
      if (m * kTileK >= S) break;
      const int k = m * kTileK + kt;
      if (k >= S) break;
      const int n = (int)ncount[k];
      const float inv = (a.normalize == SUPRA_NORM_NONE) ? 1.f : (n > 0 ? 1.f / (float)n : 0.f);
      float v[FB];
      if constexpr (FB == 1) {
        v[0] = acc.s[m] * inv;
      } else {
#pragma unroll
        for (int q = 0; q < FB / 2; q++) {
          v[2 * q] = acc.p[m][q].x * inv;
          v[2 * q + 1] = acc.p[m][q].y * inv;
        }
      }
      if (a.rf) {
#pragma unroll
        for (int b = 0; b < FB; b++)
          if (f0 + b < a.F) a.rf[((size_t)(f0 + b) * a.L + line) * S + k] = v[b];
      }
      if (a.do_epilogue) {
        const int pk = fir_pad(k + kHalo);
#pragma unroll
        for (int q4 = 0; q4 < (FB + 3) / 4; q4++) {
          float4 x;
          x.x = v[4 * q4];
          x.y = (4 * q4 + 1 < FB) ? v[(4 * q4 + 1) % FB] : 0.f;
          x.z = (4 * q4 + 2 < FB) ? v[(4 * q4 + 2) % FB] : 0.f;
          x.w = (4 * q4 + 3 < FB) ? v[(4 * q4 + 3) % FB] : 0.f;
          sm.line[(size_t)q4 * span + pk] = x;
        }
      }
    }
  }
  if (!a.do_epilogue) return;
  const int ng = (FB + 3) / 4, span = fir_span(S);
  // zero halos: padded positions of k' in [0, kHalo) and [kHalo + S, S + 2 kHalo + 4)
  for (int i = threadIdx.x; i < ng * (2 * kHalo + 4); i += blockDim.x) {
    const int q4 = i / (2 * kHalo + 4), r = i - q4 * (2 * kHalo + 4);
    const int kp = r < kHalo ? r : S + r;
    sm.line[(size_t)q4 * span + fir_pad(kp)] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  // ---- epilogue: work items = (frame group, 4 consecutive outputs) ----
  const int nblk = (S + 3) / 4;
  float bmax[4] = {0.f, 0.f, 0.f, 0.f};
  int curg = -1;
  for (int it = threadIdx.x; it < ng * nblk; it += blockDim.x) {
    const int q4 = it / nblk, blk = it - q4 * nblk;
    if (q4 != curg) {
      if (curg >= 0 && !a.ref_fixed)
        for (int q = 0; q < 4 && 4 * curg + q < FB; q++) atomicMax(&sm.smax[4 * curg + q], __float_as_uint(bmax[q]));
      curg = q4;
      bmax[0] = bmax[1] = bmax[2] = bmax[3] = 0.f;
    }
    fir_block<FB>(a, sm.line + (size_t)q4 * span, 4 * blk, line, f0 + 4 * q4, bmax);
  }
  if (!a.ref_fixed) {
    if (curg >= 0)
      for (int q = 0; q < 4 && 4 * curg + q < FB; q++) atomicMax(&sm.smax[4 * curg + q], __float_as_uint(bmax[q]));
    __syncthreads();
    if (threadIdx.x < FB && f0 + (int)threadIdx.x < a.F)
      atomicMax(&a.frame_max[f0 + threadIdx.x], sm.smax[threadIdx.x]);
  }
}

size_t das_smem_bytes(int FB, int S, int nent_max) {
  size_t off[6];
  return layout_bytes(FB, S, nent_max, off);
}

// Frames per CTA: registers hold NT x FB accumulators (<= 64), the smem
// footprint must allow 2 CTAs per SM, and never more frames than the call.
int das_frames_per_cta(int fb_max, int S, int F, int nent_max) {
  const int nt = das_nt(S);
  int fb = fb_max;
  while (fb > 1 && (fb > F || fb * nt > 64 || das_smem_bytes(fb, S, nent_max) > 113 * 1024)) fb >>= 1;
  return fb;
}

template <int FB, int NT, bool T0>
static cudaError_t launch_k(const CUtensorMap& tm, const DasArgs& a, cudaStream_t st) {
  const size_t smem = das_smem_bytes(FB, a.S, a.entries_per_group);
  auto kern = das_fused_kernel<FB, NT, T0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.nlines, (a.F + FB - 1) / FB);
  kern<<<grid, 256, smem, st>>>(tm, a);
  return cudaGetLastError();
}

template <bool T0>
static cudaError_t launch_t0(const CUtensorMap& tm, const DasArgs& a, int fb, cudaStream_t st) {
  const int nt = das_nt(a.S);
  switch (fb) {
    case 8: return nt == 4 ? launch_k<8, 4, T0>(tm, a, st) : launch_k<8, 8, T0>(tm, a, st);
    case 4:
      return nt == 4 ? launch_k<4, 4, T0>(tm, a, st)
                     : (nt == 8 ? launch_k<4, 8, T0>(tm, a, st) : launch_k<4, 16, T0>(tm, a, st));
    case 2:
      return nt == 4 ? launch_k<2, 4, T0>(tm, a, st)
                     : (nt == 8 ? launch_k<2, 8, T0>(tm, a, st) : launch_k<2, 16, T0>(tm, a, st));
    default:
      return nt == 4 ? launch_k<1, 4, T0>(tm, a, st)
                     : (nt == 8 ? launch_k<1, 8, T0>(tm, a, st) : launch_k<1, 16, T0>(tm, a, st));
  }
}

cudaError_t launch_das(const CUtensorMap& tm, const DasArgs& a, int fb, cudaStream_t st) {
  return a.t0fs != 0.f ? launch_t0<true>(tm, a, fb, st) : launch_t0<false>(tm, a, fb, st);
}

}  // namespace supra
