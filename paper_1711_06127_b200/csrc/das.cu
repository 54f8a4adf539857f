// das.cu -- sm_100a delay-and-sum receive beamforming with the fused
// IQ-envelope / log-compression epilogue (
// S:133).
//
// One CTA = one scanline x FB frames, the whole line (all depth tiles), so
// the FIR epilogue needs no halo exchange and RF never touches HBM unless
// asked for.  Warp-specialised:
//   warp 8 (producer): per stage, 32 lanes each bulk-copy (cp.async.bulk,
//     TMA 1D -> UBLKCP) one (aperture entry, frame) window of int16 samples
//     -- only the samples the tile's delays reference -- into a 4-stage
//     shared-memory ring, completion tracked by mbarrier tx-counts.
//   warps 0-7 (consumers): one output depth sample k per thread per 256-
//     sample tile; for every aperture entry the closed-form split delay
//     tau = k + delta, delta = |q + h d| - h (h = k/2, sample units), one
//     MUFU.RSQ plus a Newton correction, Hann weight, linear interpolation,
//     and the weighted sum for all FB frames (geometry amortised over FB).
// Aperture entries are pre-sorted by k_enter (binary64, reading #6), so the
// members of a tile are a prefix of the list and per-lane membership is an
// integer compare.  After the last tile the RF line sits in shared memory and
// the epilogue runs the 65-tap complex FIR, |.|, and either 20 log10 against
// a fixed reference or env + per-frame max for the frame-max reference.
#include "internal.h"
#include "epilogue.cuh"

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

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// delta = |q + h d| - h in samples, cancellation-free (reading #30):
// r0 = r2 * rsqrt(r2), delta0 = r0 - h, one Newton step on
// f(delta) = delta (delta + 2h) - num with 1/(2 r) ~ y/2 (no RCP).
__device__ __forceinline__ float split_delay(float A, float B, float kf, float h, float h2) {
  float num = fmaf(kf, B, A);             // |q|^2 + 2 h (d.q),   2h = k
  float r2 = fmaxf(h2 + num, 1e-20f);     // |q + h d|^2
  float y = rsqrtf(r2);                   // MUFU.RSQ
  float r0 = r2 * y;
  float d0 = r0 - h;
  float R = fmaf(d0, d0 + kf, -num);      // residual of delta (delta + 2h) = num
  return fmaf(-0.5f * y, R, d0);
}

// floor / fraction via the 1.5*2^23 magic (round-down add): exact for
// |x| < 2^22, stays on the FMA/ALU pipes.
__device__ __forceinline__ void split_floor(float x, int& i, float& f) {
  float t = __fadd_rd(x, 12582912.0f);
  i = __float_as_int(t) - 0x4B400000;
  f = x - (t - 12582912.0f);
}

// int16 -> float via the 2^23 + 2^15 magic: bits (u ^ 0x4B008000) for the
// zero-extended 16-bit value u are the float 2^23 + 2^15 + v.
__device__ __forceinline__ float magic16(uint32_t u) { return __int_as_float((int)(u ^ 0x4B008000u)); }
constexpr float kMagic16 = 8421376.0f;  // 2^23 + 2^15

struct SmemLayout {
  int16_t* stage;      // [kStages][32][kWin]
  int* hdr;            // [kStages][32] window start ws
  DasEntry* ent;       // [kStages][32]
  uint64_t* full;      // [kStages]
  uint64_t* empty;     // [kStages]
  float2* fir;         // [T]
  float* rf;           // [FB][S + 2P]
  unsigned* smax;      // [8]
};

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t layout_bytes(int FB, int S, int T, size_t* off) {
  const int P = (T - 1) / 2;
  size_t o = 0;
  off[0] = o; o = align16(o + sizeof(int16_t) * kStages * kCopiesPerStage * kWin);
  off[1] = o; o = align16(o + sizeof(int) * kStages * kCopiesPerStage);
  off[2] = o; o = align16(o + sizeof(DasEntry) * kStages * kCopiesPerStage);
  off[3] = o; o = align16(o + sizeof(uint64_t) * kStages);
  off[4] = o; o = align16(o + sizeof(uint64_t) * kStages);
  off[5] = o; o = align16(o + sizeof(float2) * T);
  off[6] = o; o = align16(o + sizeof(float) * (size_t)FB * (S + 2 * P));
  off[7] = o; o = align16(o + sizeof(unsigned) * 8);
  return o;
}

__device__ __forceinline__ SmemLayout carve(unsigned char* base, int FB, int S, int T) {
  size_t off[8];
  layout_bytes(FB, S, T, off);
  SmemLayout L;
  L.stage = (int16_t*)(base + off[0]);
  L.hdr = (int*)(base + off[1]);
  L.ent = (DasEntry*)(base + off[2]);
  L.full = (uint64_t*)(base + off[3]);
  L.empty = (uint64_t*)(base + off[4]);
  L.fir = (float2*)(base + off[5]);
  L.rf = (float*)(base + off[6]);
  L.smax = (unsigned*)(base + off[7]);
  return L;
}

}  // namespace

template <int FB>
__global__ void __launch_bounds__(288, (FB <= 4 ? 2 : 1)) das_fused_kernel(const DasArgs a) {
  constexpr int EC = kCopiesPerStage / FB;  // aperture entries per stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = a.S, T = a.fir_taps, P = (T - 1) / 2;
  SmemLayout sm = carve(smem_raw, FB, S, T);
  const int line = blockIdx.x;
  const int f0 = blockIdx.y * FB;
  const int g = a.line_group[line];
  const DasEntry* __restrict__ ents = a.entries + (size_t)g * a.entries_per_group;
  const int* __restrict__ ntile = a.ntile + (size_t)g * a.ntiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float4 dir = a.line_dir[line];

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; i++) {
      mbar_init(&sm.full[i], 32);
      mbar_init(&sm.empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < T; i += blockDim.x) sm.fir[i] = a.fir[i];
  if (threadIdx.x < 8) sm.smax[threadIdx.x] = 0u;
  if (a.do_epilogue) {  // zero the FIR halos of the RF lines
    const int stride = S + 2 * P;
    for (int i = threadIdx.x; i < FB * 2 * P; i += blockDim.x) {
      int b = i / (2 * P), j = i - b * 2 * P;
      sm.rf[b * stride + (j < P ? j : S + j)] = 0.f;
    }
  }
  __syncthreads();

  if (warp == 8) {
    // ------------------------------ producer ------------------------------
    const int jl = lane / FB, b = lane - jl * FB;
    const int f = f0 + b;
    const int ev = a.line_event[line];
    const int16_t* src_frame = a.raw + ((size_t)f * a.E + ev) * (size_t)a.C * S;
    int s = 0;
    for (int t = 0; t < a.ntiles; t++) {
      const int nt = ntile[t];
      const int nch = (nt + EC - 1) / EC;
      const int k0 = t * kTileK, k1 = min(k0 + kTileK, S) - 1;
      for (int c = 0; c < nch; c++, s++) {
        const int buf = s % kStages;
        if (s >= kStages) mbar_wait(&sm.empty[buf], ((s / kStages) - 1) & 1);
        const int j = c * EC + jl;
        const DasEntry e = ents[j];
        int16_t* dst = sm.stage + ((size_t)buf * kCopiesPerStage + lane) * kWin;
        int ws = 0, a0 = 0, a1 = 0;
        if (j < nt) {
          const float B = fmaf(dir.z, e.qz, fmaf(dir.y, e.qy, dir.x * e.qx));
          const int kb = max(k0, e.kenter);
          const float kbf = (float)kb, k1f = (float)k1;
          const float tb = kbf + split_delay(e.A, B, kbf, 0.5f * kbf, 0.25f * kbf * kbf) + a.t0fs;
          const float te = k1f + split_delay(e.A, B, k1f, 0.5f * k1f, 0.25f * k1f * k1f) + a.t0fs;
          ws = ((int)floorf(tb) - 2) & ~7;
          int we = ((int)floorf(te) + 4 + 7) & ~7;
          if (we - ws > kWin) we = ws + kWin;
          if (f < a.F) {
            a0 = max(ws, 0);
            a1 = min(we, S);
            bool zf = false;
            for (int i = ws; i < min(a0, we); i++) { dst[i - ws] = 0; zf = true; }
            for (int i = max(a1, ws); i < we; i++) { dst[i - ws] = 0; zf = true; }
            if (zf) fence_proxy_async();
          }
        }
        if (b == 0) {
          sm.hdr[buf * kCopiesPerStage + jl] = ws;
          sm.ent[buf * kCopiesPerStage + jl] = e;
        }
        if (a1 > a0) {
          const unsigned bytes = (unsigned)(a1 - a0) * 2u;
          mbar_arrive_tx(&sm.full[buf], bytes);
          bulk_g2s(dst + (a0 - ws), src_frame + (size_t)e.elem * S + a0, bytes, &sm.full[buf]);
        } else {
          mbar_arrive(&sm.full[buf]);
        }
      }
    }
  } else {
    // ------------------------------ consumers -----------------------------
    const int kt = warp * 32 + lane;
    int s = 0;
    const int stride = S + 2 * P;
    for (int t = 0; t < a.ntiles; t++) {
      const int k = t * kTileK + kt;
      const bool kval = k < S;
      const float kf = (float)k, h = 0.5f * kf, h2 = h * h;
      const float inv_k = k > 0 ? 1.0f / kf : 0.f;
      float acc[FB];
#pragma unroll
      for (int b = 0; b < FB; b++) acc[b] = 0.f;
      int cnt = 0;
      const int nt = ntile[t];
      const int nch = (nt + EC - 1) / EC;
      for (int c = 0; c < nch; c++, s++) {
        const int buf = s % kStages;
        mbar_wait(&sm.full[buf], (s / kStages) & 1);
        const DasEntry* se = sm.ent + buf * kCopiesPerStage;
        const int* sh = sm.hdr + buf * kCopiesPerStage;
        const int16_t* st = sm.stage + (size_t)buf * kCopiesPerStage * kWin;
#pragma unroll
        for (int jl = 0; jl < EC; jl++) {
          const DasEntry e = se[jl];
          const int ws = sh[jl];
          const bool mem = kval && (k >= e.kenter);
          const float B = fmaf(dir.z, e.qz, fmaf(dir.y, e.qy, dir.x * e.qx));
          const float delta = split_delay(e.A, B, kf, h, h2) + a.t0fs;
          int di;
          float fr;
          split_floor(delta, di, fr);
          int idx = k + di - ws;
          idx = min(max(idx, 0), kWin - 2);
          const float u = e.cu * inv_k;
          float w = fmaf(a.win_b, __cosf(3.14159265f * u), a.win_a);
          w = mem ? w : 0.f;
          cnt += mem ? 1 : 0;
          const float wf = w * fr;
          const unsigned short* px = (const unsigned short*)(st + (size_t)jl * FB * kWin + idx);
#pragma unroll
          for (int b = 0; b < FB; b++) {
            const float m0 = magic16(px[b * kWin]);
            const float m1 = magic16(px[b * kWin + 1]);
            acc[b] = fmaf(w, m0 - kMagic16, acc[b]);
            acc[b] = fmaf(wf, m1 - m0, acc[b]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[buf]);
      }
      if (kval) {
        const float inv = (a.normalize == SUPRA_NORM_NONE) ? 1.f : (cnt > 0 ? 1.f / (float)cnt : 0.f);
#pragma unroll
        for (int b = 0; b < FB; b++) {
          const float v = acc[b] * inv;
          if (a.do_epilogue) sm.rf[b * stride + P + k] = v;
          if (a.rf && f0 + b < a.F) a.rf[((size_t)(f0 + b) * a.L + line) * S + k] = v;
        }
      }
    }
  }
  if (!a.do_epilogue) return;
  __syncthreads();
  fused_epilogue<FB>(sm.rf, sm.fir, T, S, a.L, line, f0, a.F, a.ref_fixed, a.log_k1, a.log_k0,
                     a.env_out, a.y_out, a.y_type, a.frame_max, sm.smax);
}

size_t das_smem_bytes(int FB, int S, int T) {
  size_t off[8];
  return layout_bytes(FB, S, T, off);
}

int das_max_frames_per_cta(int S, int T, int F) {
  // largest FB whose footprint still allows 2 CTAs per SM (228 KB), capped by F
  for (int fb = 4; fb > 1; fb >>= 1)
    if (fb <= F && das_smem_bytes(fb, S, T) <= 112 * 1024) return fb;
  return 1;
}

template <int FB>
static cudaError_t launch_fb(const DasArgs& a, cudaStream_t st) {
  const size_t smem = das_smem_bytes(FB, a.S, a.fir_taps);
  cudaError_t e = cudaFuncSetAttribute(das_fused_kernel<FB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.L, (a.F + FB - 1) / FB);
  das_fused_kernel<FB><<<grid, 288, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_das(const DasArgs& a, int fb, size_t, cudaStream_t st) {
  while (fb > 1 && fb > a.F) fb >>= 1;
  switch (fb) {
    case 8: return launch_fb<8>(a, st);
    case 4: return launch_fb<4>(a, st);
    case 2: return launch_fb<2>(a, st);
    default: return launch_fb<1>(a, st);
  }
}

}  // namespace supra
