// das.cu -- sm_100a delay-and-sum receive beamforming with the fused
// IQ-envelope / log-compression epilogue (
// S:133).
//
// One CTA = one scanline x FB frames, all depth tiles of the line.
// Warp-specialised, 9 warps:
//   warp 8 (producer): per stage, 32 lanes each bulk-copy (cp.async.bulk ->
//     SASS UBLKCP, the 1-D TMA) one (aperture entry, frame) window of int16
//     samples -- only the samples the tile's delays reference -- into a
//     4-stage shared-memory ring; completion via mbarrier tx-counts.  The
//     producer also writes a per-stage entry record {|q|^2/2, d.q, pi*cu,
//     k_enter} and the window start, so consumers do no dot products.
//   warps 0-7 (consumers): one output depth sample k per thread per 256-
//     sample tile; per aperture entry: the closed-form split delay
//     tau = k + delta, delta = |q + h d| - h (h = k/2, sample units) with one
//     MUFU.RSQ and a Newton correction (reading #30), magic-number floor,
//     Hann weight (MUFU.COS), then for every frame pair the int16 -> f32
//     magic conversion, linear interpolation and accumulation in packed
//     f32x2 (FADD2/FFMA2): geometry is amortised over the FB frames.
// Aperture entries are pre-sorted by k_enter (binary64, reading #6): the
// members of a tile are a prefix of the list, per-lane membership is one
// integer compare.  RF lines go to a 4-tile ring in shared memory; after
// each tile the consumers run the 65-tap complex FIR of the previous tile
// (symmetric form, taps in the constant bank), |.|, and either 20 log10
// against a fixed reference or env + per-frame max (frame-max reference).
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

// 4-D TMA tile load (SASS UTMALDG): box {kWin/2 sample pairs, 1 channel,
// 1 event, FB frames} at coordinates (c0, c1, c2, c3); out-of-range
// coordinates (samples < 0 or >= S, frames >= F) are zero-filled by the TMA
// unit, which is exactly the zero padding of reading #10.
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// Named barrier over the 256 consumer threads (warps 0-7) only.
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ float rsqrt_ftz(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
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
__device__ __forceinline__ float magic16(uint32_t u) { return __int_as_float((int)(u ^ 0x4B008000u)); }
constexpr float kMagic16 = 8421376.0f;  // 2^23 + 2^15
constexpr float kFloorMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kFloorMagicBits = 0x4B400000;

__host__ __device__ constexpr size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct SmemLayout {
  int16_t* stage;  // [kStages][EC][block]: FB x kWin int16 per entry
  float4* rec;     // [kStages][32] {Ah, B, pi*cu, k_enter bits}
  int* ws;         // [kStages][32]
  uint64_t* full;  // [kStages]
  uint64_t* empty; // [kStages]
  float* ring;     // [kRing][FB]  (frame fastest)
  unsigned* smax;  // [8]
};

// One staged entry block: FB frames x kWin samples, 128-byte aligned (TMA).
__host__ __device__ constexpr int block_bytes(int FB) { return (FB * kWin * 2 + 127) & ~127; }

__host__ __device__ inline size_t layout_bytes(int FB, size_t* off) {
  size_t o = 0;
  off[0] = o; o = align16(o + (size_t)kStages * (kCopiesPerStage / FB) * block_bytes(FB));
  off[1] = o; o = align16(o + sizeof(float4) * kStages * kCopiesPerStage);
  off[2] = o; o = align16(o + sizeof(int) * kStages * kCopiesPerStage);
  off[3] = o; o = align16(o + sizeof(uint64_t) * kStages);
  off[4] = o; o = align16(o + sizeof(uint64_t) * kStages);
  off[5] = o; o = align16(o + sizeof(float) * (size_t)kRing * FB);
  off[6] = o; o = align16(o + sizeof(unsigned) * 8);
  return o;
}

__device__ __forceinline__ SmemLayout carve(unsigned char* base, int FB) {
  size_t off[7];
  layout_bytes(FB, off);
  SmemLayout L;
  L.stage = (int16_t*)(base + off[0]);
  L.rec = (float4*)(base + off[1]);
  L.ws = (int*)(base + off[2]);
  L.full = (uint64_t*)(base + off[3]);
  L.empty = (uint64_t*)(base + off[4]);
  L.ring = (float*)(base + off[5]);
  L.smax = (unsigned*)(base + off[6]);
  return L;
}

// ---------------------------------------------------------------------------
// Envelope + log of one output sample k for all FB frames from the RF ring.
// b[k] = c0 x[k] + sum_{j>=1} c_j (x[k-j] + x[k+j]) + i s_j (x[k-j] - x[k+j])
// (reading #18; symmetric h), env = 2|b|.
template <int FB>
__device__ __forceinline__ void fir_output(const DasArgs& a, const float* ring, int k, int line, int f0,
                                           float* bmax) {
  const int P = (a.fir_taps - 1) / 2;
  const int p0 = k & (kRing - 1);
  float env[FB];
  if constexpr (FB == 1) {
    float re = a.fir_c[0] * ring[p0], im = 0.f;
#pragma unroll
    for (int j = 1; j <= kMaxHalfTaps; j++) {
      if (j > P) break;
      const float xm = ring[(k - j) & (kRing - 1)];
      const float xp = ring[(k + j) & (kRing - 1)];
      re = fmaf(a.fir_c[j], xm + xp, re);
      im = fmaf(a.fir_s[j], xm - xp, im);
    }
    env[0] = 2.f * sqrtf(fmaf(re, re, im * im));
  } else {
    constexpr int NP = FB / 2;
    float2 re[NP], im[NP];
    const float2* r2 = reinterpret_cast<const float2*>(ring);
#pragma unroll
    for (int q = 0; q < NP; q++) {
      re[q] = __fmul2_rn(make_float2(a.fir_c[0], a.fir_c[0]), r2[p0 * NP + q]);
      im[q] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int j = 1; j <= kMaxHalfTaps; j++) {
      if (j > P) break;
      const int pm = (k - j) & (kRing - 1), pp = (k + j) & (kRing - 1);
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const float2 xm = r2[pm * NP + q], xp = r2[pp * NP + q];
        re[q] = __ffma2_rn(make_float2(a.fir_c[j], a.fir_c[j]), __fadd2_rn(xm, xp), re[q]);
        im[q] = __ffma2_rn(make_float2(a.fir_s[j], a.fir_s[j]), sub2(xm, xp), im[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < NP; q++) {
      const float2 e2 = __ffma2_rn(re[q], re[q], __fmul2_rn(im[q], im[q]));
      env[2 * q] = 2.f * sqrtf(e2.x);
      env[2 * q + 1] = 2.f * sqrtf(e2.y);
    }
  }
  if (k >= a.S) return;
#pragma unroll
  for (int b = 0; b < FB; b++) {
    const int f = f0 + b;
    if (f >= a.F) break;
    const size_t o = ((size_t)f * a.L + line) * a.S + k;
    if (a.ref_fixed) {
      const float e = env[b];
      const float y = e > 0.f ? fminf(fmaxf(fmaf(a.log_k1, log2f(e), a.log_k0), 0.f), 1.f) : 0.f;
      if (a.y_type == SUPRA_T_U8) ((uint8_t*)a.y_out)[o] = (uint8_t)floorf(255.f * y + 0.5f);
      else ((float*)a.y_out)[o] = y;
    } else {
      a.env_out[o] = env[b];
      bmax[b] = fmaxf(bmax[b], env[b]);
    }
  }
}

}  // namespace

template <int FB, bool T0>
__global__ void __launch_bounds__(288, 2) das_fused_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const DasArgs a) {
  constexpr int EC = kCopiesPerStage / FB;  // aperture entries per stage
  constexpr int BLK = block_bytes(FB) / 2;  // int16 elements per entry block
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int S = a.S;
  SmemLayout sm = carve(smem_raw, FB);
  const int line = blockIdx.x;
  const int f0 = blockIdx.y * FB;
  const int g = a.line_group[line];
  const DasEntry* __restrict__ ents = a.entries + (size_t)g * a.entries_per_group;
  const int* __restrict__ ntile = a.ntile + (size_t)g * a.ntiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; i++) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 8) sm.smax[threadIdx.x] = 0u;
  // ring slot 3 holds "tile -1": zeros for the FIR's left edge (k < 0)
  for (int i = threadIdx.x; i < kTileK * FB; i += blockDim.x) sm.ring[3 * kTileK * FB + i] = 0.f;
  __syncthreads();

  if (warp == 8) {
    // ------------------------------ producer ------------------------------
    // lane jl < EC owns entry c*EC + jl of each stage: it computes the
    // window, writes the entry record and issues one 4-D TMA covering the
    // window for all FB frames.
    const int ev = a.line_event[line];
    const float4 dir = a.line_dir[line];
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    int s = 0;
    for (int t = 0; t < a.ntiles; t++) {
      const int nt = ntile[t];
      const int nch = (nt + EC - 1) / EC;
      const int k0 = t * kTileK, k1 = min(k0 + kTileK, S) - 1;
      for (int c = 0; c < nch; c++, s++) {
        const int buf = s % kStages;
        if (s >= kStages) mbar_wait(&sm.empty[buf], ((s / kStages) - 1) & 1);
        const int j = c * EC + lane;
        const bool valid = lane < EC && j < nt;
        int ws = 0, kenter = 0x7fffffff;
        if (lane < EC) {
          const DasEntry e = ents[j];
          const float B = fmaf(dir.z, e.qz, fmaf(dir.y, e.qy, dir.x * e.qx));
          const float Ah = 0.5f * e.A;
          if (valid) {
            kenter = e.kenter;
            const int kb = max(k0, e.kenter);
            const float hb = 0.5f * (float)kb;
            const float tb = (float)kb + split_delay(Ah, B, hb, kb > 0 ? hb * hb : 1e-20f) + a.t0fs;
            // window [ws, ws + kWin): ws <= floor(tau(kb)) - 2, 8-aligned; the
            // end floor(tau(k1)) + 3 <= ws + kWin because d tau / dk <= 1.
            ws = ((int)floorf(tb) - 2) & ~7;
          }
          sm.rec[buf * kCopiesPerStage + lane] = make_float4(Ah, B, 3.14159265358979f * e.cu,
                                                             __int_as_float(kenter));
          sm.ws[buf * kCopiesPerStage + lane] = ws;
        }
        const unsigned nvalid = __popc(__ballot_sync(0xffffffffu, valid));
        if (lane == 0) mbar_arrive_tx(&sm.full[buf], nvalid * (unsigned)(FB * kWin * 2));
        __syncwarp();
        if (valid) {
          int16_t* dst = sm.stage + ((size_t)buf * EC + lane) * BLK;
          tma_load_4d(dst, &tmap, ws >> 1, ents[j].elem, ev, f0, &sm.full[buf]);
        }
      }
    }
  } else {
    // ------------------------------ consumers -----------------------------
    const int kt = warp * 32 + lane;
    float bmax[FB];
#pragma unroll
    for (int b = 0; b < FB; b++) bmax[b] = 0.f;
    int s = 0;
    for (int t = 0; t < a.ntiles; t++) {
      const int k = t * kTileK + kt;
      const bool kval = k < S;
      const float kf = (float)k, h = 0.5f * kf;
      const float h2 = k > 0 ? h * h : 1e-20f;   // r2 > 0 even at k = 0, q = 0
      const float inv_k = k > 0 ? 1.0f / kf : 0.f;
      const int kmw = k - kFloorMagicBits;
      float acc1 = 0.f;
      float2 acc2[FB / 2 > 0 ? FB / 2 : 1];
#pragma unroll
      for (int q = 0; q < FB / 2; q++) acc2[q] = make_float2(0.f, 0.f);
      int cnt = 0;
      const int nt = ntile[t];
      const int nch = (nt + EC - 1) / EC;
      for (int c = 0; c < nch; c++, s++) {
        const int buf = s % kStages;
        mbar_wait(&sm.full[buf], (s / kStages) & 1);
        const float4* rec = sm.rec + buf * kCopiesPerStage;
        const int* wsb = sm.ws + buf * kCopiesPerStage;
        const unsigned short* st = (const unsigned short*)(sm.stage + (size_t)buf * EC * BLK);
#pragma unroll
        for (int jl = 0; jl < EC; jl++) {
          const float4 r = rec[jl];
          const int ws = wsb[jl];
          const bool mem = kval && (k >= __float_as_int(r.w));
          float delta = split_delay(r.x, r.y, h, h2);
          if (T0) delta += a.t0fs;
          const float tf = __fadd_rd(delta, kFloorMagic);
          int idx = __float_as_int(tf) + kmw - ws;
          const float fr = delta - (tf - kFloorMagic);
          idx = mem ? idx : 0;
          float w = fmaf(__cosf(r.z * inv_k), a.win_b, a.win_a);
          w = mem ? w : 0.f;
          const float wf = w * fr;
          cnt += mem ? 1 : 0;
          const unsigned short* px = st + jl * BLK + idx;
          if constexpr (FB == 1) {
            const float m0 = magic16(px[0]), m1 = magic16(px[1]);
            acc1 = fmaf(w, m0 - kMagic16, acc1);
            acc1 = fmaf(wf, m1 - m0, acc1);
          } else {
#pragma unroll
            for (int q = 0; q < FB / 2; q++) {
              const float2 m0 = make_float2(magic16(px[(2 * q) * kWin]), magic16(px[(2 * q + 1) * kWin]));
              const float2 m1 =
                  make_float2(magic16(px[(2 * q) * kWin + 1]), magic16(px[(2 * q + 1) * kWin + 1]));
              acc2[q] = __ffma2_rn(make_float2(w, w), __fadd2_rn(m0, make_float2(-kMagic16, -kMagic16)),
                                   acc2[q]);
              acc2[q] = __ffma2_rn(make_float2(wf, wf), sub2(m1, m0), acc2[q]);
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[buf]);
      }
      // ---- tile done: RF = sum / N  (reading #7; 0 when N = 0) ----
      const float inv = (a.normalize == SUPRA_NORM_NONE) ? 1.f : (cnt > 0 ? 1.f / (float)cnt : 0.f);
      float v[FB];
      if constexpr (FB == 1) {
        v[0] = kval ? acc1 * inv : 0.f;
      } else {
#pragma unroll
        for (int q = 0; q < FB / 2; q++) {
          v[2 * q] = kval ? acc2[q].x * inv : 0.f;
          v[2 * q + 1] = kval ? acc2[q].y * inv : 0.f;
        }
      }
      if (a.rf && kval) {
#pragma unroll
        for (int b = 0; b < FB; b++)
          if (f0 + b < a.F) a.rf[((size_t)(f0 + b) * a.L + line) * S + k] = v[b];
      }
      if (a.do_epilogue) {
        float* slot = sm.ring + (size_t)(k & (kRing - 1)) * FB;
#pragma unroll
        for (int b = 0; b < FB; b++) slot[b] = v[b];
        consumer_sync();
        if (t >= 1) fir_output<FB>(a, sm.ring, k - kTileK, line, f0, bmax);
      }
    }
    if (a.do_epilogue) {
      // zero the slot after the last tile (the FIR's right edge, k >= S)
      const int kz = a.ntiles * kTileK + kt;
      float* slot = sm.ring + (size_t)(kz & (kRing - 1)) * FB;
#pragma unroll
      for (int b = 0; b < FB; b++) slot[b] = 0.f;
      consumer_sync();
      fir_output<FB>(a, sm.ring, (a.ntiles - 1) * kTileK + kt, line, f0, bmax);
      if (!a.ref_fixed) {
#pragma unroll
        for (int b = 0; b < FB; b++) {
          float m = bmax[b];
          for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
          if (lane == 0) atomicMax(&sm.smax[b], __float_as_uint(m));
        }
        consumer_sync();
        if (kt < FB && f0 + kt < a.F) atomicMax(&a.frame_max[f0 + kt], sm.smax[kt]);
      }
    }
  }
}

size_t das_smem_bytes(int FB, int, int) {
  size_t off[7];
  return layout_bytes(FB, off);
}

int das_max_frames_per_cta(int, int, int F) {
  for (int fb = 8; fb > 1; fb >>= 1)
    if (fb <= F) return fb;
  return 1;
}

template <int FB, bool T0>
static cudaError_t launch_fb(const CUtensorMap& tm, const DasArgs& a, cudaStream_t st) {
  const size_t smem = das_smem_bytes(FB, a.S, a.fir_taps);
  cudaError_t e = cudaFuncSetAttribute(das_fused_kernel<FB, T0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(a.L, (a.F + FB - 1) / FB);
  das_fused_kernel<FB, T0><<<grid, 288, smem, st>>>(tm, a);
  return cudaGetLastError();
}

template <bool T0>
static cudaError_t launch_t0(const CUtensorMap& tm, const DasArgs& a, int fb, cudaStream_t st) {
  switch (fb) {
    case 8: return launch_fb<8, T0>(tm, a, st);
    case 4: return launch_fb<4, T0>(tm, a, st);
    case 2: return launch_fb<2, T0>(tm, a, st);
    default: return launch_fb<1, T0>(tm, a, st);
  }
}

int das_frames_per_cta(int fb, int F) {
  while (fb > 1 && fb > F) fb >>= 1;
  return fb;
}

cudaError_t launch_das(const CUtensorMap& tm, const DasArgs& a, int fb, cudaStream_t st) {
  return a.t0fs != 0.f ? launch_t0<true>(tm, a, fb, st) : launch_t0<false>(tm, a, fb, st);
}

}  // namespace supra
