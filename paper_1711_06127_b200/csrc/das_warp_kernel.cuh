// das_warp_kernel.cuh -- single-frame delay-and-sum (FB = 1: one volume or frame per
// call, e.g. the 3D C4 volume) with the receive aperture split across the
// warps of the CTA, and
// the same fused envelope / log epilogue as das.cu.
//
// With one frame per CTA the per-tap geometry cannot be amortised over
// frames, and in das_fused_kernel every warp pays the per-entry bookkeeping
// (ring wait, record, tile dispatch, release atomics) for only 8 output
// samples per lane.  Here each WARP owns whole aperture entries instead:
//   * CTA = one scanline; lane l of every warp holds the RF of all S = 32 NTL
//     output samples k = 32 t + l (NTL accumulators, packed f32x2 over tile
//     pairs t = 2p, 2p+1);
//   * warp w beamforms entries j = w, w + 4, ... of the line's k_enter-sorted
//     aperture list; each warp has its own ring of NSW trace stages, filled
//     by its lane 0 with one TMA per entry (the referenced window from
//     tau(k_enter) to the end of the record; samples past S are TMA zeros);
//   * per entry the warp jumps (switch fall-through) to the first tile pair
//     holding a member sample and runs the remaining pairs straight-line;
//   * the 4 partial sums are added in warp order through shared memory
//     (deterministic), divided by N(k), and the FIR/envelope/log epilogue
//     runs on the line exactly as in das_fused_kernel.
// Hann apodisation: w = sin^2(pi (1 - min(u, 1)) / 2) = 0.5 (1 + cos pi u)
// for u = rho / R <= 1 and exactly 0 beyond the aperture (u > 1), so the
// tile code needs no membership predicate (membership itself stays the
// binary64 k_enter / N(k) tables of reading #6: a boundary sample has w = 0
// either way).  Other windows use the k >= k_enter predicate.
#pragma once
// (Kernel template and launcher; instantiated per mode in das_warp_inst*.cu.)
#include "das_common.cuh"

namespace supra {

namespace {

// 4 warps per CTA, 3 CTAs per SM: 12 warps per SM with up to 168 registers
// each (64 accumulators + the tile-pair temporaries without spills).
constexpr int kWarps = 4;
constexpr int kThreads = 32 * kWarps;
constexpr int kCtasPerSm = 3;
constexpr int kMaxWarpStages = 4;
constexpr size_t kWarpSmemBudget = 75 * 1024;

struct WarpLayout {
  size_t rk, ring, bars, smax, total;
  int nsw;
};

// [rk table: 1/max(k,1) for the tile pairs, S floats -- also the guard below
//  the ring for the (zero-weight) reads of non-member lanes, i0 >= 0 >
//  ws - S] [ring: kWarps x NSW stages] [mbarriers] [frame max].
// The epilogue's partial sums [kWarps][S] f32 and the FIR line buffer alias
// the ring.
__host__ __device__ inline WarpLayout warp_layout(int S, int rows, int P) {
  WarpLayout w;
  const size_t sb = stage_bytes(1, rows);
  const size_t epi_red = align128((size_t)kWarps * S * 4);
  const size_t epi_line = align128((size_t)fir_span(S, P) * 16);
  const size_t epi = epi_red > epi_line ? epi_red : epi_line;
  const size_t fixed = align128((size_t)S * 4) + align128(8 * kWarps * kMaxWarpStages) + align128(4 * 16);
  long n = fixed >= kWarpSmemBudget ? 0 : (long)((kWarpSmemBudget - fixed) / (kWarps * sb));
  w.nsw = n < 2 ? 2 : (n > kMaxWarpStages ? kMaxWarpStages : (int)n);
  const size_t ring = (size_t)w.nsw * kWarps * sb;
  size_t o = 0;
  w.rk = o;   o = align128(o + (size_t)S * 4);
  w.ring = o; o = align128(o + (ring > epi ? ring : epi));
  w.bars = o; o = align128(o + 8 * kWarps * kMaxWarpStages);
  w.smax = o; o = align128(o + 4 * 16);
  w.total = o;
  return w;
}

// Per-entry constants of the tile code.
struct EntryCtx {
  float Ah, B, cu;  // |q|^2/2, d.q (samples), 2 F rho / dr (u = cu / k)
  int wsl;          // ws + magic bits - lane:  idx = bits(floor tf) - wsl + 32 t
  uint32_t abase;   // sbase - 2 wsl: the stage address of x[i0] is 2 bits(floor tf) + abase + 64 t
  int kenter;
  uint32_t sbase;   // shared address of the entry's stage
};

// Window start of entry e for this line (also recomputed by the consumer:
// the same code, so the same value).
__device__ __forceinline__ int entry_ws(const DasEntry& e, const float4& dir, float t0fs, float& Ah, float& B) {
  B = fmaf(dir.z, e.qz, fmaf(dir.y, e.qy, dir.x * e.qx));
  Ah = 0.5f * e.A;
  const int kb = e.kenter;
  const float hb = 0.5f * (float)kb;
  const float tb = (float)kb + split_delay(Ah, B, hb, kb > 0 ? hb * hb : 1e-20f) + t0fs;
  return ((int)floorf(tb) - 2) & ~(kRowSamples - 1);
}

// Tile pair (2p, 2p+1): output samples k = 64 p + lane and k + 32.
// FIRST: the entry's first group of tile pairs (it holds k_enter): the only
// one with non-member samples, so the only one needing the aperture clamp
// (Hann) or the k >= k_enter predicate (other windows).
template <int PP, bool HANN, int MODE, bool FIRST>
__device__ __forceinline__ void pair_tap(const DasArgs& a, const EntryCtx& c, const float2* rkt, int lane,
                                         float2 lanef, float2& acc) {
  const float2 h = __ffma2_rn(lanef, make_float2(0.5f, 0.5f), make_float2(32.0f * PP, 32.0f * PP + 16.0f));
  float2 hh = __fmul2_rn(h, h);
  if (PP == 0 && lane == 0) hh.x = 1e-20f;  // r2 > 0 even at k = 0, q = 0
  float2 delta = split_delay2(c.Ah, c.B, h, hh);
  if (MODE >= 1) delta = __fadd2_rn(delta, make_float2(a.t0fs, a.t0fs));  // t0 (+ 1/2 for nearest)
  const float2 tf = add_rm2(delta, make_float2(kFloorMagic, kFloorMagic));

  const float2 fr = sub2(delta, sub2(tf, make_float2(kFloorMagic, kFloorMagic)));
  const float2 rk = rkt[PP * 32 + lane];
  float2 u = __fmul2_rn(make_float2(c.cu, c.cu), rk);
  float2 w;
  if constexpr (HANN) {
    if constexpr (FIRST) {
      u.x = fminf(u.x, 1.0f);
      u.y = fminf(u.y, 1.0f);
    }
    const float2 v = __ffma2_rn(u, make_float2(-1.57079632679f, -1.57079632679f),
                                make_float2(1.57079632679f, 1.57079632679f));
    const float2 sn = make_float2(__sinf(v.x), __sinf(v.y));
    w = __fmul2_rn(sn, sn);
  } else {
    const int k = 64 * PP + lane;
    w = __ffma2_rn(make_float2(__cosf(3.14159265358979f * u.x), __cosf(3.14159265358979f * u.y)),
                   make_float2(a.win_b, a.win_b), make_float2(a.win_a, a.win_a));
    if constexpr (FIRST) {
      w.x = k >= c.kenter ? w.x : 0.f;
      w.y = k + 32 >= c.kenter ? w.y : 0.f;
    }
  }
  // linear interpolation v = x0 + f (x1 - x0), then acc += w v: 3 packed
  // FP32 ops per pair (the FP32 pipe, not issue, bounds this kernel)
  // one IMAD per tap for the address; the tile offset is a load immediate
  const uint32_t p0 = 2u * (uint32_t)__float_as_int(tf.x) + c.abase;
  const uint32_t p1 = 2u * (uint32_t)__float_as_int(tf.y) + c.abase;
  const float2 x0 = make_float2(lds_s16f(p0, 128 * PP), lds_s16f(p1, 128 * PP + 64));
  if constexpr (MODE == 2) {  // nearest sample x~[floor(tau + 1/2)]
    acc = __ffma2_rn(w, x0, acc);
  } else {
    const float2 x1 = make_float2(lds_s16f(p0, 128 * PP + 2), lds_s16f(p1, 128 * PP + 66));
    const float2 v = __ffma2_rn(fr, sub2(x1, x0), x0);
    acc = __ffma2_rn(w, v, acc);
  }
}

// Pairs from the group of kGroup pairs holding p0 to NP-1 (NP = NTL / 2),
// by switch fall-through: one indirect jump per entry, then straight-line
// code.  Case labels only at group boundaries, so each group of kGroup
// pairs is one basic block the compiler can interleave (a label per pair
// serialises the pairs' dependency chains); the up to kGroup - 1 extra
// leading pairs carry zero weight (k < k_enter).
constexpr int kGroup = 4;
template <int G0, int NP, bool HANN, int MODE, bool FIRST>
__device__ __forceinline__ void pair_group(const DasArgs& a, const EntryCtx& c, const float2* rkt, int lane,
                                           float2 lanef, float2* acc) {
  constexpr int q = G0 * kGroup < NP ? G0 * kGroup : 0;
  pair_tap<q + 0, HANN, MODE, FIRST>(a, c, rkt, lane, lanef, acc[q + 0]);
  pair_tap<q + 1, HANN, MODE, FIRST>(a, c, rkt, lane, lanef, acc[q + 1]);
  pair_tap<q + 2, HANN, MODE, FIRST>(a, c, rkt, lane, lanef, acc[q + 2]);
  pair_tap<q + 3, HANN, MODE, FIRST>(a, c, rkt, lane, lanef, acc[q + 3]);
}
#define SUPRA_FIRST(g)                                                                         \
  case g:                                                                                      \
    if constexpr ((g) * kGroup < NP) pair_group<(g), NP, HANN, MODE, true>(a, c, rkt, lane, lanef, acc); \
    break;
#define SUPRA_REST(g)                                                                          \
  case g:                                                                                      \
    if constexpr ((g) * kGroup < NP) pair_group<(g), NP, HANN, MODE, false>(a, c, rkt, lane, lanef, acc); \
    [[fallthrough]];
// The entry's first group (membership handled), then the remaining groups
// by fall-through (all members: no clamp / predicate).
template <int NP, bool HANN, int MODE>
__device__ __forceinline__ void entry_pairs(int p0, const DasArgs& a, const EntryCtx& c, const float2* rkt, int lane,
                                            float2 lanef, float2* acc) {
  static_assert(NP % kGroup == 0 && NP / kGroup <= 8, "pair groups");
  const int g0 = p0 / kGroup;
  switch (g0) {
    SUPRA_FIRST(0) SUPRA_FIRST(1) SUPRA_FIRST(2) SUPRA_FIRST(3) SUPRA_FIRST(4) SUPRA_FIRST(5) SUPRA_FIRST(6)
    SUPRA_FIRST(7)
    default:
      break;
  }
  switch (g0 + 1) {
    SUPRA_REST(1) SUPRA_REST(2) SUPRA_REST(3) SUPRA_REST(4) SUPRA_REST(5) SUPRA_REST(6) SUPRA_REST(7)
    default:
      break;
  }
}
#undef SUPRA_FIRST
#undef SUPRA_REST

}  // namespace

// NTL = S / 32 tiles per lane (32 or 64); the raw tensor map is das.cu's
// with box rows das_rows_nt(NTL / 8) (the whole record from a window start).
template <int NTL, bool HANN, int MODE>
__global__ void __launch_bounds__(kThreads, kCtasPerSm) das_warp_kernel(const __grid_constant__ CUtensorMap tmap,
                                                         const DasArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NP = NTL / 2;
  constexpr int S = NTL * 32;
  constexpr int ROWS = NTL + 2;  // das_rows_nt(NTL / 8)
  const int P = (a.fir_taps - 1) / 2;
  const WarpLayout Lw = warp_layout(S, ROWS, P);
  float2* rkt = (float2*)(smem_raw + Lw.rk);
  unsigned char* ring = smem_raw + Lw.ring;
  uint64_t* full = (uint64_t*)(smem_raw + Lw.bars);
  unsigned* smax = (unsigned*)(smem_raw + Lw.smax);
  const int NSW = Lw.nsw;
  const size_t SB = stage_bytes(1, ROWS);
  const int line = a.line0 + blockIdx.x;
  const int fm = blockIdx.y;
  const int f0 = a.fbase + fm;
  if (a.pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // (primary line, mirror variant) of this line (DasArgs::cta, MIR = 1):
  // the primary's group, direction and entry order, the variant's channels
  const int pline = a.cta[(size_t)line * 9], var = a.cta[(size_t)line * 9 + 5];
  const int g = a.line_group[pline];
  const DasEntry* __restrict__ ents = a.entries + (size_t)g * a.entries_per_group;
  const int32_t* __restrict__ ech = a.ech + (size_t)g * a.entries_per_group * 4;
  const int np = a.nentries[g];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ev = a.line_event[line];
  const float4 dir = a.line_dir[pline];

  // 1/max(k,1) for tile pairs: rkt[p*32 + l] = (k = 64p + l, k + 32)
  for (int i = threadIdx.x; i < S / 2; i += blockDim.x) {
    const int p = i >> 5, l = i & 31;
    rkt[i] = make_float2(rcp_ftz(fmaxf((float)(64 * p + l), 1.f)), rcp_ftz((float)(64 * p + l + 32)));
  }
  if (threadIdx.x < 16) smax[threadIdx.x] = 0u;
  if (lane == 0) {
    for (int s = 0; s < NSW; s++) mbar_init(&full[warp * kMaxWarpStages + s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (warp == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  __syncthreads();  // rk table and barriers visible

  auto produce = [&](int j, int slot) {  // lane 0
    const DasEntry e = ents[j];
    float Ah, B;
    const int ws = entry_ws(e, dir, a.t0fs, Ah, B);
    uint64_t* bar = &full[warp * kMaxWarpStages + slot];
    mbar_arrive_tx(bar, (unsigned)(ROWS * kRowSamples * 2));
    tma_load_5d(ring + (size_t)(warp * NSW + slot) * SB, &tmap, 0, ws / kRowSamples, ech[j * 4 + var], ev, fm, bar);
  };
  if (lane == 0 && SUPRA_DBG(a) != 2)
    for (int s = 0; s < NSW; s++)
      if (warp + kWarps * s < np) produce(warp + kWarps * s, s);

  float2 acc[NP];
#pragma unroll
  for (int p = 0; p < NP; p++) acc[p] = make_float2(0.f, 0.f);
  const float2 lanef = make_float2((float)lane, (float)lane);
  int slot = 0;
  unsigned phase = 0;
  for (int j = warp; j < np; j += kWarps) {
    const DasEntry e = ents[j];
    EntryCtx c;
    const int ws = entry_ws(e, dir, a.t0fs, c.Ah, c.B);
    c.cu = e.cu;
    c.kenter = e.kenter;
    c.wsl = ws + kFloorMagicBits - lane;
    c.sbase = smem_u32(ring + (size_t)(warp * NSW + slot) * SB);
    c.abase = c.sbase - 2u * (uint32_t)c.wsl;
    if (SUPRA_DBG(a) != 2) mbar_wait(&full[warp * kMaxWarpStages + slot], phase);
    // opaque per-entry copy of the lane coordinate: keeps the compiler from
    // hoisting the 2 NP per-pair (h, h^2) constants out of the entry loop
    // (they would be spilled to local memory)
    float2 lf = lanef;
    asm volatile("" : "+f"(lf.x), "+f"(lf.y));
    if (SUPRA_DBG(a) != 1) entry_pairs<NP, HANN, MODE>(e.kenter >> 6, a, c, rkt, lane, lf, acc);
    __syncwarp();
    if (lane == 0 && j + kWarps * NSW < np && SUPRA_DBG(a) != 2) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      produce(j + kWarps * NSW, slot);
    }
    if (++slot == NSW) {
      slot = 0;
      phase ^= 1u;
    }
  }
  __syncthreads();  // every warp is done with its ring

  // ---- sum the warps' partials in warp order; RF = sum / N (reading #7) ----
  float* red = (float*)ring;
#pragma unroll
  for (int p = 0; p < NP; p++) {
    red[warp * S + 64 * p + lane] = acc[p].x;
    red[warp * S + 64 * p + 32 + lane] = acc[p].y;
  }
  __syncthreads();
  const uint16_t* ncount = a.ncount + (size_t)g * a.S;
  float v[S / kThreads];
#pragma unroll
  for (int m = 0; m < S / kThreads; m++) {
    const int k = threadIdx.x + kThreads * m;
    float s = red[k];
#pragma unroll
    for (int w = 1; w < kWarps; w++) s += red[w * S + k];
    const int n = (int)ncount[k];
    const float inv = (a.normalize == SUPRA_NORM_NONE) ? 1.f : (n > 0 ? 1.f / (float)n : 0.f);
    v[m] = s * inv;
    if (a.rf) a.rf[((size_t)f0 * a.L + line) * S + k] = v[m];
  }
  if (!a.do_epilogue) {
    // a PDL secondary still retires only after the primary grid
    if (a.pdl_wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  __syncthreads();  // partials read: the ring becomes the FIR line buffer
  float4* lineb = (float4*)ring;
  const int kbase = -2 * P;
#pragma unroll
  for (int m = 0; m < S / kThreads; m++)
    lineb[fir_pad(threadIdx.x + kThreads * m - kbase)] = make_float4(v[m], 0.f, 0.f, 0.f);
  for (int i = threadIdx.x; i < 3 * P + 4; i += blockDim.x)  // zeros before 0 and past S
    lineb[fir_pad(i < 2 * P ? i : S + i)] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  float bmax[4] = {0.f, 0.f, 0.f, 0.f};
  const int2 vout[1] = {make_int2(line, f0)};
  if (P == 32)  // (4 it - kbase = 4 it + 2P: a multiple of 4)
    for (int it = threadIdx.x; it < S / 4; it += blockDim.x) fir_block<1, 32>(a, lineb, kbase, 4 * it, S, vout, bmax);
  else
    for (int it = threadIdx.x; it < S / 4; it += blockDim.x) fir_block<1>(a, lineb, kbase, 4 * it, S, vout, bmax);
  if (!a.ref_fixed) {
    atomicMax(&smax[0], __float_as_uint(bmax[0]));
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(&a.frame_max[f0], smax[0]);
  }
  if (a.pdl_wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline size_t das_warp_smem_bytes_impl(int S, int fir_taps) {
  return warp_layout(S, S / 32 + 2, (fir_taps - 1) / 2).total;
}

template <int NTL, bool HANN, int MODE>
cudaError_t launch_w(const CUtensorMap& tm, const DasArgs& a, cudaStream_t st) {
  const size_t smem = das_warp_smem_bytes_impl(NTL * 32, a.fir_taps);
  auto kern = das_warp_kernel<NTL, HANN, MODE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nlines, a.Fmap);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl_wait_end ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, tm, a);
}

}  // namespace supra
