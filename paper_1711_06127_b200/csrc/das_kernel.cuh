// das_kernel.cuh -- sm_100a delay-and-sum receive beamforming with the fused
// IQ-envelope / log-compression epilogue (
// S:133).
//
// One CTA = one scanline x FB frames (256 threads, 2 CTAs per SM).  Depth is
// processed in passes of PL = 256 NT samples; in a pass every thread keeps
// the RF of its NT output samples k = k0 + kt + 256 m for all FB frames in
// registers (FB x NT = 64 accumulators, packed f32x2).  Per pass the loop
// runs over the line's receive-aperture entries (channels sorted by
// aperture entry depth k_enter in binary64, reading #6) that are members
// somewhere in the pass:
//   * per entry ONE 5-D TMA (cp.async.bulk.tensor -> SASS UTMALDG) fetches
//     the entry's referenced trace window for the pass, for all FB frames,
//     into a shared-memory ring; samples < 0 or >= S come back as zeros
//     (the TMA out-of-bounds fill = the zero padding of reading #10).  The
//     last warp to release a ring slot refills it -- no producer warp.
//   * per entry and output tile: the closed-form split delay tau = k + delta,
//     delta = |q + h d| - h (h = k/2 in sample units) with one MUFU.RSQ +
//     Newton correction (reading #30), magic-number floor, Hann weight
//     (MUFU.COS), then per frame pair two sign-extending LDS.S16 + I2FP and
//     the interpolating accumulation in FFMA2: the geometry is amortised
//     over the FB frames.
// After a pass RF = sum / N (N from a binary64-derived count table) goes to
// a padded shared-memory line buffer (aliasing the drained ring) and the
// 65-tap complex FIR runs over the outputs whose taps are complete, as a
// sliding window (4 outputs x 4 frames per thread, taps in the constant
// bank); the last 2P RF samples carry over to the next pass.  |.|, then
// 20 log10 against a fixed reference, or env + per-frame max for the
// frame-max reference (finalised by finalize_kernel).
#pragma once
// (Kernel templates and their launcher; explicit instantiations are spread
// over das_inst*.cu so the heavy straight-line variants compile in parallel.)
#include "internal.h"

#include <cstdio>
#include <cstdlib>

#include "das_common.cuh"

namespace supra {

namespace {


__device__ __forceinline__ int sel4(int4 v, int i) { return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w)); }

struct SmemLayout {
  int16_t* stage;   // [NS][stage_bytes]
  float4* line;     // FIR line buffer, aliases the stage ring between passes
  float4* rec;      // [nent] {|q|^2/2, d.q, pi*cu, k_enter | (ws/32 + 1) << 13 | rcut << 21}
  uint2* chx;       // [nent] channels of line slots 0..3, 16 bits each
  float4* carry;    // [ngroups][2P] RF tail of the previous pass
  uint64_t* full;   // [kMaxStages]
  unsigned* rel;    // [kMaxStages] warps done with the slot (last one refills it)
  unsigned* smax;   // [16] per-frame envelope max (float bits)
  int2* vout;       // [16] (line, frame) of every virtual frame
  int2* slot;       // [4] (event, mirror variant) of every line slot
};

// Layout: the fixed-size control block (mbarriers, release counters, frame
// maxima, output slots) first, at constant offsets, then the ring (which
// doubles as the FIR line buffer), then the per-entry records.  Constant
// offsets are load immediates and cost no registers in the tap loop.
constexpr size_t kCtlFull = 0, kCtlRel = 64, kCtlSmax = 96, kCtlVout = 160, kCtlSlot = 288, kCtlBytes = 384;
static_assert(kMaxStages * 8 <= kCtlRel && kCtlRel + kMaxStages * 4 <= kCtlSmax && kCtlSmax + 16 * 4 <= kCtlVout &&
                  kCtlVout + 16 * 8 <= kCtlSlot && kCtlSlot + 4 * 8 <= kCtlBytes,
              "DAS control block layout");

// Bytes of everything except the ring; ring stages fill the rest of the
// per-CTA budget (2 CTAs per SM), between 3 and kMaxStages.
__host__ __device__ inline size_t fixed_bytes(int FB, int nent_max, int P, int MIR) {
  return kCtlBytes + align128(sizeof(float4) * nent_max) + align128(sizeof(uint2) * nent_max) +
         align128(sizeof(float4) * fir_groups(FB) * 2 * (P > 0 ? P : 1));
}
// CTAs per SM: 3 for short passes (NT = 2: <= 85 registers), else 2 (128
// registers; at 85 the 16-accumulator shapes <4,4> and <1,4,MIR=4> spill
// 640 bytes); the per-CTA shared-memory budget follows.
__host__ __device__ constexpr int das_ctas_per_sm(int VF, int NT) { return NT == 2 ? 3 : 2; }
__host__ __device__ constexpr size_t das_smem_budget(int VF, int NT) {
  return das_ctas_per_sm(VF, NT) == 3 ? 75 * 1024 : 113 * 1024;
}

__host__ __device__ inline int das_stages(int FB, int NT, int nent_max, int P, int MIR) {
  const size_t fixed = fixed_bytes(FB, nent_max, P, MIR);
  const size_t sb = stage_bytes(FB, das_rows_nt(NT));
  const size_t budget = das_smem_budget(FB, NT);
  const long n = fixed >= budget ? 0 : (long)((budget - fixed) / sb);
  return n < 3 ? 3 : (n > kMaxStages ? kMaxStages : (int)n);
}

__host__ __device__ inline size_t layout_bytes(int FB, int NT, int nent_max, int P, int MIR, size_t* off) {
  const size_t ring = (size_t)das_stages(FB, NT, nent_max, P, MIR) * stage_bytes(FB, das_rows_nt(NT));
  const size_t fb = align128((size_t)fir_groups(FB) * fir_span(NT * kTileK, P) * 16);
  size_t o = kCtlBytes;
  off[0] = o; o = align128(o + (ring > fb ? ring : fb));
  off[1] = o; o = align128(o + sizeof(float4) * nent_max);
  off[2] = o; o = align128(o + sizeof(uint2) * nent_max);
  off[3] = o; o = align128(o + sizeof(float4) * fir_groups(FB) * 2 * (P > 0 ? P : 1));
  return o;
}

__device__ __forceinline__ SmemLayout carve(unsigned char* base, int FB, int NT, int nent_max, int P, int MIR) {
  size_t off[9];
  layout_bytes(FB, NT, nent_max, P, MIR, off);
  SmemLayout L;
  L.stage = (int16_t*)(base + off[0]);
  L.line = (float4*)(base + off[0]);
  L.rec = (float4*)(base + off[1]);
  L.chx = (uint2*)(base + off[2]);
  L.carry = (float4*)(base + off[3]);
  L.full = (uint64_t*)(base + kCtlFull);
  L.rel = (unsigned*)(base + kCtlRel);
  L.smax = (unsigned*)(base + kCtlSmax);
  L.vout = (int2*)(base + kCtlVout);
  L.slot = (int2*)(base + kCtlSlot);
  return L;
}

}  // namespace

// Accumulators of one thread: NT output samples x FB frames.
// FB = 1: tiles (2i, 2i+1) packed in s2[i]; FB >= 2: frame pairs in p[m][q].
template <int FB, int NT>
struct Acc {
  float2 s2[FB == 1 ? NT / 2 : 1];
  float2 p[FB >= 2 ? NT : 1][FB >= 2 ? FB / 2 : 1];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int m = 0; m < NT; m++) {
      if constexpr (FB == 1) {
        if (m % 2 == 0) s2[m / 2] = make_float2(0.f, 0.f);
      } else {
#pragma unroll
        for (int q = 0; q < FB / 2; q++) p[m][q] = make_float2(0.f, 0.f);
      }
    }
  }
  __device__ __forceinline__ float s(int m) const { return (m & 1) ? s2[m / 2].y : s2[m / 2].x; }
};

// Per-tile tap geometry: index of x[i0] in the staged window and the two
// interpolation weights.
struct TapGeo {
  uint32_t addr;  // shared byte address of x[i0] minus the tile's 512 m (a load immediate)
  float w0, w1;
};

// Specialisation granularity of the first active tile (code size).
__host__ __device__ constexpr int tile_gran(int NT) { return NT <= 8 ? 1 : 2; }

// Accumulate one tile's tap for all FB frames (per frame pair: 4 sign-
// extending LDS.S16 + I2FP, 2 FFMA2; frames at immediate offsets).
template <int FB, int NT, int M>
__device__ __forceinline__ void tile_accumulate(const TapGeo& g, float2* accp) {
  constexpr int FR = (NT * 8 + 2) * kRowSamples;
  constexpr int MO = 2 * M * kTileK;  // the tile's offset, folded into the load immediates
  uint32_t pa = g.addr;
  // opaque copy: keeps one materialised address so the FB loads below use
  // immediate offsets instead of one address add each
  asm("mov.b32 %0, %0;" : "+r"(pa));
#pragma unroll
  for (int q = 0; q < FB / 2; q++) {
    const float2 x0 = make_float2(lds_s16f(pa, MO + 2 * (2 * q) * FR), lds_s16f(pa, MO + 2 * (2 * q + 1) * FR));
    const float2 x1 =
        make_float2(lds_s16f(pa, MO + 2 * (2 * q) * FR + 2), lds_s16f(pa, MO + 2 * (2 * q + 1) * FR + 2));
    accp[q] = __ffma2_rn(make_float2(g.w0, g.w0), x0, accp[q]);
    accp[q] = __ffma2_rn(make_float2(g.w1, g.w1), x1, accp[q]);
  }
}

// Geometry of tile m alone (scalar).  The warp's first member tile is >= M0
// and k_enter < k0 + (M0 + gran) * 256, so only the first gran tiles can
// hold non-members (their weight and index are zeroed).  Outputs k >= S are
// computed but never stored; their taps stay inside the window.
template <int NT, int M0, bool T0>
__device__ __forceinline__ TapGeo tile_geo(int m, const DasArgs& a, const float4& r, int kenter, int wsm,
                                           uint32_t sbase, int kt, int k0, float kt0f) {
  const int k = k0 + m * kTileK + kt;
  const bool mem = !(m < M0 + tile_gran(NT)) || k >= kenter;
  const float kf = __fadd_rn(kt0f, (float)(m * kTileK));
  const float h = __fmul_rn(0.5f, kf);
  // h^2 + 1e-20: r2 > 0 even at k = 0, q = 0; for k >= 1 (h^2 >= 1/4) the
  // sum rounds to h^2 exactly, and k = 0 may sit in any tile (pass shift)
  const float h2 = __fmaf_rn(h, h, 1e-20f);
  float delta = split_delay(r.x, r.y, h, h2);
  if (T0) delta = __fadd_rn(delta, a.t0fs);
  const float tf = __fadd_rd(delta, kFloorMagic);
  // &x[i0] - 512 m = sbase + 2 (i0 - ws) - 512 m = 2 bits(tf) + (sbase - 2 wsm)  (wsm = ws + magic - k0 - kt)
  const uint32_t ad = 2u * (uint32_t)__float_as_int(tf) + (sbase - 2u * (uint32_t)wsm);
  // explicit _rn intrinsics: no FMA contraction, so each lane computes
  // exactly what tile_geo2's packed operations compute (bitwise equality
  // across launch shapes, where a tile is computed alone or in a pair)
  const float fr = __fmul_rn(__fsub_rn(delta, __fsub_rn(tf, kFloorMagic)), a.fr_scale);
  float w = fmaf(__cosf(__fmul_rn(r.z, rcp_ftz(fmaxf(kf, 1.f)))), a.win_b, a.win_a);
  w = mem ? w : 0.f;
  // linear interpolation as two weights: w (1-f) x[i0] + w f x[i0+1]
  const float w1 = __fmul_rn(w, fr);
  return TapGeo{mem ? ad : sbase - 2u * (uint32_t)(m * kTileK), __fsub_rn(w, w1), w1};
}

// Geometry of tiles m, m+1 together in packed f32x2 (FFMA2 / FADD2.RM /
// FMUL2: about 40 % fewer issued instructions than two scalar tiles; the
// per-lane arithmetic is the same, so results are identical).
template <int NT, int M0, bool T0>
__device__ __forceinline__ void tile_geo2(int m, const DasArgs& a, const float4& r, int kenter, int wsm,
                                          uint32_t sbase, int kt, int k0, float kt0f, TapGeo& g0, TapGeo& g1) {
  const int ka = k0 + m * kTileK + kt;
  const bool mem0 = !(m < M0 + tile_gran(NT)) || ka >= kenter;
  const bool mem1 = !(m + 1 < M0 + tile_gran(NT)) || ka + kTileK >= kenter;
  const float2 kf = make_float2(kt0f + (float)(m * kTileK), kt0f + (float)((m + 1) * kTileK));
  const float2 h = __fmul2_rn(kf, make_float2(0.5f, 0.5f));
  const float2 h2 = __ffma2_rn(h, h, make_float2(1e-20f, 1e-20f));  // (tile_geo)
  float2 delta = split_delay2(r.x, r.y, h, h2);
  if (T0) delta = __fadd2_rn(delta, make_float2(a.t0fs, a.t0fs));
  const float2 tf = add_rm2(delta, make_float2(kFloorMagic, kFloorMagic));
  const uint32_t ab = sbase - 2u * (uint32_t)wsm;
  const uint32_t ad0 = 2u * (uint32_t)__float_as_int(tf.x) + ab, ad1 = 2u * (uint32_t)__float_as_int(tf.y) + ab;
  const float2 fr = __fmul2_rn(sub2(delta, sub2(tf, make_float2(kFloorMagic, kFloorMagic))),
                               make_float2(a.fr_scale, a.fr_scale));
  const float2 u = __fmul2_rn(make_float2(r.z, r.z),
                              make_float2(rcp_ftz(fmaxf(kf.x, 1.f)), rcp_ftz(fmaxf(kf.y, 1.f))));
  float2 w = __ffma2_rn(make_float2(__cosf(u.x), __cosf(u.y)), make_float2(a.win_b, a.win_b),
                        make_float2(a.win_a, a.win_a));
  w.x = mem0 ? w.x : 0.f;
  w.y = mem1 ? w.y : 0.f;
  const float2 w1 = __fmul2_rn(w, fr);
  const float2 w0 = sub2(w, w1);
  g0 = TapGeo{mem0 ? ad0 : sbase - 2u * (uint32_t)(m * kTileK), w0.x, w1.x};
  g1 = TapGeo{mem1 ? ad1 : sbase - 2u * (uint32_t)((m + 1) * kTileK), w0.y, w1.y};
}

// Tile pairs (M, M+1), (M+2, M+3), ... of an entry (compile-time recursion so
// the tile index is a template argument: its offset is a load immediate).
template <int FB, int NT, int M0, bool T0, int M>
__device__ __forceinline__ void tile_pairs(const DasArgs& a, const float4& r, int kenter, int wsm, uint32_t sbase,
                                           int kt, int k0, float kt0f, Acc<FB, NT>& acc) {
  if constexpr (M + 1 < NT) {
    TapGeo g0, g1;
    tile_geo2<NT, M0, T0>(M, a, r, kenter, wsm, sbase, kt, k0, kt0f, g0, g1);
    if constexpr (FB == 1) {
      constexpr int o0 = 2 * M * kTileK, o1 = 2 * (M + 1) * kTileK;
      const float2 x0 = make_float2(lds_s16f(g0.addr, o0), lds_s16f(g1.addr, o1));
      const float2 x1 = make_float2(lds_s16f(g0.addr, o0 + 2), lds_s16f(g1.addr, o1 + 2));
      acc.s2[M / 2] = __ffma2_rn(make_float2(g0.w0, g1.w0), x0, acc.s2[M / 2]);
      acc.s2[M / 2] = __ffma2_rn(make_float2(g0.w1, g1.w1), x1, acc.s2[M / 2]);
    } else {
      tile_accumulate<FB, NT, M>(g0, acc.p[M]);
      tile_accumulate<FB, NT, M + 1>(g1, acc.p[M + 1]);
    }
    tile_pairs<FB, NT, M0, T0, M + 2>(a, r, kenter, wsm, sbase, kt, k0, kt0f, acc);
  }
}

// One aperture entry, output tiles M0 .. NT-1 of the pass (straight-line):
// an odd first tile alone, then tile pairs (2i, 2i+1) in packed geometry.
// kt0f = (float)(k0 + kt): the thread's first output sample in the pass.
template <int FB, int NT, int M0, bool T0>
__device__ __forceinline__ void entry_tiles(const DasArgs& a, const float4& r, int kenter, int wsm,
                                            const unsigned short* st, int kt, int k0, float kt0f,
                                            Acc<FB, NT>& acc) {
  const uint32_t sbase = smem_u32(st);
  if constexpr (M0 & 1) {
    const TapGeo g = tile_geo<NT, M0, T0>(M0, a, r, kenter, wsm, sbase, kt, k0, kt0f);
    if constexpr (FB == 1) {
      float& s1 = acc.s2[M0 / 2].y;
      s1 = fmaf(g.w0, lds_s16f(g.addr, 2 * M0 * kTileK), s1);
      s1 = fmaf(g.w1, lds_s16f(g.addr, 2 * M0 * kTileK + 2), s1);
    } else {
      tile_accumulate<FB, NT, M0>(g, acc.p[M0]);
    }
  }
  tile_pairs<FB, NT, M0, T0, ((M0 + 1) & ~1)>(a, r, kenter, wsm, sbase, kt, k0, kt0f, acc);
}

template <int FB, int NT, bool T0, int G = 0>
__device__ __forceinline__ void dispatch_tiles(int g, const DasArgs& a, const float4& r, int kenter, int wsm,
                                               const unsigned short* st, int kt, int k0, float kt0f,
                                               Acc<FB, NT>& acc) {
  constexpr int M0 = G * tile_gran(NT);
  if constexpr (M0 < NT) {
    if (g == G) entry_tiles<FB, NT, M0, T0>(a, r, kenter, wsm, st, kt, k0, kt0f, acc);
    else dispatch_tiles<FB, NT, T0, G + 1>(g, a, r, kenter, wsm, st, kt, k0, kt0f, acc);
  }
}

// FB frames x MIR mirror lines = VF virtual frames per CTA.  Virtual frame
// v = m FB + f is frame f of the CTA's line slot m; the stage holds the
// windows [v][rows][32] (one TMA per slot, FB frames each), and the tap
// geometry computed for the primary line is applied to all VF.
template <int FB, int NT, bool T0, int MIR>
__global__ void __launch_bounds__(256, das_ctas_per_sm(FB * MIR, NT)) das_fused_kernel(const __grid_constant__ CUtensorMap tmap,
                                                          const DasArgs a,
                                                          const __grid_constant__ RawMaps rmaps) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int VF = FB * MIR;
  constexpr int PL = NT * kTileK;                 // samples per pass
  constexpr int FR = (NT * 8 + 2) * kRowSamples;  // int16 elements per frame in a stage
  const int S = a.S;
  const int P = (a.fir_taps - 1) / 2;
  const size_t SB = stage_bytes(VF, NT * 8 + 2);
  SmemLayout sm = carve(smem_raw, VF, NT, a.entries_per_group, P, MIR);
  const int32_t* cd = a.cta + (size_t)(a.cta_base + (int)blockIdx.x) * 9;
  const int pline = cd[0];          // primary line: group, direction, entry order
  const int fm = blockIdx.y * FB;   // first frame of the CTA in the tensor map
  const int f0 = a.fbase + fm;      // ... and in the call
  if (a.pdl_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int g = a.line_group[pline];
  const DasEntry* __restrict__ ents = a.entries + (size_t)g * a.entries_per_group;
  const int32_t* __restrict__ ech = a.ech + (size_t)g * a.entries_per_group * 4;
  const int nent = a.nentries[g];
  const int lane = threadIdx.x & 31;
  const float4 dir = a.line_dir[pline];
  const int NS = das_stages(VF, NT, a.entries_per_group, P, MIR);
  const int ng = fir_groups(VF);
  const int span = fir_span(PL, P);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; i++) {
      mbar_init(&sm.full[i], 1);
      sm.rel[i] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (a.row_cut && (int)threadIdx.x < S / kRowSamples)
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&rmaps.m[threadIdx.x]))
                 : "memory");
  if (threadIdx.x < 16) {
    sm.smax[threadIdx.x] = 0u;
    // output (line, frame) of virtual frame v; frame -1: none
    const int v = threadIdx.x, m = v < VF ? v / FB : 0;
    sm.vout[v] = make_int2(cd[1 + m], (v < VF && f0 + v % FB < a.F) ? f0 + v % FB : -1);
    if (v < MIR) sm.slot[v] = make_int2(a.line_event[cd[1 + v]], cd[5 + v]);
  }

  const int kt = threadIdx.x;
  const int kwarp_last = (kt | 31);
  float bmax[4] = {0.f, 0.f, 0.f, 0.f};
  int curg = -1;
  int buf = 0;           // ring slot of the next entry (continues across passes)
  unsigned phase = 0;    // its mbarrier parity
  auto flush_max = [&]() {  // per real frame (v % FB)
    if (curg >= 0 && !a.ref_fixed)
      for (int q = 0; q < 4 && 4 * curg + q < VF; q++)
        atomicMax(&sm.smax[(4 * curg + q) % FB], __float_as_uint(bmax[q]));
  };

  // Passes end at S: the first starts at kfirst = S - ceil(S / PL) PL <= 0,
  // so a record that is not a multiple of PL loses its remainder in the
  // first pass, where the tiles of negative k -- below every k_enter -- are
  // skipped by the member-tile dispatch, instead of computing the last
  // pass's tiles past S (Table 1, S = 2368: 12 -> ~9.3 tiles per line and
  // entry; C4p, S = 3648 in one 4096-sample pass: 16 -> ~15.3).  Member
  // order per output is that of the global entry sequence whatever the
  // pass boundaries, so the results do not change.
  const int kfirst = S - ((S + PL - 1) / PL) * PL;
  for (int k0 = kfirst; k0 < S; k0 += PL) {
    const int kend = min(S, k0 + PL);
    // entries with a member sample in the pass: the k_enter-sorted prefix
    // with k_enter < kend
    int np = 0;
    for (int i0 = 0; i0 < nent; i0 += blockDim.x) {
      const int i = i0 + threadIdx.x;
      np += __syncthreads_count(i < nent && ents[i].kenter < kend);
    }
    // Entry records of the pass, in device order.  The order is ONE global
    // sequence per line group -- the k_enter-sorted list taken alternately
    // from its long-trace (early k_enter) and short-trace ends, so
    // consecutive ring entries carry similar work -- filtered to the pass's
    // prefix (entries [0, np)).  Filtering keeps the relative order, so the
    // members of any output sample k are summed in the same order whatever
    // the pass boundaries (NT), frame grouping (FB) or batch size: the RF of
    // a frame is bitwise independent of the call it is beamformed in
    // (S:164).  Non-members inside a pass add an exact +0.  The i-th record
    // of the filtered sequence, with h = nent - np entries outside the pass:
    // i < h -> entry i; else t = i - h, j = h + t/2, entry j (t even) or
    // nent - 1 - j (t odd).
    // Window [ws, ws + rows*32), rows = PL/32 + 2, ws <= floor(tau(kb)) - 2
    // and 32-aligned, kb = max(k_enter, k0): d tau/dk in [0, 1] keeps
    // i0(k) + 1 inside the window for every member k of the pass; reads
    // outside the record come back as TMA zeros.
    const int hcut = nent - np;
    for (int i = threadIdx.x; i < np; i += blockDim.x) {
      int ei = i;
      if (i >= hcut) {
        const int t = i - hcut, jj = hcut + (t >> 1);
        ei = (t & 1) ? nent - 1 - jj : jj;
      }
      const DasEntry e = ents[ei];
      const float B = fmaf(dir.z, e.qz, fmaf(dir.y, e.qy, dir.x * e.qx));
      const float Ah = 0.5f * e.A;
      const int kb = max(e.kenter, k0);
      const float hb = 0.5f * (float)kb;
      const float tb = (float)kb + split_delay(Ah, B, hb, kb > 0 ? hb * hb : 1e-20f) + a.t0fs;
      const int ws = ((int)floorf(tb) - 2) & ~(kRowSamples - 1);
      // exclusive end row of the pass's referenced samples: i0 + 1 <=
      // floor(tau(kend - 1)) + 1 for every member k < kend (+1 margin)
      const int kl = kend - 1;
      const float hl = 0.5f * (float)kl;
      const float tl = (float)kl + split_delay(Ah, B, hl, kl > 0 ? hl * hl : 1e-20f) + a.t0fs;
      const int rcut = max(1, min(S / kRowSamples, ((int)floorf(tl) + 3 + kRowSamples - 1) / kRowSamples));
      // k_enter < S <= 4096 (13 bits), ws / 32 + 1 in [0, 129] and rcut in
      // [1, 128] (8 bits each)
      sm.rec[i] = make_float4(Ah, B, 3.14159265358979f * e.cu,
                              __int_as_float(e.kenter | ((ws / kRowSamples + 1) << 13) | (rcut << 21)));
      // channels of the line slots, resolved here (off the refill path:
      // a global load in produce() would sit between a slot's release and
      // its refill)
      const int4 ch4 = *reinterpret_cast<const int4*>(ech + (size_t)ei * 4);
      const int c0 = sel4(ch4, sm.slot[0].y);
      sm.chx[i] = make_uint2((unsigned)c0 | (MIR > 1 ? (unsigned)sel4(ch4, sm.slot[1].y) << 16 : 0u),
                             MIR > 2 ? (unsigned)sel4(ch4, sm.slot[2].y) | ((unsigned)sel4(ch4, sm.slot[3].y) << 16) : 0u);
    }
    __syncthreads();  // records visible; the previous pass is done with the line buffer

    // TMA of entry jj's window (all FB frames) into ring slot `buf`.
    auto produce = [&](int jj, int buf) {
      const int w = __float_as_int(sm.rec[jj].w);
      const int wsrow = ((w >> 13) & 0xFF) - 1;
      // rows at or past rcut are out of bounds in rmaps.m[rcut - 1]: zero
      // fill, no DRAM read (the box size, and so the tx count, is fixed)
      const CUtensorMap* m = a.row_cut ? &rmaps.m[((w >> 21) & 0xFF) - 1] : &tmap;
      mbar_arrive_tx(&sm.full[buf], (unsigned)(VF * FR * 2));
      const uint2 cx = sm.chx[jj];
#pragma unroll
      for (int s = 0; s < MIR; s++) {  // slot s: its event, its (mirrored) channel
        const unsigned cw = s < 2 ? cx.x : cx.y;
        tma_load_5d((unsigned char*)sm.stage + buf * SB + (size_t)s * FB * FR * 2, m, 0, wsrow,
                    (int)((s & 1) ? cw >> 16 : cw & 0xFFFFu), sm.slot[s].x, fm, &sm.full[buf]);
      }
    };
    if (threadIdx.x == 0 && SUPRA_DBG(a) != 2) {
      // the ring was last written through the generic proxy (line buffer)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int jj = 0, b = buf; jj < NS && jj < np; jj++, b = (b + 1 == NS ? 0 : b + 1)) produce(jj, b);
    }

    Acc<VF, NT> acc;
    acc.zero();
    const float kt0f = (float)(k0 + kt);
    for (int j = 0; j < np; j++) {
      if (SUPRA_DBG(a) != 2) mbar_wait(&sm.full[buf], phase);
      const float4 r = sm.rec[j];
      const int kenter = __float_as_int(r.w) & 0x1FFF;
      const int wsm = (((__float_as_int(r.w) >> 13) & 0xFF) - 1) * kRowSamples + kFloorMagicBits - k0 - kt;
      const unsigned short* st = (const unsigned short*)((const unsigned char*)sm.stage + buf * SB);
      // first tile of the pass in which this WARP has a member sample
      // (warp-uniform): straight-line code from there (the chains of
      // consecutive tiles interleave); tiles where all 32 of the warp's k
      // are < k_enter are skipped.
      int m0 = kenter - k0 - kwarp_last;
      m0 = m0 <= 0 ? 0 : (m0 + kTileK - 1) / kTileK;
      if (SUPRA_DBG(a) != 1 && m0 < NT)
        dispatch_tiles<VF, NT, T0>(m0 / tile_gran(NT), a, r, kenter, wsm, st, kt, k0, kt0f, acc);
      // release the slot; the last warp to release it refills it (no warp
      // ever waits for another to issue a copy)
      __syncwarp();
      if (lane == 0) {
        const unsigned prev = atom_add_acqrel(&sm.rel[buf], 1u);
        if (prev == (blockDim.x / 32) - 1) {
          sm.rel[buf] = 0u;
          if (j + NS < np && SUPRA_DBG(a) != 2) {
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
    __syncthreads();  // every warp is done with the ring: it becomes the line buffer

    // ---- RF = sum / N (reading #7; 0 when N = 0) ----
    const uint16_t* ncount = a.ncount + (size_t)g * S;
    const int kbase = k0 - 2 * P;  // line buffer position b = k - kbase
#pragma unroll
    for (int m = 0; m < NT; m++) {
      const int k = k0 + m * kTileK + kt;
      float v[VF];
      if (k >= 0 && k < S) {
        const int n = (int)ncount[k];
        const float inv = (a.normalize == SUPRA_NORM_NONE) ? 1.f : (n > 0 ? 1.f / (float)n : 0.f);
        if constexpr (VF == 1) {
          v[0] = acc.s(m) * inv;
        } else {
#pragma unroll
          for (int q = 0; q < VF / 2; q++) {
            v[2 * q] = acc.p[m][q].x * inv;
            v[2 * q + 1] = acc.p[m][q].y * inv;
          }
        }
        if (a.rf) {
#pragma unroll
          for (int b = 0; b < VF; b++) {
            const int2 lf = sm.vout[b];
            if (lf.y >= 0) a.rf[((size_t)lf.y * a.L + lf.x) * S + k] = v[b];
          }
        }
      } else {
#pragma unroll
        for (int b = 0; b < VF; b++) v[b] = 0.f;  // zero padding before 0 and past the record
      }
      if (a.do_epilogue) {
        const int pk = fir_pad(k - kbase);
#pragma unroll
        for (int q4 = 0; q4 < (VF + 3) / 4; q4++) {
          float4 x;
          x.x = v[4 * q4];
          x.y = (4 * q4 + 1 < VF) ? v[(4 * q4 + 1) % VF] : 0.f;
          x.z = (4 * q4 + 2 < VF) ? v[(4 * q4 + 2) % VF] : 0.f;
          x.w = (4 * q4 + 3 < VF) ? v[(4 * q4 + 3) % VF] : 0.f;
          sm.line[(size_t)q4 * span + pk] = x;
        }
      }
    }
    if (!a.do_epilogue) continue;
    // carried RF tail (or zeros before k = 0) and zeros after the pass
    const int tail = P + 4;
    for (int i = threadIdx.x; i < ng * (2 * P + tail); i += blockDim.x) {
      const int q4 = i / (2 * P + tail), r = i - q4 * (2 * P + tail);
      if (r < 2 * P)
        sm.line[(size_t)q4 * span + fir_pad(r)] =
            k0 == kfirst ? make_float4(0.f, 0.f, 0.f, 0.f) : sm.carry[q4 * 2 * P + r];
      else
        sm.line[(size_t)q4 * span + fir_pad(PL + r)] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    // ---- epilogue: outputs whose taps are complete in this pass ----
    const int o_begin = k0 == kfirst ? 0 : k0 - P;
    const int o_end = kend == S ? S : k0 + PL - P;
    const int nblk = o_end > o_begin ? (o_end - o_begin + 3) / 4 : 0;
    // (o_begin - kbase = 2P - kfirst or P: a multiple of 4 for the 65-tap
    // default, S and PL being multiples of 32)
    const bool p32 = P == 32;
    for (int it = threadIdx.x; it < ng * nblk; it += blockDim.x) {
      const int q4 = it / nblk, blk = it - q4 * nblk;
      if (q4 != curg) {
        flush_max();
        curg = q4;
        bmax[0] = bmax[1] = bmax[2] = bmax[3] = 0.f;
      }
      if (p32)
        fir_block<VF, 32>(a, sm.line + (size_t)q4 * span, kbase, o_begin + 4 * blk, o_end, sm.vout + 4 * q4, bmax);
      else
        fir_block<VF>(a, sm.line + (size_t)q4 * span, kbase, o_begin + 4 * blk, o_end, sm.vout + 4 * q4, bmax);
    }
    // RF tail k in [k0 + PL - 2P, k0 + PL) for the next pass's first outputs
    if (kend < S)
      for (int i = threadIdx.x; i < ng * 2 * P; i += blockDim.x) {
        const int q4 = i / (2 * P), r = i - q4 * 2 * P;
        sm.carry[i] = sm.line[(size_t)q4 * span + fir_pad(PL + r)];
      }
    // (the __syncthreads at the top of the next pass orders these reads
    // before the ring is refilled)
  }
  if (a.do_epilogue && !a.ref_fixed) {
    flush_max();
    __syncthreads();
    if (threadIdx.x < FB && f0 + (int)threadIdx.x < a.F)
      atomicMax(&a.frame_max[f0 + threadIdx.x], sm.smax[threadIdx.x]);
  }
  // secondary launch of a split call: complete only after the primary grid
  // (so work queued behind this kernel also sees the primary's results)
  if (a.pdl_wait_end) asm volatile("griddepcontrol.wait;" ::: "memory");
}

inline size_t das_smem_bytes_impl(int FB, int NT, int nent_max, int fir_taps, int MIR) {
  size_t off[9];
  return layout_bytes(FB, NT, nent_max, (fir_taps - 1) / 2, MIR, off);
}

template <int FB, int NT, bool T0, int MIR>
cudaError_t launch_k(const CUtensorMap& tm, const DasArgs& a, const RawMaps& maps, cudaStream_t st) {
  const size_t smem = das_smem_bytes_impl(FB * MIR, NT, a.entries_per_group, a.fir_taps, MIR);
  auto kern = das_fused_kernel<FB, NT, T0, MIR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.nlines / MIR, (a.Fmap + FB - 1) / FB);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.pdl_wait_end ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, tm, a, maps);
}

}  // namespace supra
