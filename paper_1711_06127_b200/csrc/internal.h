// internal.h -- types shared by the host library (host.cpp) and the sm_100a
// kernels (das.cu, epilogue.cu, scanconv.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "supra_bf.h"

namespace supra {

// DAS kernel geometry.  A consumer thread owns output samples
// k = kt + kTileK * m (m = 0 .. NT-1) of its line.
constexpr int kTileK = 256;
// Staged traces are fetched in rows of kRowSamples samples (the 5-D tensor
// map splits the time axis into rows so one TMA box covers a whole trace).
constexpr int kRowSamples = 32;
// Maximum stages in the trace ring (one aperture entry per stage).
constexpr int kMaxStages = 8;
// FIR half-length limit (fir_taps <= 2*kMaxHalfTaps + 1 = 129).
constexpr int kMaxHalfTaps = 64;
// Frequency-compounding bands (SUPRA_MAX_BANDS).
constexpr int kMaxBands = SUPRA_MAX_BANDS;
// Largest record the DAS kernel holds per line (NT = 16 tiles).
constexpr int kMaxSamples = 16 * kTileK;
// Output tiles per thread and pass (a template parameter of the DAS kernel,
// NT in {4, 8, 16}; a pass covers kTileK * NT samples of depth) and the
// trace rows one TMA box fetches for that NT (the stage's frame stride).
inline __host__ __device__ int das_nt(int S) {  // largest useful NT for S
  const int t = (S + kTileK - 1) / kTileK;
  return t <= 4 ? 4 : (t <= 8 ? 8 : 16);
}
inline __host__ __device__ int das_rows_nt(int nt) { return nt * (kTileK / kRowSamples) + 2; }
// DAS launch shape: virtual frames per CTA (fb = frames x mir mirror lines)
// x tiles per pass (nt), fb * nt <= 64; mir lines share one delay set.
struct DasShape {
  int fb, nt, mir = 1;
};

// One receive-aperture entry of a line group (lines sharing an origin),
// sorted by k_enter.  Lengths in "sample units" (mm * fs / (1000 c)), in
// which the focal depth of output sample k is h = k/2.
struct __align__(16) DasEntry {
  float qx, qy, qz;  // (line origin - element position) in samples
  float A;           // |q|^2, rounded from binary64
  float cu;          // 4 F rho_s:  u = rho/R = cu / k  (R = z/(2F))
  int32_t elem;      // channel index
  int32_t kenter;    // first k with (2F) rho <= k dr (binary64 predicate); >= S: never
  int32_t pad;
};

struct DasArgs {
  const int16_t* raw;      // [F][E][C][S]
  int F, E, C, S, L;
  int dec, Sd;             // envelope decimation: line image [F][L][Sd], Sd = S / dec, keeps k = dec q
  int entries_per_group;   // row stride of `entries`
  int line0, nlines;           // lines [line0, line0 + nlines) of every frame are beamformed
  int fbase, Fmap;             // frames [fbase, fbase + Fmap) of the call, = frames [0, Fmap) of the tensor map
  int pdl_trigger;             // primary of a split call: let the secondary start on free SMs
  int pdl_wait_end;            // secondary: launched programmatically, retire after the primary
  // CTA descriptors {primary line, line[4], variant[4]} for the launch's
  // lines per CTA (MIR = 1: one per line; 2: x-mirror pairs, row-major over
  // lx < Lx/2; 4: quads over lx < Lx/2, ly < Ly/2): the
  // primary's group, direction and entry order serve every line of the
  // CTA; slot s reads entry j from channel ech[g][j][variant[s]] (mirror
  // symmetry, host.cpp build_mirror_tables)
  const int32_t* cta;
  int cta_base;                // descriptor of CTA b: cta[cta_base + b]
  const int32_t* ech;          // [G][entries_per_group][4]
  const int32_t* line_group;   // [L]
  const DasEntry* entries;     // [G][entries_per_group], sorted by kenter (ascending)
  const int32_t* nentries;     // [G]: entries with kenter < S
  const uint16_t* ncount;      // [G][S]: N(k) = #entries with kenter <= k
  const float4* line_dir;      // [L] (dx, dy, dz, 0)
  const int32_t* line_event;   // [L]
  float t0fs;                  // t0 * fs (samples); + 1/2 for nearest-sample lookup
  float fr_scale;              // 1: linear interpolation; 0: nearest sample (x~[floor(tau + 1/2)])
  float win_a, win_b;          // w = a + b cos(pi u)
  int normalize;               // 0 count, 1 none
  // outputs
  float* rf;                   // [F][L][S] or null
  int do_epilogue;             // 1: FIR + envelope (+ log) epilogue
  const float2* fir;           // [nbands][T] complex taps g_j = h_j e^{+i w j}, j = -P..P
  int fir_taps;
  // the same taps split by symmetry (reading #18): c_j = Re g_j (even),
  // s_j = Im g_{-j} = -Im g_j ... stored for j = 0..P as c[b][j] = Re g_j,
  // s[b][j] = Im g_j of band b; passed by value so the unrolled FIR reads
  // them from the constant bank (uniform-register operands of FFMA2).
  int nbands;                  // 1 .. kMaxBands (frequency compounding)
  float band_w[kMaxBands];     // env = sum_b band_w[b] env_b
  float fir_c[kMaxBands][kMaxHalfTaps + 1];
  float fir_s[kMaxBands][kMaxHalfTaps + 1];
  int ref_fixed;               // 1: y written directly; 0: env written + frame max
  float log_k1, log_k0;        // y = k1 log2(env) + k0 (fixed reference)
  float* env_out;              // [F][L][S] f32 (frame-max mode)
  void* y_out;                 // [F][L][S] (fixed mode)
  int y_type;                  // SUPRA_T_F32 / SUPRA_T_U8
  unsigned* frame_max;         // [F] float bits (frame-max mode)
  int debug_skip;              // measurement only: skip the tap loop (TMA pipeline alone)
  int vec_out;                 // 1: line outputs 16-byte aligned (4 consecutive samples per store)
  // 1: windows use the row-cut tensor maps of the launch's RawMaps kernel
  // parameter (exact windows); 0: every window uses the launch's map
  int row_cut;
};

// Row-cut tensor maps, passed BY VALUE as a __grid_constant__ kernel
// parameter (16 KB; kernel parameters may be up to 32 KB since CUDA 12.1):
// m[r - 1] is the launch's raw map with only r time rows in range, so a
// window box whose rows past the pass's last referenced row are out of
// bounds reads them as zeros without DRAM traffic (exact windows, one TMA
// per entry).  Being a parameter, the set lives in the launch itself: no
// device allocation, no host synchronisation, and a captured CUDA graph
// keeps its own copy.
struct RawMaps {
  CUtensorMap m[kMaxSamples / kRowSamples];
};

struct EnvArgs {  // standalone epilogue on an RF buffer
  const float* rf;
  int F, L, S;
  int dec, Sd;         // line image [F][L][Sd], k = dec q
  const float2* fir;   // [nbands][T]
  int fir_taps;
  int nbands;
  float band_w[kMaxBands];
  int ref_fixed;
  float log_k1, log_k0;
  float* env_out;
  void* y_out;
  int y_type;
  unsigned* frame_max;
};

struct FinalizeArgs {  // env -> y with a per-frame (or fixed) reference
  const float* env;    // [F][frame_stride], elements [offset, offset + per_frame) of each frame
  long long per_frame; // elements converted per frame (L*S, or nlines*S for a line range)
  long long frame_stride, offset;
  int F;
  const unsigned* frame_max;  // [F] float bits of the reference; NULL -> fixed_ref
  float fixed_ref;
  float DR_k;          // 20 log10(2) / DR
  void* y_out;
  int y_type;
};

// Linear scan-conversion tile: 256 columns x kScRows rows per CTA; the
// staged slab holds at most kScMaxLines lines x kScMaxK samples (checked at
// create: the tile's columns must span <= kScMaxLines - 1 line pitches).
constexpr int kScRows = 32;
// lines the 32 columns of one warp may touch (+1), checked at create
constexpr int kScWarpLinesMax = 11;
constexpr int kScMaxLines = 64;
constexpr int kScMaxK = 64;

// Linear (separable) scan conversion table entries.
struct ScAxis {
  int32_t i0;   // -1: invalid
  float f;
};

// Sector / pyramid: per output row (iz, iy) the valid x range [xlo, xhi),
// the index of its first entry and the row's lateral-y fraction fy (for the
// pyramid u_y = atan2(Y, Z) / dtheta_y + (Ly-1)/2 depends on the row only,
// reading #13; 0 in 2D).  Entries (8 bytes) hold the line-image offset of
// the (i0x, i0y, k0) corner (0xFFFFFFFF: invalid) and fx, fz as unorm16
// (q = round(65535 f); |f - q/65535| <= 7.7e-6, i.e. <= 2.3e-5 in y or
// 0.0012 dB at DR = 50 dB -- inside the 0.01 dB contract; the integer
// indices stay bit-exact).
struct ScRow {
  int32_t xlo, xhi;
  uint32_t off;
  float fy;
};
struct __align__(8) ScEntry {
  uint32_t base;  // (i0y*Lx + i0x)*S + k0, or 0xFFFFFFFF
  uint32_t fxz;   // fx_q | fz_q << 16
};
constexpr uint32_t kScInvalid = 0xFFFFFFFFu;

struct ScArgs {
  const void* line_img;  // [F][Ly][Lx][S]
  int in_type;
  int F, Lx, Ly, S;
  int nx, ny, nz;
  void* img;             // [F][nz][ny][nx]
  int out_type;
  uint8_t* mask;         // [nz][ny][nx] or null
  // linear
  const ScAxis* ax;      // [nx]
  const ScAxis* az;      // [nz]
  const int32_t* blk_kmin;  // [ceil(nz / kScRows)]: smallest valid k0 of the row block, -1 if none
  int slab_k;            // samples per line staged per row block
  const int32_t* col_l0;    // [ceil(nx / 256)]: first line the column tile touches
  const int32_t* col_nl;    // [ceil(nx / 256)]: lines it touches (0: none valid)
  int tiled;             // 1: tiled separable kernel; 0: direct per-pixel kernel
  int slab_tma;          // 1: stage the slab with 1-D bulk copies (f32), 2: one 2-D tensor copy (f32 or u8 line image)
  int slab_box_k, slab_box_l;  // staged segment: samples (16 bytes multiple) x lines
  // table
  const ScRow* rows;     // [nz*ny]
  const ScEntry* ent;
  int is3d;
  // non-NULL: line_img holds the envelope (f32) and every interpolation
  // corner is log-compressed on load against frame_max[f] (float bits),
  // y = clamp(1 + DR_k (log2 env - log2 ref), 0, 1) -- finalize_kernel's
  // expression, so the image equals finalize + scan conversion bitwise
  const unsigned* frame_max;
  float DR_k;
};

#ifdef __CUDACC__
// The measurement-only debug modes exist in -DSUPRA_DEV_KNOBS builds only;
// the product kernels always run the whole path (the checks fold away).
#ifdef SUPRA_DEV_KNOBS
#define SUPRA_DBG(a) ((a).debug_skip)
#else
#define SUPRA_DBG(a) 0
#endif
// log2 via MUFU.LG2: absolute error <= 2^-22.6 (PTX ISA), i.e. <= 1.6e-6 dB
// after the 20 log10 2 scale -- far inside the 0.01 dB contract.
__device__ __forceinline__ float lg2_approx(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
#endif

// Launchers (return cudaGetLastError()).
// raw is addressed through a 5-D tensor map {16 sample pairs (u32), S/32
// rows, C, E, F} with box {16, das_rows_nt(nt), 1, 1, fb} for sh = das_shape().
// allow_warp: a single-frame CALL may use the warp-split kernel (its own sum
// order); every multi-frame call, remainder launches included, uses
// das_fused_kernel, whose results are bitwise independent of the batch.
cudaError_t launch_das(const CUtensorMap& raw_map, const DasArgs& a, const RawMaps& maps, DasShape sh,
                       bool allow_warp, cudaStream_t st);
DasShape das_shape(int fb_max, int S, int F, int nent_max, int fir_taps, int mir = 1);
// One frame per CTA (fb = 1) with the aperture split across warps
// (das_warp.cu); same tensor map as launch_das for that shape.
bool das_warp_ok(int fb, int S, float t0fs);
cudaError_t launch_das_warp(const CUtensorMap& raw_map, const DasArgs& a, cudaStream_t st);
size_t das_smem_bytes(int fb, int nt, int nent_max, int fir_taps, int mir);
cudaError_t launch_envlog(const EnvArgs& a, cudaStream_t st);
cudaError_t launch_finalize(const FinalizeArgs& a, cudaStream_t st);
// iv[e * C + c] = 16-byte chunk range [lo, hi) of trace (e, c) (lo | hi << 16)
cudaError_t launch_stage_raw(const void* src, void* dst, const uint32_t* iv, int traces_per_frame, int S,
                             int frames, cudaStream_t st);
cudaError_t launch_sc_linear(const ScArgs& a, const CUtensorMap* slab_map, cudaStream_t st);
cudaError_t launch_sc_table(const ScArgs& a, int line_img_bytes_per_frame, cudaStream_t st);

}  // namespace supra
