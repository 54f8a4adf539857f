// das.cu -- launch-shape selection and dispatch of the DAS batch kernel
// (das_kernel.cuh); the kernel variants are instantiated in das_inst*.cu.
#include <cstdio>
#include <cstdlib>

#include "das_kernel.cuh"

namespace supra {

extern template cudaError_t launch_k<16, 4, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<16, 4, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<8, 8, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<8, 8, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<8, 4, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<8, 4, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 16, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 16, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 8, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 8, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 4, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 4, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 16, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 16, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 8, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 8, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 4, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 4, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 16, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 16, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 8, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 8, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 4, false, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 4, true, 1>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
// mirror-line variants (MIR = 2, 4 lines per CTA; t0 = 0 only)
extern template cudaError_t launch_k<1, 8, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 16, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 8, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 16, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<8, 4, false, 2>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 8, false, 4>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 16, false, 4>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 4, false, 4>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<2, 8, false, 4>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<4, 4, false, 4>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);
extern template cudaError_t launch_k<1, 4, false, 4>(const CUtensorMap&, const DasArgs&, const RawMaps&, cudaStream_t);

size_t das_smem_bytes(int FB, int NT, int nent_max, int fir_taps, int mir) {
  return das_smem_bytes_impl(FB, NT, nent_max, fir_taps, mir);
}

// (virtual frames per CTA, tiles per pass) for `mir` mirror lines per CTA:
// the first feasible candidate -- VF x NT accumulators <= 64 per thread,
// passes no longer than the record, the shared-memory footprint allows 2
// CTAs per SM with >= 3 ring stages, and never more frames (VF / mir) than
// the call (or fb_max).  Only instantiated (VF / mir, NT, mir) are listed.
DasShape das_shape(int fb_max, int S, int F, int nent_max, int fir_taps, int mir) {
  static const int cand1[][2] = {{16, 4}, {8, 8}, {8, 4}, {4, 16}, {4, 8}, {4, 4}, {2, 16},
                                 {2, 8},  {2, 4}, {1, 16}, {1, 8}, {1, 4}};
  static const int cand2[][2] = {{16, 4}, {4, 16}, {4, 8}, {2, 16}, {2, 8}};
  static const int cand4[][2] = {{16, 4}, {8, 8}, {8, 4}, {4, 16}, {4, 8}, {4, 4}};
  const int(*cand)[2] = mir == 4 ? cand4 : (mir == 2 ? cand2 : cand1);
  const int ncand = mir == 4 ? 6 : (mir == 2 ? 5 : 12);
  const int ntmax = das_nt(S);
  const int P = (fir_taps - 1) / 2;
  int ofb = 0, ont = 0;
#ifdef SUPRA_DEV_KNOBS
  // dev override (A/B measurements only): SUPRA_BF_SHAPE=<vf>x<nt> for
  // mir = 1, SUPRA_BF_MIRSHAPE=<vf>x<nt> for mir > 1 (a listed candidate)
  if (const char* ev = std::getenv(mir == 1 ? "SUPRA_BF_SHAPE" : "SUPRA_BF_MIRSHAPE"))
    std::sscanf(ev, "%dx%d", &ofb, &ont);
#endif
  for (int ci = -1; ci < ncand; ci++) {
    const int vf = ci < 0 ? ofb : cand[ci][0], nt = ci < 0 ? ont : cand[ci][1];
    if (ci < 0) {  // the override must be one of the instantiated candidates
      bool listed = false;
      for (int j = 0; j < ncand; j++) listed = listed || (cand[j][0] == ofb && cand[j][1] == ont);
      if (!listed) continue;
    }
    const int fb = vf / mir;
    if (fb > fb_max || (fb > F && fb > 1) || nt > ntmax) continue;
    const size_t fixed = fixed_bytes(vf, nent_max, P, mir);
    const size_t ring = 3 * stage_bytes(vf, das_rows_nt(nt));
    const size_t fir = align128((size_t)fir_groups(vf) * fir_span(nt * kTileK, P) * 16);
    if (fixed + (ring > fir ? ring : fir) > das_smem_budget(vf, nt)) continue;
    return DasShape{vf, nt, mir};
  }
  return mir == 1 ? DasShape{1, 4, 1} : DasShape{0, 0, mir};  // {0, ...}: no feasible mirror shape
}

template <bool T0>
static cudaError_t launch_t0(const CUtensorMap& tm, const DasArgs& a, const RawMaps& m, DasShape sh,
                             cudaStream_t st) {
  const int nt = sh.nt;
  switch (sh.fb) {
    case 16: return launch_k<16, 4, T0, 1>(tm, a, m, st);
    case 8: return nt == 4 ? launch_k<8, 4, T0, 1>(tm, a, m, st) : launch_k<8, 8, T0, 1>(tm, a, m, st);
    case 4:
      return nt == 4 ? launch_k<4, 4, T0, 1>(tm, a, m, st)
                     : (nt == 8 ? launch_k<4, 8, T0, 1>(tm, a, m, st) : launch_k<4, 16, T0, 1>(tm, a, m, st));
    case 2:
      return nt == 4 ? launch_k<2, 4, T0, 1>(tm, a, m, st)
                     : (nt == 8 ? launch_k<2, 8, T0, 1>(tm, a, m, st) : launch_k<2, 16, T0, 1>(tm, a, m, st));
    default:
      return nt == 4 ? launch_k<1, 4, T0, 1>(tm, a, m, st)
                     : (nt == 8 ? launch_k<1, 8, T0, 1>(tm, a, m, st) : launch_k<1, 16, T0, 1>(tm, a, m, st));
  }
}

// sh.fb = virtual frames = frames per CTA x sh.mir
static cudaError_t launch_mir(const CUtensorMap& tm, const DasArgs& a, const RawMaps& m, DasShape sh,
                              cudaStream_t st) {
  const int fb = sh.fb / sh.mir, nt = sh.nt;
  if (sh.mir == 2) {
    if (fb == 8) return launch_k<8, 4, false, 2>(tm, a, m, st);
    if (fb == 2) return nt == 8 ? launch_k<2, 8, false, 2>(tm, a, m, st) : launch_k<2, 16, false, 2>(tm, a, m, st);
    return nt == 8 ? launch_k<1, 8, false, 2>(tm, a, m, st) : launch_k<1, 16, false, 2>(tm, a, m, st);
  }
  if (fb == 4) return launch_k<4, 4, false, 4>(tm, a, m, st);
  if (fb == 2) return nt == 4 ? launch_k<2, 4, false, 4>(tm, a, m, st) : launch_k<2, 8, false, 4>(tm, a, m, st);
  if (nt == 4) return launch_k<1, 4, false, 4>(tm, a, m, st);
  return nt == 8 ? launch_k<1, 8, false, 4>(tm, a, m, st) : launch_k<1, 16, false, 4>(tm, a, m, st);
}

cudaError_t launch_das(const CUtensorMap& tm, const DasArgs& a, const RawMaps& m, DasShape sh, bool allow_warp,
                       cudaStream_t st) {
  if (sh.mir > 1) return launch_mir(tm, a, m, sh, st);
  bool warp = allow_warp && das_warp_ok(sh.fb, a.S, a.t0fs);
#ifdef SUPRA_DEV_KNOBS
  if (std::getenv("SUPRA_BF_NO_WARP")) warp = false;  // A/B measurements only
#endif
  if (warp) return launch_das_warp(tm, a, st);
  return a.t0fs != 0.f ? launch_t0<true>(tm, a, m, sh, st) : launch_t0<false>(tm, a, m, sh, st);
}

}  // namespace supra
