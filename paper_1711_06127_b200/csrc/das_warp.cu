// das_warp.cu -- dispatch of the single-frame warp-split DAS kernel
// (das_warp_kernel.cuh; variants instantiated in das_warp_inst*.cu).
#include "das_warp_kernel.cuh"

namespace supra {

extern template cudaError_t launch_w<32, false, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<64, false, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<32, true, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<64, true, 0>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<32, false, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<64, false, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<32, true, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<64, true, 1>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<32, false, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<64, false, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<32, true, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);
extern template cudaError_t launch_w<64, true, 2>(const CUtensorMap&, const DasArgs&, cudaStream_t);

// Usable for one frame per CTA when the record is exactly 32 NTL samples
// (and |t0| keeps non-member reads inside the guard below the ring).
bool das_warp_ok(int fb, int S, float t0fs) {
  return fb == 1 && (S == 1024 || S == 2048) && fabsf(t0fs) < 0.5f * (float)S;
}

size_t das_warp_smem_bytes(int S, int fir_taps) { return das_warp_smem_bytes_impl(S, fir_taps); }

template <bool HANN, int MODE>
static cudaError_t launch_w2(const CUtensorMap& tm, const DasArgs& a, cudaStream_t st) {
  return a.S == 1024 ? launch_w<32, HANN, MODE>(tm, a, st) : launch_w<64, HANN, MODE>(tm, a, st);
}

cudaError_t launch_das_warp(const CUtensorMap& tm, const DasArgs& a, cudaStream_t st) {
  const bool hann = a.win_a == 0.5f && a.win_b == 0.5f;
  const int mode = a.fr_scale == 0.f ? 2 : (a.t0fs != 0.f ? 1 : 0);
  if (mode == 2) return hann ? launch_w2<true, 2>(tm, a, st) : launch_w2<false, 2>(tm, a, st);
  if (mode == 1) return hann ? launch_w2<true, 1>(tm, a, st) : launch_w2<false, 1>(tm, a, st);
  return hann ? launch_w2<true, 0>(tm, a, st) : launch_w2<false, 0>(tm, a, st);
}

}  // namespace supra
