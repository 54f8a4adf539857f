// stage.cu -- end-to-end input staging (supra_bf_stage_raw): copy, for every
// (frame, event, channel) trace, only the sample range the beamformer reads
// (host-computed hull, 16-byte rounded) from src to dst.  src may be
// page-locked host memory: the device reads it over PCIe (UVA), so the
// host->device transfer carries the referenced bytes only (C2: 41 % of a
// frame, SURVEY 8(d) "Fetch windows, not whole rows").
#include "internal.h"

namespace supra {

#ifndef STAGE_U
#define STAGE_U 8
#endif
// One warp per trace, 8 traces per CTA; lane i moves 16-byte chunks
// i, i + 32, ... of the trace's range, STAGE_U loads in flight per lane.
// Measured (C2, 16 pinned frames): ~49 GB/s over PCIe for STAGE_U = 2..16
// (device-initiated reads; the copy engine reaches ~55 GB/s on whole
// frames), so 830-850 frames/s end to end against 409 for whole frames.
__global__ void __launch_bounds__(256) stage_raw_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                                        const uint32_t* __restrict__ iv, int traces_per_frame,
                                                        int s8, long long traces) {
  const long long tr = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (tr >= traces) return;
  const int lane = threadIdx.x & 31;
  const uint32_t w = iv[tr % traces_per_frame];
  const int c0 = (int)(w & 0xFFFFu), c1 = (int)(w >> 16);  // 16-byte chunk range [c0, c1)
  const size_t base = (size_t)tr * s8;
  int i = c0 + lane;
  for (; i + 32 * (STAGE_U - 1) < c1; i += 32 * STAGE_U) {
    int4 v[STAGE_U];
#pragma unroll
    for (int u = 0; u < STAGE_U; u++) v[u] = src[base + i + 32 * u];
#pragma unroll
    for (int u = 0; u < STAGE_U; u++) dst[base + i + 32 * u] = v[u];
  }
  for (; i < c1; i += 32) dst[base + i] = src[base + i];
}

cudaError_t launch_stage_raw(const void* src, void* dst, const uint32_t* iv, int traces_per_frame, int S,
                             int frames, cudaStream_t st) {
  const long long traces = (long long)traces_per_frame * frames;
  if (traces == 0) return cudaSuccess;
  stage_raw_kernel<<<(unsigned)((traces + 7) / 8), 256, 0, st>>>((const int4*)src, (int4*)dst, iv,
                                                                  traces_per_frame, S / 8, traces);
  return cudaGetLastError();
}

}  // namespace supra
