// dev aid: TMA throughput of the DAS staging pattern -- one 5-D box per
// "entry" {P pairs, rows, 1 channel, 1 event, FB frames} from an int16
// [F][E][C][S] buffer into a ring of NS stages, 2 CTAs x 256 threads per SM,
// one elected thread issuing, the CTA releasing a stage when all warps saw
// it.  Varies the row width (P = 16, 32, 64 pairs = 64/128/256 B) at a
// fixed window (samples per box) to see whether the per-row request rate,
// not bytes, bounds the copy.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(256, 2) k(const __grid_constant__ CUtensorMap tm, int nent, int rows, int fb,
                                            int ns, unsigned stage_bytes, int C, int E, int win_rows_per_step,
                                            int S_rows, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[8];
  __shared__ unsigned rel[8];
  const int line = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ns; i++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      rel[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto produce = [&](int j, int b) {
    const int ch = j % C, ev = line % E;
    const int r0 = (j * win_rows_per_step) % (S_rows - rows + 1);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[b])), "r"(stage_bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(sa(sm + (size_t)b * stage_bytes)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(r0), "r"(ch), "r"(ev), "r"(0), "r"(sa(&full[b]))
        : "memory");
  };
  if (threadIdx.x == 0)
    for (int j = 0; j < ns && j < nent; j++) produce(j, j);
  unsigned phase = 0, acc = 0;
  int b = 0;
  for (int j = 0; j < nent; j++) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            sa(&full[b])),
        "r"(phase)
        : "memory");
    acc += sm[(size_t)b * stage_bytes + (threadIdx.x * 4) % stage_bytes];
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
      unsigned prev = atomicAdd(&rel[b], 1u);
      if (prev == 7) {
        rel[b] = 0;
        if (j + ns < nent) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          produce(j + ns, b);
        }
      }
    }
    if (++b == ns) { b = 0; phase ^= 1; }
  }
  if (acc == 0xFFFFFFFF) sink[0] = acc;
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  const int F = 16, E = 256, C = 128, S = 2048;  // C2-like: 128 MiB per frame
  int16_t* raw;
  size_t bytes = (size_t)F * E * C * S * 2;
  cudaMalloc(&raw, bytes);
  cudaMemset(raw, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int lines = 148 * 2 * 4;
  printf("window samples, row bytes, FB, stages: GB/s of box bytes\n");
  for (int fb : {16, 4}) {
    for (int pairs : {16, 32, 64}) {
      const int rs = pairs * 2;                    // samples per row
      const int win = 1088;                        // samples per window (C2 NT=4)
      const int rows = (win + rs - 1) / rs;
      const unsigned stage = (unsigned)(fb * rows * rs * 2);
      int ns = (int)((110 * 1024) / stage);
      if (ns > 8) ns = 8;
      if (ns < 2) ns = 2;
      CUtensorMap tm;
      cuuint64_t dims[5] = {(cuuint64_t)pairs, (cuuint64_t)S / rs, (cuuint64_t)C, (cuuint64_t)E, (cuuint64_t)F};
      cuuint64_t str[4] = {(cuuint64_t)rs * 2, (cuuint64_t)S * 2, (cuuint64_t)C * S * 2, (cuuint64_t)E * C * S * 2};
      cuuint32_t box[5] = {(cuuint32_t)pairs, (cuuint32_t)rows, 1, 1, (cuuint32_t)fb};
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, raw, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
      const size_t smem = (size_t)ns * stage;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int nent = 256;
      for (int rep = 0; rep < 2; rep++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        k<<<lines, 256, smem>>>(tm, nent, rows, fb, ns, stage, C, E, 7, S / rs, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double gb = (double)lines * nent * stage / 1e9;
        if (rep) printf("win %d row %3d B fb %2d ns %d: %.0f GB/s (%.1f ns per box per SM) %s\n", win, rs * 2, fb, ns,
                        gb / (ms * 1e-3), ms * 1e6 / ((double)lines * nent / 148), cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
