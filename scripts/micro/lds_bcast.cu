// Microbenchmark (dev aid): shared-memory wavefronts of 32/64/128-bit loads
// when the 32 lanes of a warp read only a few distinct addresses (the linear
// scan conversion's pixel loop: lanes = columns, ~6 distinct lines per warp).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_bcast lds_bcast.cu
// Run under: ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_op_shared_ld.sum ./lds_bcast
#include <cstdio>

template <int W>
__global__ void k(float* out, int distinct, int iters) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  // lane -> one of `distinct` consecutive W-float slots
  const int slot = (lane * distinct) / 32;
  float acc = 0.f;
  int base = 0;
  for (int it = 0; it < iters; it++) {
    const float* p = s + ((base + slot * W) & 2047);
    if constexpr (W == 1) {
      acc += p[0];
    } else if constexpr (W == 2) {
      float2 v = *reinterpret_cast<const float2*>(p);
      acc += v.x + v.y;
    } else {
      float4 v = *reinterpret_cast<const float4*>(p);
      acc += v.x + v.y + v.z + v.w;
    }
    base += 64;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  float* o;
  cudaMalloc(&o, 1 << 20);
  const int iters = 1000;
  for (int d : {1, 6, 8, 16, 32}) {
    k<1><<<1, 32>>>(o, d, iters);
    k<2><<<1, 32>>>(o, d, iters);
    k<4><<<1, 32>>>(o, d, iters);
  }
  cudaDeviceSynchronize();
  printf("done (read the ncu metrics per launch: order d=1,6,8,16,32 x W=1,2,4)\n");
  return 0;
}
