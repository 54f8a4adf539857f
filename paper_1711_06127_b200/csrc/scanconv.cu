// scanconv.cu -- scan conversion of the log-compressed line image onto the
// Cartesian output grid (readings #21-#23).
//
// The integer part of the inverse map (validity, i0, k0) and the fractions
// come from binary64 tables built at create (host.cpp), so indices are
// bit-exact; the kernels are pure gathers + bilinear/trilinear blends.
//   linear 2D : separable -- u depends only on x, v only on z: two 1-D tables.
//   sector 2D / pyramid 3D : per output row (iz, iy) the contiguous valid x
//               range and 16-byte entries (corner offset, fx, fy, fz).
#include <algorithm>

#include "internal.h"

namespace supra {

namespace {

__device__ __forceinline__ float load_y(const void* p, int type, size_t i) {
  if (type == SUPRA_T_U8) return (float)((const uint8_t*)p)[i] * (1.0f / 255.0f);
  return __ldg((const float*)p + i);
}

__device__ __forceinline__ void store_img(void* p, int type, size_t i, float v) {
  if (type == SUPRA_T_U8) ((uint8_t*)p)[i] = (uint8_t)floorf(255.f * v + 0.5f);
  else ((float*)p)[i] = v;
}

}  // namespace

// grid (ceil(nx/128), nz, F); block 128: one pixel per thread, x fastest.
__global__ void __launch_bounds__(128) sc_linear_kernel(const ScArgs a) {
  const int ix = blockIdx.x * blockDim.x + threadIdx.x;
  const int iz = blockIdx.y, f = blockIdx.z;
  if (ix >= a.nx) return;
  const ScAxis ax = a.ax[ix], az = a.az[iz];
  const bool ok = ax.i0 >= 0 && az.i0 >= 0;
  float v = 0.f;
  if (ok) {
    const size_t L = (size_t)a.Lx;
    const size_t b = ((size_t)f * L + ax.i0) * a.S + az.i0;
    const float y00 = load_y(a.line_img, a.in_type, b);
    const float y01 = load_y(a.line_img, a.in_type, b + 1);
    const float y10 = load_y(a.line_img, a.in_type, b + a.S);
    const float y11 = load_y(a.line_img, a.in_type, b + a.S + 1);
    const float fx = ax.f, fz = az.f;
    v = (1.f - fz) * ((1.f - fx) * y00 + fx * y10) + fz * ((1.f - fx) * y01 + fx * y11);
  }
  const size_t o = (size_t)iz * a.nx + ix;
  store_img(a.img, a.out_type, (size_t)f * a.nz * a.nx + o, v);
  if (a.mask && f == 0) a.mask[o] = ok ? 1 : 0;
}

// grid (nz*ny, F); block 256 looping over x.
__global__ void __launch_bounds__(256) sc_table_kernel(const ScArgs a) {
  const int r = blockIdx.x, f = blockIdx.y;
  const ScRow row = a.rows[r];
  const size_t S = (size_t)a.S, LS = (size_t)a.Lx * a.S;
  const size_t fbase = (size_t)f * a.Ly * LS;
  const size_t obase = ((size_t)f * a.nz * a.ny + r) * a.nx;
  for (int ix = threadIdx.x; ix < a.nx; ix += blockDim.x) {
    float v = 0.f;
    bool ok = false;
    if (ix >= row.xlo && ix < row.xhi) {
      const ScEntry e = a.ent[row.off + (ix - row.xlo)];
      if (e.base >= 0) {
        ok = true;
        const size_t b = fbase + (size_t)e.base;
        const float fx = e.fx, fz = e.fz;
        const float y000 = load_y(a.line_img, a.in_type, b);
        const float y001 = load_y(a.line_img, a.in_type, b + 1);
        const float y100 = load_y(a.line_img, a.in_type, b + S);
        const float y101 = load_y(a.line_img, a.in_type, b + S + 1);
        float v0 = (1.f - fz) * ((1.f - fx) * y000 + fx * y100) + fz * ((1.f - fx) * y001 + fx * y101);
        if (a.is3d) {
          const float fy = e.fy;
          const float y010 = load_y(a.line_img, a.in_type, b + LS);
          const float y011 = load_y(a.line_img, a.in_type, b + LS + 1);
          const float y110 = load_y(a.line_img, a.in_type, b + LS + S);
          const float y111 = load_y(a.line_img, a.in_type, b + LS + S + 1);
          float v1 = (1.f - fz) * ((1.f - fx) * y010 + fx * y110) + fz * ((1.f - fx) * y011 + fx * y111);
          v = (1.f - fy) * v0 + fy * v1;
        } else {
          v = v0;
        }
      }
    }
    store_img(a.img, a.out_type, obase + ix, v);
    if (a.mask && f == 0) a.mask[(size_t)r * a.nx + ix] = ok ? 1 : 0;
  }
}

cudaError_t launch_sc_linear(const ScArgs& a, cudaStream_t st) {
  dim3 grid((a.nx + 127) / 128, a.nz, a.F);
  sc_linear_kernel<<<grid, 128, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sc_table(const ScArgs& a, cudaStream_t st) {
  dim3 grid(a.nz * a.ny, a.F);
  sc_table_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace supra
