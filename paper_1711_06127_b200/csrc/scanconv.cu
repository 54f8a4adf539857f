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
#include <cstdlib>

#include "internal.h"

namespace supra {

namespace {

__device__ __forceinline__ float load_y(const void* p, int type, size_t i) {
  if (type == SUPRA_T_U8) return (float)((const uint8_t*)p)[i] * (1.0f / 255.0f);
  return __ldg((const float*)p + i);
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ void store_img(void* p, int type, size_t i, float v) {
  if (type == SUPRA_T_U8) ((uint8_t*)p)[i] = (uint8_t)floorf(255.f * v + 0.5f);
  else ((float*)p)[i] = v;
}

}  // namespace

// Linear 2D, tiled and separable: one CTA per (256 output columns x
// kScRows output rows, frame); one thread per column.  Because u depends
// only on x and v only on z (reading #21), the bilinear blend factors into a
// depth lerp per (row, line) followed by a lateral lerp per pixel:
//   t[r][l] = lerp(y[l][k0], y[l][k0+1], fz(r)),
//   out[r][x] = lerp(t[r][i0], t[r][i0+1], fx(x)).
// The slab of the line image the tile touches (lines [l0, l0+nl) x ks
// samples from the row block's smallest k0, both host-computed) is staged in
// shared memory with one 1-D bulk copy (TMA) per line.
template <bool U8OUT>
__global__ void __launch_bounds__(256) sc_linear_tiled_kernel(const ScArgs a) {
  __shared__ __align__(128) float slab[kScMaxLines * kScMaxK];
  __shared__ float tz[kScRows * (kScMaxLines + 2)];
  __shared__ ScAxis saz[kScRows];
  __shared__ __align__(8) uint64_t bar;
  const int cb = blockIdx.x, rb = blockIdx.y, f = blockIdx.z;
  const int x = cb * 256 + threadIdx.x;
  const int z0 = rb * kScRows;
  const int ks = a.slab_k;
  const int kmin = a.blk_kmin[rb];
  const int l0 = a.col_l0[cb], nl = a.col_nl[cb];
  const int Lx = a.Lx, S = a.S, nx = a.nx;
  const int rows = min(kScRows, a.nz - z0);
  const size_t fbase = (size_t)f * Lx * S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool use_tma = a.in_type == SUPRA_T_F32 && a.slab_tma;
  const int kstride = use_tma ? a.slab_box_k : ks;    // slab row stride (samples)
  const int kal = kmin & ~3;                           // 16-byte aligned segment start
  if (use_tma) {
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\nfence.mbarrier_init.release.cluster;" ::"r"(b),
                   "r"(32)
                   : "memory");
    }
    __syncthreads();
    if (warp == 0) {
      // one 1-D bulk copy (TMA, UBLKCP) per line segment [kal, kal + box_k)
      // (clipped to the record), lanes take lines
      const float* src = (const float*)a.line_img + fbase;
      const int seg = min(a.slab_box_k, S - kal);
      unsigned bytes = 0;
      for (int l = lane; l < nl && kmin >= 0; l += 32) bytes += (unsigned)seg * 4u;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
      for (int l = lane; l < nl && kmin >= 0; l += 32)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                (uint32_t)__cvta_generic_to_shared(slab + l * a.slab_box_k)),
            "l"(src + (size_t)(l0 + l) * S + kal), "r"((unsigned)seg * 4u), "r"(b)
            : "memory");
    }
  }
  if (kmin >= 0 && nl > 0 && !use_tma) {
    if (a.in_type == SUPRA_T_F32) {
      const float* src = (const float*)a.line_img + fbase;
      for (int l = warp; l < nl; l += 8)
        for (int kk = lane; kk < ks; kk += 32)
          cp_async4(slab + l * ks + kk, src + (size_t)(l0 + l) * S + min(kmin + kk, S - 1));
    } else {
      for (int l = warp; l < nl; l += 8)
        for (int kk = lane; kk < ks; kk += 32)
          slab[l * ks + kk] = load_y(a.line_img, a.in_type, fbase + (size_t)(l0 + l) * S + min(kmin + kk, S - 1));
    }
  }
  if (threadIdx.x < rows) cp_async8(saz + threadIdx.x, a.az + z0 + threadIdx.x);
  asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
  const ScAxis ax = x < nx ? a.ax[x] : ScAxis{-1, 0.f};
  __syncthreads();
  if (use_tma) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&bar))
        : "memory");
  }
  // depth lerp t[r][l]; rows without a valid k0 and the spare pair of
  // columns [kScMaxLines, kScMaxLines+1] are zero, so the pixel loop below
  // needs no predicates (invalid columns read the zero pair with fx = 0)
  constexpr int TZS = kScMaxLines + 2;
  if ((int)threadIdx.x < nl) {
    const float* y = slab + threadIdx.x * kstride - (use_tma ? kal : kmin);
    for (int r = 0; r < rows; r++) {
      const ScAxis az = saz[r];
      tz[r * TZS + threadIdx.x] = az.i0 >= 0 ? fmaf(az.f, y[az.i0 + 1] - y[az.i0], y[az.i0]) : 0.f;
    }
  }
  if (threadIdx.x < 2 * kScRows) tz[(threadIdx.x >> 1) * TZS + kScMaxLines + (threadIdx.x & 1)] = 0.f;
  __syncthreads();
  if (x >= nx) return;
  const bool colok = ax.i0 >= 0;
  const float* tcol = tz + (colok ? ax.i0 - l0 : kScMaxLines);
  const float fx = colok ? ax.f : 0.f;
  const size_t out0 = ((size_t)f * a.nz + z0) * nx + x;
  if (U8OUT) {
    uint8_t* o = (uint8_t*)a.img + out0;
#pragma unroll 8
    for (int r = 0; r < rows; r++, o += nx) {
      const float t0 = tcol[r * TZS], t1 = tcol[r * TZS + 1];
      *o = (uint8_t)floorf(fmaf(255.f, fmaf(fx, t1 - t0, t0), 0.5f));
    }
  } else {
    float* o = (float*)a.img + out0;
#pragma unroll 8
    for (int r = 0; r < rows; r++, o += nx) {
      const float t0 = tcol[r * TZS], t1 = tcol[r * TZS + 1];
      *o = fmaf(fx, t1 - t0, t0);
    }
  }
  if (a.mask && f == 0)
    for (int r = 0; r < rows; r++) a.mask[(size_t)(z0 + r) * nx + x] = (colok && saz[r].i0 >= 0) ? 1 : 0;
}

// Linear 2D, direct (grids too coarse for the tiled kernel's slab): one
// pixel per thread, gathers through L1.
__global__ void __launch_bounds__(256) sc_linear_direct_kernel(const ScArgs a) {
  const size_t n = (size_t)a.nz * a.nx;
  const int f = blockIdx.y;
  for (size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (size_t)gridDim.x * blockDim.x) {
    const int iz = (int)(p / a.nx), ix = (int)(p - (size_t)iz * a.nx);
    const ScAxis ax = a.ax[ix], az = a.az[iz];
    const bool ok = ax.i0 >= 0 && az.i0 >= 0;
    float v = 0.f;
    if (ok) {
      const size_t b = ((size_t)f * a.Lx + ax.i0) * a.S + az.i0;
      const float y00 = load_y(a.line_img, a.in_type, b), y01 = load_y(a.line_img, a.in_type, b + 1);
      const float y10 = load_y(a.line_img, a.in_type, b + a.S), y11 = load_y(a.line_img, a.in_type, b + a.S + 1);
      const float t0 = fmaf(az.f, y01 - y00, y00), t1 = fmaf(az.f, y11 - y10, y10);
      v = fmaf(ax.f, t1 - t0, t0);
    }
    store_img(a.img, a.out_type, (size_t)f * n + p, v);
    if (a.mask && f == 0) a.mask[p] = ok ? 1 : 0;
  }
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
  if (!a.tiled) {
    dim3 g2(std::min<size_t>(((size_t)a.nz * a.nx + 255) / 256, 148 * 8), a.F);
    sc_linear_direct_kernel<<<g2, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  dim3 grid((a.nx + 255) / 256, (a.nz + kScRows - 1) / kScRows, a.F);
  if (a.out_type == SUPRA_T_U8) sc_linear_tiled_kernel<true><<<grid, 256, 0, st>>>(a);
  else sc_linear_tiled_kernel<false><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sc_table(const ScArgs& a, cudaStream_t st) {
  dim3 grid(a.nz * a.ny, a.F);
  sc_table_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace supra
