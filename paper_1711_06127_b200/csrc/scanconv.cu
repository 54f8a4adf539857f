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
#include <type_traits>

#include "internal.h"

namespace supra {

namespace {

__device__ __forceinline__ float load_y(const void* p, int type, size_t i) {
  if (type == SUPRA_T_U8) return (float)((const uint8_t*)p)[i] * (1.0f / 255.0f);
  return __ldg((const float*)p + i);
}

// log compression of an envelope sample against log2(ref) (finalize_kernel's
// expression; ref = 0: all-zero frame -> 0)
__device__ __forceinline__ float y_of_env(float e, float ref, float lref, float DR_k) {
  return (e > 0.f && ref > 0.f) ? fminf(fmaxf(fmaf(DR_k, lg2_approx(e) - lref, 1.f), 0.f), 1.f) : 0.f;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

__device__ __forceinline__ void store_img(void* p, int type, size_t i, float v) {
  if (type == SUPRA_T_U8) ((uint8_t*)p)[i] = (uint8_t)floorf(255.f * v + 0.5f);
  else ((float*)p)[i] = v;
}

}  // namespace

// Linear 2D, tiled and separable: one CTA per (256 output columns x
// kScRows output rows) and a group of `fpc` frames; one thread per column.
// Because u depends only on x and v only on z (reading #21), the bilinear
// blend factors into a depth lerp per (row, line) followed by a lateral lerp
// per pixel:
//   t[r][l] = lerp(y[l][k0], y[l][k0+1], fz(r)),
//   out[r][x] = lerp(t[r][i0], t[r][i0+1], fx(x)).
// The slab of the line image the tile touches (lines [l0, l0+nl) x ks
// samples from the row block's smallest k0, both host-computed) is staged in
// shared memory with one 1-D bulk copy (TMA) per line.  The CTA walks its
// frames with two slab buffers (the next frame's copies in flight while the
// current one is blended; tables read once per CTA).  Each warp does the
// depth lerp only for the few lines its 32 columns touch (lane = output
// row) into its own small buffer, so the two phases need only __syncwarp;
// a per-buffer "empty" mbarrier (8 warp arrivals) gates the refill.
constexpr int kScWarpLines = kScWarpLinesMax + 1;  // + the zero pair
// Slab elements of one buffer (as sized by launch_sc_linear): a multiple of
// 128 bytes, so both buffers are 128-byte aligned TMA destinations.
__host__ __device__ inline int sc_slab_elems(int box_l, int box_k, int slab_k, int elem_bytes) {
  const int q = 128 / elem_bytes;
  return (box_l * (box_k > slab_k ? box_k : slab_k) + q - 1) / q * q;
}
// IN8: u8 line image (log-compressed, y = v / 255), staged as bytes -- a
// quarter of the f32 slab -- by the same 2-D tensor copy.
template <bool U8OUT, bool IN8>
__global__ void __launch_bounds__(256) sc_linear_tiled_kernel(const __grid_constant__ CUtensorMap tm,
                                                              const ScArgs a, int fpc) {
  using T = typename std::conditional<IN8, uint8_t, float>::type;
  // the two slab buffers live in dynamic shared memory (the pair buffers
  // below are static; together they exceed the 48 KB static limit)
  extern __shared__ __align__(128) unsigned char slab_raw[];
  const int slab_elems = sc_slab_elems(a.slab_box_l, a.slab_box_k, a.slab_k, (int)sizeof(T));
  auto slab = [&](int b) { return reinterpret_cast<T*>(slab_raw) + b * slab_elems; };
  // per warp and output row: pairs {t(j), t(j+1) - t(j)} of the depth-lerped
  // lines (u8: t scaled to 255 t + 1/2), so a pixel is one LDS.64 + FFMA;
  // odd row stride in 8-byte units: conflict-free 64-bit row writes
  constexpr int TZS = kScWarpLines + 1;
  __shared__ float2 tzw[8][kScRows * TZS];
  __shared__ ScAxis saz[kScRows];
  __shared__ __align__(8) uint64_t full[2], empty[2];
  const int cb = blockIdx.x, rb = blockIdx.y;
  const int fbeg = blockIdx.z * fpc, fend = min(a.F, fbeg + fpc);
  const int x = cb * 256 + threadIdx.x;
  const int z0 = rb * kScRows;
  const int ks = a.slab_k;
  const int kmin = a.blk_kmin[rb];
  const int l0 = a.col_l0[cb], nl = a.col_nl[cb];
  const int Lx = a.Lx, S = a.S, nx = a.nx;
  const int rows = min(kScRows, a.nz - z0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool use_tma = a.slab_tma != 0;
  const int kstride = use_tma ? a.slab_box_k : ks;    // slab row stride (samples)
  const int kal = kmin & (IN8 ? ~15 : ~3);             // 16-byte aligned segment start
  if (threadIdx.x == 0) {
    for (int b = 0; b < 2; b++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[b])),
                   "r"(32)
                   : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[b])),
                   "r"(8)
                   : "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < rows) saz[threadIdx.x] = a.az[z0 + threadIdx.x];
  const ScAxis ax = x < nx ? a.ax[x] : ScAxis{-1, 0.f};
  // lines this warp's columns touch: [wl0, wl0 + wnl) (slab-relative)
  const bool colok = ax.i0 >= 0;
  const unsigned wlo = __reduce_min_sync(0xffffffffu, colok ? (unsigned)(ax.i0 - l0) : 0xffffffffu);
  const unsigned whi = __reduce_max_sync(0xffffffffu, colok ? (unsigned)(ax.i0 - l0 + 1) : 0u);
  const int wl0 = wlo == 0xffffffffu ? 0 : (int)wlo;
  const int wnl = wlo == 0xffffffffu ? 0 : (int)(whi - wlo + 1);  // <= kScWarpLines - 1 (checked at create)
  float2* tz = tzw[warp];
  // zero pair for invalid columns (u8: {1/2, 0} -> floor(1/2) = 0), and
  // per-column pointers
  const float2* tcol = tz + (colok ? ax.i0 - l0 - wl0 : kScWarpLines - 1);
  const float fx = colok ? ax.f : 0.f;
  for (int r = lane; r < kScRows; r += 32) tz[r * TZS + kScWarpLines - 1] = make_float2(U8OUT ? 0.5f : 0.f, 0.f);
  __syncthreads();
  auto wait = [](uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
            (uint32_t)__cvta_generic_to_shared(bar)),
        "r"(parity)
        : "memory");
  };
  // slab_tma == 2: ONE 2-D tensor copy (UTMALDG) of the box {box_k samples,
  // box_l lines} at (kal, f Lx + l0) of the [F Lx][S] line image; lines past
  // the tile's nl are staged but unused, samples/rows past the image read 0.
  // slab_tma == 1: one 1-D bulk copy (UBLKCP) per line segment
  // [kal, kal + box_k) (clipped to the record), lanes of warp 0 take lines.
  auto issue = [&](int f, int b) {
    if (a.slab_tma == 2) {
      const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&full[b]);
      const unsigned bytes =
          (lane == 0 && kmin >= 0 && nl > 0) ? (unsigned)(a.slab_box_k * a.slab_box_l * (int)sizeof(T)) : 0u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes) : "memory");
      if (bytes)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"((uint32_t)__cvta_generic_to_shared(slab(b))),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(kal), "r"(f * Lx + l0), "r"(bb)
            : "memory");
      return;
    }
    // (1-D bulk copies: f32 line images only, see run_sc)
    const float* src = (const float*)a.line_img + (size_t)f * Lx * S;
    const int seg = min(a.slab_box_k, S - kal);
    const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&full[b]);
    unsigned bytes = 0;
    for (int l = lane; l < nl && kmin >= 0; l += 32) bytes += (unsigned)seg * 4u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(bytes) : "memory");
    for (int l = lane; l < nl && kmin >= 0; l += 32)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              (uint32_t)__cvta_generic_to_shared(reinterpret_cast<float*>(slab(b)) + l * a.slab_box_k)),
          "l"(src + (size_t)(l0 + l) * S + kal), "r"((unsigned)seg * 4u), "r"(bb)
          : "memory");
  };
  if (use_tma && warp == 0 && fbeg < fend) issue(fbeg, 0);
  const ScAxis az = saz[lane < rows ? lane : 0];
  for (int f = fbeg; f < fend; f++) {
    const int it = f - fbeg, b = use_tma ? (it & 1) : 0;
    if (use_tma) {
      // refill the other buffer with the next frame once every warp has
      // finished its depth lerp on it (previous iteration)
      if (warp == 0 && f + 1 < fend) {
        if (it >= 1) wait(&empty[b ^ 1], (unsigned)(((it - 1) >> 1) & 1));
        issue(f + 1, b ^ 1);
      }
      wait(&full[b], (unsigned)((it >> 1) & 1));
    } else {
      if (it > 0) __syncthreads();  // every warp is done with slab(0)
      if (kmin >= 0 && nl > 0) {
        const size_t fbase = (size_t)f * Lx * S;
        if constexpr (!IN8) {
          const float* src = (const float*)a.line_img + fbase;
          for (int l = warp; l < nl; l += 8)
            for (int kk = lane; kk < ks; kk += 32)
              cp_async4(slab(0) + l * ks + kk, src + (size_t)(l0 + l) * S + min(kmin + kk, S - 1));
          asm volatile("cp.async.commit_group;\ncp.async.wait_all;" ::: "memory");
        } else {
          const uint8_t* src = (const uint8_t*)a.line_img + fbase;
          for (int l = warp; l < nl; l += 8)
            for (int kk = lane; kk < ks; kk += 32) slab(0)[l * ks + kk] = src[(size_t)(l0 + l) * S + min(kmin + kk, S - 1)];
        }
      }
      __syncthreads();
    }
    // depth lerp of this warp's lines: lane = output row; rows without a
    // valid k0 are zero.  With frame_max the slab holds the envelope and each
    // corner is log-compressed first (y_of_env).
    float ref = 0.f, lref = 0.f;
    if (a.frame_max) {
      ref = __uint_as_float(a.frame_max[f]);
      lref = ref > 0.f ? lg2_approx(ref) : 0.f;
    }
    // (rows without a valid k0 read the slab's first samples and select 0:
    // every read stays inside the slab, the loop has no divergent branch)
    const bool rowok = lane < rows && az.i0 >= 0;
    const T* py = slab(b) + wl0 * kstride + (rowok ? az.i0 - (use_tma ? kal : kmin) : 0);
    float2* pt = tz + lane * TZS;
    float tprev = 0.f;
    // u8 samples: y = fl(v fl(1/255)) (load_y's expression), rounded on its
    // own (no contraction into the lerp), as if staged from an f32 image
    auto yv = [](T v) { return IN8 ? __fmul_rn((float)v, 1.0f / 255.0f) : (float)v; };
    if (!IN8 && a.frame_max) {
      for (int j = 0; j < wnl; j++, py += kstride) {
        const float y0 = y_of_env(yv(py[0]), ref, lref, a.DR_k), y1 = y_of_env(yv(py[1]), ref, lref, a.DR_k);
        float t = rowok ? fmaf(az.f, y1 - y0, y0) : 0.f;
        if (U8OUT) t = fmaf(255.f, t, 0.5f);
        if (j > 0 && lane < rows) pt[j - 1] = make_float2(tprev, t - tprev);
        tprev = t;
      }
    } else {
      for (int j = 0; j < wnl; j++, py += kstride) {
        const float y0 = yv(py[0]), y1 = yv(py[1]);
        float t = rowok ? fmaf(az.f, y1 - y0, y0) : 0.f;
        if (U8OUT) t = fmaf(255.f, t, 0.5f);
        if (j > 0 && lane < rows) pt[j - 1] = make_float2(tprev, t - tprev);
        tprev = t;
      }
    }
    __syncwarp();
    if (use_tma && lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[b]))
                   : "memory");
    if (x < nx) {
      const size_t out0 = ((size_t)f * a.nz + z0) * nx + x;
      if (U8OUT) {
        // u8 = floor(255 y + 1/2) (reading #20) by the magic-number floor
        // (FADD.RM on the full-rate FP32 pipe; F2I is quarter rate): the
        // low byte of the float bits of fl(255y + 1/2) + 1.5 2^23, rounded
        // toward -inf, is the integer
        uint8_t* o = (uint8_t*)a.img + out0;
#pragma unroll 8
        for (int r = 0; r < rows; r++, o += nx) {
          const float2 t = tcol[r * TZS];  // {255 t0 + 1/2, 255 (t1 - t0)}
          *o = (uint8_t)__float_as_uint(__fadd_rd(fmaf(fx, t.y, t.x), 12582912.0f));
        }
      } else {
        float* o = (float*)a.img + out0;
#pragma unroll 8
        for (int r = 0; r < rows; r++, o += nx) {
          const float2 t = tcol[r * TZS];  // {t0, t1 - t0}
          *o = fmaf(fx, t.y, t.x);
        }
      }
      if (a.mask && f == 0)
        for (int r = 0; r < rows; r++) a.mask[(size_t)(z0 + r) * nx + x] = (colok && saz[r].i0 >= 0) ? 1 : 0;
    }
    __syncwarp();  // this warp's tz is free for the next frame
  }
}

// Linear 2D, direct (grids too coarse for the tiled kernel's slab): one
// pixel per thread, gathers through L1.
__global__ void __launch_bounds__(256) sc_linear_direct_kernel(const ScArgs a) {
  const size_t n = (size_t)a.nz * a.nx;
  const int f = blockIdx.y;
  const float ref = a.frame_max ? __uint_as_float(a.frame_max[f]) : 0.f;
  const float lref = ref > 0.f ? lg2_approx(ref) : 0.f;
  auto load_y = [&](const void* p, int type, size_t i) {
    const float v = ::supra::load_y(p, type, i);
    return a.frame_max ? y_of_env(v, ref, lref, a.DR_k) : v;
  };
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

// u32 -> f32 on the full-rate ALU path (I2FP.F32.U32); the compiler's
// choice for values it knows to be 8/16-bit, I2F.U16, runs at quarter rate.
__device__ __forceinline__ float u2f(uint32_t x) {
  float y;
  asm("cvt.rn.f32.u32 %0, %1;" : "=f"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

// Sector 2D / pyramid 3D: each warp walks output rows (iz, iy) with a
// stride of the grid's warp count, for a group of `fpc` frames per CTA.
// Over the row's valid column range [xlo, xhi) lane l takes
// x = x0 + 32 j + l (j < 4: coalesced 8-byte entry loads and output
// stores); the columns outside it are written as zeros.  Each entry is read
// ONCE and applied to every frame of the group, so a frame costs the corner
// gathers of the L2-resident line image, the blend and the store.  While a
// row is blended the next row's record is loaded and its entry span
// bulk-prefetched into L2 (the entry loads were the DRAM-latency stall:
// long-scoreboard on the first use of each entry, ~18 % of samples).
// Offsets within a frame are 32-bit (L * S < 2^31, checked at create).
// Measured (C4p, u8 line image): latency-bound on the corner gathers
// (long-scoreboard 45 % of the stall samples), not by DRAM (22 %); staging
// the entries in shared memory (bulk copies, per-warp double buffers or
// per-CTA row blocks) and z-major warp tiles were slower.
__device__ __forceinline__ void l2_prefetch_span(const void* p, uint32_t bytes) {
  const uintptr_t a0 = (uintptr_t)p & ~(uintptr_t)15;
  const uint32_t n = (uint32_t)((((uintptr_t)p + bytes + 15) & ~(uintptr_t)15) - a0);
  if (n)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"(n) : "memory");
}

template <int IN_T, int OUT_T, bool IS3D, bool LOGLOAD>
__global__ void __launch_bounds__(256, 4) sc_table_kernel(const ScArgs a, int fpc) {
  constexpr int V = 4;  // voxels per lane and chunk
  const int lane = threadIdx.x & 31;
  const int nrows = a.nz * a.ny;
  const int rstride = gridDim.x * 8;
  int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= nrows) return;
  const int f0 = blockIdx.y * fpc, f1 = min(a.F, f0 + fpc);
  auto prefetch_row = [&](const ScRow& q) {
    if (lane == 0 && q.xhi > q.xlo)
      l2_prefetch_span(reinterpret_cast<const uint2*>(a.ent) + q.off, (uint32_t)(q.xhi - q.xlo) * 8u);
  };
  ScRow nrow = a.rows[r];
  prefetch_row(nrow);
  ScRow nnrow = r + rstride < nrows ? a.rows[r + rstride] : nrow;
  for (; r < nrows; r += rstride) {
    const ScRow row = nrow;
    if (r + rstride < nrows) {
      // next row: its entries into L2 now; the record after it loads while
      // this row is blended
      nrow = nnrow;
      prefetch_row(nrow);
      if (r + 2 * rstride < nrows) nnrow = a.rows[r + 2 * rstride];
    }
    const uint32_t S = (uint32_t)a.S, LS = (uint32_t)a.Lx * S;
    const size_t fstride = (size_t)a.Ly * LS;  // line-image elements per frame
    const size_t ostride = (size_t)a.nz * a.ny * a.nx;
    const float fy = row.fy;
    using InT = typename std::conditional<IN_T == SUPRA_T_U8, uint8_t, float>::type;
    // u8 line images are blended as integers 0..255 (exact in f32) and scaled
    // by 1/255 once at the end
    constexpr float kInScale = IN_T == SUPRA_T_U8 ? 1.0f / 255.0f : 1.0f;
    const uint2* rent = reinterpret_cast<const uint2*>(a.ent) + row.off - row.xlo;  // entry of column x: rent[x]
    // columns outside the row's valid range [xlo, xhi): zeros (and mask 0)
    {
      const int xlo = max(0, min(row.xlo, a.nx)), xhi = max(xlo, min(row.xhi, a.nx));
      for (int f = f0; f < f1; f++) {
        const size_t ob = (size_t)f * ostride + (size_t)r * a.nx;
        for (int x = lane; x < xlo; x += 32) {
          if constexpr (OUT_T == SUPRA_T_U8) ((uint8_t*)a.img)[ob + x] = 0;
          else ((float*)a.img)[ob + x] = 0.f;
        }
        for (int x = xhi + lane; x < a.nx; x += 32) {
          if constexpr (OUT_T == SUPRA_T_U8) ((uint8_t*)a.img)[ob + x] = 0;
          else ((float*)a.img)[ob + x] = 0.f;
        }
      }
      if (a.mask && f0 == 0) {
        for (int x = lane; x < xlo; x += 32) a.mask[(size_t)r * a.nx + x] = 0;
        for (int x = xhi + lane; x < a.nx; x += 32) a.mask[(size_t)r * a.nx + x] = 0;
      }
    }
    // the valid range, in chunks of 32 V columns
    const int xend = min(row.xhi, a.nx);
    for (int x0 = max(0, row.xlo); x0 < xend; x0 += 32 * V) {
      uint32_t base[V];
      float fx[V], fz[V];
  #pragma unroll
      for (int j = 0; j < V; j++) {
        const int x = x0 + 32 * j + lane;
        base[j] = kScInvalid;
        uint32_t q = 0u;
        if (x >= row.xlo && x < row.xhi) {
          const uint2 e = __ldg(rent + x);
          base[j] = e.x;
          q = e.y;
        }
        fx[j] = u2f(q & 0xFFFFu) * (1.0f / 65535.0f);
        fz[j] = u2f(q >> 16) * (1.0f / 65535.0f);
        if (a.mask && f0 == 0 && x < xend) a.mask[(size_t)r * a.nx + x] = base[j] != kScInvalid ? 1 : 0;
      }
      for (int f = f0; f < f1; f++) {
        float ref = 0.f, lref = 0.f;
        if constexpr (LOGLOAD) {
          ref = __uint_as_float(a.frame_max[f]);
          lref = ref > 0.f ? lg2_approx(ref) : 0.f;
        }
        const InT* lf = (const InT*)a.line_img + (size_t)f * fstride;
        auto ld = [&](const InT* p) {
          float y;
          if constexpr (IN_T == SUPRA_T_U8) y = u2f(__ldg(p));
          else y = __ldg(p);
          if constexpr (LOGLOAD) y = y_of_env(y, ref, lref, a.DR_k);
          return y;
        };
        const size_t ob = (size_t)f * ostride + (size_t)r * a.nx;
  #pragma unroll
        for (int j = 0; j < V; j++) {
          const int x = x0 + 32 * j + lane;
          float v = 0.f;
          if (base[j] != kScInvalid) {
            const InT* p0 = lf + base[j];  // corner (i0x, i0y, k0)
            const InT* p1 = p0 + S;        // (i0x + 1, i0y, k0)
            const float t0 = lerpf(ld(p0), ld(p0 + 1), fz[j]);
            const float t1 = lerpf(ld(p1), ld(p1 + 1), fz[j]);
            v = lerpf(t0, t1, fx[j]);
            if constexpr (IS3D) {
              const InT* p2 = p0 + LS;  // (i0x, i0y + 1, k0)
              const InT* p3 = p2 + S;
              const float t2 = lerpf(ld(p2), ld(p2 + 1), fz[j]);
              const float t3 = lerpf(ld(p3), ld(p3 + 1), fz[j]);
              v = lerpf(v, lerpf(t2, t3, fx[j]), fy);
            }
            v *= kInScale;
          }
          if (x < xend) {
            // u8 = floor(255 v + 1/2) by the magic-number floor (FADD.RM; the
            // F2I conversion runs at quarter rate)
            if constexpr (OUT_T == SUPRA_T_U8)
              ((uint8_t*)a.img)[ob + x] = (uint8_t)__float_as_uint(__fadd_rd(fmaf(255.f, v, 0.5f), 12582912.0f));
            else ((float*)a.img)[ob + x] = v;
          }
        }
      }
    }
  }  // rows
}

cudaError_t launch_sc_linear(const ScArgs& a, const CUtensorMap* slab_map, cudaStream_t st) {
  if (!a.tiled) {
    dim3 g2(std::min<size_t>(((size_t)a.nz * a.nx + 255) / 256, 148 * 8), a.F);
    sc_linear_direct_kernel<<<g2, 256, 0, st>>>(a);
    return cudaGetLastError();
  }
  // frames per CTA: enough CTAs for ~8 waves of 148 SMs x 4 resident,
  // the rest of the frames walked by each CTA with double-buffered staging
  const long tiles = (long)((a.nx + 255) / 256) * ((a.nz + kScRows - 1) / kScRows);
  // (C2, 2-D TMA slab, us per 100 frames: 4 waves 191, 8: 187, 16: 189, 32: 207)
  const long want = 148L * 4 * 8;
  int fpc = (int)std::max<long>(1, (tiles * a.F + want - 1) / want);
  fpc = std::min(fpc, a.F);
  dim3 grid((a.nx + 255) / 256, (a.nz + kScRows - 1) / kScRows, (a.F + fpc - 1) / fpc);
  CUtensorMap none{};
  const CUtensorMap& tm = slab_map ? *slab_map : none;
  const bool in8 = a.in_type == SUPRA_T_U8;
  const size_t smem =
      2 * (size_t)sc_slab_elems(a.slab_box_l, a.slab_box_k, a.slab_k, in8 ? 1 : 4) * (in8 ? 1 : 4);
  auto go = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, st>>>(tm, a, fpc);
  };
  if (a.out_type == SUPRA_T_U8) in8 ? go(sc_linear_tiled_kernel<true, true>) : go(sc_linear_tiled_kernel<true, false>);
  else in8 ? go(sc_linear_tiled_kernel<false, true>) : go(sc_linear_tiled_kernel<false, false>);
  return cudaGetLastError();
}

template <int IN_T, int OUT_T, bool IS3D, bool LG>
static cudaError_t launch_tab(const ScArgs& a, int line_img_bytes_per_frame, cudaStream_t st) {
  // frames per CTA: every table entry is read once per group while the
  // group's line images stay L2-resident (<= 48 MB of the 126 MB L2); the
  // grid keeps >= 2 waves of 4 CTAs per SM
  const long tiles = ((long)a.nz * a.ny + 7) / 8;
  const long cap = std::max<long>(1, (48L << 20) / std::max(1, line_img_bytes_per_frame));
  const long fill = std::max<long>(1, tiles * a.F / (148L * 4 * 2));
  const int fpc = (int)std::min<long>({(long)a.F, cap, fill, 16L});
  // each warp walks ~4 rows (the next row's entries prefetched into L2
  // while the current one is blended), at least 2 waves of 4 CTAs per SM
  const long ctas = std::min<long>(tiles, std::max<long>(148L * 4 * 2, (tiles + 3) / 4));
  dim3 grid((unsigned)ctas, (a.F + fpc - 1) / fpc);
  sc_table_kernel<IN_T, OUT_T, IS3D, LG><<<grid, 256, 0, st>>>(a, fpc);
  return cudaGetLastError();
}

template <int IN_T, int OUT_T, bool IS3D>
static cudaError_t launch_tab_lg(const ScArgs& a, int bytes, cudaStream_t st) {
  return a.frame_max ? launch_tab<IN_T, OUT_T, IS3D, true>(a, bytes, st)
                     : launch_tab<IN_T, OUT_T, IS3D, false>(a, bytes, st);
}

cudaError_t launch_sc_table(const ScArgs& a, int bytes, cudaStream_t st) {
  const bool u8in = a.in_type == SUPRA_T_U8, u8out = a.out_type == SUPRA_T_U8;
  if (a.is3d) {
    if (u8in) return u8out ? launch_tab_lg<SUPRA_T_U8, SUPRA_T_U8, true>(a, bytes, st)
                           : launch_tab_lg<SUPRA_T_U8, SUPRA_T_F32, true>(a, bytes, st);
    return u8out ? launch_tab_lg<SUPRA_T_F32, SUPRA_T_U8, true>(a, bytes, st)
                 : launch_tab_lg<SUPRA_T_F32, SUPRA_T_F32, true>(a, bytes, st);
  }
  if (u8in) return u8out ? launch_tab_lg<SUPRA_T_U8, SUPRA_T_U8, false>(a, bytes, st)
                         : launch_tab_lg<SUPRA_T_U8, SUPRA_T_F32, false>(a, bytes, st);
  return u8out ? launch_tab_lg<SUPRA_T_F32, SUPRA_T_U8, false>(a, bytes, st)
               : launch_tab_lg<SUPRA_T_F32, SUPRA_T_F32, false>(a, bytes, st);
}

}  // namespace supra
