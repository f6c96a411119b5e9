// sconv_1x1.cuh — 1x1 sparse convolution (stride 1, no padding) for sm_100a.
//
// What it computes: Alg.2 of the paper for K = 1, where the
// stretched column index is c*H*W and the convolution is the sparse x dense
// product out[n][m][p] = act(bias[m] + sum_c W[m][c] * x[n][c][p]) (the SpMM
// special case, SURVEY 8(c) "1x1, s=1, p=0 equals a sparse x dense matmul").
//
// How: a 1x1 filter has no spatial window to keep in
// registers, so the per-nonzero dispatch of sconv_tiled has nothing to
// amortise.  Instead each warp owns R output channels x (32 lanes x V pixels)
// and walks, in ascending c, the input channels where ANY of its R rows has a
// nonzero (records {byte offset of x[c] in the slab, w[0..R-1]}, zeros for the
// rows without one).  Per record: V/4 LDS.128 of x + R*V FFMA, no branches.
// Multiplying by an explicit 0.0f leaves every accumulator bitwise unchanged
// (acc is never -0: it starts at +0 and x is finite), so each row still sees
// exactly its CSR terms in ascending c — the same bits as every other variant.
//   * Pixels are flattened over the batch (g = n*HW + p): a CTA tile is TP =
//     32*V*WP consecutive pixels, so small images waste no lanes.
//   * The input tile [CC][TP] of each channel chunk is staged by cp.async
//     (16-byte copies when HW % 4 == 0) through an NS-stage mbarrier pipeline.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "escoin_internal.h"
#include "sconv_tiled.cuh"

namespace escoin {

__device__ __forceinline__ void cp_async16z(unsigned dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}

// SPARSE = 0: row blocks (records per visited channel, R weights each, zeros
// included).  SPARSE = 1: exact row lists — per warp and chunk a header of R
// counts, then for each of the R rows its nonzeros {byte offset, w} in
// ascending c; each nonzero costs V/4 LDS.128 + V FFMA and nothing is wasted
// (shared-memory bound at ~25% of the FFMA peak: one x load per FMA).
// VW-wide vector loads/stores (VW = 4, 2, 1).
template <int VW>
__device__ __forceinline__ void lds_vec(float (&d)[VW], const char* p) {
  if constexpr (VW == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    d[0] = t.x, d[1] = t.y, d[2] = t.z, d[3] = t.w;
  } else if constexpr (VW == 2) {
    const float2 t = *reinterpret_cast<const float2*>(p);
    d[0] = t.x, d[1] = t.y;
  } else {
    d[0] = *reinterpret_cast<const float*>(p);
  }
}
template <int VW>
__device__ __forceinline__ void stg_vec(float* p, const float (&v)[VW]) {
  if constexpr (VW == 4) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  else if constexpr (VW == 2) *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  else *p = v[0];
}

template <int R, int V, int MINB, int TAG, int SPARSE>
__global__ void __launch_bounds__(kTiledThreads, MINB) sconv1x1_kernel(const TiledArgs a) {
  // lane pixels: V4 groups of VW consecutive pixels; group j of lane l at tile
  // offset wp*32*V + j*32*VW + l*VW (each group load is one coalesced LDS)
  constexpr int VW = V >= 4 ? 4 : V;
  constexpr int V4 = V / VW;
  constexpr int GB = 32 * VW * 4;  // bytes between a lane's groups
  constexpr int RS4 = (1 + R + 3) / 4;  // int4 units per record

  extern __shared__ __align__(16) float smem[];
  __shared__ __align__(8) unsigned long long bars[2 * kMaxStages];
  const int NS = a.NS;
  int2* const recbase = reinterpret_cast<int2*>(smem + NS * a.stage_floats);
  const unsigned full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[kMaxStages]);

  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % a.WM, wp = warp / a.WM;
  const int HW = a.H * a.W;
  const int64_t npix = static_cast<int64_t>(a.N) * HW;
  const int64_t g0 = static_cast<int64_t>(blockIdx.y) * a.TP;  // first (flat) pixel of the tile
  const int TP4 = a.TP / 4;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8u * s, kTiledThreads);
      mbar_init(empty0 + 8u * s, kTiledThreads / 32);
    }
  }
  __syncthreads();

  const int* const sched = a.sched + static_cast<int64_t>(a.sched_off[b]) * a.sched_stride;
  const int nact = a.sched_off[b + 1] - a.sched_off[b];

  // Staging map: the tile's pixels are QN units (16-byte groups when HW % 4 ==
  // 0, else single floats); QN is a power of two.  Thread t owns unit
  // q = t % QN (+ 256 k when QN > 256) for channel rows t / QN + k * 256 / QN,
  // so the (image, pixel) split of its units — 64-bit divisions — is done
  // once here, not per chunk.
  const int U = a.vec16 ? 4 : 1;  // floats per unit
  const int QN = a.TP / U;
  constexpr int kMaxQ = 4;        // units per thread when QN > 256
  const int nq = QN > kTiledThreads ? QN / kTiledThreads : 1;
  const int cl0 = QN >= kTiledThreads ? 0 : threadIdx.x / QN, cl_step = QN >= kTiledThreads ? 1 : kTiledThreads / QN;
  int64_t qbase[kMaxQ];  // element offset of (n, p) in the input (channel 0), or -1 past the batch
#pragma unroll
  for (int k = 0; k < kMaxQ; ++k) {
    const int64_t g = g0 + static_cast<int64_t>((threadIdx.x % QN) + k * kTiledThreads) * U;
    const int64_t n = g / HW;
    qbase[k] = (k < nq && g < npix) ? n * a.C * HW + (g - n * HW) : -1;
  }

  // Stage chunk ai: x[n][c0 + cl][p] for the tile's pixels -> slab[cl][g - g0]
  // (zero beyond the batch / beyond C), and the chunk's records.
  auto stage = [&](int ai) {
    const int st = ai % NS;
    if (ai >= NS) mbar_wait(empty0 + 8u * st, ((ai / NS) - 1) & 1);
    const int* e = sched + ai * a.sched_stride;
    const int c0 = e[0] * a.CC, rs = e[1], rc = e[2];
    const int ncl = min(a.CC, a.C - c0);
    const unsigned sb = smem_addr(smem + st * a.stage_floats);
#pragma unroll
    for (int k = 0; k < kMaxQ; ++k) {
      if (k >= nq) break;
      const int q = (threadIdx.x % QN) + k * kTiledThreads;
      for (int cl = cl0; cl < a.CC; cl += cl_step) {
        const bool ok = cl < ncl && qbase[k] >= 0;
        const float* src = ok ? a.in + qbase[k] + static_cast<int64_t>(c0 + cl) * HW : a.in;
        const unsigned dst = sb + 4u * static_cast<unsigned>(cl * a.TP + q * U);
        if (a.vec16) cp_async16z(dst, src, ok ? 16 : 0);
        else cp_async4(dst, src, ok ? 4 : 0);
      }
    }
    const unsigned rb = smem_addr(recbase + st * a.stage_recs);
    for (int i = threadIdx.x; i < (rc >> 1); i += kTiledThreads) cp_async16(rb + 16u * i, a.recs + rs + 2 * i);
    cp_async_arrive(full0 + 8u * st);
  };

  float acc[R][V];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int v = 0; v < V; ++v) acc[r][v] = 0.0f;

  const int lane_off = wp * 32 * V + lane * VW;
  if (nact > 0) stage(0);
  for (int ai = 0; ai < nact; ++ai) {
    const int st = ai % NS;
    if (ai + 1 < nact) stage(ai + 1);
    mbar_wait(full0 + 8u * st, (ai / NS) & 1);
    const char* xs = reinterpret_cast<const char*>(smem + st * a.stage_floats + lane_off);
    if constexpr (SPARSE) {
      const int* hdr = reinterpret_cast<const int*>(recbase + st * a.stage_recs + sched[ai * a.sched_stride + 3 + wm]);
      const int2* e = reinterpret_cast<const int2*>(hdr + 4 * ((R + 3) / 4));
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int n = hdr[r];
        auto term = [&](int2 t, float (&x)[V4][VW]) {
          const float w = __int_as_float(t.y);
#pragma unroll
          for (int j = 0; j < V4; ++j)
#pragma unroll
            for (int k = 0; k < VW; ++k) acc[r][VW * j + k] = fmaf(w, x[j][k], acc[r][VW * j + k]);
        };
        // two terms per step: both loads first (independent), then the FMAs in
        // ascending c (the accumulation order of every variant)
        int i = 0;
#pragma unroll 1
        for (; i + 2 <= n; i += 2) {
          const int2 t0 = e[i], t1 = e[i + 1];
          float x0[V4][VW], x1[V4][VW];
#pragma unroll
          for (int j = 0; j < V4; ++j) {
            lds_vec<VW>(x0[j], xs + t0.x + GB * j);
            lds_vec<VW>(x1[j], xs + t1.x + GB * j);
          }
          term(t0, x0);
          term(t1, x1);
        }
        if (i < n) {
          const int2 t0 = e[i];
          float x0[V4][VW];
#pragma unroll
          for (int j = 0; j < V4; ++j) lds_vec<VW>(x0[j], xs + t0.x + GB * j);
          term(t0, x0);
        }
        e += n;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8u * st);
      continue;
    }
    const int4* rp = reinterpret_cast<const int4*>(recbase + st * a.stage_recs + sched[ai * a.sched_stride + 3 + wm]);
    const int cnt = rp[0].x;
    rp += 1;
#pragma unroll 2
    for (int i = 0; i < cnt; ++i) {
      float w[RS4 * 4];
#pragma unroll
      for (int k = 0; k < RS4; ++k) {
        const int4 t = rp[k];
        w[4 * k + 0] = __int_as_float(t.x);
        w[4 * k + 1] = __int_as_float(t.y);
        w[4 * k + 2] = __int_as_float(t.z);
        w[4 * k + 3] = __int_as_float(t.w);
      }
      const int off = __float_as_int(w[0]);  // byte offset of channel row c_local in the slab
      rp += RS4;
#pragma unroll
      for (int j = 0; j < V4; ++j) {
        float x[VW];
        lds_vec<VW>(x, xs + off + GB * j);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int k = 0; k < VW; ++k) acc[r][VW * j + k] = fmaf(w[1 + r], x[k], acc[r][VW * j + k]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8u * st);
  }

  // Epilogue (reading R#10): v = acc + bias[m]; ReLU; NCHW store.
  if (a.debug & 4 && acc[0][0] != 12345.0f) return;
  int64_t obase[V4];  // output offset of group j for channel 0 (vec16), -1 past the batch
#pragma unroll
  for (int j = 0; j < V4; ++j) {
    const int64_t g = g0 + lane_off + 32 * VW * j;
    const int64_t n = g / HW;
    obase[j] = g < npix ? n * a.M * HW + (g - n * HW) : -1;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int m = (b * a.WM + wm) * R + r;
    if (m >= a.M) break;
    const float bv = a.bias ? __ldg(a.bias + m) : 0.0f;
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const int64_t g = g0 + lane_off + 32 * VW * j;
      float v[VW];
#pragma unroll
      for (int k = 0; k < VW; ++k) {
        v[k] = __fadd_rn(acc[r][VW * j + k], bv);
        if (a.relu) v[k] = v[k] > 0.0f ? v[k] : 0.0f;
      }
      if (a.vec16) {  // HW % 4 == 0: a group never straddles two images
        if (obase[j] >= 0) stg_vec<VW>(a.out + obase[j] + static_cast<int64_t>(m) * HW, v);
      } else {
#pragma unroll
        for (int k = 0; k < VW; ++k) {
          if (g + k < npix) {
            const int64_t n = (g + k) / HW, p = g + k - n * HW;
            a.out[(n * a.M + m) * HW + p] = v[k];
          }
        }
      }
    }
  }
}

template <int R, int V, int MINB, int TAG, int SPARSE>
int launch_1x1(const TiledArgs& a, cudaStream_t s) {
  auto kern = sconv1x1_kernel<R, V, MINB, TAG, SPARSE>;
  if (a.smem_bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  dim3 grid(a.B, a.ntiles);
  kern<<<grid, kTiledThreads, a.smem_bytes, s>>>(a);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace escoin
