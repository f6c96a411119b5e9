// sconv_tiled.cuh — register-tiled direct sparse convolution for sm_100a.
//
// What it computes: Alg.2 of the paper with dynamic indexing
// (§3.1), stride and virtual zero padding, bias + ReLU fused:
//   out[n][m][oh][ow] = act(bias[m] + sum_{j in row m} value[j] *
//                            X~[n][colidx[j] + oh*S*Wp + ow*S])
// How:
//   * CTA = (m-block of WM groups x Q output channels) x (pixel tile of NB
//     images x TR patch-rows x all PC patch-columns).  Warp (wm, wp): output
//     channels of group wm, pixel slots [32 wp, 32 wp + 32).  Lane = one
//     PH x PW output patch.  All lanes of a warp walk the same records, so
//     every branch is warp-uniform (the paper's "avoid unstructured
//     computation") and weights are smem broadcasts.
//   * Input channels are processed in chunks of CC; for each chunk the CTA
//     stages the zero-padded input slab [NB][CC][SR][SCs] (pad_in fused into
//     the load via cp.async zero-fill, P:705 / reading R#9) and the chunk's
//     records into shared memory, double-buffered.
//   * Per input channel c each lane loads its XH x XW input window into
//     registers once (vector LDS), then runs the bucket of records of
//     (group, c): each record = one nonzero weight, dispatched by code
//     q*K*K + kh*K + kw to PH*PW FFMAs on compile-time registers
//     (bucket_loop, generated inline PTX).  Partial sums stay in registers
//     for the whole reduction.
//   * Accumulation order per output channel: ascending (c, kh, kw) ==
//     ascending colidx, from 0.0f, fp32 FMA — identical to the paper-mapping
//     kernel, hence bitwise-identical results across variants.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "escoin_internal.h"

namespace escoin {

// Runs a warp's whole record stream of one channel chunk (mode 0): records
// dispatch FFMA blocks; NEXT records reload the window registers x from
// wbase + payload (row stride rowb bytes); DONE returns.
template <int K, int S, int PH, int PW, int Q, int TAG>
__device__ void chunk_loop(float* acc, float* x, unsigned& p, unsigned wbase, unsigned rowb);

// Mode 3: same stream as mode 0; every lane computes its patch for TWO images
// (an image pair interleaved in shared memory), one FFMA2 per pixel with the
// weight as a broadcast operand — no register duplication.
template <int K, int S, int PH, int PW, int Q, int TAG>
__device__ void chunk_loop3(unsigned long long* acc, unsigned long long* x, unsigned& p, unsigned wbase,
                            unsigned rowb);

// Mode 2: same stream as mode 0, FFMA2 on horizontal output-pixel pairs.
template <int K, int S, int PH, int PW, int Q, int TAG>
__device__ void chunk_loop2(unsigned long long* acc, unsigned long long* x, unsigned& p, unsigned wbase,
                            unsigned rowb);

// Dense-bucket sweep (mode 1): wp = shared address of the bucket's Q*K*K
// weights in (tap, q) order, zeros for absent taps.
template <int K, int S, int PH, int PW, int Q, int TAG>
__device__ void bucket_mask(float* acc, const float* x, unsigned wp);

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async4(unsigned dst, const void* src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// Completion of this thread's outstanding cp.async copies counts as one
// arrival on the mbarrier (whose expected count covers every thread).
__device__ __forceinline__ void cp_async_arrive(unsigned bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

template <int K, int S, int PH, int PW, int Q, int MINB, int MODE, int TAG>
__global__ void __launch_bounds__(kTiledThreads, MINB) sconv_tiled_kernel(const TiledArgs a) {
  constexpr int P = PH * PW;
  constexpr int XH = (PH - 1) * S + K, XW = (PW - 1) * S + K;
  // Vector (LDS.128) window loads need every lane's window to start on a
  // 16-byte boundary: true when PW*S is a multiple of 4, or when a patch spans
  // the whole row (PC == 1, all windows start at column 0).
  constexpr bool VEC_ALWAYS = ((PW * S) % 4) == 0;
  constexpr int XWV = (XW + 3) / 4;
  constexpr int IP = MODE == 3 ? 2 : 1;  // images per lane (interleaved innermost in smem)

  // NS stages of {input slab, records}; stage s: slab smem + s*stage_floats,
  // records recbase + s*stage_recs.  full[s]: the chunk's copies landed (one
  // cp.async arrival per thread); empty[s]: every warp finished reading it.
  extern __shared__ __align__(16) float smem[];
  __shared__ __align__(8) unsigned long long bars[2 * kMaxStages];
  const int NS = a.NS;
  int2* const recbase = reinterpret_cast<int2*>(smem + NS * a.stage_floats);
  const unsigned full0 = smem_addr(&bars[0]), empty0 = smem_addr(&bars[kMaxStages]);

  const int b = blockIdx.x;
  const int tile = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % a.WM, wp = warp / a.WM;
  const int slot = wp * 32 + lane;
  int n0, pr0, img, pr, pc;
  if (a.flat) {
    // flat: slots enumerate (image, patch-row) pairs; this CTA owns 32*WP of them
    const int g0 = tile * a.WP * 32, g = g0 + slot;
    n0 = g0 / a.PR;
    pr0 = 0;
    img = g / a.PR - n0;
    pr = g - (g / a.PR) * a.PR;
    pc = 0;
  } else {
    n0 = (tile / a.tiles_r) * a.NB * IP;  // a.NB counts image groups of IP images
    pr0 = (tile % a.tiles_r) * a.TR;
    const int per_img = a.TR * a.PCs;
    img = slot / per_img;
    pr = (slot - img * per_img) / a.PCs;
    pc = slot - img * per_img - pr * a.PCs;
  }
  const bool active = (img < a.NB) && (n0 + img * IP < a.N) && (pr0 + pr < a.PR) && (pc < a.PC);
  if (pc >= a.PC) pc = a.PC - 1;  // pad lanes re-read a neighbour's window: a broadcast, not a bank conflict
  if (!(img < a.NB) || !(n0 + img * IP < a.N) || !(pr0 + pr < a.PR)) { img = 0; pr = 0; pc = 0; }
  const int win_off = img * a.CC * a.plane + pr * PH * S * a.SCs + pc * PW * S * IP;

  // Staging map (pad_in fused, reading R#9).  Every slab cell outside the
  // real input (padding ring, rows beyond the image) is zeroed once below and
  // never written again; per chunk only the interior rows are copied.  The
  // interior of one plane is a CONTIGUOUS run of nrow*W floats in the NCHW
  // input (rows y0 .. y0+nrow-1), so element e of that run goes to smem cell
  // (r_lo + e / W) * SCs + pad + e % W; each thread owns e = tid + i*256 and
  // copies it for every (image, channel) plane of the chunk.
  const int y_first = pr0 * PH * S - a.pad;               // global row of slab row 0
  const int r_lo = y_first < 0 ? -y_first : 0;            // first interior slab row
  const int y0 = y_first + r_lo;                          // its global row (>= 0)
  const int nrow = max(0, min(a.SR - r_lo, a.H - y0));    // interior rows in the slab
  const int nint = nrow * a.W;                            // interior floats per plane
  {
    float4* z = reinterpret_cast<float4*>(smem);
    for (int i = threadIdx.x; i < (NS * a.stage_floats) / 4; i += kTiledThreads) z[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full0 + 8u * s, kTiledThreads);
      mbar_init(empty0 + 8u * s, kTiledThreads / 32);
    }
  }
  __syncthreads();

  const int* const sched = a.sched + static_cast<int64_t>(a.sched_off[b]) * a.sched_stride;
  const int nact = a.sched_off[b + 1] - a.sched_off[b];
  const int64_t HW = static_cast<int64_t>(a.H) * a.W;

  // Stage chunk ai into buffer ai % NS (after every warp released the chunk
  // that used it before), then arrive on full[ai % NS] when the copies land.
  auto stage = [&](int ai) {
    const int st = ai % NS;
    if (ai >= NS) mbar_wait(empty0 + 8u * st, ((ai / NS) - 1) & 1);
    const int* e = sched + ai * a.sched_stride;
    const int c0 = e[0] * a.CC, rs = e[1], rc = e[2];
    const unsigned sb = smem_addr(smem + st * a.stage_floats);
    if (a.mos && (!(a.debug & 1) || ai < NS)) {
      // mosaic: slab row r = super input row y_first + r; segment (r, image
      // column j) holds W floats of image n = block * mos + j, or stays zero
      // (separator rows, rows above the batch, images beyond N)
      const int RP = a.H + a.pad, CP = a.W + a.pad;
      const int ncl = min(a.CC, a.C - c0);
      for (int ee = threadIdx.x; ee < a.SR * a.mos * a.W; ee += kTiledThreads) {
        const int t = ee / a.W, x = ee - t * a.W;
        const int r = t / a.mos, j = t - r * a.mos;
        const int Y = y_first + r;
        if (Y < 0) continue;
        const int blk = Y / RP, y = Y - blk * RP, n = blk * a.mos + j;
        if (y >= a.H || n >= a.N) continue;
        unsigned sp = sb + 4u * static_cast<unsigned>(r * a.SCs + a.pad + j * CP + x);
        const float* g = a.in + ((static_cast<int64_t>(n) * a.C + c0) * a.H + y) * a.W + x;
        int cl = 0;
#pragma unroll 4
        for (; cl < ncl; ++cl) {
          cp_async4(sp, g, 4);
          sp += 4u * a.plane;
          g += HW;
        }
        for (; cl < a.CC; ++cl) {
          cp_async4(sp, a.in, 0);
          sp += 4u * a.plane;
        }
      }
    } else if (!(a.debug & 1) || ai < NS)
    // thread-owned interior elements ee; planes (image, channel) in the inner loop
    for (int ee = threadIdx.x; ee < nint; ee += kTiledThreads) {
      const int r = ee / a.W;
      const unsigned so = sb + 4u * static_cast<unsigned>((r_lo + r) * a.SCs + (a.pad + ee - r * a.W) * IP);
      const float* gbase = a.in + static_cast<int64_t>(y0) * a.W + ee;
      for (int im = 0; im < a.NB * IP; ++im) {
        const int n = n0 + im;
        const int ncl = n < a.N ? min(a.CC, a.C - c0) : 0;  // valid planes; the rest are re-zeroed
        const float* g = gbase + (static_cast<int64_t>(n < a.N ? n : 0) * a.C + c0) * HW;
        unsigned sp = so + 4u * static_cast<unsigned>((im / IP) * a.CC * a.plane + (im % IP));
        int cl = 0;
#pragma unroll 4
        for (; cl < ncl; ++cl) {
          cp_async4(sp, g, 4);
          sp += 4u * a.plane;
          g += HW;
        }
        for (; cl < a.CC; ++cl) {
          cp_async4(sp, a.in, 0);
          sp += 4u * a.plane;
        }
      }
    }
    const unsigned rb = smem_addr(recbase + st * a.stage_recs);
    for (int i = threadIdx.x; i < (rc >> 1); i += kTiledThreads) cp_async16(rb + 16u * i, a.recs + rs + 2 * i);
    cp_async_arrive(full0 + 8u * st);
  };

  float acc[Q * P];
#pragma unroll
  for (int i = 0; i < Q * P; ++i) acc[i] = 0.0f;
  float xw[MODE == 0 ? XH * XW : 1];  // mode 0: window registers, reloaded inside chunk_loop
#pragma unroll
  for (int i = 0; i < (MODE == 0 ? XH * XW : 1); ++i) xw[i] = 0.0f;
  constexpr int NACC2 = MODE == 2 ? Q * P / 2 : 1;
  constexpr int NX2 = MODE == 2 ? XH * (XW - 1) : 1;
  unsigned long long acc2[NACC2], xw2[NX2];  // mode 2: pairs
  constexpr int NACC3 = MODE == 3 ? Q * P : 1;
  constexpr int NX3 = MODE == 3 ? XH * XW : 1;
  unsigned long long acc3[NACC3], xw3[NX3];  // mode 3: (image 2g, image 2g+1) pairs
#pragma unroll
  for (int i = 0; i < NACC3; ++i) acc3[i] = 0ull;
#pragma unroll
  for (int i = 0; i < NX3; ++i) xw3[i] = 0ull;
#pragma unroll
  for (int i = 0; i < NACC2; ++i) acc2[i] = 0ull;
#pragma unroll
  for (int i = 0; i < NX2; ++i) xw2[i] = 0ull;

  // Pipeline without CTA barriers: chunk ai+1 is issued at the top of
  // iteration ai into buffer (ai+1) % NS, which requires every warp to have
  // released chunk ai+1-NS.  With NS = 3 a warp may run up to two chunks ahead
  // of the slowest warp (per-warp record counts differ chunk by chunk), where a
  // per-chunk __syncthreads would make every chunk cost the slowest warp's time.
  if (nact > 0) stage(0);
  for (int ai = 0; ai < nact; ++ai) {
    const int st = ai % NS;
    if (ai + 1 < nact) stage(ai + 1);
    mbar_wait(full0 + 8u * st, (ai / NS) & 1);
    const float* slab = smem + st * a.stage_floats + win_off;
    auto load_window = [&](float* x, int cl) {
      const float* src = slab + cl * a.plane;
      if (VEC_ALWAYS || a.PC == 1) {
#pragma unroll
        for (int r = 0; r < XH; ++r) {
#pragma unroll
          for (int v = 0; v < XWV; ++v) {
            const float4 t = *reinterpret_cast<const float4*>(src + r * a.SCs + 4 * v);
            if (4 * v + 0 < XW) x[r * XW + 4 * v + 0] = t.x;
            if (4 * v + 1 < XW) x[r * XW + 4 * v + 1] = t.y;
            if (4 * v + 2 < XW) x[r * XW + 4 * v + 2] = t.z;
            if (4 * v + 3 < XW) x[r * XW + 4 * v + 3] = t.w;
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < XH; ++r)
#pragma unroll
          for (int c = 0; c < XW; ++c) x[r * XW + c] = src[r * a.SCs + c];
      }
    };
    const int2* ws = recbase + st * a.stage_recs + sched[ai * a.sched_stride + 3 + wm];
    if constexpr (MODE == 0) {
      unsigned p = smem_addr(ws);
      chunk_loop<K, S, PH, PW, Q, TAG>(acc, xw, p, smem_addr(slab), 4u * a.SCs);
    } else if constexpr (MODE == 2) {
      unsigned p = smem_addr(ws);
      chunk_loop2<K, S, PH, PW, Q, TAG>(acc2, xw2, p, smem_addr(slab), 4u * a.SCs);
    } else if constexpr (MODE == 3) {
      unsigned p = smem_addr(ws);
      chunk_loop3<K, S, PH, PW, Q, TAG>(acc3, xw3, p, smem_addr(slab), 4u * a.SCs);
    } else if constexpr (MODE == 6) {
      // Tap records (no dispatch): {byte offset of tap (c, kh, kw) from the
      // lane's window origin, w[0..Q-1]} for every tap where any of the warp's
      // Q output channels has a nonzero (absent weights +0.0f: adds exact
      // zeros, so each channel still accumulates exactly its CSR terms in
      // ascending (c, kh, kw)).  Lanes own 32 consecutive output columns,
      // each PH rows of one column: per tap, PH scalar LDS (conflict-free at
      // stride 1, 2-way at stride 2; immediate row offsets, slab row stride
      // SCS6) and Q*PH FFMAs.
      static_assert(PW == 1, "tap-record mode: column patches");
      constexpr int SCS6 = 31 * S + K;  // slab row stride: 32 output columns at stride S
      constexpr int RS4 = (1 + Q + 3) / 4;
      const int4* rp = reinterpret_cast<const int4*>(ws);
      const int cnt = rp[0].x;
      rp += 1;
      const char* sb = reinterpret_cast<const char*>(slab);
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
        rp += RS4;
        const float* b = reinterpret_cast<const float*>(sb + __float_as_int(w[0]));
        float xv[PH];
#pragma unroll
        for (int v = 0; v < PH; ++v) xv[v] = b[v * S * SCS6];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int v = 0; v < PH; ++v) acc[q * P + v] = fmaf(w[1 + q], xv[v], acc[q * P + v]);
      }
    } else if constexpr (MODE == 7) {
      // Row records (no dispatch, CSR order kept): lanes own one output row
      // segment of PW pixels each (flat (image, row) slots).  One record per
      // (c, kh) where any of the warp's Q channels has a nonzero: {byte offset
      // of input row kh of channel c from the lane's window origin, kw-mask,
      // then w[kw][q]} — the lane loads its PW+K-1 input values of that row
      // once (vector LDS) and, for every kw with a nonzero (warp-uniform
      // branch), does Q*PW FFMAs; kw ascends inside the record, records ascend
      // in (c, kh), so each channel accumulates exactly in CSR order.
      static_assert(PH == 1 && S == 1, "row-record mode: full-row patches, stride 1");
      constexpr int XR = PW + K - 1;
      constexpr int XV = (XR + 3) / 4;
      constexpr int RS4 = 1 + (K * Q + 3) / 4;
      const int4* rp = reinterpret_cast<const int4*>(ws);
      const int cnt = rp[0].x;
      rp += 1;
      const char* sb = reinterpret_cast<const char*>(slab);
#pragma unroll 1
      for (int i = 0; i < cnt; ++i) {
        const int4 hd = rp[0];
        float w[(RS4 - 1) * 4];
#pragma unroll
        for (int k = 0; k < RS4 - 1; ++k) {
          const int4 t = rp[1 + k];
          w[4 * k + 0] = __int_as_float(t.x);
          w[4 * k + 1] = __int_as_float(t.y);
          w[4 * k + 2] = __int_as_float(t.z);
          w[4 * k + 3] = __int_as_float(t.w);
        }
        rp += RS4;
        const float4* b = reinterpret_cast<const float4*>(sb + hd.x);
        float xr[XV * 4];
#pragma unroll
        for (int v = 0; v < XV; ++v) {
          const float4 t = b[v];
          xr[4 * v + 0] = t.x;
          xr[4 * v + 1] = t.y;
          xr[4 * v + 2] = t.z;
          xr[4 * v + 3] = t.w;
        }
        const unsigned mask = static_cast<unsigned>(hd.y);
#pragma unroll
        for (int kw = 0; kw < K; ++kw) {
          if (mask & (1u << kw)) {
#pragma unroll
            for (int q = 0; q < Q; ++q)
#pragma unroll
              for (int px = 0; px < PW; ++px) acc[q * P + px] = fmaf(w[kw * Q + q], xr[px + kw], acc[q * P + px]);
          }
        }
      }
    } else {
      // warp stream: per bucket {c, 0, 0, 0} + Q*K*K weights (16-byte padded); c < 0 ends
      constexpr int NW4 = (Q * K * K + 3) / 4;
      const int4* b4 = reinterpret_cast<const int4*>(ws);
      int cl = b4->x;
      while (cl >= 0) {
        float x[XH * XW];
        load_window(x, cl);
        const int cl_next = b4[1 + NW4].x;
        bucket_mask<K, S, PH, PW, Q, TAG>(acc, x, smem_addr(b4 + 1));
        b4 += 1 + NW4;
        cl = cl_next;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8u * st);
  }

  if constexpr (MODE == 2) {
#pragma unroll
    for (int i = 0; i < Q * P / 2; ++i) {
      acc[2 * i] = __uint_as_float(static_cast<unsigned>(acc2[i] & 0xffffffffull));
      acc[2 * i + 1] = __uint_as_float(static_cast<unsigned>(acc2[i] >> 32));
    }
  }

  // Epilogue (reading R#10): v = acc + bias[m]; ReLU; NCHW store.
  if (a.mos) {
    // mosaic: super output row R -> (image block, oh), column X -> (image column, ow)
    if (active && !(a.debug & 4 && acc[0] != 12345.0f)) {
      const int RP = a.H + a.pad, CP = a.W + a.pad;
      int rb[PH], ro[PH], cj[PW], co[PW];
#pragma unroll
      for (int ph = 0; ph < PH; ++ph) {
        const int R = (pr0 + pr) * PH + ph;
        rb[ph] = R / RP;
        ro[ph] = R - rb[ph] * RP;
      }
#pragma unroll
      for (int pw = 0; pw < PW; ++pw) {
        const int X = pc * PW + pw;
        cj[pw] = X / CP;
        co[pw] = X - cj[pw] * CP;
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int m = (b * a.WM + wm) * Q + q;
        if (m < a.M) {
          const float bv = a.bias ? __ldg(a.bias + m) : 0.0f;
#pragma unroll
          for (int ph = 0; ph < PH; ++ph) {
#pragma unroll
            for (int pw = 0; pw < PW; ++pw) {
              const int n = rb[ph] * a.mos + cj[pw];
              if (ro[ph] < a.H && co[pw] < a.W && cj[pw] < a.mos && n < a.N) {
                float v = __fadd_rn(acc[q * P + ph * PW + pw], bv);
                if (a.relu) v = v > 0.0f ? v : 0.0f;
                a.out[((static_cast<int64_t>(n) * a.M + m) * a.E + ro[ph]) * a.F + co[pw]] = v;
              }
            }
          }
        }
      }
    }
  } else if (active && !(a.debug & 4 && acc[0] != 12345.0f)) {
#pragma unroll
    for (int j = 0; j < IP; ++j) {
      const int n = n0 + img * IP + j;
      if (n >= a.N) break;
      if constexpr (MODE == 3) {
#pragma unroll
        for (int i = 0; i < Q * P; ++i)
          acc[i] = __uint_as_float(static_cast<unsigned>(j == 0 ? (acc3[i] & 0xffffffffull) : (acc3[i] >> 32)));
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int m = (b * a.WM + wm) * Q + q;
        if (m < a.M) {
          const float bv = a.bias ? __ldg(a.bias + m) : 0.0f;
          float* o = a.out + (static_cast<int64_t>(n) * a.M + m) * a.E * a.F;
#pragma unroll
          for (int ph = 0; ph < PH; ++ph) {
            const int oh = (pr0 + pr) * PH + ph;
#pragma unroll
            for (int pw = 0; pw < PW; ++pw) {
              const int ow = pc * PW + pw;
              if (oh < a.E && ow < a.F) {
                float v = __fadd_rn(acc[q * P + ph * PW + pw], bv);
                if (a.relu) v = v > 0.0f ? v : 0.0f;
                o[oh * a.F + ow] = v;
              }
            }
          }
        }
      }
    }
  }
}

template <int K, int S, int PH, int PW, int Q, int MINB, int MODE, int TAG>
int launch_tiled(const TiledArgs& a, cudaStream_t s) {
  auto kern = sconv_tiled_kernel<K, S, PH, PW, Q, MINB, MODE, TAG>;
  if (a.smem_bytes > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
    if (e != cudaSuccess) return static_cast<int>(e);
  }
  dim3 grid(a.B, a.ntiles);
  kern<<<grid, kTiledThreads, a.smem_bytes, s>>>(a);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace escoin
