// dense_tc.cu — dense implicit-GEMM convolution on the 5th-generation tensor
// cores (tcgen05 + TMEM), sm_100a.  A MEASURED COMPARISON POINT, not the
// method: north_star keeps "a dense tcgen05 implicit-GEMM only as a measured
// comparison point"; it multiplies every weight, zeros
// included, and never reads the CSR.
//
//   D[m][p] = sum_k A[m][k] * B[k][p],  k = (c, kh, kw) (dense pruned weights,
//   row-major [M][C*K*K]),  p = (n, oh, ow) flat over the batch,
//   B[k][p] = X~[n][c][oh*s + kh][ow*s + kw] (implicit im2col, virtual padding)
//   out[n][m][oh][ow] = act(D[m][p] + bias[m])
//
// Precision: NSPLIT = 1 is plain TF32 (the tensor core reads the top 19 bits
// of each fp32 operand, ~1e-3 relative error); NSPLIT = 3 is "3xTF32" — x = hi + lo with hi, lo both
// TF32, D += Ahi*Bhi + Ahi*Blo + Alo*Bhi — which recovers FP32-level accuracy
// (the dropped lo*lo term is ~2^-22 relative) at 3x the tensor-core work.
//
// CTA (544 threads): warps 0-15 gather operand tiles into shared memory and run
// the epilogue; warp 16 owns TMEM (alloc / dealloc) and one elected lane issues
// tcgen05.mma.  Tile 128 (m) x 128 (p) x 32 (k) per stage, operands K-major in
// the canonical 128-byte-swizzled layout (8-row x 128-byte atoms, SBO = 1024 B),
// NS-stage mbarrier pipeline (full: 512 producer arrivals; empty: tcgen05.commit).
// The accumulator lives in TMEM (128 lanes x 128 fp32 columns); the epilogue
// reads it with tcgen05.ld.32x32b (warp w: TMEM lanes 32*(w%4).., columns
// 32*(w/4)..).
#include <cstdint>

#include "escoin_internal.h"

namespace escoin {

namespace {

constexpr int kBM = 128, kBN = 128, kBK = 32;
constexpr int kPW = 16;                          // producer / epilogue warps
constexpr int kProducers = kPW * 32;
constexpr int kKPT = kBK * kBN / kProducers;     // k per producer thread per chunk (8)
constexpr int kAPT = kBM * (kBK / 4) / kProducers;  // A 16-byte chunks per producer thread (2)
constexpr int kThreadsTC = kProducers + 32;     // + MMA / TMEM warp
constexpr int kTileBytes = kBM * kBK * 4;       // 16 KB per operand tile (kBM == kBN)

struct DenseArgs {
  const float* in;
  const float* w;     // [M][Kd] dense pruned weights (block-diagonal for groups)
  const float* bias;  // [M] or null
  float* out;
  int N, C, H, W, M, K, S, pad, E, F, relu;
  int Kd;             // C*K*K
  int64_t npix;       // N*E*F
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint32_t b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(b) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(b),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a0), "r"(a1), "r"(a2), "r"(a3)
               : "memory");
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
}

// K-major, 128-byte swizzle: element (row, k) of a [rows][32] fp32 tile.
__device__ __forceinline__ uint32_t sw128(int row, int k) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ row) & 7) << 4) + (k & 3) * 4;
}

// UMMA shared-memory descriptor: K-major SWIZZLE_128B, SBO = 1024 B, version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                 // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;         // SBO
  d |= static_cast<uint64_t>(1) << 46;                 // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = kBN.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(kBN >> 3) << 17) | (uint32_t(kBM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

template <int NSPLIT>
__global__ void __launch_bounds__(kThreadsTC, 1) dense_tc_kernel(const DenseArgs a, int NS) {
  constexpr int NT = NSPLIT == 1 ? 2 : 4;  // operand tiles per stage: A,B or Ahi,Alo,Bhi,Blo
  extern __shared__ __align__(1024) uint8_t dsm[];
  // 1024-byte aligned tile area
  const uint32_t tiles_s = (smem_u32(dsm) + 1023u) & ~1023u;  // shared-window address of the tiles
  __shared__ __align__(8) unsigned long long bars[2 * 8 + 1];
  __shared__ uint32_t tmem_base_sh;
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[8]), done = smem_u32(&bars[16]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM;
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kBN;
  const int nk = (a.Kd + kBK - 1) / kBK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      bar_init(full0 + 8 * s, kProducers);
      bar_init(empty0 + 8 * s, 1);
    }
    bar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == kPW) {  // TMEM: 128 lanes x 128 fp32 columns for the accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base_sh)),
                 "n"(kBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base_sh;

  if (warp < kPW) {
    // ---------------- producers: implicit im2col (B) and weights (A)
    // B: thread t owns pixel row pr = t % 128 and k in [16*(t/128), +16) of
    // every chunk (16-byte stores: the 8 rows of a swizzle atom hit 8 distinct
    // 16-byte bank groups).  A: 16-byte chunks of weight rows, vector loads when the
    // rows are 16-byte aligned (Kd % 4 == 0).
    const int t = threadIdx.x;
    const int pr = t & (kBN - 1), q0 = t >> 7;  // pixel row, k-slice of kKPT
    const int64_t pg = p0 + pr;
    const bool pvalid = pg < a.npix;
    int n = 0, oh = 0, ow = 0;
    if (pvalid) {
      const int64_t EF = static_cast<int64_t>(a.E) * a.F;
      n = static_cast<int>(pg / EF);
      const int rem = static_cast<int>(pg - static_cast<int64_t>(n) * EF);
      oh = rem / a.F;
      ow = rem - oh * a.F;
    }
    const int iy0 = oh * a.S - a.pad, ix0 = ow * a.S - a.pad;
    const float* xn = a.in + static_cast<int64_t>(n) * a.C * a.H * a.W;
    const float* xpix = xn + static_cast<int64_t>(iy0) * a.W + ix0;  // tap (0,0) of channel 0 (may lie in the padding)
    const int KK = a.K * a.K;
    uint64_t tapmask = 0;  // bit kh*K + kw: tap inside the image (K*K <= 64)
    if (pvalid && KK <= 64)
      for (int kh = 0; kh < a.K; ++kh)
        for (int kw = 0; kw < a.K; ++kw)
          if (iy0 + kh >= 0 && iy0 + kh < a.H && ix0 + kw >= 0 && ix0 + kw < a.W) tapmask |= 1ull << (kh * a.K + kw);
    const bool avec = (a.Kd & 3) == 0;
    auto split = [](float v, uint32_t& hi, uint32_t& lo) {
      if (NSPLIT == 1) {
        hi = __float_as_uint(v);  // the tensor core reads the top 19 bits (TF32)
        lo = 0;
      } else {
        hi = to_tf32(v);
        lo = to_tf32(v - __uint_as_float(hi));
      }
    };
    if constexpr (NSPLIT == 1) {
      // TF32: no conversion (the tensor core reads the top 19 bits), so the
      // operands go global -> shared with cp.async (zero-fill for padding and
      // ragged edges) and the thread runs kLag stages ahead of its own
      // completions: stage i is released to the MMA (proxy fence + full
      // arrive) once its copies have landed, kLag stages later.
      constexpr int kLag = 3;
      for (int i = 0; i < nk + kLag; ++i) {
        if (i < nk) {
          const int s = i % NS;
          if (i >= NS) bar_wait(empty0 + 8 * s, ((i / NS) - 1) & 1);
          const uint32_t tA = tiles_s + static_cast<uint32_t>(s * NT * kTileBytes), tB = tA + kTileBytes;
          const int k0 = i * kBK;
#pragma unroll
          for (int j = 0; j < kAPT; ++j) {
            const int idx = t + j * kProducers;
            const int row = idx >> 3, ch = idx & 7;
            const int m = m0 + row, k = k0 + ch * 4;
            const uint32_t off = sw128(row, ch * 4);
            const float* src = a.w + static_cast<int64_t>(m < a.M ? m : 0) * a.Kd + k;
            if (avec && m < a.M && k + 3 < a.Kd) {
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(tA + off), "l"(src) : "memory");
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const bool ok = m < a.M && k + e < a.Kd;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(tA + off + 4 * e),
                             "l"(ok ? src + e : a.w), "r"(ok ? 4 : 0)
                             : "memory");
              }
            }
          }
          const int kb = k0 + q0 * kKPT;
          int c = kb / KK, r = kb - c * KK;
          int kh = r / a.K, kw = r - kh * a.K;
          int64_t off = (static_cast<int64_t>(c) * a.H + kh) * a.W + kw;
#pragma unroll
          for (int e = 0; e < kKPT; ++e) {
            const bool ok = c < a.C && (KK <= 64 ? ((tapmask >> r) & 1ull) != 0
                                                   : (pvalid && iy0 + kh >= 0 && iy0 + kh < a.H && ix0 + kw >= 0 &&
                                                      ix0 + kw < a.W));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(tB + sw128(pr, q0 * kKPT + e)),
                         "l"(ok ? xpix + off : a.in), "r"(ok ? 4 : 0)
                         : "memory");
            ++off;
            ++r;
            if (++kw == a.K) {
              kw = 0;
              off += a.W - a.K;
              if (++kh == a.K) {
                kh = 0;
                r = 0;
                ++c;
                off += static_cast<int64_t>(a.H - a.K) * a.W;
              }
            }
          }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        if (i >= kLag) {  // stage i - kLag has landed: hand it to the tensor core
          asm volatile("cp.async.wait_group %0;\n" ::"n"(kLag) : "memory");
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          bar_arrive(full0 + 8 * ((i - kLag) % NS));
        }
      }
    } else
    for (int i = 0; i < nk; ++i) {
      const int s = i % NS;
      if (i >= NS) bar_wait(empty0 + 8 * s, ((i / NS) - 1) & 1);
      const uint32_t st = tiles_s + static_cast<uint32_t>(s * NT * kTileBytes);
      const uint32_t tA = st;                                       // A hi (A lo follows for 3xTF32)
      const uint32_t tB = st + (NSPLIT == 1 ? 1 : 2) * kTileBytes;  // B hi (B lo follows)
      const int k0 = i * kBK;
#pragma unroll
      for (int j = 0; j < kAPT; ++j) {
        const int idx = t + j * kProducers;
        const int row = idx >> 3, ch = idx & 7;
        const int m = m0 + row, k = k0 + ch * 4;
        float v[4];
        if (avec && m < a.M && k + 3 < a.Kd) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(a.w + static_cast<int64_t>(m) * a.Kd + k));
          v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e)
            v[e] = (m < a.M && k + e < a.Kd) ? __ldg(a.w + static_cast<int64_t>(m) * a.Kd + k + e) : 0.0f;
        }
        uint32_t hi[4], lo[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) split(v[e], hi[e], lo[e]);
        const uint32_t off = sw128(row, ch * 4);
        sts128(tA + off, hi[0], hi[1], hi[2], hi[3]);
        if (NSPLIT == 3) sts128(tA + kTileBytes + off, lo[0], lo[1], lo[2], lo[3]);
      }
      // B: kKPT consecutive k of this thread's pixel, 16-byte stores.  One
      // division per stage; then the tap index r = kh*K + kw and the input
      // offset advance incrementally, and the tap's validity (padding) is one
      // bit of the pixel's window mask.
      {
        const int kb = k0 + q0 * kKPT;
        int c = kb / KK, r = kb - c * KK;
        int kh = r / a.K, kw = r - kh * a.K;
        int64_t off = (static_cast<int64_t>(c) * a.H + kh) * a.W + kw;
        float vv[kKPT];
#pragma unroll
        for (int e = 0; e < kKPT; ++e) {  // all loads first (memory-level parallelism), then stores
          const bool ok = c < a.C && (KK <= 64 ? ((tapmask >> r) & 1ull) != 0
                                                 : (pvalid && iy0 + kh >= 0 && iy0 + kh < a.H && ix0 + kw >= 0 &&
                                                    ix0 + kw < a.W));
          vv[e] = ok ? __ldg(xpix + off) : 0.0f;
          ++off;
          ++r;
          if (++kw == a.K) {
            kw = 0;
            off += a.W - a.K;
            if (++kh == a.K) {
              kh = 0;
              r = 0;
              ++c;
              off += static_cast<int64_t>(a.H - a.K) * a.W;
            }
          }
        }
#pragma unroll
        for (int j = 0; j < kKPT / 4; ++j) {
          uint32_t hi[4], lo[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) split(vv[4 * j + e], hi[e], lo[e]);
          const uint32_t soff = sw128(pr, q0 * kKPT + j * 4);
          sts128(tB + soff, hi[0], hi[1], hi[2], hi[3]);
          if (NSPLIT == 3) sts128(tB + kTileBytes + soff, lo[0], lo[1], lo[2], lo[3]);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> async proxy (MMA)
      bar_arrive(full0 + 8 * s);
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer
    for (int i = 0; i < nk; ++i) {
      const int s = i % NS;
      bar_wait(full0 + 8 * s, (i / NS) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t st = tiles_s + static_cast<uint32_t>(s * NT * kTileBytes);
      const uint32_t aHi = st, aLo = st + kTileBytes;
      const uint32_t bHi = st + (NSPLIT == 1 ? 1 : 2) * kTileBytes, bLo = bHi + kTileBytes;
#pragma unroll
      for (int j = 0; j < kBK / 8; ++j) {  // UMMA_K = 8 tf32 = 32 bytes of the 128-byte row
        const uint32_t acc = (i > 0 || j > 0) ? 1u : 0u;
        if (NSPLIT == 3) {
          mma_tf32(tmem, umma_desc(aLo + 32 * j), umma_desc(bHi + 32 * j), acc);
          mma_tf32(tmem, umma_desc(aHi + 32 * j), umma_desc(bLo + 32 * j), 1u);
          mma_tf32(tmem, umma_desc(aHi + 32 * j), umma_desc(bHi + 32 * j), 1u);
        } else {
          mma_tf32(tmem, umma_desc(aHi + 32 * j), umma_desc(bHi + 32 * j), acc);
        }
      }
      // frees the stage once these MMAs have read it
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(empty0 + 8 * s)
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(done) : "memory");
  }

  // ---------------- epilogue: warps 0-15, TMEM lane quarter w%4, column quarter w/4
  if (warp < kPW) {
    bar_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const int q = warp & 3, half = warp >> 2;  // half = column slice of kBN / (kPW / 4)
    const int m = m0 + q * 32 + lane;
    const float bv = (a.bias && m < a.M) ? __ldg(a.bias + m) : 0.0f;
    const int64_t EF = static_cast<int64_t>(a.E) * a.F;
#pragma unroll 1
    for (int cb = 0; cb < kBN / (kPW / 4); cb += 16) {
      const int col = half * (kBN / (kPW / 4)) + cb;
      uint32_t v[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
          "%15}, [%16];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + (static_cast<uint32_t>(q * 32) << 16) + col));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      if (m < a.M) {
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int64_t pg = p0 + col + e;
          if (pg < a.npix) {
            const int64_t nn = pg / EF, rem = pg - nn * EF;
            float o = __uint_as_float(v[e]) + bv;
            if (a.relu) o = o > 0.0f ? o : 0.0f;
            a.out[(nn * a.M + m) * EF + rem] = o;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == kPW) {
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kBN));
  }
}

}  // namespace

int launch_dense_tc(const float* in, const float* w, const float* bias, float* out, int N, int C, int H, int W,
                    int M, int K, int S, int pad, int relu, int nsplit, cudaStream_t s) {
  DenseArgs a;
  a.in = in;
  a.w = w;
  a.bias = bias;
  a.out = out;
  a.N = N;
  a.C = C;
  a.H = H;
  a.W = W;
  a.M = M;
  a.K = K;
  a.S = S;
  a.pad = pad;
  a.E = (H + 2 * pad - K) / S + 1;
  a.F = (W + 2 * pad - K) / S + 1;
  a.relu = relu;
  a.Kd = C * K * K;
  a.npix = static_cast<int64_t>(N) * a.E * a.F;
  const int NT = nsplit == 1 ? 2 : 4;
  const int NS = nsplit == 1 ? 6 : 3;
  const int smem = NS * NT * kTileBytes + 1024;
  dim3 grid(static_cast<unsigned>((a.npix + kBN - 1) / kBN), (M + kBM - 1) / kBM);
  if (grid.x > 0x7fffffffu || grid.y > 65535) return static_cast<int>(cudaErrorInvalidValue);
  cudaError_t e;
  if (nsplit == 1) {
    e = cudaFuncSetAttribute(dense_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    dense_tc_kernel<1><<<grid, kThreadsTC, smem, s>>>(a, NS);
  } else {
    e = cudaFuncSetAttribute(dense_tc_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return static_cast<int>(e);
    dense_tc_kernel<3><<<grid, kThreadsTC, smem, s>>>(a, NS);
  }
  return static_cast<int>(cudaGetLastError());
}

}  // namespace escoin
