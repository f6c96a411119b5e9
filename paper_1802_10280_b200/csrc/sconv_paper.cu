// sconv_paper.cu — the paper's own data-to-thread mapping, on sm_100a.
//
// Variant 0 of escoin_sconv_forward and the fallback for any (K, stride)
// without a register-tiled variant.  It follows §3.2/§3.3 directly:
//   * one thread block per output channel m ("We assign the work of
//     processing one output channel to a thread block"), grid.y = image n;
//   * one thread per output element, consecutive threads -> consecutive
//     outputs, so input loads and output stores coalesce;
//   * the CSR row's colidx/value are loaded cooperatively into shared memory
//     (P:551-553); inputs are read through the read-only path (__ldg,
//     P:553-555); partial sums live in registers.
// Padding is virtual (reading R#9): the stretched offset is decoded once per
// nonzero when the row is staged, and out-of-range taps read 0 — the same
// fma(w, 0, acc) the tiled kernels execute, so both give identical bits.
#include "escoin_internal.h"

namespace escoin {

namespace {
constexpr int kPaperThreads = 256;
constexpr int kPaperChunk = 1024;   // nonzeros staged per pass
constexpr int kOutPerThread = 4;    // outputs per thread per pass

__global__ void __launch_bounds__(kPaperThreads) sconv_paper_kernel(
    const int* __restrict__ rowptr, const int* __restrict__ colidx, const float* __restrict__ value,
    const float* __restrict__ in, float* __restrict__ out, const float* __restrict__ bias, int relu, int C,
    int H, int W, int M, int K, int S, int pad, int E, int F) {
  __shared__ int s_off[kPaperChunk];   // c*H*W + (kh-pad)*W + (kw-pad)  (may be negative)
  __shared__ int s_khw[kPaperChunk];   // (kh << 16) | kw
  __shared__ float s_val[kPaperChunk];
  const int m = blockIdx.x;
  const int n = blockIdx.y;
  const int Hp = H + 2 * pad, Wp = W + 2 * pad;
  const int beg = __ldg(rowptr + m), end = __ldg(rowptr + m + 1);
  const float* xin = in + static_cast<int64_t>(n) * C * H * W;
  float* o = out + (static_cast<int64_t>(n) * M + m) * E * F;
  const float bv = bias ? __ldg(bias + m) : 0.0f;
  const int EF = E * F;
  for (int o0 = 0; o0 < EF; o0 += kPaperThreads * kOutPerThread) {
    float acc[kOutPerThread];
    int oh[kOutPerThread], ow[kOutPerThread];
#pragma unroll
    for (int i = 0; i < kOutPerThread; ++i) {
      acc[i] = 0.0f;
      const int e = o0 + i * kPaperThreads + threadIdx.x;
      oh[i] = e < EF ? e / F : -1000000;
      ow[i] = e < EF ? e - (e / F) * F : 0;
    }
    for (int j0 = beg; j0 < end; j0 += kPaperChunk) {
      const int cnt = min(kPaperChunk, end - j0);
      __syncthreads();
      for (int t = threadIdx.x; t < cnt; t += kPaperThreads) {
        const int off = __ldg(colidx + j0 + t);      // stretched: c*Hp*Wp + kh*Wp + kw
        const int c = off / (Hp * Wp);
        const int rem = off - c * Hp * Wp;
        const int kh = rem / Wp, kw = rem - (rem / Wp) * Wp;
        s_off[t] = c * H * W + (kh - pad) * W + (kw - pad);
        s_khw[t] = (kh << 16) | kw;
        s_val[t] = __ldg(value + j0 + t);
      }
      __syncthreads();
      for (int t = 0; t < cnt; ++t) {
        const int off = s_off[t], kh = s_khw[t] >> 16, kw = s_khw[t] & 0xffff;
        const float w = s_val[t];
#pragma unroll
        for (int i = 0; i < kOutPerThread; ++i) {
          const int y = oh[i] * S + kh - pad, x = ow[i] * S + kw - pad;
          const bool ok = (unsigned)y < (unsigned)H && (unsigned)x < (unsigned)W;
          const float v = ok ? __ldg(xin + off + oh[i] * S * W + ow[i] * S) : 0.0f;
          acc[i] = __fmaf_rn(w, v, acc[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kOutPerThread; ++i) {
      const int e = o0 + i * kPaperThreads + threadIdx.x;
      if (e < EF) {
        float v = __fadd_rn(acc[i], bv);
        if (relu) v = v > 0.0f ? v : 0.0f;
        o[e] = v;
      }
    }
  }
}
}  // namespace

int launch_paper(const int* rowptr, const int* colidx, const float* value, const float* in, float* out,
                 const float* bias, int relu, int N, int C, int H, int W, int M, int K, int S, int pad, int E,
                 int F, cudaStream_t s) {
  if (N > 65535) return static_cast<int>(cudaErrorInvalidConfiguration);
  dim3 grid(M, N);
  sconv_paper_kernel<<<grid, kPaperThreads, 0, s>>>(rowptr, colidx, value, in, out, bias, relu, C, H, W, M, K, S,
                                                     pad, E, F);
  return static_cast<int>(cudaGetLastError());
}

#include "generated/variants_table.inc"

const TiledVariant* tiled_variants(int* count) {
  *count = static_cast<int>(sizeof(kTiledVariants) / sizeof(kTiledVariants[0]));
  return kTiledVariants;
}

}  // namespace escoin
