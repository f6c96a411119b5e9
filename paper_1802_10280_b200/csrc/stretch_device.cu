// stretch_device.cu — weight stretching on the GPU (NEXT-4).
//
// Same contract as the host escoin_csr_stretch (P:310-322 CSR, P:437-442
// stretching; readings R#4-R#7): keep w != 0.0f, rows in order, inside a row
// ascending (c, kh, kw), colidx = c*Hp*Wp + kh*Wp + kw, value copied bitwise.
// Three passes over the dense [M][C][K][K] weights already in device memory:
//   1. count the nonzeros of every row            (one CTA per row)
//   2. exclusive scan of the counts -> rowptr     (one CTA)
//   3. order-preserving compaction of every row   (one CTA per row: ballot +
//      per-warp popc + CTA prefix per 256-element slice)
#include <cstdint>

#include "escoin_internal.h"

namespace escoin {

namespace {
constexpr int kSt = 256;

__global__ void __launch_bounds__(kSt) count_rows_kernel(const float* __restrict__ w, int64_t crs, int* cnt) {
  const float* row = w + static_cast<int64_t>(blockIdx.x) * crs;
  int c = 0;
  for (int64_t i = threadIdx.x; i < crs; i += kSt) c += row[i] != 0.0f;
  __shared__ int red[kSt / 32];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int i = 0; i < kSt / 32; ++i) t += red[i];
    cnt[blockIdx.x] = t;
  }
}

// Exclusive scan of cnt[0..M) into rowptr[0..M]; one CTA, sequential over
// 1024-element slices (M is a channel count: small).
__global__ void __launch_bounds__(1024) scan_rows_kernel(const int* cnt, int M, int32_t* rowptr) {
  __shared__ int s[1024];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < M; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < M ? cnt[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan
      const int t = threadIdx.x >= o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < M) rowptr[i] = carry + s[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += s[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) rowptr[M] = carry;
}

__global__ void __launch_bounds__(kSt) compact_rows_kernel(const float* __restrict__ w, int64_t crs, int K, int Hp,
                                                           int Wp, const int32_t* __restrict__ rowptr,
                                                           int32_t* __restrict__ colidx, float* __restrict__ value) {
  const int m = blockIdx.x;
  const float* row = w + static_cast<int64_t>(m) * crs;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ int wsum[kSt / 32];
  int out = rowptr[m];
  for (int64_t base = 0; base < crs; base += kSt) {
    const int64_t i = base + threadIdx.x;
    const float v = i < crs ? row[i] : 0.0f;
    const bool nz = v != 0.0f;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int k = 0; k < kSt / 32; ++k) {
      before += k < warp ? wsum[k] : 0;
      total += wsum[k];
    }
    if (nz) {
      const int pos = out + before + __popc(bal & ((1u << lane) - 1u));
      const int64_t kw = i % K, kh = (i / K) % K, c = i / (static_cast<int64_t>(K) * K);
      colidx[pos] = static_cast<int32_t>((c * Hp + kh) * Wp + kw);
      value[pos] = v;
    }
    out += total;
    __syncthreads();
  }
}
// Inverse of the stretch, for the dense engine (escoin_csr_set_kernel(ESCOIN_KERNEL_DENSE_TC)):
// scatter row m's nonzeros back to w[m][c][kh][kw] (w zeroed by the caller).  colidx decodes
// uniquely (mixed radix, R#4): c = col / (Hp*Wp), kh = (col % (Hp*Wp)) / Wp, kw = col % Wp.
__global__ void __launch_bounds__(kSt) densify_rows_kernel(const int32_t* __restrict__ rowptr,
                                                            const int32_t* __restrict__ colidx,
                                                            const float* __restrict__ value, int C, int K, int Hp,
                                                            int Wp, float* __restrict__ w) {
  const int m = blockIdx.x;
  const int64_t base = static_cast<int64_t>(m) * C * K * K;
  for (int j = rowptr[m] + threadIdx.x; j < rowptr[m + 1]; j += kSt) {
    const int col = colidx[j];
    const int c = col / (Hp * Wp), r = col % (Hp * Wp);
    w[base + (static_cast<int64_t>(c) * K + r / Wp) * K + r % Wp] = value[j];
  }
}
}  // namespace

int launch_densify(const int32_t* rowptr, const int32_t* colidx, const float* value, int M, int C, int K, int Hp,
                   int Wp, float* w, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(w, 0, sizeof(float) * size_t(M) * C * K * K, s);
  if (e != cudaSuccess) return static_cast<int>(e);
  densify_rows_kernel<<<M, kSt, 0, s>>>(rowptr, colidx, value, C, K, Hp, Wp, w);
  return static_cast<int>(cudaGetLastError());
}

int launch_stretch_count(const float* w, int M, int64_t crs, int* cnt, cudaStream_t s) {
  count_rows_kernel<<<M, kSt, 0, s>>>(w, crs, cnt);
  return static_cast<int>(cudaGetLastError());
}

int launch_stretch_scan(const int* cnt, int M, int32_t* rowptr, cudaStream_t s) {
  scan_rows_kernel<<<1, 1024, 0, s>>>(cnt, M, rowptr);
  return static_cast<int>(cudaGetLastError());
}

int launch_stretch_compact(const float* w, int M, int64_t crs, int K, int Hp, int Wp, const int32_t* rowptr,
                           int32_t* colidx, float* value, cudaStream_t s) {
  compact_rows_kernel<<<M, kSt, 0, s>>>(w, crs, K, Hp, Wp, rowptr, colidx, value);
  return static_cast<int>(cudaGetLastError());
}

}  // namespace escoin

// ------------------------------------------------------------------ split-channel reduce
// out[i] = act(((ws[0][i] + ws[1][i]) + ... + ws[ks-1][i]) + bias[m]) for the specialised kernel's split
// channels (JitPlan::ks): the partial sums are added in z order, then the bias (one fp32 add), then
// ReLU v > 0 ? v : 0 (R#10) — a fixed order, so the result does not depend on the grid or the batch
// slice; coalesced float4 when the total is a multiple of 4.
namespace escoin {
namespace {
__global__ void ks_reduce_kernel(const float* __restrict__ ws, int ks, int64_t total, int M, int EF,
                                 const float* __restrict__ bias, int relu, float* __restrict__ out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    float v = ws[i];
    for (int z = 1; z < ks; ++z) v = __fadd_rn(v, ws[int64_t(z) * total + i]);
    if (bias) v = __fadd_rn(v, bias[(i / EF) % M]);
    if (relu) v = v > 0.0f ? v : 0.0f;
    out[i] = v;
  }
}
}  // namespace

int launch_ks_reduce(const float* ws, int ks, int64_t total, int M, int EF, const float* bias, int relu, float* out,
                     cudaStream_t s) {
  if (total <= 0) return 0;
  const int threads = 256;
  const int64_t want = (total + threads - 1) / threads;
  const int blocks = int(want < 148 * 16 ? want : 148 * 16);
  ks_reduce_kernel<<<blocks, threads, 0, s>>>(ws, ks, total, M, EF, bias, relu, out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace escoin
