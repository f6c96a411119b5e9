// Box-facts microbenchmarks for the sconv design.
// Not part of the product: measures FP32 FFMA issue rate on B200 for the
// register patterns the sconv inner loop uses, and the cost of the
// warp-uniform switch dispatch over (q, kh, kw) cases.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

// ---------------------------------------------------------------- pure FFMA
// acc[i] = fma(w, x[i], acc[i]); w uniform register, x and acc per-thread.
template <int NACC>
__global__ void __launch_bounds__(256) ffma_peak(float* out, float w0, int iters) {
  float acc[NACC], x[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { acc[i] = 0.f; x[i] = threadIdx.x * 1e-3f + i; }
  float w = w0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fmaf(w, x[i], acc[i]);
    w = w * 0.999f;  // keep w live / not hoistable
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

// ---------------------------------------------------------------- dispatch
#define R4(M, b) M(b) M(b + 1) M(b + 2) M(b + 3)
#define R16(M, b) R4(M, b) R4(M, b + 4) R4(M, b + 8) R4(M, b + 12)
#define R64(M, b) R16(M, b) R16(M, b + 16) R16(M, b + 32) R16(M, b + 48)
#define R256(M, b) R64(M, b) R64(M, b + 64) R64(M, b + 128) R64(M, b + 192)

template <int Q, int K, int PH, int PW>
struct Tile {
  float acc[Q][PH][PW];
  float x[PH + K - 1][PW + K - 1];
  template <int CODE>
  __device__ __forceinline__ void apply(float w) {
    if constexpr (CODE < Q * K * K) {
      constexpr int q = CODE / (K * K), kh = (CODE / K) % K, kw = CODE % K;
#pragma unroll
      for (int ph = 0; ph < PH; ++ph)
#pragma unroll
        for (int pw = 0; pw < PW; ++pw)
          acc[q][ph][pw] = fmaf(w, x[ph + kh][pw + kw], acc[q][ph][pw]);
    }
  }
};

template <int Q, int K, int PH, int PW>
__global__ void __launch_bounds__(256, 1)
dispatch_bench(const int2* __restrict__ recs_g, int nrec, float* out, int iters) {
  extern __shared__ int2 recs[];
  for (int i = threadIdx.x; i < nrec + 2; i += blockDim.x) recs[i] = recs_g[i];
  __syncthreads();
  Tile<Q, K, PH, PW> t;
#pragma unroll
  for (int q = 0; q < Q; ++q)
#pragma unroll
    for (int a = 0; a < PH; ++a)
#pragma unroll
      for (int b = 0; b < PW; ++b) t.acc[q][a][b] = 0.f;
#pragma unroll
  for (int a = 0; a < PH + K - 1; ++a)
#pragma unroll
    for (int b = 0; b < PW + K - 1; ++b) t.x[a][b] = threadIdx.x * 1e-3f + a * 7 + b;
  for (int it = 0; it < iters; ++it) {
    const int2* p = recs;
    int2 r = p[0];
    for (;;) {
      int2 nx = p[1];
      ++p;
      const float w = __int_as_float(r.y);
      bool done = false;
      switch (r.x) {
#define CASE(i) case i: t.template apply<i>(w); break;
        R256(CASE, 0)
#undef CASE
        default: done = true; break;
      }
      if (done) break;
      r = nx;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < Q; ++q)
#pragma unroll
    for (int a = 0; a < PH; ++a)
#pragma unroll
      for (int b = 0; b < PW; ++b) s += t.acc[q][a][b];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int Q, int K, int PH, int PW>
void run_dispatch(int sms, const char* name) {
  const int nrec = 2000;
  std::vector<int2> h(nrec + 2);
  srand(1);
  for (int i = 0; i < nrec; ++i) { h[i].x = rand() % (Q * K * K); float w = 1e-6f; h[i].y = *(int*)&w; }
  h[nrec].x = 9999; h[nrec + 1].x = 9999;
  int2* d; float* o;
  CK(cudaMalloc(&d, (nrec + 2) * sizeof(int2)));
  CK(cudaMalloc(&o, 4096));
  CK(cudaMemcpy(d, h.data(), (nrec + 2) * sizeof(int2), cudaMemcpyHostToDevice));
  auto kern = dispatch_bench<Q, K, PH, PW>;
  size_t smem = (nrec + 2) * sizeof(int2);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, kern));
  int iters = 20;
  for (int blocksPerSm = 1; blocksPerSm <= 1; ++blocksPerSm) {
    kern<<<sms, 256, smem>>>(d, nrec, o, 2);
    CK(cudaDeviceSynchronize());
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<<<sms * 2, 256, smem>>>(d, nrec, o, iters);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * (double)sms * 2 * 256 * iters * nrec * PH * PW;
    printf("dispatch %-14s Q=%d K=%d P=%dx%d regs=%d spill=%zu : %.2f ms  %.1f TFLOP/s\n", name, Q, K, PH, PW,
           fa.numRegs, (size_t)fa.localSizeBytes, ms, flops / ms / 1e9);
  }
  cudaFree(d); cudaFree(o);
}

template <int NACC>
void run_peak(int sms, int blocks_per_sm) {
  float* o; CK(cudaMalloc(&o, 4096));
  int iters = 20000;
  ffma_peak<NACC><<<sms, 256>>>(o, 1.0f, 10);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  ffma_peak<NACC><<<sms * blocks_per_sm, 256>>>(o, 1.0f, iters);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  double flops = 2.0 * sms * blocks_per_sm * 256.0 * iters * NACC;
  printf("ffma_peak NACC=%d blocks/SM=%d : %.2f ms  %.1f TFLOP/s\n", NACC, blocks_per_sm, ms, flops / ms / 1e9);
  cudaFree(o);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0, memclk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaDeviceGetAttribute(&memclk, cudaDevAttrMemoryClockRate, 0);
  printf("name=%s sms=%d l2=%d smem/sm=%zu smem/block_optin=%zu regs/sm=%d clock_khz=%d memclk_khz=%d cc=%d.%d\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin,
         p.regsPerMultiprocessor, clk, memclk, p.major, p.minor);
  int sms = p.multiProcessorCount;
  run_peak<16>(sms, 4);
  run_peak<32>(sms, 4);
  run_peak<32>(sms, 8);
  run_peak<64>(sms, 2);
  run_dispatch<8, 3, 4, 4>(sms, "q8k3p4x4");
  run_dispatch<4, 3, 4, 8>(sms, "q4k3p4x8");
  run_dispatch<6, 3, 2, 13>(sms, "q6k3p2x13");
  run_dispatch<8, 5, 4, 4>(sms, "q8k5p4x4");
  run_dispatch<4, 3, 2, 8>(sms, "q4k3p2x8");
  run_dispatch<8, 3, 2, 8>(sms, "q8k3p2x8");
  return 0;
}
