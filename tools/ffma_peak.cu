// FP32 FFMA peak on this GPU (the roofline denominator's measured companion).
// Three forms: register weight (FFMA R, R, R, R), immediate weight (FFMA R, R, imm, R — the form
// the specialised sconv kernel issued up to round 2) and the paired immediate form (FFMA2 R, R.F32x2,
// imm, R.F32x2: fma.rn.f32x2 with a broadcast 32-bit immediate, two lanes' worth per instruction).  Grid = SMs x blocks/SM, 32 independent accumulators per
// thread, long unrolled loops; prints one JSON line.
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void __launch_bounds__(1024, 1) ffma(float* out, float w0, int iters) {
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  const float w = w0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 2) {  // 16 independent pairs
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        unsigned long long a2;
        asm volatile("mov.b64 %0, {%1, %2};" : "=l"(a2) : "f"(acc[i]), "f"(acc[i + 1]));
        asm volatile("{.reg .b64 t; mov.b64 t, 0x3F7FF9723F7FF972; fma.rn.f32x2 %0, %0, t, %0;}" : "+l"(a2));
        asm volatile("mov.b64 {%0, %1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(a2));
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (MODE == 1)
        asm volatile("fma.rn.f32 %0, %0, 0f3F7FF972, %0;" : "+f"(acc[i]));
      else
        asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(acc[i]) : "f"(w));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int MODE>
double run(int sms, int threads, int iters) {
  float* d;
  cudaMalloc(&d, 4096 * 4);
  ffma<MODE><<<sms, threads>>>(d, 0.9999f, 16);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    ffma<MODE><<<sms, threads>>>(d, 0.9999f, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double tf = 2.0 * 32 * iters * double(sms) * threads / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  cudaFree(d);
  return best;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 20000;
  const double reg = run<0>(p.multiProcessorCount, 1024, iters);
  const double imm = run<1>(p.multiProcessorCount, 1024, iters);
  const double imm2 = run<2>(p.multiProcessorCount, 1024, iters);
  CK(cudaGetLastError());
  const double nominal = p.multiProcessorCount * 128.0 * 2 * clk * 1e3 / 1e12;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"ffma_reg_tflops\": %.2f, \"ffma_imm_tflops\": %.2f, \"ffma2_imm_tflops\": %.2f, "
         "\"best_tflops\": %.2f, \"nominal_tflops\": %.2f, \"threads_per_sm\": 1024, \"accumulators\": 32}\n",
         p.name, p.multiProcessorCount, clk, reg, imm, imm2, std::max(reg, std::max(imm, imm2)), nominal);
  return 0;
}
