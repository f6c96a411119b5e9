// FP32 FFMA peak on this GPU (the roofline denominator's measured companion).
// Two forms: register weight (FFMA R, R, R, R) and immediate weight (FFMA R, R, imm, R — the form
// the specialised sconv kernel issues).  Grid = SMs x blocks/SM, 32 independent accumulators per
// thread, long unrolled loops; prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 1; } } while (0)

template <bool IMM>
__global__ void __launch_bounds__(1024, 1) ffma(float* out, float w0, int iters) {
  float acc[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  const float w = w0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (IMM)
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

template <bool IMM>
double run(int sms, int threads, int iters) {
  float* d;
  cudaMalloc(&d, 4096 * 4);
  ffma<IMM><<<sms, threads>>>(d, 0.9999f, 16);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  double best = 0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    ffma<IMM><<<sms, threads>>>(d, 0.9999f, iters);
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
  const double reg = run<false>(p.multiProcessorCount, 1024, iters);
  const double imm = run<true>(p.multiProcessorCount, 1024, iters);
  CK(cudaGetLastError());
  const double nominal = p.multiProcessorCount * 128.0 * 2 * clk * 1e3 / 1e12;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"ffma_reg_tflops\": %.2f, \"ffma_imm_tflops\": %.2f, "
         "\"best_tflops\": %.2f, \"nominal_tflops\": %.2f, \"threads_per_sm\": 1024, \"accumulators\": 32}\n",
         p.name, p.multiProcessorCount, clk, reg, imm, reg > imm ? reg : imm, nominal);
  return 0;
}
