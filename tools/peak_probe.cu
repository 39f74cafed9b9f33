// Microbenchmark: FP32 FFMA and FP64 DFMA issue peaks on the local GPU.
// Used only to fill the SIMT roofline denominators that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = (T)(threadIdx.x + c);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = acc[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == (T)1.2345) out[0] = s;
}

template <typename T>
double run(const char* name, int blocks, int threads, int iters) {
  T* d; cudaMalloc(&d, sizeof(T));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  fma_loop<T, 16><<<blocks, threads>>>(d, 100, (T)0.999, (T)0.001);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_loop<T, 16><<<blocks, threads>>>(d, iters, (T)0.999, (T)0.001);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 16.0 * (double)iters * blocks * threads;
  double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"probe\": \"%s\", \"tflops\": %.3f, \"ms\": %.3f}\n", name, tf, best);
  cudaFree(d);
  return tf;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  run<float>("ffma_fp32", sms * 8, 256, 20000);
  run<double>("dfma_fp64", sms * 8, 256, 4000);
  return 0;
}
