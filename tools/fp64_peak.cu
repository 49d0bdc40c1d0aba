// FP64 / FP32 arithmetic-pipe peak microbenchmark for the roofline denominator.
// Each thread runs NCHAIN independent FMA chains; total flops = 2 * fmas.
#include <cstdio>
#include <cuda_runtime.h>
#define NCHAIN 8
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T v[NCHAIN];
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) v[c] = (T)(threadIdx.x + c);
  // (NCHAIN 16 with the loop unrolled x4 measured lower: 33.6 vs 34.1 TFLOP/s,
  // profiles/fp64_peak_r02_nchain16_unroll4.jsonl)
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < NCHAIN; ++c) v[c] = v[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < NCHAIN; ++c) s += v[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename T>
double run(const char* name, int blocks, int threads, int iters) {
  T* out; cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * NCHAIN * (double)iters * blocks * threads;
  double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", name, blocks, threads, best, tf);
  cudaFree(out);
  return tf;
}
// back-to-back launches for ~seconds: the sustained figure (a kernel timed
// inside a long step runs at the sustained clock)
template <typename T>
double sustained(const char* name, int blocks, int threads, int iters, double seconds) {
  T* out; cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms1; cudaEventElapsedTime(&ms1, e0, e1);
  const int reps = (int)(seconds * 1e3 / ms1) + 1;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999999, (T)1e-7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * NCHAIN * (double)iters * blocks * threads * reps;
  double tf = flops / (ms * 1e-3) / 1e12;
  printf("{\"kernel\": \"%s_sustained\", \"blocks\": %d, \"threads\": %d, \"reps\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
         name, blocks, threads, reps, ms, tf);
  cudaFree(out);
  return tf;
}
int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
  sustained<double>("dfma", sms * 8, 256, 20000, 4.0);
  sustained<float>("ffma", sms * 8, 256, 40000, 4.0);
  for (int occ = 1; occ <= 8; occ *= 2) run<double>("dfma", sms * occ, 256, 20000);
  run<double>("dfma", sms * 16, 256, 10000);
  for (int occ = 1; occ <= 8; occ *= 2) run<float>("ffma", sms * occ, 256, 40000);
  return 0;
}
