// Measured FMA throughput (FP32 FFMA, FFMA2 pairs, FP64 DFMA) on the box —
// the compute roofline denominators for the k sweep.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void fma_loop(T *out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = (T)(threadIdx.x + q);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) x[q] = fma(x[q], a, b);
  T s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += x[q];
  if (s == (T)12345.678) out[0] = s;
}

__global__ void ffma2_loop(float *out, int iters, float a, float b) {
  unsigned long long x[8];
  for (int q = 0; q < 8; ++q) x[q] = ((unsigned long long)__float_as_uint((float)q) << 32) | __float_as_uint((float)threadIdx.x);
  unsigned long long aa, bb;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int q = 0; q < 8; ++q) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[q]) : "l"(aa), "l"(bb));
  unsigned long long s = 0;
  for (int q = 0; q < 8; ++q) s ^= x[q];
  if (s == 12345) out[0] = 1.f;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *o;
  cudaMalloc(&o, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 20000;
  const double fmas = (double)blocks * threads * iters * 8;
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    fma_loop<float><<<blocks, threads>>>(o, iters, 1.0000001f, 0.5f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("{\"ffma_tflops\": %.1f, ", 2 * fmas / ms / 1e9);
    cudaEventRecord(a);
    ffma2_loop<<<blocks, threads>>>(o, iters, 1.0000001f, 0.5f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("\"ffma2_tflops\": %.1f, ", 4 * fmas / ms / 1e9);
    cudaEventRecord(a);
    fma_loop<double><<<blocks, threads>>>((double *)o, iters, 1.0000001, 0.5);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) printf("\"dfma_tflops\": %.1f, \"sms\": %d}\n", 2 * fmas / ms / 1e9, sms);
  }
  return 0;
}
