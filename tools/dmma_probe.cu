#include <cstdio>
template <int SHAPE>
__global__ void k(double *out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = 0.5, b1 = 0.25;
  double acc[8][4];
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) acc[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (SHAPE == 0)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a0), "d"(b0));
      else
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3]) : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double *o; cudaMalloc(&o, 148 * 8 * 256 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int shape = 0; shape < 2; ++shape) for (int rep = 0; rep < 2; ++rep) {
    const int iters = 20000;
    cudaEventRecord(e0);
    if (shape == 0) k<0><<<148 * 4, 256>>>(o, iters); else k<1><<<148 * 4, 256>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fma_per = shape == 0 ? 256.0 : 512.0;
    const double flops = 2.0 * fma_per * 8 * iters * (148.0 * 4 * 256 / 32);
    printf("shape %s: %.2f ms, %.1f TFLOP/s (%s)\n", shape == 0 ? "m8n8k4" : "m16n8k4", ms, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
}
