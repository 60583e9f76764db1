// Does die-affine access raise the effective L2 capacity on B200?
//
// Random 2 KB block reads (+ optional 2 KB red.add into a second buffer, the
// SpMM's X_C gather / Y_C reduction) over a working set twice the L2:
//   mode 0: every SM draws blocks from the whole buffer;
//   mode 1: an SM of die d (die map from die_probe, argv) draws only blocks
//           with (b & 1) == d.
// Same number of accesses; lower time ⇒ each die's L2 holds its half better
// (i.e. far-homed lines are also cached near — capacity is per die).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/die_l2_probe tools/die_l2_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void run(const float4 *__restrict__ X, float *Y, long long n_blocks, int iters, int mode, int with_red,
                    unsigned long long m0, unsigned long long m1, unsigned long long m2, float *sink) {
  const unsigned s = smid();
  const unsigned long long m = s < 64 ? m0 : (s < 128 ? m1 : m2);
  const int die = (int)((m >> (s & 63)) & 1ull);
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    uint64_t r = mix(((uint64_t)warp << 20) + it);
    long long b = (long long)(r % (uint64_t)n_blocks);
    if (mode == 1) b = (b & ~1ll) | die;
    const float4 *p = X + b * 128;  // 2 KB = 128 float4
    float4 v0 = __ldcg(p + lane), v1 = __ldcg(p + lane + 32), v2 = __ldcg(p + lane + 64), v3 = __ldcg(p + lane + 96);
    acc += v0.x + v1.y + v2.z + v3.w;
    if (with_red) {
      uint64_t r2 = mix(r);
      long long c = (long long)(r2 % (uint64_t)n_blocks);
      if (mode == 1) c = (c & ~1ll) | die;
      float *y = Y + c * 512 + lane * 4;
      for (int q = 0; q < 4; ++q)
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(y + q * 128), "f"(v0.x), "f"(v1.x), "f"(v2.x),
                     "f"(v3.x)
                     : "memory");
    }
  }
  if (acc == 12345.f) *sink = acc;
}

int main(int argc, char **argv) {
  // argv[1]: 148-char die string over sm ids (from die_probe clustering)
  if (argc < 2) {
    fprintf(stderr, "usage: die_l2_probe <die-string indexed by smid>\n");
    return 1;
  }
  unsigned long long m[3] = {0, 0, 0};
  for (int i = 0; i < (int)strlen(argv[1]) && i < 192; ++i)
    if (argv[1][i] == '1') m[i / 64] |= 1ull << (i % 64);
  const long long bytes = 256ll << 20;  // X 256 MB (+ Y 256 MB with reds): 2-4x the L2
  const long long n_blocks = bytes / 2048;
  float4 *X;
  float *Y, *sink;
  cudaMalloc(&X, bytes);
  cudaMalloc(&Y, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(X, 0, bytes);
  cudaMemset(Y, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 2000;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int red = 0; red < 2; ++red)
    for (int rep = 0; rep < 2; ++rep)
      for (int mode = 0; mode < 2; ++mode) {
        run<<<sms * 4, 256>>>(X, Y, n_blocks, 50, mode, red, m[0], m[1], m[2], sink);  // warm
        cudaEventRecord(a);
        run<<<sms * 4, 256>>>(X, Y, n_blocks, iters, mode, red, m[0], m[1], m[2], sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double moved = (double)sms * 4 * 8 * iters * 2048.0 * (red ? 2 : 1);
        printf("red=%d mode=%d ms=%.3f GB/s=%.0f\n", red, mode, ms, moved / (ms / 1e3) / 1e9);
      }
  return 0;
}
