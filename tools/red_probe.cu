// Probe: random 32-byte f32 reductions into an L2-resident Y (the CSR
// kernel's transposed scatter, k = 8 f32): (0) two red.global.add.v4.f32 per
// row, (1) one TMA bulk reduction (cp.reduce.async.bulk .add.f32, 32 B from
// shared memory) per row.  Prints reductions per second for each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/red_probe tools/red_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void red_v4(float *Y, long long rows, int iters) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const long long r = (long long)(mix(t * 1000003ull + it) % (uint64_t)rows);
    float *y = Y + r * 8;
    const float v = 1.0f + it;
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(y), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(y + 4), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
  }
}

__global__ void red_bulk(float *Y, long long rows, int iters) {
  __shared__ __align__(128) float slot[256][2][8];
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int tid = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    const int b = it & 1;
    // the slot's previous bulk read must be done before it is rewritten
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    const long long r = (long long)(mix(t * 1000003ull + it) % (uint64_t)rows);
    const float v = 1.0f + it;
#pragma unroll
    for (int q = 0; q < 8; ++q) slot[tid][b][q] = v;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(&slot[tid][b][0]);
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 32;" ::"l"(Y + r * 8),
                 "r"(s)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const long long rows = 262144;  // 8 MB of Y: L2-resident, like the basis skeleton's Y
  float *Y;
  cudaMalloc(&Y, rows * 8 * 4);
  cudaMemset(Y, 0, rows * 8 * 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 400;
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 2; ++mode)
      for (int blocks_per_sm : {4, 8}) {
        const int grid = sms * blocks_per_sm;
        if (mode == 0) red_v4<<<grid, 256>>>(Y, rows, 10); else red_bulk<<<grid, 256>>>(Y, rows, 10);
        cudaEventRecord(a);
        if (mode == 0) red_v4<<<grid, 256>>>(Y, rows, iters); else red_bulk<<<grid, 256>>>(Y, rows, iters);
        cudaEventRecord(b);
        cudaError_t e = cudaEventSynchronize(b);
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)grid * 256 * iters;
        printf("%s blocks/SM=%d: %.3f ms, %.1f G row-reductions/s\n", mode ? "bulk 32B " : "2x red.v4", blocks_per_sm,
               ms, ops / (ms / 1e3) / 1e9);
      }
  return 0;
}
