// Micro-benchmark: cycles per tcgen05.mma.kind::tf32 with A in TMEM (TS mode)
// against A in shared memory (SS mode), M = 128 (and M = 64), N = 16…128, one
// accumulator or two alternating ones, issued back to back by one elected
// thread of one CTA.  Decides the operand placement of the split-TF32 SpMM
// kernel (profiles/r02/tc_ts_bench.txt).
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_ts_bench tools/tc_ts_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

// TS: A in TMEM (columns 0..63, K = 8 per MMA); else SS K-major SW128 A.
// Everything compile-time so the MMA operands are uniform immediates.
template <bool TS, int M, int N, int NACC>
__global__ void bench(int iters, long long *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  for (int e = threadIdx.x; e < 65536 / 4; e += blockDim.x) ((float *)sm)[e] = 0.001f * (e % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp_idx = __shfl_sync(0xffffffffu, (int)threadIdx.x / 32, 0);
  if (warp_idx == 0 && elect_one()) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp_idx == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tmem_base != 0) __trap();
  if (warp_idx == 0) {
    constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N / 8) << 17) | ((uint32_t)(M / 16) << 24);
    const uint64_t bd0 = sdesc(smem_u32(sm + 32768), 128, 2048, 0);
    const uint64_t ad0 = sdesc(smem_u32(sm), 16, 4096, 2);
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
      if (elect_one()) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          constexpr uint32_t d0 = 256u;
          const uint32_t d = d0 + (uint32_t)((ks % NACC) * N);
          const uint64_t bd = bd0 + (uint64_t)((ks * 256) >> 4);
          if constexpr (TS) {
            asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;"
                         ::"r"(d), "r"((uint32_t)(ks * 8)), "l"(bd), "r"(idesc));
          } else {
            const uint64_t ad = ad0 + (uint64_t)((((ks / 4) * 1024 + (ks % 4) * 32)) >> 4);
            asm volatile("tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, 1;"
                         ::"r"(d), "l"(ad), "l"(bd), "r"(idesc));
          }
        }
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    __syncwarp();
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar)));
    long long t2 = clock64();
    if (threadIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp_idx == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u));
}

template <bool TS, int M, int N, int NACC>
int run1(long long *d) {
  long long h[2];
  cudaFuncSetAttribute(bench<TS, M, N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const int iters = 4096;
  bench<TS, M, N, NACC><<<1, 128, 65536 + 4096>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("error TS=%d M=%d N=%d: %s\n", TS, M, N, cudaGetErrorString(e));
    return 1;
  }
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%s M=%3d N=%3d nacc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", TS ? "TS (A in TMEM)" : "SS K-major   ", M,
         N, NACC, (double)h[0] / iters, (double)h[1] / iters);
  return 0;
}

int main() {
  long long *d;
  cudaMalloc(&d, 16);
  int rc = 0;
  rc |= run1<true, 128, 16, 1>(d); rc |= run1<true, 128, 16, 2>(d); rc |= run1<true, 128, 32, 1>(d);
  rc |= run1<true, 128, 64, 1>(d); rc |= run1<true, 128, 128, 1>(d); rc |= run1<true, 128, 256, 1>(d);
  rc |= run1<true, 64, 16, 1>(d); rc |= run1<true, 64, 32, 1>(d); rc |= run1<true, 64, 64, 1>(d);
  rc |= run1<false, 128, 16, 1>(d); rc |= run1<false, 128, 32, 1>(d); rc |= run1<false, 128, 64, 1>(d);
  rc |= run1<false, 128, 128, 1>(d); rc |= run1<false, 64, 16, 1>(d); rc |= run1<false, 64, 64, 1>(d);
  return rc;
}
