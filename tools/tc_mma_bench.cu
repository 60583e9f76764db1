// Micro-benchmark: cycles per tcgen05.mma.kind::tf32 (M=128) for the operand
// modes the SpMM kernel uses, issued back to back by one thread, one CTA.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_mma_bench tc_mma_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

// mode: 0 SS K-major SW128 A, 1 SS MN-major BASE32B A, 2 TS (A in TMEM); nacc independent accumulators
__global__ void bench(int mode, int N, int nacc, int iters, long long *out, int style) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  for (int e = threadIdx.x; e < 65536 / 4; e += blockDim.x) ((float *)sm)[e] = 0.001f * (e % 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tmem_base;
  if (style == 2) tm = __shfl_sync(0xffffffffu, tm, 0);  // make it provably warp-uniform
  if (style >= 3) {
    if (tm != 0) __trap();  // (probe assumption)  // whole TMEM allocated by the only CTA on the SM: base is column 0
    tm = 0;
  }
  if (((style == 0 || style == 4 || style == 5) && threadIdx.x == 0) || ((style >= 1 && style != 4 && style != 5) && threadIdx.x < 32)) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode == 1 ? 1u : 0u) << 15) |
                           ((uint32_t)(N / 8) << 17) | (8u << 24);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    long long t0 = clock64();
    if (style == 5 || style == 6) {
      const uint64_t bd0 = sdesc(b0, 128, 2048, 0);
      const uint64_t ad0 = mode == 0 ? sdesc(a0, 16, 4096, 2) : sdesc(a0, 8192, 512, 1);
      const uint32_t d = tm + 128;
      for (int it = 0; it < iters; it += 8) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint64_t ad = ad0 + (uint64_t)(mode == 0 ? (((ks / 4) * 1024 + (ks % 4) * 32) >> 4) : ((ks * 1024) >> 4));
          const uint64_t bd = bd0 + (uint64_t)((ks * 256) >> 4);
          if (style == 6)
            asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|q, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(it + ks > 0)));
          else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(it + ks > 0)));
        }
      }
    } else
    for (int it = 0; it < iters; ++it) {
      const int ks = it & 7;
      const uint32_t d = tm + 128 + (uint32_t)((it % nacc) * N);
      const uint64_t bd = sdesc(b0 + ks * 256, 128, 2048, 0);
      const uint32_t acc = it >= nacc ? 1u : 0u;
      if (style >= 1 && style != 4) {
        asm volatile("{\n\t.reg .pred p, q;\n\telect.sync _|q, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t@q tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(sdesc(a0 + (ks / 4) * 1024 + (ks % 4) * 32, 16, 4096, 2)), "l"(bd), "r"(idesc), "r"(acc));
      } else if (mode == 0) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(sdesc(a0 + (ks / 4) * 1024 + (ks % 4) * 32, 16, 4096, 2)), "l"(bd), "r"(idesc), "r"(acc));
      } else if (mode == 1) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(sdesc(a0 + ks * 1024, 8192, 512, 1)), "l"(bd), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(tm + ks * 8), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
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
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

// CUTLASS-style issue: warp-uniform role branch (warp index via shfl), converged
// loop, descriptors from uniform sources, TMEM base 0, elect.sync around the MMA.
__global__ void bench2(int mode, int N, int iters, long long *out, int batched) {
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
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode == 1 ? 1u : 0u) << 15) |
                           ((uint32_t)(N / 8) << 17) | (8u << 24);
    const uint64_t bd0 = sdesc(smem_u32(sm + 32768), 128, 2048, 0);
    const uint64_t ad0 = mode == 0 ? sdesc(smem_u32(sm), 16, 4096, 2) : sdesc(smem_u32(sm), 8192, 512, 1);
    long long t0 = clock64();
    for (int it = 0; it < iters; it += 8) {
      if (batched) {
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint64_t ad = ad0 + (uint64_t)(mode == 0 ? (((ks / 4) * 1024 + (ks % 4) * 32) >> 4) : ((ks * 1024) >> 4));
            const uint64_t bd = bd0 + (uint64_t)((ks * 256) >> 4);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(128u), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(it + ks > 0)));
          }
        }
        __syncwarp();
        continue;
      }
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        const uint64_t ad = ad0 + (uint64_t)(mode == 0 ? (((ks / 4) * 1024 + (ks % 4) * 32) >> 4) : ((ks * 1024) >> 4));
        const uint64_t bd = bd0 + (uint64_t)((ks * 256) >> 4);
        if (elect_one())
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                       ::"r"(128u), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(it + ks > 0)));
        __syncwarp();
      }
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

int main() {
  long long *d, h[2];
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  const char *names[] = {"SS K-major SW128", "SS MN-major BASE32B", "TS (A in TMEM)"};
  cudaFuncSetAttribute(bench2, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int batched = 0; batched < 2; ++batched)
  for (int mode = 0; mode < 2; ++mode)
    for (int N : {16, 32, 128}) {
      bench2<<<1, 128, 65536 + 4096>>>(mode, N, 1024, d, batched);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("error bench2\n"); return 1; }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%s %-22s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", batched ? "cutlass-style+batched" : "cutlass-style", names[mode], N,
             (double)h[0] / 1024, (double)h[1] / 1024);
    }
  for (int style = 5; style < 5; ++style)
  for (int mode = 0; mode < 3; ++mode)
    for (int N : {16, 128})
      for (int nacc : {1}) {
        if (mode == 2) continue;
        if (128 + nacc * N > 512) continue;
        const int iters = 1024;
        bench<<<1, 128, 65536 + 4096>>>(mode, N, nacc, iters, d, style);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("%s %-22s N=%3d acc=%d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", style == 6 ? "warp+elect+unrolled+precomp" : style == 5 ? "unrolled+precomputed-desc" : style == 4 ? "lane0+const-tmem" : style == 3 ? "warp+elect+const-tmem" : style == 2 ? "warp+elect+shfl" : style ? "warp+elect" : "lane0-loop", names[mode], N, nacc,
               (double)h[0] / iters, (double)h[1] / iters);
      }
  return 0;
}
