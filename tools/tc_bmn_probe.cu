// Probe: tcgen05.mma kind::tf32 with A in TMEM (M = 128) and B in shared memory
// in the MN-major SWIZZLE_NONE canonical layout
//     B(kk, n) at (n % 4)·4 + (n / 4)·SBO + (kk % 8)·16 + (kk / 8)·LBO
// (idesc bit 16 = B MN-major), against the K-major layout the SpMM kernel
// uses today.  Prints the max |D − D_ref| of each over random data.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tc_bmn_probe tools/tc_bmn_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr int M = 128, N = 32, KK = 64;  // D = A (M×KK) · B (KK×N)

// mode 0: B K-major (n/8)·2048 + (kk/4)·128 + (n%8)·16 + (kk%4)·4, LBO 128, SBO 2048
// mode 1: B MN-major (n%4)·4 + (n/4)·128 + (kk%8)·16 + (kk/8)·(N/4·128), SBO 128, LBO N·32
// mode 2: mode 1 with LBO / SBO swapped in the descriptor (which field is which)
__global__ void probe(const float *A, const float *B, float *D, int mode) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < KK * N; e += blockDim.x) {
    const int kk = e / N, n = e % N;
    unsigned off = mode == 0 ? (unsigned)((n / 8) * 2048 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4)
                             : (unsigned)((n % 4) * 4 + (n / 4) * 128 + (kk % 8) * 16 + (kk / 8) * (N / 4) * 128);
    *reinterpret_cast<float *>(sm + off) = B[kk * N + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // A row m = TMEM lane m, columns 0..63
  {
    const int m = tid;  // 128 threads
    for (int c0 = 0; c0 < KK; c0 += 8) {
      uint32_t r[8];
      for (int e = 0; e < 8; ++e) r[e] = __float_as_uint(A[m * KK + c0 + e]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       ((uint32_t)(32 * warp) << 16) + (uint32_t)c0),
                   "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((mode ? 1u : 0u) << 16) | ((uint32_t)(N / 8) << 17) |
                           ((uint32_t)(M / 16) << 24);
    const uint32_t base = smem_u32(sm);
    for (int ks = 0; ks < KK / 8; ++ks) {
      uint64_t bd;
      if (mode == 0) bd = sdesc(base + ks * 256, 128, 2048);
      else if (mode == 1) bd = sdesc(base + ks * (N / 4) * 128, (N / 4) * 128, 128);
      else bd = sdesc(base + ks * (N / 4) * 128, 128, (N / 4) * 128);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(256u),
                   "r"((uint32_t)(ks * 8)), "l"(bd), "r"(idesc), "r"((uint32_t)(ks > 0)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int m = tid;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(((uint32_t)(32 * warp) << 16) + 256u + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int e = 0; e < 8; ++e) D[m * N + c0 + e] = __uint_as_float(r[e]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u));
}

// Decode: smem word w = w (w < 2048: exact in TF32), A = I (rows 0..63), so
// D[kk][n] names the word the MMA read as B(kk, n) for an MN-major descriptor
// with LBO = 256 B and SBO = 1024 B.
__global__ void decode(float *D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 2048; e += blockDim.x) reinterpret_cast<float *>(sm)[e] = (float)e;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int m = tid;
    for (int c0 = 0; c0 < 8; c0 += 8) {
      uint32_t r[8];
      for (int e = 0; e < 8; ++e) r[e] = __float_as_uint((m == c0 + e) ? 1.0f : 0.0f);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       ((uint32_t)(32 * warp) << 16) + (uint32_t)c0),
                   "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                   : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(N / 8) << 17) |
                           ((uint32_t)(M / 16) << 24);
    const uint64_t bd = sdesc(smem_u32(sm), 256, 1024);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(256u),
                 "r"(0u), "l"(bd), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
                   : "=r"(ok)
                   : "r"(smem_u32(&bar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  {
    const int m = tid;
    for (int c0 = 0; c0 < N; c0 += 8) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(((uint32_t)(32 * warp) << 16) + 256u + (uint32_t)c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int e = 0; e < 8; ++e) D[m * N + c0 + e] = __uint_as_float(r[e]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u));
}

int main() {
  std::vector<float> A(M * KK), B(KK * N), D(M * N);
  srand(1);
  // values exactly representable in TF32 so the reference is exact
  for (auto &x : A) x = (float)((rand() % 33) - 16) / 16.0f;
  for (auto &x : B) x = (float)((rand() % 33) - 16) / 16.0f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  const char *names[] = {"K-major  (LBO 128, SBO 2048)", "MN-major (LBO = K-group stride, SBO = MN-chunk stride)",
                         "MN-major (LBO = MN-chunk stride, SBO = K-group stride)"};
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    probe<<<1, 128, 64 * 1024>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < KK; ++k) s += (double)A[m * KK + k] * B[k * N + n];
        err = fmax(err, fabs(s - D[m * N + n]));
      }
    printf("%s: max err %.3g\n", names[mode], err);
  }
  cudaMemset(dD, 0, D.size() * 4);
  decode<<<1, 128, 64 * 1024>>>(dD);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("decode failed\n"); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  printf("MN-major decode (LBO 256, SBO 1024): word read as B(kk, n), kk = 0..7 rows, n = 0..31 columns\n");
  for (int kk = 0; kk < 8; ++kk) {
    for (int n = 0; n < N; ++n) printf("%5d", (int)D[kk * N + n]);
    printf("\n");
  }
  return 0;
}
