// Probe (round 2) for a pre-split tensor-core tile layout "tc2": per 32-column
// block b, [T block | T_lo block] (8 KB each, SWIZZLE_128B_BASE32B rows of 4),
// read as (a) a K-major A = [T; T_lo] (M = 128 rows, the direct product) and
// (b) an MN-major A = [Tᵀ_cb0; T_loᵀ_cb0; Tᵀ_cb1; T_loᵀ_cb1] (the transposed
// product).  Derived from tools/tc_probe.cu (round 1).
//
// The host builds the exact shared-memory image of the A operand for each
// variant; the kernel copies it verbatim into smem, runs 8 K-steps of
// M=128, N=16, K=8 tf32 MMAs into TMEM, reads TMEM back (row m -> lane m) and
// the host compares with a TF32-truncated CPU product.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc_probe tc_probe.cu
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

struct Variant {
  const char *name;
  int a_mn;         // 0 K-major, 1 MN-major
  int layout;       // descriptor layout type
  uint32_t lbo, sbo;
  uint32_t kstep_bytes;  // start-address advance per K-step (or -1: special)
};

__global__ void probe(const float *Aimg, const float *Bimg, float *out, Variant v) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float *op = (float *)sm;            // 64 KB A image
  float *Bs = (float *)(sm + 65536);  // 4 KB B image
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  int tid = threadIdx.x;
  for (int e = tid; e < 16384; e += blockDim.x) op[e] = Aimg[e];
  for (int e = tid; e < 1024; e += blockDim.x) Bs[e] = Bimg[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tm = tmem_base;
  const uint32_t a_major = (v.a_mn == 1 || v.a_mn == 4) ? 1u : 0u;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (a_major << 15) | (2u << 17) | (8u << 24);
  if (v.a_mn == 2) {
    // A in TMEM columns [32, 96): thread m writes row m (64 values) of the row-major image at op
    int w = tid / 32, lane = tid % 32;
    int m = 32 * w + lane;
    for (int half = 0; half < 4; ++half) {
      uint32_t r[16];
      for (int j = 0; j < 16; ++j) r[j] = __float_as_uint(op[m * 64 + half * 16 + j]);
      uint32_t addr = tm + ((uint32_t)(32 * w) << 16) + 32 + half * 16;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                   ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                     "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (tid == 0) {
    uint32_t a0 = smem_u32(op), b0 = smem_u32(Bs);
    const uint32_t idesc_k = idesc & ~(3u << 15);
    const int nks = (int)(v.kstep_bytes >> 16);
    for (int ks = 0; ks < nks; ++ks) {
      uint64_t bd = sdesc(b0 + ks * 256, 128, 2048, 0);
      if (v.a_mn == 2) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
            "r"(tm + 32 + ks * 8), "l"(bd), "r"(idesc_k), "r"((uint32_t)(ks > 0)));
        continue;
      }
      uint32_t aoff = v.a_mn == 3 ? (ks / 4) * 16384 + (ks % 4) * 32
                      : v.a_mn ? ks * (v.kstep_bytes & 0xFFFFu) : (ks / 4) * 1024 + (ks % 4) * 32;
      mma_tf32(tm, sdesc(a0 + aoff, v.lbo, v.sbo, v.layout), bd, idesc, ks > 0);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0,1,0,p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  int w = tid / 32, lane = tid % 32;
  if (w < 4) {
    uint32_t r[16];
    uint32_t addr = tm + ((uint32_t)(32 * w) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    int m = 32 * w + lane;
    for (int j = 0; j < 16; ++j) out[m * 16 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

static float tf32_trunc(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

int main(int argc, char **argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int nks = argc > 2 ? atoi(argv[2]) : 8;
  std::vector<float> T0(4096), T1(4096), X(64 * 16);
  srand(1);
  for (auto &x : T0) x = (rand() % 2001 - 1000) / 1000.0f;
  for (auto &x : T1) x = (rand() % 2001 - 1000) / 1000.0f;
  for (auto &x : X) x = (rand() % 2001 - 1000) / 1000.0f;
  // B image: K-major INTERLEAVE (verified): (n/8)*2048 + (k/4)*128 + (n%8)*16 + (k%4)*4
  std::vector<float> Bimg(1024);
  for (int k = 0; k < 64; ++k)
    for (int n = 0; n < 16; ++n) Bimg[((n / 8) * 2048 + (k / 4) * 128 + (n % 8) * 16 + (k % 4) * 4) / 4] = X[k * 16 + n];

  // variants: A = [T0ᵀ ; T1ᵀ] (M = column index c of tile s = m/64, K = row r) unless K-major
  Variant vars[] = {
      {"tc2 K-major BASE32B sbo=1024 (direct A=[T;Tlo])", 3, 1, 16, 1024, 0},
      {"tc2 K-major BASE32B lbo=0 sbo=1024", 3, 1, 0, 1024, 0},
      {"tc2 K-major SW128 sbo=1024 (expected BAD)", 3, 2, 16, 1024, 0},
      {"tc2 MN-major BASE32B lbo=8192 sbo=512 (transposed)", 4, 1, 8192, 512, 1024},
  };
  float *dA, *dB, *dO;
  cudaMalloc(&dA, 65536);
  cudaMalloc(&dB, 4096);
  cudaMalloc(&dO, 128 * 16 * 4);
  cudaMemcpy(dB, Bimg.data(), 4096, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  int nv = sizeof(vars) / sizeof(vars[0]);
  for (int vi = 0; vi < nv; ++vi) {
    if (only >= 0 && vi != only) continue;
    Variant v = vars[vi];
    v.kstep_bytes = (v.kstep_bytes & 0xFFFFu) | ((uint32_t)nks << 16);  // K-steps to run (high half)
    std::vector<float> A(16384, 0.0f);
    auto put = [&](uint32_t byte, float val) { A[byte / 4] = val; };
    for (int s = 0; s < 2; ++s)
      for (int r = 0; r < 64; ++r)
        for (int c = 0; c < 64; ++c) {
          float val = s ? T1[r * 64 + c] : T0[r * 64 + c];
          // tc2: block b = c/32 at b·16384; T at +0, T_lo (here T1) at +8192
          uint32_t inatom = (r % 4) * 128 + (c % 32) * 4;
          inatom ^= ((inatom >> 7) & 3) << 5;
          put((c / 32) * 16384 + s * 8192 + (r / 4) * 512 + inatom, val);
        }
    cudaMemcpy(dA, A.data(), 65536, cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, 128 * 16 * 4);
    probe<<<1, 128, 65536 + 4096>>>(dA, dB, dO, v);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%-44s CUDA error %s\n", v.name, cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> O(128 * 16);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0, maxout = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 16; ++n) {
        double ref = 0;
        const int kmax = 8 * ((int)(v.kstep_bytes >> 16));
        for (int k = 0; k < kmax; ++k) {
          float a;
          if (v.a_mn == 3) {  // K-major: M = [T rows ; T1 rows], K = column
            a = (m < 64) ? T0[m * 64 + k] : T1[(m - 64) * 64 + k];
          } else {  // MN-major: M groups of 32 = [T cb0, T1 cb0, T cb1, T1 cb1], K = row
            const int g = m / 32, cc = (g / 2) * 32 + m % 32;
            a = (g % 2) ? T1[k * 64 + cc] : T0[k * 64 + cc];
          }
          ref += (double)tf32_trunc(a) * (double)tf32_trunc(X[k * 16 + n]);
        }
        maxerr = fmax(maxerr, fabs(ref - O[m * 16 + n]));
        maxref = fmax(maxref, fabs(ref));
        maxout = fmax(maxout, fabs(O[m * 16 + n]));
      }
    printf("%-44s max|err|=%.3e max|ref|=%.3e max|out|=%.3e %s\n", v.name, maxerr, maxref, maxout,
           maxerr <= 1e-4 * maxref ? "OK" : "BAD");
  }
  return 0;
}
