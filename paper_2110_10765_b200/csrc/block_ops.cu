// Tall-skinny block products for the eigensolver (C-ABI cim_gram, cim_tsmm).
//
// cim_gram: G = Aᵀ·B in float64.
//
// LOBPCG (config C5, lobpcg.py) needs, per iteration, several Gram matrices of
// row-distributed blocks with n = 2²² rows and ≤ 64 columns (Sᵀ·AS, Sᵀ·S,
// Rᵀ·R, the Cholesky-QR passes).  cuBLAS treats them as M, N ≤ 64, K = 4M
// GEMMs and torch first materialises float64 copies of both operands; this
// kernel reads the f32 (or f64) operands once from HBM, widens them to f64 in
// shared memory and accumulates in f64 — the product is HBM-bound
// (rows·(ca+cb)·s bytes) with DFMA work rows·ca·cb.
//
// Grid-stride over slabs of rows (~24 KB per stage), a kGramStages-deep ring
// in shared memory: block-major operands (the eigensolver's work buffer) are
// staged by one thread with one bulk copy per 8-column block (cp.async.bulk
// on an mbarrier), other layouts by all threads with cp.async.  Each thread
// owns an 8×8 block of G for a residue class of the slab's rows.  Per-CTA
// partials go to a workspace and a second kernel sums them in a fixed order
// (bit-reproducible run to run).
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>

#include <cuda_runtime.h>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace {

constexpr int kGramThreads = 128;
constexpr int kMaxCols = 64;

// A column-blocked tall operand: element (r, c) at p + (c >> bw_shift)·bstride
// + r·ld + (c & (bw-1)).  One plain row-major block is bw = 64, bstride = 0.
struct Operand {
  const void *p;
  long long ld, bstride;
  int bw_shift, cols;
};

__host__ __device__ __forceinline__ int pad8(int c) { return (c + 7) & ~7; }

// Rows per slab: ~24 KB per stage whatever the column counts (6K f32 or 3K
// f64 elements), kGramStages stages in flight per CTA.
constexpr int kGramStages = 4;
__host__ __device__ __forceinline__ int slab_rows(int cap, int cbp, int es) {
  const int r = (es == 4 ? 6144 : 3072) / (cap + cbp);
  return r < 32 ? 32 : (r > 1024 ? 1024 : (r & ~7));
}

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// Shared-memory slab layout: each operand as 8-column blocks [blk][row][8],
// consecutive blocks skewed by 8 elements so the 8×8 register tiles of one
// warp (same row, different blocks) hit different banks.
__host__ __device__ __forceinline__ int sblk_stride(int slab) { return slab * 8 + 8; }

// Load modes of an operand for one slab (decided once per launch):
//  0 = blocked, bw = 8, ld = 8: each 8-column block of the slab is one
//      contiguous run → 16-byte copies with trivial addressing;
//  1 = row-major, 16-byte aligned, ld % (16/s) == 0: 16-byte copies;
//  2 = anything else: element copies.
template <typename T>
__device__ __forceinline__ void load_operand(T *dst, const Operand &o, int mode, int slab, long long r0, int nr,
                                             float inv_c) {
  constexpr int V = 16 / sizeof(T);  // elements per 16-byte chunk
  const T *base = static_cast<const T *>(o.p);
  const int sbs = sblk_stride(slab);
  const int nb8 = (o.cols + 7) / 8;
  if (mode == 0) {
    const int per = nr * 8 / V;  // chunks per block
    for (int b = 0; b < nb8; ++b) {
      const T *src = base + (long long)b * o.bstride + r0 * 8;
      T *d = dst + b * sbs;
      for (int e = threadIdx.x; e < per; e += blockDim.x) cp_async16(d + e * V, src + e * V);
    }
  } else if (mode == 1) {
    const int cpr = (o.cols + V - 1) / V;  // chunks per row
    const int n = nr * cpr;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int r = e / cpr, ch = e - r * cpr, c = ch * V;
      cp_async16(dst + (c >> 3) * sbs + r * 8 + (c & 7), base + (r0 + r) * o.ld + c);
    }
  } else {
    const int n = nr * o.cols, mask = (1 << o.bw_shift) - 1;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
      const int r = __float2int_rz(((float)e + 0.5f) * inv_c);
      const int c = e - r * o.cols;
      const T *src = base + (long long)(c >> o.bw_shift) * o.bstride + (r0 + r) * o.ld + (c & mask);
      T *d = dst + (c >> 3) * sbs + r * 8 + (c & 7);
      if constexpr (sizeof(T) == 4)
        cp_async4(d, src);
      else
        cp_async8(d, src);
    }
  }
}

template <typename T>
__device__ __forceinline__ void load8(double (&d)[8], const T *p) {
  if constexpr (sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4 *>(p);
    const float4 b = *reinterpret_cast<const float4 *>(p + 4);
    d[0] = a.x, d[1] = a.y, d[2] = a.z, d[3] = a.w, d[4] = b.x, d[5] = b.y, d[6] = b.z, d[7] = b.w;
  } else {
    const double4 a = *reinterpret_cast<const double4 *>(p);
    const double4 b = *reinterpret_cast<const double4 *>(p + 4);
    d[0] = a.x, d[1] = a.y, d[2] = a.z, d[3] = a.w, d[4] = b.x, d[5] = b.y, d[6] = b.z, d[7] = b.w;
  }
}

// A kGramStages-deep cp.async ring of slabs (input dtype); each thread owns
// an 8×8 block of G for one residue class of a slab's rows and widens its 16
// operands per row to f64 on use (16 F2F per 64 DFMA).
// block_mask: bit (bi·nbj + bj) set ⇔ output block (bi, bj) is computed (a
// caller exploiting symmetry skips the mirrored half; skipped blocks are 0).
// a_in_b: A is the first ca columns of B (same buffer and block layout; B == A
// is the special case): only B is staged and A's blocks alias B's first ones.
// FAST (f32 operands, CIM_GRAM_FAST): products and partial sums in f32
// (FFMA2 on register pairs) over at most kFastRun rows, then widened into the
// f64 accumulators — 1/kFastRun of the conversions and no DFMA in the row
// loop; each partial is a ≤ kFastRun-term f32 sum (relative error
// ≲ kFastRun·2⁻²⁴ of its absolute sum), everything above it f64.
constexpr int kFastRun = 32;

__device__ __forceinline__ unsigned long long gfma2(float t, unsigned long long x, unsigned long long acc) {
  unsigned long long tt, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(tt) : "f"(t));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(tt), "l"(x), "l"(acc));
  return r;
}

// NT threads per CTA, each owning an 8 × JW block of G.  (JW = 4 with 256
// threads halves the per-thread accumulators and doubles the resident warps
// of the 254-register 8 × 8 FAST version, but loads 1.5× the shared bytes
// per FMA: 0.382 vs 0.351 ms per LOBPCG iteration's Gram passes — 8 × 8
// stays the launch.)
template <typename T, bool FAST, int NT = kGramThreads, int JW = 8>
__global__ void __launch_bounds__(NT) gram_partial_kernel(const Operand A, const Operand B, int mode_a,
                                                                    int mode_b, long long rows,
                                                                    double *__restrict__ part, uint64_t block_mask,
                                                                    bool a_in_b) {
  extern __shared__ __align__(32) unsigned char smem_raw[];
  const int ca = A.cols, cb = B.cols;
  const int cap = pad8(ca), cbp = pad8(cb);
  const int nbi_st = a_in_b ? 0 : cap / 8;  // staged A blocks (B's are always staged)
  const int kSlab = slab_rows(8 * nbi_st, cbp, (int)sizeof(T));
  const int sbs = sblk_stride(kSlab);
  const int nbi = cap / 8, nbj = cbp / 8, nblk = nbi * nbj;
  const uint64_t live = (nblk >= 64 ? ~0ull : ((1ull << nblk) - 1)) & block_mask;
  constexpr int NH = 8 / JW;  // threads per 8×8 output block
  const int nact = max(1, __popcll(live)) * NH;
  const int stage_elems = (nbi_st + nbj) * sbs;
  T *ring = reinterpret_cast<T *>(smem_raw);
  __shared__ uint64_t full[kGramStages];  // bulk mode: slab k landed in stage k % S
  const bool bulk = mode_b == 0 && (a_in_b || mode_a == 0);
  if (bulk && threadIdx.x == 0) {
    for (int q = 0; q < kGramStages; ++q) cim::mbar_init(&full[q], 1);
    cim::fence_mbar_init();
  }
  const int red_cap = (int)((kGramStages * (size_t)stage_elems * sizeof(T)) / (sizeof(double) * cap * cbp));
  const int split = min(NT / nact, red_cap);  // row residue classes (≥ 1)
  const int t = threadIdx.x;
  const int a_idx = t % nact, grp = t / nact;
  const bool active = grp < split && live != 0;
  int blk = 0;
  const int jh = a_idx % NH;  // which JW columns of the block
  {  // the (a_idx / NH)-th live block
    uint64_t m = live;
    for (int q = 0; q < a_idx / NH; ++q) m &= m - 1;
    blk = m ? __ffsll((long long)m) - 1 : 0;
  }
  const int bi = blk / nbj, bj = blk % nbj;
  const float inv_ca = 1.0f / (float)ca, inv_cb = 1.0f / (float)cb;
  for (int e = t; e < kGramStages * stage_elems; e += NT) ring[e] = T(0);  // pads stay zero
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before the bulk copies' writes
  __syncthreads();
  double acc[8][JW];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < JW; ++j) acc[i][j] = 0.0;
  unsigned long long acc2[8][JW / 2];  // FAST: f32 pairs (row i, columns 2jp, 2jp+1)
  int run = 0;
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int jp = 0; jp < JW / 2; ++jp) {
        float lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc2[i][jp]));
        acc[i][2 * jp] += (double)lo;
        acc[i][2 * jp + 1] += (double)hi;
        acc2[i][jp] = 0ull;
      }
    run = 0;
  };
  if constexpr (FAST) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int jp = 0; jp < JW / 2; ++jp) acc2[i][jp] = 0ull;
  }

  const long long nslabs = (rows + kSlab - 1) / kSlab;
  const uint64_t pol = cim::policy_evict_first();  // streamed once
  auto issue = [&](long long k) {  // this CTA's k-th slab into ring stage k % S (rows ≥ nr never read)
    const long long sl = blockIdx.x + k * gridDim.x;
    if (bulk) {  // one bulk copy per 8-column block, issued by thread 0
      if (threadIdx.x == 0 && sl < nslabs) {
        const long long r0 = sl * kSlab;
        const int nr = (int)min((long long)kSlab, rows - r0);
        T *st = ring + (size_t)(k % kGramStages) * stage_elems;
        const uint32_t bytes = (uint32_t)nr * 8 * sizeof(T);
        cim::mbar_arrive_expect_tx(&full[k % kGramStages], bytes * (nbi_st + nbj));
        for (int b = 0; b < nbi_st; ++b)
          cim::bulk_g2s(st + b * sbs, static_cast<const T *>(A.p) + (long long)b * A.bstride + r0 * 8, bytes,
                        &full[k % kGramStages], pol);
        for (int b = 0; b < nbj; ++b)
          cim::bulk_g2s(st + (nbi_st + b) * sbs, static_cast<const T *>(B.p) + (long long)b * B.bstride + r0 * 8,
                        bytes, &full[k % kGramStages], pol);
      }
      return;
    }
    if (sl < nslabs) {
      const long long r0 = sl * kSlab;
      const int nr = (int)min((long long)kSlab, rows - r0);
      T *st = ring + (size_t)(k % kGramStages) * stage_elems;
      if (!a_in_b) load_operand(st, A, mode_a, kSlab, r0, nr, inv_ca);
      load_operand(st + nbi_st * sbs, B, mode_b, kSlab, r0, nr, inv_cb);
    }
    cp_async_commit();  // possibly empty group: keeps the wait arithmetic uniform
  };
  for (int k = 0; k < kGramStages - 1; ++k) issue(k);
  for (long long k = 0;; ++k) {
    const long long sl = blockIdx.x + k * gridDim.x;
    if (sl >= nslabs) break;
    if (bulk)
      cim::mbar_wait(&full[k % kGramStages], (uint32_t)((k / kGramStages) & 1));
    else
      cp_async_wait<kGramStages - 2>();  // slab k has landed (this thread's copies) ...
    __syncthreads();                     // ... everyone's, and slab k-1's stage is free
    issue(k + kGramStages - 1);
    const long long r0 = sl * kSlab;
    const int nr = (int)min((long long)kSlab, rows - r0);
    const T *sa = ring + (size_t)(k % kGramStages) * stage_elems + bi * sbs;
    const T *sb = ring + (size_t)(k % kGramStages) * stage_elems + (nbi_st + bj) * sbs + jh * JW;
    if (active) {
      if constexpr (FAST) {
        for (int r = grp; r < nr; r += split) {
          const float4 a0 = *reinterpret_cast<const float4 *>(sa + r * 8);
          const float4 a1 = *reinterpret_cast<const float4 *>(sa + r * 8 + 4);
          const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          unsigned long long bv[JW / 2];
#pragma unroll
          for (int q = 0; q < JW / 4; ++q) {
            const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(sb + r * 8 + 4 * q);
            bv[2 * q] = b.x, bv[2 * q + 1] = b.y;
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int jp = 0; jp < JW / 2; ++jp) acc2[i][jp] = gfma2(av[i], bv[jp], acc2[i][jp]);
          if (++run == kFastRun) flush();
        }
      } else {
        for (int r = grp; r < nr; r += split) {
          static_assert(FAST || JW == 8, "the exact path owns whole 8×8 blocks");
          double av[8], bv[8];
          load8<T>(av, sa + r * 8);
          load8<T>(bv, sb + r * 8);
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < JW; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
        }
      }
    }
  }
  if constexpr (FAST) flush();
  cp_async_wait<0>();
  // CTA reduction over the row residue classes (fixed order) in the ring
  __syncthreads();
  double *red = reinterpret_cast<double *>(smem_raw);
  if (active) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < JW; ++j) red[(size_t)grp * cap * cbp + (8 * bi + i) * cbp + 8 * bj + jh * JW + j] = acc[i][j];
  }
  __syncthreads();
  double *out = part + (size_t)blockIdx.x * ca * cb;
  for (int e = t; e < ca * cb; e += NT) {
    const int i = e / cb, j = e % cb;
    double s = 0.0;
    if ((live >> ((i >> 3) * nbj + (j >> 3))) & 1ull)
      for (int g = 0; g < split; ++g) s += red[(size_t)g * cap * cbp + i * cbp + j];
    out[e] = s;
  }
}

// One warp per output entry: lane l sums partials l, l+32, … then a fixed
// butterfly — deterministic, and ~nparts/32 dependent loads instead of nparts.
__global__ void gram_sum_kernel(const double *__restrict__ part, int nparts, int count, double *__restrict__ out) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (e >= count) return;
  double s = 0.0;
  for (int p = lane; p < nparts; p += 32) s += part[(size_t)p * count + e];
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[e] = s;
}

size_t gram_smem(int ca, int cb, size_t es, bool a_in_b = false) {
  const int cap = a_in_b ? 0 : pad8(ca), cbp = pad8(cb);
  return (size_t)kGramStages * ((cap + cbp) / 8) * sblk_stride(slab_rows(cap, cbp, (int)es)) * es;
}

int load_mode(const Operand &o, size_t es) {
  const int V = 16 / (int)es;
  const bool aligned = !(reinterpret_cast<uintptr_t>(o.p) & 15);
  if (aligned && o.bw_shift == 3 && o.ld == 8 && (o.bstride % V) == 0) return 0;
  if (aligned && (o.cols <= (1 << o.bw_shift)) && (o.ld % V) == 0 && (o.cols % V) == 0) return 1;
  return 2;
}

int gram_grid(long long rows, int ca, int cb, bool a_in_b = false, int es = 4) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int kSlab = slab_rows(a_in_b ? 0 : pad8(ca), pad8(cb), es);
  const long long slabs = (rows + kSlab - 1) / kSlab;
  return (int)std::min<long long>(slabs > 0 ? slabs : 1, 2LL * sms);
}

int bw_shift_of(int32_t bw) {
  for (int s = 2; s <= 6; ++s)
    if (bw == (1 << s)) return s;
  return -1;
}

int gram_impl(const Operand &A, const Operand &B, long long rows, int32_t dtype, double *out, void *workspace,
              uint64_t ws_bytes, cudaStream_t stream, uint64_t block_mask = ~0ull, uint32_t flags = 0) {
  const int ca = A.cols, cb = B.cols;
  if (ca < 1 || cb < 1 || ca > kMaxCols || cb > kMaxCols)
    return cim::set_error(CIM_EINVAL, "column counts must be in [1, 64]");
  if (rows < 0) return cim::set_error(CIM_EINVAL, "rows must be >= 0");
  if (dtype != CIM_F32 && dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (!out || (rows > 0 && (!A.p || !B.p))) return cim::set_error(CIM_EINVAL, "NULL pointer");
  const size_t es = dtype == CIM_F32 ? 4 : 8;
  // A = the first ca columns of B (B == A, or SᵀAS-style [S]ᵀ[S AS]): stage B only
  const bool a_in_b = A.p == B.p && A.ld == B.ld && A.bstride == B.bstride && A.bw_shift == B.bw_shift &&
                      A.cols <= B.cols;
  const int grid = gram_grid(rows, ca, cb, a_in_b, (int)es);  // ≤ the grid cim_gram_workspace_bytes assumed
  const uint64_t need = (uint64_t)grid * ca * cb * sizeof(double);
  if (!workspace || ws_bytes < need)
    return cim::set_error(CIM_EINVAL, "workspace must hold " + std::to_string(need) + " bytes");
  const size_t smem = gram_smem(ca, cb, es, a_in_b);
  const int ma = load_mode(A, es), mb = load_mode(B, es);
  if (block_mask == 0) block_mask = ~0ull;
  cudaError_t e;
  auto run = [&](auto kern, int nt) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      kern<<<grid, nt, smem, stream>>>(A, B, ma, mb, rows, static_cast<double *>(workspace), block_mask, a_in_b);
  };
  if (dtype == CIM_F32 && (flags & CIM_GRAM_FAST))
    run(gram_partial_kernel<float, true>, kGramThreads);
  else if (dtype == CIM_F32)
    run(gram_partial_kernel<float, false>, kGramThreads);
  else
    run(gram_partial_kernel<double, false>, kGramThreads);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("gram_partial_kernel: ") + cudaGetErrorString(e));
  const int count = ca * cb;
  gram_sum_kernel<<<(count * 32 + 255) / 256, 256, 0, stream>>>(static_cast<const double *>(workspace), grid, count, out);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("gram_sum_kernel: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace

extern "C" uint64_t cim_gram_workspace_bytes(int64_t rows, int32_t ca, int32_t cb) {
  if (rows < 0 || ca < 1 || cb < 1) return 0;
  // the largest grid any dtype / aliasing uses (f64: the smallest slabs)
  return (uint64_t)gram_grid(rows, ca, cb, false, 8) * (uint64_t)ca * (uint64_t)cb * sizeof(double);
}

extern "C" int cim_gram(const void *A, int64_t lda, int32_t ca, const void *B, int64_t ldb, int32_t cb, int64_t rows,
                        int32_t dtype, double *out, void *workspace, uint64_t ws_bytes, void *stream_) {
  cim::clear_error();
  if (lda < ca || ldb < cb) return cim::set_error(CIM_EINVAL, "leading dimensions must cover the columns");
  const Operand a{A, lda, 0, 6, ca}, b{B, ldb, 0, 6, cb};
  return gram_impl(a, b, rows, dtype, out, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream_));
}

extern "C" int cim_gram_blocked_ex(const void *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t ca,
                                   const void *B, int64_t ldb, int32_t b_bw, int64_t b_bstride, int32_t cb,
                                   int64_t rows, int32_t dtype, double *out, void *workspace, uint64_t ws_bytes,
                                   uint64_t block_mask, uint32_t flags, void *stream_) {
  cim::clear_error();
  const int sa = bw_shift_of(a_bw), sb = bw_shift_of(b_bw);
  if (sa < 0 || sb < 0) return cim::set_error(CIM_EINVAL, "block widths must be 4, 8, 16, 32 or 64");
  if (lda < std::min(a_bw, ca) || ldb < std::min(b_bw, cb))
    return cim::set_error(CIM_EINVAL, "leading dimensions must cover a block");
  if (flags & ~(uint32_t)CIM_GRAM_FAST) return cim::set_error(CIM_EINVAL, "unknown gram flags");
  const Operand a{A, lda, a_bstride, sa, ca}, b{B, ldb, b_bstride, sb, cb};
  return gram_impl(a, b, rows, dtype, out, workspace, ws_bytes, reinterpret_cast<cudaStream_t>(stream_), block_mask,
                   flags);
}

extern "C" int cim_gram_blocked(const void *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t ca,
                                const void *B, int64_t ldb, int32_t b_bw, int64_t b_bstride, int32_t cb, int64_t rows,
                                int32_t dtype, double *out, void *workspace, uint64_t ws_bytes, uint64_t block_mask,
                                void *stream_) {
  return cim_gram_blocked_ex(A, lda, a_bw, a_bstride, ca, B, ldb, b_bw, b_bstride, cb, rows, dtype, out, workspace,
                             ws_bytes, block_mask, 0u, stream_);
}

// ---------------------------------------------------------------------------
// Tall-skinny block times small matrix:  Out = alpha·A·C + beta·Out
// (C-ABI cim_tsmm).  A: rows × q (lda), C: q × p row-major f32 (device),
// Out: rows × p (ldo); q, p ≤ 64.  The eigensolver's block updates
// (projections, Cholesky-QR back-substitution, Ritz-vector assembly) write
// straight into column slots of a shared [P X W | AP AX AW] buffer; cuBLAS
// needs dense outputs (and runs these K ≤ 64 shapes on SIMT tiles).  One
// thread per row, C staged in shared memory: HBM-bound, rows·(q+p)·4 bytes.
// ---------------------------------------------------------------------------
namespace {

constexpr int kTsmmThreads = 256;

struct MutOperand {
  float *p;
  long long ld, bstride;
  int bw_shift;
};

__device__ __forceinline__ const float *elem(const Operand &o, long long r, int c) {
  return static_cast<const float *>(o.p) + (long long)(c >> o.bw_shift) * o.bstride + r * o.ld +
         (c & ((1 << o.bw_shift) - 1));
}
__device__ __forceinline__ float *elem(const MutOperand &o, long long r, int c) {
  return o.p + (long long)(c >> o.bw_shift) * o.bstride + r * o.ld + (c & ((1 << o.bw_shift) - 1));
}

// The small matrix C, read once per CTA into shared memory: from device
// memory, or carried in the kernel parameters (≤ kCParMax values — the
// eigensolver's coefficient matrices, computed on the host each iteration:
// no separate upload, no staging buffer).
constexpr int kCParMax = 1024;
struct DevC {
  const float *p;
  __device__ __forceinline__ float operator[](int i) const { return p[i]; }
};
struct ParC {
  float c[kCParMax];
  __device__ __forceinline__ float operator[](int i) const { return c[i]; }
};

// Generic path (any q, p, alignment): one row per thread.
template <typename CS>
__global__ void __launch_bounds__(kTsmmThreads) tsmm_scalar_kernel(const Operand A, const CS C, int p, float alpha,
                                                                   float beta, const MutOperand Out, long long rows) {
  __shared__ float sc[64 * 64];
  const int q = A.cols;
  for (int e = threadIdx.x; e < q * p; e += kTsmmThreads) sc[e] = C[e];
  __syncthreads();
  for (long long r = (long long)blockIdx.x * kTsmmThreads + threadIdx.x; r < rows;
       r += (long long)gridDim.x * kTsmmThreads) {
    for (int j = 0; j < p; ++j) {
      float acc = 0.f;
      for (int i = 0; i < q; ++i) acc = fmaf(*elem(A, r, i), sc[i * p + j], acc);
      float *o = elem(Out, r, j);
      *o = (beta == 0.f) ? alpha * acc : fmaf(beta, *o, alpha * acc);
    }
  }
}

// Vector path (q, p, leading dimensions, block strides multiples of 4,
// 16-byte aligned): each thread owns RB rows and a 16-column strip; A rows
// arrive as float4, C rows as broadcast LDS.128 (one shared load feeds 4·RB FMAs).
template <int RB, typename CS>
__global__ void __launch_bounds__(kTsmmThreads) tsmm_vec_kernel(const Operand A, const CS C, int p, float alpha,
                                                                float beta, const MutOperand Out, long long rows) {
  __shared__ __align__(16) float sc[64 * 64];
  const int q = A.cols;
  for (int e = threadIdx.x; e < q * p; e += kTsmmThreads) sc[e] = C[e];
  __syncthreads();
  const long long groups = (rows + RB - 1) / RB;
  for (long long g = (long long)blockIdx.x * kTsmmThreads + threadIdx.x; g < groups;
       g += (long long)gridDim.x * kTsmmThreads) {
    const long long r0 = g * RB;
    const int nr = (int)min((long long)RB, rows - r0);
    for (int j0 = 0; j0 < p; j0 += 16) {
      const int jq = min(16, p - j0) / 4;  // float4 column chunks in this strip
      float4 acc[RB][4];
#pragma unroll
      for (int b = 0; b < RB; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[b][c] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int i = 0; i < q; i += 4) {
        float av[RB][4];
#pragma unroll
        for (int b = 0; b < RB; ++b) {
          const float4 v =
              (b < nr) ? *reinterpret_cast<const float4 *>(elem(A, r0 + b, i)) : make_float4(0.f, 0.f, 0.f, 0.f);
          av[b][0] = v.x, av[b][1] = v.y, av[b][2] = v.z, av[b][3] = v.w;
        }
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            if (c < jq) {
              const float4 cv = *reinterpret_cast<const float4 *>(sc + (i + ii) * p + j0 + 4 * c);
#pragma unroll
              for (int b = 0; b < RB; ++b) {
                acc[b][c].x = fmaf(av[b][ii], cv.x, acc[b][c].x);
                acc[b][c].y = fmaf(av[b][ii], cv.y, acc[b][c].y);
                acc[b][c].z = fmaf(av[b][ii], cv.z, acc[b][c].z);
                acc[b][c].w = fmaf(av[b][ii], cv.w, acc[b][c].w);
              }
            }
          }
        }
      }
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        if (b >= nr) break;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (c < jq) {
            float4 *o = reinterpret_cast<float4 *>(elem(Out, r0 + b, j0 + 4 * c));
            float4 r = acc[b][c];
            if (beta == 0.f) {
              r.x *= alpha, r.y *= alpha, r.z *= alpha, r.w *= alpha;
            } else {
              const float4 prev = *o;
              r.x = fmaf(beta, prev.x, alpha * r.x), r.y = fmaf(beta, prev.y, alpha * r.y);
              r.z = fmaf(beta, prev.z, alpha * r.z), r.w = fmaf(beta, prev.w, alpha * r.w);
            }
            *o = r;
          }
        }
      }
    }
  }
}

// Block-major bw = 8 operands with C in the kernel parameters and (Q, P)
// compile-time (the eigensolver's shapes): one thread per row, the row's Q
// inputs as float4 pairs, every FMA takes its C value as a constant-bank
// operand — no shared-memory traffic, so L1 only carries the row stream
// (the generic vector kernel was L1-bound at 84% on LDS + half-sector loads).
// A row's inputs are all read before its outputs are written: in place is
// safe for any P.
template <int Q, int P>
__global__ void __launch_bounds__(256) tsmm_b8_kernel(const float *__restrict__ A, long long a_bstride,
                                                      float *Out, long long o_bstride, long long rows, float alpha,
                                                      float beta, const ParC C) {
  for (long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
       r += (long long)gridDim.x * blockDim.x) {
    float a[Q];
#pragma unroll
    for (int s = 0; s < Q / 8; ++s) {
      const float4 *src = reinterpret_cast<const float4 *>(A + s * a_bstride + r * 8);
      const float4 u = src[0], v = src[1];
      a[8 * s + 0] = u.x, a[8 * s + 1] = u.y, a[8 * s + 2] = u.z, a[8 * s + 3] = u.w;
      a[8 * s + 4] = v.x, a[8 * s + 5] = v.y, a[8 * s + 6] = v.z, a[8 * s + 7] = v.w;
    }
    float o[P];
#pragma unroll
    for (int j = 0; j < P; ++j) o[j] = 0.f;
#pragma unroll
    for (int i = 0; i < Q; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) o[j] = fmaf(a[i], C.c[i * P + j], o[j]);
#pragma unroll
    for (int s = 0; s < P / 8; ++s) {
      float4 *dst = reinterpret_cast<float4 *>(Out + s * o_bstride + r * 8);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float4 w = make_float4(alpha * o[8 * s + 4 * h], alpha * o[8 * s + 4 * h + 1], alpha * o[8 * s + 4 * h + 2],
                               alpha * o[8 * s + 4 * h + 3]);
        if (beta != 0.f) {
          const float4 prev = dst[h];
          w.x = fmaf(beta, prev.x, w.x), w.y = fmaf(beta, prev.y, w.y);
          w.z = fmaf(beta, prev.z, w.z), w.w = fmaf(beta, prev.w, w.w);
        }
        dst[h] = w;
      }
    }
  }
}

template <int Q, int P>
void launch_b8(const Operand &A, const ParC &C, float alpha, float beta, const MutOperand &Out, long long rows,
               int sms, cudaStream_t stream) {
  const long long blocks = std::min<long long>((rows + 255) / 256, 16LL * sms);
  tsmm_b8_kernel<Q, P><<<(unsigned)blocks, 256, 0, stream>>>(static_cast<const float *>(A.p), A.bstride, Out.p,
                                                             Out.bstride, rows, alpha, beta, C);
}

// true if (q, p) has a specialised bw = 8 kernel (and it was launched)
bool try_tsmm_b8(const Operand &A, const ParC &C, int p, float alpha, float beta, const MutOperand &Out,
                 long long rows, int out_bw, cudaStream_t stream) {
  const int q = A.cols;
  if (A.bw_shift != 3 || out_bw != 8 || A.ld != 8 || Out.ld != 8 || (A.bstride & 3) || (Out.bstride & 3) ||
      (reinterpret_cast<uintptr_t>(A.p) & 15) || (reinterpret_cast<uintptr_t>(Out.p) & 15))
    return false;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
#define CIM_B8(QQ, PP) \
  if (q == QQ && p == PP) { launch_b8<QQ, PP>(A, C, alpha, beta, Out, rows, sms, stream); return true; }
  CIM_B8(8, 8)
  CIM_B8(16, 8)
  CIM_B8(24, 8)
  CIM_B8(8, 16)
  CIM_B8(16, 16)
  CIM_B8(24, 16)
  CIM_B8(32, 16)
  CIM_B8(48, 16)
#undef CIM_B8
  return false;
}

template <typename CS>
int tsmm_impl(const Operand &A, const CS &C, int p, float alpha, float beta, const MutOperand &Out, long long rows,
              int out_bw, cudaStream_t stream) {
  const int q = A.cols;
  if (q < 1 || p < 1 || q > 64 || p > 64) return cim::set_error(CIM_EINVAL, "q and p must be in [1, 64]");
  if (rows < 0) return cim::set_error(CIM_EINVAL, "rows must be >= 0");
  if (rows == 0) return CIM_OK;
  if (!A.p || !Out.p) return cim::set_error(CIM_EINVAL, "NULL pointer");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int a_bw = 1 << A.bw_shift;
  const bool vec = (q % 4 == 0) && (p % 4 == 0) && (A.ld % 4 == 0) && (Out.ld % 4 == 0) && (A.bstride % 4 == 0) &&
                   (Out.bstride % 4 == 0) && (a_bw % 4 == 0) && (out_bw % 4 == 0) &&
                   !(reinterpret_cast<uintptr_t>(A.p) & 15) && !(reinterpret_cast<uintptr_t>(Out.p) & 15);
  if (vec) {
    constexpr int RB = 2;
    const long long groups = (rows + RB - 1) / RB;
    const long long blocks = std::min<long long>((groups + kTsmmThreads - 1) / kTsmmThreads, 8LL * sms);
    tsmm_vec_kernel<RB, CS><<<(unsigned)blocks, kTsmmThreads, 0, stream>>>(A, C, p, alpha, beta, Out, rows);
  } else {
    const long long blocks = std::min<long long>((rows + kTsmmThreads - 1) / kTsmmThreads, 8LL * sms);
    tsmm_scalar_kernel<CS><<<(unsigned)blocks, kTsmmThreads, 0, stream>>>(A, C, p, alpha, beta, Out, rows);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("tsmm kernel: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace

extern "C" int cim_tsmm(const float *A, int64_t lda, int32_t q, const float *C, int32_t p, float alpha, float beta,
                        float *Out, int64_t ldo, int64_t rows, void *stream_) {
  cim::clear_error();
  if (lda < q || ldo < p) return cim::set_error(CIM_EINVAL, "bad leading dimensions");
  if (!C) return cim::set_error(CIM_EINVAL, "NULL pointer");
  const Operand a{A, lda, 0, 6, q};
  const MutOperand o{Out, ldo, 0, 6};
  return tsmm_impl(a, DevC{C}, p, alpha, beta, o, rows, 64, reinterpret_cast<cudaStream_t>(stream_));
}

extern "C" int cim_tsmm_blocked(const float *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t q,
                                const float *C, int32_t p, float alpha, float beta, float *Out, int64_t ldo,
                                int32_t o_bw, int64_t o_bstride, int64_t rows, void *stream_) {
  cim::clear_error();
  const int sa = bw_shift_of(a_bw), so = bw_shift_of(o_bw);
  if (sa < 0 || so < 0) return cim::set_error(CIM_EINVAL, "block widths must be 4, 8, 16, 32 or 64");
  if (lda < std::min(a_bw, q) || ldo < std::min(o_bw, p))
    return cim::set_error(CIM_EINVAL, "leading dimensions must cover a block");
  if (!C) return cim::set_error(CIM_EINVAL, "NULL pointer");
  const Operand a{A, lda, a_bstride, sa, q};
  const MutOperand o{Out, ldo, o_bstride, so};
  return tsmm_impl(a, DevC{C}, p, alpha, beta, o, rows, o_bw, reinterpret_cast<cudaStream_t>(stream_));
}

extern "C" int cim_tsmm_blocked_hc(const float *A, int64_t lda, int32_t a_bw, int64_t a_bstride, int32_t q,
                                   const float *C_host, int32_t p, float alpha, float beta, float *Out, int64_t ldo,
                                   int32_t o_bw, int64_t o_bstride, int64_t rows, void *stream_) {
  cim::clear_error();
  const int sa = bw_shift_of(a_bw), so = bw_shift_of(o_bw);
  if (sa < 0 || so < 0) return cim::set_error(CIM_EINVAL, "block widths must be 4, 8, 16, 32 or 64");
  if (lda < std::min(a_bw, q) || ldo < std::min(o_bw, p))
    return cim::set_error(CIM_EINVAL, "leading dimensions must cover a block");
  if (!C_host) return cim::set_error(CIM_EINVAL, "NULL pointer");
  if (q < 1 || p < 1 || (long long)q * p > kCParMax)
    return cim::set_error(CIM_EUNSUPPORTED, "host C holds at most 1024 values (q*p)");
  ParC c;
  std::memcpy(c.c, C_host, sizeof(float) * (size_t)q * p);
  const Operand a{A, lda, a_bstride, sa, q};
  const MutOperand o{Out, ldo, o_bstride, so};
  if (rows > 0 && try_tsmm_b8(a, c, p, alpha, beta, o, rows, o_bw, reinterpret_cast<cudaStream_t>(stream_))) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("tsmm_b8: ") + cudaGetErrorString(e));
    return CIM_OK;
  }
  return tsmm_impl(a, c, p, alpha, beta, o, rows, o_bw, reinterpret_cast<cudaStream_t>(stream_));
}

namespace {
// ---------------------------------------------------------------------------
// Block residual W = AX − X·diag(λ) over whole slots (rows × bw, row-major;
// λ_j = 0 for j ≥ m keeps padding columns zero).  λ rides in the kernel
// parameters.  Elementwise, HBM-bound: 3·rows·bw·4 bytes.
// ---------------------------------------------------------------------------
struct LamPar {
  float l[64];
};

__global__ void __launch_bounds__(256) block_residual_kernel(const float4 *__restrict__ X,
                                                             const float4 *__restrict__ AX, float4 *__restrict__ W,
                                                             long long n4, int bw4, const LamPar lam) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (long long)gridDim.x * blockDim.x) {
    const int j = 4 * (int)(e % bw4);
    const float4 x = X[e], ax = AX[e];
    W[e] = make_float4(fmaf(-lam.l[j], x.x, ax.x), fmaf(-lam.l[j + 1], x.y, ax.y), fmaf(-lam.l[j + 2], x.z, ax.z),
                       fmaf(-lam.l[j + 3], x.w, ax.w));
  }
}
}  // namespace

extern "C" int cim_block_residual(const float *X, const float *AX, const double *lam_host, int32_t m, float *W,
                                  int64_t rows, int32_t bw, void *stream_) {
  cim::clear_error();
  if (bw < 4 || bw > 64 || (bw & 3) || m < 0 || m > bw) return cim::set_error(CIM_EINVAL, "need 4 <= bw <= 64, bw % 4 == 0, m <= bw");
  if (rows < 0) return cim::set_error(CIM_EINVAL, "rows must be >= 0");
  if (rows == 0) return CIM_OK;
  if (!X || !AX || !W || (m > 0 && !lam_host)) return cim::set_error(CIM_EINVAL, "NULL pointer");
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(AX) | reinterpret_cast<uintptr_t>(W)) & 15)
    return cim::set_error(CIM_EINVAL, "X, AX and W must be 16-byte aligned");
  LamPar lam{};
  for (int j = 0; j < m; ++j) lam.l[j] = (float)lam_host[j];
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long n4 = rows * bw / 4;
  const long long blocks = std::min<long long>((n4 + 255) / 256, 16LL * sms);
  block_residual_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream_)>>>(
      reinterpret_cast<const float4 *>(X), reinterpret_cast<const float4 *>(AX), reinterpret_cast<float4 *>(W), n4,
      bw / 4, lam);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("block_residual: ") + cudaGetErrorString(e));
  return CIM_OK;
}

namespace {
// ---------------------------------------------------------------------------
// LOBPCG Ritz update fused with the next residual (bw = 8 block-major f32
// slots): per row, [P' X'] = S·C and [AP' AX'] = AS·C (C = [C_p | C], q × 16)
// and W' = AX' − X'·diag(λ), written into five consecutive slots
// [P' X' W' AP' AX'] of the other work buffer.  One pass reads the 2·q/8
// input slots and writes five, where two tsmm passes and the residual pass
// read and wrote 2·q/8 + 7.  C and λ ride in the kernel parameters.
// ---------------------------------------------------------------------------
struct RitzPar {
  float c[48 * 16];
  float lam[8];
};

template <int Q>
__device__ __forceinline__ void ritz_load(const float *__restrict__ A, long long bstride, long long r, float (&a)[Q]) {
#pragma unroll
  for (int s = 0; s < Q / 8; ++s) {
    const float4 *src = reinterpret_cast<const float4 *>(A + s * bstride + r * 8);
    const float4 u = __ldcs(src), v = __ldcs(src + 1);  // streamed once
    a[8 * s + 0] = u.x, a[8 * s + 1] = u.y, a[8 * s + 2] = u.z, a[8 * s + 3] = u.w;
    a[8 * s + 4] = v.x, a[8 * s + 5] = v.y, a[8 * s + 6] = v.z, a[8 * s + 7] = v.w;
  }
}

template <int Q>
__device__ __forceinline__ void ritz_mul(const float (&a)[Q], const float *c, float (&o)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j] = 0.f;
#pragma unroll
  for (int i = 0; i < Q; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) o[j] = fmaf(a[i], c[i * 16 + j], o[j]);
}

__device__ __forceinline__ void st8(float *dst, const float *v) {
  float4 *d = reinterpret_cast<float4 *>(dst);
  d[0] = make_float4(v[0], v[1], v[2], v[3]);
  d[1] = make_float4(v[4], v[5], v[6], v[7]);
}

// Lane pairs share a row: the even lane multiplies the S row ([P' X']),
// the odd lane the AS row ([AP' AX']) and forms W' with X' from its partner
// (one shuffle) — half the registers of one thread per row (whose loads
// ptxas interleaved with the first product's FMAs), twice the resident
// warps.
template <int Q>
__global__ void __launch_bounds__(256) ritz_update_b8_kernel(const float *__restrict__ S, const float *__restrict__ AS,
                                                             long long bstride, float *__restrict__ Out,
                                                             long long o_bstride, long long rows, const RitzPar par) {
  const int h = threadIdx.x & 1;
  const long long step = ((long long)gridDim.x * blockDim.x) >> 1;
  for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 1; r < rows; r += step) {
    float a[Q], o[16], x[8];
    ritz_load<Q>(h ? AS : S, bstride, r, a);
    ritz_mul<Q>(a, par.c, o);
    const unsigned mask = __activemask();  // both lanes of a pair are in or out together
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __shfl_xor_sync(mask, o[8 + j], 1);  // odd lane: X' of the row
    float *dst = Out + (h ? 3 : 0) * o_bstride + r * 8;
    st8(dst, o);                  // P' | AP'
    st8(dst + o_bstride, o + 8);  // X' | AX'
    if (h) {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fmaf(-par.lam[j], x[j], o[8 + j]);
      st8(Out + 2 * o_bstride + r * 8, x);  // W' = AX' − X'Λ
    }
  }
}
}  // namespace

extern "C" int cim_ritz_update_b8(const float *S, const float *AS, int64_t bstride, int32_t q, const float *C_host,
                                  const double *lam_host, int32_t m, float *Out, int64_t o_bstride, int64_t rows,
                                  void *stream_) {
  cim::clear_error();
  if (q != 8 && q != 16 && q != 24 && q != 32 && q != 48) return cim::set_error(CIM_EINVAL, "q must be 8, 16, 24, 32 or 48");
  if (m < 0 || m > 8) return cim::set_error(CIM_EINVAL, "m must be in [0, 8]");
  if (rows < 0) return cim::set_error(CIM_EINVAL, "rows must be >= 0");
  if (rows == 0) return CIM_OK;
  if (!S || !AS || !Out || !C_host || (m > 0 && !lam_host)) return cim::set_error(CIM_EINVAL, "NULL pointer");
  if ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(AS) | reinterpret_cast<uintptr_t>(Out)) & 15 ||
      (bstride & 3) || (o_bstride & 3))
    return cim::set_error(CIM_EINVAL, "slots must be 16-byte aligned");
  RitzPar par{};
  std::memcpy(par.c, C_host, sizeof(float) * (size_t)q * 16);
  for (int j = 0; j < m; ++j) par.lam[j] = (float)lam_host[j];
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned blocks = (unsigned)std::min<long long>((rows + 255) / 256, 16LL * sms);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream_);
  switch (q) {
    case 8: ritz_update_b8_kernel<8><<<blocks, 256, 0, st>>>(S, AS, bstride, Out, o_bstride, rows, par); break;
    case 16: ritz_update_b8_kernel<16><<<blocks, 256, 0, st>>>(S, AS, bstride, Out, o_bstride, rows, par); break;
    case 24: ritz_update_b8_kernel<24><<<blocks, 256, 0, st>>>(S, AS, bstride, Out, o_bstride, rows, par); break;
    case 32: ritz_update_b8_kernel<32><<<blocks, 256, 0, st>>>(S, AS, bstride, Out, o_bstride, rows, par); break;
    default: ritz_update_b8_kernel<48><<<blocks, 256, 0, st>>>(S, AS, bstride, Out, o_bstride, rows, par); break;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("ritz_update_b8: ") + cudaGetErrorString(e));
  return CIM_OK;
}
