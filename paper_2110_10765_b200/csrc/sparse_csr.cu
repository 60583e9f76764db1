// Row-CSR path for the SMALL sparse tiles (a few dozen entries per 64-tile:
// the basis-built skeletons of the reference, pipeline.py:290-377, whose
// orbital-pair tiles hold ~16 entries each).
//
// sparse_small_kernel walks such tiles entry-parallel and issues, per entry,
// two X gathers and two vector reductions (Y_R[row] and Y_C[col]) — the
// reference's _contract_atomic discipline (pipeline.py:479-488).  Here the
// small tiles of each block row are re-laid (once, on the device) as one
// row-CSR of the upper block triangle: row i lists every (j, v) of its small
// tiles, j global.  The apply then walks rows:
//
//   Y[i] += Σ_j v·X[j]         (direct: gathered X[j], summed in registers
//                               across the row's lanes, ONE reduction per row)
//   Y[j] += v·X[i]   (j ∉ block(i): transposed; X[i] read once per row)
//
// — half the reductions and half the gathers of the entry-parallel kernel,
// and every lane of a row group has independent entries in flight.  Rows
// of the diagonal block store both triangles (a diagonal tile is stored in
// full), so their entries feed the direct product only.
//
// Build (cim_sparse_csr_count → cim_exclusive_scan_i64 → cim_sparse_csr_fill):
// per-row counts by atomics over (tile, row) segments, the device scan, then
// one thread per (block row, local row) walks its panel's small tiles in
// order and copies the row segments — a deterministic entry order.
#include <algorithm>
#include <cstdint>
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

#ifndef CIM_CSR_SYM_ILP
#define CIM_CSR_SYM_ILP 4  // entries gathered per lane per step in the symmetric row walk (2 or 4)
#endif
#ifndef CIM_CSR_SYM_MINB
#define CIM_CSR_SYM_MINB 4  // resident 256-thread blocks per SM (64 registers: 4 gathers of 32 B in flight, no spills)
#endif
#ifndef CIM_CSR_SYM_SUB
#define CIM_CSR_SYM_SUB 8  // most lanes sharing one entry's X row in the symmetric walk (1 = one lane per entry)
#endif

namespace cim {
namespace {

__global__ void csr_count_kernel(const int32_t *small, long long n_small, const int2 *tile_rc,
                                 const uint16_t *rowptr, unsigned long long *row_cnt) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_small * 64) return;
  const long long t = small[g >> 6];
  const int r = (int)(g & 63);
  const uint16_t *rp = rowptr + (size_t)t * kSpPtrStride;
  const int c = rp[r + 1] - rp[r];
  if (c > 0) atomicAdd(row_cnt + (long long)tile_rc[t].x * 64 + r, (unsigned long long)c);
}

template <typename T>
__global__ void csr_fill_kernel(const int32_t *small, const int2 *tile_rc, const long long *entry_off,
                                const uint16_t *rowptr, const uint8_t *col, const T *vals, const int32_t *panel_R,
                                const long long *panel_ptr, long long n_panels, const long long *csr_ptr,
                                int32_t *csr_col, T *csr_val) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_panels * 64) return;
  const long long pnl = g >> 6;
  const int r = (int)(g & 63);
  const long long i = (long long)panel_R[pnl] * 64 + r;
  long long cur = csr_ptr[i];
  for (long long q = panel_ptr[pnl]; q < panel_ptr[pnl + 1]; ++q) {
    const long long t = small[q];
    const uint16_t *rp = rowptr + (size_t)t * kSpPtrStride;
    const long long base = entry_off[t];
    const int C64 = tile_rc[t].y * 64;
    for (int e = rp[r]; e < rp[r + 1]; ++e) {
      csr_col[cur] = C64 + col[base + e];
      csr_val[cur] = vals[base + e];
      ++cur;
    }
  }
}

template <typename T, int KV>
__device__ __forceinline__ void ld_vec(T (&d)[KV], const T *p) {
  if constexpr (sizeof(T) * KV == 32) {
    // one 256-bit load per row slice (LDG.E.ENL2.256, sm_100): half the L1
    // requests of two 128-bit loads for the random X gathers
    uint32_t u[8];
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                 : "l"(p));
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int q = 0; q < 8; ++q) d[q] = __uint_as_float(u[q]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) d[q] = __hiloint2double((int)u[2 * q + 1], (int)u[2 * q]);
    }
  } else if constexpr (sizeof(T) == 4 && KV % 4 == 0) {
#pragma unroll
    for (int q = 0; q < KV / 4; ++q) {
      const float4 v = __ldg(reinterpret_cast<const float4 *>(p) + q);
      d[4 * q] = v.x, d[4 * q + 1] = v.y, d[4 * q + 2] = v.z, d[4 * q + 3] = v.w;
    }
  } else if constexpr (sizeof(T) == 8 && KV % 2 == 0) {
#pragma unroll
    for (int q = 0; q < KV / 2; ++q) {
      const double2 v = __ldg(reinterpret_cast<const double2 *>(p) + q);
      d[2 * q] = v.x, d[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < KV; ++q) d[q] = __ldg(p + q);
  }
}

template <typename T, int KV>
__device__ __forceinline__ void red_vec(T *p, const T (&s)[KV]) {
  if constexpr (sizeof(T) == 4 && KV % 4 == 0) {
#pragma unroll
    for (int q = 0; q < KV / 4; ++q)
      red_add_v4(reinterpret_cast<float *>(p) + 4 * q, s[4 * q], s[4 * q + 1], s[4 * q + 2], s[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < KV; ++q) red_add(p + q, s[q]);
  }
}

// LPR lanes per row (a warp holds 32 / LPR rows), KV vectors per pass.
// The rows hold one triangle: the transposed product is scattered.
template <typename T, int KV, int LPR>
__global__ void __launch_bounds__(256) csr_spmm_kernel(const long long *__restrict__ ptr,
                                                       const int32_t *__restrict__ col, const T *__restrict__ val,
                                                       long long rows, const T *__restrict__ X, T *__restrict__ Y,
                                                       int k, long long ldy) {
  const int lane = threadIdx.x & 31, sl = lane % LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (lane - sl));
  const long long groups = ((long long)gridDim.x * blockDim.x) / LPR;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPR; i < rows; i += groups) {
    const long long p0 = ptr[i], p1 = ptr[i + 1];
    if (p0 == p1) continue;  // uniform within the row group
    const long long bi = i >> 6;
    for (int v0 = 0; v0 < k; v0 += KV) {
      T xi[KV], acc[KV];
      ld_vec<T, KV>(xi, X + i * k + v0);
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = T(0);
      long long e = p0 + sl;
      for (; e + LPR < p1; e += 2 * LPR) {  // two independent entries in flight per lane
        const int j0 = __ldg(col + e), j1 = __ldg(col + e + LPR);
        const T w0 = __ldg(val + e), w1 = __ldg(val + e + LPR);
        T x0[KV], x1[KV], t[KV];
        ld_vec<T, KV>(x0, X + (long long)j0 * k + v0);
        ld_vec<T, KV>(x1, X + (long long)j1 * k + v0);
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = fma(w0, x0[q], fma(w1, x1[q], acc[q]));
        if ((j0 >> 6) != bi) {
#pragma unroll
          for (int q = 0; q < KV; ++q) t[q] = w0 * xi[q];
          red_vec<T, KV>(Y + (long long)j0 * ldy + v0, t);
        }
        if ((j1 >> 6) != bi) {
#pragma unroll
          for (int q = 0; q < KV; ++q) t[q] = w1 * xi[q];
          red_vec<T, KV>(Y + (long long)j1 * ldy + v0, t);
        }
      }
      if (e < p1) {
        const int j = __ldg(col + e);
        const T w = __ldg(val + e);
        T x[KV], t[KV];
        ld_vec<T, KV>(x, X + (long long)j * k + v0);
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = fma(w, x[q], acc[q]);
        if ((j >> 6) != bi) {
#pragma unroll
          for (int q = 0; q < KV; ++q) t[q] = w * xi[q];
          red_vec<T, KV>(Y + (long long)j * ldy + v0, t);
        }
      }
#pragma unroll
      for (int off = LPR / 2; off > 0; off >>= 1)
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] += __shfl_xor_sync(gmask, acc[q], off);
      if (sl == 0) red_vec<T, KV>(Y + i * ldy + v0, acc);
    }
  }
}

// The rows hold both triangles (csr_symmetric): gathers only, one reduction
// per row.  The walk is bound by the L1's gather wavefronts (one per X row
// slice, every entry a different line): SUB lanes share one entry, each
// gathering KV vectors of the same X row, so an entry whose row is 64 or 128
// bytes (f32 k = 16 / 32) costs one line request instead of two or four;
// LPR / SUB entries per row group per step, U of them in flight per lane.
template <typename T, int KV, int LPR, int SUB>
__global__ void __launch_bounds__(256, CIM_CSR_SYM_MINB) csr_sym_kernel(const long long *__restrict__ ptr,
                                                      const int32_t *__restrict__ col, const T *__restrict__ val,
                                                      long long rows, const T *__restrict__ X, T *__restrict__ Y,
                                                      int k, long long ldy) {
  constexpr int U = CIM_CSR_SYM_ILP, ES = LPR / SUB;
  const int lane = threadIdx.x & 31, sl = lane % LPR, es = sl / SUB, part = sl % SUB;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (lane - sl));
  const long long groups = ((long long)gridDim.x * blockDim.x) / LPR;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / LPR; i < rows; i += groups) {
    const long long p0 = ptr[i], p1 = ptr[i + 1];
    if (p0 == p1) continue;  // uniform within the row group
    for (int v0 = part * KV; v0 < k; v0 += SUB * KV) {
      T acc[KV];
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = T(0);
      long long e = p0 + es;
      for (; e + (U - 1) * ES < p1; e += U * ES) {
        int j[U];
        T w[U], x[U][KV];
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = __ldg(col + e + u * ES), w[u] = __ldg(val + e + u * ES);
#pragma unroll
        for (int u = 0; u < U; ++u) ld_vec<T, KV>(x[u], X + (long long)j[u] * k + v0);
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < KV; ++q) acc[q] = fma(w[u], x[u][q], acc[q]);
      }
      if (U > 2 && e + ES < p1) {
        const int j0 = __ldg(col + e), j1 = __ldg(col + e + ES);
        const T w0 = __ldg(val + e), w1 = __ldg(val + e + ES);
        T x0[KV], x1[KV];
        ld_vec<T, KV>(x0, X + (long long)j0 * k + v0);
        ld_vec<T, KV>(x1, X + (long long)j1 * k + v0);
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = fma(w0, x0[q], fma(w1, x1[q], acc[q]));
        e += 2 * ES;
      }
      for (; e < p1; e += ES) {
        const int j = __ldg(col + e);
        const T w = __ldg(val + e);
        T x[KV];
        ld_vec<T, KV>(x, X + (long long)j * k + v0);
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = fma(w, x[q], acc[q]);
      }
#pragma unroll
      for (int off = LPR / 2; off >= SUB; off >>= 1)
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] += __shfl_xor_sync(gmask, acc[q], off);
      if (es == 0) red_vec<T, KV>(Y + i * ldy + v0, acc);
    }
  }
}

template <typename T, int KV, int LPR>
void launch_csr_sym(const long long *ptr, const int32_t *col, const T *v, long long rows, const T *x, T *y, int k,
                    long long ldy, unsigned grid, cudaStream_t stream) {
  int sub = 1;
  if constexpr (sizeof(T) * KV == 32)  // full 32-byte slices: lanes share an entry's X row
    while (sub < CIM_CSR_SYM_SUB && sub < LPR && k % (2 * sub * KV) == 0) sub *= 2;
  switch (sub) {
    case 8: csr_sym_kernel<T, KV, LPR, 8><<<grid, 256, 0, stream>>>(ptr, col, v, rows, x, y, k, ldy); break;
    case 4: csr_sym_kernel<T, KV, LPR, 4><<<grid, 256, 0, stream>>>(ptr, col, v, rows, x, y, k, ldy); break;
    case 2: csr_sym_kernel<T, KV, LPR, 2><<<grid, 256, 0, stream>>>(ptr, col, v, rows, x, y, k, ldy); break;
    default: csr_sym_kernel<T, KV, LPR, 1><<<grid, 256, 0, stream>>>(ptr, col, v, rows, x, y, k, ldy); break;
  }
}

template <typename T, int KV>
int launch_csr_kv(const cim_sparse_tiles *S, const void *X, void *Y, int k, long long ldy, int sms,
                  cudaStream_t stream) {
  const long long rows = S->csr_rows;
  const double avg = (double)S->csr_nnz / (double)(rows > 0 ? rows : 1);
  const T *x = static_cast<const T *>(X);
  T *y = static_cast<T *>(Y);
  const T *v = static_cast<const T *>(S->csr_val);
  const long long per_block = avg >= 24.0 ? 8 : 32;  // rows per 256-thread block (LPR 32 or 8)
  const unsigned grid = (unsigned)std::min<long long>((rows + per_block - 1) / per_block, (long long)sms * 16);
  const long long *ptr = reinterpret_cast<const long long *>(S->csr_ptr);
  if (S->csr_symmetric) {
    if (avg >= 24.0) launch_csr_sym<T, KV, 32>(ptr, S->csr_col, v, rows, x, y, k, ldy, grid, stream);
    else launch_csr_sym<T, KV, 8>(ptr, S->csr_col, v, rows, x, y, k, ldy, grid, stream);
  } else {
    if (avg >= 24.0) csr_spmm_kernel<T, KV, 32><<<grid, 256, 0, stream>>>(ptr, S->csr_col, v, rows, x, y, k, ldy);
    else csr_spmm_kernel<T, KV, 8><<<grid, 256, 0, stream>>>(ptr, S->csr_col, v, rows, x, y, k, ldy);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CIM_OK : set_error(CIM_ECUDA, std::string("csr_spmm launch: ") + cudaGetErrorString(e));
}

}  // namespace

// The small tiles' contribution through the row-CSR (called by sym_spmm_sparse).
int sym_spmm_sparse_csr(const cim_sparse_tiles *S, int dtype, const void *X, void *Y, int k, long long ldy, int sms,
                        cudaStream_t stream) {
  if (!S->csr_ptr || S->csr_rows <= 0 || S->csr_nnz <= 0) return CIM_OK;
  if (!S->csr_col || !S->csr_val) return set_error(CIM_EINVAL, "csr arrays are NULL");
  if (dtype == CIM_F32) {
    if (k % 8 == 0) return launch_csr_kv<float, 8>(S, X, Y, k, ldy, sms, stream);
    if (k % 4 == 0) return launch_csr_kv<float, 4>(S, X, Y, k, ldy, sms, stream);
    if (k % 2 == 0) return launch_csr_kv<float, 2>(S, X, Y, k, ldy, sms, stream);
    return launch_csr_kv<float, 1>(S, X, Y, k, ldy, sms, stream);
  }
  if (k % 4 == 0) return launch_csr_kv<double, 4>(S, X, Y, k, ldy, sms, stream);
  if (k % 2 == 0) return launch_csr_kv<double, 2>(S, X, Y, k, ldy, sms, stream);
  return launch_csr_kv<double, 1>(S, X, Y, k, ldy, sms, stream);
}

}  // namespace cim

extern "C" int cim_sparse_csr_count(const cim_sparse_tiles *S, int64_t n_pad, int64_t *row_cnt, void *stream) {
  cim::clear_error();
  if (!S || !row_cnt || n_pad < 0) return cim::set_error(CIM_EINVAL, "bad arguments");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(row_cnt, 0, sizeof(int64_t) * (size_t)n_pad, s);
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("csr_count memset: ") + cudaGetErrorString(e));
  if (S->n_small <= 0) return CIM_OK;
  if (!S->small_tiles || !S->tile_rc || !S->rowptr) return cim::set_error(CIM_EINVAL, "NULL sparse arrays");
  const long long threads = S->n_small * 64;
  cim::csr_count_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
      S->small_tiles, S->n_small, reinterpret_cast<const int2 *>(S->tile_rc), S->rowptr,
      reinterpret_cast<unsigned long long *>(row_cnt));
  e = cudaGetLastError();
  return e == cudaSuccess ? CIM_OK : cim::set_error(CIM_ECUDA, std::string("csr_count: ") + cudaGetErrorString(e));
}

extern "C" int cim_sparse_csr_fill(const cim_sparse_tiles *S, int32_t dtype, const int32_t *panel_R,
                                   const int64_t *panel_ptr, int64_t n_panels, const int64_t *csr_ptr,
                                   int32_t *csr_col, void *csr_val, void *stream) {
  cim::clear_error();
  if (!S || n_panels < 0) return cim::set_error(CIM_EINVAL, "bad arguments");
  if (dtype != CIM_F32 && dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (n_panels == 0) return CIM_OK;
  if (!panel_R || !panel_ptr || !csr_ptr || !csr_col || !csr_val || !S->small_tiles || !S->col || !S->vals)
    return cim::set_error(CIM_EINVAL, "NULL arrays");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const long long threads = n_panels * 64;
  const unsigned grid = (unsigned)((threads + 127) / 128);
  const int2 *rc = reinterpret_cast<const int2 *>(S->tile_rc);
  const long long *off = reinterpret_cast<const long long *>(S->entry_off);
  const long long *pp = reinterpret_cast<const long long *>(panel_ptr);
  const long long *cp = reinterpret_cast<const long long *>(csr_ptr);
  if (dtype == CIM_F32)
    cim::csr_fill_kernel<float><<<grid, 128, 0, s>>>(S->small_tiles, rc, off, S->rowptr, S->col,
                                                     static_cast<const float *>(S->vals), panel_R, pp, n_panels, cp,
                                                     csr_col, static_cast<float *>(csr_val));
  else
    cim::csr_fill_kernel<double><<<grid, 128, 0, s>>>(S->small_tiles, rc, off, S->rowptr, S->col,
                                                      static_cast<const double *>(S->vals), panel_R, pp, n_panels,
                                                      cp, csr_col, static_cast<double *>(csr_val));
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CIM_OK : cim::set_error(CIM_ECUDA, std::string("csr_fill: ") + cudaGetErrorString(e));
}
