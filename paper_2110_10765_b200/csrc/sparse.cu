// Sparse ("COO-in-tile") stored tiles: the same operator, Y += U_s·X + U_s,offᵀ·X,
// for 64-tiles below the dense break-even fill (include/cim_b200.h,
// cim_sparse_tiles).  Reference skeletons are built from ragged orbital
// blocks (pipeline.py:290-377; sizes 1..100), so their 64-tiles are mostly
// sparse: streaming them as dense tiles would move 4096 values per tile for
// a few hundred entries.
//
// One warp per tile (persistent warps, global ticket counter):
//   * lane ℓ owns local rows ℓ and ℓ+32 — the direct product of a row is a
//     register accumulation over its (row-sorted) entries, flushed with one
//     vector red.global per row;
//   * the transposed product scatters v·x_r into a per-warp shared-memory
//     Y_C tile (red.shared, padded stride against bank conflicts), flushed
//     once per tile;
//   * X_C / X_R rows are read through L1 (a tile's entries hit a 64-row X
//     block repeatedly).
// k is processed in passes of KV vectors (8 f32 / 4 f64).
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

constexpr int kSpWarps = 8;  // warps per CTA

template <typename T, int KV>
__device__ __forceinline__ void ldg_vec(T (&d)[KV], const T *p) {
  if constexpr (sizeof(T) == 4 && KV % 4 == 0) {
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
    for (int q = 0; q < KV / 4; ++q) red_add_v4(reinterpret_cast<float *>(p) + 4 * q, s[4 * q], s[4 * q + 1], s[4 * q + 2], s[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < KV; ++q) red_add(p + q, s[q]);
  }
}

struct SparseParams {
  const int2 *tile_rc;
  const long long *entry_off;
  const uint16_t *rowptr;
  const uint8_t *col;
  const void *vals;
  const void *X;
  void *Y;
  unsigned int *counter;
  long long n_tiles;
  long long ldx, ldy;
  int k;
};

template <typename T, int KV>
__global__ void __launch_bounds__(kSpWarps * 32) sparse_spmm_kernel(const SparseParams p) {
  __shared__ T ycs_all[kSpWarps][64 * (KV + 1)];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T *ycs = ycs_all[w];
  const T *X = static_cast<const T *>(p.X);
  T *Y = static_cast<T *>(p.Y);
  const T *vals = static_cast<const T *>(p.vals);
  while (true) {
    unsigned int t = 0;
    if (lane == 0) t = atomicAdd(p.counter, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((long long)t >= p.n_tiles) break;
    const int2 rc = p.tile_rc[t];
    const bool diag = rc.x == rc.y;
    const long long base = p.entry_off[t];
    const uint16_t *rp = p.rowptr + (size_t)t * 65;
    const int e_lo[2] = {rp[lane], rp[lane + 32]}, e_hi[2] = {rp[lane + 1], rp[lane + 33]};
    const T *xr_blk = X + (long long)rc.x * 64 * p.ldx;
    const T *xc_blk = X + (long long)rc.y * 64 * p.ldx;
    for (int v0 = 0; v0 < p.k; v0 += KV) {
      if (!diag) {
        for (int e = lane; e < 64 * (KV + 1); e += 32) ycs[e] = T(0);
        __syncwarp();
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = lane + 32 * h;
        if (e_hi[h] == e_lo[h]) continue;
        T xr[KV], acc[KV];
        if (!diag) ldg_vec<T, KV>(xr, xr_blk + (long long)r * p.ldx + v0);
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = T(0);
        for (int e = e_lo[h]; e < e_hi[h]; ++e) {
          const int c = __ldg(p.col + base + e);
          const T v = __ldg(vals + base + e);
          T xc[KV];
          ldg_vec<T, KV>(xc, xc_blk + (long long)c * p.ldx + v0);
#pragma unroll
          for (int q = 0; q < KV; ++q) acc[q] = fma(v, xc[q], acc[q]);
          if (!diag) {
#pragma unroll
            for (int q = 0; q < KV; ++q) atomicAdd(&ycs[c * (KV + 1) + q], v * xr[q]);
          }
        }
        red_vec<T, KV>(Y + ((long long)rc.x * 64 + r) * p.ldy + v0, acc);
      }
      if (!diag) {
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = lane + 32 * h;
          T s[KV];
#pragma unroll
          for (int q = 0; q < KV; ++q) s[q] = ycs[c * (KV + 1) + q];
          red_vec<T, KV>(Y + ((long long)rc.y * 64 + c) * p.ldy + v0, s);
        }
        __syncwarp();
      }
    }
  }
}

template <typename T>
__global__ void fill_sparse_values_kernel(const int2 *tile_rc, const long long *entry_off, const uint16_t *rowptr,
                                          const uint8_t *col, long long n_tiles, long long n, int kind,
                                          uint64_t seed, int op_k, const T *mask, T *out) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long t = warp; t < n_tiles; t += nwarps) {
    const int2 rc = tile_rc[t];
    const long long base = entry_off[t];
    const uint16_t *rp = rowptr + (size_t)t * 65;
    for (int r = lane; r < 64; r += 32) {
      const uint64_t i = (uint64_t)rc.x * 64 + r;
      for (int e = rp[r]; e < rp[r + 1]; ++e) {
        const uint64_t j = (uint64_t)rc.y * 64 + col[base + e];
        const bool on = (mask == nullptr || mask[base + e] != T(0)) && i < (uint64_t)n && j < (uint64_t)n;
        out[base + e] = on ? (T)value_of_kind(kind, i, j, seed, op_k) : T(0);
      }
    }
  }
}

struct SpState {
  int sms = 0;
  unsigned int *counters = nullptr;
  int pos = 0;
};
std::mutex g_sp_mu;
std::vector<SpState> g_sp;
constexpr int kSpRing = 1024;

int sp_state(SpState **out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(CIM_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_sp_mu);
  if ((int)g_sp.size() <= dev) g_sp.resize(dev + 1);
  SpState &s = g_sp[dev];
  if (s.sms == 0) {
    cudaError_t e = cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaMalloc(&s.counters, kSpRing * sizeof(unsigned int));
    if (e != cudaSuccess) {
      s.sms = 0;
      return set_error(CIM_ECUDA, std::string("sparse state: ") + cudaGetErrorString(e));
    }
  }
  *out = &s;
  return CIM_OK;
}

template <typename T, int KV>
int launch_sparse(const cim_sparse_tiles *S, const void *X, void *Y, int k, long long ldx, long long ldy,
                  cudaStream_t stream) {
  SpState *st = nullptr;
  int rc = sp_state(&st);
  if (rc) return rc;
  unsigned int *ctr;
  {
    std::lock_guard<std::mutex> lk(g_sp_mu);
    if (st->pos >= kSpRing) st->pos = 0;
    ctr = st->counters + st->pos++;
  }
  cudaError_t e = cudaMemsetAsync(ctr, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse counter: ") + cudaGetErrorString(e));
  SparseParams p;
  p.tile_rc = reinterpret_cast<const int2 *>(S->tile_rc);
  p.entry_off = reinterpret_cast<const long long *>(S->entry_off);
  p.rowptr = S->rowptr;
  p.col = S->col;
  p.vals = S->vals;
  p.X = X;
  p.Y = Y;
  p.counter = ctr;
  p.n_tiles = S->n_tiles;
  p.ldx = ldx;
  p.ldy = ldy;
  p.k = k;
  const long long warps = std::min<long long>(S->n_tiles, (long long)st->sms * 4 * kSpWarps);
  const unsigned grid = (unsigned)((warps + kSpWarps - 1) / kSpWarps);
  sparse_spmm_kernel<T, KV><<<grid, kSpWarps * 32, 0, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse_spmm launch: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace

// Called by cim_sym_spmm after the dense tiles (Y already zeroed or accumulating).
int sym_spmm_sparse(const cim_sparse_tiles *S, int dtype, const void *X, void *Y, int k, long long ldx,
                    long long ldy, cudaStream_t stream) {
  if (!S || S->n_tiles == 0) return CIM_OK;
  if (!S->tile_rc || !S->entry_off || !S->rowptr || (S->n_entries > 0 && (!S->col || !S->vals)))
    return set_error(CIM_EINVAL, "sparse tile arrays are NULL");
  if (dtype == CIM_F32) {
    if (k % 8 == 0) return launch_sparse<float, 8>(S, X, Y, k, ldx, ldy, stream);
    if (k % 4 == 0) return launch_sparse<float, 4>(S, X, Y, k, ldx, ldy, stream);
    if (k % 2 == 0) return launch_sparse<float, 2>(S, X, Y, k, ldx, ldy, stream);
    return launch_sparse<float, 1>(S, X, Y, k, ldx, ldy, stream);
  }
  if (k % 4 == 0) return launch_sparse<double, 4>(S, X, Y, k, ldx, ldy, stream);
  if (k % 2 == 0) return launch_sparse<double, 2>(S, X, Y, k, ldx, ldy, stream);
  return launch_sparse<double, 1>(S, X, Y, k, ldx, ldy, stream);
}

}  // namespace cim

extern "C" int cim_fill_sparse_values(const cim_sparse_tiles *S, int64_t n, int32_t dtype, int32_t kind,
                                      uint64_t seed, int32_t op_k, const void *mask, void *vals_out, void *stream_) {
  cim::clear_error();
  if (!S) return cim::set_error(CIM_EINVAL, "S is NULL");
  if (dtype != CIM_F32 && dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (kind < 0 || kind > 2) return cim::set_error(CIM_EINVAL, "unknown value kind");
  if (S->n_tiles == 0) return CIM_OK;
  if (!S->tile_rc || !S->entry_off || !S->rowptr || (S->n_entries > 0 && (!S->col || !vals_out)))
    return cim::set_error(CIM_EINVAL, "NULL arrays");
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const unsigned grid = (unsigned)std::min<long long>((S->n_tiles + 7) / 8, 4096);
  const int2 *rc = reinterpret_cast<const int2 *>(S->tile_rc);
  const long long *off = reinterpret_cast<const long long *>(S->entry_off);
  if (dtype == CIM_F32)
    cim::fill_sparse_values_kernel<float><<<grid, 256, 0, stream>>>(rc, off, S->rowptr, S->col, S->n_tiles, n, kind,
                                                                    seed, op_k, static_cast<const float *>(mask),
                                                                    static_cast<float *>(vals_out));
  else
    cim::fill_sparse_values_kernel<double><<<grid, 256, 0, stream>>>(rc, off, S->rowptr, S->col, S->n_tiles, n, kind,
                                                                     seed, op_k, static_cast<const double *>(mask),
                                                                     static_cast<double *>(vals_out));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("fill_sparse_values: ") + cudaGetErrorString(e));
  return CIM_OK;
}
