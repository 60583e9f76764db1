// CIM_DETERMINISTIC: the same operator without float atomics (SURVEY.md §7
// "Nondeterminism"; §8(b) flags).  The fast kernels reduce Y_C with
// red.global, so the summation order of a column block depends on timing and
// Y is reproducible only to rounding; this validation mode is bitwise
// reproducible.  One CTA owns block row b of Y and sums, in (R, C) order,
//   direct      T·X_C   over the tiles of block row b,
//   transposed  Tᵀ·X_R  over the tiles of block column b with R < b,
// with thread (row r, vector group g) accumulating in registers in a fixed
// order and writing Y once.  Every off-diagonal tile is read twice (once per
// side) — a correctness mode, not the hot path.  The tile lists index dense
// tiles as t < n_dense and COO-in-tile sparse tiles as n_dense + s; a sparse
// tile is walked along row r (rowptr / col, direct) or column r (colptr /
// cperm, transposed) in its stored order, so the summation order is fixed.
#include <cstdint>
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

constexpr int kDetThreads = 256;  // 64 rows × 4 vector groups
constexpr int kDetMaxK = 64;

// Storage index of tile element (r, c) in fragment layout v1 (include/cim_b200.h).
template <typename T>
__device__ __forceinline__ int frag_index(int r, int c) {
  const int rg = r & 7, i = r >> 3, cg = c & 15, j = c >> 4;
  const int mb = 32 * (cg >> 2) + 4 * rg + (cg & 3);
  if constexpr (sizeof(T) == 4)
    return (i * 128 + mb) * 4 + j;
  else
    return ((2 * i + (j >> 1)) * 128 + mb) * 2 + (j & 1);
}

// Storage index of tile element (r, c) in either tile layout: fragment order
// v1 or the tensor-core layout's row-major rows with 4-element chunks
// XOR-swizzled by row (include/cim_b200.h).
template <typename T, bool TC>
__device__ __forceinline__ int tile_index(int r, int c) {
  if constexpr (TC)
    return r * 64 + (((c >> 2) ^ (r & 7)) << 2) + (c & 3);
  else
    return frag_index<T>(r, c);
}

template <typename T>
struct DetSparse {
  long long n_tiles;
  const int2 *tile_rc;
  const long long *entry_off;
  const uint16_t *rowptr, *colptr, *cperm;
  const uint8_t *col, *row;
  const T *vals;
};

template <typename T, int VMAX>
__device__ __forceinline__ void det_fma(T (&acc)[VMAX], T a, const T *x, int g, int k) {
#pragma unroll
  for (int q = 0; q < VMAX; ++q) {
    const int v = g + 4 * q;
    if (v < k) acc[q] = fma(a, x[v], acc[q]);
  }
}

template <typename T, bool TC>
__global__ void __launch_bounds__(kDetThreads) det_spmm_kernel(int n_dense, const int2 *tile_rc, const T *vals,
                                                               DetSparse<T> sp, const long long *row_ptr,
                                                               const int *row_tiles, const long long *col_ptr,
                                                               const int *col_tiles, const T *X, T *Y, int k,
                                                               long long ldy, bool accumulate) {
  const int b = blockIdx.x;
  const int r = threadIdx.x & 63, g = threadIdx.x >> 6;
  constexpr int VMAX = kDetMaxK / 4;
  T acc[VMAX];
#pragma unroll
  for (int q = 0; q < VMAX; ++q) acc[q] = T(0);
  // direct: Y_b[r] += Σ_c T[r][c] X_C[c]
  for (long long s = row_ptr[b]; s < row_ptr[b + 1]; ++s) {
    const int t = row_tiles[s];
    if (t >= n_dense) {
      const long long u = t - n_dense;
      const T *xc = X + (long long)sp.tile_rc[u].y * 64 * k;
      const long long base = sp.entry_off[u];
      const uint16_t *rp = sp.rowptr + u * kSpPtrStride;
      for (long long e = base + rp[r]; e < base + rp[r + 1]; ++e)
        det_fma<T, VMAX>(acc, sp.vals[e], xc + (long long)sp.col[e] * k, g, k);
      continue;
    }
    const int C = tile_rc[t].y;
    const T *tv = vals + (size_t)t * kTileElems;
    const T *xc = X + (long long)C * 64 * k;
    for (int c = 0; c < 64; ++c) det_fma<T, VMAX>(acc, tv[tile_index<T, TC>(r, c)], xc + (long long)c * k, g, k);
  }
  // transposed: Y_b[r] += Σ_r' T[r'][r] X_R[r'] over tiles (R, b), R < b
  for (long long s = col_ptr[b]; s < col_ptr[b + 1]; ++s) {
    const int t = col_tiles[s];
    if (t >= n_dense) {
      const long long u = t - n_dense;
      const T *xr = X + (long long)sp.tile_rc[u].x * 64 * k;
      const long long base = sp.entry_off[u];
      const uint16_t *cp = sp.colptr + u * kSpPtrStride;
      for (int q = cp[r]; q < cp[r + 1]; ++q) {
        const long long e = base + sp.cperm[base + q];
        det_fma<T, VMAX>(acc, sp.vals[e], xr + (long long)sp.row[e] * k, g, k);
      }
      continue;
    }
    const int R = tile_rc[t].x;
    const T *tv = vals + (size_t)t * kTileElems;
    const T *xr = X + (long long)R * 64 * k;
    for (int rr = 0; rr < 64; ++rr) det_fma<T, VMAX>(acc, tv[tile_index<T, TC>(rr, r)], xr + (long long)rr * k, g, k);
  }
  T *y = Y + ((long long)b * 64 + r) * ldy;
#pragma unroll
  for (int q = 0; q < VMAX; ++q) {
    const int v = g + 4 * q;
    if (v < k) y[v] = accumulate ? y[v] + acc[q] : acc[q];
  }
}

}  // namespace

int sym_spmm_deterministic(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, bool accumulate,
                           cudaStream_t stream) {
  if (H->layout != CIM_LAYOUT_FRAG && H->layout != CIM_LAYOUT_TC) return set_error(CIM_EINVAL, "unknown tile layout");
  if (k > kDetMaxK) return set_error(CIM_EUNSUPPORTED, "CIM_DETERMINISTIC supports k <= 64");
  if (!H->det_row_ptr || !H->det_row_tiles || !H->det_col_ptr || !H->det_col_tiles)
    return set_error(CIM_EINVAL, "CIM_DETERMINISTIC needs the det_* tile lists");
  if (H->n_tiles > INT32_MAX) return set_error(CIM_EUNSUPPORTED, "CIM_DETERMINISTIC: too many tiles");
  const long long nb = (H->n + kBlock - 1) / kBlock;
  const int2 *rc = reinterpret_cast<const int2 *>(H->tile_rc);
  const cim_sparse_tiles *S = H->sparse;
  const bool has_sp = S && S->n_tiles > 0;
  if (has_sp && (!S->tile_rc || !S->entry_off || !S->rowptr || !S->colptr ||
                 (S->n_entries > 0 && (!S->col || !S->row || !S->cperm || !S->vals))))
    return set_error(CIM_EINVAL, "NULL sparse arrays");
  auto run = [&](auto tag) {
    using T = decltype(tag);
    DetSparse<T> sp{};
    if (has_sp)
      sp = {S->n_tiles,  reinterpret_cast<const int2 *>(S->tile_rc), reinterpret_cast<const long long *>(S->entry_off),
            S->rowptr,   S->colptr, S->cperm, S->col, S->row, static_cast<const T *>(S->vals)};
    auto kern = H->layout == CIM_LAYOUT_TC ? det_spmm_kernel<T, true> : det_spmm_kernel<T, false>;
    kern<<<(unsigned)nb, kDetThreads, 0, stream>>>(
        (int)H->n_tiles, rc, static_cast<const T *>(H->vals), sp, reinterpret_cast<const long long *>(H->det_row_ptr),
        H->det_row_tiles, reinterpret_cast<const long long *>(H->det_col_ptr), H->det_col_tiles,
        static_cast<const T *>(X), static_cast<T *>(Y), k, ldy, accumulate);
  };
  if (H->dtype == CIM_F32)
    run(float{});
  else
    run(double{});
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("det_spmm_kernel: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace cim
