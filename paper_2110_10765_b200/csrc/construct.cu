// GPU construction of the half-stored matrix from a many-body basis — the
// reference's two-pass skeleton build (count → scan → fill,
// build_skeleton pipeline.py:290-377) straight into 64-tiles:
//
//   kept(i, j)  ⇔  popcount(lo_i ⊕ lo_j) ≤ thr          (prefilter,  sparsity.py:137-152)
//              ∧  occ_diff(occ_i, occ_j) ≤ thr        (exact walk, sparsity.py:158-178)
//   value(i,j)  =  h(i XOR j; seed)                      (pipeline.py:216-222)
//
// over the grouped basis order (group_orbitals, pipeline.py:131-159).  The
// reference enumerates orbital-pair tiles first and prunes by their keys;
// here the host prunes 64-row block pairs with a popcount lower bound built
// from each block's AND / OR of the packed words, then one thread per
// (candidate tile, local row) counts (cim_basis_count_tiles) and, after the
// caller's scan, fills dense tiles (cim_basis_fill_dense, fragment order) or
// sparse tiles (cim_basis_fill_sparse, row-sorted entries).
#include <cstdint>
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

// _occ_diff: lockstep walk of two sorted occupation lists (sparsity.py:158-178).
__device__ __forceinline__ int occ_diff(const uint16_t *a, const uint16_t *b, int n1, int n2) {
  int i1 = 0, i2 = 0, d1 = 0, d2 = 0;
  while (i1 < n1 && i2 < n2) {
    const uint16_t x = a[i1], y = b[i2];
    if (x == y) {
      ++i1;
      ++i2;
    } else if (x < y) {
      ++d1;
      ++i1;
    } else {
      ++d2;
      ++i2;
    }
  }
  return 2 * (d1 > d2 ? d1 : d2);
}

__device__ __forceinline__ bool kept(const uint64_t *lo, const uint16_t *occ, int npart, int thr, long long i,
                                     long long j) {
  if (__popcll(lo[i] ^ lo[j]) > thr) return false;
  return occ_diff(occ + i * npart, occ + j * npart, npart, npart) <= thr;
}

__global__ void basis_count_kernel(const uint64_t *lo, const uint16_t *occ, long long n, int npart, int thr,
                                   const int2 *rc, long long n_tiles, int *rowcnt) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_tiles * 64) return;
  const int2 t = rc[g >> 6];
  const long long i = (long long)t.x * 64 + (g & 63);
  int cnt = 0;
  if (i < n)
    for (int c = 0; c < 64; ++c) {
      const long long j = (long long)t.y * 64 + c;
      if (j < n && kept(lo, occ, npart, thr, i, j)) ++cnt;
    }
  rowcnt[g] = cnt;
}

template <typename T>
__global__ void basis_fill_dense_kernel(const uint64_t *lo, const uint16_t *occ, long long n, int npart, int thr,
                                        const int2 *rc, long long n_tiles, int layout, uint64_t seed, T *vals) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_tiles * (long long)kTileElems) return;
  const int2 t = rc[g / kTileElems];
  int r, c;
  layout_index_to_rc<T>(layout, (int)(g % kTileElems), r, c);
  const long long i = (long long)t.x * 64 + r, j = (long long)t.y * 64 + c;
  const bool on = i < n && j < n && kept(lo, occ, npart, thr, i, j);
  vals[g] = on ? (T)h_value((uint64_t)i, (uint64_t)j, seed) : T(0);
}

template <typename T>
__global__ void basis_fill_sparse_kernel(const uint64_t *lo, const uint16_t *occ, long long n, int npart, int thr,
                                         const int2 *rc, const long long *entry_off, const uint16_t *rowptr,
                                         long long n_tiles, uint64_t seed, uint8_t *col, uint8_t *row, T *vals) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_tiles * 64) return;
  const long long tt = g >> 6;
  const int r = (int)(g & 63);
  const int2 t = rc[tt];
  const long long i = (long long)t.x * 64 + r;
  if (i >= n) return;
  long long e = entry_off[tt] + rowptr[tt * kSpPtrStride + r];
  for (int c = 0; c < 64; ++c) {
    const long long j = (long long)t.y * 64 + c;
    if (j < n && kept(lo, occ, npart, thr, i, j)) {
      col[e] = (uint8_t)c;
      row[e] = (uint8_t)r;
      vals[e] = (T)h_value((uint64_t)i, (uint64_t)j, seed);
      ++e;
    }
  }
}

int check_basis(const uint64_t *lo, const uint16_t *occ, int64_t n, int32_t npart, int32_t thr) {
  if (n < 1 || npart < 1 || npart > 128 || thr < 0) return set_error(CIM_EINVAL, "bad basis arguments");
  if (!lo || !occ) return set_error(CIM_EINVAL, "NULL basis arrays");
  return CIM_OK;
}

}  // namespace
}  // namespace cim

extern "C" int cim_basis_count_tiles(const uint64_t *bits_lo, const uint16_t *occ, int64_t n, int32_t n_particles,
                                     int32_t threshold, const int32_t *tile_rc, int64_t n_tiles, int32_t *rowcnt,
                                     void *stream) {
  cim::clear_error();
  int rc = cim::check_basis(bits_lo, occ, n, n_particles, threshold);
  if (rc) return rc;
  if (n_tiles < 0) return cim::set_error(CIM_EINVAL, "n_tiles must be >= 0");
  if (n_tiles == 0) return CIM_OK;
  if (!tile_rc || !rowcnt) return cim::set_error(CIM_EINVAL, "NULL tile arrays");
  const long long threads = n_tiles * 64;
  cim::basis_count_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      bits_lo, occ, n, n_particles, threshold, reinterpret_cast<const int2 *>(tile_rc), n_tiles, rowcnt);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("basis_count: ") + cudaGetErrorString(e));
  return CIM_OK;
}

extern "C" int cim_basis_fill_dense(const uint64_t *bits_lo, const uint16_t *occ, int64_t n, int32_t n_particles,
                                    int32_t threshold, const int32_t *tile_rc, int64_t n_tiles, int32_t dtype,
                                    int32_t layout, uint64_t seed, void *vals, void *stream) {
  cim::clear_error();
  int rc = cim::check_basis(bits_lo, occ, n, n_particles, threshold);
  if (rc) return rc;
  if (dtype != CIM_F32 && dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (layout != CIM_LAYOUT_FRAG && layout != CIM_LAYOUT_TC)
    return cim::set_error(CIM_EINVAL, "unknown layout for dtype");
  if (n_tiles == 0) return CIM_OK;
  if (!tile_rc || !vals) return cim::set_error(CIM_EINVAL, "NULL tile arrays");
  const long long threads = n_tiles * (long long)cim::kTileElems;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int2 *t = reinterpret_cast<const int2 *>(tile_rc);
  if (dtype == CIM_F32)
    cim::basis_fill_dense_kernel<float><<<grid, 256, 0, s>>>(bits_lo, occ, n, n_particles, threshold, t, n_tiles,
                                                             layout, seed, static_cast<float *>(vals));
  else
    cim::basis_fill_dense_kernel<double><<<grid, 256, 0, s>>>(bits_lo, occ, n, n_particles, threshold, t, n_tiles,
                                                              layout, seed, static_cast<double *>(vals));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("basis_fill_dense: ") + cudaGetErrorString(e));
  return CIM_OK;
}

extern "C" int cim_basis_fill_sparse(const uint64_t *bits_lo, const uint16_t *occ, int64_t n, int32_t n_particles,
                                     int32_t threshold, const cim_sparse_tiles *S, int32_t dtype, uint64_t seed,
                                     void *stream) {
  cim::clear_error();
  int rc = cim::check_basis(bits_lo, occ, n, n_particles, threshold);
  if (rc) return rc;
  if (!S) return cim::set_error(CIM_EINVAL, "S is NULL");
  if (dtype != CIM_F32 && dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (S->n_tiles == 0) return CIM_OK;
  if (!S->tile_rc || !S->entry_off || !S->rowptr || (S->n_entries > 0 && (!S->col || !S->row || !S->vals)))
    return cim::set_error(CIM_EINVAL, "NULL sparse arrays");
  const long long threads = S->n_tiles * 64;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int2 *t = reinterpret_cast<const int2 *>(S->tile_rc);
  const long long *off = reinterpret_cast<const long long *>(S->entry_off);
  uint8_t *col = const_cast<uint8_t *>(S->col), *row = const_cast<uint8_t *>(S->row);
  if (dtype == CIM_F32)
    cim::basis_fill_sparse_kernel<float><<<grid, 256, 0, s>>>(bits_lo, occ, n, n_particles, threshold, t, off,
                                                              S->rowptr, S->n_tiles, seed, col, row,
                                                              static_cast<float *>(const_cast<void *>(S->vals)));
  else
    cim::basis_fill_sparse_kernel<double><<<grid, 256, 0, s>>>(bits_lo, occ, n, n_particles, threshold, t, off,
                                                               S->rowptr, S->n_tiles, seed, col, row,
                                                               static_cast<double *>(const_cast<void *>(S->vals)));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("basis_fill_sparse: ") + cudaGetErrorString(e));
  return CIM_OK;
}
