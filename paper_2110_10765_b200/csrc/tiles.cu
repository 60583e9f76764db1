// Repacking layer (device half) and the device twin of the reference's value
// hashes: synthetic tile values, row-major ⇄ fragment repacking, and hashing
// of explicit index arrays for parity checks.
//
// The synthetic generator replaces build_skeleton's per-entry value step
// (pipeline.py:357-368 → _h_values_np, :247-249) for matrices far beyond what
// the reference can build (C2: 2·10⁹ stored values, generated here in HBM).
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {

template <typename T>
__global__ void fill_values_kernel(const int2 *__restrict__ rc, long long n_tiles, long long n, int layout, int kind,
                                   unsigned long long seed, int op_k, T *__restrict__ vals) {
  const long long total = n_tiles * kTileElems;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e >> 12;
    const int idx = (int)(e & 4095);
    int row, col;
    layout_index_to_rc<T>(layout, idx, row, col);
    const int2 RC = rc[t];
    const long long i = (long long)RC.x * kBlock + row;
    const long long j = (long long)RC.y * kBlock + col;
    float v = 0.0f;
    if (i < n && j < n) v = value_of_kind(kind, (uint64_t)i, (uint64_t)j, seed, op_k);
    vals[e] = static_cast<T>(v);
  }
}

// vals = (mask != 0) ? value(i, j) : 0 — operator values on a stored pattern.
template <typename T>
__global__ void fill_masked_kernel(const int2 *__restrict__ rc, long long n_tiles, long long n, int layout, int kind,
                                   unsigned long long seed, int op_k, const T *__restrict__ mask,
                                   T *__restrict__ vals) {
  const long long total = n_tiles * kTileElems;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e >> 12;
    const int idx = (int)(e & 4095);
    int row, col;
    layout_index_to_rc<T>(layout, idx, row, col);
    const int2 RC = rc[t];
    const long long i = (long long)RC.x * kBlock + row;
    const long long j = (long long)RC.y * kBlock + col;
    float v = 0.0f;
    if (mask[e] != T(0) && i < n && j < n) v = value_of_kind(kind, (uint64_t)i, (uint64_t)j, seed, op_k);
    vals[e] = static_cast<T>(v);
  }
}

template <typename T>
__global__ void pack_kernel(const T *__restrict__ src, long long n_tiles, int layout, T *__restrict__ dst,
                            bool to_fragment) {
  const long long total = n_tiles * kTileElems;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e >> 12;
    const int idx = (int)(e & 4095);
    int row, col;
    layout_index_to_rc<T>(layout, idx, row, col);
    const long long rm = (t << 12) + row * kBlock + col;
    if (to_fragment)
      dst[e] = src[rm];
    else
      dst[rm] = src[e];
  }
}

__global__ void hash_kernel(const long long *__restrict__ I, const long long *__restrict__ J, long long count,
                            int kind, unsigned long long seed, int op_k, float *__restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < count;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = value_of_kind(kind, (uint64_t)I[e], (uint64_t)J[e], seed, op_k);
}

namespace {
unsigned int grid_for(long long total) {
  long long g = (total + 255) / 256;
  if (g > 148LL * 32) g = 148LL * 32;
  if (g < 1) g = 1;
  return (unsigned int)g;
}
int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return CIM_OK;
}
}  // namespace
}  // namespace cim

using namespace cim;

static bool layout_ok(int32_t layout, int32_t dtype) {
  return layout == CIM_LAYOUT_FRAG || layout == CIM_LAYOUT_TC;
}

extern "C" int cim_fill_synthetic_values(const int32_t *tile_rc, int64_t n_tiles, int64_t n, int32_t dtype,
                                         int32_t layout, int32_t kind, uint64_t seed, int32_t op_k, void *vals,
                                         void *stream) {
  clear_error();
  if (n_tiles < 0 || n < 1 || kind < 0 || kind > 2) return set_error(CIM_EINVAL, "bad arguments");
  if (!layout_ok(layout, dtype)) return set_error(CIM_EINVAL, "bad layout for dtype");
  if (n_tiles == 0) return CIM_OK;
  if (!tile_rc || !vals) return set_error(CIM_EINVAL, "NULL arrays");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long long total = n_tiles * (long long)kTileElems;
  if (dtype == CIM_F32)
    fill_values_kernel<float><<<grid_for(total), 256, 0, st>>>(reinterpret_cast<const int2 *>(tile_rc), n_tiles, n,
                                                               layout, kind, seed, op_k, static_cast<float *>(vals));
  else if (dtype == CIM_F64)
    fill_values_kernel<double><<<grid_for(total), 256, 0, st>>>(reinterpret_cast<const int2 *>(tile_rc), n_tiles, n,
                                                                layout, kind, seed, op_k, static_cast<double *>(vals));
  else
    return set_error(CIM_EINVAL, "bad dtype");
  return check_launch("fill_values_kernel");
}

extern "C" int cim_fill_masked_values(const int32_t *tile_rc, int64_t n_tiles, int64_t n, int32_t dtype,
                                      int32_t layout, int32_t kind, uint64_t seed, int32_t op_k, const void *mask,
                                      void *vals, void *stream) {
  clear_error();
  if (n_tiles < 0 || n < 1 || kind < 0 || kind > 2) return set_error(CIM_EINVAL, "bad arguments");
  if (!layout_ok(layout, dtype)) return set_error(CIM_EINVAL, "bad layout for dtype");
  if (n_tiles == 0) return CIM_OK;
  if (!tile_rc || !vals || !mask) return set_error(CIM_EINVAL, "NULL arrays");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long long total = n_tiles * (long long)kTileElems;
  if (dtype == CIM_F32)
    fill_masked_kernel<float><<<grid_for(total), 256, 0, st>>>(reinterpret_cast<const int2 *>(tile_rc), n_tiles, n,
                                                               layout, kind, seed, op_k, static_cast<const float *>(mask),
                                                               static_cast<float *>(vals));
  else if (dtype == CIM_F64)
    fill_masked_kernel<double><<<grid_for(total), 256, 0, st>>>(reinterpret_cast<const int2 *>(tile_rc), n_tiles,
                                                                n, layout, kind, seed, op_k, static_cast<const double *>(mask),
                                                                static_cast<double *>(vals));
  else
    return set_error(CIM_EINVAL, "bad dtype");
  return check_launch("fill_masked_kernel");
}

static int pack_common(const void *src, int64_t n_tiles, int32_t dtype, int32_t layout, void *dst, void *stream,
                       bool to_frag) {
  clear_error();
  if (n_tiles < 0) return set_error(CIM_EINVAL, "bad n_tiles");
  if (!layout_ok(layout, dtype)) return set_error(CIM_EINVAL, "bad layout for dtype");
  if (n_tiles == 0) return CIM_OK;
  if (!src || !dst) return set_error(CIM_EINVAL, "NULL arrays");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long long total = n_tiles * (long long)kTileElems;
  if (dtype == CIM_F32)
    pack_kernel<float><<<grid_for(total), 256, 0, st>>>(static_cast<const float *>(src), n_tiles, layout,
                                                        static_cast<float *>(dst), to_frag);
  else if (dtype == CIM_F64)
    pack_kernel<double><<<grid_for(total), 256, 0, st>>>(static_cast<const double *>(src), n_tiles, layout,
                                                         static_cast<double *>(dst), to_frag);
  else
    return set_error(CIM_EINVAL, "bad dtype");
  return check_launch("pack_kernel");
}

extern "C" int cim_pack_tiles(const void *src, int64_t n_tiles, int32_t dtype, int32_t layout, void *dst,
                              void *stream) {
  return pack_common(src, n_tiles, dtype, layout, dst, stream, true);
}

extern "C" int cim_unpack_tiles(const void *src, int64_t n_tiles, int32_t dtype, int32_t layout, void *dst,
                                void *stream) {
  return pack_common(src, n_tiles, dtype, layout, dst, stream, false);
}

extern "C" int cim_hash_values(const int64_t *i, const int64_t *j, int64_t count, int32_t kind, uint64_t seed,
                               int32_t op_k, float *out, void *stream) {
  clear_error();
  if (count < 0 || kind < 0 || kind > 2) return set_error(CIM_EINVAL, "bad arguments");
  if (count == 0) return CIM_OK;
  if (!i || !j || !out) return set_error(CIM_EINVAL, "NULL arrays");
  hash_kernel<<<grid_for(count), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const long long *>(i), reinterpret_cast<const long long *>(j), count, kind, seed, op_k, out);
  return check_launch("hash_kernel");
}
