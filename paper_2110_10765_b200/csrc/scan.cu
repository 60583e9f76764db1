// Device exclusive scan — the reference's scan motif (scan_serial,
// scan.py:131-139; the offsets of CountsAndOffsets, scan.py:45-65) for the
// count → scan → fill construction (build_skeleton, pipeline.py:319-330).
//
// Reduce-then-scan over 4096-item chunks (256 threads × 16 items, staged
// through shared memory so global loads and stores stay coalesced):
//   1. chunk_sum_kernel: one int64 sum per chunk;
//   2. chunk_scan_kernel: one CTA scans the chunk sums (looping over them in
//      4096-sum pieces with a running carry) and writes the total to y[n];
//   3. chunk_apply_kernel: every chunk scans its items on top of its offset.
// Integer adds in a fixed order: bitwise deterministic, any int64 values.
// The per-tile row scan of the sparse build (cim_sparse_tile_offsets) is a
// warp-shuffle scan of each tile's 64 row counts, then the scan above over
// the padded tile sizes.
#include <cstdint>
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanChunk = kScanThreads * kScanItems;  // 4096

// Exclusive scan of one value per thread across the block; returns the
// thread's exclusive prefix and sets `total` (every thread) to the block sum.
__device__ __forceinline__ long long block_exclusive_scan(long long v, long long &total) {
  __shared__ long long warp_tot[kScanThreads / 32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  long long incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += u;
  }
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  long long base = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < kScanThreads / 32; ++q) {
    const long long t = warp_tot[q];
    base += q < w ? t : 0;
    tot += t;
  }
  __syncthreads();  // warp_tot reusable by the next call
  total = tot;
  return base + incl - v;
}

// Load chunk `c` into shared memory (coalesced), zero past n.
__device__ __forceinline__ void load_chunk(const long long *x, long long n, long long c, long long *sm) {
  const long long base = c * kScanChunk;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int idx = it * kScanThreads + threadIdx.x;
    const long long g = base + idx;
    sm[idx] = g < n ? x[g] : 0;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kScanThreads) chunk_sum_kernel(const long long *x, long long n, long long *sums) {
  __shared__ long long sm[kScanChunk];
  load_chunk(x, n, blockIdx.x, sm);
  long long s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) s += sm[threadIdx.x * kScanItems + it];
  long long tot;
  block_exclusive_scan(s, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// sums → exclusive chunk offsets (in place); y_total ← Σ sums.
__global__ void __launch_bounds__(kScanThreads) chunk_scan_kernel(long long *sums, long long n_chunks,
                                                                  long long *y_total) {
  __shared__ long long sm[kScanChunk];
  long long carry = 0;
  for (long long c = 0; c * kScanChunk < n_chunks; ++c) {
    load_chunk(sums, n_chunks, c, sm);
    long long loc[kScanItems];
    long long s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      loc[it] = s;
      s += sm[threadIdx.x * kScanItems + it];
    }
    long long tot;
    const long long pre = block_exclusive_scan(s, tot);
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) sm[threadIdx.x * kScanItems + it] = carry + pre + loc[it];
    __syncthreads();
    const long long base = c * kScanChunk;
#pragma unroll
    for (int it = 0; it < kScanItems; ++it) {
      const int idx = it * kScanThreads + threadIdx.x;
      if (base + idx < n_chunks) sums[base + idx] = sm[idx];
    }
    __syncthreads();
    carry += tot;
  }
  if (threadIdx.x == 0) *y_total = carry;
}

__global__ void __launch_bounds__(kScanThreads) chunk_apply_kernel(const long long *x, long long n,
                                                                   const long long *offs, long long *y) {
  __shared__ long long sm[kScanChunk];
  load_chunk(x, n, blockIdx.x, sm);
  long long loc[kScanItems];
  long long s = 0;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    loc[it] = s;
    s += sm[threadIdx.x * kScanItems + it];
  }
  long long tot;
  const long long pre = offs[blockIdx.x] + block_exclusive_scan(s, tot);
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) sm[threadIdx.x * kScanItems + it] = pre + loc[it];
  __syncthreads();
  const long long base = (long long)blockIdx.x * kScanChunk;
#pragma unroll
  for (int it = 0; it < kScanItems; ++it) {
    const int idx = it * kScanThreads + threadIdx.x;
    if (base + idx < n) y[base + idx] = sm[idx];
  }
}

// One warp per tile: shuffle scan of the 64 row counts (two per lane).
__global__ void tile_row_scan_kernel(const int *rowcnt, long long n_tiles, int align, short *rowptr,
                                     long long *counts, long long *padded) {
  const long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n_tiles) return;
  const int a = rowcnt[t * 64 + 2 * lane], b = rowcnt[t * 64 + 2 * lane + 1];
  int incl = a + b;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += u;
  }
  const int excl = incl - a - b;
  short *rp = rowptr + t * kSpPtrStride;
  rp[2 * lane] = (short)excl;
  rp[2 * lane + 1] = (short)(excl + a);
  if (lane == 31) {
    rp[64] = (short)incl;
    counts[t] = incl;
    padded[t] = (long long)(incl + align - 1) / align * align;
  }
  if (lane >= 1 && lane < 8) rp[64 + lane] = 0;
}

int launch_scan(const long long *x, long long n, long long *y, cudaStream_t s) {
  const long long n_chunks = (n + kScanChunk - 1) / kScanChunk;
  if (n == 0) {
    const cudaError_t e = cudaMemsetAsync(y, 0, sizeof(long long), s);
    return e == cudaSuccess ? CIM_OK : set_error(CIM_ECUDA, std::string("scan: ") + cudaGetErrorString(e));
  }
  long long *sums = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&sums), sizeof(long long) * (size_t)n_chunks, s);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("scan scratch: ") + cudaGetErrorString(e));
  chunk_sum_kernel<<<(unsigned)n_chunks, kScanThreads, 0, s>>>(x, n, sums);
  chunk_scan_kernel<<<1, kScanThreads, 0, s>>>(sums, n_chunks, y + n);
  chunk_apply_kernel<<<(unsigned)n_chunks, kScanThreads, 0, s>>>(x, n, sums, y);
  e = cudaGetLastError();
  cudaFreeAsync(sums, s);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("scan: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace
}  // namespace cim

extern "C" int cim_exclusive_scan_i64(const int64_t *x, int64_t n, int64_t *y, void *stream) {
  cim::clear_error();
  if (n < 0) return cim::set_error(CIM_EINVAL, "n must be >= 0");
  if (!y || (n > 0 && !x)) return cim::set_error(CIM_EINVAL, "NULL x / y");
  if (n > 0 && x != y && x < y + n + 1 && y < x + n)
    return cim::set_error(CIM_EINVAL, "x and y overlap without being the same array");
  if ((n + cim::kScanChunk - 1) / cim::kScanChunk > 0x7fffffffll) return cim::set_error(CIM_EINVAL, "n too large");
  return cim::launch_scan(reinterpret_cast<const long long *>(x), n, reinterpret_cast<long long *>(y),
                          reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int cim_sparse_tile_offsets(const int32_t *rowcnt, int64_t n_tiles, int32_t align, int16_t *rowptr,
                                       int64_t *counts, int64_t *entry_off, void *stream) {
  cim::clear_error();
  if (n_tiles < 0) return cim::set_error(CIM_EINVAL, "n_tiles must be >= 0");
  if (align < 1) return cim::set_error(CIM_EINVAL, "align must be >= 1");
  if (!entry_off || (n_tiles > 0 && (!rowcnt || !rowptr || !counts)))
    return cim::set_error(CIM_EINVAL, "NULL arrays");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (n_tiles > 0) {
    const long long threads = n_tiles * 32;
    // padded sizes go to entry_off[1..n_tiles] first, then scan in place shifted by one
    cim::tile_row_scan_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, s>>>(
        rowcnt, n_tiles, align, rowptr, reinterpret_cast<long long *>(counts),
        reinterpret_cast<long long *>(entry_off) + 1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("tile_row_scan: ") + cudaGetErrorString(e));
  }
  // entry_off[0..n) = exclusive scan of padded sizes, entry_off[n] = total.  The
  // padded sizes sit at entry_off[1..n]; the scan reads them into shared
  // memory chunk by chunk, so scan a staging copy to keep reads ahead of writes.
  long long *tmp = nullptr;
  if (n_tiles > 0) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void **>(&tmp), sizeof(long long) * (size_t)n_tiles, s);
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("offsets scratch: ") + cudaGetErrorString(e));
    e = cudaMemcpyAsync(tmp, entry_off + 1, sizeof(long long) * (size_t)n_tiles, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("offsets copy: ") + cudaGetErrorString(e));
  }
  const int rc = cim::launch_scan(tmp, n_tiles, reinterpret_cast<long long *>(entry_off), s);
  if (tmp) cudaFreeAsync(tmp, s);
  return rc;
}
