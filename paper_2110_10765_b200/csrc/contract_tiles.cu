// The reference's observables operator over ORBITAL tiles — the literal
// drop-in of contract_observables / contract_oracle (pipeline.py:534-589):
//
//   accum[v, k] = Σ_(tiles (r, c)) Σ_(i ∈ r, j ∈ c, kept(i, j)) c[v,i] · O_ij(k) · c[v,j]
//
// where kept(i, j) is the count predicate the reference re-walks each tile
// with (_collect_pairs → count_pairs "combined" + _fill_tile_cols,
// pipeline.py:428-458, :270-280: popcount(lo_i ⊕ lo_j) ≤ thr and the
// lockstep occupation difference ≤ thr) and O_ij(k) is _op_value
// (pipeline.py:224-232).  Nothing is materialised: one warp walks one tile's
// |r|·|c| candidate pairs (lanes over the flattened pair index), evaluates
// the predicate and, for kept pairs, hashes O once per operator and adds
// c[v,i]·O·c[v,j] into per-lane accumulators (an 8-vector × 8-operator chunk);
// warps reduce with shuffles, the block in shared memory, and one f64
// atomic per (v, k) per block lands the sum.
//
// Two product modes: the reference's f32 arithmetic ((c_vi·o)·c_vj rounded
// in f32, pipeline.py:470-474) summed per lane in f32 and across lanes in
// f64 (contract_observables), or everything in f64 (contract_oracle,
// pipeline.py:573-589: c.astype(float64)·o·c).
#include <cstdint>
#include <string>
#include <type_traits>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

constexpr int kCtNV = 8;  // vectors per chunk
constexpr int kCtKS = 8;  // operators per chunk
constexpr int kCtThreads = 256;

__device__ __forceinline__ int occ_diff_walk(const uint16_t *a, const uint16_t *b, int n) {  // sparsity.py:132-151
  int i1 = 0, i2 = 0, d1 = 0, d2 = 0;
  while (i1 < n && i2 < n) {
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

template <bool kF64>
__global__ void __launch_bounds__(kCtThreads) contract_tiles_kernel(
    const uint64_t *__restrict__ lo, const uint16_t *__restrict__ occ, int npart, int thr,
    const int4 *__restrict__ tiles, long long n_tiles, const float *__restrict__ c, long long ldc, int v0, int nv,
    int k0, int ks, int identity, uint64_t seed, double *__restrict__ accum, int m_ops) {
  using Acc = typename std::conditional<kF64, double, float>::type;
  Acc acc[kCtNV][kCtKS];
#pragma unroll
  for (int v = 0; v < kCtNV; ++v)
#pragma unroll
    for (int k = 0; k < kCtKS; ++k) acc[v][k] = Acc(0);

  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * kCtThreads + threadIdx.x) >> 5;
  const long long n_warps = ((long long)gridDim.x * kCtThreads) >> 5;
  for (long long t = warp; t < n_tiles; t += n_warps) {
    const int4 tr = tiles[t];  // r0, r1, c0, c1
    const int nc = tr.w - tr.z;
    const long long np = (long long)(tr.y - tr.x) * nc;
    for (long long p = lane; p < np; p += 32) {
      const long long i = tr.x + p / nc, j = tr.z + p % nc;
      if (__popcll(lo[i] ^ lo[j]) > thr) continue;
      if (occ_diff_walk(occ + i * npart, occ + j * npart, npart) > thr) continue;
      float o[kCtKS];
      if (identity) {
#pragma unroll
        for (int k = 0; k < kCtKS; ++k) o[k] = i == j ? 1.0f : 0.0f;
      } else {
        const uint64_t a = (uint64_t)(i < j ? i : j), b = (uint64_t)(i < j ? j : i);
        const uint64_t u = mix64(a + kGolden * b);  // k-independent prefix (pipeline.py:229)
#pragma unroll
        for (int k = 0; k < kCtKS; ++k)
          o[k] = k < ks ? to_unit(mix64(mix64(u ^ ((uint64_t)(k0 + k) + 1ull) * kMix1) ^ seed)) : 0.0f;
      }
#pragma unroll
      for (int v = 0; v < kCtNV; ++v) {
        if (v < nv) {
          const float ci = c[i * ldc + v0 + v], cj = c[j * ldc + v0 + v];
#pragma unroll
          for (int k = 0; k < kCtKS; ++k) {
            if constexpr (kF64)
              acc[v][k] += (double)ci * (double)o[k] * (double)cj;
            else
              acc[v][k] += __fmul_rn(__fmul_rn(ci, o[k]), cj);
          }
        }
      }
    }
  }
  // warp → block → one f64 atomic per (v, k) per block
  __shared__ double part[kCtThreads / 32][kCtNV * kCtKS];
  const int w = threadIdx.x >> 5;
#pragma unroll
  for (int v = 0; v < kCtNV; ++v)
#pragma unroll
    for (int k = 0; k < kCtKS; ++k) {
      double s = (double)acc[v][k];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (lane == 0) part[w][v * kCtKS + k] = s;
    }
  __syncthreads();
  if (threadIdx.x < kCtNV * kCtKS) {
    const int v = threadIdx.x / kCtKS, k = threadIdx.x % kCtKS;
    if (v < nv && k < ks) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < kCtThreads / 32; ++q) s += part[q][threadIdx.x];
      atomicAdd(accum + (long long)(v0 + v) * m_ops + (k0 + k), s);
    }
  }
}

}  // namespace
}  // namespace cim

extern "C" int cim_contract_tiles(const uint64_t *bits_lo, const uint16_t *occ, int64_t n, int32_t n_particles,
                                  int32_t threshold, const int32_t *tile_ranges, int64_t n_tiles, const float *c,
                                  int64_t ldc, int32_t n_vec, int32_t m_ops, int32_t kind, uint64_t seed,
                                  double *accum, uint32_t flags, void *stream) {
  cim::clear_error();
  if (n < 1 || n_particles < 1 || n_particles > 128 || threshold < 0)
    return cim::set_error(CIM_EINVAL, "bad basis arguments");
  if (!bits_lo || !occ) return cim::set_error(CIM_EINVAL, "NULL basis arrays");
  if (n_tiles < 0) return cim::set_error(CIM_EINVAL, "n_tiles must be >= 0");
  if (n_vec < 1 || m_ops < 1) return cim::set_error(CIM_EINVAL, "n_vec and m_ops must be >= 1");
  if (ldc < n_vec) return cim::set_error(CIM_EINVAL, "ldc must be >= n_vec");
  if (kind != CIM_VALUES_OP_HASH && kind != CIM_VALUES_IDENTITY)
    return cim::set_error(CIM_EINVAL, "kind must be CIM_VALUES_OP_HASH or CIM_VALUES_IDENTITY");
  if (!c || !accum) return cim::set_error(CIM_EINVAL, "NULL c / accum");
  if (n_tiles > 0 && !tile_ranges) return cim::set_error(CIM_EINVAL, "NULL tile_ranges");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!(flags & CIM_ACCUMULATE)) {
    const cudaError_t e = cudaMemsetAsync(accum, 0, sizeof(double) * (size_t)n_vec * (size_t)m_ops, s);
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("contract_tiles memset: ") + cudaGetErrorString(e));
  }
  if (n_tiles == 0) return CIM_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (n_tiles + cim::kCtThreads / 32 - 1) / (cim::kCtThreads / 32);
  const unsigned grid = (unsigned)(want < (long long)sms * 8 ? want : (long long)sms * 8);
  const int4 *t = reinterpret_cast<const int4 *>(tile_ranges);
  const bool f64 = (flags & CIM_CONTRACT_EXACT_F64) != 0;
  const int identity = kind == CIM_VALUES_IDENTITY;
  for (int v0 = 0; v0 < n_vec; v0 += cim::kCtNV)
    for (int k0 = 0; k0 < m_ops; k0 += cim::kCtKS) {
      const int nv = n_vec - v0 < cim::kCtNV ? n_vec - v0 : cim::kCtNV;
      const int ks = m_ops - k0 < cim::kCtKS ? m_ops - k0 : cim::kCtKS;
      if (f64)
        cim::contract_tiles_kernel<true><<<grid, cim::kCtThreads, 0, s>>>(
            bits_lo, occ, n_particles, threshold, t, n_tiles, c, ldc, v0, nv, k0, ks, identity, seed, accum, m_ops);
      else
        cim::contract_tiles_kernel<false><<<grid, cim::kCtThreads, 0, s>>>(
            bits_lo, occ, n_particles, threshold, t, n_tiles, c, ldc, v0, nv, k0, ks, identity, seed, accum, m_ops);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess)
        return cim::set_error(CIM_ECUDA, std::string("contract_tiles: ") + cudaGetErrorString(e));
    }
  return CIM_OK;
}
