// The observables contraction fused into one tile walk:
//
//   accum[v, k] = Σ_(i,j) c[v,i] · O_ij(k) · c[v,j]
//
// over the full symmetric pattern of a stored HalfTiles (contract_observables,
// pipeline.py:534-570; kernels _contract_array_clause / _contract_atomic,
// :461-531).  O_ij(k) is the reference's symmetric hash (_op_value,
// pipeline.py:224-232) or the identity, computed on the fly — nothing is
// materialised.  The pattern is the set of nonzero stored elements; an
// off-diagonal tile (R < C) stands for its pairs and their mirror images
// (weight 2, O and the c-products are symmetric), a diagonal tile is stored in
// full (weight 1).
//
// One CTA (256 threads) walks tiles in a grid-stride loop.  Per tile the CTA
// turns the stored values (dense fragment / tc layout, or COO-in-tile sparse
// entries) into 64 row bitmasks in shared memory and stages the 64-row
// blocks c[·, R] and c[·, C] (≤ 16 vectors).  Thread (row r, slot s) then walks
// the set bits of its row in its column range: per pair it forms
// p_v = w·c[v,i]·c[v,j] once, the k-independent hash prefix
// mix64(lo + φ·hi) once, and for each of its ≤ 4 operators two mix64 and one
// int→f32 conversion, accumulating acc[k][v] += p_v·O_ij(k) in f32 registers —
// the "per-(v,k) register reduction".  Slots split the operators (GK groups of
// KS ≤ 4, chosen from m so no hash is computed for nothing when m < 4) and,
// when there are fewer operator groups, the columns; the identity operator
// is one walk added to every column.  At the end each warp reduces its
// accumulators with shuffles and adds them to the f64 accum with one atomic
// per (v, k).  The host loops over chunks of 16 vectors and 16 operators.
// The work per pair is integer hashing (~34 ALU-pipe ops per operator for
// two 64-bit mix64 and the conversion): the kernel is ALU-bound (ncu: ALU
// pipe 71%), not HBM-bound.
#include <algorithm>
#include <cstdint>
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

constexpr int kCtThreads = 256;
#ifndef CIM_CT_MINB4
#define CIM_CT_MINB4 2  // resident CTAs per SM the register budget targets (KS = 4; A/B knob)
#endif
#define CIM_CT_MINB(KS) ((KS) == 4 ? CIM_CT_MINB4 : 3)
// small-tile kernel: ~150 registers per thread (8 operators × 8 vectors of
// accumulators), so 4-warp blocks let three blocks share an SM where one
// 8-warp block left 8 warps resident
constexpr int kCtSmallThreads = 128;

template <typename T>
struct ContractArgs {
  long long n, n_dense;
  const int2 *rc;
  const T *vals;
  int layout;
  long long n_sparse;
  const int2 *sp_rc;
  const long long *sp_off;
  const uint16_t *sp_rowptr;
  const uint8_t *sp_col, *sp_row;
  const T *sp_vals;
  const int32_t *sp_list;  // optional: the sparse tiles this kernel walks (else all n_sparse)
  const float *c;  // (n, n_vec) row-major
  int n_vec, v0, nv;
  int m_ops, k0, kc;
  uint64_t seed;
  double *accum;  // (n_vec, m_ops) row-major
};

// NV vectors per launch, GK operator groups of KS operators per thread
// (GK·KS ≥ the launch's operator count), IDENT: the identity operator (same
// value for every k — one walk, added to every column of accum).
template <typename T, int NV, int GK, int KS, bool IDENT>
__global__ void __launch_bounds__(kCtThreads, CIM_CT_MINB(KS)) contract_kernel(ContractArgs<T> a) {
  __shared__ unsigned rowmask[64][2];  // 32-bit words: shared atomicOr is native at 32 bits
  __shared__ __align__(16) float xr[64][NV];
  __shared__ __align__(16) float xc[64][NV];
  const int tid = threadIdx.x;
  const int r = tid & 63, slot = tid >> 6;
  const int kg = slot % GK;
  constexpr int S = 4 / GK;  // column splits
  const int cs = slot / GK;
  const unsigned long long colrange =
      S == 1 ? ~0ull : (((1ull << (64 / S)) - 1ull) << (cs * (64 / S)));
  uint64_t kq[KS];
#pragma unroll
  for (int q = 0; q < KS; ++q) kq[q] = (uint64_t)(a.k0 + kg + GK * q + 1) * kMix1;
  float acc[KS][NV];
#pragma unroll
  for (int q = 0; q < KS; ++q)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[q][v] = 0.f;

  const long long total = a.n_dense + a.n_sparse;
  for (long long t = blockIdx.x; t < total; t += gridDim.x) {
    const bool dense = t < a.n_dense;
    const long long u = dense ? t : (a.sp_list ? (long long)a.sp_list[t - a.n_dense] : t - a.n_dense);
    const int2 RC = dense ? a.rc[u] : a.sp_rc[u];
    if (tid < 128) rowmask[tid >> 1][tid & 1] = 0u;
    // stage the two c blocks (zero outside the matrix / vector chunk)
    for (int e = tid; e < 2 * 64 * NV; e += kCtThreads) {
      const int side = e / (64 * NV), rr = (e / NV) & 63, v = e % NV;
      const long long row = (long long)(side ? RC.y : RC.x) * 64 + rr;
      const float x = (row < a.n && v < a.nv) ? a.c[row * a.n_vec + a.v0 + v] : 0.f;
      (side ? xc : xr)[rr][v] = x;
    }
    __syncthreads();
    if (dense) {
      const T *tv = a.vals + u * kTileElems;
#pragma unroll 4
      for (int e = tid; e < kTileElems; e += kCtThreads) {
        if (tv[e] != T(0)) {
          int rr, cc;
          layout_index_to_rc<T>(a.layout, e, rr, cc);
          atomicOr(&rowmask[rr][cc >> 5], 1u << (cc & 31));
        }
      }
    } else {
      const long long base = a.sp_off[u];
      const int cnt = a.sp_rowptr[u * kSpPtrStride + 64];
      for (int e = tid; e < cnt; e += kCtThreads)
        if (a.sp_vals[base + e] != T(0)) {
          const int cc = a.sp_col[base + e];
          atomicOr(&rowmask[a.sp_row[base + e]][cc >> 5], 1u << (cc & 31));
        }
    }
    __syncthreads();
    const long long i = (long long)RC.x * 64 + r;
    unsigned long long m = (((unsigned long long)rowmask[r][1] << 32) | rowmask[r][0]) & colrange;
    if (i >= a.n) m = 0ull;
    const float w = RC.x == RC.y ? 1.f : 2.f;
    float ci[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) ci[v] = w * xr[r][v];
    while (m) {
      const int cc = __ffsll((long long)m) - 1;
      m &= m - 1;
      const long long j = (long long)RC.y * 64 + cc;
      float p[NV];
#pragma unroll
      for (int v = 0; v < NV; v += 4) {
        const float4 x4 = *reinterpret_cast<const float4 *>(&xc[cc][v]);
        p[v] = ci[v] * x4.x;
        p[v + 1] = ci[v + 1] * x4.y;
        p[v + 2] = ci[v + 2] * x4.z;
        p[v + 3] = ci[v + 3] * x4.w;
      }
      if constexpr (IDENT) {
        if (i == j)
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[0][v] += p[v];
      } else {
        const uint64_t lo = (uint64_t)(i < j ? i : j), hi = (uint64_t)(i < j ? j : i);
        const uint64_t base = mix64(lo + kGolden * hi);
#pragma unroll
        for (int q = 0; q < KS; ++q) {  // operators past the launch's count are computed and dropped
          const float o = to_unit(mix64(mix64(base ^ kq[q]) ^ a.seed));
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[q][v] = fmaf(p[v], o, acc[q][v]);
        }
      }
    }
    __syncthreads();
  }
  // warp reduction (a warp's 32 threads share one slot), one f64 atomic per (v, k)
  const int lane = tid & 31;
#pragma unroll
  for (int q = 0; q < KS; ++q) {
    const int kl = kg + GK * q;
    if (!IDENT && kl >= a.kc) continue;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float s = acc[q][v];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && v < a.nv) {
        double *dst = a.accum + (long long)(a.v0 + v) * a.m_ops;
        if (IDENT)
          for (int k = 0; k < a.m_ops; ++k) atomicAdd(dst + k, (double)s);
        else
          atomicAdd(dst + a.k0 + kl, (double)s);
      }
    }
  }
}

// Small sparse tiles (the cim_sparse_tiles.small_tiles list — basis-built
// skeletons hold millions of tiles of a few dozen entries): staging two
// 64-row c blocks and 64 row masks per tile would cost more than the tile's
// pairs.  One warp per tile, lane per entry: c[i, ·] and c[j, ·] are read
// straight from global memory (L2-resident for these n), then the same
// per-pair work as contract_kernel into per-thread accumulators for KS
// operators.  The host loops over operator chunks of KS.
template <typename T, int NV, int KS, bool IDENT>
__global__ void __launch_bounds__(kCtSmallThreads) contract_small_kernel(ContractArgs<T> a, const int32_t *list, long long n_list) {
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  uint64_t kq[KS];
#pragma unroll
  for (int q = 0; q < KS; ++q) kq[q] = (uint64_t)(a.k0 + q + 1) * kMix1;
  float acc[KS][NV];
#pragma unroll
  for (int q = 0; q < KS; ++q)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[q][v] = 0.f;
  // 32 tiles' metadata per warp load round (lane = tile), broadcast by shuffles
  for (long long c0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; c0 < n_list; c0 += nw * 32) {
    long long my_base = 0;
    int my_cnt = 0;
    int2 my_rc = make_int2(0, 0);
    if (c0 + lane < n_list) {
      const long long u = __ldg(list + c0 + lane);
      my_base = __ldg(a.sp_off + u);
      my_cnt = __ldg(a.sp_rowptr + u * kSpPtrStride + 64);
      my_rc = __ldg(a.sp_rc + u);
    }
    // one stored entry (tile RC, entry index eidx) into the accumulators
    auto entry = [&](int2 RC, long long eidx) {
      if (__ldg(a.sp_vals + eidx) == T(0)) return;
      const long long i = (long long)RC.x * 64 + __ldg(a.sp_row + eidx);
      const long long j = (long long)RC.y * 64 + __ldg(a.sp_col + eidx);
      if (i >= a.n || j >= a.n) return;
      const float wgt = RC.x == RC.y ? 1.f : 2.f;
      float p[NV];
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const bool on = v < a.nv;
        const float ci = on ? __ldg(a.c + i * a.n_vec + a.v0 + v) : 0.f;
        const float cj = on ? __ldg(a.c + j * a.n_vec + a.v0 + v) : 0.f;
        p[v] = wgt * ci * cj;
      }
      if constexpr (IDENT) {
        if (i == j)
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[0][v] += p[v];
      } else {
        const uint64_t lo = (uint64_t)(i < j ? i : j), hi = (uint64_t)(i < j ? j : i);
        const uint64_t hb = mix64(lo + kGolden * hi);
#pragma unroll
        for (int q = 0; q < KS; ++q) {
          const float o = to_unit(mix64(mix64(hb ^ kq[q]) ^ a.seed));
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[q][v] = fmaf(p[v], o, acc[q][v]);
        }
      }
    };
    if (__all_sync(0xffffffffu, my_cnt <= 24)) {
      // tiny tiles: the chunk's entries as one flat range (as sparse_small_kernel)
      int my_end = my_cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, my_end, o);
        if (lane >= o) my_end += v;
      }
      const int total = __shfl_sync(0xffffffffu, my_end, 31);
      for (int f0 = 0; f0 < total; f0 += 32) {  // warp-uniform trip count for the shuffles
        const int f = f0 + lane;
        const int fq = f < total ? f : total - 1;
        int q = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1)
          if (__shfl_sync(0xffffffffu, my_end, q + step - 1) <= fq) q += step;
        const int end_q = __shfl_sync(0xffffffffu, my_end, q), cnt_q = __shfl_sync(0xffffffffu, my_cnt, q);
        const long long eidx = __shfl_sync(0xffffffffu, my_base, q) + (fq - (end_q - cnt_q));
        const int2 RC = make_int2(__shfl_sync(0xffffffffu, my_rc.x, q), __shfl_sync(0xffffffffu, my_rc.y, q));
        if (f < total) entry(RC, eidx);
      }
      continue;
    }
    const int n_here = (int)(n_list - c0 < 32 ? n_list - c0 : 32);
    for (int t = 0; t < n_here; ++t) {
      const int cnt = __shfl_sync(0xffffffffu, my_cnt, t);
      if (cnt == 0) continue;
      const long long base = __shfl_sync(0xffffffffu, my_base, t);
      const int2 RC = make_int2(__shfl_sync(0xffffffffu, my_rc.x, t), __shfl_sync(0xffffffffu, my_rc.y, t));
      for (int e = lane; e < cnt; e += 32) entry(RC, base + e);
    }
  }
#pragma unroll
  for (int q = 0; q < KS; ++q) {
    if (!IDENT && q >= a.kc) continue;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float s = acc[q][v];
#pragma unroll
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && v < a.nv) {
        double *dst = a.accum + (long long)(a.v0 + v) * a.m_ops;
        if (IDENT)
          for (int k = 0; k < a.m_ops; ++k) atomicAdd(dst + k, (double)s);
        else
          atomicAdd(dst + a.k0 + q, (double)s);
      }
    }
  }
}

template <typename T, int NV>
void launch_small_nv(const ContractArgs<T> &a, bool ident, const int32_t *list, long long n_list, int grid,
                     cudaStream_t s) {
  if (ident)
    contract_small_kernel<T, NV, 1, true><<<grid, kCtSmallThreads, 0, s>>>(a, list, n_list);
  else if (a.kc == 1)
    contract_small_kernel<T, NV, 1, false><<<grid, kCtSmallThreads, 0, s>>>(a, list, n_list);
  else if (a.kc <= 4)
    contract_small_kernel<T, NV, 4, false><<<grid, kCtSmallThreads, 0, s>>>(a, list, n_list);
  else
    contract_small_kernel<T, NV, 8, false><<<grid, kCtSmallThreads, 0, s>>>(a, list, n_list);
}

template <typename T, int NV>
void launch_nv(const ContractArgs<T> &a, bool ident, int grid, cudaStream_t s) {
  if (ident)
    contract_kernel<T, NV, 1, 1, true><<<grid, kCtThreads, 0, s>>>(a);
  else if (a.kc == 1)
    contract_kernel<T, NV, 1, 1, false><<<grid, kCtThreads, 0, s>>>(a);
  else if (a.kc == 2)
    contract_kernel<T, NV, 1, 2, false><<<grid, kCtThreads, 0, s>>>(a);
  else if (a.kc <= 4)
    contract_kernel<T, NV, 1, 4, false><<<grid, kCtThreads, 0, s>>>(a);
  else if (a.kc <= 8)
    contract_kernel<T, NV, 2, 4, false><<<grid, kCtThreads, 0, s>>>(a);
  else
    contract_kernel<T, NV, 4, 4, false><<<grid, kCtThreads, 0, s>>>(a);
}

template <typename T>
int run_contract(const cim_half_tiles *H, const float *c, int n_vec, int m_ops, int kind, uint64_t seed,
                 double *accum, cudaStream_t stream) {
  ContractArgs<T> a{};
  a.n = H->n;
  a.n_dense = H->n_tiles;
  a.rc = reinterpret_cast<const int2 *>(H->tile_rc);
  a.vals = static_cast<const T *>(H->vals);
  a.layout = H->layout;
  const cim_sparse_tiles *S = H->sparse;
  if (S && S->n_tiles > 0) {
    a.n_sparse = S->n_tiles;
    a.sp_rc = reinterpret_cast<const int2 *>(S->tile_rc);
    a.sp_off = reinterpret_cast<const long long *>(S->entry_off);
    a.sp_rowptr = S->rowptr;
    a.sp_col = S->col;
    a.sp_row = S->row;
    a.sp_vals = static_cast<const T *>(S->vals);
  }
  a.c = c;
  a.n_vec = n_vec;
  a.m_ops = m_ops;
  a.seed = seed;
  a.accum = accum;
  // the sparse split of cim_sparse_tiles: staged tiles through the mask
  // kernel, small ones entry-parallel (NULL lists: every tile in the mask kernel)
  const bool listed = S && S->n_tiles > 0 && (S->staged_tiles || S->small_tiles);
  const int32_t *small = listed ? S->small_tiles : nullptr;
  const long long n_small = (listed && S->small_tiles) ? S->n_small : 0;
  if (listed) {
    a.sp_list = S->staged_tiles;
    a.n_sparse = S->staged_tiles ? S->n_staged : 0;
  }
  const long long total = a.n_dense + a.n_sparse;
  if (total == 0 && n_small == 0) return CIM_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)(total < (long long)sms * 8 ? total : (long long)sms * 8);
  const int grid_small = (int)std::min<long long>((n_small + kCtSmallThreads - 1) / kCtSmallThreads,
                                                  (long long)sms * 32);  // 32 tiles per warp
  const bool ident = kind == CIM_VALUES_IDENTITY;
  if (n_small > 0) {
    constexpr int kSmallKs = 8;
    for (int v0 = 0; v0 < n_vec; v0 += 8) {
      a.v0 = v0;
      a.nv = n_vec - v0 < 8 ? n_vec - v0 : 8;
      for (int k0 = 0; k0 < (ident ? 1 : m_ops); k0 += kSmallKs) {
        a.k0 = k0;
        a.kc = m_ops - k0 < kSmallKs ? m_ops - k0 : kSmallKs;
        if (a.nv <= 4)
          launch_small_nv<T, 4>(a, ident, small, n_small, grid_small, stream);
        else
          launch_small_nv<T, 8>(a, ident, small, n_small, grid_small, stream);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess)
          return set_error(CIM_ECUDA, std::string("contract_small_kernel: ") + cudaGetErrorString(e));
      }
    }
  }
  if (total == 0) return CIM_OK;
  for (int v0 = 0; v0 < n_vec; v0 += 16) {
    a.v0 = v0;
    a.nv = n_vec - v0 < 16 ? n_vec - v0 : 16;
    for (int k0 = 0; k0 < (ident ? 1 : m_ops); k0 += 16) {
      a.k0 = k0;
      a.kc = m_ops - k0 < 16 ? m_ops - k0 : 16;
      if (a.nv <= 4)
        launch_nv<T, 4>(a, ident, grid, stream);
      else if (a.nv <= 8)
        launch_nv<T, 8>(a, ident, grid, stream);
      else
        launch_nv<T, 16>(a, ident, grid, stream);
      const cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("contract_kernel: ") + cudaGetErrorString(e));
    }
  }
  return CIM_OK;
}

}  // namespace
}  // namespace cim

extern "C" int cim_contract_observables(const cim_half_tiles *H, const float *c, int32_t n_vec, int32_t m_ops,
                                        int32_t kind, uint64_t seed, double *accum, uint32_t flags, void *stream_) {
  cim::clear_error();
  if (!H) return cim::set_error(CIM_EINVAL, "H is NULL");
  if (H->block != cim::kBlock) return cim::set_error(CIM_EINVAL, "block must be 64");
  if (H->n < 1) return cim::set_error(CIM_EINVAL, "n must be >= 1");
  if (H->dtype != CIM_F32 && H->dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (H->layout != CIM_LAYOUT_FRAG && H->layout != CIM_LAYOUT_TC) return cim::set_error(CIM_EINVAL, "unknown tile layout");
  if (n_vec < 1 || m_ops < 1) return cim::set_error(CIM_EINVAL, "n_vec and m_ops must be >= 1");
  if (kind != CIM_VALUES_OP_HASH && kind != CIM_VALUES_IDENTITY)
    return cim::set_error(CIM_EINVAL, "kind must be CIM_VALUES_OP_HASH or CIM_VALUES_IDENTITY");
  if (!c || !accum) return cim::set_error(CIM_EINVAL, "c and accum must be non-NULL");
  if (H->n_tiles > 0 && (!H->tile_rc || !H->vals)) return cim::set_error(CIM_EINVAL, "tile arrays are NULL");
  const cim_sparse_tiles *S = H->sparse;
  if (S && S->n_tiles > 0 &&
      (!S->tile_rc || !S->entry_off || !S->rowptr || (S->n_entries > 0 && (!S->col || !S->row || !S->vals))))
    return cim::set_error(CIM_EINVAL, "NULL sparse arrays");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream_);
  if (!(flags & CIM_ACCUMULATE)) {
    const cudaError_t e = cudaMemsetAsync(accum, 0, sizeof(double) * (size_t)n_vec * m_ops, s);
    if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("zeroing accum: ") + cudaGetErrorString(e));
  }
  if (H->dtype == CIM_F32) return cim::run_contract<float>(H, c, n_vec, m_ops, kind, seed, accum, s);
  return cim::run_contract<double>(H, c, n_vec, m_ops, kind, seed, accum, s);
}
