// Sparse ("COO-in-tile") stored tiles: the same operator, Y += U_s·X + U_s,offᵀ·X,
// for 64-tiles below the dense break-even fill (include/cim_b200.h,
// cim_sparse_tiles).  Reference skeletons are built from ragged orbital
// blocks (pipeline.py:290-377; sizes 1..100), so their 64-tiles are mostly
// sparse: streaming them as dense tiles would move 4096 values per tile for
// a few hundred entries.
//
// One warp per tile (persistent warps, global ticket counter), two passes,
// both register reductions — no atomics inside a tile (shared-memory f32
// atomicAdd is a CAS loop on sm_100; a first version built on it ran 4×
// slower than streaming the tiles dense):
//   * direct: lane ℓ owns local rows ℓ, ℓ+32 and walks their row-sorted
//     entries, acc += v·X_C[col]; one vector red.global per row;
//   * transposed (off-diagonal tiles): lane ℓ owns local columns ℓ, ℓ+32 and
//     walks them through the column permutation, acc += v·X_R[row]; one
//     vector red.global per column.
// X rows are read through L1 (a tile's entries hit one 64-row X block
// repeatedly).  k is processed in passes of KV vectors (8 f32 / 4 f64).
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace {

constexpr int kSpWarps = 4;  // warps per CTA

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
  const uint16_t *rowptr, *colptr;
  const uint8_t *col, *row;
  const uint16_t *cperm;
  const void *vals;
  const void *X;
  void *Y;
  unsigned int *counter;
  long long n_tiles;
  long long ldx, ldy;
  int k;
};

// Per-warp double-buffered shared staging: a tile's entry arrays (≤ kSpCap
// entries) and the X_C / X_R slices, filled with cp.async while the previous
// tile is being multiplied.
constexpr int kSpCap = 1024;

template <typename T, int KV>
struct SpStage {
  uint8_t col[kSpCap];
  uint8_t row[kSpCap];
  uint16_t cperm[kSpCap];
  alignas(16) T val[kSpCap];
  alignas(16) T xc[64 * KV];
  alignas(16) T xr[64 * KV];
};

__device__ __forceinline__ void cp16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

__device__ __forceinline__ void copy16_async(void *dst, const void *src, int bytes, int lane) {
  const char *s = static_cast<const char *>(src);
  char *d = static_cast<char *>(dst);
  for (int q = lane; q < bytes / 16; q += 32) cp16(d + 16 * q, s + 16 * q);
}

template <typename T, int KV>
__device__ __forceinline__ void lds_vec(T (&d)[KV], const T *p) {
  if constexpr (sizeof(T) == 4 && KV % 4 == 0) {
#pragma unroll
    for (int q = 0; q < KV / 4; ++q) {
      const float4 v = reinterpret_cast<const float4 *>(p)[q];
      d[4 * q] = v.x, d[4 * q + 1] = v.y, d[4 * q + 2] = v.z, d[4 * q + 3] = v.w;
    }
  } else if constexpr (sizeof(T) == 8 && KV % 2 == 0) {
#pragma unroll
    for (int q = 0; q < KV / 2; ++q) {
      const double2 v = reinterpret_cast<const double2 *>(p)[q];
      d[2 * q] = v.x, d[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < KV; ++q) d[q] = p[q];
  }
}

// One tile's header, held in registers: its lane's row/column pointer
// values (rows lane, lane+32, and 64), entry range, position.
struct SpHdr {
  int2 rc;
  long long base;
  int ne;             // padded entry count
  uint16_t r0, r1, r64, c0, c1, c64;
};

__device__ __forceinline__ SpHdr load_hdr(const SparseParams &p, long long t, int lane) {
  SpHdr h;
  h.rc = p.tile_rc[t];
  h.base = p.entry_off[t];
  h.ne = (int)(p.entry_off[t + 1] - h.base);
  const uint16_t *rp = p.rowptr + (size_t)t * 65, *cp = p.colptr + (size_t)t * 65;
  h.r0 = rp[lane], h.r1 = rp[lane + 32], h.r64 = rp[64];
  h.c0 = cp[lane], h.c1 = cp[lane + 32], h.c64 = cp[64];
  return h;
}

// Bounds of a lane's two rows (or columns) from the held pointer values.
__device__ __forceinline__ void bounds(int lane, int v0, int v1, int v64, int (&lo)[2], int (&hi)[2]) {
  const int n0 = __shfl_down_sync(0xffffffffu, v0, 1), n1 = __shfl_down_sync(0xffffffffu, v1, 1);
  const int b32 = __shfl_sync(0xffffffffu, v1, 0);
  lo[0] = v0, lo[1] = v1;
  hi[0] = lane < 31 ? n0 : b32;
  hi[1] = lane < 31 ? n1 : v64;
}

// X slices are staged for every staged tile (kSpStageX = 0): reading the
// few X rows of a sparse tile through L1 instead measured 2× slower at 2%
// fill (dependent global loads per entry); the threshold stays as a knob.
constexpr int kSpStageX = 0;

template <typename T, int KV>
__device__ __forceinline__ void issue_stage(SpStage<T, KV> &st, const SparseParams &p, const SpHdr &h, int v0,
                                            int lane) {
  const T *vals = static_cast<const T *>(p.vals);
  const T *X = static_cast<const T *>(p.X);
  // entries are re-staged for every vector pass (the other buffer holds them
  // only for the previous step)
  copy16_async(st.col, p.col + h.base, h.ne, lane);
  copy16_async(st.row, p.row + h.base, h.ne, lane);
  copy16_async(st.cperm, p.cperm + h.base, 2 * h.ne, lane);
  copy16_async(st.val, vals + h.base, h.ne * (int)sizeof(T), lane);
  if (h.ne < kSpStageX) return;
  constexpr int CPR = KV * (int)sizeof(T) / 16;  // 16-byte chunks per X row slice
  const T *xc = X + (long long)h.rc.y * 64 * p.ldx + v0;
  const T *xr = X + (long long)h.rc.x * 64 * p.ldx + v0;
  for (int q = lane; q < 64 * CPR; q += 32) {
    const int r = q / CPR, c = q % CPR;
    cp16(reinterpret_cast<char *>(st.xc) + 16 * q, reinterpret_cast<const char *>(xc + (long long)r * p.ldx) + 16 * c);
    if (h.rc.x != h.rc.y)
      cp16(reinterpret_cast<char *>(st.xr) + 16 * q,
           reinterpret_cast<const char *>(xr + (long long)r * p.ldx) + 16 * c);
  }
}

// Two register-reduction passes over one tile, operands in the stage
// (STAGED) or straight from global memory (tiles above kSpCap entries).
template <typename T, int KV, bool STAGED, bool XST>
__device__ __forceinline__ void tile_passes(int lane, const SpHdr &h, const SparseParams &p, const SpStage<T, KV> *st,
                                            int v0) {
  const bool diag = h.rc.x == h.rc.y;
  const T *X = static_cast<const T *>(p.X);
  T *Y = static_cast<T *>(p.Y);
  const uint8_t *col = STAGED ? st->col : p.col + h.base;
  const uint8_t *row = STAGED ? st->row : p.row + h.base;
  const uint16_t *cperm = STAGED ? st->cperm : p.cperm + h.base;
  const T *val = STAGED ? st->val : static_cast<const T *>(p.vals) + h.base;
  const T *xc = XST ? st->xc : X + (long long)h.rc.y * 64 * p.ldx + v0;
  const T *xr = XST ? st->xr : X + (long long)h.rc.x * 64 * p.ldx + v0;
  const long long xs = XST ? KV : p.ldx;
  int lo[2], hi[2];
  bounds(lane, h.r0, h.r1, h.r64, lo, hi);
  T *y_r = Y + (long long)h.rc.x * 64 * p.ldy + v0;
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {  // direct: rows lane, lane+32
    if (lo[k2] == hi[k2]) continue;
    T acc[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = T(0);
    int e = lo[k2];
    for (; e + 2 <= hi[k2]; e += 2) {  // two independent load chains per iteration
      const int c0 = col[e], c1 = col[e + 1];
      const T v0_ = val[e], v1_ = val[e + 1];
      T x0[KV], x1[KV];
      if constexpr (XST) {
        lds_vec<T, KV>(x0, xc + c0 * xs);
        lds_vec<T, KV>(x1, xc + c1 * xs);
      } else {
        ldg_vec<T, KV>(x0, xc + c0 * xs);
        ldg_vec<T, KV>(x1, xc + c1 * xs);
      }
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = fma(v1_, x1[q], fma(v0_, x0[q], acc[q]));
    }
    if (e < hi[k2]) {
      const int c = col[e];
      const T v = val[e];
      T x[KV];
      if constexpr (XST)
        lds_vec<T, KV>(x, xc + c * xs);
      else
        ldg_vec<T, KV>(x, xc + c * xs);
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = fma(v, x[q], acc[q]);
    }
    red_vec<T, KV>(y_r + (long long)(lane + 32 * k2) * p.ldy, acc);
  }
  if (diag) return;
  bounds(lane, h.c0, h.c1, h.c64, lo, hi);
  T *y_c = Y + (long long)h.rc.y * 64 * p.ldy + v0;
#pragma unroll
  for (int k2 = 0; k2 < 2; ++k2) {  // transposed: columns lane, lane+32
    if (lo[k2] == hi[k2]) continue;
    T acc[KV];
#pragma unroll
    for (int q = 0; q < KV; ++q) acc[q] = T(0);
    int qi = lo[k2];
    for (; qi + 2 <= hi[k2]; qi += 2) {
      const int e0 = cperm[qi], e1 = cperm[qi + 1];
      const int r0 = row[e0], r1 = row[e1];
      const T v0_ = val[e0], v1_ = val[e1];
      T x0[KV], x1[KV];
      if constexpr (XST) {
        lds_vec<T, KV>(x0, xr + r0 * xs);
        lds_vec<T, KV>(x1, xr + r1 * xs);
      } else {
        ldg_vec<T, KV>(x0, xr + r0 * xs);
        ldg_vec<T, KV>(x1, xr + r1 * xs);
      }
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = fma(v1_, x1[q], fma(v0_, x0[q], acc[q]));
    }
    if (qi < hi[k2]) {
      const int e = cperm[qi];
      const int r = row[e];
      const T v = val[e];
      T x[KV];
      if constexpr (XST)
        lds_vec<T, KV>(x, xr + r * xs);
      else
        ldg_vec<T, KV>(x, xr + r * xs);
#pragma unroll
      for (int q = 0; q < KV; ++q) acc[q] = fma(v, x[q], acc[q]);
    }
    red_vec<T, KV>(y_c + (long long)(lane + 32 * k2) * p.ldy, acc);
  }
}

// Static contiguous tile chunks per warp; software pipeline: the header of
// tile i+1 and its staged operands load while tile i is multiplied.
template <typename T, int KV>
__global__ void __launch_bounds__(kSpWarps * 32) sparse_spmm_kernel(const SparseParams p) {
  extern __shared__ __align__(16) unsigned char sp_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SpStage<T, KV> *stage = reinterpret_cast<SpStage<T, KV> *>(sp_smem) + 2 * w;
  const long long gw = (long long)blockIdx.x * kSpWarps + w, nw = (long long)gridDim.x * kSpWarps;
  const long long t_lo = p.n_tiles * gw / nw, t_hi = p.n_tiles * (gw + 1) / nw;
  if (t_lo >= t_hi) return;
  const int npass = (p.k + KV - 1) / KV;
  // X slices stage in 16-byte chunks: narrower passes read X through L1
  constexpr bool kStageable = (KV * sizeof(T)) % 16 == 0;
  // flattened (tile, pass) steps; step s → tile t_lo + s / npass, pass s % npass
  const long long nsteps = (t_hi - t_lo) * npass;
  SpHdr cur = load_hdr(p, t_lo, lane);
  bool cur_staged = kStageable && cur.ne <= kSpCap && (p.ldx * (long long)sizeof(T)) % 16 == 0;
  if constexpr (kStageable)
    if (cur_staged) issue_stage<T, KV>(stage[0], p, cur, 0, lane);
  cp_commit();
  for (long long s = 0; s < nsteps; ++s) {
    const long long t = t_lo + s / npass;
    const int v0 = (int)(s % npass) * KV;
    // prefetch the next step (same tile next pass, or the next tile)
    SpHdr nxt = cur;
    bool nxt_staged = false;
    if (s + 1 < nsteps) {
      const long long tn = t_lo + (s + 1) / npass;
      if (tn != t) nxt = load_hdr(p, tn, lane);
      nxt_staged = kStageable && nxt.ne <= kSpCap && (p.ldx * (long long)sizeof(T)) % 16 == 0;
      __syncwarp();  // everyone is done with the buffer being refilled (step s-1's)
      if constexpr (kStageable)
        if (nxt_staged) issue_stage<T, KV>(stage[(s + 1) & 1], p, nxt, (int)((s + 1) % npass) * KV, lane);
    }
    cp_commit();
    cp_wait1();  // this step's stage has landed (this lane's copies) ...
    __syncwarp();  // ... and everyone's
    if (kStageable && cur_staged) {
      if (cur.ne >= kSpStageX)
        tile_passes<T, KV, true, true>(lane, cur, p, &stage[s & 1], v0);
      else
        tile_passes<T, KV, true, false>(lane, cur, p, &stage[s & 1], v0);
    } else {
      tile_passes<T, KV, false, false>(lane, cur, p, nullptr, v0);
    }
    cur = nxt;
    cur_staged = nxt_staged;
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
  SparseParams p;
  p.tile_rc = reinterpret_cast<const int2 *>(S->tile_rc);
  p.entry_off = reinterpret_cast<const long long *>(S->entry_off);
  p.rowptr = S->rowptr;
  p.colptr = S->colptr;
  p.col = S->col;
  p.row = S->row;
  p.cperm = S->cperm;
  p.vals = S->vals;
  p.X = X;
  p.Y = Y;
  p.counter = nullptr;
  p.n_tiles = S->n_tiles;
  p.ldx = ldx;
  p.ldy = ldy;
  p.k = k;
  const size_t smem = 2 * kSpWarps * sizeof(SpStage<T, KV>);
  static std::once_flag attr_once;
  std::call_once(attr_once, [&] {
    cudaFuncSetAttribute(sparse_spmm_kernel<T, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sparse_spmm_kernel<T, KV>, kSpWarps * 32, smem) != cudaSuccess ||
      occ < 1)
    occ = 1;
  const long long warps = std::min<long long>(S->n_tiles, (long long)st->sms * occ * kSpWarps);
  const unsigned grid = (unsigned)((warps + kSpWarps - 1) / kSpWarps);
  sparse_spmm_kernel<T, KV><<<grid, kSpWarps * 32, smem, stream>>>(p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse_spmm launch: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace

// Called by cim_sym_spmm after the dense tiles (Y already zeroed or accumulating).
int sym_spmm_sparse(const cim_sparse_tiles *S, int dtype, const void *X, void *Y, int k, long long ldx,
                    long long ldy, cudaStream_t stream) {
  if (!S || S->n_tiles == 0) return CIM_OK;
  if (!S->tile_rc || !S->entry_off || !S->rowptr || !S->colptr ||
      (S->n_entries > 0 && (!S->col || !S->row || !S->cperm || !S->vals)))
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

// ---------------------------------------------------------------------------
// Device construction of synthetic sparse tiles — the reference's
// count → scan → fill motif (build_skeleton: count_pairs, counts_to_offsets,
// fill_rows; pipeline.py:290-377) on the GPU:
//   1. cim_sparse_count_rows: per (tile, local row) the number of kept
//      entries, kept(i, j) ⇔ mix64(mix64(min ⊕ 0x5bd1e995·max) ⊕ seed) < fill·2⁶⁴
//      (symmetric in i, j, so diagonal tiles stay symmetric);
//   2. the caller scans the counts (rowptr per tile, entry_off over tiles);
//   3. cim_sparse_fill_entries writes columns (row-sorted) and values
//      value_of_kind(i, j) — h(i XOR j; seed) by default, bit-exact to the
//      reference hash.
// ---------------------------------------------------------------------------
namespace cim {
namespace {

__device__ __forceinline__ bool keep_entry(uint64_t i, uint64_t j, uint64_t thresh, uint64_t seed) {
  const uint64_t lo = i < j ? i : j, hi = i < j ? j : i;
  return mix64(mix64(lo ^ (hi * 0x5bd1e995ull)) ^ seed) < thresh;
}

__global__ void sparse_count_rows_kernel(const int2 *tile_rc, long long n_tiles, long long n, uint64_t thresh,
                                         uint64_t seed, int32_t *rowcnt) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_tiles * 64) return;
  const long long t = g >> 6;
  const int r = (int)(g & 63);
  const int2 rc = tile_rc[t];
  const uint64_t i = (uint64_t)rc.x * 64 + r;
  int cnt = 0;
  if (i < (uint64_t)n) {
    for (int c = 0; c < 64; ++c) {
      const uint64_t j = (uint64_t)rc.y * 64 + c;
      if (j < (uint64_t)n && keep_entry(i, j, thresh, seed)) ++cnt;
    }
  }
  rowcnt[g] = cnt;
}

template <typename T>
__global__ void sparse_fill_entries_kernel(const int2 *tile_rc, const long long *entry_off, const uint16_t *rowptr,
                                           long long n_tiles, long long n, uint64_t thresh, uint64_t seed, int kind,
                                           uint64_t value_seed, int op_k, uint8_t *col, uint8_t *rowi, T *vals) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_tiles * 64) return;
  const long long t = g >> 6;
  const int r = (int)(g & 63);
  const int2 rc = tile_rc[t];
  const uint64_t i = (uint64_t)rc.x * 64 + r;
  long long e = entry_off[t] + rowptr[t * 65 + r];
  if (i >= (uint64_t)n) return;
  for (int c = 0; c < 64; ++c) {
    const uint64_t j = (uint64_t)rc.y * 64 + c;
    if (j < (uint64_t)n && keep_entry(i, j, thresh, seed)) {
      col[e] = (uint8_t)c;
      rowi[e] = (uint8_t)r;
      vals[e] = (T)value_of_kind(kind, i, j, value_seed, op_k);
      ++e;
    }
  }
}

uint64_t fill_threshold(double fill) {
  if (fill >= 1.0) return ~0ull;
  if (fill <= 0.0) return 0ull;
  return (uint64_t)(fill * 18446744073709551616.0);
}

}  // namespace
}  // namespace cim

extern "C" int cim_sparse_count_rows(const int32_t *tile_rc, int64_t n_tiles, int64_t n, double fill, uint64_t seed,
                                     int32_t *rowcnt, void *stream_) {
  cim::clear_error();
  if (n_tiles < 0 || n < 1 || !(fill >= 0.0 && fill <= 1.0)) return cim::set_error(CIM_EINVAL, "bad arguments");
  if (n_tiles == 0) return CIM_OK;
  if (!tile_rc || !rowcnt) return cim::set_error(CIM_EINVAL, "NULL arrays");
  const long long threads = n_tiles * 64;
  cim::sparse_count_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream_)>>>(
      reinterpret_cast<const int2 *>(tile_rc), n_tiles, n, cim::fill_threshold(fill), seed, rowcnt);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("sparse_count_rows: ") + cudaGetErrorString(e));
  return CIM_OK;
}

extern "C" int cim_sparse_fill_entries(const cim_sparse_tiles *S, int64_t n, int32_t dtype, double fill, uint64_t seed,
                                       int32_t kind, uint64_t value_seed, int32_t op_k, void *stream_) {
  cim::clear_error();
  if (!S || n < 1 || !(fill >= 0.0 && fill <= 1.0)) return cim::set_error(CIM_EINVAL, "bad arguments");
  if (dtype != CIM_F32 && dtype != CIM_F64) return cim::set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (kind < 0 || kind > 2) return cim::set_error(CIM_EINVAL, "unknown value kind");
  if (S->n_tiles == 0) return CIM_OK;
  if (!S->tile_rc || !S->entry_off || !S->rowptr || (S->n_entries > 0 && (!S->col || !S->vals)))
    return cim::set_error(CIM_EINVAL, "NULL arrays");
  const long long threads = S->n_tiles * 64;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  const int2 *rc = reinterpret_cast<const int2 *>(S->tile_rc);
  const long long *off = reinterpret_cast<const long long *>(S->entry_off);
  uint8_t *col = const_cast<uint8_t *>(S->col);
  uint8_t *rowi = const_cast<uint8_t *>(S->row);
  if (S->n_entries > 0 && !rowi) return cim::set_error(CIM_EINVAL, "NULL row array");
  if (dtype == CIM_F32)
    cim::sparse_fill_entries_kernel<float><<<grid, 256, 0, stream>>>(rc, off, S->rowptr, S->n_tiles, n,
                                                                     cim::fill_threshold(fill), seed, kind, value_seed,
                                                                     op_k, col, rowi, static_cast<float *>(const_cast<void *>(S->vals)));
  else
    cim::sparse_fill_entries_kernel<double><<<grid, 256, 0, stream>>>(rc, off, S->rowptr, S->n_tiles, n,
                                                                      cim::fill_threshold(fill), seed, kind, value_seed,
                                                                      op_k, col, rowi, static_cast<double *>(const_cast<void *>(S->vals)));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("sparse_fill_entries: ") + cudaGetErrorString(e));
  return CIM_OK;
}

// Column index of row-sorted sparse tiles (warp per tile): lane ℓ counts the
// entries of columns ℓ and ℓ+32, a warp scan gives colptr, then the lanes
// fill cperm with tile-relative entry indices in row order.
namespace cim {
namespace {

__global__ void sparse_build_columns_kernel(const long long *entry_off, const uint16_t *rowptr, const uint8_t *col,
                                            long long n_tiles, uint16_t *colptr, uint16_t *cperm) {
  const int lane = threadIdx.x & 31;
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long t = warp; t < n_tiles; t += nwarps) {
    const long long base = entry_off[t];
    const uint16_t *rp = rowptr + (size_t)t * 65;
    const uint8_t *cl = col + base;
    int cnt[2] = {0, 0};
    for (int r = 0; r < 64; ++r) {  // count: lane owns columns lane, lane+32
      const int e0 = rp[r], e1 = rp[r + 1];
      for (int e = e0; e < e1; ++e) {
        const int c = cl[e];
        if ((c & 31) == lane) ++cnt[c >> 5];
      }
    }
    // exclusive scan over the 64 columns (lane-major: c = lane, then lane+32)
    int incl0 = cnt[0];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl0, d);
      if (lane >= d) incl0 += y;
    }
    const int tot0 = __shfl_sync(0xffffffffu, incl0, 31);
    int incl1 = cnt[1];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl1, d);
      if (lane >= d) incl1 += y;
    }
    int pos[2] = {incl0 - cnt[0], tot0 + incl1 - cnt[1]};
    uint16_t *cpt = colptr + (size_t)t * 65;
    cpt[lane + 1] = (uint16_t)(pos[0] + cnt[0]);
    cpt[lane + 33] = (uint16_t)(pos[1] + cnt[1]);
    if (lane == 0) cpt[0] = 0;
    for (int r = 0; r < 64; ++r) {  // fill in row order
      const int e0 = rp[r], e1 = rp[r + 1];
      for (int e = e0; e < e1; ++e) {
        const int c = cl[e];
        if ((c & 31) == lane) cperm[base + pos[c >> 5]++] = (uint16_t)e;
      }
    }
  }
}

}  // namespace
}  // namespace cim

extern "C" int cim_sparse_build_columns(const cim_sparse_tiles *S, void *stream_) {
  cim::clear_error();
  if (!S) return cim::set_error(CIM_EINVAL, "S is NULL");
  if (S->n_tiles == 0) return CIM_OK;
  if (!S->entry_off || !S->rowptr || !S->colptr || (S->n_entries > 0 && (!S->col || !S->cperm)))
    return cim::set_error(CIM_EINVAL, "NULL arrays");
  const unsigned grid = (unsigned)std::min<long long>((S->n_tiles + 7) / 8, 8192);
  cim::sparse_build_columns_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream_)>>>(
      reinterpret_cast<const long long *>(S->entry_off), S->rowptr, S->col, S->n_tiles,
      const_cast<uint16_t *>(S->colptr), const_cast<uint16_t *>(S->cperm));
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cim::set_error(CIM_ECUDA, std::string("sparse_build_columns: ") + cudaGetErrorString(e));
  return CIM_OK;
}
