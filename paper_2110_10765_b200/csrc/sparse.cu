// Sparse ("COO-in-tile") stored tiles: the same operator, Y += U_s·X + U_s,offᵀ·X,
// for 64-tiles below the dense break-even fill (include/cim_b200.h,
// cim_sparse_tiles).  Reference skeletons are built from ragged orbital
// blocks (pipeline.py:290-377; sizes 1..100), so their 64-tiles are mostly
// sparse: streaming them as dense tiles would move 4096 values per tile for
// a few hundred entries.
//
// Ring design (v5, the dense kernel's structure with variable-size stages):
// a producer warp bulk-copies each tile's pointers, entry arrays and X_C /
// X_R blocks into shared memory; 128 consumer threads (local row / column r,
// vector half h) then run both products as register reductions —
//   * direct: thread r walks row r's row-sorted entries, acc += v·X_C[col];
//   * transposed (off-diagonal tiles): thread r walks column r through the
//     column permutation, acc += v·X_R[row];
// one vector red.global per row / column and vector half.  No atomics inside
// a tile (shared-memory f32 atomicAdd is a CAS loop on sm_100; a first
// version built on it ran 4× slower than streaming the tiles dense).
// Tiles of at most cim_sparse_small_max() padded entries skip the ring and go
// to sparse_small_kernel (entry-parallel, straight from global memory); the
// split is the staged_tiles / small_tiles lists of cim_sparse_tiles.
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "common.cuh"
#include "counter_ring.h"
#include "host_util.h"

namespace cim {
namespace {


template <typename T, int KV>
__device__ __forceinline__ void ldg_vec(T (&d)[KV], const T *p) {
  if constexpr (sizeof(T) * KV == 32) {  // one 256-bit gather (LDG.E.ENL2.256, sm_100)
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
  int small_max;  // tiles with ≤ small_max (padded) entries go to sparse_small_kernel
  int cap;        // staged entries per stage (kSpCap or kSpCapSmall)
  const int32_t *staged;  // optional list of the staged tiles (else scan all, skipping small ones)
  long long n_staged;
};

// ---------------------------------------------------------------------------
// Kernel v5: the dense kernel's producer / consumer ring with variable-size
// stages.  A producer warp takes tiles from a ticket counter and bulk-copies
// (cp.async.bulk, mbarrier complete_tx) each tile's row / column pointers,
// entry arrays and X_C / X_R blocks into a ring of shared-memory stages; the
// 4 consumer warps (128 threads: local row / column r, vector half h) walk
// the tile from shared memory.  Tiles above kSpCap entries are flagged and
// walked from global memory instead.
// ---------------------------------------------------------------------------
// Staged entries per tile: 1024, or 512 when every staged tile fits (the
// storage says so in cim_sparse_tiles.staged_max_entries): 8.4 KB stages
// instead of 12.3 KB let three CTAs share an SM instead of two (5%-fill
// tiles 1.32 → 1.15 ms); larger tiles go through the global-memory path.
constexpr int kSpCap = 1024;
constexpr int kSpCapSmall = 512;
constexpr int kSpSmallDefault = 128;
constexpr int kSpConsumers = 128;
constexpr unsigned kSpBig = 1u, kSpTerm = 2u, kSpSkew = 4u;
constexpr int kSpSkewMin = 256;
constexpr int kSpFlatMax = 24;  // small-tile chunks whose tiles all hold ≤ this many entries walk one flat entry range  // tiles above this many (padded) entries stage X in skewed chunks

struct SpStageHdr {
  int R, C, ne;
  unsigned flags;
  long long t;  // tile index (global fallback)
  long long pad;
};

// X_C / X_R blocks are staged as kXChunks copies of 64/kXChunks rows, chunk q
// shifted by q·kXSkew bytes: lanes gathering random rows then spread over
// more banks (ncu: 44% of the shared-load wavefronts were bank conflicts
// with one contiguous 2 KB copy).  Row c lives at c·k + (c / rows-per-chunk)·skew.
#ifdef CIM_SP_NO_SKEW
constexpr int kXChunks = 1, kXSkew = 0;
#else
constexpr int kXChunks = 4, kXSkew = 16;
#endif

struct SpLayout {  // byte offsets inside one stage
  unsigned rp, cp, col, row, cperm, val, xc, xr, bytes;
};

__host__ __device__ __forceinline__ SpLayout sp_layout(int k, int es, int cap) {
  SpLayout L;
  L.rp = 32;
  L.cp = L.rp + 2 * kSpPtrStride;
  L.col = L.cp + 2 * kSpPtrStride;
  L.row = L.col + cap;
  L.cperm = L.row + cap;
  L.val = L.cperm + 2 * cap;
  L.xc = L.val + cap * es;
  L.xr = L.xc + 64 * k * es + kXChunks * kXSkew;
  L.bytes = (L.xr + 64 * k * es + kXChunks * kXSkew + 127) & ~127u;
  return L;
}

template <bool GLOBAL, typename U>
__device__ __forceinline__ U ld1(const U *p) {
  if constexpr (GLOBAL)
    return __ldg(p);
  else
    return *p;
}

template <bool GLOBAL, typename T, int KV>
__device__ __forceinline__ void ldx(T (&d)[KV], const T *p) {
  if constexpr (GLOBAL) {
    ldg_vec<T, KV>(d, p);
  } else if constexpr (sizeof(T) == 4 && KV % 4 == 0) {
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

// One tile, both products, by one warp: lane owns local rows / columns
// lane and lane+32 and KV vectors per pass (k in passes of KV).
template <bool GLOBAL, typename T, int KV>
__device__ __forceinline__ void sp_tile(int lane, int R, int C, const uint16_t *rp, const uint16_t *cp,
                                        const uint8_t *col, const uint8_t *row, const uint16_t *cperm,
                                        const T *val, const T *xc, const T *xr, int k, T *Y, long long ldy,
                                        int skew = 0) {  // skew: elements added per 64/kXChunks rows of X
  const bool diag = R == C;
#pragma unroll
  for (int hh = 0; hh < 2; ++hh) {
    const int r = lane + 32 * hh;
    const int e0 = ld1<GLOBAL>(rp + r), e1 = ld1<GLOBAL>(rp + r + 1);
    const int q0 = diag ? 0 : ld1<GLOBAL>(cp + r), q1 = diag ? 0 : ld1<GLOBAL>(cp + r + 1);
    for (int v0 = 0; v0 < k; v0 += KV) {
      if (e1 > e0) {  // direct: row r
        T acc[KV];
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = T(0);
        for (int e = e0; e < e1; ++e) {
          const int c = ld1<GLOBAL>(col + e);
          const T w = ld1<GLOBAL>(val + e);
          T x[KV];
          ldx<GLOBAL, T, KV>(x, xc + (long long)c * k + (GLOBAL ? 0 : (c / (64 / kXChunks)) * skew) + v0);
#pragma unroll
          for (int q = 0; q < KV; ++q) acc[q] = fma(w, x[q], acc[q]);
        }
        red_vec<T, KV>(Y + ((long long)R * 64 + r) * ldy + v0, acc);
      }
      if (q1 > q0) {  // transposed: column r
        T acc[KV];
#pragma unroll
        for (int q = 0; q < KV; ++q) acc[q] = T(0);
        for (int qi = q0; qi < q1; ++qi) {
          const int e = ld1<GLOBAL>(cperm + qi);
          const int rr = ld1<GLOBAL>(row + e);
          const T w = ld1<GLOBAL>(val + e);
          T x[KV];
          ldx<GLOBAL, T, KV>(x, xr + (long long)rr * k + (GLOBAL ? 0 : (rr / (64 / kXChunks)) * skew) + v0);
#pragma unroll
          for (int q = 0; q < KV; ++q) acc[q] = fma(w, x[q], acc[q]);
        }
        red_vec<T, KV>(Y + ((long long)C * 64 + r) * ldy + v0, acc);
      }
    }
  }
}

template <typename T, int KV>
__global__ void __launch_bounds__(kSpConsumers + 32) sparse_spmm_kernel(const SparseParams p, int S) {
  extern __shared__ __align__(128) unsigned char sp_smem[];
  const SpLayout L = sp_layout(p.k, (int)sizeof(T), p.cap);
  uint64_t *full = reinterpret_cast<uint64_t *>(sp_smem + (size_t)S * L.bytes);
  uint64_t *empty = full + S;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // one consumer warp per stage
    }
    fence_mbar_init();
  }
  __syncthreads();
  const T *X = static_cast<const T *>(p.X);
  T *Y = static_cast<T *>(p.Y);
  const T *vals = static_cast<const T *>(p.vals);
  const unsigned xblk = 64u * (unsigned)p.k * (unsigned)sizeof(T);

  if (tid >= kSpConsumers) {
    // ======================= producer warp =======================
    // Tickets are chunks of 32 tiles: the whole warp loads a chunk's headers
    // at once (one memory latency per 32 tiles), lane 0 then streams them.
    const int lane = tid & 31;
    const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    unsigned int t0 = 0;
    const long long n_items = p.staged ? p.n_staged : p.n_tiles;
    if (lane == 0) t0 = atomicAdd(p.counter, 32u);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    while ((long long)t0 < n_items) {
      unsigned int t_next = 0;
      if (lane == 0) t_next = atomicAdd(p.counter, 32u);  // prefetch the next chunk's ticket
      const long long it = (long long)t0 + lane;
      const bool valid = it < n_items;
      const long long t = valid ? (p.staged ? (long long)__ldg(p.staged + it) : it) : 0;
      const int2 my_rc = valid ? p.tile_rc[t] : make_int2(0, 0);
      const long long my_b = valid ? p.entry_off[t] : 0, my_e = valid ? p.entry_off[t + 1] : 0;
      const int cnt = (int)min(32LL, n_items - (long long)t0);
      for (int q = 0; q < cnt; ++q) {
        const int R = __shfl_sync(0xffffffffu, my_rc.x, q), C = __shfl_sync(0xffffffffu, my_rc.y, q);
        const long long base = __shfl_sync(0xffffffffu, my_b, q);
        const int ne = (int)(__shfl_sync(0xffffffffu, my_e, q) - base);
        const long long tt = __shfl_sync(0xffffffffu, t, q);
        if (!p.staged && ne <= p.small_max) continue;  // empty, or walked by sparse_small_kernel (warp-uniform)
        if (lane == 0) {
          mbar_wait_backoff(&empty[stage], phase ^ 1u);
          unsigned char *st = sp_smem + (size_t)stage * L.bytes;
          SpStageHdr *h = reinterpret_cast<SpStageHdr *>(st);
          const bool diag = R == C, big = ne > p.cap;
          h->R = R;
          h->C = C;
          h->ne = ne;
          const bool skew = ne > kSpSkewMin;  // denser tiles: more random X rows per tile, spread the banks
          h->flags = big ? kSpBig : (skew ? kSpSkew : 0u);
          h->t = tt;
          if (big) {
            mbar_arrive(&full[stage]);
          } else {
            const unsigned bytes = 4u * kSpPtrStride + 4u * (unsigned)ne + (unsigned)(ne * (int)sizeof(T)) + xblk +
                                   (diag ? 0u : xblk);
            mbar_arrive_expect_tx(&full[stage], bytes);
            bulk_g2s(st + L.rp, p.rowptr + (size_t)tt * kSpPtrStride, 2 * kSpPtrStride, &full[stage], pol_stream);
            bulk_g2s(st + L.cp, p.colptr + (size_t)tt * kSpPtrStride, 2 * kSpPtrStride, &full[stage], pol_stream);
            if (ne > 0) {
              bulk_g2s(st + L.col, p.col + base, ne, &full[stage], pol_stream);
              bulk_g2s(st + L.row, p.row + base, ne, &full[stage], pol_stream);
              bulk_g2s(st + L.cperm, p.cperm + base, 2 * ne, &full[stage], pol_stream);
              bulk_g2s(st + L.val, vals + base, ne * (int)sizeof(T), &full[stage], pol_stream);
            }
            if (skew) {
              const unsigned xch = xblk / kXChunks;
              for (int q = 0; q < kXChunks; ++q) {
                bulk_g2s(st + L.xc + q * (xch + kXSkew), X + ((long long)C * 64 + q * (64 / kXChunks)) * p.k, xch,
                         &full[stage], pol_keep);
                if (!diag)
                  bulk_g2s(st + L.xr + q * (xch + kXSkew), X + ((long long)R * 64 + q * (64 / kXChunks)) * p.k, xch,
                           &full[stage], pol_keep);
              }
            } else {
              bulk_g2s(st + L.xc, X + (long long)C * 64 * p.k, xblk, &full[stage], pol_keep);
              if (!diag) bulk_g2s(st + L.xr, X + (long long)R * 64 * p.k, xblk, &full[stage], pol_keep);
            }
          }
        }
        __syncwarp();
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
      t0 = __shfl_sync(0xffffffffu, t_next, 0);
    }
    if (lane == 0)  // one terminator per consumer warp (stage s belongs to warp s % 4)
      for (int q = 0; q < kSpConsumers / 32; ++q) {
        mbar_wait_backoff(&empty[stage], phase ^ 1u);
        reinterpret_cast<SpStageHdr *>(sp_smem + (size_t)stage * L.bytes)->flags = kSpTerm;
        mbar_arrive(&full[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    return;
  }

  // ======================= consumer warps =======================
  // warp w consumes stages w, w+4, w+8, ... (S is a multiple of 4): four
  // tiles in flight per CTA, one per warp.
  const int w = tid >> 5, lane = tid & 31;
  constexpr int NW = kSpConsumers / 32;
  int stage = w;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(&full[stage], phase);
    const unsigned char *st = sp_smem + (size_t)stage * L.bytes;
    const SpStageHdr h = *reinterpret_cast<const SpStageHdr *>(st);
    if (h.flags & kSpTerm) break;
    if (h.flags & kSpBig) {
      const long long t = h.t, base = p.entry_off[t];
      sp_tile<true, T, KV>(lane, h.R, h.C, p.rowptr + (size_t)t * kSpPtrStride, p.colptr + (size_t)t * kSpPtrStride,
                           p.col + base, p.row + base, p.cperm + base, vals + base, X + (long long)h.C * 64 * p.k,
                           X + (long long)h.R * 64 * p.k, p.k, Y, p.ldy);
    } else {
      sp_tile<false, T, KV>(lane, h.R, h.C, reinterpret_cast<const uint16_t *>(st + L.rp),
                            reinterpret_cast<const uint16_t *>(st + L.cp), st + L.col, st + L.row,
                            reinterpret_cast<const uint16_t *>(st + L.cperm), reinterpret_cast<const T *>(st + L.val),
                            reinterpret_cast<const T *>(st + L.xc), reinterpret_cast<const T *>(st + L.xr), p.k, Y,
                            p.ldy, (h.flags & kSpSkew) ? kXSkew / (int)sizeof(T) : 0);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    stage += NW;
    if (stage >= S) {
      stage -= S;
      phase ^= 1u;
    }
  }
}

// Small tiles (≤ small_max entries, typically a few dozen): staging them
// through the ring costs the producer ~8 bulk copies and two 2 KB X blocks
// per tile for a few dozen entries, so the producer lane becomes the
// bottleneck on skeletons with millions of such tiles.  Here one warp takes
// one tile straight from global memory, entry-parallel: lane e reads entry e
// (row, col, value — coalesced), gathers X_C[col] and X_R[row] from L2 and
// adds v·X_C[col] into Y_R[row] and v·X_R[row] into Y_C[col] with vector
// reds.  One dependent load level instead of rowptr → entries → X, and every
// lane busy; rows of a tiny tile rarely repeat, so per-entry reds cost about
// what per-row reductions would.  Grid-stride over the small-tile list.
template <typename T, int KV>
__global__ void __launch_bounds__(256) sparse_small_kernel(const SparseParams p, const int32_t *list,
                                                             long long n_list) {
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const T *X = static_cast<const T *>(p.X);
  T *Y = static_cast<T *>(p.Y);
  const T *vals = static_cast<const T *>(p.vals);
  const long long n_items = list ? n_list : p.n_tiles;
  // Chunks of 32 tiles per warp: lane l fetches tile l's metadata (list
  // entry, entry offset, count, (R, C)) in one round of loads, then the warp
  // walks the chunk's tiles with the metadata broadcast by shuffles — one
  // dependent load level per tile (entries → X) instead of four.
  for (long long c0 = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; c0 < n_items; c0 += nw * 32) {
    const long long it = c0 + lane;
    long long my_base = 0;
    int my_cnt = 0;
    int2 my_rc = make_int2(0, 0);
    if (it < n_items) {
      const long long t = list ? (long long)__ldg(list + it) : it;
      my_base = __ldg(p.entry_off + t);
      bool take = true;
      if (!list) {
        const int ne = (int)(__ldg(p.entry_off + t + 1) - my_base);
        take = ne > 0 && ne <= p.small_max;
      }
      if (take) {
        my_cnt = __ldg(p.rowptr + (size_t)t * kSpPtrStride + 64);
        my_rc = __ldg(p.tile_rc + t);
      }
    }
    if (__all_sync(0xffffffffu, my_cnt <= kSpFlatMax)) {
      // the chunk's entries as one flat range (inclusive scan of the counts),
      // lanes striding over it — a warp stays busy however small the tiles
      int my_end = my_cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, my_end, o);
        if (lane >= o) my_end += v;
      }
      const int total = __shfl_sync(0xffffffffu, my_end, 31);
      for (int f0 = 0; f0 < total; f0 += 32) {  // warp-uniform trip count: the shuffles need every lane
        const int f = f0 + lane;
        const bool on = f < total;
        const int fq = on ? f : total - 1;
        int q = 0;  // first tile whose inclusive end exceeds fq
#pragma unroll
        for (int step = 16; step; step >>= 1)
          if (__shfl_sync(0xffffffffu, my_end, q + step - 1) <= fq) q += step;
        const int end_q = __shfl_sync(0xffffffffu, my_end, q), cnt_q = __shfl_sync(0xffffffffu, my_cnt, q);
        const long long base = __shfl_sync(0xffffffffu, my_base, q) + (fq - (end_q - cnt_q));
        const int R = __shfl_sync(0xffffffffu, my_rc.x, q), C = __shfl_sync(0xffffffffu, my_rc.y, q);
        if (!on) continue;
        const T *xr = X + (long long)R * 64 * p.k, *xc = X + (long long)C * 64 * p.k;
        T *yr = Y + (long long)R * 64 * p.ldy, *yc = Y + (long long)C * 64 * p.ldy;
        const int c = __ldg(p.col + base), r = __ldg(p.row + base);
        const T v = __ldg(vals + base);
        for (int v0 = 0; v0 < p.k; v0 += KV) {
          T x[KV], a[KV];
          ldg_vec<T, KV>(x, xc + (long long)c * p.k + v0);
#pragma unroll
          for (int qq = 0; qq < KV; ++qq) a[qq] = v * x[qq];
          red_vec<T, KV>(yr + (long long)r * p.ldy + v0, a);
          if (R != C) {
            ldg_vec<T, KV>(x, xr + (long long)r * p.k + v0);
#pragma unroll
            for (int qq = 0; qq < KV; ++qq) a[qq] = v * x[qq];
            red_vec<T, KV>(yc + (long long)c * p.ldy + v0, a);
          }
        }
      }
      continue;
    }
    const int n_here = (int)min(32LL, n_items - c0);
    for (int q = 0; q < n_here; ++q) {  // larger tiles: one tile at a time, lanes over its entries
      const int cnt = __shfl_sync(0xffffffffu, my_cnt, q);
      if (cnt == 0) continue;
      const long long base = __shfl_sync(0xffffffffu, my_base, q);
      const int R = __shfl_sync(0xffffffffu, my_rc.x, q), C = __shfl_sync(0xffffffffu, my_rc.y, q);
      const T *xr = X + (long long)R * 64 * p.k, *xc = X + (long long)C * 64 * p.k;
      T *yr = Y + (long long)R * 64 * p.ldy, *yc = Y + (long long)C * 64 * p.ldy;
      for (int e = lane; e < cnt; e += 32) {
        const int c = __ldg(p.col + base + e), r = __ldg(p.row + base + e);
        const T v = __ldg(vals + base + e);
        for (int v0 = 0; v0 < p.k; v0 += KV) {
          T x[KV], a[KV];
          ldg_vec<T, KV>(x, xc + (long long)c * p.k + v0);
#pragma unroll
          for (int qq = 0; qq < KV; ++qq) a[qq] = v * x[qq];
          red_vec<T, KV>(yr + (long long)r * p.ldy + v0, a);
          if (R != C) {
            ldg_vec<T, KV>(x, xr + (long long)r * p.k + v0);
#pragma unroll
            for (int qq = 0; qq < KV; ++qq) a[qq] = v * x[qq];
            red_vec<T, KV>(yc + (long long)c * p.ldy + v0, a);
          }
        }
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
    const uint16_t *rp = rowptr + (size_t)t * kSpPtrStride;
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

}  // namespace
int sym_spmm_sparse_csr(const cim_sparse_tiles *S, int dtype, const void *X, void *Y, int k, long long ldy, int sms,
                        cudaStream_t stream);  // sparse_csr.cu
namespace {

struct SpState {
  int sms = 0;
  CounterRing *ring = nullptr;  // ticket counters (counter_ring.h)
};
std::mutex g_sp_mu;
std::vector<SpState> g_sp;
CounterRing g_sp_rings[64];
constexpr int kSpRingBlocks = 256;

int sp_state(SpState **out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(CIM_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_sp_mu);
  if ((int)g_sp.size() <= dev) g_sp.resize(dev + 1);
  SpState &s = g_sp[dev];
  if (s.sms == 0) {
    if (dev >= 64) return set_error(CIM_EUNSUPPORTED, "device index >= 64");
    cudaError_t e = cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) {
      s.sms = 0;
      return set_error(CIM_ECUDA, std::string("sparse state: ") + cudaGetErrorString(e));
    }
    s.ring = &g_sp_rings[dev];
    const int rc = s.ring->init(kSpRingBlocks);
    if (rc) {
      s.sms = 0;
      return rc;
    }
  }
  *out = &s;
  return CIM_OK;
}

// Small-tile threshold in (padded) entries: CIM_SPARSE_SMALL overrides (A/B
// sweeps; 0 = every tile through the ring).
int sparse_small_max() {
  static const int v = [] {
    const char *e = std::getenv("CIM_SPARSE_SMALL");
    return e ? std::atoi(e) : kSpSmallDefault;
  }();
  return v;
}

template <typename T, int KV>
int launch_sparse(const cim_sparse_tiles *S, const void *X, void *Y, int k, long long ldx, long long ldy,
                  cudaStream_t stream) {
  SpState *st = nullptr;
  int rc = sp_state(&st);
  if (rc) return rc;
  if (ldx != k) return set_error(CIM_EINVAL, "sparse tiles need dense X rows (ldx == k)");
  const int cap = (S->staged_max_entries > 0 && S->staged_max_entries <= kSpCapSmall) ? kSpCapSmall : kSpCap;
  const SpLayout L = sp_layout(k, (int)sizeof(T), cap);
  // 8 stages (2 per consumer warp) when two CTAs fit per SM, else 4
#ifdef CIM_SP_STAGES
  int stages = CIM_SP_STAGES;  // A/B experiments (a multiple of 4)
#else
  int stages = ((size_t)8 * L.bytes + 128 <= 113 * 1024) ? 8 : 4;
#endif
  const size_t smem = (size_t)stages * L.bytes + 16 * (size_t)stages;  // + full / empty mbarriers
  const bool listed0 = S->staged_tiles != nullptr || S->small_tiles != nullptr;
  const bool csr0 = S->csr_ptr && S->csr_rows > 0;
  const long long n_ring0 = (csr0 && S->csr_all) ? 0 : listed0 ? (S->staged_tiles ? S->n_staged : 0) : S->n_tiles;
  if (n_ring0 > 0 && smem > 227 * 1024) return set_error(CIM_EUNSUPPORTED, "k too large for the sparse-tile stages");
  CounterLease lease;
  if (const int lrc = lease.take(*st->ring, stream, 1)) return lrc;
  unsigned int *ctr = lease.ctr;
  cudaError_t e = cudaSuccess;
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
  p.counter = ctr;
  p.n_tiles = S->n_tiles;
  p.ldx = ldx;
  p.ldy = ldy;
  p.k = k;
  p.small_max = sparse_small_max();
  p.cap = cap;
  p.staged = S->staged_tiles;
  p.n_staged = S->staged_tiles ? S->n_staged : 0;
  const bool listed = S->staged_tiles != nullptr || S->small_tiles != nullptr;
  const bool csr = S->csr_ptr && S->csr_rows > 0;
  const long long n_ring = (csr && S->csr_all) ? 0 : listed ? p.n_staged : S->n_tiles;
  if (n_ring > 0) {
    e = cudaFuncSetAttribute(sparse_spmm_kernel<T, KV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse attr: ") + cudaGetErrorString(e));
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sparse_spmm_kernel<T, KV>, kSpConsumers + 32, smem) !=
            cudaSuccess ||
        occ < 1)
      occ = 1;
    const long long grid = std::min<long long>(n_ring, (long long)st->sms * occ);
    sparse_spmm_kernel<T, KV><<<(unsigned)grid, kSpConsumers + 32, smem, stream>>>(p, stages);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse_spmm launch: ") + cudaGetErrorString(e));
  }
  const long long n_small = listed ? (S->small_tiles ? S->n_small : 0) : (p.small_max > 0 ? S->n_tiles : 0);
  if (S->csr_ptr && S->csr_rows > 0) return sym_spmm_sparse_csr(S, sizeof(T) == 4 ? CIM_F32 : CIM_F64, X, Y, k, ldy,
                                                                st->sms, stream);
  if (n_small > 0) {
    const long long g2 = std::min<long long>((n_small + 255) / 256, (long long)st->sms * 16);  // 32 tiles / warp
    sparse_small_kernel<T, KV><<<(unsigned)g2, 256, 0, stream>>>(p, listed ? S->small_tiles : nullptr,
                                                                 listed ? S->n_small : 0);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse_small launch: ") + cudaGetErrorString(e));
  }
  return CIM_OK;
}

}  // namespace
}  // namespace cim

extern "C" int32_t cim_sparse_small_max(void) { return cim::sparse_small_max(); }

namespace cim {
namespace {
// Does the staged ring for W-wide vector blocks fit in shared memory (the
// plan of launch_sparse)?
template <typename T>
bool sparse_stage_fits(const cim_sparse_tiles *S, int W) {
  const int cap = (S->staged_max_entries > 0 && S->staged_max_entries <= kSpCapSmall) ? kSpCapSmall : kSpCap;
  const SpLayout L = sp_layout(W, (int)sizeof(T), cap);
  const int stages = ((size_t)8 * L.bytes + 128 <= 113 * 1024) ? 8 : 4;
  return (size_t)stages * L.bytes + 16 * (size_t)stages <= 227 * 1024;
}

// X (n_pad × k) → pass-major slices (passes × n_pad × W), 16-byte chunks.
__global__ void sparse_pass_major_kernel(const uint4 *__restrict__ X, uint4 *__restrict__ Xp, long long rows,
                                         int row_chunks, int w_chunks) {
  const long long total = rows * row_chunks;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / row_chunks;
    const int c = (int)(e - r * row_chunks);
    const int ps = c / w_chunks, cc = c - ps * w_chunks;
    Xp[((long long)ps * rows + r) * w_chunks + cc] = X[e];
  }
}

// Widths whose staged X blocks (64·k values each for X_C and X_R) exceed the
// shared-memory ring (f64 k = 64) run as column passes of the largest W that
// fits, each on a pass-major copy of X (stream-ordered allocation) writing
// its W columns of Y in place.
template <typename T, int KV>
int sparse_dispatch(const cim_sparse_tiles *S, const void *X, void *Y, int k, long long ldx, long long ldy,
                    long long n_pad, cudaStream_t stream) {
  const bool listed = S->staged_tiles != nullptr || S->small_tiles != nullptr;
  const bool csr_all = S->csr_ptr && S->csr_rows > 0 && S->csr_all;
  const bool ring = !csr_all && (listed ? (S->staged_tiles != nullptr && S->n_staged > 0) : S->n_tiles > 0);
  if (!ring || sparse_stage_fits<T>(S, k)) return launch_sparse<T, KV>(S, X, Y, k, ldx, ldy, stream);
  int W = k;
  while (W % (2 * KV) == 0 && (W / 2 * (int)sizeof(T)) % 16 == 0 && !sparse_stage_fits<T>(S, W)) W /= 2;
  if (!sparse_stage_fits<T>(S, W) || ldx != k || n_pad <= 0)
    return set_error(CIM_EUNSUPPORTED, "k too large for the sparse-tile stages");
  const int passes = k / W;
  void *Xp = nullptr;
  cudaError_t e = cudaMallocAsync(&Xp, (size_t)n_pad * k * sizeof(T), stream);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sparse pass scratch: ") + cudaGetErrorString(e));
  const int row_chunks = k * (int)sizeof(T) / 16, w_chunks = W * (int)sizeof(T) / 16;
  const long long total = n_pad * row_chunks;
  sparse_pass_major_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 4096), 256, 0, stream>>>(
      static_cast<const uint4 *>(X), static_cast<uint4 *>(Xp), n_pad, row_chunks, w_chunks);
  int rc = CIM_OK;
  e = cudaGetLastError();
  if (e != cudaSuccess) rc = set_error(CIM_ECUDA, std::string("sparse pass-major copy: ") + cudaGetErrorString(e));
  for (int ps = 0; ps < passes && rc == CIM_OK; ++ps)
    rc = launch_sparse<T, KV>(S, static_cast<const T *>(Xp) + (size_t)ps * n_pad * W, static_cast<T *>(Y) + ps * W, W,
                              W, ldy, stream);
  cudaFreeAsync(Xp, stream);
  return rc;
}
}  // namespace

// Called by cim_sym_spmm after the dense tiles (Y already zeroed or accumulating).
int sym_spmm_sparse(const cim_sparse_tiles *S, int dtype, const void *X, void *Y, int k, long long ldx,
                    long long ldy, long long n_pad, cudaStream_t stream) {
  if (!S || S->n_tiles == 0) return CIM_OK;
  if (!S->tile_rc || !S->entry_off || !S->rowptr || !S->colptr ||
      (S->n_entries > 0 && (!S->col || !S->row || !S->cperm || !S->vals)))
    return set_error(CIM_EINVAL, "sparse tile arrays are NULL");
  if (dtype == CIM_F32) {
    if (k % 8 == 0) return sparse_dispatch<float, 8>(S, X, Y, k, ldx, ldy, n_pad, stream);
    if (k % 4 == 0) return sparse_dispatch<float, 4>(S, X, Y, k, ldx, ldy, n_pad, stream);
    if (k % 2 == 0) return sparse_dispatch<float, 2>(S, X, Y, k, ldx, ldy, n_pad, stream);
    return sparse_dispatch<float, 1>(S, X, Y, k, ldx, ldy, n_pad, stream);
  }
  if (k % 4 == 0) return sparse_dispatch<double, 4>(S, X, Y, k, ldx, ldy, n_pad, stream);
  if (k % 2 == 0) return sparse_dispatch<double, 2>(S, X, Y, k, ldx, ldy, n_pad, stream);
  return sparse_dispatch<double, 1>(S, X, Y, k, ldx, ldy, n_pad, stream);
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
  long long e = entry_off[t] + rowptr[t * kSpPtrStride + r];
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
    const uint16_t *rp = rowptr + (size_t)t * kSpPtrStride;
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
    uint16_t *cpt = colptr + (size_t)t * kSpPtrStride;
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
