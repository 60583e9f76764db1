// One-pass half-stored symmetric SpMM for sm_100a:  Y = U·X + U_offᵀ·X.
//
// Each stored 64×64 tile is streamed from HBM exactly once per pass by a
// single-thread producer (cp.async.bulk into a multi-stage shared-memory
// ring, mbarrier-synchronised) and used by 128 consumer threads per vector
// group for BOTH products:
//
//   direct      acc_r[row][v] += T[row][col] · X_C[col][v]   (Y_R, block row)
//   transposed  acc_c[col][v] += T[row][col] · X_R[row][v]   (Y_C, block col)
//
// Thread ↔ data map (fragment layout v1, include/cim_b200.h): consumer mb owns
// rows rg+8i (i<8) and columns cg+16j (j<4) of every tile, so one LDS.128 per
// micro-row feeds 4·2·KV FMAs with all operands in registers.
//
//  * acc_r lives in registers across a whole work unit (a run of tiles of one
//    block row) and is reduced once per unit: a 2-step butterfly over the 4
//    lanes that share rows, then (f32, k % 4 == 0) one red.global.add.v4 per
//    lane and row — no cross-warp barrier — or (otherwise) a 4-warp sum
//    through shared memory first.
//  * acc_c is reduced per tile inside the warp (the 8 lanes sharing columns):
//    for the packed k = 8 path by a 3-step register butterfly
//    (reduce_cols_shfl), otherwise through a bank-swizzled per-warp scratch;
//    then red.global.add.v4 into Y_C.
//  * Two independent sub-CTAs (own ring + producer + consumers) share one CTA
//    when the accumulators are small (sub_ctas).
//
// Diagonal tiles (R == C) are stored in full and only feed the direct product
// (the packed path runs their transposed FMAs too and discards them).
// The reference reaches this arithmetic only as a pair walk
// (_contract_array_clause / _contract_atomic, pipeline.py:461-488) over the
// full COO from _collect_pairs (pipeline.py:428-458).
//
// Compile-time switches for A/B experiments (tools/build_variant.sh; the
// shipped build defines none): CIM_NO_K8 (generic kernel for every k),
// CIM_ROWFLUSH_SMEM (4-warp shared-memory row sum before the row flush),
// CIM_DIAG_BRANCH (separate diagonal-tile body in the generic kernel),
// CIM_K8_X_NORMAL / CIM_K8_Y_LAST (L2 policies of X copies / Y atomics),
// CIM_K8_ROW_PASSES (multi-pass widths over whole k-wide X rows instead of a
// pass-major copy).  Their measured effects are in profiles/r01/SUMMARY.md
// and DESIGN.md §5.
#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "common.cuh"
#include "counter_ring.h"
#include "host_util.h"

namespace cim {

enum : int { HDR_FIRST = 1, HDR_LAST = 2, HDR_DIAG = 4, HDR_TERM = 8 };

struct __align__(16) StageHdr {
  int R, C, flags, pad;
};

// Wide-register kernel stage header: the Y row blocks this tile updates,
// resolved by the producer (X / Y may live in per-rank chunks, possibly in
// peer GPUs' memory — cim_sym_spmm_chunked).
struct __align__(16) WideHdr {
  int R, C, flags, pad;
  unsigned char *yr, *yc;  // Y block rows of R and C (already offset to the chunk)
};

constexpr int kMaxChunks = 8;

struct SpmmParams {
  const int4 *units;    // (R, t0, t1, 0)
  const int2 *tile_rc;  // (R, C)
  const unsigned char *vals;
  const unsigned char *X;
  unsigned char *Y;
  unsigned int *counter;
  long long n_units;
  long long ldy;  // elements
  int k;          // row length of X (all vectors)
  int v_base;     // first vector handled by this pass
  int stages;
  unsigned int stage_bytes;
  unsigned int tile_bytes;
  unsigned int xblk_bytes;  // 64·k·sizeof(T)
  unsigned int sub_bytes;   // shared memory per sub-CTA
  // chunked X / Y (wide-register kernel): block row b lives in chunk
  // b / chunk_blocks at block b % chunk_blocks; one chunk = plain X / Y
  int n_chunks, chunk_blocks;
  const unsigned char *xch[kMaxChunks];
  unsigned char *ych[kMaxChunks];
  // three-ring kernel, paired passes: work item i = (unit i / n_pass, pass
  // i % n_pass); pass q stages X from the pass-major slice at q·xpass_bytes
  // and writes Y columns q·KROW … (n_pass = 1: plain single pass)
  int n_pass;
  long long xpass_bytes;
};

template <typename T>
struct Chunk;  // 16-byte vector of T
template <>
struct Chunk<float> {
  using V = float4;
  static constexpr int N = 4;
};
template <>
struct Chunk<double> {
  using V = double2;
  static constexpr int N = 2;
};

// Load KV consecutive elements (16-byte aligned when KV·sizeof(T) ≥ 16).
template <typename T, int KV>
__device__ __forceinline__ void load_vec(T (&d)[KV], const T *s) {
  if constexpr (KV * sizeof(T) >= 16) {
    using V = typename Chunk<T>::V;
    constexpr int C = Chunk<T>::N;
#pragma unroll
    for (int q = 0; q < KV / C; ++q) {
      const V v = reinterpret_cast<const V *>(s)[q];
      if constexpr (C == 4) {
        d[4 * q + 0] = v.x;
        d[4 * q + 1] = v.y;
        d[4 * q + 2] = v.z;
        d[4 * q + 3] = v.w;
      } else {
        d[2 * q + 0] = v.x;
        d[2 * q + 1] = v.y;
      }
    }
  } else if constexpr (KV == 2 && sizeof(T) == 4) {
    const float2 v = *reinterpret_cast<const float2 *>(s);
    d[0] = v.x;
    d[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < KV; ++q) d[q] = s[q];
  }
}

// One micro-row of the tile for this thread: 4 values, columns cg+16j.
template <typename T>
__device__ __forceinline__ void load_trow(T (&t)[4], const T *Ts, int i, int mb) {
  if constexpr (sizeof(T) == 4) {
    const float4 v = reinterpret_cast<const float4 *>(Ts)[i * 128 + mb];
    t[0] = v.x;
    t[1] = v.y;
    t[2] = v.z;
    t[3] = v.w;
  } else {
    const double2 a = reinterpret_cast<const double2 *>(Ts)[(2 * i + 0) * 128 + mb];
    const double2 b = reinterpret_cast<const double2 *>(Ts)[(2 * i + 1) * 128 + mb];
    t[0] = a.x;
    t[1] = a.y;
    t[2] = b.x;
    t[3] = b.y;
  }
}

template <typename T, int KV, bool DIAG>
__device__ __forceinline__ void tile_fma(const T *__restrict__ Ts, const T *__restrict__ XC,
                                         const T *__restrict__ XR, int mb, int rg, int cg, int k, int v0,
                                         T (&acc_r)[8][KV], T (&acc_c)[4][KV]) {
  T xc[4][KV];
#pragma unroll
  for (int j = 0; j < 4; ++j) load_vec<T, KV>(xc[j], XC + (cg + 16 * j) * k + v0);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    T t[4];
    load_trow<T>(t, Ts, i, mb);
    T xr[KV];
    if constexpr (!DIAG) load_vec<T, KV>(xr, XR + (rg + 8 * i) * k + v0);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int v = 0; v < KV; ++v) {
        acc_r[i][v] = fma(t[j], xc[j][v], acc_r[i][v]);
        if constexpr (!DIAG) acc_c[j][v] = fma(t[j], xr[v], acc_c[j][v]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Packed FP32 path (sm_100 FFMA2): accumulators are register pairs holding two
// consecutive vectors, and every FMA is  acc[v:v+2] += t · x[v:v+2]  with t a
// broadcast scalar — one FFMA2 instruction for two FMAs, halving the issue
// cost of the inner loop.
// ---------------------------------------------------------------------------
typedef unsigned long long u64;

__device__ __forceinline__ u64 fma2(float t, u64 x, u64 acc) {
  u64 tt, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(tt) : "f"(t));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(tt), "l"(x), "l"(acc));
  return r;
}

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}

__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

__device__ __forceinline__ void unpack2(u64 x, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
}

template <int P>  // P = KV/2 pairs, 8-byte aligned source
__device__ __forceinline__ void load_pairs(u64 (&d)[P], const float *s) {
  if constexpr (P >= 2) {
#pragma unroll
    for (int q = 0; q < P / 2; ++q) {
      const ulonglong2 v = reinterpret_cast<const ulonglong2 *>(s)[q];
      d[2 * q] = v.x;
      d[2 * q + 1] = v.y;
    }
  } else {
    d[0] = *reinterpret_cast<const u64 *>(s);
  }
}

// X_R chunk order for KV = 8 (two 16-byte chunks per row): lanes with rg ≥ 4
// read the upper chunk first, so one LDS.128 of the warp touches 8 rows ×
// alternating chunks = 8 distinct bank quads (1 wavefront instead of 2).  Their
// acc_c slots 0-1 then hold vectors 4-7 and slots 2-3 vectors 0-3, which is
// exactly the exchange pattern of the first butterfly step of
// reduce_cols_shfl (every lane sends slots 2-3, keeps 0-1).
template <int KV>
__device__ __forceinline__ int xr_chunk_swap(int rg) {
  return (KV == 8) ? (rg >> 2) : 0;
}

template <int KV, bool DIAG>
__device__ __forceinline__ void tile_fma2(const float *__restrict__ Ts, const float *__restrict__ XC,
                                          const float *__restrict__ XR, int mb, int rg, int cg, int k, int v0,
                                          u64 (&ar)[8][KV / 2], u64 (&ac)[4][KV / 2]) {
  constexpr int P = KV / 2;
  u64 xc[4][P];
#pragma unroll
  for (int j = 0; j < 4; ++j) load_pairs<P>(xc[j], XC + (cg + 16 * j) * k + v0);
  const int sw = xr_chunk_swap<KV>(rg);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 t4 = reinterpret_cast<const float4 *>(Ts)[i * 128 + mb];
    const float t[4] = {t4.x, t4.y, t4.z, t4.w};
    u64 xr[P];
    if constexpr (!DIAG) {
      const float *row = XR + (rg + 8 * i) * k + v0;
      if constexpr (KV == 8) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(row + 4 * sw);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(row + 4 * (sw ^ 1));
        xr[0] = a.x;
        xr[1] = a.y;
        xr[2] = b.x;
        xr[3] = b.y;
      } else {
        load_pairs<P>(xr, row);
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int q = 0; q < P; ++q) {
        ar[i][q] = fma2(t[j], xc[j][q], ar[i][q]);
        if constexpr (!DIAG) ac[j][q] = fma2(t[j], xr[q], ac[j][q]);
      }
    }
  }
}

// Store a chunk-sized run of outputs with one vector reduction when possible.
template <typename T, int KV>
__device__ __forceinline__ void red_chunk(T *ybase, long long ldy, int e0, const T (&s)[Chunk<T>::N]) {
  constexpr int C = Chunk<T>::N;
  if constexpr (KV >= C) {
    // chunk = one row (or column) index, C consecutive vectors
    const int r = e0 / KV, v = e0 % KV;
    T *p = ybase + (long long)r * ldy + v;
    if constexpr (sizeof(T) == 4) {
      red_add_v4(reinterpret_cast<float *>(p), s[0], s[1], s[2], s[3]);
    } else {
      red_add(p, s[0]);
      red_add(p + 1, s[1]);
    }
  } else {
#pragma unroll
    for (int x = 0; x < C; ++x) {
      const int e = e0 + x, r = e / KV, v = e % KV;
      red_add(ybase + (long long)r * ldy + v, s[x]);
    }
  }
}

// Per-tile reduction of acc_c over the 8 lanes (rg) that share columns.
// scr: this warp's scratch, 32 lanes × 4·KV elements.
template <typename T, int KV>
__device__ __forceinline__ void reduce_cols(T (&acc)[4][KV], T *scr, int lane, int w, T *yblk, long long ldy) {
  using V = typename Chunk<T>::V;
  constexpr int C = Chunk<T>::N;
  constexpr int NCH = (4 * KV) / C;  // chunks per lane
  static_assert((4 * KV) % C == 0, "KV too small for chunking");
  const T *flat = &acc[0][0];
  V *sv = reinterpret_cast<V *>(scr);
  __syncwarp();
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    V v;
    if constexpr (C == 4) {
      v = make_float4(flat[4 * q], flat[4 * q + 1], flat[4 * q + 2], flat[4 * q + 3]);
    } else {
      v = make_double2(flat[2 * q], flat[2 * q + 1]);
    }
    sv[q * 32 + (lane ^ ((q & 1) << 2))] = v;
  }
  __syncwarp();
  if (lane < 4 * NCH) {
    const int cg_lo = lane & 3, q = lane >> 2;
    T s[C];
    V part[8];
#pragma unroll
    for (int rg = 0; rg < 8; ++rg) part[rg] = sv[q * 32 + ((rg * 4 + cg_lo) ^ ((q & 1) << 2))];
    if constexpr (C == 4) {
      // pairwise tree of packed adds: 3 levels × 2 FADD2 instead of 28 FADD
      u64 lo[8], hi[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        lo[r] = pack2(part[r].x, part[r].y);
        hi[r] = pack2(part[r].z, part[r].w);
      }
#pragma unroll
      for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
        for (int r = 0; r < w2; ++r) {
          lo[r] = add2(lo[r], lo[r + w2]);
          hi[r] = add2(hi[r], hi[r + w2]);
        }
      unpack2(lo[0], s[0], s[1]);
      unpack2(hi[0], s[2], s[3]);
    } else {
      T a[8], b[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        a[r] = part[r].x;
        b[r] = part[r].y;
      }
#pragma unroll
      for (int w2 = 4; w2 >= 1; w2 >>= 1)
#pragma unroll
        for (int r = 0; r < w2; ++r) {
          a[r] += a[r + w2];
          b[r] += b[r + w2];
        }
      s[0] = a[0];
      s[1] = b[0];
    }
    // flat element e = j·KV + v ; column = cg + 16·j
    const int cg = w * 4 + cg_lo;
    const int e0 = q * C;
    if constexpr (KV >= C) {
      const int j = e0 / KV, v = e0 % KV;
      T *p = yblk + (long long)(cg + 16 * j) * ldy + v;
      if constexpr (sizeof(T) == 4) {
        red_add_v4(reinterpret_cast<float *>(p), s[0], s[1], s[2], s[3]);
      } else {
        red_add(p, s[0]);
        red_add(p + 1, s[1]);
      }
    } else {
#pragma unroll
      for (int x = 0; x < C; ++x) {
        const int e = e0 + x, j = e / KV, v = e % KV;
        red_add(yblk + (long long)(cg + 16 * j) * ldy + v, s[x]);
      }
    }
  }
}

__device__ __forceinline__ u64 shfl_xor_u64(u64 v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// KV = 8 packed path: per-tile reduction of acc_c over the 8 lanes (rg = lane
// bits 2-4) that share columns, entirely in registers — a 3-step reduce-scatter
// butterfly (16 + 8 + 4 SHFL per lane) instead of a shared-memory round trip.
// ac[j][q]: column cg + 16j, vector pair q (pairs swapped for rg ≥ 4, see
// xr_chunk_swap).  Afterwards lane holds column cg + 16·((lane>>2)&3), vectors
// 4·(lane>>4) .. +3, flushed with one red.global.add.v4.f32.
__device__ __forceinline__ void reduce_cols_shfl(const u64 (&ac)[4][4], int lane, int cg, float *yblk,
                                                 long long ldy, uint64_t ypol) {
  u64 a[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) a[j][q] = add2(ac[j][q], shfl_xor_u64(ac[j][q + 2], 16));
  const bool b3 = lane & 8;
  u64 b[2][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const u64 send = b3 ? a[m][q] : a[m + 2][q];
      const u64 keep = b3 ? a[m + 2][q] : a[m][q];
      b[m][q] = add2(keep, shfl_xor_u64(send, 8));
    }
  const bool b2 = lane & 4;
  u64 c[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const u64 send = b2 ? b[0][q] : b[1][q];
    const u64 keep = b2 ? b[1][q] : b[0][q];
    c[q] = add2(keep, shfl_xor_u64(send, 4));
  }
  const int j = (lane >> 2) & 3, h = lane >> 4;
  float s0, s1, s2, s3;
  unpack2(c[0], s0, s1);
  unpack2(c[1], s2, s3);
  red_add_v4(yblk + (long long)(cg + 16 * j) * ldy + 4 * h, s0, s1, s2, s3, ypol);
}

// Per-unit reduction of acc_r over the 16 threads (4 lanes × 4 warps) that
// share rows.  scr: group scratch, 4 warps × 64·KV elements.
template <typename T, int KV>
__device__ __forceinline__ void reduce_rows(T (&acc)[8][KV], T *scr, int lane, int w, int rg, int gt, int bar_id,
                                            T *yblk, long long ldy) {
  using V = typename Chunk<T>::V;
  constexpr int C = Chunk<T>::N;
  // butterfly over lane bit 0: keep rows i + 4·b0
  const bool b0 = lane & 1;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int v = 0; v < KV; ++v) {
      const T send = b0 ? acc[i][v] : acc[i + 4][v];
      const T keep = b0 ? acc[i + 4][v] : acc[i][v];
      acc[i][v] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
  }
  // butterfly over lane bit 1: keep rows i + 2·b1 (+4·b0)
  const bool b1 = lane & 2;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int v = 0; v < KV; ++v) {
      const T send = b1 ? acc[i][v] : acc[i + 2][v];
      const T keep = b1 ? acc[i + 2][v] : acc[i][v];
      acc[i][v] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
  }
  const int i0 = (b0 ? 4 : 0) + (b1 ? 2 : 0);
#ifndef CIM_ROWFLUSH_SMEM
  if constexpr (sizeof(T) == 4 && KV % 4 == 0) {
    // No cross-warp sum: each lane flushes its 2 rows straight to L2 with
    // vector reductions (4× the row atomics, but no named barrier per unit —
    // the barrier wait was ~7% of the consumer stall samples; 1.86 → 1.76 ms).
#pragma unroll
    for (int ri = 0; ri < 2; ++ri) {
      T *yr = yblk + (long long)(rg + 8 * (i0 + ri)) * ldy;
#pragma unroll
      for (int c = 0; c < KV / 4; ++c)
        red_add_v4(reinterpret_cast<float *>(yr + 4 * c), acc[ri][4 * c], acc[ri][4 * c + 1], acc[ri][4 * c + 2],
                   acc[ri][4 * c + 3]);
    }
    return;
  }
#endif
  named_bar_sync(bar_id, kGroupThreads);  // previous unit's readers are done
  T *mine = scr + w * 64 * KV;
  // every lane now holds distinct rows: rg + 8·(i0 + ri)
#pragma unroll
  for (int ri = 0; ri < 2; ++ri) {
    const int row = rg + 8 * (i0 + ri);
#pragma unroll
    for (int v = 0; v < KV; ++v) mine[row * KV + v] = acc[ri][v];
  }
  named_bar_sync(bar_id, kGroupThreads);
  constexpr int NOUT = 64 * KV / C;  // output chunks
  for (int c = gt; c < NOUT; c += kGroupThreads) {
    T s[C];
    const V a = reinterpret_cast<const V *>(scr)[c];
    const V b = reinterpret_cast<const V *>(scr + 64 * KV)[c];
    const V d = reinterpret_cast<const V *>(scr + 128 * KV)[c];
    const V e = reinterpret_cast<const V *>(scr + 192 * KV)[c];
    if constexpr (C == 4) {
      s[0] = (a.x + b.x) + (d.x + e.x);
      s[1] = (a.y + b.y) + (d.y + e.y);
      s[2] = (a.z + b.z) + (d.z + e.z);
      s[3] = (a.w + b.w) + (d.w + e.w);
    } else {
      s[0] = (a.x + b.x) + (d.x + e.x);
      s[1] = (a.y + b.y) + (d.y + e.y);
    }
    red_chunk<T, KV>(yblk, ldy, c * C, s);
  }
}

// Independent sub-CTAs (own ring, producer warp and consumer groups) packed
// into one CTA: two when a thread carries at most 8 vectors' worth of
// accumulators in total, else one (same residency as two 5-warp CTAs per SM;
// one launch slot, one shared-memory carve-out).
template <typename T, int KV, int NG>
constexpr int sub_ctas() {
  return (KV * NG * (int)sizeof(T) <= 32) ? 2 : 1;
}

// Shared-memory column-reduction scratch (elements); the KV = 8 packed path
// reduces in registers and needs none.
template <typename T, int KV, int NG>
constexpr int col_scratch_elems() {
  return (sizeof(T) == 4 && KV == 8) ? 0 : NG * 4 * 32 * 4 * KV;
}

// KX: the X row length when it is known at compile time (single pass, k =
// KV·NG), else 0.  A constant k turns every shared-memory operand address into
// one per-thread base plus an immediate, which keeps the inner loop free of
// address registers (a runtime k made ptxas precompute and spill them).
template <typename T, int KV, int NG, int KX>
__global__ void __launch_bounds__(sub_ctas<T, KV, NG>() * (NG * kGroupThreads + 32), 1)
    sym_spmm_kernel(const SpmmParams p) {
  extern __shared__ __align__(128) unsigned char smem_all[];
  constexpr int NCONS = NG * kGroupThreads;
  const int sub = threadIdx.x / (NCONS + 32);
  const int tid = threadIdx.x % (NCONS + 32);
  unsigned char *smem = smem_all + (size_t)sub * p.sub_bytes;
  const int S = p.stages;
  unsigned char *stage_base = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
  uint64_t *empty = full + S;
  T *scr_c = reinterpret_cast<T *>(smem + (size_t)S * p.stage_bytes + 128);  // barriers fit in 128 B (S ≤ 8)
  T *scr_r = scr_c + col_scratch_elems<T, KV, NG>();

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NG * 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const unsigned int tile_bytes = p.tile_bytes, xblk = p.xblk_bytes;

  if (tid >= NCONS) {
    // ======================= producer warp =======================
    const int lane = tid & 31;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    unsigned int u = 0;
    if (lane == 0) u = atomicAdd(p.counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    while ((long long)u < p.n_units) {
      const int4 unit = p.units[u];
      unsigned int u_next = 0;
      if (lane == 0) u_next = atomicAdd(p.counter, 1u);  // prefetch the next ticket
      const int R = unit.x, t0 = unit.y, t1 = unit.z;
      const unsigned char *xr_src = p.X + (size_t)R * xblk;
      for (int tb = t0; tb < t1; tb += 32) {
        const int t = tb + lane;
        const int myC = (t < t1) ? p.tile_rc[t].y : 0;
        const int cnt = min(32, t1 - tb);
        for (int q = 0; q < cnt; ++q) {
          const int C = __shfl_sync(0xffffffffu, myC, q);
          if (lane == 0) {
            mbar_wait_backoff(&empty[stage], phase ^ 1u);
            unsigned char *st = stage_base + (size_t)stage * p.stage_bytes;
            const int tt = tb + q;
            const bool diag = (C == R);
            const int flags = (tt == t0 ? HDR_FIRST : 0) | (tt == t1 - 1 ? HDR_LAST : 0) | (diag ? HDR_DIAG : 0);
            StageHdr *h = reinterpret_cast<StageHdr *>(st + tile_bytes + 2 * xblk);
            *h = StageHdr{R, C, flags, 0};
            mbar_arrive_expect_tx(&full[stage], tile_bytes + (diag ? xblk : 2 * xblk));
            bulk_g2s(st, p.vals + (size_t)tt * tile_bytes, tile_bytes, &full[stage], pol_stream);
            bulk_g2s(st + tile_bytes, p.X + (size_t)C * xblk, xblk, &full[stage], pol_keep);
            if (!diag) bulk_g2s(st + tile_bytes + xblk, xr_src, xblk, &full[stage], pol_keep);
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      u = __shfl_sync(0xffffffffu, u_next, 0);
    }
    if (lane == 0) {
      mbar_wait_backoff(&empty[stage], phase ^ 1u);
      StageHdr *h = reinterpret_cast<StageHdr *>(stage_base + (size_t)stage * p.stage_bytes + tile_bytes + 2 * xblk);
      *h = StageHdr{0, 0, HDR_TERM, 0};
      mbar_arrive(&full[stage]);
    }
    return;
  }

  // ======================= consumer groups =======================
  const int g = tid / kGroupThreads;
  const int gt = tid % kGroupThreads;  // micro-block id
  const int w = gt >> 5, lane = tid & 31;
  const int rg = frag_rg(gt), cg = frag_cg(gt);
  const int k = KX > 0 ? KX : p.k;
  const int v0 = p.v_base + g * KV;
  T *my_scr_c = scr_c + (g * 4 + w) * 32 * 4 * KV;
  T *my_scr_r = scr_r + g * 4 * 64 * KV;
  T *Y = reinterpret_cast<T *>(p.Y);

  constexpr bool PACKED = (sizeof(T) == 4) && (KV % 2 == 0);
  using AccE = typename std::conditional<PACKED, u64, T>::type;
  constexpr int NA = PACKED ? KV / 2 : KV;  // accumulator elements per row / column
  AccE acc_r[8][NA];
  AccE acc_c[4][NA];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int v = 0; v < NA; ++v) acc_r[i][v] = AccE(0);

  int stage = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(&full[stage], phase);
    const unsigned char *st = stage_base + (size_t)stage * p.stage_bytes;
    const StageHdr h = *reinterpret_cast<const StageHdr *>(st + tile_bytes + 2 * xblk);
    if (h.flags & HDR_TERM) break;
    if (h.flags & HDR_FIRST) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int v = 0; v < NA; ++v) acc_r[i][v] = AccE(0);
    }
    const T *Ts = reinterpret_cast<const T *>(st);
    const T *XC = reinterpret_cast<const T *>(st + tile_bytes);
    const T *XR = reinterpret_cast<const T *>(st + tile_bytes + xblk);
    const bool diag = h.flags & HDR_DIAG;
    if (PACKED || !diag) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < NA; ++v) acc_c[j][v] = AccE(0);
    }
    if constexpr (PACKED) {
#ifdef CIM_DIAG_BRANCH
      if (diag)
        tile_fma2<KV, true>(Ts, XC, XR, gt, rg, cg, k, v0, acc_r, acc_c);
      else
        tile_fma2<KV, false>(Ts, XC, XR, gt, rg, cg, k, v0, acc_r, acc_c);
#else
      // One code path for every tile: a diagonal tile also runs the
      // transposed FMAs (against X_C, which is X_R there) and just skips their
      // flush.  Two inlined bodies made ptxas reconcile the accumulator
      // registers with ~64 MOVs per off-diagonal tile, more than the 6.7%
      // extra FFMA2 work this costs on diagonal tiles.
      tile_fma2<KV, false>(Ts, XC, diag ? XC : XR, gt, rg, cg, k, v0, acc_r, acc_c);
#endif
    } else {
      if (diag)
        tile_fma<T, KV, true>(Ts, XC, XR, gt, rg, cg, k, v0, acc_r, acc_c);
      else
        tile_fma<T, KV, false>(Ts, XC, XR, gt, rg, cg, k, v0, acc_r, acc_c);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
    if constexpr (PACKED && KV == 8) {
      if (!diag) reduce_cols_shfl(acc_c, lane, cg, Y + (long long)h.C * kBlock * p.ldy + v0, p.ldy, policy_evict_normal());
    } else if (!diag) {
      T fc[4][KV];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int v = 0; v < NA; ++v) {
          if constexpr (PACKED) {
            unpack2(acc_c[j][v], fc[j][2 * v], fc[j][2 * v + 1]);
          } else {
            fc[j][v] = acc_c[j][v];
          }
        }
      reduce_cols<T, KV>(fc, my_scr_c, lane, w, Y + (long long)h.C * kBlock * p.ldy + v0, p.ldy);
    }
    if (h.flags & HDR_LAST) {
      T fr[8][KV];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int v = 0; v < NA; ++v) {
          if constexpr (PACKED) {
            unpack2(acc_r[i][v], fr[i][2 * v], fr[i][2 * v + 1]);
          } else {
            fr[i][v] = acc_r[i][v];
          }
        }
      reduce_rows<T, KV>(fr, my_scr_r, lane, w, rg, gt, 1 + sub * NG + g, Y + (long long)h.R * kBlock * p.ldy + v0, p.ldy);
    }
  }
}


// ---------------------------------------------------------------------------
// k = 8 f32 specialisation (the BASELINE headline): register-reallocated
// warpgroups, X_R resident in registers for a whole work unit.
//
// CTA = 3 warpgroups.  WG0 and WG1 are the consumer groups of two independent
// sub-rings (sub 0, sub 1); WG2 holds their two producer warps (warps 8, 9;
// warps 10-11 leave at once).  setmaxnreg moves registers from WG2 (→ 40) to
// the consumers (→ 232): per SM sub-partition 2 × 232 + 40 ≤ 512 registers
// per lane.  With 232 registers a consumer keeps, besides acc_r (8 rows × 8
// vectors) and acc_c (4 columns × 8), the unit's X_R rows (8 × 8) in
// registers, so a tile costs 8 LDS.128 of T + 8 of X_C per thread instead of
// 32, and the producer copies X_R only with a unit's first tile.
// ---------------------------------------------------------------------------
// Element traits of the wide-register kernel: every accumulator / operand
// register slot is 8 bytes — a pair of f32 vectors (FFMA2 / FADD2 on register
// pairs) or one f64 vector (DFMA).  A warpgroup covers 4 slots = 8 f32 or
// 4 f64 vectors, so the thread map, the X_R chunk swap and the butterflies are
// the same code for both dtypes.
template <typename T>
struct WideE;
template <>
struct WideE<float> {
  using E = u64;
  static constexpr int VPG = 8;  // vectors per warpgroup
  static __device__ __forceinline__ E zero() { return 0ull; }
  static __device__ __forceinline__ E fma(float t, E x, E acc) { return fma2(t, x, acc); }
  static __device__ __forceinline__ E add(E a, E b) { return add2(a, b); }
  static __device__ __forceinline__ E shfl_xor(E v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
  static __device__ __forceinline__ E from_bits(u64 b) { return b; }
  static __device__ __forceinline__ void trow(float (&t)[4], const float *Ts, int i, int gt) {
    const float4 v = reinterpret_cast<const float4 *>(Ts)[i * 128 + gt];
    t[0] = v.x, t[1] = v.y, t[2] = v.z, t[3] = v.w;
  }
  // slots a, b (4 consecutive vectors) → Y
  static __device__ __forceinline__ void flush(float *y, E a, E b, uint64_t pol) {
    float s0, s1, s2, s3;
    unpack2(a, s0, s1);
    unpack2(b, s2, s3);
    red_add_v4(y, s0, s1, s2, s3, pol);
  }
};
template <>
struct WideE<double> {
  using E = double;
  static constexpr int VPG = 4;
  static __device__ __forceinline__ E zero() { return 0.0; }
  static __device__ __forceinline__ E fma(double t, E x, E acc) { return ::fma(t, x, acc); }
  static __device__ __forceinline__ E add(E a, E b) { return a + b; }
  static __device__ __forceinline__ E shfl_xor(E v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }
  static __device__ __forceinline__ E from_bits(u64 b) { return __longlong_as_double((long long)b); }
  static __device__ __forceinline__ void trow(double (&t)[4], const double *Ts, int i, int gt) {
    const double2 a = reinterpret_cast<const double2 *>(Ts)[(2 * i + 0) * 128 + gt];
    const double2 b = reinterpret_cast<const double2 *>(Ts)[(2 * i + 1) * 128 + gt];
    t[0] = a.x, t[1] = a.y, t[2] = b.x, t[3] = b.y;
  }
  static __device__ __forceinline__ void flush(double *y, E a, E b, uint64_t) {
    red_add(y, a);
    red_add(y + 1, b);
  }
};

// The column butterfly of reduce_cols_shfl for any element type.
template <typename T>
__device__ __forceinline__ void reduce_cols_wide(const typename WideE<T>::E (&ac)[4][4], int lane, int cg, T *yblk,
                                                 long long ldy, uint64_t ypol) {
  using W = WideE<T>;
  using E = typename W::E;
  E a[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int q = 0; q < 2; ++q) a[j][q] = W::add(ac[j][q], W::shfl_xor(ac[j][q + 2], 16));
  const bool b3 = lane & 8;
  E b[2][2];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const E send = b3 ? a[m][q] : a[m + 2][q];
      const E keep = b3 ? a[m + 2][q] : a[m][q];
      b[m][q] = W::add(keep, W::shfl_xor(send, 8));
    }
  const bool b2 = lane & 4;
  E c[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const E send = b2 ? b[0][q] : b[1][q];
    const E keep = b2 ? b[1][q] : b[0][q];
    c[q] = W::add(keep, W::shfl_xor(send, 4));
  }
  const int j = (lane >> 2) & 3, h = lane >> 4;
  W::flush(yblk + (long long)(cg + 16 * j) * ldy + (W::VPG / 2) * h, c[0], c[1], ypol);
}

constexpr int kK8Threads = 384;
constexpr int kK8ConsumerRegs = 232;
constexpr int kK8ProducerRegs = 40;

// G = 8-vector groups sharing one ring (k = 8·G): G = 1 → two independent
// sub-rings (WG0, WG1); G = 2 → one ring whose every tile feeds both consumer
// warpgroups (vectors 0-7 and 8-15), the tile streamed from HBM once.
// KROW: the X / Y row length (k); k > 8·G runs as passes of 8·G vectors
// (v_base), each streaming the tiles once more.
template <typename T, int G, int KROW>
__global__ void __launch_bounds__(kK8Threads, 1) sym_spmm_k8_kernel(const SpmmParams p) {
  using W = WideE<T>;
  using E = typename W::E;
  constexpr int VPG = W::VPG;
  extern __shared__ __align__(128) unsigned char smem_all[];
  constexpr int K = KROW;
  constexpr int SUBS = 2 / G;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int wg = warp >> 2;
  const int S = p.stages;
  const unsigned int tile_bytes = p.tile_bytes, xblk = p.xblk_bytes;

  if (threadIdx.x < SUBS) {
    unsigned char *sm = smem_all + (size_t)threadIdx.x * p.sub_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)S * p.stage_bytes);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&full[S + s], 4 * G);  // empty[s]: one arrival per consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (wg == 2) {
    // ======================= producer warps =======================
    setmaxnreg_dec<kK8ProducerRegs>();
    if (warp >= 8 + SUBS) return;
    const int sub = warp - 8;
    const size_t ybytes = (size_t)kBlock * p.ldy * sizeof(T);  // one Y block row
    unsigned char *smem = smem_all + (size_t)sub * p.sub_bytes;
    unsigned char *stage_base = smem;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
    uint64_t *empty = full + S;
    // paired passes (n_pass > 1) re-read each tile right away: keep it in L2
    const uint64_t pol_stream = p.n_pass > 1 ? policy_evict_normal() : policy_evict_first();
#ifdef CIM_K8_X_NORMAL
    const uint64_t pol_keep = policy_evict_normal();
#else
    const uint64_t pol_keep = policy_evict_last();
#endif
    int stage = 0;
    uint32_t phase = 0;
    unsigned int u = 0;
    const long long n_items = p.n_units * p.n_pass;
    if (lane == 0) u = atomicAdd(p.counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    while ((long long)u < n_items) {
      const unsigned int ui = u / (unsigned)p.n_pass, pass = u - ui * (unsigned)p.n_pass;
      const int4 unit = p.units[ui];
      unsigned int u_next = 0;
      if (lane == 0) u_next = atomicAdd(p.counter, 1u);  // prefetch the next ticket
      const int R = unit.x, t0 = unit.y, t1 = unit.z;
      const size_t xpo = (size_t)pass * (size_t)p.xpass_bytes;  // pass slice of X (paired passes: n_chunks = 1)
      for (int tb = t0; tb < t1; tb += 32) {
        const int t = tb + lane;
        const int myC = (t < t1) ? p.tile_rc[t].y : 0;
        const int cnt = min(32, t1 - tb);
        for (int q = 0; q < cnt; ++q) {
          const int C = __shfl_sync(0xffffffffu, myC, q);
          if (lane == 0) {
            mbar_wait_backoff(&empty[stage], phase ^ 1u);
            unsigned char *st = stage_base + (size_t)stage * p.stage_bytes;
            const int tt = tb + q;
            const bool diag = (C == R), first = (tt == t0);
            const int flags = (first ? HDR_FIRST : 0) | (tt == t1 - 1 ? HDR_LAST : 0) | (diag ? HDR_DIAG : 0);
            const int oc = C / p.chunk_blocks, lc = C - oc * p.chunk_blocks;
            const int orr = R / p.chunk_blocks, lr = R - orr * p.chunk_blocks;
            WideHdr *h = reinterpret_cast<WideHdr *>(st + tile_bytes + 2 * xblk);
            *h = WideHdr{R, C, flags, (int)pass * KROW, p.ych[orr] + (size_t)lr * ybytes,
                         p.ych[oc] + (size_t)lc * ybytes};
            const bool need_xr = first && !diag;  // a diagonal first tile has X_R = X_C
            mbar_arrive_expect_tx(&full[stage], tile_bytes + (need_xr ? 2 * xblk : xblk));
            bulk_g2s(st, p.vals + (size_t)tt * tile_bytes, tile_bytes, &full[stage], pol_stream);
            bulk_g2s(st + tile_bytes, p.xch[oc] + xpo + (size_t)lc * xblk, xblk, &full[stage], pol_keep);
            if (need_xr)
              bulk_g2s(st + tile_bytes + xblk, p.xch[orr] + xpo + (size_t)lr * xblk, xblk, &full[stage], pol_keep);
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      u = __shfl_sync(0xffffffffu, u_next, 0);
    }
    if (lane == 0) {
      mbar_wait_backoff(&empty[stage], phase ^ 1u);
      WideHdr *h = reinterpret_cast<WideHdr *>(stage_base + (size_t)stage * p.stage_bytes + tile_bytes + 2 * xblk);
      *h = WideHdr{0, 0, HDR_TERM, 0, nullptr, nullptr};
      mbar_arrive(&full[stage]);
    }
    return;
  }

  // ======================= consumer warpgroups =======================
  setmaxnreg_inc<kK8ConsumerRegs>();
  const int sub = wg / G;
  const int v0 = p.v_base + VPG * (wg % G);  // this warpgroup's vectors v0 .. v0+VPG-1
  unsigned char *smem = smem_all + (size_t)sub * p.sub_bytes;
  unsigned char *stage_base = smem;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
  uint64_t *empty = full + S;
  const int gt = threadIdx.x & 127;  // micro-block id
  const int rg = frag_rg(gt), cg = frag_cg(gt);
  const int sw = xr_chunk_swap<8>(rg);
  const long long ldy = p.ldy;
#ifdef CIM_K8_Y_LAST
  const uint64_t ypol = policy_evict_last();
#else
  const uint64_t ypol = policy_evict_normal();
#endif

  E ar[8][4], ac[4][4], xr[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) ar[i][q] = W::zero(), xr[i][q] = W::zero();

  int stage = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(&full[stage], phase);
    const unsigned char *st = stage_base + (size_t)stage * p.stage_bytes;
    const WideHdr h = *reinterpret_cast<const WideHdr *>(st + tile_bytes + 2 * xblk);
    if (h.flags & HDR_TERM) {
      // chunked (peer-memory) Y: make this thread's remote reductions visible
      // system-wide before the kernel ends and the ranks' barrier follows
      if (p.n_chunks > 1) __threadfence_system();
      break;
    }
    const T *Ts = reinterpret_cast<const T *>(st);
    const T *XC = reinterpret_cast<const T *>(st + tile_bytes);
    const bool diag = h.flags & HDR_DIAG;
    if (h.flags & HDR_FIRST) {
      const T *XR = diag ? XC : reinterpret_cast<const T *>(st + tile_bytes + xblk);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // a row slice = 4 slots = two 16-byte chunks, read in swapped order for rg ≥ 4
        const unsigned char *row = reinterpret_cast<const unsigned char *>(XR + (rg + 8 * i) * K + v0);
        const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(row + 16 * sw);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(row + 16 * (sw ^ 1));
        xr[i][0] = W::from_bits(a.x);
        xr[i][1] = W::from_bits(a.y);
        xr[i][2] = W::from_bits(b.x);
        xr[i][3] = W::from_bits(b.y);
#pragma unroll
        for (int q = 0; q < 4; ++q) ar[i][q] = W::zero();
      }
    }
    E xc[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned char *row = reinterpret_cast<const unsigned char *>(XC + (cg + 16 * j) * K + v0);
      const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(row);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(row + 16);
      xc[j][0] = W::from_bits(a.x);
      xc[j][1] = W::from_bits(a.y);
      xc[j][2] = W::from_bits(b.x);
      xc[j][3] = W::from_bits(b.y);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) ac[j][q] = W::zero();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      T t[4];
      W::trow(t, Ts, i, gt);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ar[i][q] = W::fma(t[j], xc[j][q], ar[i][q]);
          ac[j][q] = W::fma(t[j], xr[i][q], ac[j][q]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
    // a diagonal tile's transposed FMAs (against X_R = X_C) are discarded
    if (!diag) reduce_cols_wide<T>(ac, lane, cg, reinterpret_cast<T *>(h.yc) + v0 + h.pad, ldy, ypol);
    if (h.flags & HDR_LAST) {
      // rows rg + 8i over the 4 lanes sharing them: 2 butterfly steps, then
      // each lane flushes 2 rows × VPG vectors (no cross-warp barrier)
      const bool b0 = lane & 1, b1 = lane & 2;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const E send = b0 ? ar[i][q] : ar[i + 4][q];
          const E keep = b0 ? ar[i + 4][q] : ar[i][q];
          ar[i][q] = W::add(keep, W::shfl_xor(send, 1));
        }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const E send = b1 ? ar[i][q] : ar[i + 2][q];
          const E keep = b1 ? ar[i + 2][q] : ar[i][q];
          ar[i][q] = W::add(keep, W::shfl_xor(send, 2));
        }
      const int i0 = (b0 ? 4 : 0) + (b1 ? 2 : 0);
      T *yblk = reinterpret_cast<T *>(h.yr) + v0 + h.pad;
#pragma unroll
      for (int ri = 0; ri < 2; ++ri) {
        T *yr = yblk + (long long)(rg + 8 * (i0 + ri)) * ldy;
        W::flush(yr, ar[ri][0], ar[ri][1], ypol);
        W::flush(yr + VPG / 2, ar[ri][2], ar[ri][3], ypol);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Three-ring variant of the wide-register kernel (KROW = one warpgroup's
// vectors: f32 k = 8, f64 k = 4).  The two-ring kernel above keeps a unit's
// X_R rows in registers, which costs 64 of its 232 registers and leaves room
// for only two consumer warps per scheduler; ncu shows it issue-limited
// (51% issue, FMA pipe 59%, `wait` the top stall) while DRAM runs at 92% of
// the copy peak, so at k = 8 it is simultaneously at its byte and its issue
// bound.  Here X_R rows are read from the stage with every tile instead
// (the producer copies X_R per tile: an L2 hit after the unit's first tile),
// which brings the consumers to 160 registers and a CTA to three
// independent rings (WG0-WG2 consumers, WG3 = three producer warps):
// three consumer warps per scheduler for the same FFMA2 stream.  The first
// micro-row of a tile initialises the transposed accumulators with a
// multiply (no zeroing moves).
// ---------------------------------------------------------------------------
constexpr int kR3Threads = 512;
constexpr int kR3ConsumerRegs = 160;
constexpr int kR3ProducerRegs = 32;

__device__ __forceinline__ u64 mul2s(float t, u64 x) {
  u64 tt, r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(tt) : "f"(t));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(tt), "l"(x));
  return r;
}

template <typename T>
__device__ __forceinline__ typename WideE<T>::E wide_mul(T t, typename WideE<T>::E x) {
  if constexpr (sizeof(T) == 4)
    return mul2s(t, x);
  else
    return t * x;
}

template <typename T, int KROW>
__global__ void __launch_bounds__(kR3Threads, 1) sym_spmm_k8r3_kernel(const SpmmParams p) {
  using W = WideE<T>;
  using E = typename W::E;
  constexpr int VPG = W::VPG;
  static_assert(KROW == VPG, "one warpgroup's vectors per row");
  extern __shared__ __align__(128) unsigned char smem_all[];
  constexpr int K = KROW;
  constexpr int SUBS = 3;
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);  // warp-uniform
  const int lane = threadIdx.x & 31;
  const int wg = warp >> 2;
  const int S = p.stages;
  const unsigned int tile_bytes = p.tile_bytes, xblk = p.xblk_bytes;

  if (threadIdx.x < SUBS) {
    unsigned char *sm = smem_all + (size_t)threadIdx.x * p.sub_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sm + (size_t)S * p.stage_bytes);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&full[S + s], 4);  // empty[s]: one arrival per consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (wg == 3) {
    // ======================= producer warps (12, 13, 14) =======================
    setmaxnreg_dec<kR3ProducerRegs>();
    if (warp >= 12 + SUBS) return;
    const int sub = warp - 12;
    const size_t ybytes = (size_t)kBlock * p.ldy * sizeof(T);
    unsigned char *smem = smem_all + (size_t)sub * p.sub_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
    uint64_t *empty = full + S;
    // paired passes read every tile n_pass times back to back: keep tiles in
    // L2 (evict_normal) so the later passes of a unit hit; one pass streams
    const uint64_t pol_tile = p.n_pass > 1 ? policy_evict_normal() : policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    const long long n_items = p.n_units * p.n_pass;
    // work-item metadata software-pipelined as in the tensor-core producer:
    // holding item i+1's unit header and item i+2's ticket at the start of
    // item i, load item i+1's first 32 tile columns and item i+2's header,
    // and claim item i+3 — no dependent global load between two items' copies
    const int4 zero4 = make_int4(0, 0, 0, 0);
    unsigned int u = 0, u1 = 0, u2 = 0;
    if (lane == 0) {
      u = atomicAdd(p.counter, 1u);
      u1 = atomicAdd(p.counter, 1u);
      u2 = atomicAdd(p.counter, 1u);
    }
    u = __shfl_sync(0xffffffffu, u, 0);
    u1 = __shfl_sync(0xffffffffu, u1, 0);
    u2 = __shfl_sync(0xffffffffu, u2, 0);
    int4 unit = (long long)u < n_items ? p.units[u / (unsigned)p.n_pass] : zero4;
    int4 unit1 = (long long)u1 < n_items ? p.units[u1 / (unsigned)p.n_pass] : zero4;
    int myC0 = (unit.y + lane < unit.z) ? p.tile_rc[unit.y + lane].y : 0;
    while ((long long)u < n_items) {
      const int myC1 = (unit1.y + lane < unit1.z) ? p.tile_rc[unit1.y + lane].y : 0;
      const int4 unit2 = (long long)u2 < n_items ? p.units[u2 / (unsigned)p.n_pass] : zero4;
      unsigned int u3 = 0;
      if (lane == 0) u3 = atomicAdd(p.counter, 1u);
      const unsigned int ui = u / (unsigned)p.n_pass, pass = u - ui * (unsigned)p.n_pass;
      const int R = unit.x, t0 = unit.y, t1 = unit.z;
      const int orr = R / p.chunk_blocks, lr = R - orr * p.chunk_blocks;
      const unsigned char *xs = p.xch[0] + (size_t)pass * (size_t)p.xpass_bytes;  // pass slice (n_chunks = 1)
      for (int tb = t0; tb < t1; tb += 32) {
        const int t = tb + lane;
        const int myC = tb == t0 ? myC0 : ((t < t1) ? p.tile_rc[t].y : 0);
        const int cnt = min(32, t1 - tb);
        for (int q = 0; q < cnt; ++q) {
          const int C = __shfl_sync(0xffffffffu, myC, q);
          if (lane == 0) {
            mbar_wait_backoff(&empty[stage], phase ^ 1u);
            unsigned char *st = smem + (size_t)stage * p.stage_bytes;
            const int tt = tb + q;
            const bool diag = (C == R);
            const int flags = (tt == t0 ? HDR_FIRST : 0) | (tt == t1 - 1 ? HDR_LAST : 0) | (diag ? HDR_DIAG : 0);
            const int oc = C / p.chunk_blocks, lc = C - oc * p.chunk_blocks;
            WideHdr *h = reinterpret_cast<WideHdr *>(st + tile_bytes + 2 * xblk);
            *h = WideHdr{R, C, flags, (int)pass * KROW, p.ych[orr] + (size_t)lr * ybytes,
                         p.ych[oc] + (size_t)lc * ybytes};
            mbar_arrive_expect_tx(&full[stage], tile_bytes + (diag ? xblk : 2 * xblk));
            bulk_g2s(st, p.vals + (size_t)tt * tile_bytes, tile_bytes, &full[stage], pol_tile);
            if (p.n_pass == 1) {
              bulk_g2s(st + tile_bytes, p.xch[oc] + (size_t)lc * xblk, xblk, &full[stage], pol_keep);
              if (!diag)  // X_R with every tile (L2-resident across the unit)
                bulk_g2s(st + tile_bytes + xblk, p.xch[orr] + (size_t)lr * xblk, xblk, &full[stage], pol_keep);
            } else {
              bulk_g2s(st + tile_bytes, xs + (size_t)C * xblk, xblk, &full[stage], pol_keep);
              if (!diag) bulk_g2s(st + tile_bytes + xblk, xs + (size_t)R * xblk, xblk, &full[stage], pol_keep);
            }
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      u = u1;
      unit = unit1;
      myC0 = myC1;
      u1 = u2;
      unit1 = unit2;
      u2 = __shfl_sync(0xffffffffu, u3, 0);
    }
    if (lane == 0) {
      mbar_wait_backoff(&empty[stage], phase ^ 1u);
      WideHdr *h = reinterpret_cast<WideHdr *>(smem + (size_t)stage * p.stage_bytes + tile_bytes + 2 * xblk);
      *h = WideHdr{0, 0, HDR_TERM, 0, nullptr, nullptr};
      mbar_arrive(&full[stage]);
    }
    return;
  }

  // ======================= consumer warpgroups (rings 0, 1, 2) =======================
  setmaxnreg_inc<kR3ConsumerRegs>();
  const int sub = wg;
  constexpr int v0 = 0;  // staged X rows hold exactly this item's KROW vectors
  unsigned char *smem = smem_all + (size_t)sub * p.sub_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * p.stage_bytes);
  uint64_t *empty = full + S;
  const int gt = threadIdx.x & 127;
  const int rg = frag_rg(gt), cg = frag_cg(gt);
  const int sw = xr_chunk_swap<8>(rg);
  const long long ldy = p.ldy;
  const uint64_t ypol = policy_evict_normal();

  E ar[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) ar[i][q] = W::zero();

  int stage = 0;
  uint32_t phase = 0;
  while (true) {
    mbar_wait(&full[stage], phase);
    const unsigned char *st = smem + (size_t)stage * p.stage_bytes;
    const WideHdr h = *reinterpret_cast<const WideHdr *>(st + tile_bytes + 2 * xblk);
    if (h.flags & HDR_TERM) {
      if (p.n_chunks > 1) __threadfence_system();
      break;
    }
    const T *Ts = reinterpret_cast<const T *>(st);
    const T *XC = reinterpret_cast<const T *>(st + tile_bytes);
    const bool diag = h.flags & HDR_DIAG;
    const T *XR = diag ? XC : reinterpret_cast<const T *>(st + tile_bytes + xblk);
    if (h.flags & HDR_FIRST) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) ar[i][q] = W::zero();
    }
    E xc[4][4], ac[4][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned char *row = reinterpret_cast<const unsigned char *>(XC + (cg + 16 * j) * K + v0);
      const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(row);
      const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(row + 16);
      xc[j][0] = W::from_bits(a.x);
      xc[j][1] = W::from_bits(a.y);
      xc[j][2] = W::from_bits(b.x);
      xc[j][3] = W::from_bits(b.y);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      T t[4];
      W::trow(t, Ts, i, gt);
      E xr[4];
      {
        const unsigned char *row = reinterpret_cast<const unsigned char *>(XR + (rg + 8 * i) * K + v0);
        const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(row + 16 * sw);
        const ulonglong2 b = *reinterpret_cast<const ulonglong2 *>(row + 16 * (sw ^ 1));
        xr[0] = W::from_bits(a.x);
        xr[1] = W::from_bits(a.y);
        xr[2] = W::from_bits(b.x);
        xr[3] = W::from_bits(b.y);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          ar[i][q] = W::fma(t[j], xc[j][q], ar[i][q]);
          ac[j][q] = (i == 0) ? wide_mul<T>(t[j], xr[q]) : W::fma(t[j], xr[q], ac[j][q]);
        }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }
    if (!diag) reduce_cols_wide<T>(ac, lane, cg, reinterpret_cast<T *>(h.yc) + h.pad, ldy, ypol);
    if (h.flags & HDR_LAST) {
      const bool b0 = lane & 1, b1 = lane & 2;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const E send = b0 ? ar[i][q] : ar[i + 4][q];
          const E keep = b0 ? ar[i + 4][q] : ar[i][q];
          ar[i][q] = W::add(keep, W::shfl_xor(send, 1));
        }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const E send = b1 ? ar[i][q] : ar[i + 2][q];
          const E keep = b1 ? ar[i + 2][q] : ar[i][q];
          ar[i][q] = W::add(keep, W::shfl_xor(send, 2));
        }
      const int i0 = (b0 ? 4 : 0) + (b1 ? 2 : 0);
      T *yblk = reinterpret_cast<T *>(h.yr) + h.pad;
#pragma unroll
      for (int ri = 0; ri < 2; ++ri) {
        T *yr = yblk + (long long)(rg + 8 * (i0 + ri)) * ldy;
        W::flush(yr, ar[ri][0], ar[ri][1], ypol);
        W::flush(yr + VPG / 2, ar[ri][2], ar[ri][3], ypol);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

struct DeviceState {
  int sms = 0;
  CounterRing *ring = nullptr;  // scheduler ticket counters (counter_ring.h)
  // one grow-only scratch buffer per device (pass-major X copies); users on
  // any stream are ordered through scratch_ev (waited before use, recorded
  // after the user's kernels are queued) under scratch_mu
  void *scratch = nullptr;
  size_t scratch_bytes = 0;
  cudaEvent_t scratch_ev = nullptr;
};
constexpr int kCounterBlocks = 512;
CounterRing g_rings[64];
std::mutex g_mu;
std::vector<DeviceState> g_dev;

int device_state(DeviceState **out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return set_error(CIM_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_mu);
  if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
  DeviceState &d = g_dev[dev];
  if (d.sms == 0) {
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("cudaDeviceGetAttribute: ") + cudaGetErrorString(e));
    if (dev >= 64) return set_error(CIM_EUNSUPPORTED, "device index >= 64");
    d.ring = &g_rings[dev];
    const int rc = d.ring->init(kCounterBlocks);
    if (rc) return rc;
    d.sms = sms;
  }
  *out = &d;
  return CIM_OK;
}

std::mutex g_scratch_mu;

// The device's scratch buffer of at least `bytes` for work queued on
// `stream` (call with g_scratch_mu held until scratch_done): `stream` first
// waits for the buffer's previous user; a too-small buffer is released after
// that user (cudaFreeAsync on the now-ordered stream) and regrown.
int scratch_begin(DeviceState *d, cudaStream_t stream, size_t bytes, void **out) {
  cudaError_t e = cudaSuccess;
  if (d->scratch_ev) e = cudaStreamWaitEvent(stream, d->scratch_ev, 0);
  else e = cudaEventCreateWithFlags(&d->scratch_ev, cudaEventDisableTiming);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("scratch event: ") + cudaGetErrorString(e));
  if (d->scratch_bytes < bytes) {
    if (d->scratch) cudaFreeAsync(d->scratch, stream);
    d->scratch = nullptr;
    d->scratch_bytes = 0;
    e = cudaMallocAsync(&d->scratch, bytes, stream);
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("scratch: ") + cudaGetErrorString(e));
    d->scratch_bytes = bytes;
  }
  *out = d->scratch;
  return CIM_OK;
}

int scratch_done(DeviceState *d, cudaStream_t stream) {
  const cudaError_t e = cudaEventRecord(d->scratch_ev, stream);
  return e == cudaSuccess ? CIM_OK : set_error(CIM_ECUDA, std::string("scratch event: ") + cudaGetErrorString(e));
}

struct LaunchCfg {
  int KV, NG, passes;
};

bool pick_cfg_default(int dtype, int k, LaunchCfg &c);

// CIM_SPLIT=<KV>x<NG> forces a vector split when that variant is compiled
// (tuning experiments only; the default table below is what ships).
bool pick_cfg(int dtype, int k, LaunchCfg &c) {
  if (!pick_cfg_default(dtype, k, c)) return false;
  if (const char *e = getenv("CIM_SPLIT")) {
    int kv = 0, ng = 0;
    if (sscanf(e, "%dx%d", &kv, &ng) == 2 && kv > 0 && ng > 0 && k % (kv * ng) == 0) {
      c.KV = kv;
      c.NG = ng;
      c.passes = k / (kv * ng);
    }
  }
  return true;
}

bool pick_cfg_default(int dtype, int k, LaunchCfg &c) {
  if (k < 1 || k > 64) return false;
  if (dtype == CIM_F32) {
    if (k == 1 || k == 2 || k == 4) {
      c = {k, 1, 1};
      return true;
    }
    if (k % 8 == 0) {
      const int m = k / 8;
      c = {8, (m % 2 == 0) ? 2 : 1, 0};
      c.passes = m / c.NG;
      return true;
    }
    return false;
  }
  if (dtype == CIM_F64) {
    if (k == 1 || k == 2) {
      c = {k, 1, 1};
      return true;
    }
    if (k % 4 == 0) {
      const int m = k / 4;
      c = {4, (m % 2 == 0) ? 2 : 1, 0};
      c.passes = m / c.NG;
      return true;
    }
    return false;
  }
  return false;
}

template <typename T, int KV, int NG, int KX = 0>
int launch_kernel(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, int passes,
                  cudaStream_t stream, DeviceState *ds) {
  static std::mutex mu;
  static int attr_set_dev_mask = 0;
  const unsigned int tile_bytes = kTileElems * sizeof(T);
  const unsigned int xblk = (unsigned int)(kBlock * k * sizeof(T));
  const unsigned int stage_bytes = (tile_bytes + 2 * xblk + sizeof(StageHdr) + 127u) & ~127u;
  const size_t scratch = (size_t)col_scratch_elems<T, KV, NG>() * sizeof(T) + (size_t)NG * 4 * 64 * KV * sizeof(T);
  constexpr int subs = sub_ctas<T, KV, NG>();
  const size_t budget = (size_t)(227 * 1024) / subs;
  if (budget < scratch + 128 + 2 * (size_t)stage_bytes) return set_error(CIM_EUNSUPPORTED, "k too large for smem");
  int S = (int)((budget - scratch - 128) / stage_bytes);
  S = std::min(S, 8);
  const size_t sub_bytes = ((size_t)S * stage_bytes + 128 + scratch + 127) & ~(size_t)127;
  const size_t smem = subs * sub_bytes;
  const int threads = subs * (NG * kGroupThreads + 32);

  auto kern = sym_spmm_kernel<T, KV, NG, KX>;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    // attribute must cover the largest smem we ever request; set to the max once per device
    if (!(attr_set_dev_mask & (1 << dev))) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess)
        return set_error(CIM_ECUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
      attr_set_dev_mask |= (1 << dev);
    }
  }
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  if (e != cudaSuccess || occ < 1) occ = 1;
  long long grid = (long long)ds->sms * occ;
  grid = std::min<long long>(grid, H->n_units);
  if (grid < 1) return CIM_OK;

  CounterLease lease;
  if (const int rc = lease.take(*ds->ring, stream, passes)) return rc;
  unsigned int *ctr = lease.ctr;

  for (int ps = 0; ps < passes; ++ps) {
    SpmmParams p;
    p.units = reinterpret_cast<const int4 *>(H->units);
    p.tile_rc = reinterpret_cast<const int2 *>(H->tile_rc);
    p.vals = reinterpret_cast<const unsigned char *>(H->vals);
    p.X = reinterpret_cast<const unsigned char *>(X);
    p.Y = reinterpret_cast<unsigned char *>(Y);
    p.counter = ctr + ps;
    p.n_units = H->n_units;
    p.ldy = ldy;
    p.k = k;
    p.v_base = ps * KV * NG;
    p.stages = S;
    p.stage_bytes = stage_bytes;
    p.tile_bytes = tile_bytes;
    p.xblk_bytes = xblk;
    p.sub_bytes = (unsigned int)sub_bytes;
    kern<<<(unsigned int)grid, threads, smem, stream>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sym_spmm launch: ") + cudaGetErrorString(e));
  }
  return CIM_OK;
}

struct Chunks {  // X / Y as per-rank chunks (cim_sym_spmm_chunked); n = 1: plain X / Y
  int n = 1, blocks = 1 << 30;
  const void *x[kMaxChunks] = {};
  void *y[kMaxChunks] = {};
};

template <typename T, int G, int KROW>
int launch_k8(const cim_half_tiles *H, const Chunks &ck, long long ldy, cudaStream_t stream, DeviceState *ds,
              int n_pass = 1, long long xpass_bytes = 0) {
  static std::mutex attr_mu;
  static bool attr_done[64] = {};
  constexpr int SUBS = 2 / G;
  constexpr int passes = KROW / (WideE<T>::VPG * G);
  const unsigned int tile_bytes = kTileElems * sizeof(T);
  const unsigned int xblk = kBlock * KROW * sizeof(T);
  const unsigned int stage_bytes = (tile_bytes + 2 * xblk + sizeof(WideHdr) + 127u) & ~127u;
  const size_t budget = (size_t)(227 * 1024) / SUBS;
  int S = std::min((int)((budget - 128) / stage_bytes), 8);
  if (S < 2) return set_error(CIM_EUNSUPPORTED, "k too large for the k8 kernel's stages");
  const size_t sub_bytes = ((size_t)S * stage_bytes + 128 + 127) & ~(size_t)127;
  const size_t smem = SUBS * sub_bytes;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaSuccess;
  {
    // set once per device; a failure is reported on every call (and retried)
    std::lock_guard<std::mutex> lk(attr_mu);
    if (!attr_done[dev & 63]) {
      e = cudaFuncSetAttribute(sym_spmm_k8_kernel<T, G, KROW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess)
        return set_error(CIM_ECUDA, std::string("cudaFuncSetAttribute(k8): ") + cudaGetErrorString(e));
      attr_done[dev & 63] = true;
    }
  }
  long long grid = std::min<long long>(ds->sms, (H->n_units * n_pass + SUBS - 1) / SUBS);
  if (grid < 1) return CIM_OK;
  CounterLease lease;
  if (const int rc = lease.take(*ds->ring, stream, passes)) return rc;
  unsigned int *ctr = lease.ctr;
  for (int ps = 0; ps < passes; ++ps) {
    SpmmParams p;
    p.units = reinterpret_cast<const int4 *>(H->units);
    p.tile_rc = reinterpret_cast<const int2 *>(H->tile_rc);
    p.vals = reinterpret_cast<const unsigned char *>(H->vals);
    p.X = reinterpret_cast<const unsigned char *>(ck.x[0]);
    p.Y = reinterpret_cast<unsigned char *>(ck.y[0]);
    p.counter = ctr + ps;
    p.n_units = H->n_units;
    p.ldy = ldy;
    p.k = KROW;
    p.v_base = ps * WideE<T>::VPG * G;
    p.stages = S;
    p.stage_bytes = stage_bytes;
    p.tile_bytes = tile_bytes;
    p.xblk_bytes = xblk;
    p.sub_bytes = (unsigned int)sub_bytes;
    p.n_chunks = ck.n;
    p.chunk_blocks = ck.blocks;
    p.n_pass = n_pass;
    p.xpass_bytes = xpass_bytes;
    for (int c = 0; c < kMaxChunks; ++c) {
      p.xch[c] = reinterpret_cast<const unsigned char *>(ck.x[c < ck.n ? c : 0]);
      p.ych[c] = reinterpret_cast<unsigned char *>(ck.y[c < ck.n ? c : 0]);
    }
    sym_spmm_k8_kernel<T, G, KROW><<<(unsigned int)grid, kK8Threads, smem, stream>>>(p);
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sym_spmm_k8 launch: ") + cudaGetErrorString(e));
  }
  return CIM_OK;
}

template <typename T, int KROW>
int launch_k8r3(const cim_half_tiles *H, const Chunks &ck, long long ldy, cudaStream_t stream, DeviceState *ds,
                int n_pass = 1, long long xpass_bytes = 0) {
  static std::mutex attr_mu;
  static bool attr_done[64] = {};
  constexpr int SUBS = 3;
  const unsigned int tile_bytes = kTileElems * sizeof(T);
  const unsigned int xblk = kBlock * KROW * sizeof(T);
  const unsigned int stage_bytes = (tile_bytes + 2 * xblk + sizeof(WideHdr) + 127u) & ~127u;
  const size_t budget = (size_t)(227 * 1024) / SUBS;
  int S = std::min((int)((budget - 128) / stage_bytes), 8);
  if (S < 2) return set_error(CIM_EUNSUPPORTED, "k too large for the three-ring kernel's stages");
  const size_t sub_bytes = ((size_t)S * stage_bytes + 128 + 127) & ~(size_t)127;
  const size_t smem = SUBS * sub_bytes;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaError_t e = cudaSuccess;
  {
    std::lock_guard<std::mutex> lk(attr_mu);
    if (!attr_done[dev & 63]) {
      e = cudaFuncSetAttribute(sym_spmm_k8r3_kernel<T, KROW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess)
        return set_error(CIM_ECUDA, std::string("cudaFuncSetAttribute(k8r3): ") + cudaGetErrorString(e));
      attr_done[dev & 63] = true;
    }
  }
  long long grid = std::min<long long>(ds->sms, (H->n_units * n_pass + SUBS - 1) / SUBS);
  if (grid < 1) return CIM_OK;
  CounterLease lease;
  if (const int rc = lease.take(*ds->ring, stream, 1)) return rc;
  SpmmParams p;
  p.n_pass = n_pass;
  p.xpass_bytes = xpass_bytes;
  p.units = reinterpret_cast<const int4 *>(H->units);
  p.tile_rc = reinterpret_cast<const int2 *>(H->tile_rc);
  p.vals = reinterpret_cast<const unsigned char *>(H->vals);
  p.X = reinterpret_cast<const unsigned char *>(ck.x[0]);
  p.Y = reinterpret_cast<unsigned char *>(ck.y[0]);
  p.counter = lease.ctr;
  p.n_units = H->n_units;
  p.ldy = ldy;
  p.k = KROW;
  p.v_base = 0;
  p.stages = S;
  p.stage_bytes = stage_bytes;
  p.tile_bytes = tile_bytes;
  p.xblk_bytes = xblk;
  p.sub_bytes = (unsigned int)sub_bytes;
  p.n_chunks = ck.n;
  p.chunk_blocks = ck.blocks;
  for (int c = 0; c < kMaxChunks; ++c) {
    p.xch[c] = reinterpret_cast<const unsigned char *>(ck.x[c < ck.n ? c : 0]);
    p.ych[c] = reinterpret_cast<unsigned char *>(ck.y[c < ck.n ? c : 0]);
  }
  sym_spmm_k8r3_kernel<T, KROW><<<(unsigned int)grid, kR3Threads, smem, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sym_spmm_k8r3 launch: ") + cudaGetErrorString(e));
  return CIM_OK;
}

// CIM_K8_PAIRED=0 keeps one launch per pass for multi-pass widths (A/B).
bool use_paired() {
  static const bool v = [] {
    const char *e = std::getenv("CIM_K8_PAIRED");
    return !(e && std::atoi(e) == 0);
  }();
  return v;
}

// CIM_K8_RINGS=2 selects the two-ring kernel for the one-warpgroup widths
// (A/B); the three-ring kernel is the default.
bool use_r3() {
  static const bool v = [] {
    const char *e = std::getenv("CIM_K8_RINGS");
    return !(e && std::atoi(e) == 2);
  }();
  return v;
}

// X (n_pad × k, row-major) → pass-major slices Xp[ps] (n_pad × W): each
// 16-byte chunk of a row goes to its pass slice.
__global__ void pass_major_kernel(const uint4 *__restrict__ X, uint4 *__restrict__ Xp, long long rows, int row_chunks,
                                  int w_chunks) {
  const long long total = rows * row_chunks;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / row_chunks;
    const int c = (int)(e - r * row_chunks);
    const int ps = c / w_chunks, cc = c - ps * w_chunks;
    Xp[((long long)ps * rows + r) * w_chunks + cc] = X[e];
  }
}

// k = passes × W with W = the kernel's vectors per pass: run each pass as its
// own W-wide apply on a pass-major copy of X (Y written in place with its
// row stride), so a pass stages only its W columns of X_C / X_R instead of
// whole k-wide rows.
template <typename T, int G>
int launch_k8_passes(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, cudaStream_t stream,
                     DeviceState *ds) {
  constexpr int W = WideE<T>::VPG * G;
  const int passes = k / W;
  const long long n_pad = (H->n + kBlock - 1) / kBlock * kBlock;
  void *Xp = nullptr;
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  int rc = scratch_begin(ds, stream, (size_t)n_pad * k * sizeof(T), &Xp);
  if (rc) return rc;
  const int row_chunks = k * (int)sizeof(T) / 16, w_chunks = W * (int)sizeof(T) / 16;
  const long long total = n_pad * row_chunks;
  pass_major_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 16LL * ds->sms), 256, 0, stream>>>(
      static_cast<const uint4 *>(X), static_cast<uint4 *>(Xp), n_pad, row_chunks, w_chunks);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("pass_major_kernel: ") + cudaGetErrorString(e));
  if (use_paired()) {  // one launch, a unit's passes adjacent in the ticket order (tiles hit L2)
    Chunks ck;
    ck.x[0] = Xp;
    ck.y[0] = Y;
    rc = launch_k8<T, G, W>(H, ck, ldy, stream, ds, passes, n_pad * W * (long long)sizeof(T));
  } else {
    for (int ps = 0; ps < passes && rc == CIM_OK; ++ps) {
      Chunks ck;
      ck.x[0] = static_cast<const T *>(Xp) + (size_t)ps * n_pad * W;
      ck.y[0] = static_cast<T *>(Y) + ps * W;
      rc = launch_k8<T, G, W>(H, ck, ldy, stream, ds);
    }
  }
  const int rc2 = scratch_done(ds, stream);
  return rc ? rc : rc2;
}

// k = passes × KROW on the three-ring kernel in ONE launch: work items are
// (unit, pass) pairs, the passes of a unit adjacent in the ticket order, so
// a tile read from HBM by its first pass is still in L2 for the others.
template <typename T, int KROW>
int launch_k8r3_paired(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, cudaStream_t stream,
                       DeviceState *ds) {
  const int passes = k / KROW;
  const long long n_pad = (H->n + kBlock - 1) / kBlock * kBlock;
  void *Xp = nullptr;
  std::lock_guard<std::mutex> lk(g_scratch_mu);
  int rc = scratch_begin(ds, stream, (size_t)n_pad * k * sizeof(T), &Xp);
  if (rc) return rc;
  const int row_chunks = k * (int)sizeof(T) / 16, w_chunks = KROW * (int)sizeof(T) / 16;
  const long long total = n_pad * row_chunks;
  pass_major_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 16LL * ds->sms), 256, 0, stream>>>(
      static_cast<const uint4 *>(X), static_cast<uint4 *>(Xp), n_pad, row_chunks, w_chunks);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("pass_major_kernel: ") + cudaGetErrorString(e));
  Chunks ck;
  ck.x[0] = Xp;
  ck.y[0] = Y;
  rc = launch_k8r3<T, KROW>(H, ck, ldy, stream, ds, passes, n_pad * KROW * (long long)sizeof(T));
  const int rc2 = scratch_done(ds, stream);
  return rc ? rc : rc2;
}

// CIM_K8_PAIRED_F64=1 runs f64 k > 4 as paired four-vector passes on the
// three-ring kernel (A/B; off by default until measured faster).
bool use_paired_f64() {
  static const bool v = [] {
    const char *e = std::getenv("CIM_K8_PAIRED_F64");
    return e && std::atoi(e) == 1;
  }();
  return v;
}

// The wide-register kernel for (dtype, k), or EUNSUPPORTED.
int launch_wide(const cim_half_tiles *H, int k, const Chunks &ck, long long ldy, cudaStream_t stream,
                DeviceState *ds) {
  if (H->dtype == CIM_F32) {
    switch (k) {
      case 8: return use_r3() ? launch_k8r3<float, 8>(H, ck, ldy, stream, ds) : launch_k8<float, 1, 8>(H, ck, ldy, stream, ds);
      case 16: return launch_k8<float, 2, 16>(H, ck, ldy, stream, ds);
      case 24: return launch_k8<float, 1, 24>(H, ck, ldy, stream, ds);
      case 32: return launch_k8<float, 2, 32>(H, ck, ldy, stream, ds);
      case 48: return launch_k8<float, 2, 48>(H, ck, ldy, stream, ds);
      case 64: return launch_k8<float, 2, 64>(H, ck, ldy, stream, ds);
    }
  } else {
    switch (k) {
      case 4: return launch_k8<double, 1, 4>(H, ck, ldy, stream, ds);  // HBM-bound (0.96): the two-ring kernel is 1% faster
      case 8: return launch_k8<double, 2, 8>(H, ck, ldy, stream, ds);
      case 12: return launch_k8<double, 1, 12>(H, ck, ldy, stream, ds);
      case 16: return launch_k8<double, 2, 16>(H, ck, ldy, stream, ds);
      case 32: return launch_k8<double, 2, 32>(H, ck, ldy, stream, ds);
    }
  }
  return set_error(CIM_EUNSUPPORTED, "no single-launch wide kernel for (dtype, k) (multi-pass widths run through "
                                     "cim_sym_spmm only)");
}

bool wide_supported(int dtype, int k) {
  if (dtype == CIM_F32) return k % 8 == 0 && k >= 8 && k <= 64;  // k > 8: paired passes of 8 (or 16 / 8)
  // f64 k = 20, 28 and k > 32: column passes of the wide kernel (a
  // generic-kernel stage with whole 64-row X blocks of that many doubles
  // does not fit shared memory)
  return k == 4 || k == 8 || k == 12 || k == 16 || k == 32 || (k > 16 && k <= 64 && k % 4 == 0 && k != 24);
}

}  // namespace
}  // namespace cim

using namespace cim;

namespace cim {
int sym_spmm_tc_dispatch(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, cudaStream_t stream,
                         int sms, unsigned int *counter);
int sym_spmm_dmma_dispatch(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy,
                           cudaStream_t stream, int sms, unsigned int *counter);
}

extern "C" int cim_sym_spmm_supported(int32_t dtype, int32_t k) {
  LaunchCfg c;
  return pick_cfg(dtype, k, c) ? 1 : 0;
}

extern "C" int cim_layout_supports(int32_t layout, int32_t dtype, int32_t k) {
  if (layout == CIM_LAYOUT_FRAG) return cim_sym_spmm_supported(dtype, k);
  if (layout == CIM_LAYOUT_TC) {
    if (dtype == CIM_F32) return (k >= 8 && k <= 64 && k % 8 == 0) ? 1 : 0;
    return ((k >= 8 && k <= 32 && k % 8 == 0) || k == 64) ? 1 : 0;  // f64: DMMA kernel (k = 64: two column passes)
  }
  return 0;
}

namespace cim {
int sym_spmm_sparse(const cim_sparse_tiles *S, int dtype, const void *X, void *Y, int k, long long ldx,
                    long long ldy, long long n_pad, cudaStream_t stream);
int sym_spmm_deterministic(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, bool accumulate,
                           cudaStream_t stream);
}

// Dense tiles (and the Y zeroing); the sparse tiles follow in cim_sym_spmm.
static int sym_spmm_dense(const cim_half_tiles *H, const void *X, void *Y, int32_t k, int64_t ldx, int64_t ldy,
                          uint32_t flags, void *stream_) {
  clear_error();
  if (!H) return set_error(CIM_EINVAL, "H is NULL");
  if (H->block != kBlock) return set_error(CIM_EINVAL, "block must be 64");
  if (H->n < 1) return set_error(CIM_EINVAL, "n must be >= 1");
  if (H->dtype != CIM_F32 && H->dtype != CIM_F64) return set_error(CIM_EINVAL, "dtype must be CIM_F32 or CIM_F64");
  if (!X || !Y) return set_error(CIM_EINVAL, "X and Y must be non-NULL");
  if (k < 1) return set_error(CIM_EINVAL, "k must be >= 1");
  if (ldx != k) return set_error(CIM_EINVAL, "X must be dense row-major (ldx == k)");
  if (ldy < k) return set_error(CIM_EINVAL, "ldy must be >= k");
  if (H->n_tiles < 0 || H->n_units < 0) return set_error(CIM_EINVAL, "negative tile/unit count");
  if (H->n_tiles > 0 && (!H->tile_rc || !H->units || !H->vals)) return set_error(CIM_EINVAL, "tile arrays are NULL");
  const size_t es = H->dtype == CIM_F32 ? 4 : 8;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(Y) & 15) ||
      (reinterpret_cast<uintptr_t>(H->vals) & 15))
    return set_error(CIM_EINVAL, "X, Y and vals must be 16-byte aligned");
  if ((ldy * (int64_t)es) % 16 != 0 && k * es >= 16) return set_error(CIM_EINVAL, "ldy*sizeof(T) must be a multiple of 16");
  if (H->layout != CIM_LAYOUT_FRAG && H->layout != CIM_LAYOUT_TC) return set_error(CIM_EINVAL, "unknown tile layout");
  if (!cim_layout_supports(H->layout, H->dtype, k)) return set_error(CIM_EUNSUPPORTED, "unsupported (layout, dtype, k)");
  LaunchCfg cfg{};
  if (H->layout == CIM_LAYOUT_FRAG) pick_cfg(H->dtype, k, cfg);

  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  DeviceState *ds = nullptr;
  int rc = device_state(&ds);
  if (rc) return rc;
  const int64_t nb = (H->n + kBlock - 1) / kBlock;
  const int64_t n_pad = nb * kBlock;
  if (flags & CIM_DETERMINISTIC)  // writes every row block itself: no zeroing, no atomics
    return sym_spmm_deterministic(H, X, Y, k, ldy, (flags & CIM_ACCUMULATE) != 0, stream);
  if (!(flags & CIM_ACCUMULATE)) {
    cudaError_t e = (ldy == k) ? cudaMemsetAsync(Y, 0, (size_t)n_pad * k * es, stream)
                               : cudaMemset2DAsync(Y, (size_t)ldy * es, 0, (size_t)k * es, (size_t)n_pad, stream);
    if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("zeroing Y: ") + cudaGetErrorString(e));
  }
  if (H->n_tiles == 0 || H->n_units == 0) return CIM_OK;

  if (H->layout == CIM_LAYOUT_TC) {
    if ((reinterpret_cast<uintptr_t>(Y) & 15) || (ldy % 4)) return set_error(CIM_EINVAL, "TC path needs 16-B aligned Y rows");
    // widths above one launch (f64 k > 32: the DMMA kernel's register-resident
    // accumulators) run as column passes of W on a pass-major copy of X, each
    // writing its W columns of Y in place (row stride ldy)
    const int W = (H->dtype == CIM_F64 && k > 32) ? 32 : k;
    if (W == k) {
      CounterLease lease;
      if (const int lrc = lease.take(*ds->ring, stream, 1)) return lrc;
      if (H->dtype == CIM_F64) return sym_spmm_dmma_dispatch(H, X, Y, k, ldy, stream, ds->sms, lease.ctr);
      return sym_spmm_tc_dispatch(H, X, Y, k, ldy, stream, ds->sms, lease.ctr);
    }
    if (k % W != 0) return set_error(CIM_EUNSUPPORTED, "tensor-core layout: k must be a multiple of 32 above 32 (f64)");
    const int passes = k / W;
    void *Xp = nullptr;
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    int rc = scratch_begin(ds, stream, (size_t)n_pad * k * es, &Xp);
    if (rc) return rc;
    const int row_chunks = k * (int)es / 16, w_chunks = W * (int)es / 16;
    const long long total = n_pad * row_chunks;
    pass_major_kernel<<<(unsigned)std::min<long long>((total + 255) / 256, 16LL * ds->sms), 256, 0, stream>>>(
        static_cast<const uint4 *>(X), static_cast<uint4 *>(Xp), n_pad, row_chunks, w_chunks);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = set_error(CIM_ECUDA, std::string("pass_major_kernel: ") + cudaGetErrorString(e));
    CounterLease lease;
    if (!rc) rc = lease.take(*ds->ring, stream, passes);
    for (int ps = 0; ps < passes && rc == CIM_OK; ++ps)
      rc = sym_spmm_dmma_dispatch(H, static_cast<const unsigned char *>(Xp) + (size_t)ps * n_pad * W * es,
                                  static_cast<unsigned char *>(Y) + (size_t)ps * W * es, W, ldy, stream, ds->sms,
                                  lease.ctr + ps);
    const int rc2 = scratch_done(ds, stream);
    return rc ? rc : rc2;
  }

#ifndef CIM_NO_K8
  if (H->layout == CIM_LAYOUT_FRAG && wide_supported(H->dtype, k)) {
#ifndef CIM_K8_ROW_PASSES
    // multi-pass widths: one W-wide apply per pass on a pass-major copy of X
    if (H->dtype == CIM_F32 && k > 8 && k % 8 == 0 && use_r3() && use_paired())
      return launch_k8r3_paired<float, 8>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F64 && k > 4 && k % 4 == 0 && use_r3() && use_paired_f64())
      return launch_k8r3_paired<double, 4>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F32 && k > 16 && k % 16 == 0) return launch_k8_passes<float, 2>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F32 && k > 16) return launch_k8_passes<float, 1>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F64 && (k == 16 || k == 32)) return launch_k8_passes<double, 2>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F64 && k == 12) return launch_k8_passes<double, 1>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F64 && k > 32 && k % 8 == 0) return launch_k8_passes<double, 2>(H, X, Y, k, ldy, stream, ds);
    if (H->dtype == CIM_F64 && k > 16 && k % 8 == 4) return launch_k8_passes<double, 1>(H, X, Y, k, ldy, stream, ds);
#endif
    Chunks ck;
    ck.x[0] = X;
    ck.y[0] = Y;
    return launch_wide(H, k, ck, ldy, stream, ds);
  }
#endif
  if (H->dtype == CIM_F32) {
    switch (cfg.KV * 10 + cfg.NG) {
      case 11:
        if (k == 1) return launch_kernel<float, 1, 1, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 1, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 21:
        if (k == 2) return launch_kernel<float, 2, 1, 2>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 2, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 41:
        if (k == 4) return launch_kernel<float, 4, 1, 4>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 4, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 42:
        if (k == 8) return launch_kernel<float, 4, 2, 8>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 4, 2>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 24:
        if (k == 8) return launch_kernel<float, 2, 4, 8>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 2, 4>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 81:
        if (k == 8) return launch_kernel<float, 8, 1, 8>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 8, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 82:
        if (k == 16) return launch_kernel<float, 8, 2, 16>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<float, 8, 2>(H, X, Y, k, ldy, cfg.passes, stream, ds);
    }
  } else {
    switch (cfg.KV * 10 + cfg.NG) {
      case 11:
        if (k == 1) return launch_kernel<double, 1, 1, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<double, 1, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 21:
        if (k == 2) return launch_kernel<double, 2, 1, 2>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<double, 2, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 41:
        if (k == 4) return launch_kernel<double, 4, 1, 4>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<double, 4, 1>(H, X, Y, k, ldy, cfg.passes, stream, ds);
      case 42:
        if (k == 8) return launch_kernel<double, 4, 2, 8>(H, X, Y, k, ldy, cfg.passes, stream, ds);
        return launch_kernel<double, 4, 2>(H, X, Y, k, ldy, cfg.passes, stream, ds);
    }
  }
  return set_error(CIM_EUNSUPPORTED, "no kernel for (dtype, k)");
}

extern "C" int cim_sym_spmm(const cim_half_tiles *H, const void *X, void *Y, int32_t k, int64_t ldx, int64_t ldy,
                            uint32_t flags, void *stream_) {
  const int rc = sym_spmm_dense(H, X, Y, k, ldx, ldy, flags, stream_);
  if (rc != CIM_OK || (flags & CIM_DETERMINISTIC) || !H->sparse || H->sparse->n_tiles == 0) return rc;
  return sym_spmm_sparse(H->sparse, H->dtype, X, Y, k, ldx, ldy, (H->n + kBlock - 1) / kBlock * kBlock,
                         reinterpret_cast<cudaStream_t>(stream_));
}

extern "C" int cim_sym_spmm_chunked(const cim_half_tiles *H, const void *const *X_chunks, void *const *Y_chunks,
                                    int32_t n_chunks, int64_t chunk_rows, int32_t k, int64_t ldy, void *stream_) {
  clear_error();
  if (!H) return set_error(CIM_EINVAL, "H is NULL");
  if (n_chunks < 1 || n_chunks > kMaxChunks) return set_error(CIM_EINVAL, "n_chunks must be in [1, 8]");
  if (chunk_rows < kBlock || chunk_rows % kBlock) return set_error(CIM_EINVAL, "chunk_rows must be a positive multiple of 64");
  if (!X_chunks || !Y_chunks) return set_error(CIM_EINVAL, "chunk arrays are NULL");
  const int64_t nb = (H->n + kBlock - 1) / kBlock;
  if ((int64_t)n_chunks * (chunk_rows / kBlock) < nb) return set_error(CIM_EINVAL, "chunks do not cover the matrix rows");
  if (H->layout != CIM_LAYOUT_FRAG) return set_error(CIM_EUNSUPPORTED, "chunked apply needs fragment-layout tiles");
  if (H->sparse && H->sparse->n_tiles > 0) return set_error(CIM_EUNSUPPORTED, "chunked apply: dense tiles only");
  if (!wide_supported(H->dtype, k)) return set_error(CIM_EUNSUPPORTED, "chunked apply: (dtype, k) has no wide kernel");
  if (ldy < k) return set_error(CIM_EINVAL, "ldy must be >= k");
  const size_t es = H->dtype == CIM_F32 ? 4 : 8;
  Chunks ck;
  ck.n = n_chunks;
  ck.blocks = (int)(chunk_rows / kBlock);
  for (int c = 0; c < n_chunks; ++c) {
    if (!X_chunks[c] || !Y_chunks[c]) return set_error(CIM_EINVAL, "NULL chunk pointer");
    if ((reinterpret_cast<uintptr_t>(X_chunks[c]) & 15) || (reinterpret_cast<uintptr_t>(Y_chunks[c]) & 15))
      return set_error(CIM_EINVAL, "chunks must be 16-byte aligned");
    ck.x[c] = X_chunks[c];
    ck.y[c] = Y_chunks[c];
  }
  if ((ldy * (int64_t)es) % 16) return set_error(CIM_EINVAL, "ldy*sizeof(T) must be a multiple of 16");
  DeviceState *ds = nullptr;
  int rc = device_state(&ds);
  if (rc) return rc;
  if (H->n_tiles == 0 || H->n_units == 0) return CIM_OK;
  return launch_wide(H, k, ck, ldy, reinterpret_cast<cudaStream_t>(stream_), ds);
}
