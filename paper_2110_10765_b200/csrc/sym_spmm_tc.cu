// Tensor-core (tcgen05, kind::tf32) variant of the half-stored symmetric SpMM
//   Y = U·X + U_offᵀ·X          (f32 values and vectors, k ∈ {8, 16})
//
// FP32 accuracy from TF32 tensor cores by splitting both operands into a
// TF32 "hi" part and an exactly-representable remainder "lo" and summing all
// four partial products (hi·hi + hi·lo + lo·hi + lo·lo) in FP32:
//   T = T_hi + T_lo   with T_hi = trunc_tf32(T) (what the MMA reads from raw
//                     FP32 bits) and T_lo = T − T_hi (exact);
//   X = X_hi + X_lo   with X_hi = rna_tf32(X), X_lo = X − X_hi (exact).
// The residual error per product is < 2⁻¹⁹·|T||X| (the MMA truncates T_lo and
// X_lo to TF32 once more), far inside the FP32 gates of tests/test_gpu_parity.
//
// Each 64×64 tile is streamed from HBM once (one 16 KB cp.async.bulk; the HBM
// layout is the SWIZZLE_128B_BASE32B MN-major operand layout, so the tile
// lands in shared memory ready to be the A operand of the transposed product):
//
//   direct      D_dir[128×2k] += [T_hi ; T_lo] · [X_C,hi | X_C,lo]
//               A from TMEM (the splitter warpgroup writes rows with
//               tcgen05.st), accumulated in TMEM across the whole work unit;
//   transposed  D_tr [128×2k]  = [T_hiᵀ ; T_loᵀ] · [X_R,hi | X_R,lo]
//               A from shared memory, MN-major (the raw tile + the splitter's
//               lo copy at +16 KB = two more M groups of the same descriptor).
//
// Warp roles (one CTA of 16 warps per SM, persistent):
//   warp 0       producer: work-unit tickets, bulk copies into an S-stage ring
//   warp 1       TMEM allocator + single-thread MMA issuer (tcgen05.mma/commit)
//   warps 4–7    splitter group 0 (even tiles) ┐ T_lo, TMEM A rows (4 buffers),
//   warps 8–11   splitter group 1 (odd tiles)  ┘ X hi/lo → K-major B operands
//   warps 12–15  epilogue: tcgen05.ld → hi/lo row sums → red.global.add.v4.f32
// The reference reaches this arithmetic only as its per-pair contraction
// kernels (pipeline.py:461-531) over the COO of _collect_pairs (:428-458).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

namespace cim {
namespace tc {
unsigned long long *g_tc_dbg = nullptr;
int g_tc_dbg_ctas = 0;

enum : int { HDR_FIRST = 1, HDR_LAST = 2, HDR_DIAG = 4, HDR_TERM = 8 };

struct TcParams {
  const int4 *units;
  const int2 *tile_rc;
  const unsigned char *vals;
  const unsigned char *X;
  unsigned char *Y;
  unsigned int *counter;
  long long n_units;
  long long ldy;
  unsigned int stages;
  unsigned int stage_bytes;
  unsigned int xblk;      // 64·k·4
  unsigned int off_xc, off_xr, off_bc, off_hdr;  // inside a stage
  unsigned int off_br;    // 2 × B_R
  unsigned int off_xch;   // epilogue exchange, 4 × 64·k floats
  unsigned int off_meta;  // 4 × int4
  unsigned int off_bars;
  unsigned int off_tmem;
  unsigned long long *dbg;  // optional per-CTA role timers (CIM_TC_PROFILE=1), else null
};

// role-timer slots (per CTA, cycles): see tools/tc_profile.py
enum : int {
  DBG_SPL_WAIT_FULL = 0, DBG_SPL_WAIT_ADIR, DBG_SPL_WORK, DBG_MMA_WAIT_SPLIT, DBG_MMA_WAIT_TR, DBG_MMA_WAIT_DIR,
  DBG_MMA_WAIT_META, DBG_MMA_ISSUE, DBG_EPI_WAIT_META, DBG_EPI_WAIT_TR, DBG_EPI_WAIT_DIR, DBG_EPI_WORK,
  DBG_TILES, DBG_TOTAL, DBG_SLOTS = 16
};

// ----------------------------------------------------------------------------
// tcgen05 wrappers
// ----------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// D[tmem] (+)= A[smem desc] · B[smem desc]
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

// D[tmem] (+)= A[tmem] · B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}

__device__ __forceinline__ void tmem_st16(uint32_t addr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(addr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t addr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr)
      : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ float trunc_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

typedef unsigned long long u64;
__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpack2(u64 x, float &a, float &b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {  // a - b, exact here (b = trunc(a))
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// instruction descriptor: D f32, A/B tf32, M = 128, N = 2·KV
template <int KV>
__device__ __forceinline__ uint32_t idesc(bool a_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((uint32_t)(2 * KV / 8) << 17) | (8u << 24);
}

// Split a 64×KV block of X (row-major, row stride k = KV) into the K-major
// INTERLEAVE B operand [X_hi | X_lo] (N = 2·KV rows of 64 K-values):
//   B(n, kk) at (n/8)·2048 + (kk/4)·128 + (n%8)·16 + (kk%4)·4.
// 64 threads (t64): lane → (v%8, kk%4) so each STS hits 32 distinct banks.
template <int KV>
__device__ __forceinline__ void split_x(const float *__restrict__ Xs, unsigned char *B, int t64) {
  const int lane = t64 & 31, half = t64 >> 5;
  const int v8 = lane >> 2, kq = lane & 3;
#pragma unroll
  for (int it = 0; it < KV; ++it) {
    // groups: kk/4 ∈ [0,16), v/8 ∈ [0, KV/8): 16·KV/8 groups, half takes every other
    const int g = 2 * it + half;
    const int kk = (g & 15) * 4 + kq;
    const int v = (g >> 4) * 8 + v8;
    const float x = Xs[kk * KV + v];
    const float hi = rna_tf32(x);
    const float lo = x - hi;
    const int n_hi = v, n_lo = KV + v;
    const int base = (kk >> 2) * 128 + (kk & 3) * 4;
    *reinterpret_cast<float *>(B + (n_hi >> 3) * 2048 + (n_hi & 7) * 16 + base) = hi;
    *reinterpret_cast<float *>(B + (n_lo >> 3) * 2048 + (n_lo & 7) * 16 + base) = lo;
  }
}

#define CIM_T0() const long long _t0 = dbg ? clock64() : 0
#define CIM_ACC(slot) \
  do {                \
    if (dbg) acc[slot] += clock64() - _t0; \
  } while (0)

template <int KV>
__global__ void __launch_bounds__(512, 1) sym_spmm_tc_kernel(const TcParams p) {
  const bool dbg = p.dbg != nullptr;
  long long acc[DBG_SLOTS];
#pragma unroll
  for (int i = 0; i < DBG_SLOTS; ++i) acc[i] = 0;
  const long long t_kernel0 = clock64();
  constexpr int N = 2 * KV;
  extern __shared__ unsigned char smem_raw[];
  // 1 KB alignment by pointer arithmetic on the shared pointer itself, so the
  // compiler keeps the shared address space (LDS/STS, not generic LD/ST)
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index broadcast so the compiler treats role branches as warp-uniform
  // (keeps MMA operands in uniform registers: no R2UR waterfall per MMA)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int S = (int)p.stages;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bars);
  uint64_t *full = bars, *empty = bars + S, *splitf = bars + 2 * S;
  uint64_t *adir_e = bars + 3 * S, *tr_f = adir_e + 4, *tr_e = tr_f + 2, *dir_f = tr_e + 2, *dir_e = dir_f + 2;
  uint64_t *meta_f = dir_e + 2, *meta_e = meta_f + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + p.off_tmem);
  int4 *meta = reinterpret_cast<int4 *>(smem + p.off_meta);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&splitf[s], 128);
    }
    for (int b = 0; b < 4; ++b) mbar_init(&adir_e[b], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tr_f[b], 1);
      mbar_init(&tr_e[b], 4);
      mbar_init(&dir_f[b], 1);
      mbar_init(&dir_e[b], 4);
    }
    for (int b = 0; b < 4; ++b) {
      mbar_init(&meta_f[b], 1);
      mbar_init(&meta_e[b], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // The only CTA on the SM allocated all 512 columns, so the base is column 0;
  // using the constant keeps every TMEM operand address compile-time uniform.
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0;
  // TMEM map: 4 direct-product A buffers (64 columns each: hi rows | lo rows),
  // then 2 buffers × NSPLIT accumulators of N columns for each product.  The
  // K loop of a product alternates between its NSPLIT accumulators so that
  // consecutive MMAs are independent (small-N MMAs into one accumulator
  // serialise on the accumulator dependency).
  constexpr int NSPLIT = 2;
  const uint32_t t_adir = tmem;                             // 4 × 64 columns
  const uint32_t t_dtr = tmem + 256;                        // 2 × NSPLIT × N
  const uint32_t t_ddir = tmem + 256 + 2 * NSPLIT * N;      // 2 × NSPLIT × N

  const unsigned int SB = p.stage_bytes, xblk = p.xblk;

  if (warp == 0) {
    // ================================ producer ================================
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    unsigned int u = 0;
    int useq = 0;  // units handled by this CTA so far
    if (lane == 0) u = atomicAdd(p.counter, 1u);
    u = __shfl_sync(0xffffffffu, u, 0);
    while ((long long)u < p.n_units) {
      const int4 unit = p.units[u];
      unsigned int u_next = 0;
      if (lane == 0) u_next = atomicAdd(p.counter, 1u);
      const int R = unit.x, t0 = unit.y, t1 = unit.z;
      for (int tb = t0; tb < t1; tb += 32) {
        const int t = tb + lane;
        const int myC = (t < t1) ? p.tile_rc[t].y : 0;
        const int cnt = min(32, t1 - tb);
        for (int q = 0; q < cnt; ++q) {
          const int C = __shfl_sync(0xffffffffu, myC, q);
          if (lane == 0) {
            mbar_wait_backoff(&empty[stage], phase ^ 1u);
            unsigned char *st = smem + (size_t)stage * SB;
            const int tt = tb + q;
            const int flags = (tt == t0 ? HDR_FIRST : 0) | (tt == t1 - 1 ? HDR_LAST : 0) | (C == R ? HDR_DIAG : 0);
            *reinterpret_cast<int4 *>(st + p.off_hdr) = make_int4(R, C, flags, useq);
            mbar_arrive_expect_tx(&full[stage], 16384u + 2u * xblk);
            bulk_g2s(st, p.vals + (size_t)tt * 16384u, 16384u, &full[stage], pol_stream);
            bulk_g2s(st + p.off_xc, p.X + (size_t)C * xblk, xblk, &full[stage], pol_keep);
            bulk_g2s(st + p.off_xr, p.X + (size_t)R * xblk, xblk, &full[stage], pol_keep);
          }
          __syncwarp();
          if (++stage == S) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
      ++useq;
      u = __shfl_sync(0xffffffffu, u_next, 0);
    }
    if (lane == 0) {
      // one TERM per splitter group (they take alternate stages)
      for (int e = 0; e < 2; ++e) {
        mbar_wait_backoff(&empty[stage], phase ^ 1u);
        *reinterpret_cast<int4 *>(smem + (size_t)stage * SB + p.off_hdr) = make_int4(0, 0, HDR_TERM, 0);
        mbar_arrive(&full[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ===============================
    // The whole warp runs this loop (converged, uniform control flow); one
    // elected lane issues the tcgen05 instructions.
    const uint32_t id_k = idesc<KV>(false), id_mn = idesc<KV>(true);
    const uint32_t smem_base = smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0, t = 0, ntr = 0, u = 0;
    while (true) {
      {
        CIM_T0();
        mbar_wait(&splitf[stage], phase);
        CIM_ACC(DBG_MMA_WAIT_SPLIT);
      }
      tc_fence_after();
      unsigned char *st = smem + (size_t)stage * SB;
      const int4 h = *reinterpret_cast<const int4 *>(st + p.off_hdr);
      {
        CIM_T0();
        mbar_wait(&meta_e[t & 3], ((t >> 2) & 1) ^ 1);
        CIM_ACC(DBG_MMA_WAIT_META);
      }
      if (elect_one()) {
        meta[t & 3] = h;
        mbar_arrive(&meta_f[t & 3]);
      }
      __syncwarp();
      // flags as warp votes → uniform predicates
      const bool term = __any_sync(0xffffffffu, h.z & HDR_TERM);
      if (term) break;
      const bool first = __any_sync(0xffffffffu, h.z & HDR_FIRST);
      const bool last = __any_sync(0xffffffffu, h.z & HDR_LAST);
      const bool diag = __any_sync(0xffffffffu, h.z & HDR_DIAG);
      const uint32_t ub = u & 1;
      if (first) {
        CIM_T0();
        mbar_wait(&dir_e[ub], ((u >> 1) & 1) ^ 1);
        CIM_ACC(DBG_MMA_WAIT_DIR);
        tc_fence_after();
      }
      if (!diag) {
        CIM_T0();
        mbar_wait(&tr_e[ntr & 1], ((ntr >> 1) & 1) ^ 1);
        CIM_ACC(DBG_MMA_WAIT_TR);
        tc_fence_after();
      }
      const uint32_t st_addr = smem_base + (uint32_t)stage * SB;
      const uint64_t bdesc_c = sdesc(st_addr + p.off_bc, 128, 2048, 0);
      const uint64_t bdesc_r = sdesc(smem_base + p.off_br + (u & 3) * (uint32_t)(N * 256), 128, 2048, 0);
      const uint64_t adesc_t = sdesc(st_addr, 8192, 512, 1);
      const uint32_t a_t = t_adir + (t & 3) * 64;
      const uint32_t d_dir = t_ddir + ub * NSPLIT * N;
      const uint32_t d_tr = t_dtr + (ntr & 1) * NSPLIT * N;
      if (elect_one()) {
        // interleave the two products and alternate accumulators along K;
        // descriptors advance by constants (start-address field is addr >> 4)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const uint32_t sp = (uint32_t)(ks % NSPLIT) * N;
          mma_ts(d_dir + sp, a_t + ks * 8, bdesc_c + (uint64_t)(ks * 16), id_k, (first && ks < NSPLIT) ? 0u : 1u);
          if (!diag)
            mma_ss(d_tr + sp, adesc_t + (uint64_t)(ks * 64), bdesc_r + (uint64_t)(ks * 16), id_mn,
                   ks < NSPLIT ? 0u : 1u);
        }
        tc_commit(&empty[stage]);
        tc_commit(&adir_e[t & 3]);
        if (!diag) tc_commit(&tr_f[ntr & 1]);
        if (last) tc_commit(&dir_f[ub]);
      }
      __syncwarp();
      if (!diag) ++ntr;
      if (last) ++u;
      ++t;
      if (dbg) acc[DBG_TILES] += 1;
      if (++stage == S) {
        stage = 0;
        phase ^= 1u;
      }
    }
  } else if (warp >= 4 && warp < 12) {
    // =============================== splitters ===============================
    const int grp = (warp - 4) >> 2;  // group 0: tiles 0,2,4,…  group 1: tiles 1,3,5,…
    const int q = warp & 3;           // TMEM lane quarter
    const int r = 32 * (q & 1) + lane;  // tile row handled by this thread
    const bool is_lo = q >= 2;
    const int t64 = (q & 1) * 32 + lane;  // 0..63 for q < 2
    uint32_t t = grp;
    int stage = grp % S;
    uint32_t phase = (uint32_t)(grp / S) & 1u;
    while (true) {
      {
        CIM_T0();
        mbar_wait(&full[stage], phase);
        CIM_ACC(DBG_SPL_WAIT_FULL);
      }
      unsigned char *st = smem + (size_t)stage * SB;
      const int4 h = *reinterpret_cast<const int4 *>(st + p.off_hdr);
      if (h.z & HDR_TERM) {
        mbar_arrive(&splitf[stage]);
        break;
      }
      const uint32_t buf = t & 3;
      {
        CIM_T0();
        mbar_wait(&adir_e[buf], ((t >> 2) & 1) ^ 1);
        CIM_ACC(DBG_SPL_WAIT_ADIR);
      }
      const long long _tw = dbg ? clock64() : 0;
      tc_fence_after();
      // Row r of the tile: 16 chunks of 4 values from the BASE32B layout.  The
      // hi warps (q<2) store hi rows to TMEM lanes 0-63 and the lo remainders
      // of chunks 8-15 to shared memory; the lo warps (q≥2) store lo rows to
      // TMEM lanes 64-127 and the lo remainders of chunks 0-7 to shared memory
      // (the transposed product's extra M groups), which balances the work.
      const uint32_t lane_base = ((uint32_t)(32 * q) << 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float4 x[4];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c4 = 4 * j + cc;
          uint32_t in = (uint32_t)(((r & 3) << 7) + ((c4 & 7) << 4));
          in ^= ((in >> 7) & 3u) << 5;
          x[cc] = *reinterpret_cast<const float4 *>(st + (uint32_t)(c4 >> 3) * 8192u + (uint32_t)(r >> 2) * 512u + in);
        }
        uint32_t r16[16];
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int c4 = 4 * j + cc;
          const bool store_lo = is_lo ? (c4 < 8) : (c4 >= 8);
          float4 lo = x[cc];
          if (is_lo || store_lo) {
            const u64 a = pack2(x[cc].x, x[cc].y), b = pack2(x[cc].z, x[cc].w);
            const u64 ta = pack2(trunc_tf32(x[cc].x), trunc_tf32(x[cc].y));
            const u64 tb2 = pack2(trunc_tf32(x[cc].z), trunc_tf32(x[cc].w));
            unpack2(sub2(a, ta), lo.x, lo.y);
            unpack2(sub2(b, tb2), lo.z, lo.w);
          }
          if (store_lo) {
            uint32_t in = (uint32_t)(((r & 3) << 7) + ((c4 & 7) << 4));
            in ^= ((in >> 7) & 3u) << 5;
            *reinterpret_cast<float4 *>(st + 16384u + (uint32_t)(c4 >> 3) * 8192u + (uint32_t)(r >> 2) * 512u + in) = lo;
          }
          const float4 w = is_lo ? lo : x[cc];
          r16[4 * cc + 0] = __float_as_uint(w.x);
          r16[4 * cc + 1] = __float_as_uint(w.y);
          r16[4 * cc + 2] = __float_as_uint(w.z);
          r16[4 * cc + 3] = __float_as_uint(w.w);
        }
        tmem_st16(t_adir + buf * 64 + lane_base + 16 * j, r16);
      }
      if (!is_lo) {
        split_x<KV>(reinterpret_cast<const float *>(st + p.off_xc), st + p.off_bc, t64);
        if (h.z & HDR_FIRST)
          split_x<KV>(reinterpret_cast<const float *>(st + p.off_xr),
                      smem + p.off_br + (uint32_t)(h.w & 3) * (uint32_t)(N * 256), t64);
      }
      tmem_wait_st();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_fence_before();
      mbar_arrive(&splitf[stage]);
      if (dbg) acc[DBG_SPL_WORK] += clock64() - _tw;
      t += 2;
      stage += 2;
      if (stage >= S) {
        stage -= S;
        phase ^= 1u;
      }
    }
  } else if (warp >= 12) {
    // =============================== epilogue ================================
    const int q = warp & 3;
    const int m = 32 * q + lane;  // TMEM lane = D row
    float *xch = reinterpret_cast<float *>(smem + p.off_xch);  // 4 × [64][KV]
    float *Y = reinterpret_cast<float *>(p.Y);
    const long long ldy = p.ldy;
    uint32_t t = 0, ntr = 0, u = 0;
    while (true) {
      {
        CIM_T0();
        mbar_wait(&meta_f[t & 3], (t >> 2) & 1);
        CIM_ACC(DBG_EPI_WAIT_META);
      }
      const long long _tw = dbg ? clock64() : 0;
      const int4 h = meta[t & 3];
      __syncwarp();
      if (lane == 0) mbar_arrive(&meta_e[t & 3]);
      if (h.z & HDR_TERM) break;
      // --- transposed product of this tile: Y_C += (rows m and m+64 of D_tr) ---
      if (!(h.z & HDR_DIAG)) {
        const uint32_t tb = ntr & 1;
        {
          CIM_T0();
          mbar_wait(&tr_f[tb], (ntr >> 1) & 1);
          CIM_ACC(DBG_EPI_WAIT_TR);
        }
        tc_fence_after();
        float y[KV];
#pragma unroll
        for (int e = 0; e < KV; ++e) y[e] = 0.0f;
#pragma unroll
        for (int cb = 0; cb < NSPLIT * N / 16; ++cb) {
          uint32_t r16[16];
          tmem_ld16(t_dtr + tb * NSPLIT * N + ((uint32_t)(32 * q) << 16) + 16 * cb, r16);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) y[(16 * cb + e) % KV] += __uint_as_float(r16[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tr_e[tb]);
        float *xb = xch + (tb) * 64 * KV;
        if (q >= 2) {
#pragma unroll
          for (int e = 0; e < KV; ++e) xb[(m - 64) * KV + e] = y[e];
        }
        named_bar_sync(1, 128);
        if (q < 2) {
#pragma unroll
          for (int e = 0; e < KV; ++e) y[e] += xb[m * KV + e];
          float *yp = Y + ((long long)h.y * kBlock + m) * ldy;
#pragma unroll
          for (int e = 0; e < KV; e += 4) red_add_v4(yp + e, y[e], y[e + 1], y[e + 2], y[e + 3]);
        }
        ++ntr;
      }
      // --- direct product of the unit: Y_R += rows m and m+64 of D_dir ---
      if (h.z & HDR_LAST) {
        const uint32_t ub = u & 1;
        {
          CIM_T0();
          mbar_wait(&dir_f[ub], (u >> 1) & 1);
          CIM_ACC(DBG_EPI_WAIT_DIR);
        }
        tc_fence_after();
        float y[KV];
#pragma unroll
        for (int e = 0; e < KV; ++e) y[e] = 0.0f;
#pragma unroll
        for (int cb = 0; cb < NSPLIT * N / 16; ++cb) {
          uint32_t r16[16];
          tmem_ld16(t_ddir + ub * NSPLIT * N + ((uint32_t)(32 * q) << 16) + 16 * cb, r16);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e) y[(16 * cb + e) % KV] += __uint_as_float(r16[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dir_e[ub]);
        float *xb = xch + (2 + ub) * 64 * KV;
        if (q >= 2) {
#pragma unroll
          for (int e = 0; e < KV; ++e) xb[(m - 64) * KV + e] = y[e];
        }
        named_bar_sync(1, 128);
        if (q < 2) {
#pragma unroll
          for (int e = 0; e < KV; ++e) y[e] += xb[m * KV + e];
          float *yp = Y + ((long long)h.x * kBlock + m) * ldy;
#pragma unroll
          for (int e = 0; e < KV; e += 4) red_add_v4(yp + e, y[e], y[e + 1], y[e + 2], y[e + 3]);
        }
        ++u;
      }
      if (dbg) acc[DBG_EPI_WORK] += clock64() - _tw;
      ++t;
    }
  }
  if (dbg && lane == 0 && (warp == 1 || warp == 4 || warp == 8 || warp == 12)) {
    acc[DBG_TOTAL] = clock64() - t_kernel0;
    unsigned long long *o = p.dbg + ((size_t)blockIdx.x * 4 + (warp == 1 ? 0 : warp == 4 ? 1 : warp == 8 ? 2 : 3)) * DBG_SLOTS;
    for (int i = 0; i < DBG_SLOTS; ++i) o[i] = (unsigned long long)acc[i];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));  // tmem == 0
  }
}

// ----------------------------------------------------------------------------
// host launcher
// ----------------------------------------------------------------------------
template <int KV>
int launch(const cim_half_tiles *H, const void *X, void *Y, long long ldy, cudaStream_t stream, int sms,
           unsigned int *counter) {
  static std::mutex mu;
  static int attr_mask = 0;
  const unsigned int xblk = 64u * KV * 4u;
  const unsigned int bbytes = (unsigned int)(2 * KV) * 256u;  // B operand (N = 2·KV rows × 64 K × 4 B)
  TcParams p{};
  p.off_xc = 32768;
  p.off_xr = p.off_xc + xblk;
  p.off_bc = p.off_xr + xblk;
  p.off_hdr = p.off_bc + bbytes;
  p.stage_bytes = (p.off_hdr + 16 + 1023) & ~1023u;
  const size_t fixed = 4 * (size_t)bbytes + 4 * 64 * KV * 4 + 64 + 8 * 64 + 64;
  const size_t budget = 227 * 1024 - 1024;  // minus manual 1 KB alignment slack
  int S = (int)((budget - fixed) / p.stage_bytes);
  S = std::min(S, 8);
  if (S < 2) return set_error(CIM_EUNSUPPORTED, "tensor-core path: k too large for shared memory");
  p.stages = S;
  size_t off = (size_t)S * p.stage_bytes;
  p.off_br = (unsigned int)off;
  off += 4 * (size_t)bbytes;
  p.off_xch = (unsigned int)off;
  off += 4 * 64 * KV * 4;
  p.off_meta = (unsigned int)off;
  off += 64;
  p.off_bars = (unsigned int)off;
  off += (3 * S + 12 + 8) * 8;
  off = (off + 15) & ~size_t(15);
  p.off_tmem = (unsigned int)off;
  off += 16;
  const size_t smem = off + 1024;

  auto kern = sym_spmm_tc_kernel<KV>;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(attr_mask & (1 << dev))) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess)
        return set_error(CIM_ECUDA, std::string("cudaFuncSetAttribute(tc): ") + cudaGetErrorString(e));
      attr_mask |= (1 << dev);
    }
  }
  p.units = reinterpret_cast<const int4 *>(H->units);
  p.tile_rc = reinterpret_cast<const int2 *>(H->tile_rc);
  p.vals = reinterpret_cast<const unsigned char *>(H->vals);
  p.X = reinterpret_cast<const unsigned char *>(X);
  p.Y = reinterpret_cast<unsigned char *>(Y);
  p.counter = counter;
  p.n_units = H->n_units;
  p.ldy = ldy;
  p.xblk = xblk;
  const long long grid = std::min<long long>(sms, H->n_units);
  p.dbg = nullptr;
  if (const char *e = getenv("CIM_TC_PROFILE")) {
    if (e[0] == '1') {
      static unsigned long long *dbuf = nullptr;
      if (!dbuf) cudaMalloc(&dbuf, 1024 * 4 * DBG_SLOTS * sizeof(unsigned long long));
      cudaMemsetAsync(dbuf, 0, 1024 * 4 * DBG_SLOTS * sizeof(unsigned long long), stream);
      p.dbg = dbuf;
      g_tc_dbg = dbuf;
      g_tc_dbg_ctas = (int)grid;
    }
  }
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("counter memset: ") + cudaGetErrorString(e));
  kern<<<(unsigned int)grid, 512, smem, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sym_spmm_tc launch: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace tc

// Entry used by cim_sym_spmm for CIM_LAYOUT_TC tiles.
int sym_spmm_tc_dispatch(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, cudaStream_t stream,
                         int sms, unsigned int *counter) {
  if (k == 8) return tc::launch<8>(H, X, Y, ldy, stream, sms, counter);
  if (k == 16) return tc::launch<16>(H, X, Y, ldy, stream, sms, counter);
  return set_error(CIM_EUNSUPPORTED, "tensor-core path supports k in {8, 16}");
}

}  // namespace cim

// Debug export of the last profiled launch's role timers (CIM_TC_PROFILE=1).
extern "C" CIM_API int cim_tc_profile_read(unsigned long long *host_out, int max_ctas) {
  if (!cim::tc::g_tc_dbg) return 0;
  const int n = std::min(max_ctas, cim::tc::g_tc_dbg_ctas);
  cudaMemcpy(host_out, cim::tc::g_tc_dbg, (size_t)n * 4 * cim::tc::DBG_SLOTS * sizeof(unsigned long long),
             cudaMemcpyDeviceToHost);
  return n;
}
