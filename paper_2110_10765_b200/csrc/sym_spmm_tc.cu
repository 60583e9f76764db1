// Tensor-core (tcgen05, kind::tf32) half-stored symmetric SpMM
//   Y = U·X + U_offᵀ·X          (f32 tiles and vectors, k ∈ 8ℕ, k ≤ 64)
//
// FP32 accuracy from TF32 tensor cores ("3×TF32"): the MMA reads the top 19
// bits of each FP32 operand, so with  T = hi(T) + lo(T),  lo(T) = T − hi(T)
// (exact), and the same split of X,
//   T·X ≈ hi(T)·hi(X) + lo(T)·hi(X) + hi(T)·lo(X)
// with a residual below 2⁻²⁰·|T||X| per product (lo·lo and the truncation of
// the lo parts), far inside the FP32 gates of tests/test_gpu_parity.py.  The
// three partial products are concatenated along K, so ONE accumulator per
// tile sums them inside the tensor core (no hi/lo bookkeeping in the
// epilogue).
//
// Both products of a tile come out of one MMA chain with M = 128:
//
//   A (TMEM, 128 lanes × 128 columns) = [ T  | lo(T)  ]   lanes  0-63: row r of T
//                                       [ Tᵀ | lo(T)ᵀ ]   lanes 64-127: column c of T
//   B (smem, K-major, N = 2k)          = [ X_C | X_R ]   (hi, and lo in a second copy)
//   D (TMEM, 128 × 2k) = Σ_ks  A_hi·B_hi + A_lo·B_hi + A_hi·B_lo   (24 MMAs, K = 8 each)
//
//   D[r][v]        = (T·X_C)[r][v]      → Y_R  (direct product, lanes 0-63, columns 0..k-1)
//   D[64+c][k+v]   = (Tᵀ·X_R)[c][v]     → Y_C  (transposed product, lanes 64-127, columns k..2k-1)
//
// (the other two quadrants of D are discarded).  With A in TMEM the MMA
// issues at its N/2-cycle floor (tools/tc_ts_bench.cu: 9 / 16 / 32 / 64
// cycles per K = 8 step at N = 16 / 32 / 64 / 128, against 79-118 with A
// read from shared memory — the bound of the round-1 variant).  The tile is
// read from shared memory twice by the splitters (as rows and as columns;
// the HBM layout CIM_LAYOUT_TC makes both patterns bank-conflict-free) and
// written to TMEM with tcgen05.st; each stored tile is still streamed from
// HBM exactly once.
//
// Warp roles (one CTA of 16 warps per SM, persistent, work units by ticket):
//   warp 0        producer: bulk copies (tile 16 KB, X_C, X_R) into an S-stage ring
//   warp 1        TMEM allocator + MMA issuer (one elected lane)
//   warps 4–7     splitter group 0 (even tiles) ┐ T → TMEM A buffer (NA buffers),
//   warps 8–11    splitter group 1 (odd tiles)  ┘ X_C / X_R → K-major B hi / lo
//   warps 12–15   epilogue: tcgen05.ld of D; lanes 0-63 sum the direct product
//                 over the work unit (one reduction per row of Y_R), lanes
//                 64-127 reduce the transposed product into Y_C per tile
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

enum : int { HDR_FIRST = 1, HDR_LAST = 2, HDR_DIAG = 4, HDR_TERM = 8, HDR_TERM2 = 16, HDR_XR = 32 };

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
  unsigned int xblk;                  // 64·k·4
  unsigned int off_xc, off_xr, off_hdr;  // inside a stage
  unsigned int off_b;                 // NA B buffers (k·1024 B each)
  unsigned int off_hdrj;              // NA int4 headers (splitter → MMA)
  unsigned int off_meta;              // ND int4 headers (MMA → epilogue)
  unsigned int off_bars;
  unsigned int off_tmem;
  unsigned int off_ebuf;  // 4 staging blocks of 64·k floats for bulk Y reductions (0 = red.v4 per row)
  int xpol, ypol;         // L2 policies (A/B, CIM_TC_XPOL / CIM_TC_YPOL): 0 evict_last/normal, 1 evict_first, 2 evict_normal/last
};

// Role timers (tools/tc_profile.py; compiled in only with -DCIM_TC_PROF): lane 0
// of one warp per role accumulates clock64 deltas per slot.  Roles: 0 MMA
// issuer, 1 splitter row warp, 2 splitter column warp, 3 epilogue direct
// warp, 4 epilogue transposed warp.
enum : int { P_WAIT0 = 0, P_WAIT1, P_WAIT2, P_WORK0, P_WORK1, P_WORK2, P_WORK3, P_TILES = 14, P_TOTAL = 15, P_SLOTS = 16 };
constexpr int kProfRoles = 6, kProfCtas = 160;  // role 5: the producer lane
#ifdef CIM_TC_PROF
__device__ unsigned long long g_prof[kProfCtas][kProfRoles][P_SLOTS];
#define TPROF_DECL long long _pa[P_SLOTS] = {0}; long long _pt = clock64(); const long long _p0 = _pt
#define TPROF(slot) do { const long long _n = clock64(); _pa[slot] += _n - _pt; _pt = _n; } while (0)
#define TPROF_TILE() (_pa[P_TILES] += 1)
#define TPROF_DUMP(role) do { if (lane == 0 && blockIdx.x < kProfCtas) { _pa[P_TOTAL] = clock64() - _p0; \
    for (int _i = 0; _i < P_SLOTS; ++_i) g_prof[blockIdx.x][role][_i] = (unsigned long long)_pa[_i]; } } while (0)
#else
#define TPROF_DECL
#define TPROF(slot)
#define TPROF_TILE()
#define TPROF_DUMP(role)
#endif

// ----------------------------------------------------------------------------
// tcgen05 wrappers
// ----------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
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

// shared-memory matrix descriptor, SWIZZLE_NONE (layout 0) unless given
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

__device__ __forceinline__ void tmem_ld8(uint32_t addr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr)
               : "memory");
}

__device__ __forceinline__ void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One 64 × k block of partial sums (staged in shared memory) → the 64
// contiguous rows of a dense Y block: one bulk reduction (UBLKRED.ADD.F32)
// instead of 64·k/4 red.global.add.v4.f32 from the epilogue warps.
__device__ __forceinline__ void bulk_red_f32(float *dst, const void *src, unsigned bytes, int ypol = 0) {
  if (ypol == 0) {
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
  } else {
    const uint64_t pol = ypol == 1 ? policy_evict_first() : policy_evict_last();
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.L2::cache_hint.add.f32 [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(pol)
                 : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// lo(x) = x − (x with the low 13 mantissa bits cleared): exact in FP32
__device__ __forceinline__ float lo_tf32(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// lo() of 16 words, two at a time (FADD2: x − trunc(x) per lane pair)
__device__ __forceinline__ void lo16(const uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int e = 0; e < 16; e += 2) {
    unsigned long long a, b, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(hi[e]), "r"(hi[e + 1]));
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "r"(hi[e] & 0xFFFFE000u), "r"(hi[e + 1] & 0xFFFFE000u));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo[e]), "=r"(lo[e + 1]) : "l"(r));
  }
}

// instruction descriptor: D f32, A/B tf32 (K-major), M = 128, N = 2·K
template <int K>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(2 * K / 8) << 17) | (8u << 24);
}

// Buffer counts (TMEM: NA·128 + ND·2K ≤ 512 columns).
template <int K>
struct Cfg {
  static constexpr int N = 2 * K;
  static constexpr int NA = K <= 24 ? 3 : 2;
  static constexpr int ND = (512 - NA * 128) / N < 4 ? (512 - NA * 128) / N : 4;
  static constexpr unsigned BBYTES = (unsigned)K * 1024u;  // 4K rows × 64 K-values × 4 B
  static_assert(K % 8 == 0 && K >= 8 && K <= 64, "K must be a multiple of 8 in [8, 64]");
  static_assert(ND >= 2, "TMEM budget");
};

// B(n, kk) of the K-major SWIZZLE_NONE operand: 8-row × 16-byte core
// matrices, K-adjacent ones 128 B apart (LBO), N-adjacent 8-row groups
// 2048 B apart (SBO).
__device__ __forceinline__ unsigned b_off(int n, int kk) {
  return (unsigned)((n >> 3) * 2048 + (kk >> 2) * 128 + (n & 7) * 16 + (kk & 3) * 4);
}

// Build B = [X_C,hi | X_R,hi | X_C,lo | X_R,lo] (N = 4K rows, K-major) from
// the staged row-major X blocks (the X_R rows only when `with_r`: a B buffer
// keeps the X_R part of the last block row it was built for); t = 0..127.
// One item = (vector v, four K-values kk0..kk0+3): four word loads, one
// 16-byte store of the hi values and one of the lo values.  Lanes take
// consecutive v, so a warp's 16-byte stores land in 8 distinct bank groups
// (4 wavefronts for 512 B, the minimum).
template <int K>
__device__ __forceinline__ void build_b(const float *__restrict__ Xc, const float *__restrict__ Xr,
                                        unsigned char *B, int t, bool with_r) {
  constexpr int ITEMS = 16 * K;  // per source block
#pragma unroll
  for (int src = 0; src < 2; ++src) {
    if (src == 1 && !with_r) break;
    const float *Xs = src ? Xr : Xc;
#pragma unroll
    for (int e = t; e < ITEMS; e += 128) {
      const int v = e % K, kk4 = e / K;
      const float *x = Xs + (4 * kk4) * K + v;
      float4 hi, lo;
      hi.x = x[0];
      hi.y = x[K];
      hi.z = x[2 * K];
      hi.w = x[3 * K];
      lo.x = lo_tf32(hi.x);
      lo.y = lo_tf32(hi.y);
      lo.z = lo_tf32(hi.z);
      lo.w = lo_tf32(hi.w);
      const int n = src * K + v;
      *reinterpret_cast<float4 *>(B + b_off(n, 4 * kk4)) = hi;
      *reinterpret_cast<float4 *>(B + b_off(n + 2 * K, 4 * kk4)) = lo;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(512, 1) sym_spmm_tc_kernel(const TcParams p) {
  using C = Cfg<K>;
  constexpr int N = C::N, NA = C::NA, ND = C::ND;
  extern __shared__ unsigned char smem_raw[];
  // 1 KB alignment by pointer arithmetic on the shared pointer itself (keeps
  // the shared address space: LDS/STS, not generic LD/ST)
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, lane = tid & 31;
  // warp index broadcast so role branches are warp-uniform (MMA operands in
  // uniform registers)
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int S = (int)p.stages;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + p.off_bars);
  uint64_t *full = bars, *empty = bars + S;
  uint64_t *splitf = bars + 2 * S, *ab_empty = splitf + NA;
  uint64_t *d_full = ab_empty + NA, *d_empty = d_full + ND, *meta_f = d_empty + ND;
  uint64_t *hdr_ready = meta_f + ND;  // [S]: tile producer → X producer, the stage's header is written
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + p.off_tmem);
  int4 *hdrj = reinterpret_cast<int4 *>(smem + p.off_hdrj);
  int4 *meta = reinterpret_cast<int4 *>(smem + p.off_meta);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
      mbar_init(&hdr_ready[s], 1);
    }
    for (int j = 0; j < NA; ++j) {
      mbar_init(&splitf[j], 4);
      mbar_init(&ab_empty[j], 1);
    }
    for (int d = 0; d < ND; ++d) {
      mbar_init(&d_full[d], 1);
      mbar_init(&d_empty[d], 4);
      mbar_init(&meta_f[d], 1);
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
  // the constant keeps every TMEM operand address compile-time uniform.
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t t_a = 0;              // NA × 128 columns
  constexpr uint32_t t_d = NA * 128;       // ND × N columns
  const unsigned int SB = p.stage_bytes;

  if (warp == 0) {
    // ================================ producer ================================
    TPROF_DECL;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = p.xpol == 1 ? policy_evict_first() : p.xpol == 2 ? policy_evict_normal() : policy_evict_last();
    const unsigned int xblk = p.xblk;
    int stage = 0;
    uint32_t phase = 0;
    unsigned int u = 0;
    // B buffer j = (tile seq) % NA keeps the X_R part of the last non-diagonal
    // tile built into it: X_R is staged and split only when that row changes
    int xr_of[NA];
#pragma unroll
    for (int b = 0; b < NA; ++b) xr_of[b] = -1;
    uint32_t seq = 0;
    // Work-unit metadata is software-pipelined so that no dependent global
    // load (ticket → unit → tile columns) sits between two units' copies:
    // at the start of unit i the producer already holds unit i+1 and the
    // ticket of unit i+2; it then loads unit i+1's first 32 tile columns,
    // unit i+2's header, and claims the ticket of unit i+3.  (One producer
    // lane per SM: exposed metadata latency drained the ring — the splitters
    // waited 40% of their time for data at k = 8.)
    const long long n_units = p.n_units;
    const int4 zero4 = make_int4(0, 0, 0, 0);
    unsigned int u1 = 0, u2 = 0;
    if (lane == 0) {
      u = atomicAdd(p.counter, 1u);
      u1 = atomicAdd(p.counter, 1u);
      u2 = atomicAdd(p.counter, 1u);
    }
    u = __shfl_sync(0xffffffffu, u, 0);
    u1 = __shfl_sync(0xffffffffu, u1, 0);
    u2 = __shfl_sync(0xffffffffu, u2, 0);
    int4 unit = (long long)u < n_units ? p.units[u] : zero4;
    int4 unit1 = (long long)u1 < n_units ? p.units[u1] : zero4;
    int myC0 = (unit.y + lane < unit.z) ? p.tile_rc[unit.y + lane].y : 0;
    while ((long long)u < n_units) {
      const int myC1 = (unit1.y + lane < unit1.z) ? p.tile_rc[unit1.y + lane].y : 0;
      const int4 unit2 = (long long)u2 < n_units ? p.units[u2] : zero4;
      unsigned int u3 = 0;
      if (lane == 0) u3 = atomicAdd(p.counter, 1u);
      const int R = unit.x, t0 = unit.y, t1 = unit.z;
      for (int tb = t0; tb < t1; tb += 32) {
        const int t = tb + lane;
        const int myC = tb == t0 ? myC0 : ((t < t1) ? p.tile_rc[t].y : 0);
        const int cnt = min(32, t1 - tb);
        for (int q = 0; q < cnt; ++q) {
          const int Cb = __shfl_sync(0xffffffffu, myC, q);
          if (lane == 0) {
            TPROF(P_WORK0);
            mbar_wait_backoff(&empty[stage], phase ^ 1u);
            TPROF(P_WAIT0);
            unsigned char *st = smem + (size_t)stage * SB;
            const int tt = tb + q;
            const bool diag = Cb == R;
            const int jb = (int)(seq % NA);
            int have = -1;
#pragma unroll
            for (int b = 0; b < NA; ++b) have = (b == jb) ? xr_of[b] : have;
            const bool need_xr = !diag && have != R;
            if (need_xr) {
#pragma unroll
              for (int b = 0; b < NA; ++b) xr_of[b] = (b == jb) ? R : xr_of[b];
            }
            const int flags = (tt == t0 ? HDR_FIRST : 0) | (tt == t1 - 1 ? HDR_LAST : 0) | (diag ? HDR_DIAG : 0) |
                              (need_xr ? HDR_XR : 0);
            *reinterpret_cast<int4 *>(st + p.off_hdr) = make_int4(R, Cb, flags, 0);
            // all of the stage's bytes are expected before the X producer
            // (warp 2) may issue its copies: complete_tx never precedes expect_tx
            mbar_arrive_expect_tx(&full[stage], 16384u + (need_xr ? 2u * xblk : xblk));
            mbar_arrive(&hdr_ready[stage]);
            bulk_g2s(st, p.vals + (size_t)tt * 16384u, 16384u, &full[stage], pol_stream);
          }
          __syncwarp();
          ++seq;
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
    TPROF_TILE();
    TPROF_DUMP(5);
    if (lane == 0) {
      // one terminator per splitter group (they take alternate tiles); only
      // the first travels on to the MMA issuer and the epilogue
      for (int e = 0; e < 2; ++e) {
        mbar_wait_backoff(&empty[stage], phase ^ 1u);
        *reinterpret_cast<int4 *>(smem + (size_t)stage * SB + p.off_hdr) = make_int4(0, 0, e ? HDR_TERM2 : HDR_TERM, 0);
        mbar_arrive(&hdr_ready[stage]);
        mbar_arrive(&full[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 2) {
    // ============================ X-block producer ============================
    // The X_C (and, when the B buffer's row changes, X_R) copies of every
    // stage, issued by a second warp: a bulk-copy issue blocks its warp while
    // the copy engine's queue is full, and with one producer warp issuing all
    // three copies per tile the producer was busy 85% of the time at k = 8
    // (role timers) — the ring, not the DRAM, paced the kernel.
    if (lane == 0) {
      const uint64_t pol_keep = p.xpol == 1 ? policy_evict_first() : p.xpol == 2 ? policy_evict_normal() : policy_evict_last();
      const unsigned int xblk = p.xblk;
      int stage = 0;
      uint32_t phase = 0;
      while (true) {
        mbar_wait(&hdr_ready[stage], phase);
        unsigned char *st = smem + (size_t)stage * SB;
        const int4 h = *reinterpret_cast<const int4 *>(st + p.off_hdr);
        if (h.z & HDR_TERM2) break;
        if (!(h.z & HDR_TERM)) {
          bulk_g2s(st + p.off_xc, p.X + (size_t)h.y * xblk, xblk, &full[stage], pol_keep);
          if (h.z & HDR_XR) bulk_g2s(st + p.off_xr, p.X + (size_t)h.x * xblk, xblk, &full[stage], pol_keep);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
  } else if (warp == 1) {
    // ============================== MMA issuer ===============================
    constexpr uint32_t idesc = idesc_tf32<K>();
    const uint32_t b_base = smem_u32(smem + p.off_b);
    uint32_t t = 0;
    TPROF_DECL;
    while (true) {
      const uint32_t j = t % NA, d = t % ND;
      TPROF(P_WORK0);
      mbar_wait(&splitf[j], (t / NA) & 1u);
      TPROF(P_WAIT0);
      tc_fence_after();
      const int4 h = hdrj[j];
      mbar_wait(&d_empty[d], ((t / ND) & 1u) ^ 1u);  // the epilogue has drained D_d (and read meta[d])
      TPROF(P_WAIT1);
      tc_fence_after();
      if (elect_one()) {
        meta[d] = h;
        mbar_arrive(&meta_f[d]);
      }
      __syncwarp();
      if (__any_sync(0xffffffffu, h.z & HDR_TERM)) break;
      const uint32_t bh = b_base + j * C::BBYTES;
      const uint64_t bdesc_hi = sdesc(bh, 128, 2048, 0);
      const uint64_t bdesc_lo = sdesc(bh + (uint32_t)(N / 8) * 2048u, 128, 2048, 0);
      const uint32_t a = t_a + j * 128, dd = t_d + d * N;
      if (elect_one()) {
#ifndef CIM_TC_NO_MMA
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          // K step ks: 8 K-values = two core matrices along K (256 B → +16 in desc units)
          mma_ts(dd, a + ks * 8, bdesc_hi + (uint64_t)(ks * 16), idesc, ks > 0 ? 1u : 0u);
          mma_ts(dd, a + 64 + ks * 8, bdesc_hi + (uint64_t)(ks * 16), idesc, 1u);
          mma_ts(dd, a + ks * 8, bdesc_lo + (uint64_t)(ks * 16), idesc, 1u);
        }
#endif
        tc_commit(&ab_empty[j]);
        tc_commit(&d_full[d]);
      }
      __syncwarp();
      TPROF_TILE();
      ++t;
    }
    TPROF_DUMP(0);
  } else if (warp >= 4 && warp < 12) {
    // =============================== splitters ===============================
    const int grp = (warp - 4) >> 2;  // group 0: tiles 0,2,4,…  group 1: tiles 1,3,5,…
    const int q = warp & 3;           // TMEM lane quarter
    const int m = 32 * q + lane;      // TMEM lane: row m (m < 64) or column m − 64 of the tile
    const int t128 = (warp - 4 - 4 * grp) * 32 + lane;  // 0..127 inside the group
    const uint32_t lane_field = (uint32_t)(32 * q) << 16;
    // column threads: byte offset of (r, c) within row r for r % 8 = 0..7
    const int c = m - 64;
    uint32_t coff[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) coff[s] = (uint32_t)(((((c >> 2) ^ s) & 15) << 4) + (c & 3) * 4);
    uint32_t t = grp;
    int stage = grp % S;
    uint32_t phase = (uint32_t)(grp / S) & 1u;
    TPROF_DECL;
    while (true) {
      TPROF(P_WORK3);
      mbar_wait(&full[stage], phase);
      TPROF(P_WAIT0);
      unsigned char *st = smem + (size_t)stage * SB;
      const int4 h = *reinterpret_cast<const int4 *>(st + p.off_hdr);
      const uint32_t j = t % NA;
      if (h.z & HDR_TERM2) break;
      mbar_wait(&ab_empty[j], ((t / NA) & 1u) ^ 1u);
      TPROF(P_WAIT1);
      if (h.z & HDR_TERM) {
        if (t128 == 0) hdrj[j] = h;
        __syncwarp();
        if (lane == 0) mbar_arrive(&splitf[j]);
        break;
      }
      tc_fence_after();
      const bool diag = h.z & HDR_DIAG;
      const uint32_t a = t_a + j * 128 + lane_field;
#ifndef CIM_TC_NO_ROWS
      if (m < 64) {
#else
      if (false) {
#endif
        // row m: 16 chunks of 4 values, chunk j at (j ^ m%8)·16
        const unsigned char *row = st + m * 256;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int ch = 4 * jj + cc;
            const float4 v = *reinterpret_cast<const float4 *>(row + (((ch ^ (m & 7)) & 15) << 4));
            hi[4 * cc + 0] = __float_as_uint(v.x);
            hi[4 * cc + 1] = __float_as_uint(v.y);
            hi[4 * cc + 2] = __float_as_uint(v.z);
            hi[4 * cc + 3] = __float_as_uint(v.w);
          }
#pragma unroll
          lo16(hi, lo);
          tmem_st16(a + 16 * jj, hi);
          tmem_st16(a + 64 + 16 * jj, lo);
        }
      }
#ifndef CIM_TC_NO_COLS
      else if (!diag) {
#else
      else if (false) {
#endif
        // column c: one word per row; a warp reads 32 consecutive columns of one row
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int rr = 0; rr < 16; ++rr) {
            const int r = 16 * jj + rr;
            hi[rr] = *reinterpret_cast<const uint32_t *>(st + r * 256 + coff[r & 7]);
          }
#pragma unroll
          lo16(hi, lo);
          tmem_st16(a + 16 * jj, hi);
          tmem_st16(a + 64 + 16 * jj, lo);
        }
      }
      TPROF(P_WORK0);
#ifndef CIM_TC_NO_BUILDB
      build_b<K>(reinterpret_cast<const float *>(st + p.off_xc), reinterpret_cast<const float *>(st + p.off_xr),
                 smem + p.off_b + j * C::BBYTES, t128, (h.z & HDR_XR) != 0);
#endif
      if (t128 == 0) hdrj[j] = h;
      // stage consumed: the producer may refill it
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      TPROF(P_WORK1);
      tmem_wait_st();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B stores → async proxy (MMA)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&splitf[j]);
      TPROF(P_WORK2);
      TPROF_TILE();
      t += 2;
      stage += 2;
      if (stage >= S) {
        stage -= S;
        phase ^= 1u;
      }
    }
    if (grp == 0 && (q == 0 || q == 2)) TPROF_DUMP(q == 0 ? 1 : 2);
  } else if (warp >= 12) {
    // =============================== epilogue ================================
    const int q = warp & 3;
    const int m = 32 * q + lane;  // D row
    const uint32_t lane_field = (uint32_t)(32 * q) << 16;
    float *Y = reinterpret_cast<float *>(p.Y);
    const long long ldy = p.ldy;
    float acc[K];
#pragma unroll
    for (int e = 0; e < K; ++e) acc[e] = 0.0f;
    // bulk Y reductions: warps 12-13 (direct) and 14-15 (transposed) each
    // stage a 64 × K block, their lane 0 of warp 12 / 14 issues it
    const bool bulk = p.off_ebuf != 0;
    const bool issuer = (q == 0 || q == 2) && lane == 0;
    float *ebuf = reinterpret_cast<float *>(smem + p.off_ebuf);
    int eb_dir = 0, eb_tr = 0;
    uint32_t t = 0;
    TPROF_DECL;
    while (true) {
      const uint32_t d = t % ND;
      const uint32_t ph = (t / ND) & 1u;
      TPROF(P_WORK0);
      mbar_wait(&meta_f[d], ph);
      TPROF(P_WAIT0);
      const int4 h = meta[d];
      if (h.z & HDR_TERM) {
        if (bulk && issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        break;
      }
      mbar_wait(&d_full[d], ph);
      TPROF(P_WAIT1);
      tc_fence_after();
      const bool diag = h.z & HDR_DIAG;
      const uint32_t dcol = t_d + d * N + lane_field;
      if (q < 2) {
        // direct product row m of the tile: D columns 0..K-1, summed over the unit
        if (h.z & HDR_FIRST) {
#pragma unroll
          for (int e = 0; e < K; ++e) acc[e] = 0.0f;
        }
#pragma unroll
        for (int cb = 0; cb < K / 8; ++cb) {
          uint32_t r8[8];
          tmem_ld8(dcol + 8 * cb, r8);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[8 * cb + e] += __uint_as_float(r8[e]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&d_empty[d]);
#ifndef CIM_TC_NO_RED
        if (h.z & HDR_LAST) {
#else
        if (false) {
#endif
          if (bulk) {
            float *eb = ebuf + (size_t)eb_dir * 64 * K;
            if (issuer) bulk_wait_read_le1();
            named_bar_sync(1, 64);
#pragma unroll
            for (int e = 0; e < K; e += 4)
              *reinterpret_cast<float4 *>(eb + m * K + e) = make_float4(acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_bar_sync(1, 64);
            if (issuer) bulk_red_f32(Y + (long long)h.x * kBlock * K, eb, 64u * K * 4u, p.ypol);
            eb_dir ^= 1;
          } else {
            float *yp = Y + ((long long)h.x * kBlock + m) * ldy;
#pragma unroll
            for (int e = 0; e < K; e += 4) red_add_v4(yp + e, acc[e], acc[e + 1], acc[e + 2], acc[e + 3]);
          }
        }
      } else {
        // transposed product column m − 64 of the tile: D columns K..2K-1 → Y_C
        if (!diag) {
          float *eb = ebuf + (size_t)(2 + eb_tr) * 64 * K;
          if (bulk) {
            if (issuer) bulk_wait_read_le1();
            named_bar_sync(2, 64);
          }
          float *yp = Y + ((long long)h.y * kBlock + (m - 64)) * ldy;
#pragma unroll
          for (int cb = 0; cb < K / 8; ++cb) {
            uint32_t r8[8];
            tmem_ld8(dcol + K + 8 * cb, r8);
            tmem_wait_ld();
#ifndef CIM_TC_NO_RED
            if (bulk) {
              float *row = eb + (m - 64) * K + 8 * cb;
              *reinterpret_cast<float4 *>(row) = make_float4(__uint_as_float(r8[0]), __uint_as_float(r8[1]),
                                                             __uint_as_float(r8[2]), __uint_as_float(r8[3]));
              *reinterpret_cast<float4 *>(row + 4) = make_float4(__uint_as_float(r8[4]), __uint_as_float(r8[5]),
                                                                 __uint_as_float(r8[6]), __uint_as_float(r8[7]));
            } else {
              red_add_v4(yp + 8 * cb, __uint_as_float(r8[0]), __uint_as_float(r8[1]), __uint_as_float(r8[2]),
                         __uint_as_float(r8[3]));
              red_add_v4(yp + 8 * cb + 4, __uint_as_float(r8[4]), __uint_as_float(r8[5]), __uint_as_float(r8[6]),
                         __uint_as_float(r8[7]));
            }
#endif
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[d]);
          if (bulk) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            named_bar_sync(2, 64);
            if (issuer) bulk_red_f32(Y + (long long)h.y * kBlock * K, eb, 64u * K * 4u, p.ypol);
            eb_tr ^= 1;
          }
        } else {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&d_empty[d]);
        }
      }
      TPROF_TILE();
      ++t;
    }
    if (q == 0 || q == 2) TPROF_DUMP(q == 0 ? 3 : 4);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(0u));
  }
}

// ----------------------------------------------------------------------------
// host launcher
// ----------------------------------------------------------------------------
template <int K>
int launch(const cim_half_tiles *H, const void *X, void *Y, long long ldy, cudaStream_t stream, int sms,
           unsigned int *counter) {
  using Cf = Cfg<K>;
  static std::mutex mu;
  static int attr_mask = 0;
  const unsigned int xblk = 64u * K * 4u;
  TcParams p{};
  p.off_xc = 16384;
  p.off_xr = p.off_xc + xblk;
  p.off_hdr = p.off_xr + xblk;
  p.stage_bytes = (p.off_hdr + 16 + 127) & ~127u;
  const size_t fixed = (size_t)Cf::NA * Cf::BBYTES + 16 * (Cf::NA + Cf::ND) + 8 * (3 * Cf::NA + 3 * Cf::ND) + 64 + 8 * 8;
  const size_t budget = 227 * 1024 - 1024;  // minus the manual 1 KB alignment slack
  // bulk Y reductions need dense Y rows and 4 staging blocks; keep them unless
  // they would cost ring stages below 4
  const size_t ebytes = 4 * (size_t)64 * K * 4;
  const int S_scalar = std::min(8, (int)((budget - fixed - 8 * 2 * 8) / p.stage_bytes)) & ~1;
  const int S_bulk = std::min(8, (int)((budget - fixed - ebytes - 8 * 2 * 8) / p.stage_bytes)) & ~1;
  const bool use_bulk = ldy == K && (S_bulk >= 4 || S_bulk == S_scalar) && !std::getenv("CIM_TC_SCALAR_RED");
  int S = use_bulk ? S_bulk : S_scalar;
  // The two consumer groups take alternate tiles; with an odd ring a stage
  // would alternate between the groups, and a group running ahead could
  // pass a parity wait on a stage one fill behind (phase aliasing).  An even
  // ring keeps every stage with one group.
  S &= ~1;
  if (S < 2) return set_error(CIM_EUNSUPPORTED, "tensor-core path: k too large for shared memory");
  p.stages = (unsigned)S;
  size_t off = (size_t)S * p.stage_bytes;
  p.off_b = (unsigned int)off;
  off += (size_t)Cf::NA * Cf::BBYTES;
  p.off_hdrj = (unsigned int)off;
  off += 16 * Cf::NA;
  p.off_meta = (unsigned int)off;
  off += 16 * Cf::ND;
  p.off_bars = (unsigned int)off;
  off += 8 * (3 * (size_t)S + 2 * Cf::NA + 3 * Cf::ND);
  off = (off + 15) & ~size_t(15);
  p.off_tmem = (unsigned int)off;
  off += 16;
  off = (off + 127) & ~size_t(127);
  p.off_ebuf = use_bulk ? (unsigned int)off : 0u;
  if (use_bulk) off += ebytes;
  const size_t smem = off + 1024;
  if (smem > 227 * 1024) return set_error(CIM_EUNSUPPORTED, "tensor-core path: shared-memory plan too large");

  auto kern = sym_spmm_tc_kernel<K>;
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
  p.xpol = std::getenv("CIM_TC_XPOL") ? std::atoi(std::getenv("CIM_TC_XPOL")) : 0;
  p.ypol = std::getenv("CIM_TC_YPOL") ? std::atoi(std::getenv("CIM_TC_YPOL")) : 0;
  const long long grid = std::min<long long>(sms, H->n_units);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("counter memset: ") + cudaGetErrorString(e));
  kern<<<(unsigned int)grid, 512, smem, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sym_spmm_tc launch: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace tc

// Entry used by cim_sym_spmm for CIM_LAYOUT_TC tiles (k a multiple of 8, ≤ 64).
int sym_spmm_tc_dispatch(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy, cudaStream_t stream,
                         int sms, unsigned int *counter) {
  switch (k) {
    case 8: return tc::launch<8>(H, X, Y, ldy, stream, sms, counter);
    case 16: return tc::launch<16>(H, X, Y, ldy, stream, sms, counter);
    case 24: return tc::launch<24>(H, X, Y, ldy, stream, sms, counter);
    case 32: return tc::launch<32>(H, X, Y, ldy, stream, sms, counter);
    case 40: return tc::launch<40>(H, X, Y, ldy, stream, sms, counter);
    case 48: return tc::launch<48>(H, X, Y, ldy, stream, sms, counter);
    case 56: return tc::launch<56>(H, X, Y, ldy, stream, sms, counter);
    case 64: return tc::launch<64>(H, X, Y, ldy, stream, sms, counter);
  }
  return set_error(CIM_EUNSUPPORTED, "tensor-core path supports k in 8N, k <= 64");
}

}  // namespace cim

// Role timers of the last CIM_TC_PROF launch (tools/tc_profile.py): copies
// [ctas][5 roles][16 slots] cycle counts; 0 when profiling is not compiled in.
extern "C" CIM_API int cim_tc_profile_read(unsigned long long *host_out, int max_ctas) {
#ifdef CIM_TC_PROF
  const int n = max_ctas < cim::tc::kProfCtas ? max_ctas : cim::tc::kProfCtas;
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(host_out, cim::tc::g_prof, (size_t)n * cim::tc::kProfRoles * cim::tc::P_SLOTS * 8);
  return n;
#else
  (void)host_out;
  (void)max_ctas;
  return 0;
#endif
}
