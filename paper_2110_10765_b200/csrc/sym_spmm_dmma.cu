// FP64 tensor-core (DMMA) half-stored symmetric SpMM
//   Y = U·X + U_offᵀ·X          (f64 tiles and vectors, k ∈ {8, 16, 24, 32})
//
// The FP64 path of the tile layout CIM_LAYOUT_TC (row-major tiles whose
// 4-element chunks are XOR-swizzled by row % 8 — 32-byte chunks for f64).
// mma.sync m8n8k4 f64 (SASS DMMA.8x8x4) does 256 FMAs per warp instruction
// against 32 for DFMA at the same FP64 peak on B200 (tools/dmma_probe.cu:
// 37.1 TFLOP/s vs the measured DFMA 34.1), so the kernel is no longer bound
// by issue slots and register-resident accumulators: the DFMA kernel ran the
// compute-bound widths at ~42% of the FP64 pipe, shared-memory bound
// (L1/TEX 94%: each warpgroup re-read the 32 KB tile per 4 vectors).
//
// Per stored tile (T, 64 × 64) and 8·NB vectors, consumer warp w (0..3):
//   direct      rows 16w..16w+15:  D[r][v] += Σ_c T[r][c] · X_C[c][v]
//               A = T (8×4 fragments, row-major), B = X_C (4×8, col-major)
//   transposed  cols 16w..16w+15:  E[c][v]  = Σ_r T[r][c] · X_R[r][v]
//               A = Tᵀ (the same smem tile read transposed), B = X_R
// Each tile element is read from shared memory once per product for all k
// vectors (the A fragment is reused across the NB column blocks).  D stays
// in registers across the tiles of one block row (flushed with red.global
// when the row changes), E is reduced into Y_C per tile.
//
// Roles (one CTA per SM, persistent): warp 8 is the producer (work units by
// ticket, bulk copies of tile / X_C / X_R into an S-stage ring); warps 0-3
// and 4-7 are two consumer groups taking alternate tiles.
// The reference reaches this arithmetic only as its per-pair contraction
// kernels (pipeline.py:461-531) over the COO of _collect_pairs (:428-458).
#include <algorithm>
#include <cstdlib>
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cuda.h>  // CUtensorMap and its enums (the encoder comes through cudaGetDriverEntryPoint)
#include <cstdio>
#include <mutex>
#include <string>

#include "cim_b200.h"
#include "common.cuh"
#include "host_util.h"

#ifndef CIM_DMMA_TMA_X
#define CIM_DMMA_TMA_X 1  // k = 16 / 32: X blocks by TMA tensor copies with the 128-byte swizzle
#endif

namespace cim {
namespace dmma {

enum : int { HDR_DIAG = 4, HDR_TERM = 8 };

struct DmParams {
  const int4 *units;
  const int2 *tile_rc;
  const unsigned char *vals;
  const unsigned char *X;
  double *Y;
  unsigned int *counter;
  long long n_units;
  long long ldy;
  unsigned int stages, stage_bytes, xblk;
  unsigned int off_xc, off_xr, off_hdr, off_bars;
  unsigned int off_ebuf;  // 2 groups × 2 staging blocks of 64·K doubles (bulk flush), 0 = scalar reds
  alignas(64) CUtensorMap tmx;  // k ∈ {16, 32}: X as a 2-D tensor (K × n_pad doubles), 16 × 64 boxes, 128-B swizzle
};

// X blocks through TMA with the 128-byte swizzle (k = 16, 32): the m8n8k4 B
// fragment reads rows 4kb + q4 of X at one column, and with 128-byte (or
// 256-byte) rows every X row starts on the same bank — 8 wavefronts per
// 8-byte fragment load from a row-major stage.  The swizzle stores the
// 16-byte chunk j of row r of each 16-column box at chunk j ^ (r % 8): the
// four rows land on different banks (4 wavefronts, the two lanes of a bank
// pair read different rows).
template <int K>
struct XSwz {
  static constexpr bool on = CIM_DMMA_TMA_X && (K == 16 || K == 32);
};

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

constexpr int kTileBytes = 4096 * 8;
constexpr int kThreads = 288;  // 2 consumer groups × 4 warps + 1 producer warp

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// One 64 × K block of partial sums → Y rows Rb·64 … Rb·64+63 (dense, ldy = K)
// with one bulk reduction: UBLKRED.ADD.F64 does the read-modify-write of the
// whole contiguous 64·K·8-byte block at the L2, where scalar red.global.add.f64
// (there is no vector form for f64) needed 64·K separate atomic operations.
__device__ __forceinline__ void bulk_red_f64(double *dst, const void *src, unsigned bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

template <int K>
__global__ void __launch_bounds__(kThreads, 1) sym_spmm_dmma_kernel(const __grid_constant__ DmParams p) {
  constexpr int NB = K / 8;  // 8-vector column blocks
  constexpr bool SWZ = XSwz<K>::on;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // the 128-byte swizzle needs 1024-byte aligned boxes (1 KB of slack is allocated)
  unsigned char *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int S = (int)p.stages;
  const unsigned SB = p.stage_bytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.off_bars), *empty = full + S;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 8) {
    // ================================ producer ================================
    const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();
    const unsigned xblk = p.xblk;
    int stage = 0;
    uint32_t phase = 0;
    // work-unit metadata software-pipelined (see the tcgen05 kernel's producer)
    const long long n_units = p.n_units;
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
            mbar_wait_backoff(&empty[stage], phase ^ 1u);
            unsigned char *st = smem + (size_t)stage * SB;
            const bool diag = Cb == R;
            *reinterpret_cast<int4 *>(smem + p.off_hdr + 16 * stage) = make_int4(R, Cb, diag ? HDR_DIAG : 0, 0);
            mbar_arrive_expect_tx(&full[stage], (unsigned)kTileBytes + (diag ? xblk : 2u * xblk));
            bulk_g2s(st, p.vals + (size_t)(tb + q) * kTileBytes, kTileBytes, &full[stage], pol_stream);
            if constexpr (SWZ) {
#pragma unroll
              for (int hb = 0; hb < K / 16; ++hb) {
                tma_load_2d(st + p.off_xc + hb * 8192, &p.tmx, 16 * hb, Cb * kBlock, &full[stage], pol_keep);
                if (!diag) tma_load_2d(st + p.off_xr + hb * 8192, &p.tmx, 16 * hb, R * kBlock, &full[stage], pol_keep);
              }
            } else {
              bulk_g2s(st + p.off_xc, p.X + (size_t)Cb * xblk, xblk, &full[stage], pol_keep);
              if (!diag) bulk_g2s(st + p.off_xr, p.X + (size_t)R * xblk, xblk, &full[stage], pol_keep);
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
    if (lane == 0)
      for (int e = 0; e < 2; ++e) {  // one terminator per consumer group
        mbar_wait_backoff(&empty[stage], phase ^ 1u);
        *reinterpret_cast<int4 *>(smem + p.off_hdr + 16 * stage) = make_int4(0, 0, HDR_TERM, 0);
        mbar_arrive(&full[stage]);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
    return;
  }
  if (warp > 8) return;

  // ============================== consumers ==============================
  const int grp = warp >> 2, w = warp & 3;
  const int g = lane >> 2, q4 = lane & 3;  // fragment row / column group of this lane
  const long long ldy = p.ldy;
  // direct A: row 16w + 8rb + g, chunk kb swizzled by g (= row % 8)
  const unsigned a_dir = (unsigned)((16 * w + g) * 512 + q4 * 8 + (g << 5));
  // transposed A: T[4kb + q4][16w + 8cb + g]; row % 8 = 4(kb&1) + q4, chunk 4w + 2cb + g/4
  unsigned a_tr[2][2];
#pragma unroll
  for (int cb = 0; cb < 2; ++cb)
#pragma unroll
    for (int par = 0; par < 2; ++par) {
      const int chunk = 4 * w + 2 * cb + (g >> 2);
      a_tr[cb][par] = (unsigned)(q4 * 512 + ((chunk ^ (4 * par + q4)) << 5) + (g & 3) * 8);
    }
  // B fragments: X[4kb + q4][8nb + g] — row-major stage, or (SWZ) box nb/2,
  // row r = 4kb + q4 at r·128, chunk (4(nb&1) + g/2) ^ (r % 8), half g&1
  const unsigned b_off = (unsigned)(q4 * K * 8 + g * 8);
  unsigned b_swz[2][NB];
#pragma unroll
  for (int par = 0; par < 2; ++par)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb)
      b_swz[par][nb] = (unsigned)((nb >> 1) * 8192 + q4 * 128 + (((4 * (nb & 1) + (g >> 1)) ^ (4 * par + q4)) << 4) +
                                  (g & 1) * 8);

  double acc[2][NB][2];
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
  int curR = -1;
  // partial sums of one 64-row block (fragments f[2][NB][2] of rows / columns
  // 16w + 8·blk + g) → Y block row Rb
  const bool bulk = p.off_ebuf != 0;
  const bool issuer = w == 0 && lane == 0;
  int eb = 0;  // staging buffer of this group's next bulk flush
  auto flush = [&](int Rb, double (&f)[2][NB][2]) {
    if (bulk) {
      double *ebuf = reinterpret_cast<double *>(smem + p.off_ebuf + (size_t)(2 * grp + eb) * 64 * K * 8);
      if (issuer) bulk_wait_read_le1();  // the flush that last used this buffer has read it
      named_bar_sync(1 + grp, 128);
#pragma unroll
      for (int blk = 0; blk < 2; ++blk)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
          *reinterpret_cast<double2 *>(ebuf + (16 * w + 8 * blk + g) * K + 8 * nb + 2 * q4) =
              make_double2(f[blk][nb][0], f[blk][nb][1]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      named_bar_sync(1 + grp, 128);
      if (issuer) bulk_red_f64(p.Y + (long long)Rb * kBlock * K, ebuf, 64u * K * 8u);
      eb ^= 1;
    } else {
#pragma unroll
      for (int blk = 0; blk < 2; ++blk) {
        double *y = p.Y + ((long long)Rb * kBlock + 16 * w + 8 * blk + g) * ldy + 2 * q4;
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) {
          red_add(y + 8 * nb, f[blk][nb][0]);
          red_add(y + 8 * nb + 1, f[blk][nb][1]);
        }
      }
    }
  };
  auto flush_direct = [&](int R) {
    flush(R, acc);
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int nb = 0; nb < NB; ++nb) acc[rb][nb][0] = acc[rb][nb][1] = 0.0;
  };

  int stage = grp % S;
  uint32_t phase = (uint32_t)(grp / S) & 1u;
  while (true) {
    mbar_wait(&full[stage], phase);
    const unsigned char *st = smem + (size_t)stage * SB;
    const int4 h = *reinterpret_cast<const int4 *>(smem + p.off_hdr + 16 * stage);
    if (h.z & HDR_TERM) {
      if (curR >= 0) flush_direct(curR);
      if (bulk && issuer) bulk_wait_all();
      break;
    }
    if (h.x != curR) {
      if (curR >= 0) flush_direct(curR);
      curR = h.x;
    }
    const unsigned char *Xc = st + p.off_xc, *Xr = st + p.off_xr;
    // ---- direct: acc[rb][nb] += T[rows] · X_C ----
#pragma unroll 4
    for (int kb = 0; kb < 16; ++kb) {
      double b[NB];
#pragma unroll
      for (int nb = 0; nb < NB; ++nb)
          b[nb] = SWZ ? *reinterpret_cast<const double *>(Xc + b_swz[kb & 1][nb] + kb * 512)
                      : *reinterpret_cast<const double *>(Xc + b_off + kb * 32 * K + nb * 64);
#pragma unroll
      for (int rb = 0; rb < 2; ++rb) {
        const double a = *reinterpret_cast<const double *>(st + ((a_dir + rb * 8 * 512) ^ (unsigned)(kb << 5)));
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) dmma(acc[rb][nb][0], acc[rb][nb][1], a, b[nb]);
      }
    }
    const bool diag = h.z & HDR_DIAG;
    if (!diag) {
      // ---- transposed: E[cb][nb] = Tᵀ[cols] · X_R ----
      double e[2][NB][2];
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int nb = 0; nb < NB; ++nb) e[cb][nb][0] = e[cb][nb][1] = 0.0;
#pragma unroll 4
      for (int kb = 0; kb < 16; ++kb) {
        double b[NB];
#pragma unroll
        for (int nb = 0; nb < NB; ++nb)
          b[nb] = SWZ ? *reinterpret_cast<const double *>(Xr + b_swz[kb & 1][nb] + kb * 512)
                      : *reinterpret_cast<const double *>(Xr + b_off + kb * 32 * K + nb * 64);
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          const double a = *reinterpret_cast<const double *>(st + kb * 2048 + a_tr[cb][kb & 1]);
#pragma unroll
          for (int nb = 0; nb < NB; ++nb) dmma(e[cb][nb][0], e[cb][nb][1], a, b[nb]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      flush(h.y, e);
    } else {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
    stage += 2;
    if (stage >= S) {
      stage -= S;
      phase ^= 1u;
    }
  }
}

template <int K>
int launch(const cim_half_tiles *H, const void *X, void *Y, long long ldy, cudaStream_t stream, int sms,
           unsigned int *counter) {
  static std::mutex mu;
  static int attr_mask = 0;
  const unsigned xblk = 64u * K * 8u;
  DmParams p{};
  p.off_xc = kTileBytes;
  p.off_xr = p.off_xc + xblk;
  p.stage_bytes = kTileBytes + 2 * xblk;  // a multiple of 1024 (swizzled TMA boxes stay aligned)
  // stages, then the bulk-flush staging blocks, the stage headers and the barriers
  const size_t budget = 227 * 1024 - 1024 - 32 * 8;
  // bulk flushes need dense Y rows and 2 groups × 2 staging blocks; keep them
  // unless they would cost ring stages
  const size_t ebytes = 4 * (size_t)64 * K * 8;
  const int S_scalar = std::min(8, (int)(budget / p.stage_bytes)) & ~1;
  const int S_bulk = std::min(8, (int)((budget - ebytes) / p.stage_bytes)) & ~1;
  const bool use_bulk = ldy == K && (S_bulk >= 4 || S_bulk == S_scalar) && !std::getenv("CIM_DMMA_SCALAR_RED");
  int S = use_bulk ? S_bulk : S_scalar;
  // The two consumer groups take alternate tiles; with an odd ring a stage
  // would alternate between the groups, and a group running ahead could
  // pass a parity wait on a stage one fill behind (phase aliasing).  An even
  // ring keeps every stage with one group.
  S &= ~1;
  if (S < 2) return set_error(CIM_EUNSUPPORTED, "DMMA path: k too large for shared memory");
  p.stages = (unsigned)S;
  p.off_ebuf = use_bulk ? (unsigned)S * p.stage_bytes : 0u;
  p.off_hdr = (unsigned)((size_t)S * p.stage_bytes + (use_bulk ? ebytes : 0));
  p.off_bars = p.off_hdr + 16u * (unsigned)S;
  const size_t smem = p.off_bars + 16 * (size_t)S + 1024;
  if constexpr (XSwz<K>::on) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
          return set_error(CIM_ECUDA, "cuTensorMapEncodeTiled not available");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
      }
    }
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)((H->n + kBlock - 1) / kBlock * kBlock)};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 8};
    const cuuint32_t box[2] = {16, (cuuint32_t)kBlock}, estr[2] = {1, 1};
    const CUresult r = encode(&p.tmx, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void *>(X), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_error(CIM_EINVAL, "cuTensorMapEncodeTiled(X) failed (alignment?)");
  }
  auto kern = sym_spmm_dmma_kernel<K>;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(attr_mask & (1 << dev))) {
      const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess)
        return set_error(CIM_ECUDA, std::string("cudaFuncSetAttribute(dmma): ") + cudaGetErrorString(e));
      attr_mask |= (1 << dev);
    }
  }
  p.units = reinterpret_cast<const int4 *>(H->units);
  p.tile_rc = reinterpret_cast<const int2 *>(H->tile_rc);
  p.vals = reinterpret_cast<const unsigned char *>(H->vals);
  p.X = reinterpret_cast<const unsigned char *>(X);
  p.Y = reinterpret_cast<double *>(Y);
  p.counter = counter;
  p.n_units = H->n_units;
  p.ldy = ldy;
  p.xblk = xblk;
  const long long grid = std::min<long long>(sms, H->n_units);
  cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("counter memset: ") + cudaGetErrorString(e));
  kern<<<(unsigned)grid, kThreads, smem, stream>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(CIM_ECUDA, std::string("sym_spmm_dmma launch: ") + cudaGetErrorString(e));
  return CIM_OK;
}

}  // namespace dmma

// Entry used by cim_sym_spmm for f64 CIM_LAYOUT_TC tiles.
int sym_spmm_dmma_dispatch(const cim_half_tiles *H, const void *X, void *Y, int k, long long ldy,
                           cudaStream_t stream, int sms, unsigned int *counter) {
  switch (k) {
    case 8: return dmma::launch<8>(H, X, Y, ldy, stream, sms, counter);
    case 16: return dmma::launch<16>(H, X, Y, ldy, stream, sms, counter);
    case 24: return dmma::launch<24>(H, X, Y, ldy, stream, sms, counter);
    case 32: return dmma::launch<32>(H, X, Y, ldy, stream, sms, counter);
  }
  return set_error(CIM_EUNSUPPORTED, "f64 tensor-core path supports k in {8, 16, 24, 32}");
}

}  // namespace cim
