// Shared device helpers: mbarrier / bulk-copy PTX wrappers, the reference
// value hashes, and the fragment-layout index map.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cim {

constexpr int kBlock = 64;          // tile edge
constexpr int kTileElems = 4096;    // 64 × 64
constexpr int kGroupThreads = 128;  // consumer threads per group = micro-blocks per tile
constexpr int kSpPtrStride = 72;    // uint16 row / column pointers per sparse tile (65 used; 144 B, 16-B aligned)

// ---------------------------------------------------------------------------
// Fragment layout v1 (include/cim_b200.h): micro-block mb ∈ [0,128) owns rows
// rg + 8i (i < 8) and columns cg + 16j (j < 4).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int frag_rg(int mb) { return (mb & 31) >> 2; }
__host__ __device__ __forceinline__ int frag_cg(int mb) { return ((mb >> 5) << 2) | (mb & 3); }

// Element index inside a tile's fragment-ordered storage → (row, col).
template <typename T>
__host__ __device__ __forceinline__ void frag_index_to_rc(int idx, int &row, int &col) {
  if constexpr (sizeof(T) == 4) {
    const int j = idx & 3, mb = (idx >> 2) & 127, i = idx >> 9;
    row = frag_rg(mb) + 8 * i;
    col = frag_cg(mb) + 16 * j;
  } else {
    const int jj = idx & 1, mb = (idx >> 1) & 127, h = (idx >> 8) & 1, i = idx >> 9;
    row = frag_rg(mb) + 8 * i;
    col = frag_cg(mb) + 16 * (2 * h + jj);
  }
}

// TC layout (CIM_LAYOUT_TC, f32): row-major rows of 256 B whose 16-byte
// chunks are XOR-swizzled by the row: byte(r,c) = r·256 + ((c/4 ^ r%8)·16) +
// (c%4)·4.  Row r read as 16-byte chunks by 32 threads (one row each) and
// one row read as words by 32 threads (one column each) are both
// bank-conflict-free — the two access patterns of the split-TF32 kernel.
__host__ __device__ __forceinline__ int tc_byte(int row, int col) {
  return row * 256 + ((((col >> 2) ^ (row & 7)) & 15) << 4) + (col & 3) * 4;
}
__host__ __device__ __forceinline__ void tc_index_to_rc(int idx, int &row, int &col) {
  row = idx >> 6;
  const int pc = (idx >> 2) & 15;
  col = ((pc ^ (row & 7)) << 2) | (idx & 3);
}

template <typename T>
__host__ __device__ __forceinline__ void layout_index_to_rc(int layout, int idx, int &row, int &col) {
  if (layout == 1)  // the same element map for f32 (16-byte chunks) and f64 (32-byte chunks)
    tc_index_to_rc(idx, row, col);
  else
    frag_index_to_rc<T>(idx, row, col);
}

// ---------------------------------------------------------------------------
// Reference value hashes, bit-exact twins of pipeline.py:199-263.
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // pipeline.py:199
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;    // pipeline.py:200
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;    // pipeline.py:201

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // pipeline.py:204-209
  z += kGolden;
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}

// top 53 bits → [0,1) → [-1,1), rounded once to f32 (pipeline.py:212-215).
// The reference's f64 value m·2⁻⁵³·2 − 1 (m = u >> 11) is exactly
// (m − 2⁵²)·2⁻⁵², so one int64 → f32 round-to-nearest conversion and an exact
// power-of-two scale give the same bits without f64 arithmetic.
__host__ __device__ __forceinline__ float to_unit(uint64_t u) {
  const long long s = static_cast<long long>(u >> 11) - (1ll << 52);
  return static_cast<float>(s) * 0x1p-52f;
}

__host__ __device__ __forceinline__ float h_value(uint64_t i, uint64_t j, uint64_t seed) {  // :218-221
  return to_unit(mix64(mix64(i ^ j) ^ seed));
}

__host__ __device__ __forceinline__ float op_value(uint64_t i, uint64_t j, uint64_t k, uint64_t seed) {  // :224-232
  const uint64_t lo = i < j ? i : j, hi = i < j ? j : i;
  uint64_t u = mix64(lo + kGolden * hi);
  u = mix64(u ^ ((k + 1ull) * kMix1));
  return to_unit(mix64(u ^ seed));
}

__host__ __device__ __forceinline__ float value_of_kind(int kind, uint64_t i, uint64_t j, uint64_t seed, int op_k) {
  if (kind == 0) return h_value(i, j, seed);
  if (kind == 1) return op_value(i, j, static_cast<uint64_t>(op_k), seed);
  return i == j ? 1.0f : 0.0f;
}

// ---------------------------------------------------------------------------
// PTX wrappers (sm_90+ mbarrier / cp.async.bulk; used on sm_100a)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}

// try_wait with a suspend-time hint (ns): the thread sleeps in hardware until
// the phase completes or the hint expires.
__device__ __forceinline__ bool mbar_try_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity), "r"(ns)
      : "memory");
  return ok != 0;
}

// Producer-side wait: it is almost always the ring that is full (consumers are
// the slower side), so back off instead of spinning — a spinning producer lane
// steals issue slots from the consumer warps on its SM sub-partition.
__device__ __forceinline__ void mbar_wait_backoff(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait_hint(a, parity, 0x4000u)) {
    __nanosleep(128);
  }
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// One-instruction bulk copy global → shared, completing on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Warpgroup register reallocation (all 128 threads of the warpgroup execute it).
template <int N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Fire-and-forget global reductions (no return value → REDG).
__device__ __forceinline__ void red_add(float *p, float a) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}
__device__ __forceinline__ void red_add(double *p, double a) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(a) : "memory");
}
__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d, uint64_t policy) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void red_add_v2(float *p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}

}  // namespace cim
