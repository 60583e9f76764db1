/*
 * TEST INFRASTRUCTURE — CPU restatement of the half-stored symmetric SpMM.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * --impl reference) load this library, as the checker / CPU baseline.  The
 * product (paper_2110_10765_b200/) never links or calls it.
 *
 * What it restates from the reference package cimotifs:
 *   - value hash h(i XOR j; seed) = f32(to_unit(mix64(mix64(i^j) ^ seed)))
 *     (pkg/src/cimotifs/pipeline.py:204-221, numpy twin :235-249);
 *   - the reference's parallel merge discipline for a multi-output
 *     accumulation: numba prange over work items with a privatized output
 *     array merged after the loop (_contract_array_clause, pipeline.py:461-476;
 *     _reduce_array_clause, reduce.py:88-117), here OpenMP over block rows
 *     with per-thread private Y for the scattered Hᵀ·X part;
 *   - f32 accumulation without FMA contraction (numba fastmath off), the
 *     reference's arithmetic for f32 inputs; an f64-accumulating variant is the
 *     parity oracle.
 * The SpMM itself has no reference implementation; its
 * definition is Y[R] += T·X[C], Y[C] += Tᵀ·X[R] for stored tiles R < C.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define B 64

static inline uint64_t mix64(uint64_t z) { /* pipeline.py:204-209 */
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline float h_value(uint64_t i, uint64_t j, uint64_t seed) { /* pipeline.py:212-221 */
  uint64_t u = mix64(mix64(i ^ j) ^ seed);
  double d = (double)(u >> 11) * (1.0 / 9007199254740992.0);
  d = d * 2.0 - 1.0;
  return (float)d;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Row-major dense tile values h(i XOR j; seed) for each (R, C) (0 outside n). */
void oracle_fill_h(const int32_t *rc, int64_t n_tiles, int64_t n, uint64_t seed, float *tiles, int threads) {
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int64_t r0 = (int64_t)rc[2 * t] * B, c0 = (int64_t)rc[2 * t + 1] * B;
    float *T = tiles + t * B * B;
    for (int a = 0; a < B; ++a)
      for (int b = 0; b < B; ++b) {
        const int64_t i = r0 + a, j = c0 + b;
        T[a * B + b] = (i < n && j < n) ? h_value((uint64_t)i, (uint64_t)j, seed) : 0.0f;
      }
  }
}

/*
 * f32 SpMM over tiles [0, n_tiles) (sorted by R).  X: (rows, k) row-major
 * indexed by global row; Y likewise (zeroed here).  `col_map` maps a block
 * index to a compact slot for the per-thread private transposed buffers
 * (slots in [0, n_slots)), so a bounded sample of a huge matrix needs only
 * n_slots·64·k floats per thread.  Returns 0, or 1 on allocation failure.
 */
int oracle_sym_spmm_f32(int64_t n_tiles, const int32_t *rc, const float *tiles, const float *X, int k, float *Y,
                        int64_t y_rows, const int32_t *col_map, int64_t n_slots, const int32_t *slot_block,
                        int threads) {
  if (threads < 1) threads = 1;
  memset(Y, 0, (size_t)y_rows * k * sizeof(float));
  /* block-row starts */
  int64_t n_rows = 0;
  int64_t *row_start = (int64_t *)malloc(sizeof(int64_t) * (n_tiles + 1));
  if (!row_start) return 1;
  for (int64_t t = 0; t < n_tiles; ++t)
    if (t == 0 || rc[2 * t] != rc[2 * (t - 1)]) row_start[n_rows++] = t;
  row_start[n_rows] = n_tiles;
  const size_t priv_elems = (size_t)n_slots * B * k;
  float *priv = (float *)calloc((size_t)threads * priv_elems, sizeof(float));
  if (!priv) {
    free(row_start);
    return 1;
  }
#pragma omp parallel num_threads(threads)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    float *P = priv + (size_t)tid * priv_elems;
    float acc[B * 64];
#pragma omp for schedule(dynamic, 4)
    for (int64_t r = 0; r < n_rows; ++r) {
      const int64_t R = rc[2 * row_start[r]];
      memset(acc, 0, sizeof(float) * B * k);
      const float *XR = X + R * B * k;
      for (int64_t t = row_start[r]; t < row_start[r + 1]; ++t) {
        const int64_t C = rc[2 * t + 1];
        const float *T = tiles + t * B * B;
        const float *XC = X + C * B * k;
        /* direct: acc[a][v] += T[a][b] * XC[b][v] */
        for (int a = 0; a < B; ++a) {
          float *ya = acc + a * k;
          for (int b = 0; b < B; ++b) {
            const float tv = T[a * B + b];
            const float *xb = XC + b * k;
            for (int v = 0; v < k; ++v) {
              float prod = tv * xb[v];
              ya[v] = ya[v] + prod;
            }
          }
        }
        if (C != R) {
          /* transposed: P[slot(C)][b][v] += T[a][b] * XR[a][v] */
          float *pc = P + (size_t)col_map[C] * B * k;
          for (int a = 0; a < B; ++a) {
            const float *xa = XR + a * k;
            for (int b = 0; b < B; ++b) {
              const float tv = T[a * B + b];
              float *yb = pc + b * k;
              for (int v = 0; v < k; ++v) {
                float prod = tv * xa[v];
                yb[v] = yb[v] + prod;
              }
            }
          }
        }
      }
      float *YR = Y + R * B * k;
      for (int e = 0; e < B * k; ++e) YR[e] += acc[e];
    }
    /* merge of the privatized arrays (the array_clause `a += part` step) */
#pragma omp barrier
#pragma omp for schedule(static)
    for (int64_t s = 0; s < n_slots; ++s) {
      float *YC = Y + (int64_t)slot_block[s] * B * k;
      for (int th = 0; th < threads; ++th) {
        const float *ps = priv + (size_t)th * priv_elems + (size_t)s * B * k;
        for (int e = 0; e < B * k; ++e) YC[e] += ps[e];
      }
    }
  }
  free(priv);
  free(row_start);
  return 0;
}

/* f64-accumulating single-thread oracle (any value dtype given as double). */
void oracle_sym_spmm_f64(int64_t n_tiles, const int32_t *rc, const double *tiles, const double *X, int k, double *Y,
                         int64_t y_rows) {
  memset(Y, 0, (size_t)y_rows * k * sizeof(double));
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int64_t R = rc[2 * t], C = rc[2 * t + 1];
    const double *T = tiles + t * B * B;
    for (int a = 0; a < B; ++a)
      for (int b = 0; b < B; ++b) {
        const double tv = T[a * B + b];
        if (tv == 0.0) continue;
        for (int v = 0; v < k; ++v) {
          Y[(R * B + a) * k + v] += tv * X[(C * B + b) * k + v];
          if (C != R) Y[(C * B + b) * k + v] += tv * X[(R * B + a) * k + v];
        }
      }
  }
}
