/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * C restatement of the reference's dense product (tiles.py:197-212
 * reference_gemm) and of its per-tile rank-1 update (tiles.py:154-172
 * accumulate_product).  Per output element the operation sequence is the
 * reference's: start at 0, then for k = 0, 1, ... one IEEE multiply and one
 * IEEE add (compile with -ffp-contract=off: no FMA), so results are
 * bit-identical to the numpy reference for float64 and float32 inputs.  The
 * loops are cache-blocked over rows/columns and parallelised over row blocks;
 * neither changes any element's k order, so every thread count gives the same
 * bits.  Also the CPU baseline timed by bench.py (cpu_baseline, kind "port").
 */
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RB 64   /* rows per block                                 */
#define CB 256  /* columns per block (accumulator block in cache) */
#define KB 256  /* k values per pass over the accumulator block   */

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

#define DEFINE_GEMM(NAME, T)                                                                  \
  void NAME(const T* a, const T* b, T* c, int64_t m, int64_t k, int64_t n, int threads) {      \
    int64_t nrb = (m + RB - 1) / RB;                                                          \
    if (threads <= 0) threads = oracle_max_threads();                                         \
    _Pragma("omp parallel for schedule(dynamic) num_threads(threads)")                        \
    for (int64_t rb = 0; rb < nrb; ++rb) {                                                    \
      int64_t i0 = rb * RB, i1 = i0 + RB < m ? i0 + RB : m;                                  \
      for (int64_t j0 = 0; j0 < n; j0 += CB) {                                                \
        int64_t j1 = j0 + CB < n ? j0 + CB : n;                                               \
        for (int64_t i = i0; i < i1; ++i)                                                     \
          for (int64_t j = j0; j < j1; ++j) c[i * n + j] = (T)0;                              \
        for (int64_t k0 = 0; k0 < k; k0 += KB) {                                              \
          int64_t k1 = k0 + KB < k ? k0 + KB : k;                                             \
          for (int64_t i = i0; i < i1; ++i) {                                                 \
            T* ci = c + i * n;                                                                \
            const T* ai = a + i * k;                                                          \
            for (int64_t kk = k0; kk < k1; ++kk) {                                            \
              const T av = ai[kk];                                                            \
              const T* bk = b + kk * n;                                                       \
              for (int64_t j = j0; j < j1; ++j) {                                             \
                T p = av * bk[j]; /* rounded product */                                       \
                ci[j] = ci[j] + p; /* rounded sum, k ascending */                             \
              }                                                                               \
            }                                                                                 \
          }                                                                                   \
        }                                                                                     \
      }                                                                                       \
    }                                                                                         \
  }

DEFINE_GEMM(oracle_gemm_f64, double)
DEFINE_GEMM(oracle_gemm_f32, float)

/* tiles.py:170-171 literally: for kk in range(kk_count): out += outer(a[:,kk], b[kk,:]).
 * a is m x k, b is k x n, out m x n (all row-major, contiguous); kk_count <= k. */
#define DEFINE_RANK1(NAME, T)                                                                  \
  void NAME(const T* a, const T* b, T* out, int64_t m, int64_t k, int64_t n, int64_t kk_count) {\
    for (int64_t kk = 0; kk < kk_count; ++kk)                                                 \
      for (int64_t i = 0; i < m; ++i) {                                                       \
        const T av = a[i * k + kk];                                                           \
        T* oi = out + i * n;                                                                  \
        const T* bk = b + kk * n;                                                             \
        for (int64_t j = 0; j < n; ++j) {                                                     \
          T p = av * bk[j];                                                                   \
          oi[j] = oi[j] + p;                                                                  \
        }                                                                                     \
      }                                                                                       \
  }

DEFINE_RANK1(oracle_rank1_f64, double)
DEFINE_RANK1(oracle_rank1_f32, float)
