/* A pure-C client of the drop-in boundary (include/tilerun_b200.h): no Python,
 * no torch.  Builds a 2-device machine (both logical devices on GPU 0 unless
 * more GPUs are visible), multiplies two host matrices through the scheduled
 * runtime (tr_gemm = Runtime.multiply, scheduler.py:559-612) in the
 * FP32-accurate and exact precisions, checks the results against a naive
 * k-ascending product (the reference's tiles.py:197-212 arithmetic: exact mode
 * must match it bit for bit) and prints the reference's counters.
 *
 *   gcc -O2 -std=c11 examples/c_client.c -Iinclude -Lpaper_1511_04348_b200 \
 *       -ltilerun_b200 -Wl,-rpath,$PWD/paper_1511_04348_b200 -o c_client && ./c_client
 * Exit code 0 = both products correct, 2 = no GPU, 1 = failure. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tilerun_b200.h"

#define CHECK(call)                                                        \
  do {                                                                     \
    int st_ = (call);                                                      \
    if (st_ != 0) {                                                        \
      fprintf(stderr, "%s -> %d: %s\n", #call, st_, tr_last_error());      \
      return 1;                                                            \
    }                                                                      \
  } while (0)

static int run_precision(const tr_machine* m, int precision, const double* a, const double* b, int M, int K, int N,
                         const double* ref, double* err_out, int* bitwise_out, tr_cache_stats* stats_out) {
  tr_session* s = NULL;
  CHECK(tr_session_create(m, 128, precision, TR_FLAG_STEAL | TR_FLAG_COHERENCE, 0, &s));
  double* c = calloc((size_t)M * N, sizeof(double));
  tr_matrix ma = {a, M, K, K, TR_DTYPE_F64, TR_LOC_HOST};
  tr_matrix mb = {b, K, N, N, TR_DTYPE_F64, TR_LOC_HOST};
  tr_matrix mc = {c, M, N, N, TR_DTYPE_F64, TR_LOC_HOST};
  tr_gemm_report rep;
  memset(&rep, 0, sizeof(rep));
  CHECK(tr_gemm(s, &ma, 1, 0, &mb, 2, 0, &mc, 3, &rep));
  double num = 0, den = 0;
  int bitwise = 1;
  for (int64_t i = 0; i < (int64_t)M * N; ++i) {
    num += (c[i] - ref[i]) * (c[i] - ref[i]);
    den += ref[i] * ref[i];
    bitwise &= c[i] == ref[i];
  }
  *err_out = sqrt(num / den);
  *bitwise_out = bitwise;
  *stats_out = rep.cache;
  printf("precision %d: %lld tasks, %lld launches, rel err %.3e, bitwise %d | host_fetches %lld l1 %lld l2 %lld "
         "writebacks %lld\n",
         precision, (long long)rep.total_tasks, (long long)rep.gpu_launches, *err_out, bitwise,
         (long long)rep.cache.host_fetches, (long long)rep.cache.l1_hits, (long long)rep.cache.l2_hits,
         (long long)rep.cache.writebacks);
  free(c);
  CHECK(tr_session_destroy(s));
  return 0;
}

int main(void) {
  if (tr_abi_version() != 1) return 1;
  int32_t gpus = 0;
  if (tr_cuda_device_count(&gpus) != 0 || gpus < 1) {
    fprintf(stderr, "no CUDA device\n");
    return 2;
  }
  const int M = 300, K = 260, N = 270, T = 128;
  double* a = malloc(sizeof(double) * M * K);
  double* b = malloc(sizeof(double) * K * N);
  double* ref = calloc((size_t)M * N, sizeof(double));
  srand(7);
  for (int i = 0; i < M * K; ++i) a[i] = (double)rand() / RAND_MAX - 0.5;
  for (int i = 0; i < K * N; ++i) b[i] = (double)rand() / RAND_MAX - 0.5;
  /* tiles.py:209-211: out += a[:, k] * b[k, :], k ascending, a rounded multiply then a rounded add */
  for (int k = 0; k < K; ++k)
    for (int i = 0; i < M; ++i) {
      const double aik = a[i * K + k];
      for (int j = 0; j < N; ++j) {
        volatile double p = aik * b[k * N + j];
        ref[i * N + j] = ref[i * N + j] + p;
      }
    }
  tr_device_spec dev[2];
  memset(dev, 0, sizeof(dev));
  for (int d = 0; d < 2; ++d) {
    dev[d].device_id = d;
    dev[d].kind = TR_KIND_ACCELERATOR;
    dev[d].capacity_tiles = -1;
    dev[d].slots = 4;
    dev[d].gpu = gpus > 1 ? d : 0;
    dev[d].flops_per_unit = 1.0;
    dev[d].host_bandwidth = 1.0;
  }
  int64_t hops[4] = {0, 1, 1, 0};
  tr_machine m = {2, dev, hops, 8, NULL, 0.0};
  const int g = (M + T - 1) / T, gk = (K + T - 1) / T, gn = (N + T - 1) / T;
  double err;
  int bitwise;
  tr_cache_stats st;
  if (run_precision(&m, TR_PREC_FP32ACC, a, b, M, K, N, ref, &err, &bitwise, &st) || err > 1e-5) return 1;
  /* unbounded caches: every input tile crosses the host link once (test_acceptance.py:95-107) */
  if (st.host_fetches != (int64_t)g * gk + (int64_t)gk * gn || st.writebacks != (int64_t)g * gn) return 1;
  if (run_precision(&m, TR_PREC_EXACT, a, b, M, K, N, ref, &err, &bitwise, &st) || !bitwise) return 1;
  printf("c client ok\n");
  free(a);
  free(b);
  free(ref);
  return 0;
}
