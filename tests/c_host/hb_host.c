/* A non-Python host driving the B200 HyperBall path through the C-ABI only
 * (include/hyperball_b200.h): seed, one hb_union_step_v2 per iteration until no counter
 * changes, finalizers -- what INTEGRATION.md section 2 describes for a C / JNI / cgo host.
 * Test infrastructure (tests/test_gpu_c_host.py compares its output with the golden
 * cases produced by the reference).
 *
 *   hb_host <graph.bin> <b> <seed> <out.bin>
 *   graph.bin: int64 n, int64 m, int64 offsets[n + 1], int32 successors[m]  (G^T CSR)
 *   out.bin:   int64 t, uint8 registers[n * 2^b], double harmonic[n], closeness[n], lin[n]
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include "hyperball_b200.h"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 2; } } while (0)
#define HB(x) do { if ((x) != 0) { fprintf(stderr, "%s: %s\n", #x, hb_last_error()); \
    return 3; } } while (0)

/* hll.py alpha / estimator_constants / lc_table, restated for the host */
static double alpha(int p) {
  if (p == 16) return 0.673;
  if (p == 32) return 0.697;
  if (p == 64) return 0.709;
  return 0.7213 / (1.0 + 1.079 / p);
}

int main(int argc, char **argv) {
  if (argc != 5) { fprintf(stderr, "usage: hb_host graph.bin b seed out.bin\n"); return 1; }
  FILE *f = fopen(argv[1], "rb");
  if (!f) return 1;
  int64_t n, m;
  if (fread(&n, 8, 1, f) != 1 || fread(&m, 8, 1, f) != 1) return 1;
  int64_t *off = (int64_t *)malloc(8 * (size_t)(n + 1));
  int32_t *suc = (int32_t *)malloc(4 * (size_t)(m > 0 ? m : 1));
  if (fread(off, 8, (size_t)(n + 1), f) != (size_t)(n + 1)) return 1;
  if (m > 0 && fread(suc, 4, (size_t)m, f) != (size_t)m) return 1;
  fclose(f);
  const int b = atoi(argv[2]);
  const uint64_t seed = strtoull(argv[3], NULL, 10);
  const int p = 1 << b;
  const size_t rows = (size_t)n * (size_t)p, words = (size_t)((n + 31) / 32);

  double *lc = (double *)calloc((size_t)p + 1, 8);
  for (int v = 1; v <= p; v++) lc[v] = (double)p * log((double)p / (double)v);
  const double alpha_p2 = (alpha(p) * p) * p, lc_cut = 2.5 * p;

  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  int64_t *d_off; int32_t *d_suc; uint8_t *d_cur, *d_nxt; uint32_t *d_prev, *d_now;
  double *d_est, *d_sd, *d_sr, *d_lc, *d_h, *d_c, *d_l; uint64_t *d_cnt;
  CK(cudaMalloc((void **)&d_off, 8 * (size_t)(n + 1)));
  CK(cudaMalloc((void **)&d_suc, 4 * (size_t)(m > 0 ? m : 1)));
  CK(cudaMalloc((void **)&d_cur, rows)); CK(cudaMalloc((void **)&d_nxt, rows));
  CK(cudaMalloc((void **)&d_prev, 4 * words)); CK(cudaMalloc((void **)&d_now, 4 * words));
  CK(cudaMalloc((void **)&d_est, 8 * (size_t)n)); CK(cudaMalloc((void **)&d_sd, 8 * (size_t)n));
  CK(cudaMalloc((void **)&d_sr, 8 * (size_t)n)); CK(cudaMalloc((void **)&d_lc, 8 * (size_t)(p + 1)));
  CK(cudaMalloc((void **)&d_h, 8 * (size_t)n)); CK(cudaMalloc((void **)&d_c, 8 * (size_t)n));
  CK(cudaMalloc((void **)&d_l, 8 * (size_t)n)); CK(cudaMalloc((void **)&d_cnt, 16));
  CK(cudaMemcpy(d_off, off, 8 * (size_t)(n + 1), cudaMemcpyHostToDevice));
  if (m > 0) CK(cudaMemcpy(d_suc, suc, 4 * (size_t)m, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_lc, lc, 8 * (size_t)(p + 1), cudaMemcpyHostToDevice));
  CK(cudaMemset(d_sd, 0, 8 * (size_t)n)); CK(cudaMemset(d_sr, 0, 8 * (size_t)n));
  CK(cudaMemset(d_prev, 0xFF, 4 * words));           /* every counter "changed" at t = 0 */

  /* engine.py:153-162: seed both buffers (the lazy double buffer reads nxt's old rows) */
  HB(hb_seed(d_cur, d_est, n, b, 5, seed, NULL, NULL, d_lc, alpha_p2, lc_cut, s));
  CK(cudaMemcpyAsync(d_nxt, d_cur, rows, cudaMemcpyDeviceToDevice, s));

  int64_t t = 0;
  for (;;) {
    t++;
    hb_step_args a;
    memset(&a, 0, sizeof a);
    a.struct_size = sizeof a;
    a.n = n; a.lo = 0; a.hi = n; a.offsets = d_off; a.succ = d_suc;
    a.cur = d_cur; a.nxt = d_nxt; a.chg_prev = d_prev; a.chg_now = d_now;
    a.est = d_est; a.b = b; a.dense = t == 1; a.clear_chg_now = 1; a.t = t;
    a.lc_table = d_lc; a.alpha_p2 = alpha_p2; a.lc_cut = lc_cut;
    a.sum_dist = d_sd; a.sum_recip = d_sr;
    a.light_max_deg = INT64_MAX; a.item_arcs = 64;   /* one group per node, no heavy split */
    a.nch_out = d_cnt; a.merged_out = d_cnt + 1; a.stream = s;
    HB(hb_union_step_v2(&a));
    uint64_t cnt[2];
    CK(cudaMemcpyAsync(cnt, d_cnt, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    uint8_t *tr = d_cur; d_cur = d_nxt; d_nxt = tr;       /* swap (engine.py:393) */
    uint32_t *tb = d_prev; d_prev = d_now; d_now = tb;
    if (cnt[0] == 0) break;
  }
  HB(hb_finalize(n, NULL, d_sd, d_sr, d_est, d_c, d_h, d_l, s));
  uint8_t *regs = (uint8_t *)malloc(rows > 0 ? rows : 1);
  double *h = (double *)malloc(8 * (size_t)n), *c = (double *)malloc(8 * (size_t)n),
         *l = (double *)malloc(8 * (size_t)n);
  CK(cudaMemcpyAsync(regs, d_cur, rows, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(h, d_h, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(c, d_c, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(l, d_l, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  FILE *o = fopen(argv[4], "wb");
  if (!o) return 1;
  fwrite(&t, 8, 1, o);
  fwrite(regs, 1, rows, o);
  fwrite(h, 8, (size_t)n, o);
  fwrite(c, 8, (size_t)n, o);
  fwrite(l, 8, (size_t)n, o);
  fclose(o);
  printf("hb_host: n=%lld m=%lld b=%d t=%lld\n", (long long)n, (long long)m, b, (long long)t);
  return 0;
}
