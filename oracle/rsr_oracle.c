/*
 * CPU oracle / CPU baseline for the RSR / RSR++ hot path — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference `rsr` package (arxiv 2411.06360,
 * /root/reference/pkg/src/rsr).  The reference's compiled inner loops are
 * Numba `@njit` functions (no C sources exist to compile), so this file is the
 * "port" CPU baseline that bench.py times and the parity tests check against.
 * The product library (paper_2411_06360_b200/lib/librsr_b200.so) never links it.
 *
 * Pinned against the reference's own outputs by tests/test_oracle_golden.py
 * (golden vectors from tests/golden/make_golden.py, which imports the real
 * reference).
 *
 *   preprocess : indexer.py:251-278 (stable per-block ordering, bincount+cumsum)
 *                restated as an explicit stable counting sort.
 *   multiply   : kernels.py:127-177 (`_run_blocks`, scatter u[bucket[r]] += v[r]
 *                four blocks at a time, then `_product_fold` kernels.py:74-91 or
 *                `_product_dense` kernels.py:63-71), fp64.
 *   parallel   : kernels.py:209-239 (block ranges [i*nb/W, (i+1)*nb/W) per worker,
 *                disjoint output slices), pthreads instead of a ThreadPoolExecutor.
 *   naive      : core.py:135-143 (`_naive_ternary`, ascending-row fp64 sum).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Keys of one binary half of a ternary matrix for every block (indexer.py:215-219):
 * key(r, b) = MSB-first bits of [A[r, c] == sign] over the block's columns. */
void rsr_oracle_keys_ternary(const int8_t* A, int64_t n, int64_t m, int k, int sign,
                             uint16_t* keys /* [nb][n] */) {
  int64_t nb = (m + k - 1) / k;
  for (int64_t b = 0; b < nb; ++b) {
    int64_t c0 = b * k;
    int w = (int)((m - c0) < k ? (m - c0) : k);
    for (int64_t r = 0; r < n; ++r) {
      const int8_t* row = A + r * m + c0;
      unsigned key = 0;
      for (int c = 0; c < w; ++c) key = (key << 1) | (unsigned)(row[c] == sign);
      keys[b * n + r] = (uint16_t)key;
    }
  }
}

/* Stable counting sort of one block's keys (indexer.py:269,274-276):
 * seg[j] = #rows with key < j (seg[2^w] = n), perm lists rows by ascending key,
 * ties in ascending row order. */
void rsr_oracle_sort_block(const uint16_t* keys, int64_t n, int w, uint32_t* perm, int64_t* seg) {
  int64_t nbk = (int64_t)1 << w;
  int64_t* cursor = (int64_t*)calloc((size_t)nbk, sizeof(int64_t));
  for (int64_t r = 0; r < n; ++r) cursor[keys[r]]++;
  int64_t run = 0;
  for (int64_t j = 0; j < nbk; ++j) {
    int64_t c = cursor[j];
    seg[j] = run;
    cursor[j] = run;
    run += c;
  }
  seg[nbk] = run;
  for (int64_t r = 0; r < n; ++r) perm[cursor[keys[r]]++] = (uint32_t)r;
  free(cursor);
}

static void product_fold(const double* u, double* buf, int w, double* out) {
  int64_t half = ((int64_t)1 << w) >> 1;
  double acc = 0.0;
  for (int64_t t = 0; t < half; ++t) {
    acc += u[2 * t + 1];
    buf[t] = u[2 * t] + u[2 * t + 1];
  }
  out[w - 1] = acc;
  int64_t size = half;
  for (int c = w - 2; c >= 0; --c) {
    half = size >> 1;
    acc = 0.0;
    for (int64_t t = 0; t < half; ++t) {
      acc += buf[2 * t + 1];
      buf[t] = buf[2 * t] + buf[2 * t + 1];
    }
    out[c] = acc;
    size = half;
  }
}

static void product_dense(const double* u, int w, double* out) {
  int64_t nseg = (int64_t)1 << w;
  for (int c = 0; c < w; ++c) {
    int shift = w - 1 - c;
    double acc = 0.0;
    for (int64_t j = 0; j < nseg; ++j) acc += u[j] * (double)((j >> shift) & 1);
    out[c] = acc;
  }
}

/* kernels.py:127-177: blocks [b0, b1) of one half, scatter form, 4 blocks per row pass. */
void rsr_oracle_run_blocks(const double* v, const uint16_t* keys /* [nb][n] */, int64_t n,
                           int64_t m, int k, int64_t b0, int64_t b1, int use_fold, double* out) {
  int64_t kbuf = (int64_t)1 << k;
  double* u = (double*)malloc(sizeof(double) * (size_t)(4 * kbuf + (kbuf > 1 ? kbuf / 2 : 1)));
  double *u0 = u, *u1 = u + kbuf, *u2 = u + 2 * kbuf, *u3 = u + 3 * kbuf, *buf = u + 4 * kbuf;
  int64_t b = b0;
#define WIDTH(bb) ((int)(((m - (bb) * k) < k) ? (m - (bb) * k) : k))
  while (b + 4 <= b1) {
    int w0 = WIDTH(b), w1 = WIDTH(b + 1), w2 = WIDTH(b + 2), w3 = WIDTH(b + 3);
    memset(u0, 0, sizeof(double) * ((size_t)1 << w0));
    memset(u1, 0, sizeof(double) * ((size_t)1 << w1));
    memset(u2, 0, sizeof(double) * ((size_t)1 << w2));
    memset(u3, 0, sizeof(double) * ((size_t)1 << w3));
    const uint16_t *g0 = keys + b * n, *g1 = g0 + n, *g2 = g1 + n, *g3 = g2 + n;
    for (int64_t r = 0; r < n; ++r) {
      double x = v[r];
      u0[g0[r]] += x;
      u1[g1[r]] += x;
      u2[g2[r]] += x;
      u3[g3[r]] += x;
    }
    if (use_fold) {
      product_fold(u0, buf, w0, out + b * k);
      product_fold(u1, buf, w1, out + (b + 1) * k);
      product_fold(u2, buf, w2, out + (b + 2) * k);
      product_fold(u3, buf, w3, out + (b + 3) * k);
    } else {
      product_dense(u0, w0, out + b * k);
      product_dense(u1, w1, out + (b + 1) * k);
      product_dense(u2, w2, out + (b + 2) * k);
      product_dense(u3, w3, out + (b + 3) * k);
    }
    b += 4;
  }
  while (b < b1) {
    int w = WIDTH(b);
    memset(u0, 0, sizeof(double) * ((size_t)1 << w));
    const uint16_t* g0 = keys + b * n;
    for (int64_t r = 0; r < n; ++r) u0[g0[r]] += v[r];
    if (use_fold) product_fold(u0, buf, w, out + b * k);
    else product_dense(u0, w, out + b * k);
    ++b;
  }
#undef WIDTH
  free(u);
}

typedef struct {
  const double* v;
  const uint16_t* keys;
  int64_t n, m, b0, b1;
  int k, use_fold;
  double* out;
} task_t;

static void* task_main(void* arg) {
  task_t* t = (task_t*)arg;
  rsr_oracle_run_blocks(t->v, t->keys, t->n, t->m, t->k, t->b0, t->b1, t->use_fold, t->out);
  return NULL;
}

/* kernels.py:209-239 — halves = 1 (binary) or 2 (ternary: keys_pos, keys_neg),
 * W workers over block ranges, result = pos - neg. scratch: m doubles (ternary). */
void rsr_oracle_multiply_parallel(const double* v, const uint16_t* keys_pos,
                                  const uint16_t* keys_neg, int64_t n, int64_t m, int k,
                                  int use_fold, int workers, double* out, double* scratch) {
  int64_t nb = (m + k - 1) / k;
  int halves = keys_neg ? 2 : 1;
  double* outs[2] = {out, scratch};
  const uint16_t* keys[2] = {keys_pos, keys_neg};
  if (workers < 1) workers = 1;
  task_t* tasks = (task_t*)calloc((size_t)(2 * workers), sizeof(task_t));
  pthread_t* th = (pthread_t*)calloc((size_t)(2 * workers), sizeof(pthread_t));
  int nt = 0;
  for (int h = 0; h < halves; ++h)
    for (int i = 0; i < workers; ++i) {
      int64_t lo = i * nb / workers, hi = (i + 1) * nb / workers;
      if (lo < hi) {
        task_t t = {v, keys[h], n, m, lo, hi, k, use_fold, outs[h]};
        tasks[nt++] = t;
      }
    }
  if (workers == 1) {
    for (int i = 0; i < nt; ++i) task_main(&tasks[i]);
  } else {
    for (int i = 0; i < nt; ++i) pthread_create(&th[i], NULL, task_main, &tasks[i]);
    for (int i = 0; i < nt; ++i) pthread_join(th[i], NULL);
  }
  if (halves == 2)
    for (int64_t j = 0; j < m; ++j) out[j] = out[j] - scratch[j];
  free(tasks);
  free(th);
}

/* core.py:135-143 — the "standard" dense multiply, ascending i. */
void rsr_oracle_naive_ternary(const double* v, const int8_t* A, int64_t n, int64_t m, double* out) {
  for (int64_t j = 0; j < m; ++j) out[j] = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double vi = v[i];
    const int8_t* row = A + i * m;
    for (int64_t j = 0; j < m; ++j) out[j] += vi * (double)row[j];
  }
}
