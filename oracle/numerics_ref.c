/*
 * CPU restatement of the B200 hot path's numerics (TEST INFRASTRUCTURE ONLY:
 * imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * as the checker / CPU baseline, never by the product).
 *
 * PARITY UNPINNED for numerics: the reference has no attention, GEMM or token
 * code (it prices jobs with cost_model.cpp:75-94 and SPEC.md:19-23 puts real
 * kernels out of scope), so there are no reference golden vectors to pin
 * this file to. It follows the reference's KV geometry instead:
 *   - head-blocks of block_tokens=16 tokens x head_dim=128, bf16
 *     (kv_manager.cpp:25-40),
 *   - a 16-token row of a request costs 2*L*H blocks (kv_manager.cpp:30-35),
 *   - decode context ctx = prompt + 1 + steps_done (scheduler.cpp:107),
 * and the physical table layout of this repo's pool (csrc/include/mux/kv.hpp):
 *   rowlist[slot][row] -> row record; rowrec[rec][(layer*H + head)*2 + kv].
 *
 * Build: gcc -O3 -march=x86-64-v3 -shared -fPIC -pthread numerics_ref.c -o _build/libnumerics_ref.so
 * (no -ffast-math: the attention restatement relies on IEEE -INFINITY / exp
 * semantics, and the summation orders below are the ones written).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline float bf16_to_f32(uint16_t v) {
  uint32_t u = ((uint32_t)v) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline uint16_t f32_to_bf16(float f) { /* round to nearest even */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

typedef struct {
  const uint16_t* q;       /* [B][H][128] */
  const uint16_t* pool;    /* [blocks][16][128] */
  const int32_t* rowrec;
  const int32_t* rowlist;
  const int32_t* slots;
  const int32_t* ctx;
  int B, H, L, layer, max_rows;
  float* out;              /* [B][H][128] */
  int next;                /* work counter (guarded) */
  pthread_mutex_t mu;
} attn_job;

/* softmax(q.K^T / sqrt(128)) V for one (request, head), double accumulation. */
static void attend_one(const attn_job* j, int b, int h) {
  const int D = 128;
  const int ctx = j->ctx[b];
  const int slot = j->slots[b];
  const int64_t row_width = 2LL * j->L * j->H;
  double qv[128];
  for (int d = 0; d < D; ++d) qv[d] = bf16_to_f32(j->q[((int64_t)b * j->H + h) * D + d]);
  double* s = (double*)malloc(sizeof(double) * (ctx > 0 ? ctx : 1));
  double m = -INFINITY;
  const double scale = 1.0 / sqrt(128.0);
  for (int t = 0; t < ctx; ++t) {
    int row = t / 16, in = t % 16;
    int32_t rr = j->rowlist[(int64_t)slot * j->max_rows + row];
    int32_t kid = j->rowrec[(int64_t)rr * row_width + ((int64_t)j->layer * j->H + h) * 2 + 0];
    const uint16_t* k = j->pool + (int64_t)kid * 16 * D + (int64_t)in * D;
    double acc = 0.0;
    for (int d = 0; d < D; ++d) acc += qv[d] * bf16_to_f32(k[d]);
    s[t] = acc * scale;
    if (s[t] > m) m = s[t];
  }
  double l = 0.0, o[128];
  for (int d = 0; d < D; ++d) o[d] = 0.0;
  for (int t = 0; t < ctx; ++t) {
    int row = t / 16, in = t % 16;
    int32_t rr = j->rowlist[(int64_t)slot * j->max_rows + row];
    int32_t vid = j->rowrec[(int64_t)rr * row_width + ((int64_t)j->layer * j->H + h) * 2 + 1];
    const uint16_t* v = j->pool + (int64_t)vid * 16 * D + (int64_t)in * D;
    double p = exp(s[t] - m);
    l += p;
    for (int d = 0; d < D; ++d) o[d] += p * bf16_to_f32(v[d]);
  }
  float* out = j->out + ((int64_t)b * j->H + h) * D;
  for (int d = 0; d < D; ++d) out[d] = ctx > 0 ? (float)(o[d] / l) : 0.f;
  free(s);
}

static void* attn_worker(void* arg) {
  attn_job* j = (attn_job*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int w = j->next++;
    pthread_mutex_unlock(&j->mu);
    if (w >= j->B * j->H) break;
    attend_one(j, w / j->H, w % j->H);
  }
  return NULL;
}

/* Paged head-wise decode attention for one layer (the K1 restatement). */
int ref_decode_attention(const uint16_t* q, const uint16_t* pool, const int32_t* rowrec,
                         const int32_t* rowlist, const int32_t* slots, const int32_t* ctx, int B,
                         int H, int L, int layer, int max_rows, float* out, int nthreads) {
  attn_job j;
  j.q = q; j.pool = pool; j.rowrec = rowrec; j.rowlist = rowlist; j.slots = slots; j.ctx = ctx;
  j.B = B; j.H = H; j.L = L; j.layer = layer; j.max_rows = max_rows; j.out = out; j.next = 0;
  pthread_mutex_init(&j.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, attn_worker, &j);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  pthread_mutex_destroy(&j.mu);
  return 0;
}

/* ---- CPU baseline: one bf16-weight GEMV batch (decode projection) --------
 * y[b][n] = sum_k x[b][k] * W[n][k], bf16 inputs, fp32 accumulation, threaded
 * over output rows. Used by bench.py's cpu_baseline leg to time a bounded
 * sample of the decode step on the host cores. */
typedef struct {
  const float* xf; const uint16_t* w; float* y;
  int B, N, K, next; pthread_mutex_t mu;
} gemv_job;

/* fp32 dot product over 16 independent lane sums (a fixed order the
 * compiler can vectorise without -ffast-math), then a fixed lane reduction. */
static float dot_f32(const float* a, const float* b, int n) {
  float acc[16] = {0};
  int i = 0;
  for (; i + 16 <= n; i += 16)
    for (int l = 0; l < 16; ++l) acc[l] += a[i + l] * b[i + l];
  for (; i < n; ++i) acc[i & 15] += a[i] * b[i];
  float s = 0.f;
  for (int l = 0; l < 16; ++l) s += acc[l];
  return s;
}

static void* gemv_worker(void* arg) {
  gemv_job* j = (gemv_job*)arg;
  enum { ROWS = 16 };
  float* wf = (float*)malloc(sizeof(float) * ROWS * (size_t)j->K);
  for (;;) {
    pthread_mutex_lock(&j->mu);
    int n0 = j->next;
    j->next += ROWS;
    pthread_mutex_unlock(&j->mu);
    if (n0 >= j->N) break;
    int n1 = n0 + ROWS < j->N ? n0 + ROWS : j->N;
    for (int n = n0; n < n1; ++n) {
      const uint16_t* wr = j->w + (int64_t)n * j->K;
      float* dst = wf + (size_t)(n - n0) * j->K;
      for (int k = 0; k < j->K; ++k) dst[k] = bf16_to_f32(wr[k]);
    }
    for (int b = 0; b < j->B; ++b) {
      const float* xb = j->xf + (int64_t)b * j->K;
      for (int n = n0; n < n1; ++n)
        j->y[(int64_t)b * j->N + n] = dot_f32(wf + (size_t)(n - n0) * j->K, xb, j->K);
    }
  }
  free(wf);
  return NULL;
}

/* y[b][n] = sum_k x[b][k] * W[n][k]; bf16 in, fp32 accumulate, threaded over
 * blocks of output rows (weights streamed once, activations cache-resident). */
int ref_gemv_bf16(const uint16_t* x, const uint16_t* w, float* y, int B, int N, int K, int nthreads) {
  gemv_job j;
  float* xf = (float*)malloc(sizeof(float) * (size_t)B * K);
  for (int64_t i = 0; i < (int64_t)B * K; ++i) xf[i] = bf16_to_f32(x[i]);
  j.xf = xf; j.w = w; j.y = y; j.B = B; j.N = N; j.K = K; j.next = 0;
  pthread_mutex_init(&j.mu, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
  for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, gemv_worker, &j);
  for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
  free(th);
  free(xf);
  pthread_mutex_destroy(&j.mu);
  return 0;
}

/* bf16 conversions exposed for tests. */
void ref_f32_to_bf16(const float* in, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = f32_to_bf16(in[i]);
}
