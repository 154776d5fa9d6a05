/* C restatement of the reference's MoL scoring for large parity checks (TEST INFRASTRUCTURE ONLY:
 * only tests/, __graft_entry__.smoke() and bench.py's oracle legs load it; the product never does).
 *
 * It computes exactly what oracle/molr_oracle.py computes (and what the reference computes with
 * NumPy + OpenBLAS) for one (query, item) pair, in fp32, without materialising any (U, X, G)
 * intermediate, multithreaded over items with pthreads, so the full-corpus exact scores of BASELINE's
 * configs (ML-1M: 22.4M pairs; 100M items x a few queries) can be recomputed on the host cores:
 *
 *   cl[a*k_x+b] = <u_a, x_b> / tau                       mol.py:139-158 (component_logits; / tau at 158)
 *   h           = silu(cl @ W1 + b1)                      mol.py:84-85   (Mlp.__call__, cross net, no out bias)
 *   cw          = h @ W2
 *   pi          = softmax_rows(silu(uw * gate_pre + cw))  mol.py:186-188 (decomposed_gating, inference)
 *   score       = sum_g pi[g] * cl[g]                     mol.py:197-205 (mol_score)
 *   silu(x) = x * expit(x) = x / (1 + exp(-x))            numerics.py:73-75
 *   softmax: max-shifted, e / sum(e)                      numerics.py:61-66
 *
 * Summation order differs from OpenBLAS's sgemm (which is itself unpinned): agreement
 * with the NumPy restatement is checked to ~1e-7 absolute in tests/test_oracle_c.py, far inside the
 * parity tolerance 1e-3 |s| + 1e-6.
 *
 * Item inputs may be f32 or bf16 (uint16 bit patterns, widened exactly), so a device cache can be
 * streamed back in its storage format without a host-side f32 copy of the corpus.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define MAXG 256
/* x86-64-v3 (AVX2 + FMA) clone where the host has it, baseline otherwise (resolved at load time,
 * so the library built here runs on any x86-64 host) */
#if defined(__x86_64__) && defined(__GNUC__) && !defined(__clang__)
#define MOLO_CLONES __attribute__((target_clones("arch=x86-64-v3", "default")))
#else
#define MOLO_CLONES
#endif
#define MAXH 1024

static inline float bf16_to_f32(uint16_t v) {
  uint32_t u = (uint32_t)v << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

static inline float load_item(const void* p, int dtype, int64_t i) {
  return dtype ? bf16_to_f32(((const uint16_t*)p)[i]) : ((const float*)p)[i];
}

/* exp(x) in float: x = n ln2 + r (Cody-Waite, |r| <= ln2/2), e^r by a degree-7 Taylor/minimax
 * polynomial, 2^n through the exponent bits.  Max relative error ~2 ulp against expf over the
 * range used here (|x| < 87, clamped), written branch-free so the array loops below vectorize. */
static inline float exp_f(float x) {
  x = x < -87.0f ? -87.0f : x;
  x = x > 88.0f ? 88.0f : x;
  const float n = (x * 1.44269504088896341f + 12582912.0f) - 12582912.0f; /* round half-even */
  float r = x - n * 0.693145751953125f;
  r = r - n * 1.428606765330187045e-06f;
  float p = 1.9875691500e-4f;
  p = p * r + 1.3981999507e-3f;
  p = p * r + 8.3334519073e-3f;
  p = p * r + 4.1665795894e-2f;
  p = p * r + 1.6666665459e-1f;
  p = p * r + 5.0000001201e-1f;
  p = p * r * r + r + 1.0f;
  union {
    int32_t i;
    float f;
  } e;
  e.i = ((int32_t)n + 127) << 23;
  return p * e.f;
}

/* silu over an array: x * expit(x) = x / (1 + e^-x)  (numerics.py:73-75) */
static inline void silu_rows(float* x, int n) {
  for (int i = 0; i < n; ++i) x[i] = x[i] / (1.0f + exp_f(-x[i]));
}

/* One query against one item: returns the MoL score.  xt is the item's components transposed
 * (d, k_x), gp its gate pre-activations (G).  Generic shapes. */
static float score_one(int k_u, int k_x, int d, int H, const float* u, const float* uw, const float* W1,
                       const float* b1, const float* W2, float tau, const float* xt, const float* gp) {
  const int G = k_u * k_x;
  float cl[MAXG], cw[MAXG], z[MAXG], h[MAXH];
  for (int a = 0; a < k_u; ++a) {
    float acc[64];
    for (int b = 0; b < k_x; ++b) acc[b] = 0.0f;
    for (int k = 0; k < d; ++k) {
      const float ua = u[a * d + k];
      const float* xr = xt + k * k_x;
      for (int b = 0; b < k_x; ++b) acc[b] += ua * xr[b];
    }
    for (int b = 0; b < k_x; ++b) cl[a * k_x + b] = acc[b] / tau;
  }
  for (int j = 0; j < H; ++j) h[j] = 0.0f;
  for (int g = 0; g < G; ++g) {
    const float c = cl[g];
    const float* w = W1 + (int64_t)g * H;
    for (int j = 0; j < H; ++j) h[j] += c * w[j];
  }
  for (int j = 0; j < H; ++j) h[j] += b1[j];
  silu_rows(h, H);
  for (int g = 0; g < G; ++g) cw[g] = 0.0f;
  for (int j = 0; j < H; ++j) {
    const float hj = h[j];
    const float* w = W2 + (int64_t)j * G;
    for (int g = 0; g < G; ++g) cw[g] += hj * w[g];
  }
  for (int g = 0; g < G; ++g) z[g] = uw[g] * gp[g] + cw[g];
  silu_rows(z, G);
  float m = -INFINITY;
  for (int g = 0; g < G; ++g) m = z[g] > m ? z[g] : m;
  for (int g = 0; g < G; ++g) z[g] = exp_f(z[g] - m);
  float se = 0.0f;
  for (int g = 0; g < G; ++g) se += z[g];
  float s = 0.0f;
  for (int g = 0; g < G; ++g) s += (z[g] / se) * cl[g];
  return s;
}

/* The production shape (k_u = k_x = 8, d = 64, H = 128, G = 64) written with 8-wide GCC vector
 * types (one ymm register in the x86-64-v3 clone, two xmm otherwise), so every contraction runs as
 * independent vector FMA chains.  Same arithmetic as score_one (per-element results differ only by
 * summation order). */
enum { PKU = 8, PKX = 8, PD = 64, PH = 128, PG = 64 };
typedef float v8f __attribute__((vector_size(32)));
typedef int32_t v8i __attribute__((vector_size(32)));

static inline __attribute__((always_inline)) v8f splat(float x) { return (v8f){x, x, x, x, x, x, x, x}; }
static inline __attribute__((always_inline)) v8f ldv(const float* p) {
  v8f v;
  memcpy(&v, p, sizeof v);
  return v;
}
static inline __attribute__((always_inline)) v8f vsel(v8i m, v8f a, v8f b) { /* m ? a : b, lanewise (C has no vector ?:) */
  v8i ai, bi;
  memcpy(&ai, &a, sizeof ai);
  memcpy(&bi, &b, sizeof bi);
  const v8i r = (ai & m) | (bi & ~m);
  v8f out;
  memcpy(&out, &r, sizeof out);
  return out;
}
static inline __attribute__((always_inline)) v8f vmax(v8f a, v8f b) { return vsel(a > b, a, b); }
static inline __attribute__((always_inline)) v8f exp_v(v8f x) { /* exp_f on 8 lanes */
  x = vmax(x, splat(-87.0f));
  x = vsel(x > splat(88.0f), splat(88.0f), x);
  const v8f n = (x * 1.44269504088896341f + 12582912.0f) - 12582912.0f;
  v8f r = x - n * 0.693145751953125f;
  r = r - n * 1.428606765330187045e-06f;
  v8f p = splat(1.9875691500e-4f);
  p = p * r + 1.3981999507e-3f;
  p = p * r + 8.3334519073e-3f;
  p = p * r + 4.1665795894e-2f;
  p = p * r + 1.6666665459e-1f;
  p = p * r + 5.0000001201e-1f;
  p = p * r * r + r + 1.0f;
  const v8i e = (__builtin_convertvector(n, v8i) + 127) << 23;
  v8f s;
  memcpy(&s, &e, sizeof s);
  return p * s;
}
static inline __attribute__((always_inline)) v8f silu_v(v8f x) { return x / (1.0f + exp_v(-x)); }
static inline __attribute__((always_inline)) float hmax(v8f v) {
  float m = v[0];
  for (int i = 1; i < 8; ++i) m = v[i] > m ? v[i] : m;
  return m;
}
static inline __attribute__((always_inline)) float hsum(v8f v) {
  float s = 0.0f;
  for (int i = 0; i < 8; ++i) s += v[i];
  return s;
}

static inline __attribute__((always_inline)) float score_prod(const float* restrict u, const float* restrict uw, const float* restrict W1,
                               const float* restrict b1, const float* restrict W2, float tau,
                               const float* restrict xt, const float* restrict gp) {
  /* component logits: row a of cl = sum_k u[a,k] * xt[k, 0..7], then / tau (mol.py:156-158) */
  v8f cl[PKU];
  for (int a = 0; a < PKU; ++a) cl[a] = splat(0.0f);
  for (int k = 0; k < PD; ++k) {
    const v8f x = ldv(xt + k * PKX);
    for (int a = 0; a < PKU; ++a) cl[a] += u[a * PD + k] * x;
  }
  float cls[PG];
  for (int a = 0; a < PKU; ++a) {
    cl[a] = cl[a] / tau;
    memcpy(cls + a * PKX, &cl[a], sizeof(v8f));
  }
  /* cross net layer 1: h = silu(cl @ W1 + b1), two passes of 8 vector accumulators */
  v8f h[PH / 8];
  for (int jb = 0; jb < PH / 8; jb += 8) {
    v8f acc[8];
    for (int v = 0; v < 8; ++v) acc[v] = splat(0.0f);
    for (int g = 0; g < PG; ++g) {
      const float c = cls[g];
      for (int v = 0; v < 8; ++v) acc[v] += c * ldv(W1 + g * PH + (jb + v) * 8);
    }
    for (int v = 0; v < 8; ++v) h[jb + v] = silu_v(acc[v] + ldv(b1 + (jb + v) * 8));
  }
  float hs[PH];
  memcpy(hs, h, sizeof hs);
  /* layer 2: cw = h @ W2 */
  v8f cw[PG / 8];
  for (int v = 0; v < PG / 8; ++v) cw[v] = splat(0.0f);
  for (int j = 0; j < PH; ++j) {
    const float hj = hs[j];
    for (int v = 0; v < PG / 8; ++v) cw[v] += hj * ldv(W2 + j * PG + v * 8);
  }
  /* pi = softmax(silu(uw * gate_pre + cw)); score = sum pi * cl */
  v8f z[PG / 8];
  v8f m = splat(-INFINITY);
  for (int v = 0; v < PG / 8; ++v) {
    z[v] = silu_v(ldv(uw + v * 8) * ldv(gp + v * 8) + cw[v]);
    m = vmax(m, z[v]);
  }
  const float mx = hmax(m);
  v8f se = splat(0.0f);
  for (int v = 0; v < PG / 8; ++v) {
    z[v] = exp_v(z[v] - mx);
    se += z[v];
  }
  const float sum = hsum(se);
  v8f s = splat(0.0f);
  for (int v = 0; v < PG / 8; ++v) s += (z[v] / sum) * cl[v];
  return hsum(s);
}

/* ---- a minimal pthread parallel-for over [0, n) in dynamic chunks (no OpenMP in this image) ---- */
typedef struct {
  void (*body)(void* arg, int64_t lo, int64_t hi, float* scratch);
  void* arg;
  int64_t n, chunk;
  int64_t next;
  pthread_mutex_t mu;
  size_t scratch_floats;
} pfor_t;

static void* pfor_worker(void* p) {
  pfor_t* f = (pfor_t*)p;
  float* scratch = (float*)malloc(sizeof(float) * (f->scratch_floats ? f->scratch_floats : 1));
  for (;;) {
    pthread_mutex_lock(&f->mu);
    const int64_t lo = f->next;
    f->next += f->chunk;
    pthread_mutex_unlock(&f->mu);
    if (lo >= f->n) break;
    const int64_t hi = lo + f->chunk < f->n ? lo + f->chunk : f->n;
    f->body(f->arg, lo, hi, scratch);
  }
  free(scratch);
  return NULL;
}

static int default_threads(void) {
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

static void pfor(int nthreads, int64_t n, int64_t chunk, size_t scratch_floats,
                 void (*body)(void*, int64_t, int64_t, float*), void* arg) {
  if (nthreads <= 0) nthreads = default_threads();
  if (nthreads > 256) nthreads = 256;
  pfor_t f = {body, arg, n, chunk > 0 ? chunk : 1, 0, PTHREAD_MUTEX_INITIALIZER, scratch_floats};
  pthread_t th[256];
  int started = 0;
  for (int t = 1; t < nthreads; ++t)
    if (pthread_create(&th[started], NULL, pfor_worker, &f) == 0) ++started;
  pfor_worker(&f);
  for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

typedef struct {
  int k_u, k_x, d, H, embs_dtype, gp_dtype, B;
  const void *item_embs, *gate_pre;
  const float *user_embs, *uw, *W1, *b1, *W2;
  float tau;
  float* out;
  int64_t ld;
  const int64_t *offs, *ids; /* candidate mode */
  int q;                     /* candidate mode: current query */
} job_t;

static inline void load_item_block(const job_t* J, int64_t i, float* xt, float* gp) {
  const int G = J->k_u * J->k_x;
  for (int b = 0; b < J->k_x; ++b)
    for (int k = 0; k < J->d; ++k) xt[k * J->k_x + b] = load_item(J->item_embs, J->embs_dtype, (i * J->k_x + b) * J->d + k);
  for (int g = 0; g < G; ++g) gp[g] = load_item(J->gate_pre, J->gp_dtype, i * G + g);
}

#define PROD(J) ((J)->k_u == PKU && (J)->k_x == PKX && (J)->d == PD && (J)->H == PH)

MOLO_CLONES static void scores_body(void* a, int64_t lo, int64_t hi, float* xt) {
  const job_t* J = (const job_t*)a;
  const int G = J->k_u * J->k_x;
  float gp[MAXG];
  for (int64_t i = lo; i < hi; ++i) {
    load_item_block(J, i, xt, gp);
    for (int q = 0; q < J->B; ++q)
      J->out[(int64_t)q * J->ld + i] = PROD(J) ? score_prod(J->user_embs + (int64_t)q * PKU * PD, J->uw + (int64_t)q * PG, J->W1, J->b1, J->W2, J->tau, xt, gp) : score_one(J->k_u, J->k_x, J->d, J->H, J->user_embs + (int64_t)q * J->k_u * J->d,
                                                 J->uw + (int64_t)q * G, J->W1, J->b1, J->W2, J->tau, xt, gp);
  }
}

MOLO_CLONES static void cand_body(void* a, int64_t lo, int64_t hi, float* xt) {
  const job_t* J = (const job_t*)a;
  const int G = J->k_u * J->k_x;
  float gp[MAXG];
  for (int64_t j = lo; j < hi; ++j) {
    load_item_block(J, J->ids[j], xt, gp);
    J->out[j] = PROD(J) ? score_prod(J->user_embs + (int64_t)J->q * PKU * PD, J->uw + (int64_t)J->q * PG, J->W1, J->b1, J->W2, J->tau, xt, gp) : score_one(J->k_u, J->k_x, J->d, J->H, J->user_embs + (int64_t)J->q * J->k_u * J->d,
                          J->uw + (int64_t)J->q * G, J->W1, J->b1, J->W2, J->tau, xt, gp);
  }
}

/* Scores of B queries against items [0, n): out (B, ld) row-major, column i = item i.
 * item_embs (n, k_x, d) and gate_pre (n, G) in f32 (dtype 0) or bf16 bits (dtype 1).
 * nthreads <= 0: one thread per online core.  Returns 0, or -1 for unsupported shapes. */
int molo_scores(int64_t n, int k_u, int k_x, int d, int H, const void* item_embs, int embs_dtype,
                const void* gate_pre, int gp_dtype, int B, const float* user_embs, const float* uw,
                const float* W1, const float* b1, const float* W2, float tau, float* out, int64_t ld,
                int nthreads) {
  if (k_u * k_x > MAXG || H > MAXH || k_x > 64 || n < 0 || B < 0) return -1;
  job_t J = {k_u, k_x, d, H, embs_dtype, gp_dtype, B, item_embs, gate_pre, user_embs, uw, W1, b1, W2, tau, out, ld,
             NULL, NULL, 0};
  pfor(nthreads, n, 256, (size_t)k_x * d, scores_body, &J);
  return 0;
}

/* Scores of B queries, each against its own candidate list (ids into the item arrays):
 * offs (B+1), ids (offs[B]) -> out (offs[B]).  score_candidates (mol.py:329-345). */
int molo_score_candidates(int k_u, int k_x, int d, int H, const void* item_embs, int embs_dtype, const void* gate_pre,
                          int gp_dtype, int B, const float* user_embs, const float* uw, const float* W1,
                          const float* b1, const float* W2, float tau, const int64_t* offs, const int64_t* ids,
                          float* out, int nthreads) {
  if (k_u * k_x > MAXG || H > MAXH || k_x > 64 || B < 0) return -1;
  job_t J = {k_u, k_x, d, H, embs_dtype, gp_dtype, 1, item_embs, gate_pre, user_embs, uw, W1, b1, W2, tau, out, 0,
             offs, ids, 0};
  for (int q = 0; q < B; ++q) {
    J.q = q;
    /* cand_body writes out[j] for j in [offs[q], offs[q+1]) */
    const int64_t lo = offs[q], hi = offs[q + 1];
    job_t Jq = J;
    Jq.ids = ids + lo;
    Jq.out = out + lo;
    pfor(nthreads, hi - lo, 64, (size_t)k_x * d, cand_body, &Jq);
  }
  return 0;
}

/* Exact top-k of each row of scores (B, n) by (score desc, id asc) = np.lexsort((ids, -scores))
 * (mol.py:407).  ids are id_offset + column.  Merges into (and returns) the caller's running lists
 * out_ids/out_scores (B, k), which must be initialised to (-1, -inf) before the first call, so a
 * corpus can be scored chunk by chunk. */
static int key_less(float sa, int64_t ia, float sb, int64_t ib) { /* a ranks after b */
  if (sa != sb) return sa < sb;
  return ia > ib;
}

typedef struct {
  const float* scores;
  int64_t n, ld, id_offset;
  int k;
  int64_t* out_ids;
  float* out_scores;
} merge_t;

static void merge_body(void* a, int64_t lo, int64_t hi, float* unused) {
  (void)unused;
  const merge_t* M = (const merge_t*)a;
  const int k = M->k;
  for (int64_t q = lo; q < hi; ++q) {
    int64_t* ri = M->out_ids + q * k;
    float* rs = M->out_scores + q * k;
    const float* s = M->scores + q * M->ld;
    for (int64_t c = 0; c < M->n; ++c) {
      const float v = s[c];
      const int64_t id = M->id_offset + c;
      /* the list is sorted best-first; the last slot is the current k-th */
      if (ri[k - 1] >= 0 && !key_less(rs[k - 1], ri[k - 1], v, id)) continue;
      int p = k - 1;
      while (p > 0 && (ri[p - 1] < 0 || key_less(rs[p - 1], ri[p - 1], v, id))) {
        rs[p] = rs[p - 1];
        ri[p] = ri[p - 1];
        --p;
      }
      rs[p] = v;
      ri[p] = id;
    }
  }
}

int molo_topk_merge(int B, int64_t n, const float* scores, int64_t ld, int64_t id_offset, int k, int64_t* out_ids,
                    float* out_scores, int nthreads) {
  if (k < 1 || B < 0 || n < 0) return -1;
  merge_t M = {scores, n, ld, id_offset, k, out_ids, out_scores};
  pfor(nthreads, B, 1, 0, merge_body, &M);
  return 0;
}

int molo_num_threads(void) { return default_threads(); }
