/* TEST INFRASTRUCTURE ONLY — see vnt_oracle.h.  Plain-C restatement of the
 * reference hot path.  Reduction exactness is restated with Shewchuk's
 * non-overlapping-partials summation + a correct final rounding (the published
 * algorithm behind CPython's math.fsum), which yields the same correctly
 * rounded sum the reference obtains with its 71-limb fixed-point accumulator
 * (exact_sum.cpp:15-104): both return the real sum rounded once to nearest-even,
 * so results are bit-identical while the mechanism is independent.
 * Compile with -ffp-contract=off: the reference's x86-64 build has no FMA. */
#include "vnt_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.cpp */
static const uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

static uint64_t mix64(uint64_t z) { /* rng.cpp:16-20 */
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t vo_rng_key(uint64_t seed) { return mix64(seed + kGolden); } /* rng.cpp:33 */

static uint64_t split_u64(uint64_t key, uint64_t stream) { /* rng.cpp:35-37 */
  return mix64(key ^ mix64(stream + kGolden));
}

uint64_t vo_rng_split_label(uint64_t key, const char* label) { /* rng.cpp:22-29,39-41 */
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const unsigned char* p = (const unsigned char*)label; *p; ++p) {
    h ^= *p;
    h *= 0x100000001B3ULL;
  }
  return split_u64(key, h);
}

static uint64_t rng_bits(uint64_t key, uint64_t c) { return mix64(key + c * kGolden); }

double vo_rng_normal(uint64_t key, uint64_t c) { /* rng.cpp:51-58 */
  const double u1 = (double)((rng_bits(key, 2 * c) >> 11) + 1) * 0x1.0p-53;
  const double u2 = (double)(rng_bits(key, 2 * c + 1) >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.141592653589793 * u2);
}

/* --------------------------------------------------------------- data.cpp */
int vo_synth_batch(uint64_t seed, uint64_t n, uint64_t in_w, uint64_t out_w,
                   uint64_t start, uint64_t count, double* x, double* y) {
  if (n == 0 || in_w == 0 || out_w == 0) return 2;
  const uint64_t base = vo_rng_key(seed);
  const uint64_t tkey = vo_rng_split_label(base, "teacher");
  const uint64_t xkey = vo_rng_split_label(base, "examples");
  double* teacher = (double*)malloc(sizeof(double) * in_w * out_w);
  double* logits = (double*)malloc(sizeof(double) * out_w);
  const double scale = 1.0 / sqrt((double)in_w);
  for (uint64_t k = 0; k < in_w * out_w; ++k) teacher[k] = vo_rng_normal(tkey, k) * scale;
  for (uint64_t r = 0; r < count; ++r) { /* data.cpp:67-105 */
    const uint64_t id = (start + r) % n;
    double* xr = x + r * in_w;
    for (uint64_t j = 0; j < in_w; ++j) xr[j] = vo_rng_normal(xkey, id * in_w + j);
    double mx = -1e300;
    for (uint64_t o = 0; o < out_w; ++o) {
      double z = 0.0;
      for (uint64_t j = 0; j < in_w; ++j) z += xr[j] * teacher[j * out_w + o];
      logits[o] = z;
      if (z > mx) mx = z;
    }
    double norm = 0.0;
    for (uint64_t o = 0; o < out_w; ++o) {
      logits[o] = exp(logits[o] - mx);
      norm += logits[o];
    }
    for (uint64_t o = 0; o < out_w; ++o) y[r * out_w + o] = logits[o] / norm;
  }
  free(teacher);
  free(logits);
  return 0;
}

/* -------------------------------------------------------------- model.cpp */
uint64_t vo_param_count(const uint64_t* w, uint32_t nw) {
  uint64_t p = 0;
  for (uint32_t l = 0; l + 1 < nw; ++l) p += w[l] * w[l + 1] + w[l + 1];
  return p;
}

int vo_init_params(const uint64_t* w, uint32_t nw, uint64_t seed, double* out) {
  const uint64_t key = vo_rng_split_label(vo_rng_key(seed), "init");
  uint64_t off = 0;
  for (uint32_t l = 0; l + 1 < nw; ++l) {
    const double scale = 1.0 / sqrt((double)w[l]);
    for (uint64_t k = 0; k < w[l] * w[l + 1]; ++k) out[off + k] = vo_rng_normal(key, off + k) * scale;
    off += w[l] * w[l + 1];
    for (uint64_t k = 0; k < w[l + 1]; ++k) out[off + k] = 0.0;
    off += w[l + 1];
  }
  return 0;
}

/* ----------------------------------------------- exact summation (Shewchuk) */
typedef struct {
  uint32_t n, cap;
  double* p;
} esum;

static void esum_add(esum* s, double x) {
  if (x == 0.0) return;
  uint32_t i = 0;
  for (uint32_t j = 0; j < s->n; ++j) {
    double y = s->p[j];
    if (fabs(x) < fabs(y)) {
      const double t = x;
      x = y;
      y = t;
    }
    const double hi = x + y;
    const double lo = y - (hi - x);
    if (lo != 0.0) s->p[i++] = lo;
    x = hi;
  }
  if (i >= s->cap) {
    s->cap = s->cap ? 2 * s->cap : 4;
    s->p = (double*)realloc(s->p, sizeof(double) * s->cap);
  }
  s->p[i] = x;
  s->n = i + 1;
}

static double esum_total(const esum* s) {
  int n = (int)s->n;
  double hi = 0.0, lo = 0.0;
  if (n > 0) {
    hi = s->p[--n];
    while (n > 0) {
      const double x = hi, y = s->p[--n];
      hi = x + y;
      lo = y - (hi - x);
      if (lo != 0.0) break;
    }
    if (n > 0 && ((lo < 0.0 && s->p[n - 1] < 0.0) || (lo > 0.0 && s->p[n - 1] > 0.0))) {
      const double y = lo * 2.0;
      const double x = hi + y;
      if (y == x - hi) hi = x;
    }
  }
  return hi;
}

static void esum_merge(esum* into, const esum* from) {
  for (uint32_t i = 0; i < from->n; ++i) esum_add(into, from->p[i]);
}

static void esum_clear(esum* s) { s->n = 0; }

/* Per-example forward/backward, model.cpp:238-343, adding into exact sums. */
typedef struct {
  const uint64_t* w;
  uint32_t nw;
  int act, loss;
  uint64_t P;
  uint64_t *woff, *boff;
  double **pre, **a, *delta, *dprev, *grad, *probs;
} fbws;

static double activate(int act, double z) {
  if (act == 0) return z > 0.0 ? z : 0.0;
  if (act == 1) return tanh(z);
  return z;
}

static double activate_grad(int act, double z) {
  if (act == 0) return z > 0.0 ? 1.0 : 0.0;
  if (act == 1) {
    const double t = tanh(z);
    return 1.0 - t * t;
  }
  return 1.0;
}

static void fbws_init(fbws* ws, const uint64_t* w, uint32_t nw, int act, int loss) {
  ws->w = w;
  ws->nw = nw;
  ws->act = act;
  ws->loss = loss;
  ws->P = vo_param_count(w, nw);
  ws->woff = (uint64_t*)malloc(sizeof(uint64_t) * nw);
  ws->boff = (uint64_t*)malloc(sizeof(uint64_t) * nw);
  uint64_t off = 0, maxw = 0;
  for (uint32_t l = 0; l + 1 < nw; ++l) {
    ws->woff[l] = off;
    off += w[l] * w[l + 1];
    ws->boff[l] = off;
    off += w[l + 1];
  }
  for (uint32_t l = 0; l < nw; ++l) maxw = w[l] > maxw ? w[l] : maxw;
  ws->pre = (double**)malloc(sizeof(double*) * nw);
  ws->a = (double**)malloc(sizeof(double*) * nw);
  for (uint32_t l = 0; l < nw; ++l) {
    ws->pre[l] = (double*)calloc(w[l], sizeof(double));
    ws->a[l] = (double*)calloc(w[l], sizeof(double));
  }
  ws->delta = (double*)calloc(maxw, sizeof(double));
  ws->dprev = (double*)calloc(maxw, sizeof(double));
  ws->grad = (double*)calloc(ws->P, sizeof(double));
  ws->probs = (double*)calloc(w[nw - 1], sizeof(double));
}

static void fbws_free(fbws* ws) {
  for (uint32_t l = 0; l < ws->nw; ++l) {
    free(ws->pre[l]);
    free(ws->a[l]);
  }
  free(ws->pre);
  free(ws->a);
  free(ws->delta);
  free(ws->dprev);
  free(ws->grad);
  free(ws->probs);
  free(ws->woff);
  free(ws->boff);
}

/* One example: fills ws->grad, returns the example loss. */
static double example_grad(fbws* ws, const double* params, const double* x, const double* y) {
  const uint64_t* w = ws->w;
  const uint32_t L = ws->nw - 1;
  memcpy(ws->a[0], x, sizeof(double) * w[0]);
  for (uint32_t l = 0; l < L; ++l) { /* model.cpp:275-287 */
    const uint64_t in = w[l], out = w[l + 1];
    const double* W = params + ws->woff[l];
    const double* b = params + ws->boff[l];
    for (uint64_t o = 0; o < out; ++o) {
      double z = b[o];
      for (uint64_t i = 0; i < in; ++i) z += ws->a[l][i] * W[i * out + o];
      ws->pre[l + 1][o] = z;
      ws->a[l + 1][o] = (l + 1 < L) ? activate(ws->act, z) : z;
    }
  }
  const uint64_t ow = w[L];
  const double* oa = ws->a[L];
  double loss = 0.0;
  if (ws->loss == 0) { /* model.cpp:294-302 */
    for (uint64_t o = 0; o < ow; ++o) {
      const double d = oa[o] - y[o];
      loss += d * d;
      ws->delta[o] = 2.0 * d / (double)ow;
    }
    loss /= (double)ow;
  } else { /* model.cpp:303-315 */
    double mx = oa[0];
    for (uint64_t o = 1; o < ow; ++o) mx = oa[o] > mx ? oa[o] : mx;
    double norm = 0.0;
    for (uint64_t o = 0; o < ow; ++o) {
      ws->probs[o] = exp(oa[o] - mx);
      norm += ws->probs[o];
    }
    const double lognorm = log(norm);
    for (uint64_t o = 0; o < ow; ++o) {
      ws->probs[o] /= norm;
      loss -= y[o] * (oa[o] - mx - lognorm);
      ws->delta[o] = ws->probs[o] - y[o];
    }
  }
  for (uint32_t l = L; l-- > 0;) { /* model.cpp:317-338 */
    const uint64_t in = w[l], out = w[l + 1];
    double* gw = ws->grad + ws->woff[l];
    double* gb = ws->grad + ws->boff[l];
    for (uint64_t o = 0; o < out; ++o) gb[o] = ws->delta[o];
    for (uint64_t i = 0; i < in; ++i)
      for (uint64_t o = 0; o < out; ++o) gw[i * out + o] = ws->a[l][i] * ws->delta[o];
    if (l > 0) {
      const double* W = params + ws->woff[l];
      for (uint64_t i = 0; i < in; ++i) {
        double acc = 0.0;
        for (uint64_t o = 0; o < out; ++o) acc += W[i * out + o] * ws->delta[o];
        ws->dprev[i] = acc * activate_grad(ws->act, ws->pre[l][i]);
      }
      double* t = ws->delta;
      ws->delta = ws->dprev;
      ws->dprev = t;
    }
  }
  return loss;
}

static esum* esum_vec(uint64_t n) { return (esum*)calloc(n, sizeof(esum)); }

static void esum_vec_free(esum* v, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) free(v[i].p);
  free(v);
}

int vo_forward_backward(const uint64_t* w, uint32_t nw, int act, int loss,
                        const double* params, const double* x, const double* y,
                        uint64_t count, double* grads, double* loss_out) {
  fbws ws;
  fbws_init(&ws, w, nw, act, loss);
  esum* g = esum_vec(ws.P);
  esum ls = {0, 0, NULL};
  for (uint64_t r = 0; r < count; ++r) {
    esum_add(&ls, example_grad(&ws, params, x + r * w[0], y + r * w[nw - 1]));
    for (uint64_t k = 0; k < ws.P; ++k) esum_add(&g[k], ws.grad[k]);
  }
  const double inv = 1.0 / (double)count; /* model.cpp:352-356 */
  for (uint64_t k = 0; k < ws.P; ++k) grads[k] = esum_total(&g[k]) * inv;
  *loss_out = esum_total(&ls) * inv;
  esum_vec_free(g, ws.P);
  free(ls.p);
  fbws_free(&ws);
  return 0;
}

int vo_forward_backward_wide_masked(const uint64_t* w, uint32_t nw, int act, int loss,
                                    const double* params, const double* x, const double* y,
                                    uint64_t count, const float* const* act_ext, double tau,
                                    double* grads, double* loss_out, uint64_t* n_amb,
                                    uint64_t* n_conf);

/* Wide-model variant of vo_forward_backward (same per-example arithmetic,
 * model.cpp:270-338, without materialising the P-sized per-example gradient):
 * per-example activations and deltas are kept (examples in parallel), then
 * each gradient element sum_r a_r[i] d_r[o] over examples ascending is
 * accumulated with Neumaier compensation — within an ulp or two of the exactly
 * rounded sum the reference's ExactVectorAccumulator produces (tests pin it
 * to vo_forward_backward on small models) — and scaled by 1/count. */
int vo_forward_backward_wide(const uint64_t* w, uint32_t nw, int act, int loss,
                             const double* params, const double* x, const double* y,
                             uint64_t count, double* grads, double* loss_out) {
  return vo_forward_backward_wide_masked(w, nw, act, loss, params, x, y, count, NULL, 0.0, grads,
                                         loss_out, NULL, NULL);
}

/* relu only: where |z| <= tau * max_o |z| for a hidden unit of an example
 * (an fp32 computation cannot resolve the sign there), relu' is taken from
 * the caller's activations act_ext[l][r * w[l] + o] > 0 instead of z > 0
 * (counted in *n_amb); elsewhere a disagreement between the two signs is
 * counted in *n_conf. */
int vo_forward_backward_wide_masked(const uint64_t* w, uint32_t nw, int act, int loss,
                                    const double* params, const double* x, const double* y,
                                    uint64_t count, const float* const* act_ext, double tau,
                                    double* grads, double* loss_out, uint64_t* n_amb,
                                    uint64_t* n_conf) {
  const uint32_t L = nw - 1;
  uint64_t sw = 0, woff[64], boff[64], off = 0;
  if (L > 63 || count == 0) return 1;
  for (uint32_t l = 0; l < L; ++l) {
    woff[l] = off;
    off += w[l] * w[l + 1];
    boff[l] = off;
    off += w[l + 1];
  }
  for (uint32_t l = 0; l <= L; ++l) sw += w[l];
  /* per example: a[0..L] (layer inputs / outputs) and d[1..L] (dLoss/dz) */
  double* A = (double*)malloc(sizeof(double) * sw * count);
  double* D = (double*)malloc(sizeof(double) * sw * count);
  double* EL = (double*)malloc(sizeof(double) * count);
  unsigned char* MK = (unsigned char*)calloc(sw * count, 1);   /* relu' per hidden unit */
  uint64_t amb = 0, conf = 0;
  uint64_t aoff[65];
  aoff[0] = 0;
  for (uint32_t l = 0; l < L; ++l) aoff[l + 1] = aoff[l] + w[l];
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : amb, conf)
  for (uint64_t r = 0; r < count; ++r) {
    double* a = A + r * sw;
    unsigned char* mk = MK + r * sw;
    double* d = D + r * sw;
    double* pre = (double*)malloc(sizeof(double) * sw);
    memcpy(a, x + r * w[0], sizeof(double) * w[0]);
    for (uint32_t l = 0; l < L; ++l) {
      const uint64_t in = w[l], out = w[l + 1];
      const double* W = params + woff[l];
      double* z = pre + aoff[l + 1];
      for (uint64_t o = 0; o < out; ++o) z[o] = params[boff[l] + o];
      for (uint64_t i = 0; i < in; ++i) {   /* i ascending per output, as the reference */
        const double ai = a[aoff[l] + i];
        const double* Wr = W + i * out;
        for (uint64_t o = 0; o < out; ++o) z[o] += ai * Wr[o];
      }
      double zmax = 0.0;
      for (uint64_t o = 0; o < out; ++o) zmax = fabs(z[o]) > zmax ? fabs(z[o]) : zmax;
      for (uint64_t o = 0; o < out; ++o) {
        if (l + 1 == L) {
          a[aoff[l + 1] + o] = z[o];
          continue;
        }
        a[aoff[l + 1] + o] = activate(act, z[o]);
        mk[aoff[l + 1] + o] = z[o] > 0.0;
        if (act == 0 && act_ext && act_ext[l + 1]) {
          const int on = act_ext[l + 1][r * out + o] > 0.0f;
          if (fabs(z[o]) <= tau * zmax) {
            amb += on != (z[o] > 0.0);
            mk[aoff[l + 1] + o] = (unsigned char)on;
            a[aoff[l + 1] + o] = on ? fabs(z[o]) : 0.0;
          } else {
            conf += on != (z[o] > 0.0);
          }
        }
      }
    }
    const uint64_t ow = w[L];
    const double* oa = a + aoff[L];
    double* dl = d + aoff[L];
    double lo = 0.0;
    if (loss == 0) {
      for (uint64_t o = 0; o < ow; ++o) {
        const double df = oa[o] - y[r * ow + o];
        lo += df * df;
        dl[o] = 2.0 * df / (double)ow;
      }
      lo /= (double)ow;
    } else {
      double mx = oa[0];
      for (uint64_t o = 1; o < ow; ++o) mx = oa[o] > mx ? oa[o] : mx;
      double norm = 0.0;
      for (uint64_t o = 0; o < ow; ++o) {
        dl[o] = exp(oa[o] - mx);
        norm += dl[o];
      }
      const double lognorm = log(norm);
      for (uint64_t o = 0; o < ow; ++o) {
        dl[o] /= norm;
        lo -= y[r * ow + o] * (oa[o] - mx - lognorm);
        dl[o] = dl[o] - y[r * ow + o];
      }
    }
    EL[r] = lo;
    for (uint32_t l = L - 1; l >= 1; --l) {
      const uint64_t in = w[l], out = w[l + 1];
      const double* W = params + woff[l];
      const double* dn = d + aoff[l + 1];
      for (uint64_t i = 0; i < in; ++i) {
        double acc = 0.0;
        const double* Wr = W + i * out;
        for (uint64_t o = 0; o < out; ++o) acc += Wr[o] * dn[o];
        d[aoff[l] + i] = act == 0 ? (mk[aoff[l] + i] ? acc : 0.0)
                                  : acc * activate_grad(act, pre[aoff[l] + i]);
      }
    }
    free(pre);
  }
  const double inv = 1.0 / (double)count;
  for (uint32_t l = 0; l < L; ++l) {
    const uint64_t in = w[l], out = w[l + 1];
#pragma omp parallel for schedule(static)
    for (uint64_t i = 0; i <= in; ++i) {   /* i == in: the bias */
      double* s = (double*)calloc(out, sizeof(double));
      double* c = (double*)calloc(out, sizeof(double));
      for (uint64_t r = 0; r < count; ++r) {
        const double ai = i < in ? A[r * sw + aoff[l] + i] : 1.0;
        const double* dn = D + r * sw + aoff[l + 1];
        for (uint64_t o = 0; o < out; ++o) {
          const double v = ai * dn[o], t = s[o] + v;
          c[o] += fabs(s[o]) >= fabs(v) ? (s[o] - t) + v : (v - t) + s[o];
          s[o] = t;
        }
      }
      double* g = grads + (i < in ? woff[l] + i * out : boff[l]);
      for (uint64_t o = 0; o < out; ++o) g[o] = (s[o] + c[o]) * inv;
      free(s);
      free(c);
    }
  }
  esum ls = {0, 0, NULL};
  for (uint64_t r = 0; r < count; ++r) esum_add(&ls, EL[r]);
  *loss_out = esum_total(&ls) * inv;
  free(ls.p);
  free(A);
  free(D);
  free(EL);
  free(MK);
  if (n_amb) *n_amb = amb;
  if (n_conf) *n_conf = conf;
  return 0;
}

void vo_sgd_momentum(double* w, double* v, const double* g, uint64_t n, double lr, double mu) {
  for (uint64_t i = 0; i < n; ++i) {
    v[i] = mu * v[i] + g[i];
    w[i] -= lr * v[i];
  }
}

/* ------------------------------------------------ LayerStats, model.cpp:101-139 */
typedef struct {
  double count;
  double *mean, *m2;
} lstats;

static void lstats_combine(lstats* a, const lstats* b, uint64_t width) {
  if (b->count == 0) return;
  if (a->count == 0) {
    a->count = b->count;
    memcpy(a->mean, b->mean, sizeof(double) * width);
    memcpy(a->m2, b->m2, sizeof(double) * width);
    return;
  }
  const double n = a->count + b->count;
  for (uint64_t j = 0; j < width; ++j) {
    const double delta = b->mean[j] - a->mean[j];
    a->m2[j] += b->m2[j] + delta * delta * (a->count * b->count / n);
    a->mean[j] += delta * (b->count / n);
  }
  a->count = n;
}

static void lstats_observe(lstats* s, uint64_t rows, uint64_t width, const double* data,
                           lstats* scratch) {
  if (rows == 0) return;
  scratch->count = (double)rows;
  for (uint64_t j = 0; j < width; ++j) scratch->mean[j] = scratch->m2[j] = 0.0;
  for (uint64_t r = 0; r < rows; ++r)
    for (uint64_t j = 0; j < width; ++j) scratch->mean[j] += data[r * width + j];
  for (uint64_t j = 0; j < width; ++j) scratch->mean[j] /= scratch->count;
  for (uint64_t r = 0; r < rows; ++r)
    for (uint64_t j = 0; j < width; ++j) {
      const double d = data[r * width + j] - scratch->mean[j];
      scratch->m2[j] += d * d;
    }
  lstats_combine(s, scratch, width);
}

/* ------------------------------------------- Trainer (runner + virtual_exec) */
typedef struct {
  char id[32];
  lstats st;
} odev;

typedef struct {
  uint64_t* w;
  uint32_t nw;
  int act, loss;
  uint64_t B, V, n, data_seed, step;
  double lr;
  uint64_t P;
  double* params;
  uint32_t G;
  odev* devs;          /* sorted by id (World order) */
  uint32_t* node_dev;  /* node -> index into devs */
  fbws ws;
  esum* dev_acc;
  double *x, *y;
  lstats scratch;
} otrainer;

static int cmp_dev(const void* a, const void* b) { return strcmp(((const odev*)a)->id, ((const odev*)b)->id); }

static void lstats_alloc(lstats* s, uint64_t w) {
  s->count = 0;
  s->mean = (double*)calloc(w, sizeof(double));
  s->m2 = (double*)calloc(w, sizeof(double));
}

void* vo_trainer_create(const uint64_t* widths, uint32_t nw, int act, int loss, uint64_t seed,
                        uint64_t B, uint64_t V, double lr, uint64_t data_seed,
                        uint64_t dataset_size, uint32_t G) {
  if (nw < 2 || B == 0 || V == 0 || B % V != 0 || G == 0 || V < G || !(lr > 0)) return NULL;
  otrainer* t = (otrainer*)calloc(1, sizeof(otrainer));
  t->w = (uint64_t*)malloc(sizeof(uint64_t) * nw);
  memcpy(t->w, widths, sizeof(uint64_t) * nw);
  t->nw = nw;
  t->act = act;
  t->loss = loss;
  t->B = B;
  t->V = V;
  t->n = dataset_size ? dataset_size : B;
  t->data_seed = data_seed;
  t->lr = lr;
  t->P = vo_param_count(widths, nw);
  t->params = (double*)malloc(sizeof(double) * t->P);
  vo_init_params(widths, nw, seed, t->params);
  t->G = G;
  t->devs = (odev*)calloc(G, sizeof(odev));
  for (uint32_t d = 0; d < G; ++d) {
    snprintf(t->devs[d].id, sizeof t->devs[d].id, "gpu%u", d);
    lstats_alloc(&t->devs[d].st, widths[0]);
  }
  /* make_uniform_mapping deals nodes over the devices in *input* order
   * (virtual_exec.cpp:94-97); the World is sorted by id (.cpp:200-203). */
  t->node_dev = (uint32_t*)malloc(sizeof(uint32_t) * V);
  char name[32];
  qsort(t->devs, G, sizeof(odev), cmp_dev);
  for (uint64_t k = 0; k < V; ++k) {
    snprintf(name, sizeof name, "gpu%u", (unsigned)(k % G));
    for (uint32_t d = 0; d < G; ++d)
      if (!strcmp(t->devs[d].id, name)) t->node_dev[k] = d;
  }
  fbws_init(&t->ws, t->w, nw, act, loss);
  t->dev_acc = esum_vec(t->P);
  t->x = (double*)malloc(sizeof(double) * B * widths[0]);
  t->y = (double*)malloc(sizeof(double) * B * widths[nw - 1]);
  lstats_alloc(&t->scratch, widths[0]);
  return t;
}

void vo_trainer_destroy(void* h) {
  otrainer* t = (otrainer*)h;
  if (!t) return;
  for (uint32_t d = 0; d < t->G; ++d) {
    free(t->devs[d].st.mean);
    free(t->devs[d].st.m2);
  }
  free(t->devs);
  free(t->node_dev);
  esum_vec_free(t->dev_acc, t->P);
  fbws_free(&t->ws);
  free(t->x);
  free(t->y);
  free(t->scratch.mean);
  free(t->scratch.m2);
  free(t->params);
  free(t->w);
  free(t);
}

int vo_trainer_step(void* h, double* loss_out) {
  otrainer* t = (otrainer*)h;
  const uint64_t in = t->w[0], ow = t->w[t->nw - 1], micro = t->B / t->V;
  vo_synth_batch(t->data_seed, t->n, in, ow, (t->step * t->B) % t->n, t->B, t->x, t->y);
  /* Exact sums are order-free, so one accumulator over all devices' nodes gives
   * the same merged result as per-device buffers merged by id
   * (virtual_exec.cpp:146-168). Stats are per device, nodes ascending. */
  for (uint64_t k = 0; k < t->P; ++k) esum_clear(&t->dev_acc[k]);
  esum ls = {0, 0, NULL};
  for (uint32_t d = 0; d < t->G; ++d) {
    for (uint64_t node = 0; node < t->V; ++node) {
      if (t->node_dev[node] != d) continue;
      const double* xs = t->x + node * micro * in;
      const double* ys = t->y + node * micro * ow;
      for (uint64_t r = 0; r < micro; ++r) {
        esum_add(&ls, example_grad(&t->ws, t->params, xs + r * in, ys + r * ow));
        for (uint64_t k = 0; k < t->P; ++k) esum_add(&t->dev_acc[k], t->ws.grad[k]);
      }
      lstats_observe(&t->devs[d].st, micro, in, xs, &t->scratch);
    }
  }
  const double inv = 1.0 / (double)t->B;
  for (uint64_t k = 0; k < t->P; ++k) {
    const double g = esum_total(&t->dev_acc[k]) * inv;
    t->params[k] -= t->lr * g; /* model.cpp:370-372 */
  }
  if (loss_out) *loss_out = esum_total(&ls) / (double)t->B;
  free(ls.p);
  t->step += 1;
  return 0;
}

int vo_trainer_params(void* h, double* out, uint64_t n) {
  otrainer* t = (otrainer*)h;
  if (n != t->P) return 6;
  memcpy(out, t->params, sizeof(double) * n);
  return 0;
}

int vo_trainer_input_stats(void* h, uint32_t idx, double* count, double* mean, double* m2,
                           uint64_t width) {
  otrainer* t = (otrainer*)h;
  if (idx >= t->G || width != t->w[0]) return 6;
  *count = t->devs[idx].st.count;
  memcpy(mean, t->devs[idx].st.mean, sizeof(double) * width);
  memcpy(m2, t->devs[idx].st.m2, sizeof(double) * width);
  return 0;
}

int vo_trainer_resize(void* h, uint32_t G2) {
  otrainer* t = (otrainer*)h;
  if (G2 == 0 || G2 > t->V) return 2;
  const uint64_t in = t->w[0];
  odev* nd = (odev*)calloc(G2, sizeof(odev));
  for (uint32_t d = 0; d < G2; ++d) snprintf(nd[d].id, sizeof nd[d].id, "gpu%u", d);
  qsort(nd, G2, sizeof(odev), cmp_dev);
  /* survivors / removed / added in ascending id (elastic.cpp:151-168) */
  uint32_t *surv = malloc(sizeof(uint32_t) * t->G), ns = 0;   /* old index */
  uint32_t *rem = malloc(sizeof(uint32_t) * t->G), nr = 0;    /* old index */
  uint32_t *add = malloc(sizeof(uint32_t) * G2), na = 0;      /* new index */
  for (uint32_t d = 0; d < t->G; ++d) {
    int found = 0;
    for (uint32_t e = 0; e < G2; ++e) found |= !strcmp(t->devs[d].id, nd[e].id);
    if (found) surv[ns++] = d; else rem[nr++] = d;
  }
  for (uint32_t e = 0; e < G2; ++e) {
    int found = 0;
    for (uint32_t d = 0; d < t->G; ++d) found |= !strcmp(t->devs[d].id, nd[e].id);
    if (!found) add[na++] = e;
  }
  if (ns == 0) { free(nd); free(surv); free(rem); free(add); return 8; }
  /* removed lineages merge into survivors round-robin (elastic.cpp:162-165, 201-219) */
  for (uint32_t s = 0; s < ns; ++s)
    for (uint32_t i = s; i < nr; i += ns)
      lstats_combine(&t->devs[surv[s]].st, &t->devs[rem[i]].st, in);
  for (uint32_t e = 0; e < G2; ++e) {
    lstats_alloc(&nd[e].st, in);
    for (uint32_t d = 0; d < t->G; ++d)
      if (!strcmp(t->devs[d].id, nd[e].id)) lstats_combine(&nd[e].st, &t->devs[d].st, in);
  }
  /* added devices copy a survivor's (post-merge) state (elastic.cpp:166-168, 222-236) */
  for (uint32_t i = 0; i < na; ++i) {
    const lstats* src = &t->devs[surv[i % ns]].st;
    lstats_combine(&nd[add[i]].st, src, in);
  }
  for (uint32_t d = 0; d < t->G; ++d) {
    free(t->devs[d].st.mean);
    free(t->devs[d].st.m2);
  }
  free(t->devs);
  t->devs = nd;
  t->G = G2;
  /* node n -> sorted_new[n % G'] (elastic.cpp:137-141) */
  for (uint64_t k = 0; k < t->V; ++k) t->node_dev[k] = (uint32_t)(k % G2);
  free(surv);
  free(rem);
  free(add);
  return 0;
}
