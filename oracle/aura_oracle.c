/*
 * aura_oracle.c -- TEST INFRASTRUCTURE ONLY. CPU restatement of the
 * reference hot path; see aura_oracle.h for the anchors and the pinning
 * status. Compiled with -O2 -ffp-contract=off so every real operation
 * rounds exactly as the reference's (the C-vs-reference comparison in
 * tests/test_oracle.py is bit-exact).
 *
 * Channel loops run on OpenMP threads (so the full-length parity runs at the
 * BASELINE sizes take seconds, not minutes); every channel's arithmetic is
 * unchanged and every cross-channel sum stays serial in channel order, so
 * the results are bit-identical to a single-threaded run.
 *
 * This file is the checker for the CUDA product in paper_2509_04390_b200/;
 * the product never links or calls it.
 */
#include "aura_oracle.h"

/* real = float: the restatement (bit-exact to the reference). real = double
 * (-DAO_F64, liboracle64.so): the same algorithm in float64 with exact
 * twiddles -- the ground truth the fp32 implementations (reference, oracle,
 * GPU) are measured against at full stream lengths, where their own
 * accumulation error over K ~ 10^4 partitions is ~1e-5 of the RMS. */
typedef ao_real real;

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int n_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
static int thread_id(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}
/* parallelise a channel loop only when it carries real work */
#define AO_PAR_MIN_WORK ((size_t)1 << 18)

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

typedef struct { real re, im; } cf;

static inline cf cmul(cf a, cf b) { /* (ac - bd, ad + bc) as libstdc++ */
  cf r;
  r.re = a.re * b.re - a.im * b.im;
  r.im = a.re * b.im + a.im * b.re;
  return r;
}
static inline cf cadd(cf a, cf b) { cf r = {a.re + b.re, a.im + b.im}; return r; }
static inline cf csub(cf a, cf b) { cf r = {a.re - b.re, a.im - b.im}; return r; }
static inline cf cconj(cf a) { cf r = {a.re, -a.im}; return r; }
static inline cf cscale(real s, cf a) { cf r = {a.re * s, a.im * s}; return r; }

/* ------------------------------------------------------------------ DFT */
/* dft.hpp:34-63: twiddles in double, stored as float (f64 build: double); bit-reverse table. */
struct ao_plan {
  size_t size, half;
  cf* stage_tw;  /* half/2 entries, e^{-2 pi i j / half} */
  cf* split_tw;  /* half/2 + 1 entries, e^{-2 pi i j / size} */
  size_t* bitrev;
  cf* work;
};

ao_plan* ao_plan_new(size_t fft_size) {
  if (fft_size < 32 || (fft_size & (fft_size - 1))) return NULL;
  ao_plan* p = (ao_plan*)calloc(1, sizeof(ao_plan));
  p->size = fft_size;
  p->half = fft_size / 2;
  p->stage_tw = (cf*)malloc(sizeof(cf) * (p->half / 2));
  p->split_tw = (cf*)malloc(sizeof(cf) * (p->half / 2 + 1));
  p->bitrev = (size_t*)malloc(sizeof(size_t) * p->half);
  p->work = (cf*)malloc(sizeof(cf) * p->half);
  const double step = -2.0 * M_PI / (double)p->half;
  for (size_t j = 0; j < p->half / 2; ++j) {
    p->stage_tw[j].re = (real)cos(step * (double)j);
    p->stage_tw[j].im = (real)sin(step * (double)j);
  }
  const double sstep = -2.0 * M_PI / (double)p->size;
  for (size_t j = 0; j <= p->half / 2; ++j) {
    p->split_tw[j].re = (real)cos(sstep * (double)j);
    p->split_tw[j].im = (real)sin(sstep * (double)j);
  }
  for (size_t i = 0; i < p->half; ++i) {
    size_t r = 0, v = i;
    for (size_t b = p->half >> 1; b; b >>= 1) { r = (r << 1) | (v & 1); v >>= 1; }
    p->bitrev[i] = r;
  }
  return p;
}

void ao_plan_free(ao_plan* p) {
  if (!p) return;
  free(p->stage_tw); free(p->split_tw); free(p->bitrev); free(p->work);
  free(p);
}

/* dft.hpp:163-176: iterative radix-2 butterflies over a bit-reversed array */
static void fft_core(const ao_plan* p, cf* z) {
  const size_t n = p->half;
  for (size_t len = 2; len <= n; len <<= 1) {
    const size_t stride = n / len, h = len / 2;
    for (size_t base = 0; base < n; base += len)
      for (size_t k = 0; k < h; ++k) {
        const cf w = p->stage_tw[k * stride];
        const cf u = z[base + k];
        const cf v = cmul(z[base + k + h], w);
        z[base + k] = cadd(u, v);
        z[base + k + h] = csub(u, v);
      }
  }
}

/* dft.hpp:69-101 (z: n_f/2 complex scratch) */
static void forward_w(const ao_plan* p, const real* buf, real* spec_f, cf* z) {
  cf* spec = (cf*)spec_f;
  const size_t n = p->half;
  for (size_t m = 0; m < n; ++m) {
    z[p->bitrev[m]].re = buf[2 * m];
    z[p->bitrev[m]].im = buf[2 * m + 1];
  }
  fft_core(p, z);
  spec[0].re = z[0].re + z[0].im; spec[0].im = 0.0f;
  spec[n].re = z[0].re - z[0].im; spec[n].im = 0.0f;
  const cf mhalf_i = {0.0f, -0.5f};
  for (size_t k = 1; k <= n / 2; ++k) {
    const cf a = z[k];
    const cf b = cconj(z[n - k]);
    const cf even = cscale(0.5f, cadd(a, b));
    const cf odd = cmul(mhalf_i, csub(a, b));
    const cf rot = cmul(p->split_tw[k], odd);
    spec[k] = cadd(even, rot);
    spec[n - k] = cconj(csub(even, rot));
  }
}

void ao_forward(const ao_plan* p, const real* buf, real* spec_f) { forward_w(p, buf, spec_f, p->work); }

/* dft.hpp:124-153 (inverse_unchecked: edge imaginary parts ignored) */
static void inverse_w(const ao_plan* p, const real* spec_f, real* buf, cf* z) {
  const cf* spec = (const cf*)spec_f;
  const size_t n = p->half;
  {
    const real xe = 0.5f * (spec[0].re + spec[n].re);
    const real xo = 0.5f * (spec[0].re - spec[n].re);
    cf t = {xe, xo};
    z[p->bitrev[0]] = cconj(t);
  }
  const cf unit_i = {0.0f, 1.0f};
  for (size_t k = 1; k < n; ++k) {
    const size_t kc = n - k;
    const cf a = spec[k];
    const cf b = cconj(spec[kc]);
    const cf even = cscale(0.5f, cadd(a, b));
    cf tw;
    if (k <= n / 2) tw = p->split_tw[k];
    else { cf s = cconj(p->split_tw[kc]); tw.re = -s.re; tw.im = -s.im; }
    const cf odd = cmul(cconj(tw), cscale(0.5f, csub(a, b)));
    z[p->bitrev[k]] = cconj(cadd(even, cmul(unit_i, odd)));
  }
  fft_core(p, z);
  const real scale = 1.0f / (real)n;
  for (size_t m = 0; m < n; ++m) {
    buf[2 * m] = z[m].re * scale;
    buf[2 * m + 1] = -z[m].im * scale;
  }
}

void ao_inverse(const ao_plan* p, const real* spec_f, real* buf) { inverse_w(p, spec_f, buf, p->work); }

/* ------------------------------------------------------------ convolver */
/* One UPOLS engine = convolver.hpp:65-220 with its FDL (engine.hpp:233-279).
 * MIMO (Appendix B) = Q broadcast engines whose outputs are summed in q
 * order, the composition the survey pins. */
typedef struct {
  size_t N, bins, K, in_ch, out_ch, n_h;
  int elementwise;
  ao_plan* plan;
  cf* H;        /* out_ch x K x bins  (convolver.hpp:19-46 layout) */
  cf* fdl;      /* fdl_ch x K x bins */
  size_t* head; /* fdl_ch */
  size_t fdl_ch;
  real* window; /* in_ch x 2N */
  cf* acc;       /* bins */
  real* time;   /* 2N */
  real* pad;    /* 2N */
  int nt;        /* per-thread scratch: */
  cf* tacc;      /*   nt x bins */
  real* ttime;  /*   nt x 2N */
  cf* twork;     /*   nt x N (FFT work) */
} upols;

static void upols_partition(upols* u, size_t row, const real* taps) {
  /* convolver.hpp:19-46: split into K blocks of N taps, zero-pad to 2N */
  const int t = thread_id();
  real* pad = u->ttime + (size_t)t * 2 * u->N;
  for (size_t k = 0; k < u->K; ++k) {
    const size_t begin = k * u->N;
    size_t n = u->n_h - begin;
    if (n > u->N) n = u->N;
    memset(pad, 0, sizeof(real) * 2 * u->N);
    memcpy(pad, taps + begin, sizeof(real) * n);
    forward_w(u->plan, pad, (real*)(u->H + (row * u->K + k) * u->bins), u->twork + (size_t)t * u->N);
  }
}

static void upols_partition_rows(upols* u, size_t rows, const real* filters) {
#pragma omp parallel for schedule(dynamic, 1) if (rows * u->K * u->bins >= AO_PAR_MIN_WORK)
  for (size_t c = 0; c < rows; ++c) upols_partition(u, c, filters + c * u->n_h);
}

static int upols_init(upols* u, size_t N, size_t in_ch, size_t out_ch,
                      int elementwise, const real* filters, size_t n_h) {
  memset(u, 0, sizeof(*u));
  if (n_h == 0 || out_ch == 0) return -1;
  u->N = N; u->bins = N + 1; u->n_h = n_h;
  u->K = (n_h + N - 1) / N;
  u->in_ch = in_ch; u->out_ch = out_ch; u->elementwise = elementwise;
  u->fdl_ch = elementwise ? out_ch : 1;
  u->plan = ao_plan_new(2 * N);
  if (!u->plan) return -1;
  u->H = (cf*)calloc(out_ch * u->K * u->bins, sizeof(cf));
  u->fdl = (cf*)calloc(u->fdl_ch * u->K * u->bins, sizeof(cf));
  u->head = (size_t*)calloc(u->fdl_ch, sizeof(size_t));
  u->window = (real*)calloc(in_ch * 2 * N, sizeof(real));
  u->acc = (cf*)calloc(u->bins, sizeof(cf));
  u->time = (real*)calloc(2 * N, sizeof(real));
  u->pad = (real*)calloc(2 * N, sizeof(real));
  u->nt = n_threads();
  u->tacc = (cf*)calloc((size_t)u->nt * u->bins, sizeof(cf));
  u->ttime = (real*)calloc((size_t)u->nt * 2 * N, sizeof(real));
  u->twork = (cf*)calloc((size_t)u->nt * N, sizeof(cf));
  upols_partition_rows(u, out_ch, filters);
  return 0;
}

static void upols_free(upols* u) {
  ao_plan_free(u->plan);
  free(u->H); free(u->fdl); free(u->head); free(u->window);
  free(u->acc); free(u->time); free(u->pad);
  free(u->tacc); free(u->ttime); free(u->twork);
}

static void upols_reset(upols* u) {
  memset(u->fdl, 0, sizeof(cf) * u->fdl_ch * u->K * u->bins);
  memset(u->head, 0, sizeof(size_t) * u->fdl_ch);
  memset(u->window, 0, sizeof(real) * u->in_ch * 2 * u->N);
}

static const cf* fdl_slot(const upols* u, size_t ch, size_t age) {
  const size_t phys = (u->head[ch] + age) % u->K; /* engine.hpp:261-266 */
  return u->fdl + (ch * u->K + phys) * u->bins;
}

/* convolver.hpp:180-191: window shift, append, r2c, FDL push */
static void upols_stage1(upols* u, size_t ch, const real* in) {
  real* w = u->window + ch * 2 * u->N;
  memmove(w, w + u->N, sizeof(real) * u->N);
  memcpy(w + u->N, in, sizeof(real) * u->N);
  u->head[ch] = (u->head[ch] + u->K - 1) % u->K; /* engine.hpp:250-258 */
  forward_w(u->plan, w, (real*)(u->fdl + (ch * u->K + u->head[ch]) * u->bins),
            u->twork + (size_t)thread_id() * u->N);
}

/* stage 1 of channels [0, n): independent channels, one per thread */
static void upols_stage1_all(upols* u, size_t n, const real* in) {
#pragma omp parallel for schedule(static) if (n * u->bins * 16 >= AO_PAR_MIN_WORK)
  for (size_t c = 0; c < n; ++c) upols_stage1(u, c, in + c * u->N);
}

/* backend.hpp:212-235: newest-to-oldest fp32 complex accumulation */
static void spectral_mac(const upols* u, const cf* H, size_t K, size_t fdl_ch,
                         size_t row, cf* acc) {
  for (size_t j = 0; j < u->bins; ++j) { acc[j].re = 0.0f; acc[j].im = 0.0f; }
  for (size_t k = 0; k < K; ++k) {
    const cf* x = fdl_slot(u, fdl_ch, k);
    const cf* h = H + (row * K + k) * u->bins;
    for (size_t j = 0; j < u->bins; ++j) {
      const real xr = x[j].re, xi = x[j].im, hr = h[j].re, hi = h[j].im;
      acc[j].re += xr * hr - xi * hi;
      acc[j].im += xr * hi + xi * hr;
    }
  }
}

/* MAC of row `row` of H (K partitions) against FDL channel fdl_ch, c2r,
 * keep the last N samples (convolver.hpp:193-206), in the calling thread's
 * scratch */
static void mac_c2r(upols* u, const cf* H, size_t K, size_t fdl_ch, size_t row, real* out) {
  const int t = thread_id();
  cf* acc = u->tacc + (size_t)t * u->bins;
  real* time = u->ttime + (size_t)t * 2 * u->N;
  spectral_mac(u, H, K, fdl_ch, row, acc);
  inverse_w(u->plan, (const real*)acc, time, u->twork + (size_t)t * u->N);
  memcpy(out, time + u->N, sizeof(real) * u->N);
}

/* convolver.hpp:193-206 for every output channel (independent) */
static void upols_stage23_all(upols* u, real* out) {
#pragma omp parallel for schedule(dynamic, 1) if (u->out_ch * u->K * u->bins >= AO_PAR_MIN_WORK)
  for (size_t c = 0; c < u->out_ch; ++c)
    mac_c2r(u, u->H, u->K, u->elementwise ? c : 0, c, out + c * u->N);
}

static void upols_process(upols* u, const real* in, real* out) {
  upols_stage1_all(u, u->in_ch, in);
  upols_stage23_all(u, out);
}

struct ao_conv {
  size_t N, inputs, outputs;
  int mode;
  upols* eng;  /* 1 engine, or Q engines in MIMO mode */
  size_t n_eng;
  real* tmp;  /* outputs x N */
};

ao_conv* ao_conv_new(size_t N, size_t inputs, size_t outputs, int mode,
                     const real* filters, size_t n_h) {
  if (N < 16 || N > 8192 || (N & (N - 1)) || outputs == 0 || n_h == 0) return NULL;
  if (mode == AO_BROADCAST && inputs != 1) return NULL;
  if (mode == AO_ELEMENTWISE && inputs != outputs) return NULL;
  if (mode == AO_MIMO && inputs == 0) return NULL;
  ao_conv* c = (ao_conv*)calloc(1, sizeof(ao_conv));
  c->N = N; c->inputs = inputs; c->outputs = outputs; c->mode = mode;
  c->n_eng = mode == AO_MIMO ? inputs : 1;
  c->eng = (upols*)calloc(c->n_eng, sizeof(upols));
  c->tmp = (real*)calloc(outputs * N, sizeof(real));
  for (size_t e = 0; e < c->n_eng; ++e) {
    const int ew = mode == AO_ELEMENTWISE;
    const size_t in_ch = ew ? inputs : 1;
    if (upols_init(&c->eng[e], N, in_ch, outputs, ew,
                   filters + e * outputs * n_h, n_h)) {
      ao_conv_free(c);
      return NULL;
    }
  }
  return c;
}

void ao_conv_free(ao_conv* c) {
  if (!c) return;
  for (size_t e = 0; e < c->n_eng; ++e) upols_free(&c->eng[e]);
  free(c->eng); free(c->tmp); free(c);
}

void ao_conv_process(ao_conv* c, const real* in, real* out) {
  if (c->mode != AO_MIMO) { upols_process(&c->eng[0], in, out); return; }
  /* Appendix B: l_l = sum_q H_{l,q} * m_q, summed in q order */
  upols_process(&c->eng[0], in, out);
  for (size_t q = 1; q < c->n_eng; ++q) {
    upols_process(&c->eng[q], in + q * c->N, c->tmp);
    for (size_t i = 0; i < c->outputs * c->N; ++i) out[i] += c->tmp[i];
  }
}

void ao_conv_reset(ao_conv* c) {
  for (size_t e = 0; e < c->n_eng; ++e) upols_reset(&c->eng[e]);
}

size_t ao_conv_partitions(const ao_conv* c) { return c->eng[0].K; }

void ao_conv_spectrum(const ao_conv* c, size_t row, size_t k, real* out) {
  const size_t e = row / c->outputs, r = row % c->outputs;
  const upols* u = &c->eng[e];
  memcpy(out, u->H + (r * u->K + k) * u->bins, sizeof(cf) * u->bins);
}

/* ------------------------------------------------------------ auralizer */
/* auralizer.hpp:25-123, generalised per SURVEY.md Appendix A (NLMS on the
 * feedback-canceller spectra) and Appendix B (Q = P inputs/mics). */
struct ao_aur {
  size_t N, bins, Q, L, P, K_f;
  real gain, mu, lambda, delta;
  ao_conv* synth;      /* MIMO (or broadcast when Q == 1) */
  upols fc;            /* elementwise L -> L; H holds W for mic 0 */
  cf* W;               /* P x L x K_f x bins (W[0] aliases fc.H) */
  real* fhat;         /* P x N */
  real* mt;           /* Q x N  (m~) */
  real* fc_out;       /* N */
  real* ewin;         /* 2N error window */
  cf* E;               /* bins */
  real* power;        /* bins */
  real* scale;        /* bins */
  real* fc_l;         /* L x N: per-loudspeaker canceller outputs */
  int constrained;     /* Appendix A step 2, constrained gradient */
  real* cwork;         /* per thread: G (bins cf), 2N window, N cf FFT scratch */
  int cwork_threads;   /* threads cwork was sized for (the update loop uses no more) */
};

ao_aur* ao_aur_new(size_t N, size_t Q, size_t L, const real* synth,
                   size_t n_h, const real* fc, size_t n_hf, real gain,
                   real mu, real lambda, real delta) {
  if (Q == 0 || L == 0 || n_hf == 0) return NULL;
  ao_aur* a = (ao_aur*)calloc(1, sizeof(ao_aur));
  a->N = N; a->bins = N + 1; a->Q = Q; a->L = L; a->P = Q;
  a->gain = gain; a->mu = mu; a->lambda = lambda; a->delta = delta;
  a->synth = ao_conv_new(N, Q, L, Q == 1 ? AO_BROADCAST : AO_MIMO, synth, n_h);
  if (!a->synth) { free(a); return NULL; }
  /* the FC engine owns the shared AFC FDL X_l; W per mic is partitioned
   * with the same make_partitioned_filters transform */
  if (upols_init(&a->fc, N, L, L, 1, fc, n_hf)) { ao_aur_free(a); return NULL; }
  a->K_f = a->fc.K;
  const size_t wsz = L * a->K_f * a->bins;
  a->W = (cf*)calloc(a->P * wsz, sizeof(cf));
  memcpy(a->W, a->fc.H, sizeof(cf) * wsz);
  for (size_t p = 1; p < a->P; ++p) {
    upols_partition_rows(&a->fc, L, fc + p * L * n_hf);
    memcpy(a->W + p * wsz, a->fc.H, sizeof(cf) * wsz);
  }
  memcpy(a->fc.H, a->W, sizeof(cf) * wsz);
  a->fhat = (real*)calloc(a->P * N, sizeof(real));
  a->mt = (real*)calloc(Q * N, sizeof(real));
  a->fc_out = (real*)calloc(N, sizeof(real));
  a->ewin = (real*)calloc(2 * N, sizeof(real));
  a->E = (cf*)calloc(a->bins, sizeof(cf));
  a->power = (real*)calloc(a->bins, sizeof(real));
  a->scale = (real*)calloc(a->bins, sizeof(real));
  a->fc_l = (real*)calloc(L * N, sizeof(real));
  return a;
}

void ao_aur_free(ao_aur* a) {
  if (!a) return;
  ao_conv_free(a->synth);
  upols_free(&a->fc);
  free(a->W); free(a->fhat); free(a->mt); free(a->fc_out); free(a->ewin);
  free(a->E); free(a->power); free(a->scale); free(a->fc_l); free(a->cwork);
  free(a);
}

#define AO_CWORK(N) (6 * (N) + 2)  /* reals of constrained scratch per thread */

/* The constrained gradient of one (p, l, k): G = scale (.) conj(x) E, then
 * G' = r2c([first N samples of c2r(G), 0_N]) -- DftPlan::inverse_unchecked
 * and DftPlan::forward (dft.hpp:69-153) -- and w += G'. */
static void constrained_step(const ao_aur* a, const cf* x, cf* w, real* work) {
  const size_t N = a->N, bins = a->bins;
  cf* G = (cf*)work;
  real* buf = work + 2 * bins;
  cf* z = (cf*)(buf + 2 * N);
  for (size_t j = 0; j < bins; ++j) {
    const cf g = cmul(cconj(x[j]), a->E[j]);
    G[j].re = a->scale[j] * g.re;
    G[j].im = a->scale[j] * g.im;
  }
  inverse_w(a->fc.plan, (const real*)G, buf, z);
  for (size_t i = N; i < 2 * N; ++i) buf[i] = 0.0f;
  forward_w(a->fc.plan, buf, (real*)G, z);
  for (size_t j = 0; j < bins; ++j) {
    w[j].re += G[j].re;
    w[j].im += G[j].im;
  }
}

/* Appendix A step 2: W[p][l][k] += mu/(P+delta) * conj(X_l(age k)) E_p,
 * on the AFC FDL *before* X(l_n) is pushed (constrained: see above). */
static void nlms_update(ao_aur* a) {
  const size_t N = a->N, bins = a->bins, L = a->L, Kf = a->K_f;
  for (size_t j = 0; j < bins; ++j) a->scale[j] = a->mu / (a->power[j] + a->delta);
  for (size_t p = 0; p < a->P; ++p) {
    memset(a->ewin, 0, sizeof(real) * N);
    memcpy(a->ewin + N, a->mt + p * N, sizeof(real) * N);
    ao_forward(a->fc.plan, a->ewin, (real*)a->E);
#pragma omp parallel for schedule(static) if (L * Kf * bins >= AO_PAR_MIN_WORK) \
    num_threads(a->constrained ? a->cwork_threads : n_threads())
    for (size_t l = 0; l < L; ++l)
      for (size_t k = 0; k < Kf; ++k) {
        const cf* x = fdl_slot(&a->fc, l, k);
        cf* w = a->W + ((p * L + l) * Kf + k) * bins;
        if (a->constrained) {
          constrained_step(a, x, w, a->cwork + (size_t)thread_id() * AO_CWORK(N));
          continue;
        }
        for (size_t j = 0; j < bins; ++j) {
          const cf g = cmul(cconj(x[j]), a->E[j]);
          w[j].re += a->scale[j] * g.re;
          w[j].im += a->scale[j] * g.im;
        }
      }
  }
}

int ao_aur_set_constrained(ao_aur* a, int constrained) {
  if (constrained && !a->cwork) {
    a->cwork_threads = n_threads();
    a->cwork = (real*)calloc((size_t)a->cwork_threads * AO_CWORK(a->N), sizeof(real));
    if (!a->cwork) return -1;
  }
  a->constrained = constrained != 0;
  return 0;
}

void ao_aur_process(ao_aur* a, const real* mic, real* spk) {
  const size_t N = a->N, L = a->L, bins = a->bins;
  /* auralizer.hpp:73-76: m~ = g m - f^ (mic q pairs with estimate q) */
  for (size_t q = 0; q < a->Q; ++q)
    for (size_t i = 0; i < N; ++i)
      a->mt[q * N + i] = a->gain * mic[q * N + i] - a->fhat[q * N + i];
  if (a->mu != 0.0f) nlms_update(a);
  /* auralizer.hpp:78: synthesis */
  ao_conv_process(a->synth, a->mt, spk);
  /* auralizer.hpp:79: FC stage 1 on every loudspeaker channel */
  upols_stage1_all(&a->fc, L, spk);
  /* auralizer.hpp:79-86: per channel MAC + c2r (channels in parallel),
   * summed in time in l order */
  const size_t wsz = L * a->K_f * bins;
  for (size_t p = 0; p < a->P; ++p) {
#pragma omp parallel for schedule(dynamic, 1) if (L * a->K_f * bins >= AO_PAR_MIN_WORK)
    for (size_t l = 0; l < L; ++l) mac_c2r(&a->fc, a->W + p * wsz, a->K_f, l, l, a->fc_l + l * N);
    real* f = a->fhat + p * N;
    for (size_t i = 0; i < N; ++i) f[i] = 0.0f;
    for (size_t l = 0; l < L; ++l)
      for (size_t i = 0; i < N; ++i) f[i] += a->fc_l[l * N + i];
  }
  /* Appendix A step 5: smoothed loudspeaker power for the next update */
  if (a->mu != 0.0f) {
    for (size_t j = 0; j < bins; ++j) {
      real s = 0.0f;
      for (size_t l = 0; l < L; ++l) {
        const cf x = fdl_slot(&a->fc, l, 0)[j];
        s += x.re * x.re + x.im * x.im;
      }
      a->power[j] = a->lambda * a->power[j] + (1.0f - a->lambda) * s;
    }
  }
}

void ao_aur_reset(ao_aur* a) {
  ao_conv_reset(a->synth);
  upols_reset(&a->fc);
  memset(a->fhat, 0, sizeof(real) * a->P * a->N);
  memset(a->power, 0, sizeof(real) * a->bins);
}

void ao_aur_set_gain(ao_aur* a, real gain) { a->gain = gain; }

void ao_aur_feedback_estimate(const ao_aur* a, real* out) {
  memcpy(out, a->fhat, sizeof(real) * a->P * a->N);
}

size_t ao_aur_fc_partitions(const ao_aur* a) { return a->K_f; }
size_t ao_aur_synth_partitions(const ao_aur* a) { return ao_conv_partitions(a->synth); }

void ao_aur_coeffs(const ao_aur* a, real* out) {
  memcpy(out, a->W, sizeof(cf) * a->P * a->L * a->K_f * a->bins);
}

void ao_aur_power(const ao_aur* a, real* out) {
  memcpy(out, a->power, sizeof(real) * a->bins);
}

/* oracle.hpp:15-27 */
void ao_direct_convolve(const double* x, size_t nx, const double* h, size_t nh,
                        double* y) {
  for (size_t i = 0; i < nx + nh - 1; ++i) y[i] = 0.0;
  for (size_t tau = 0; tau < nh; ++tau) {
    const double hv = h[tau];
    if (hv == 0.0) continue;
    for (size_t t = 0; t < nx; ++t) y[t + tau] += x[t] * hv;
  }
}
