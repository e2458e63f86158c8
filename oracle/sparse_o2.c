/*
 * O2: the unfold's trace definition evaluated with sparse (CSR) operators.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): a plain, slow, obviously
 * correct CPU reference.  It shares no code with the CUDA path.
 *
 * Definition followed (Eq. 1; basis P:135-144; Eq. 5 P:162-166;
 * Eq. 9):
 *
 *     Q_sm = Tr(F_s L(F_m)),     K_s = Tr(F_s L(I/N))
 *     L(X) = -i(H X - X H) + sum_p gamma_p (L_p X L_p^+ - 1/2 (L_p^+L_p X + X L_p^+L_p))
 *
 * computed COLUMN BY COLUMN: for every generator F_m (canonical order, DESIGN.md
 * R5) the matrix X = L(F_m) is formed as a list of product terms (r, c, value)
 * from the CSR operators, sorted by (r, c) and summed; then Tr(F_s X) is
 * evaluated for every F_s whose support meets X:
 *     Tr(S_ab X) = (X_ba + X_ab)/sqrt2
 *     Tr(J_ab X) = (-i X_ba + i X_ab)/sqrt2
 *     Tr(D^l X)  = (sum_{c<l} X_cc - l X_ll)/sqrt(l(l+1))
 * (the trace restricted to the nonzero entries of F_s).  Entries with
 * |Q_sm| <= tau are not stored (R6).  Columns are independent; OpenMP
 * runs them in parallel in fixed chunks whose outputs are concatenated in
 * column order, then a stable counting sort by row gives CSR with ascending
 * columns.  Deterministic for any thread count.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o liboracle_o2.so sparse_o2.c -lm
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double _Complex zd;

typedef struct {
  int n;
  int64_t *rp; /* n+1 */
  int32_t *ci; /* nnz  */
  zd *v;       /* nnz  */
} csr_t;

typedef struct {
  int32_t r, c;
  zd v;
  double a; /* sum of |term| merged into this entry (roundoff yardstick, R6) */
} term_t;

typedef struct {
  term_t *t;
  int64_t len, cap;
} tvec_t;

static void tpush(tvec_t *tv, int32_t r, int32_t c, zd v) {
  if (tv->len == tv->cap) {
    tv->cap = tv->cap ? 2 * tv->cap : 256;
    tv->t = (term_t *)realloc(tv->t, (size_t)tv->cap * sizeof(term_t));
  }
  tv->t[tv->len].r = r;
  tv->t[tv->len].c = c;
  tv->t[tv->len].v = v;
  tv->t[tv->len].a = cabs(v);
  tv->len++;
}

typedef struct {
  int32_t *s;
  int32_t *m;
  double *v;
  double *a; /* sum|terms| of the entry (condition number = a / |v|; R7) */
  int64_t len, cap;
} ovec_t;

static void opush(ovec_t *o, int32_t s, int32_t m, double v, double a) {
  if (o->len == o->cap) {
    o->cap = o->cap ? 2 * o->cap : 1024;
    o->s = (int32_t *)realloc(o->s, (size_t)o->cap * sizeof(int32_t));
    o->m = (int32_t *)realloc(o->m, (size_t)o->cap * sizeof(int32_t));
    o->v = (double *)realloc(o->v, (size_t)o->cap * sizeof(double));
    o->a = (double *)realloc(o->a, (size_t)o->cap * sizeof(double));
  }
  o->s[o->len] = s;
  o->m[o->len] = m;
  o->v[o->len] = v;
  o->a[o->len] = a;
  o->len++;
}

static int cmp_term(const void *a, const void *b) {
  const term_t *x = (const term_t *)a, *y = (const term_t *)b;
  if (x->r != y->r) return x->r < y->r ? -1 : 1;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return 0;
}

/* Transpose (no conjugation) of a CSR matrix. */
static csr_t csr_transpose(const csr_t *A) {
  csr_t T;
  int n = A->n;
  int64_t nnz = A->rp[n];
  T.n = n;
  T.rp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  T.ci = (int32_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  T.v = (zd *)malloc((size_t)(nnz ? nnz : 1) * sizeof(zd));
  for (int64_t k = 0; k < nnz; ++k) T.rp[A->ci[k] + 1]++;
  for (int i = 0; i < n; ++i) T.rp[i + 1] += T.rp[i];
  int64_t *pos = (int64_t *)malloc((size_t)n * sizeof(int64_t));
  for (int i = 0; i < n; ++i) pos[i] = T.rp[i];
  for (int r = 0; r < n; ++r)
    for (int64_t k = A->rp[r]; k < A->rp[r + 1]; ++k) {
      int32_t c = A->ci[k];
      T.ci[pos[c]] = r;
      T.v[pos[c]] = A->v[k];
      pos[c]++;
    }
  free(pos);
  return T;
}

/* C = A^+ A (conjugate transpose of A times A), Gustavson with a dense row accumulator. */
static csr_t csr_adjoint_times_self(const csr_t *A) {
  int n = A->n;
  csr_t At = csr_transpose(A); /* row k of At = column k of A */
  csr_t C;
  C.n = n;
  C.rp = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
  zd *acc = (zd *)calloc((size_t)n, sizeof(zd));
  char *mark = (char *)calloc((size_t)n, 1);
  int32_t *touched = (int32_t *)malloc((size_t)n * sizeof(int32_t));
  int64_t cap = 1024, len = 0;
  C.ci = (int32_t *)malloc((size_t)cap * sizeof(int32_t));
  C.v = (zd *)malloc((size_t)cap * sizeof(zd));
  for (int i = 0; i < n; ++i) {
    /* (A^+ A)_ij = sum_k conj(A_ki) A_kj ; k runs over column i of A */
    int nt = 0;
    for (int64_t q = At.rp[i]; q < At.rp[i + 1]; ++q) {
      int k = At.ci[q];
      zd aki = conj(At.v[q]);
      for (int64_t w = A->rp[k]; w < A->rp[k + 1]; ++w) {
        int j = A->ci[w];
        if (!mark[j]) {
          mark[j] = 1;
          touched[nt++] = j;
          acc[j] = 0;
        }
        acc[j] += aki * A->v[w];
      }
    }
    /* sort touched columns ascending (insertion sort; rows are short) */
    for (int x = 1; x < nt; ++x) {
      int32_t key = touched[x];
      int y = x - 1;
      while (y >= 0 && touched[y] > key) {
        touched[y + 1] = touched[y];
        --y;
      }
      touched[y + 1] = key;
    }
    for (int x = 0; x < nt; ++x) {
      int j = touched[x];
      mark[j] = 0;
      if (len == cap) {
        cap *= 2;
        C.ci = (int32_t *)realloc(C.ci, (size_t)cap * sizeof(int32_t));
        C.v = (zd *)realloc(C.v, (size_t)cap * sizeof(zd));
      }
      C.ci[len] = j;
      C.v[len] = acc[j];
      ++len;
    }
    C.rp[i + 1] = len;
  }
  free(acc);
  free(mark);
  free(touched);
  free(At.rp);
  free(At.ci);
  free(At.v);
  return C;
}

typedef struct {
  int n, P;
  csr_t H, Ht;             /* H and its transpose (column access) */
  csr_t *L, *Lt, *M, *Mt;  /* L_p, L_p^T, M_p = L_p^+ L_p, M_p^T */
  const double *gamma;
} model_t;

/* Append the terms of L(F) for F given as entries (fr[i], fc[i], fv[i]). */
static void lindblad_terms(const model_t *md, int nf, const int32_t *fr, const int32_t *fc,
                           const zd *fv, tvec_t *tv) {
  for (int e = 0; e < nf; ++e) {
    int k = fr[e], c = fc[e];
    zd v = fv[e];
    /* -i (H F)_rc = -i sum_k H_rk F_kc : r over column k of H */
    for (int64_t q = md->Ht.rp[k]; q < md->Ht.rp[k + 1]; ++q)
      tpush(tv, md->Ht.ci[q], c, -I * md->Ht.v[q] * v);
    /* +i (F H)_kd = +i F_kc H_cd : d over row c of H */
    for (int64_t q = md->H.rp[c]; q < md->H.rp[c + 1]; ++q)
      tpush(tv, k, md->H.ci[q], I * v * md->H.v[q]);
    for (int p = 0; p < md->P; ++p) {
      double g = md->gamma[p];
      const csr_t *Lt = &md->Lt[p], *M = &md->M[p], *Mt = &md->Mt[p];
      /* gamma (L F L^+)_rd = gamma sum L_rk F_kc conj(L_dc) : r over column k of L, d over column c of L */
      for (int64_t q = Lt->rp[k]; q < Lt->rp[k + 1]; ++q)
        for (int64_t w = Lt->rp[c]; w < Lt->rp[c + 1]; ++w)
          tpush(tv, Lt->ci[q], Lt->ci[w], g * Lt->v[q] * v * conj(Lt->v[w]));
      /* -gamma/2 (M F)_rc = -gamma/2 sum_k M_rk F_kc : r over column k of M */
      for (int64_t q = Mt->rp[k]; q < Mt->rp[k + 1]; ++q)
        tpush(tv, Mt->ci[q], c, -0.5 * g * Mt->v[q] * v);
      /* -gamma/2 (F M)_kd = -gamma/2 F_kc M_cd : d over row c of M */
      for (int64_t q = M->rp[c]; q < M->rp[c + 1]; ++q)
        tpush(tv, k, M->ci[q], -0.5 * g * v * M->v[q]);
    }
  }
}

/* Sort the terms by (r, c) and sum duplicates in place; returns number of unique entries. */
static int64_t sum_terms(tvec_t *tv) {
  if (tv->len == 0) return 0;
  qsort(tv->t, (size_t)tv->len, sizeof(term_t), cmp_term);
  int64_t u = 0;
  for (int64_t i = 1; i < tv->len; ++i) {
    if (tv->t[i].r == tv->t[u].r && tv->t[i].c == tv->t[u].c) {
      tv->t[u].v += tv->t[i].v;
      tv->t[u].a += tv->t[i].a;
    } else
      tv->t[++u] = tv->t[i];
  }
  tv->len = u + 1;
  return tv->len;
}

/* X_rc from the sorted unique terms (0 if absent); *found tells whether it is stored;
 * *absum (if given) receives the sum of |terms| merged into it. */
static zd lookup_a(const tvec_t *tv, int32_t r, int32_t c, int *found, double *absum) {
  int64_t lo = 0, hi = tv->len - 1;
  if (absum) *absum = 0.0;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    const term_t *t = &tv->t[mid];
    if (t->r == r && t->c == c) {
      if (found) *found = 1;
      if (absum) *absum = t->a;
      return t->v;
    }
    if (t->r < r || (t->r == r && t->c < c))
      lo = mid + 1;
    else
      hi = mid - 1;
  }
  if (found) *found = 0;
  return 0;
}
static zd lookup(const tvec_t *tv, int32_t r, int32_t c, int *found) { return lookup_a(tv, r, c, found, NULL); }

static inline int64_t pidx(int64_t n, int64_t a, int64_t b) { return a * (2 * n - a - 1) / 2 + (b - a - 1); }

/* Generator m as its nonzero entries (canonical order, R4/R5). */
static int generator_entries(int n, int64_t m, int32_t *fr, int32_t *fc, zd *fv) {
  int64_t np = (int64_t)n * (n - 1) / 2;
  const double is2 = 1.0 / sqrt(2.0);
  if (m < 2 * np) {
    int64_t p = m < np ? m : m - np;
    /* decode pair p -> (a, b) by walking rows (plain; O(n)) */
    int64_t a = 0, base = 0;
    while (base + (n - 1 - a) <= p) {
      base += n - 1 - a;
      ++a;
    }
    int64_t b = a + 1 + (p - base);
    fr[0] = (int32_t)a; fc[0] = (int32_t)b;
    fr[1] = (int32_t)b; fc[1] = (int32_t)a;
    if (m < np) {            /* S_ab = (E_ab + E_ba)/sqrt2 */
      fv[0] = is2; fv[1] = is2;
    } else {                 /* J_ab = -i (E_ab - E_ba)/sqrt2 */
      fv[0] = -I * is2; fv[1] = I * is2;
    }
    return 2;
  }
  int l = (int)(m - 2 * np + 1); /* D^l = (sum_{c<l} E_cc - l E_ll)/sqrt(l(l+1)) */
  double nrm = 1.0 / sqrt((double)l * (l + 1.0));
  for (int c = 0; c < l; ++c) { fr[c] = c; fc[c] = c; fv[c] = nrm; }
  fr[l] = l; fc[l] = l; fv[l] = -(double)l * nrm;
  return l + 1;
}

/* Gap diagnostics of the stored-pattern rule (R6).  min_margin: over every entry
 * with |q| <= 1e6 tau, the smallest ||q| - tau| / (1e-16 sum|terms|) -- how many per-entry
 * roundoff bounds separate the entry from the threshold (large = the keep/drop decision
 * cannot depend on the order of summation). */
typedef struct {
  double max_dropped, min_kept, max_imag, min_margin;
} gap_t;

static void note_margin(gap_t *g, double v, double absum, double tau) {
  if (tau <= 0.0 || fabs(v) > 1e6 * tau) return;
  double bound = 1e-16 * absum;
  double r = bound > 0.0 ? fabs(fabs(v) - tau) / bound : INFINITY;
  if (r < g->min_margin) g->min_margin = r;
}

/* Project X (unique sorted terms) on every F_s: emit (s, col, Re Tr(F_s X)) with |.| > tau. */
static void project_emit(int n, const tvec_t *X, int32_t col, double tau, ovec_t *out, double *dense_out,
                         double *diagbuf, gap_t *gap) {
  int64_t np = (int64_t)n * (n - 1) / 2;
  const double is2 = 1.0 / sqrt(2.0);
  /* S/J block: every unordered pair {r, c} present in X */
  for (int64_t i = 0; i < X->len; ++i) {
    int32_t r = X->t[i].r, c = X->t[i].c;
    if (r == c) continue;
    int32_t a = r < c ? r : c, b = r < c ? c : r;
    if (r > c) { /* visit the pair once: via (a, b) when that entry is stored */
      int up = 0;
      (void)lookup(X, c, r, &up);
      if (up) continue;
    }
    double aab, aba;
    zd xab = lookup_a(X, a, b, NULL, &aab), xba = lookup_a(X, b, a, NULL, &aba);
    double absum = (aab + aba) * is2; /* sum|terms| of both Tr(S_ab X) and Tr(J_ab X) */
    zd trS = (xba + xab) * is2;          /* Tr(S_ab X) */
    zd trJ = (-I * xba + I * xab) * is2; /* Tr(J_ab X) */
    int64_t p = pidx(n, a, b);
    double vals[2] = {creal(trS), creal(trJ)};
    double ims[2] = {cimag(trS), cimag(trJ)};
    int64_t rows[2] = {p, np + p};
    for (int q = 0; q < 2; ++q) {
      if (fabs(ims[q]) > gap->max_imag) gap->max_imag = fabs(ims[q]);
      if (!dense_out) note_margin(gap, vals[q], absum, tau);
      if (dense_out) {
        dense_out[rows[q]] = vals[q];
      } else if (fabs(vals[q]) > tau) {
        opush(out, (int32_t)rows[q], col, vals[q], absum);
        if (fabs(vals[q]) < gap->min_kept) gap->min_kept = fabs(vals[q]);
      } else if (fabs(vals[q]) > gap->max_dropped) {
        gap->max_dropped = fabs(vals[q]);
      }
    }
  }
  /* D block: Tr(D^l X) = (sum_{c<l} X_cc - l X_ll)/sqrt(l(l+1)), l = 1..n-1 */
  int ndiag = 0;
  for (int64_t i = 0; i < X->len; ++i)
    if (X->t[i].r == X->t[i].c) ++ndiag;
  if (ndiag == 0) return;
  for (int c = 0; c < n; ++c) diagbuf[3 * c] = diagbuf[3 * c + 1] = diagbuf[3 * c + 2] = 0.0;
  for (int64_t i = 0; i < X->len; ++i)
    if (X->t[i].r == X->t[i].c) {
      diagbuf[3 * X->t[i].r] = creal(X->t[i].v);
      diagbuf[3 * X->t[i].r + 1] = cimag(X->t[i].v);
      diagbuf[3 * X->t[i].r + 2] = X->t[i].a;
    }
  double pre_re = diagbuf[0], pre_im = diagbuf[1]; /* sum_{c<l} X_cc, starting at l = 1 */
  double pre_a = diagbuf[2];                        /* sum_{c<l} sum|terms of X_cc| */
  for (int l = 1; l < n; ++l) {
    double nrm = 1.0 / sqrt((double)l * (l + 1.0));
    double v = (pre_re - (double)l * diagbuf[3 * l]) * nrm;
    double im = (pre_im - (double)l * diagbuf[3 * l + 1]) * nrm;
    if (fabs(im) > gap->max_imag) gap->max_imag = fabs(im);
    int64_t row = 2 * np + l - 1;
    const double dabs = (pre_a + (double)l * diagbuf[3 * l + 2]) * nrm;
    if (!dense_out) note_margin(gap, v, dabs, tau);
    if (dense_out) {
      dense_out[row] = v;
    } else if (fabs(v) > tau) {
      opush(out, (int32_t)row, col, v, dabs);
      if (fabs(v) < gap->min_kept) gap->min_kept = fabs(v);
    } else if (fabs(v) > gap->max_dropped) {
      gap->max_dropped = fabs(v);
    }
    pre_re += diagbuf[3 * l];
    pre_im += diagbuf[3 * l + 1];
    pre_a += diagbuf[3 * l + 2];
  }
}

typedef struct {
  int64_t m, nnz;
  int64_t *row_ptr;
  int32_t *col;
  double *val;
  double *absv;
  double *K;
  gap_t gap;
} o2_result;

static csr_t wrap(int n, const int64_t *rp, const int32_t *ci, const double *v) {
  csr_t A;
  A.n = n;
  A.rp = (int64_t *)rp;
  A.ci = (int32_t *)ci;
  A.v = (zd *)v;
  return A;
}

/*
 * o2_unfold: Q (CSR, |q| > tau) and K for H and dissipators {L_p, gamma_p}.
 * Operators are CSR with interleaved (re, im) values.  with_k = 0 skips K.
 * nthreads <= 0 uses the OpenMP default.  Returns a heap result (free with o2_free).
 */
void *o2_unfold(int n, const int64_t *h_rp, const int32_t *h_ci, const double *h_v, int P,
                const int64_t *const *l_rp, const int32_t *const *l_ci, const double *const *l_v,
                const double *gamma, double tau, int with_k, int nthreads) {
  model_t md;
  md.n = n;
  md.P = P;
  md.H = wrap(n, h_rp, h_ci, h_v);
  md.Ht = csr_transpose(&md.H);
  md.L = (csr_t *)calloc((size_t)(P > 0 ? P : 1), sizeof(csr_t));
  md.Lt = (csr_t *)calloc((size_t)(P > 0 ? P : 1), sizeof(csr_t));
  md.M = (csr_t *)calloc((size_t)(P > 0 ? P : 1), sizeof(csr_t));
  md.Mt = (csr_t *)calloc((size_t)(P > 0 ? P : 1), sizeof(csr_t));
  for (int p = 0; p < P; ++p) {
    md.L[p] = wrap(n, l_rp[p], l_ci[p], l_v[p]);
    md.Lt[p] = csr_transpose(&md.L[p]);
    md.M[p] = csr_adjoint_times_self(&md.L[p]);
    md.Mt[p] = csr_transpose(&md.M[p]);
  }
  md.gamma = gamma;
  int64_t M = (int64_t)n * n - 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  const int64_t CH = 256;
  int64_t nch = (M + CH - 1) / CH;
  ovec_t *outs = (ovec_t *)calloc((size_t)nch, sizeof(ovec_t));
  gap_t *gaps = (gap_t *)malloc((size_t)nch * sizeof(gap_t));
#pragma omp parallel
  {
    tvec_t tv = {0, 0, 0};
    int32_t *fr = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *fc = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    zd *fv = (zd *)malloc((size_t)n * sizeof(zd));
    double *diagbuf = (double *)malloc((size_t)3 * n * sizeof(double));
#pragma omp for schedule(dynamic, 1)
    for (int64_t ch = 0; ch < nch; ++ch) {
      gap_t g = {0.0, INFINITY, 0.0, INFINITY};
      for (int64_t m = ch * CH; m < (ch + 1) * CH && m < M; ++m) {
        int nf = generator_entries(n, m, fr, fc, fv);
        tv.len = 0;
        lindblad_terms(&md, nf, fr, fc, fv, &tv);
        sum_terms(&tv);
        project_emit(n, &tv, (int32_t)m, tau, &outs[ch], NULL, diagbuf, &g);
      }
      gaps[ch] = g;
    }
    free(tv.t);
    free(fr);
    free(fc);
    free(fv);
    free(diagbuf);
  }
  o2_result *res = (o2_result *)calloc(1, sizeof(o2_result));
  res->m = M;
  res->gap.max_dropped = 0.0;
  res->gap.min_kept = INFINITY;
  res->gap.max_imag = 0.0;
  res->gap.min_margin = INFINITY;
  int64_t nnz = 0;
  for (int64_t ch = 0; ch < nch; ++ch) {
    nnz += outs[ch].len;
    if (gaps[ch].max_dropped > res->gap.max_dropped) res->gap.max_dropped = gaps[ch].max_dropped;
    if (gaps[ch].min_kept < res->gap.min_kept) res->gap.min_kept = gaps[ch].min_kept;
    if (gaps[ch].max_imag > res->gap.max_imag) res->gap.max_imag = gaps[ch].max_imag;
    if (gaps[ch].min_margin < res->gap.min_margin) res->gap.min_margin = gaps[ch].min_margin;
  }
  res->nnz = nnz;
  res->row_ptr = (int64_t *)calloc((size_t)M + 1, sizeof(int64_t));
  res->col = (int32_t *)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  res->val = (double *)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
  res->absv = (double *)malloc((size_t)(nnz ? nnz : 1) * sizeof(double));
  /* stable counting sort by row; chunks are visited in column order */
  for (int64_t ch = 0; ch < nch; ++ch)
    for (int64_t i = 0; i < outs[ch].len; ++i) res->row_ptr[outs[ch].s[i] + 1]++;
  for (int64_t s = 0; s < M; ++s) res->row_ptr[s + 1] += res->row_ptr[s];
  int64_t *pos = (int64_t *)malloc((size_t)M * sizeof(int64_t));
  memcpy(pos, res->row_ptr, (size_t)M * sizeof(int64_t));
  for (int64_t ch = 0; ch < nch; ++ch) {
    for (int64_t i = 0; i < outs[ch].len; ++i) {
      int64_t d = pos[outs[ch].s[i]]++;
      res->col[d] = outs[ch].m[i];
      res->val[d] = outs[ch].v[i];
      res->absv[d] = outs[ch].a[i];
    }
    free(outs[ch].s);
    free(outs[ch].m);
    free(outs[ch].v);
    free(outs[ch].a);
  }
  free(pos);
  free(outs);
  free(gaps);
  /* K_s = Tr(F_s L(I/N)) */
  res->K = (double *)calloc((size_t)M, sizeof(double));
  if (with_k) {
    int32_t *fr = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    int32_t *fc = (int32_t *)malloc((size_t)n * sizeof(int32_t));
    zd *fv = (zd *)malloc((size_t)n * sizeof(zd));
    double *diagbuf = (double *)malloc((size_t)3 * n * sizeof(double));
    for (int c = 0; c < n; ++c) { fr[c] = c; fc[c] = c; fv[c] = 1.0 / n; }
    tvec_t tv = {0, 0, 0};
    lindblad_terms(&md, n, fr, fc, fv, &tv);
    sum_terms(&tv);
    gap_t g = {0.0, INFINITY, 0.0, INFINITY};
    project_emit(n, &tv, 0, 0.0, NULL, res->K, diagbuf, &g);
    if (g.max_imag > res->gap.max_imag) res->gap.max_imag = g.max_imag;
    free(tv.t);
    free(fr);
    free(fc);
    free(fv);
    free(diagbuf);
  }
  free(md.Ht.rp); free(md.Ht.ci); free(md.Ht.v);
  for (int p = 0; p < P; ++p) {
    free(md.Lt[p].rp); free(md.Lt[p].ci); free(md.Lt[p].v);
    free(md.M[p].rp); free(md.M[p].ci); free(md.M[p].v);
    free(md.Mt[p].rp); free(md.Mt[p].ci); free(md.Mt[p].v);
  }
  free(md.L); free(md.Lt); free(md.M); free(md.Mt);
  return res;
}

int64_t o2_nnz(void *r) { return ((o2_result *)r)->nnz; }

void o2_gap(void *r, double *out4) {
  o2_result *res = (o2_result *)r;
  out4[0] = res->gap.max_dropped;
  out4[1] = res->gap.min_kept;
  out4[2] = res->gap.max_imag;
  out4[3] = res->gap.min_margin;
}

void o2_fetch(void *r, int64_t *row_ptr, int32_t *col, double *val, double *K) {
  o2_result *res = (o2_result *)r;
  memcpy(row_ptr, res->row_ptr, (size_t)(res->m + 1) * sizeof(int64_t));
  if (res->nnz) {
    memcpy(col, res->col, (size_t)res->nnz * sizeof(int32_t));
    memcpy(val, res->val, (size_t)res->nnz * sizeof(double));
  }
  if (K) memcpy(K, res->K, (size_t)res->m * sizeof(double));
}

/* per-entry sum|terms| (same order as o2_fetch's col / val) */
void o2_fetch_abs(void *r, double *absv) {
  o2_result *res = (o2_result *)r;
  if (res->nnz) memcpy(absv, res->absv, (size_t)res->nnz * sizeof(double));
}

void o2_free(void *r) {
  o2_result *res = (o2_result *)r;
  free(res->row_ptr);
  free(res->col);
  free(res->val);
  free(res->absv);
  free(res->K);
  free(res);
}

int o2_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
