/*
 * coracle.c -- plain-C restatement of the reference block ILU(k) path.
 * TEST / BASELINE INFRASTRUCTURE ONLY: loaded by tests/, smoke() and the
 * cpu_baseline / --impl reference legs of bench.py; never by the product.
 *
 * It follows the reference algorithms line by line in C so that parity can be
 * checked at full size (128^3) where the numpy restatement is too slow:
 *   co_symbolic       symbolic.py:27-72   (sorted pivot queue, levels > k dropped)
 *   co_build          factor.py:302-323   (materialize :83-121, block IKJ ILU(0)
 *                     :165-205 with block_invert :38-70, point kernel :124-148,
 *                     split_ldu :230-289, csr_expand sparse.py:337-374,
 *                     build_level_schedule trisolve.py:98-118)
 *   co_apply          trisolve.py:121-182 (point-wise level-scheduled sweeps,
 *                     stored-order row reduction; OpenMP over the rows of a level)
 *   co_bsr_spmv       sparse.py:278-301 on the block matrix
 * It is itself pinned against the reference's golden vectors
 * (tests/test_oracle_golden.py::test_c_oracle_matches_reference_golden).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define CO_OK 0
#define CO_STRUCT 1
#define CO_SINGULAR 2
#define CO_ZEROPIVOT 3
#define CO_NOMEM 7

typedef struct {
    int64_t n, m;               /* m = n * bs point rows */
    int bs;
    /* factors in the reference layout */
    int64_t *lrp, *lci, *urp, *uci;
    double *lv, *uv, *dinv;     /* L / U' column-major blocks; dinv row-major (n, bs, bs) */
    int64_t nl, nu, nnzp;
    /* point expansions (zero-dropped) */
    int64_t *plrp, *plci, *purp, *puci;
    double *plv, *puv;
    /* point level schedules: level of each point row, rows in level order */
    int64_t *llev, *ulev, *lord, *uord, *lptr, *uptr;
    int64_t nll, nul;
} co_factors;

/* ------------------------------------------------------------------------ */
/* symbolic phase                                                           */
/* ------------------------------------------------------------------------ */
static void heap_push(int64_t *h, int64_t *len, int64_t v) {
    int64_t i = (*len)++;
    h[i] = v;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p] <= h[i]) break;
        int64_t t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}
static int64_t heap_pop(int64_t *h, int64_t *len) {
    int64_t top = h[0];
    h[0] = h[--(*len)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, s = i;
        if (l < *len && h[l] < h[s]) s = l;
        if (r < *len && h[r] < h[s]) s = r;
        if (s == i) break;
        int64_t t = h[s]; h[s] = h[i]; h[i] = t;
        i = s;
    }
    return top;
}
static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* grows (rp, ci) to the ILU(k) pattern; *out_rp (n+1) and *out_ci malloc'ed */
int co_symbolic(int64_t n, const int64_t *rp, const int64_t *ci, int k, int64_t **out_rp, int64_t **out_ci,
                int64_t *err_row) {
    int64_t *lev = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *touched = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *heap = malloc(sizeof(int64_t) * (n ? n : 1));
    int64_t *orp = calloc(n + 1, sizeof(int64_t));
    int64_t cap = rp[n] * 2 + 16, ocnt = 0;
    int64_t *oci = malloc(sizeof(int64_t) * cap);
    int64_t ucap = rp[n] + 16, ucnt = 0;
    int64_t *ucol = malloc(sizeof(int64_t) * ucap), *ulevv = malloc(sizeof(int64_t) * ucap);
    int64_t *uptr = calloc(n + 1, sizeof(int64_t));
    if (!lev || !touched || !heap || !orp || !oci || !ucol || !ulevv || !uptr) return CO_NOMEM;
    for (int64_t i = 0; i < n; ++i) lev[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        int64_t nt = 0, hl = 0;
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            lev[ci[t]] = 0;
            touched[nt++] = ci[t];
            if (ci[t] < i) heap_push(heap, &hl, ci[t]);
        }
        if (lev[i] != 0) {
            *err_row = i;
            return CO_STRUCT;
        }
        while (hl) {
            int64_t p = heap_pop(heap, &hl), lp = lev[p];
            for (int64_t u = uptr[p]; u < uptr[p + 1]; ++u) {
                int64_t lv = lp + ulevv[u] + 1, j = ucol[u];
                if (lv > k) continue;
                if (lev[j] < 0) {
                    lev[j] = lv;
                    touched[nt++] = j;
                    if (j < i) heap_push(heap, &hl, j);
                } else if (lv < lev[j]) {
                    lev[j] = lv;
                }
            }
        }
        qsort(touched, nt, sizeof(int64_t), cmp_i64);
        if (ocnt + nt > cap) {
            cap = 2 * (ocnt + nt);
            oci = realloc(oci, sizeof(int64_t) * cap);
        }
        for (int64_t q = 0; q < nt; ++q) {
            int64_t j = touched[q];
            oci[ocnt++] = j;
            if (j > i) {
                if (ucnt == ucap) {
                    ucap *= 2;
                    ucol = realloc(ucol, sizeof(int64_t) * ucap);
                    ulevv = realloc(ulevv, sizeof(int64_t) * ucap);
                }
                ucol[ucnt] = j;
                ulevv[ucnt++] = lev[j];
            }
            lev[j] = -1;
        }
        orp[i + 1] = ocnt;
        uptr[i + 1] = ucnt;
    }
    free(lev); free(touched); free(heap); free(ucol); free(ulevv); free(uptr);
    *out_rp = orp;
    *out_ci = oci;
    return CO_OK;
}

/* ------------------------------------------------------------------------ */
/* block inverse, block_invert (factor.py:38-70); a, inv row-major          */
/* ------------------------------------------------------------------------ */
static int block_invert(int bs, const double *a, double *inv) {
    double lu[64], amax = 0.0;
    int perm[8];
    for (int q = 0; q < bs * bs; ++q) {
        lu[q] = a[q];
        if (fabs(a[q]) > amax) amax = fabs(a[q]);
    }
    if (amax == 0.0) return CO_SINGULAR;
    if (bs == 1) {
        inv[0] = 1.0 / a[0];
        return CO_OK;
    }
    for (int r = 0; r < bs; ++r) perm[r] = r;
    for (int c = 0; c < bs; ++c) {
        int p = c;
        for (int r = c + 1; r < bs; ++r)
            if (fabs(lu[r * bs + c]) > fabs(lu[p * bs + c])) p = r;
        if (fabs(lu[p * bs + c]) < 1e-13 * amax) return CO_SINGULAR;
        if (p != c) {
            for (int q = 0; q < bs; ++q) {
                double t = lu[c * bs + q]; lu[c * bs + q] = lu[p * bs + q]; lu[p * bs + q] = t;
            }
            int t = perm[c]; perm[c] = perm[p]; perm[p] = t;
        }
        for (int r = c + 1; r < bs; ++r) {
            lu[r * bs + c] /= lu[c * bs + c];
            for (int q = c + 1; q < bs; ++q) lu[r * bs + q] -= lu[r * bs + c] * lu[c * bs + q];
        }
    }
    for (int r = 0; r < bs; ++r)
        for (int q = 0; q < bs; ++q) inv[r * bs + q] = (perm[r] == q) ? 1.0 : 0.0;
    for (int r = 1; r < bs; ++r)
        for (int q = 0; q < bs; ++q) {
            double s = 0.0;
            for (int t = 0; t < r; ++t) s += lu[r * bs + t] * inv[t * bs + q];
            inv[r * bs + q] -= s;
        }
    for (int r = bs - 1; r >= 0; --r)
        for (int q = 0; q < bs; ++q) {
            double s = 0.0;
            for (int t = r + 1; t < bs; ++t) s += lu[r * bs + t] * inv[t * bs + q];
            inv[r * bs + q] = (inv[r * bs + q] - s) / lu[r * bs + r];
        }
    return CO_OK;
}

/* column-major block (storage) <-> row-major matrix */
static void cm_to_rm(int bs, const double *cm, double *rm) {
    for (int r = 0; r < bs; ++r)
        for (int c = 0; c < bs; ++c) rm[r * bs + c] = cm[c * bs + r];
}
static void rm_to_cm(int bs, const double *rm, double *cm) {
    for (int r = 0; r < bs; ++r)
        for (int c = 0; c < bs; ++c) cm[c * bs + r] = rm[r * bs + c];
}
static void matmul(int bs, const double *a, const double *b, double *c) { /* row-major c = a b */
    for (int r = 0; r < bs; ++r)
        for (int q = 0; q < bs; ++q) {
            double s = 0.0;
            for (int t = 0; t < bs; ++t) s += a[r * bs + t] * b[t * bs + q];
            c[r * bs + q] = s;
        }
}

/* ------------------------------------------------------------------------ */
/* point expansion (sparse.py:337-374) and levels (trisolve.py:98-118)      */
/* ------------------------------------------------------------------------ */
static void expand(int64_t n, int bs, const int64_t *rp, const int64_t *ci, const double *v, int64_t **prp,
                   int64_t **pci, double **pv) {
    int64_t m = n * bs, bs2 = (int64_t)bs * bs, cnt = 0;
    int64_t *r = calloc(m + 1, sizeof(int64_t));
    int64_t cap = rp[n] * bs2 + 1;
    int64_t *c = malloc(sizeof(int64_t) * cap);
    double *w = malloc(sizeof(double) * cap);
    for (int64_t i = 0; i < n; ++i)
        for (int rr = 0; rr < bs; ++rr) {
            for (int64_t s = rp[i]; s < rp[i + 1]; ++s)
                for (int cc = 0; cc < bs; ++cc) {
                    double val = v[s * bs2 + cc * bs + rr];
                    if (val != 0.0) {
                        c[cnt] = ci[s] * bs + cc;
                        w[cnt++] = val;
                    }
                }
            r[i * bs + rr + 1] = cnt;
        }
    *prp = r;
    *pci = c;
    *pv = w;
}

static int64_t levels(int64_t m, const int64_t *rp, const int64_t *ci, int upper, int64_t *lev, int64_t **ord,
                      int64_t **ptr) {
    int64_t mx = 0;
    for (int64_t s = 0; s < m; ++s) {
        int64_t i = upper ? m - 1 - s : s, best = 0;
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t)
            if (lev[ci[t]] > best) best = lev[ci[t]];
        lev[i] = best + 1;
        if (lev[i] > mx) mx = lev[i];
    }
    int64_t *p = calloc(mx + 2, sizeof(int64_t));
    for (int64_t i = 0; i < m; ++i) p[lev[i]]++;
    for (int64_t l = 1; l <= mx + 1; ++l) p[l] += p[l - 1];
    /* p[l] = rows with level <= l ; rows of level l at [p[l-1], p[l]) ascending (stable) */
    int64_t *cur = malloc(sizeof(int64_t) * (mx + 2));
    for (int64_t l = 1; l <= mx; ++l) cur[l] = p[l - 1];
    int64_t *o = malloc(sizeof(int64_t) * (m ? m : 1));
    for (int64_t i = 0; i < m; ++i) o[cur[lev[i]]++] = i;
    free(cur);
    *ord = o;
    *ptr = p;
    return mx;
}

void co_free(co_factors *f) {
    if (!f) return;
    free(f->lrp); free(f->lci); free(f->urp); free(f->uci); free(f->lv); free(f->uv); free(f->dinv);
    free(f->plrp); free(f->plci); free(f->purp); free(f->puci); free(f->plv); free(f->puv);
    free(f->llev); free(f->ulev); free(f->lord); free(f->uord); free(f->lptr); free(f->uptr);
    free(f);
}

/* the whole build_preconditioner pipeline */
int co_build(int64_t n, int bs, const int64_t *rp, const int64_t *ci, const double *vals, int k, co_factors **out,
             int64_t *err_row) {
    int64_t *prp = NULL, *pci = NULL;
    int rc = co_symbolic(n, rp, ci, k, &prp, &pci, err_row);
    if (rc) return rc;
    const int64_t bs2 = (int64_t)bs * bs, nnzp = prp[n];
    double *pv = calloc(nnzp * bs2 + 1, sizeof(double));           /* materialize */
    for (int64_t i = 0; i < n; ++i) {
        int64_t q = prp[i];
        for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
            while (pci[q] != ci[t]) ++q;
            memcpy(pv + q * bs2, vals + t * bs2, sizeof(double) * bs2);
        }
    }
    int64_t *diag = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        int64_t d = prp[i];
        while (d < prp[i + 1] && pci[d] < i) ++d;
        diag[i] = d;
    }
    double *dinv = calloc(n * bs2 + 1, sizeof(double));             /* row-major */
    int64_t *pos = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t i = 0; i < n; ++i) pos[i] = -1;
    double A[64], B[64], C[64], D[64];
    for (int64_t i = 0; i < n && !rc; ++i) {                        /* block IKJ ILU(0) */
        for (int64_t t = prp[i]; t < prp[i + 1]; ++t) pos[pci[t]] = t;
        for (int64_t t = prp[i]; t < diag[i]; ++t) {
            int64_t p = pci[t];
            if (bs == 1) {
                pv[t] = pv[t] / pv[diag[p]];
            } else {
                cm_to_rm(bs, pv + t * bs2, A);
                matmul(bs, A, dinv + p * bs2, C);
                rm_to_cm(bs, C, pv + t * bs2);
            }
            for (int64_t u = diag[p] + 1; u < prp[p + 1]; ++u) {
                int64_t q = pos[pci[u]];
                if (q < 0) continue;
                if (bs == 1) {
                    pv[q] -= pv[t] * pv[u];
                } else {
                    cm_to_rm(bs, pv + t * bs2, A);
                    cm_to_rm(bs, pv + u * bs2, B);
                    matmul(bs, A, B, C);
                    cm_to_rm(bs, pv + q * bs2, D);
                    for (int x = 0; x < bs2; ++x) D[x] -= C[x];
                    rm_to_cm(bs, D, pv + q * bs2);
                }
            }
        }
        if (bs == 1) {
            if (fabs(pv[diag[i]]) < 1e-300) {
                *err_row = i;
                rc = CO_ZEROPIVOT;
            } else {
                dinv[i] = 1.0 / pv[diag[i]];
            }
        } else {
            cm_to_rm(bs, pv + diag[i] * bs2, A);
            if (block_invert(bs, A, dinv + i * bs2) != CO_OK) {
                *err_row = i;
                rc = CO_SINGULAR;
            }
        }
        for (int64_t t = prp[i]; t < prp[i + 1]; ++t) pos[pci[t]] = -1;
    }
    free(pos);
    if (rc) {
        free(prp); free(pci); free(pv); free(diag); free(dinv);
        return rc;
    }
    co_factors *f = calloc(1, sizeof(co_factors));
    f->n = n;
    f->bs = bs;
    f->m = n * bs;
    f->nnzp = nnzp;
    f->dinv = dinv;
    f->lrp = calloc(n + 1, sizeof(int64_t));
    f->urp = calloc(n + 1, sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) {                                /* split (factor.py:230-289) */
        f->lrp[i + 1] = f->lrp[i] + (diag[i] - prp[i]);
        f->urp[i + 1] = f->urp[i] + (prp[i + 1] - diag[i] - 1);
    }
    f->nl = f->lrp[n];
    f->nu = f->urp[n];
    f->lci = malloc(sizeof(int64_t) * (f->nl + 1));
    f->uci = malloc(sizeof(int64_t) * (f->nu + 1));
    f->lv = malloc(sizeof(double) * (f->nl * bs2 + 1));
    f->uv = malloc(sizeof(double) * (f->nu * bs2 + 1));
    for (int64_t i = 0; i < n; ++i) {
        int64_t lq = f->lrp[i], uq = f->urp[i];
        for (int64_t t = prp[i]; t < diag[i]; ++t, ++lq) {
            f->lci[lq] = pci[t];
            memcpy(f->lv + lq * bs2, pv + t * bs2, sizeof(double) * bs2);
        }
        for (int64_t t = diag[i] + 1; t < prp[i + 1]; ++t, ++uq) {
            f->uci[uq] = pci[t];
            cm_to_rm(bs, pv + t * bs2, B);
            matmul(bs, dinv + i * bs2, B, C);
            rm_to_cm(bs, C, f->uv + uq * bs2);
        }
    }
    free(prp); free(pci); free(pv); free(diag);
    expand(n, bs, f->lrp, f->lci, f->lv, &f->plrp, &f->plci, &f->plv);
    expand(n, bs, f->urp, f->uci, f->uv, &f->purp, &f->puci, &f->puv);
    f->llev = malloc(sizeof(int64_t) * (f->m + 1));
    f->ulev = malloc(sizeof(int64_t) * (f->m + 1));
    f->nll = levels(f->m, f->plrp, f->plci, 0, f->llev, &f->lord, &f->lptr);
    f->nul = levels(f->m, f->purp, f->puci, 1, f->ulev, &f->uord, &f->uptr);
    *out = f;
    return CO_OK;
}

/* sizes: [n, bs, nl, nu, m, plnnz, punnz, nll, nul] */
void co_sizes(const co_factors *f, int64_t *s) {
    s[0] = f->n; s[1] = f->bs; s[2] = f->nl; s[3] = f->nu; s[4] = f->m;
    s[5] = f->plrp[f->m]; s[6] = f->purp[f->m]; s[7] = f->nll; s[8] = f->nul;
}

void co_get(const co_factors *f, int64_t *lrp, int64_t *lci, double *lv, double *dinv, int64_t *urp, int64_t *uci,
            double *uv, int64_t *llev, int64_t *ulev) {
    const int64_t bs2 = (int64_t)f->bs * f->bs;
    if (lrp) memcpy(lrp, f->lrp, sizeof(int64_t) * (f->n + 1));
    if (lci) memcpy(lci, f->lci, sizeof(int64_t) * f->nl);
    if (lv) memcpy(lv, f->lv, sizeof(double) * f->nl * bs2);
    if (dinv) memcpy(dinv, f->dinv, sizeof(double) * f->n * bs2);
    if (urp) memcpy(urp, f->urp, sizeof(int64_t) * (f->n + 1));
    if (uci) memcpy(uci, f->uci, sizeof(int64_t) * f->nu);
    if (uv) memcpy(uv, f->uv, sizeof(double) * f->nu * bs2);
    if (llev) memcpy(llev, f->llev, sizeof(int64_t) * f->m);
    if (ulev) memcpy(ulev, f->ulev, sizeof(int64_t) * f->m);
}

/* ------------------------------------------------------------------------ */
/* apply: level-scheduled unit solves + D^-1 (trisolve.py:121-182)           */
/* ------------------------------------------------------------------------ */
static void unit_solve(int64_t m, const int64_t *rp, const int64_t *ci, const double *v, const int64_t *ord,
                       const int64_t *ptr, int64_t nlev, const double *b, double *x, int threads) {
    memcpy(x, b, sizeof(double) * m);
    for (int64_t l = 1; l <= nlev; ++l) {
        const int64_t lo = ptr[l - 1], hi = ptr[l];
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1 && hi - lo > 256)
        for (int64_t q = lo; q < hi; ++q) {
            const int64_t i = ord[q];
            double s = 0.0;
            for (int64_t t = rp[i]; t < rp[i + 1]; ++t) s += v[t] * x[ci[t]];
            x[i] = b[i] - s;
        }
    }
}

void co_apply(const co_factors *f, const double *b, double *x, double *work, int threads) {
    const int bs = f->bs;
    const int64_t bs2 = (int64_t)bs * bs;
    unit_solve(f->m, f->plrp, f->plci, f->plv, f->lord, f->lptr, f->nll, b, work, threads);
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
    for (int64_t i = 0; i < f->n; ++i)
        for (int r = 0; r < bs; ++r) {
            double s = 0.0;
            for (int c = 0; c < bs; ++c) s += f->dinv[i * bs2 + r * bs + c] * work[i * bs + c];
            x[i * bs + r] = s;
        }
    memcpy(work, x, sizeof(double) * f->m);
    unit_solve(f->m, f->purp, f->puci, f->puv, f->uord, f->uptr, f->nul, work, x, threads);
}

/* y = A x for a BSR matrix (column-major blocks) */
void co_bsr_spmv(int64_t n, int bs, const int64_t *rp, const int64_t *ci, const double *v, const double *x,
                 double *y, int threads) {
    const int64_t bs2 = (int64_t)bs * bs;
#pragma omp parallel for num_threads(threads) schedule(static) if (threads > 1)
    for (int64_t i = 0; i < n; ++i)
        for (int r = 0; r < bs; ++r) {
            double s = 0.0;
            for (int64_t t = rp[i]; t < rp[i + 1]; ++t)
                for (int c = 0; c < bs; ++c) s += v[t * bs2 + c * bs + r] * x[ci[t] * bs + c];
            y[i * bs + r] = s;
        }
}

int co_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* point expansions (zero-dropped, reference order) */
void co_get_points(const co_factors *f, int64_t *plrp, int64_t *plci, double *plv, int64_t *purp, int64_t *puci,
                   double *puv) {
    memcpy(plrp, f->plrp, sizeof(int64_t) * (f->m + 1));
    memcpy(plci, f->plci, sizeof(int64_t) * f->plrp[f->m]);
    memcpy(plv, f->plv, sizeof(double) * f->plrp[f->m]);
    memcpy(purp, f->purp, sizeof(int64_t) * (f->m + 1));
    memcpy(puci, f->puci, sizeof(int64_t) * f->purp[f->m]);
    memcpy(puv, f->puv, sizeof(double) * f->purp[f->m]);
}
