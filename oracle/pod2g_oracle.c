/*
 * pod2g_oracle.c -- CPU restatement of the reference POD-2G solve path.
 *
 * TEST INFRASTRUCTURE ONLY (see pod2g_oracle.h).  Built with
 * -ffp-contract=off so that a*b+c is never fused: the reference is compiled for
 * plain x86-64 (no FMA), and the restatement must round identically.
 *
 * Citations are relative to /root/reference/proj/include/pod2g/.
 */
#include "pod2g_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* core/types.hpp:52-57 -- sequential ascending sum */
double or_dot(int64_t n, const double* x, const double* y) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

/* core/csr.hpp:83-93 */
void or_spmv(const or_csr* A, const double* x, double* y) {
    for (int64_t i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * x[A->ci[k]];
        y[i] = s;
    }
}

/* core/csr.hpp:96-105  r = f - A u (row sum first, then subtract) */
void or_residual(const or_csr* A, const double* f, const double* u, double* r) {
    for (int64_t i = 0; i < A->n; ++i) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k) s += A->v[k] * u[A->ci[k]];
        r[i] = f[i] - s;
    }
}

/* smoothers.hpp:26-47  forward Gauss-Seidel, ascending rows.  The sum starts
 * from f_i and subtracts each off-diagonal product in column order. */
int or_gs_forward(const or_csr* K, const double* f, double* u, int64_t sweeps) {
    for (int64_t sw = 0; sw < sweeps; ++sw) {
        for (int64_t i = 0; i < K->n; ++i) {
            double sum = f[i];
            double diag = 0.0;
            for (int64_t k = K->rp[i]; k < K->rp[i + 1]; ++k) {
                const int64_t j = K->ci[k];
                if (j == i)
                    diag = K->v[k];
                else
                    sum -= K->v[k] * u[j];
            }
            if (diag == 0.0) return OR_EZERODIAG;
            u[i] = sum / diag;
        }
    }
    return OR_OK;
}

/* smoothers.hpp:51-72  backward Gauss-Seidel, descending rows */
int or_gs_backward(const or_csr* K, const double* f, double* u, int64_t sweeps) {
    for (int64_t sw = 0; sw < sweeps; ++sw) {
        for (int64_t i = K->n; i-- > 0;) {
            double sum = f[i];
            double diag = 0.0;
            for (int64_t k = K->rp[i]; k < K->rp[i + 1]; ++k) {
                const int64_t j = K->ci[k];
                if (j == i)
                    diag = K->v[k];
                else
                    sum -= K->v[k] * u[j];
            }
            if (diag == 0.0) return OR_EZERODIAG;
            u[i] = sum / diag;
        }
    }
    return OR_OK;
}

/* core/csr.hpp:125-132 */
static void extract_diagonal(const or_csr* A, double* d) {
    for (int64_t i = 0; i < A->n; ++i) {
        d[i] = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; ++k)
            if (A->ci[k] == i) d[i] = A->v[k];
    }
}

/* smoothers.hpp:75-87  u += omega * r_i / d_i per sweep, r = f - K u */
int or_jacobi_sweep(const or_csr* K, const double* f, double* u, double omega, int64_t sweeps) {
    if (!(omega > 0.0 && omega <= 1.0)) return OR_EINVAL;
    const int64_t n = K->n;
    double* diag = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* r = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    extract_diagonal(K, diag);
    for (int64_t i = 0; i < n; ++i)
        if (diag[i] == 0.0) {
            free(diag);
            free(r);
            return OR_EZERODIAG;
        }
    for (int64_t sw = 0; sw < sweeps; ++sw) {
        or_residual(K, f, u, r);
        for (int64_t i = 0; i < n; ++i) u[i] += omega * r[i] / diag[i];
    }
    free(diag);
    free(r);
    return OR_OK;
}

/* pod.hpp:27-35  z_j += phi(i,j) * u_i, rows outer */
void or_project(int64_t n, int64_t k, const double* phi, const double* u, double* z) {
    for (int64_t j = 0; j < k; ++j) z[j] = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const double ui = u[i];
        for (int64_t j = 0; j < k; ++j) z[j] += phi[i * k + j] * ui;
    }
}

/* pod.hpp:37-46 */
void or_lift(int64_t n, int64_t k, const double* phi, const double* z, double* u) {
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < k; ++j) s += phi[i * k + j] * z[j];
        u[i] = s;
    }
}

/* core/dense_solve.hpp:15-38  partial-pivot LU, row swaps, pivot floor
 * 1e-14 * max|a| (core/types.hpp:114-118) */
int or_lu_factor(int64_t n, double* a, int64_t* perm) {
    double maxabs = 0.0;
    for (int64_t i = 0; i < n * n; ++i) maxabs = fmax(maxabs, fabs(a[i]));
    const double pivot_floor = 1e-14 * maxabs;
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t k = 0; k < n; ++k) {
        int64_t p = k;
        for (int64_t i = k + 1; i < n; ++i)
            if (fabs(a[i * n + k]) > fabs(a[p * n + k])) p = i;
        if (fabs(a[p * n + k]) <= pivot_floor) return OR_ESINGULAR;
        if (p != k) {
            for (int64_t j = 0; j < n; ++j) {
                const double t = a[k * n + j];
                a[k * n + j] = a[p * n + j];
                a[p * n + j] = t;
            }
            const int64_t t = perm[k];
            perm[k] = perm[p];
            perm[p] = t;
        }
        for (int64_t i = k + 1; i < n; ++i) {
            a[i * n + k] /= a[k * n + k];
            const double lik = a[i * n + k];
            if (lik == 0.0) continue;
            for (int64_t j = k + 1; j < n; ++j) a[i * n + j] -= lik * a[k * n + j];
        }
    }
    return OR_OK;
}

/* core/dense_solve.hpp:40-56 */
void or_lu_solve(int64_t n, const double* lu, const int64_t* perm, const double* b, double* x) {
    for (int64_t i = 0; i < n; ++i) x[i] = b[perm[i]];
    for (int64_t i = 1; i < n; ++i) {
        double s = x[i];
        for (int64_t j = 0; j < i; ++j) s -= lu[i * n + j] * x[j];
        x[i] = s;
    }
    for (int64_t ii = n; ii-- > 0;) {
        double s = x[ii];
        for (int64_t j = ii + 1; j < n; ++j) s -= lu[ii * n + j] * x[j];
        x[ii] = s / lu[ii * n + ii];
    }
}

/* pod.hpp:152-165  column j: kphi = K phi_j; Kr(i,j) = sum_m phi(m,i) kphi_m */
void or_reduced_operator(const or_csr* K, int64_t k, const double* phi, double* Ac) {
    const int64_t n = K->n;
    double* col = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* kphi = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    for (int64_t j = 0; j < k; ++j) {
        for (int64_t m = 0; m < n; ++m) col[m] = phi[m * k + j];
        or_spmv(K, col, kphi);
        for (int64_t i = 0; i < k; ++i) {
            double s = 0.0;
            for (int64_t m = 0; m < n; ++m) s += phi[m * k + i] * kphi[m];
            Ac[i * k + j] = s;
        }
    }
    free(col);
    free(kphi);
}

/* pod.hpp:167-179 */
int or_reduced_solve(const or_csr* K, const double* f, int64_t k, const double* phi, double* x0,
                     double* ur) {
    double* Ac = (double*)malloc(sizeof(double) * (size_t)(k * k));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)k);
    double* fr = (double*)malloc(sizeof(double) * (size_t)k);
    double* u = (double*)malloc(sizeof(double) * (size_t)k);
    or_reduced_operator(K, k, phi, Ac);
    or_project(K->n, k, phi, f, fr);
    int st = or_lu_factor(k, Ac, perm);
    if (st == OR_OK) {
        or_lu_solve(k, Ac, perm, fr, u);
        or_lift(K->n, k, phi, u, x0);
        if (ur) memcpy(ur, u, sizeof(double) * (size_t)k);
    }
    free(Ac);
    free(perm);
    free(fr);
    free(u);
    return st;
}

/* pod.hpp:186-189  Pod2gOperator ctor: coarse LU of reduced_operator(K, basis) */
int or_pod2g_setup(or_pod2g* P, const or_csr* K, int64_t k, const double* phi, int64_t r1,
                   int64_t r2, int smoother, double omega, double* lu_storage,
                   int64_t* perm_storage) {
    P->K = K;
    P->k = k;
    P->phi = phi;
    P->r1 = r1;
    P->r2 = r2;
    P->smoother = smoother;
    P->omega = omega;
    P->lu = lu_storage;
    P->perm = perm_storage;
    if (k == 0) return OR_OK;
    or_reduced_operator(K, k, phi, lu_storage);
    return or_lu_factor(k, lu_storage, perm_storage);
}

/* smoothers.hpp:89-105 */
static int apply_smoother(const or_pod2g* P, const double* f, double* u, int64_t sweeps,
                          int adjoint) {
    if (P->smoother == OR_SMOOTHER_GS)
        return adjoint ? or_gs_backward(P->K, f, u, sweeps) : or_gs_forward(P->K, f, u, sweeps);
    return or_jacobi_sweep(P->K, f, u, P->omega, sweeps);
}

/* pod.hpp:264-267  s := 0; cycle(r, s, adjoint_post=true)
 * pod.hpp:196-207  smoother^r1; t = r - K s; e = LU^{-1} Phi^T t; s += Phi e;
 *                  adjoint smoother^r2 */
int or_pod2g_apply(const or_pod2g* P, const double* f, double* u) {
    const int64_t n = P->K->n, k = P->k;
    int st;
    for (int64_t i = 0; i < n; ++i) u[i] = 0.0;
    if ((st = apply_smoother(P, f, u, P->r1, 0)) != OR_OK) return st;
    if (k > 0) {
        double* r = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
        double* c = (double*)malloc(sizeof(double) * (size_t)k);
        double* e = (double*)malloc(sizeof(double) * (size_t)k);
        double* corr = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
        or_residual(P->K, f, u, r);
        or_project(n, k, P->phi, r, c);
        or_lu_solve(k, P->lu, P->perm, c, e);
        or_lift(n, k, P->phi, e, corr);
        for (int64_t i = 0; i < n; ++i) u[i] += 1.0 * corr[i]; /* axpy(1.0, corr, u) */
        free(r);
        free(c);
        free(e);
        free(corr);
    }
    return apply_smoother(P, f, u, P->r2, 1);
}

static double relative_residual(double rnorm, double fnorm) { /* krylov.hpp:235-237 */
    return fnorm > 0.0 ? rnorm / fnorm : rnorm;
}

/* krylov.hpp:243-297 */
int or_pcg_pod2g(const or_csr* K, const double* f, int64_t k, const double* phi,
                 const double* u0, double delta, int64_t max_iter, int smoother, double omega,
                 int64_t r1, int64_t r2, double* u, int64_t* iters, int* converged,
                 double* hist, int64_t hist_cap, int64_t* hist_len) {
    const int64_t n = K->n;
    int st = OR_OK;
    int64_t hl = 0;
#define PUSH_HIST(v)                         \
    do {                                     \
        if (hist && hl < hist_cap) hist[hl] = (v); \
        ++hl;                                \
    } while (0)

    or_pod2g P;
    double* lu = (double*)malloc(sizeof(double) * (size_t)(k * k + 1));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k + 1));
    /* identity preconditioner when k == 0 (krylov.hpp:21-25): s = r */
    if (k > 0) {
        st = or_pod2g_setup(&P, K, k, phi, r1, r2, smoother, omega, lu, perm);
        if (st != OR_OK) {
            free(lu);
            free(perm);
            *iters = 0;
            *converged = 0;
            if (hist_len) *hist_len = 0;
            return st;
        }
    }

    const double fnorm = sqrt(or_dot(n, f, f));
    if (u0)
        memcpy(u, u0, sizeof(double) * (size_t)n);
    else
        for (int64_t i = 0; i < n; ++i) u[i] = 0.0;
    double* r = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* s = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* p = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* Kp = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    or_residual(K, f, u, r);
    double rel = relative_residual(sqrt(or_dot(n, r, r)), fnorm);
    PUSH_HIST(rel);

    int64_t it = 0;
    if (rel > delta && it < max_iter) {
        if (k > 0) {
            st = or_pod2g_apply(&P, r, s);
        } else {
            memcpy(s, r, sizeof(double) * (size_t)n);
        }
        if (st != OR_OK) goto done;
        memcpy(p, s, sizeof(double) * (size_t)n);
        double rs_old = or_dot(n, r, s);
        if (rs_old <= 0.0) {
            st = OR_EBREAKDOWN;
            goto done;
        }
        while (rel > delta && it < max_iter) {
            or_spmv(K, p, Kp);
            const double pKp = or_dot(n, p, Kp);
            if (pKp <= 0.0) {
                st = OR_EBREAKDOWN;
                goto done;
            }
            const double alpha = rs_old / pKp;
            for (int64_t i = 0; i < n; ++i) u[i] += alpha * p[i];   /* axpy */
            for (int64_t i = 0; i < n; ++i) r[i] += -alpha * Kp[i]; /* axpy(-alpha) */
            if (k > 0) {
                st = or_pod2g_apply(&P, r, s);
                if (st != OR_OK) goto done;
            } else {
                memcpy(s, r, sizeof(double) * (size_t)n);
            }
            const double rs_new = or_dot(n, r, s);
            const double beta = rs_new / rs_old;
            for (int64_t i = 0; i < n; ++i) p[i] = s[i] + beta * p[i];
            rs_old = rs_new;
            ++it;
            rel = relative_residual(sqrt(or_dot(n, r, r)), fnorm);
            PUSH_HIST(rel);
            if (rs_new <= 0.0 && rel > delta) {
                st = OR_EBREAKDOWN;
                goto done;
            }
        }
    }
    for (int64_t i = 0; i < n; ++i)
        if (!isfinite(u[i])) {
            st = OR_ENONFINITE;
            break;
        }
done:
    *iters = it;
    *converged = rel <= delta;
    if (hist_len) *hist_len = hl;
    free(r);
    free(s);
    free(p);
    free(Kp);
    free(lu);
    free(perm);
#undef PUSH_HIST
    return st;
}

/* ---- batched CPU baseline: whole instances per worker thread ------------ */
typedef struct {
    int64_t n, nnz, B, k, max_iter;
    const int64_t *rp, *ci;
    const double *values, *f, *phi, *u0;
    double delta, omega;
    int smoother;
    double* u;
    int64_t* iters;
    int *converged, *status;
    int64_t next; /* guarded by mu */
    pthread_mutex_t mu;
} batch_ctx;

static void* batch_worker(void* arg) {
    batch_ctx* c = (batch_ctx*)arg;
    for (;;) {
        pthread_mutex_lock(&c->mu);
        const int64_t b = c->next++;
        pthread_mutex_unlock(&c->mu);
        if (b >= c->B) break;
        or_csr K = {c->n, c->rp, c->ci, c->values + b * c->nnz};
        c->status[b] = or_pcg_pod2g(&K, c->f + b * c->n, c->k, c->phi,
                                    c->u0 ? c->u0 + b * c->n : NULL, c->delta, c->max_iter,
                                    c->smoother, c->omega, 1, 1, c->u + b * c->n, &c->iters[b],
                                    &c->converged[b], NULL, 0, NULL);
    }
    return NULL;
}

int or_pcg_pod2g_batch(int64_t n, const int64_t* rp, const int64_t* ci, int64_t nnz,
                       const double* values, int64_t B, const double* f, int64_t k,
                       const double* phi, const double* u0, double delta, int64_t max_iter,
                       int smoother, double omega, double* u, int64_t* iters, int* converged,
                       int* status, int nthreads) {
    batch_ctx c;
    c.n = n;
    c.nnz = nnz;
    c.B = B;
    c.k = k;
    c.max_iter = max_iter;
    c.rp = rp;
    c.ci = ci;
    c.values = values;
    c.f = f;
    c.phi = phi;
    c.u0 = u0;
    c.delta = delta;
    c.omega = omega;
    c.smoother = smoother;
    c.u = u;
    c.iters = iters;
    c.converged = converged;
    c.status = status;
    c.next = 0;
    pthread_mutex_init(&c.mu, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, batch_worker, &c);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&c.mu);
    int worst = OR_OK;
    for (int64_t b = 0; b < B; ++b)
        if (status[b] != OR_OK) worst = status[b];
    return worst;
}

/* surrogate.hpp:354-357 (see the header) */
int or_surrogate_predict(int nlayers, const int64_t* widths, int act, const double* W,
                         const double* bias, const double* in_mean, const double* in_std,
                         const double* lat_mean, const double* lat_std, int64_t n,
                         const double* phi, int64_t B, const double* theta, double* x) {
    if (nlayers < 1) return OR_EINVAL;
    int64_t wmax = 0;
    for (int l = 0; l <= nlayers; ++l) wmax = widths[l] > wmax ? widths[l] : wmax;
    const int64_t p = widths[0], k = widths[nlayers];
    double* a = (double*)malloc(sizeof(double) * (size_t)wmax);
    double* z = (double*)malloc(sizeof(double) * (size_t)wmax);
    if (!a || !z) {
        free(a);
        free(z);
        return OR_EINVAL;
    }
    for (int64_t b = 0; b < B; ++b) {
        for (int64_t j = 0; j < p; ++j) a[j] = (theta[b * p + j] - in_mean[j]) / in_std[j];
        const double* Wl = W;
        const double* bl = bias;
        for (int l = 0; l < nlayers; ++l) {
            const int64_t fi = widths[l], fo = widths[l + 1];
            for (int64_t i = 0; i < fo; ++i) {
                double s = bl[i];
                for (int64_t j = 0; j < fi; ++j) s += Wl[i * fi + j] * a[j];
                z[i] = s;
            }
            if (l + 1 < nlayers)
                for (int64_t i = 0; i < fo; ++i) z[i] = act == 0 ? tanh(z[i]) : fmax(z[i], 0.0);
            for (int64_t i = 0; i < fo; ++i) a[i] = z[i];
            Wl += fo * fi;
            bl += fo;
        }
        for (int64_t i = 0; i < k; ++i) a[i] = a[i] * lat_std[i] + lat_mean[i];
        or_lift(n, k, phi, a, x + b * n);
    }
    free(a);
    free(z);
    return OR_OK;
}

/* pod.hpp:224-256 (see the header) */
int or_pod2g_solve(const or_csr* K, const double* f, int64_t k, const double* phi,
                   const double* u0, double delta, int64_t max_cycles, int64_t r1, int64_t r2,
                   double* u, int64_t* cycles, int* converged, double* hist, int64_t hist_cap,
                   int64_t* hist_len) {
    const int64_t n = K->n;
    double* lu = (double*)malloc(sizeof(double) * (size_t)(k * k > 0 ? k * k : 1));
    int64_t* perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k > 0 ? k : 1));
    double* r = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    double* c = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
    double* e = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1));
    double* corr = (double*)malloc(sizeof(double) * (size_t)(n ? n : 1));
    or_pod2g P;
    int st = or_pod2g_setup(&P, K, k, phi, r1, r2, OR_SMOOTHER_GS, 0.0, lu, perm);
    int64_t hl = 0, it = 0;
    for (int64_t i = 0; i < n; ++i) u[i] = u0 ? u0[i] : 0.0;
    if (st == OR_OK) {
        const double fnorm = sqrt(or_dot(n, f, f));
        or_residual(K, f, u, r);
        double rel = relative_residual(sqrt(or_dot(n, r, r)), fnorm);
        if (hist && hl < hist_cap) hist[hl] = rel;
        ++hl;
        while (rel > delta && it < max_cycles) {
            if ((st = or_gs_forward(K, f, u, r1)) != OR_OK) break; /* cycle(f, u) */
            if (k > 0) {
                or_residual(K, f, u, r);
                or_project(n, k, phi, r, c);
                or_lu_solve(k, lu, perm, c, e);
                or_lift(n, k, phi, e, corr);
                for (int64_t i = 0; i < n; ++i) u[i] += 1.0 * corr[i];
            }
            if ((st = or_gs_forward(K, f, u, r2)) != OR_OK) break;
            or_residual(K, f, u, r);
            rel = relative_residual(sqrt(or_dot(n, r, r)), fnorm);
            if (hist && hl < hist_cap) hist[hl] = rel;
            ++hl;
            ++it;
        }
        *converged = rel <= delta;
        if (st == OR_OK)
            for (int64_t i = 0; i < n; ++i)
                if (!isfinite(u[i])) {
                    st = OR_ENONFINITE;
                    break;
                }
    } else {
        *converged = 0;
    }
    *cycles = it;
    if (hist_len) *hist_len = hl;
    free(lu);
    free(perm);
    free(r);
    free(c);
    free(e);
    free(corr);
    return st;
}
