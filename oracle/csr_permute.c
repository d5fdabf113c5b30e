/*
 * csr_permute.c -- P K P^T for the parity tests at full c5 size (12.4 M rows,
 * 1e9 nonzeros), where tests/helpers.permute_csr's per-row Python loop is
 * far too slow.  TEST INFRASTRUCTURE ONLY (linked into the oracle library,
 * never into the product).  Not a restatement of a reference function: it
 * builds the permuted input the oracle then runs on (D1).
 *
 * New row i = old row perm[i]; each row's entries sorted by new column
 * index iperm[old col] (explicit zeros kept), exactly as permute_csr.
 * Rows are split over `threads` pthreads; the result does not depend on it.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

typedef struct {
    int64_t n, r0, r1;
    const int64_t *rp, *ci, *perm, *iperm, *nrp;
    const double* v;
    int64_t* nci;
    double* nv;
} job_t;

static void* run(void* arg) {
    job_t* J = (job_t*)arg;
    int64_t cap = 256;
    int64_t* key = (int64_t*)malloc(sizeof(int64_t) * cap);
    int64_t* src = (int64_t*)malloc(sizeof(int64_t) * cap);
    for (int64_t i = J->r0; i < J->r1; ++i) {
        const int64_t o = J->perm[i], b = J->rp[o], len = J->rp[o + 1] - b;
        if (len > cap) {
            cap = len;
            key = (int64_t*)realloc(key, sizeof(int64_t) * cap);
            src = (int64_t*)realloc(src, sizeof(int64_t) * cap);
        }
        /* insertion sort by new column (rows hold <= ~100 entries, mostly
           already in order: node blocks keep their components ascending) */
        for (int64_t q = 0; q < len; ++q) {
            const int64_t kk = J->iperm[J->ci[b + q]], ss = b + q;
            int64_t p = q;
            while (p > 0 && key[p - 1] > kk) {
                key[p] = key[p - 1];
                src[p] = src[p - 1];
                --p;
            }
            key[p] = kk;
            src[p] = ss;
        }
        const int64_t d = J->nrp[i];
        for (int64_t q = 0; q < len; ++q) {
            J->nci[d + q] = key[q];
            J->nv[d + q] = J->v[src[q]];
        }
    }
    free(key);
    free(src);
    return NULL;
}

int or_permute_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                   const int64_t* perm, int threads, int64_t* nrp, int64_t* nci, double* nv) {
    if (n < 0 || !rp || !ci || !v || !perm || !nrp || !nci || !nv) return 1;
    int64_t* iperm = (int64_t*)malloc(sizeof(int64_t) * (n > 0 ? n : 1));
    if (!iperm) return 1;
    for (int64_t i = 0; i < n; ++i) iperm[i] = -1;
    for (int64_t i = 0; i < n; ++i) {
        if (perm[i] < 0 || perm[i] >= n || iperm[perm[i]] != -1) {
            free(iperm);
            return 1; /* not a permutation */
        }
        iperm[perm[i]] = i;
    }
    nrp[0] = 0;
    for (int64_t i = 0; i < n; ++i) nrp[i + 1] = nrp[i] + (rp[perm[i] + 1] - rp[perm[i]]);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    job_t jobs[256];
    for (int t = 0; t < threads; ++t) {
        job_t J = {n, n * t / threads, n * (t + 1) / threads, rp, ci, perm, iperm, nrp, v, nci, nv};
        jobs[t] = J;
        pthread_create(&th[t], NULL, run, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(iperm);
    return 0;
}
