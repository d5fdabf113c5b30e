/*
 * pod2g_oracle.h -- CPU restatement of the reference POD-2G solve path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2207_02543_b200/) links, loads or calls this code.  It is used
 * by tests/ as the parity checker, by __graft_entry__.smoke() as the checker,
 * and by bench.py's cpu_baseline leg.
 *
 * Every function restates one reference function with the same operation
 * order (sequential sums in ascending index order, no fused multiply-add), so
 * that on identical inputs it reproduces the reference bit for bit.  That claim
 * is pinned by tests/test_oracle.py against oracle/_ref (the reference headers
 * compiled unmodified) and against the reference's own known answers.
 *
 * Index arrays are int64 (the reference's index_t is std::size_t,
 * /root/reference/proj/include/pod2g/core/types.hpp:13).
 */
#ifndef POD2G_ORACLE_H
#define POD2G_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same meaning as the product library's P2G_* codes */
enum {
    OR_OK = 0,
    OR_EINVAL = 1,      /* std::invalid_argument from require()           */
    OR_EBREAKDOWN = 2,  /* pcg_solve runtime_error: r.s<=0, pKp<=0, rs'<=0 */
    OR_ENONFINITE = 3,  /* pcg_solve: non-finite entries in solution       */
    OR_ESINGULAR = 4,   /* DenseLu: singular to working precision          */
    OR_EZERODIAG = 5    /* gauss_seidel_sweep: zero diagonal               */
};

enum { OR_SMOOTHER_GS = 0, OR_SMOOTHER_JACOBI = 1 };

typedef struct {
    int64_t n;              /* square: nrows == ncols */
    const int64_t* rp;      /* n+1 */
    const int64_t* ci;      /* nnz */
    const double* v;        /* nnz */
} or_csr;

/* core/types.hpp:52-57 */
double or_dot(int64_t n, const double* x, const double* y);
/* core/csr.hpp:83-93 */
void or_spmv(const or_csr* A, const double* x, double* y);
/* core/csr.hpp:96-105 */
void or_residual(const or_csr* A, const double* f, const double* u, double* r);
/* smoothers.hpp:26-47 */
int or_gs_forward(const or_csr* K, const double* f, double* u, int64_t sweeps);
/* smoothers.hpp:51-72 */
int or_gs_backward(const or_csr* K, const double* f, double* u, int64_t sweeps);
/* smoothers.hpp:75-87 */
int or_jacobi_sweep(const or_csr* K, const double* f, double* u, double omega, int64_t sweeps);
/* pod.hpp:27-35  z = Phi^T u, phi is n x k row-major */
void or_project(int64_t n, int64_t k, const double* phi, const double* u, double* z);
/* pod.hpp:37-46  u = Phi z */
void or_lift(int64_t n, int64_t k, const double* phi, const double* z, double* u);
/* core/dense_solve.hpp:15-38; lu is k*k in/out, perm k */
int or_lu_factor(int64_t k, double* lu, int64_t* perm);
/* core/dense_solve.hpp:40-56 */
void or_lu_solve(int64_t k, const double* lu, const int64_t* perm, const double* b, double* x);
/* pod.hpp:152-165  Ac (k x k row-major) = Phi^T K Phi */
void or_reduced_operator(const or_csr* K, int64_t k, const double* phi, double* Ac);
/* pod.hpp:167-179  x0 = Phi Ac^{-1} Phi^T f; ur (k) optional */
int or_reduced_solve(const or_csr* K, const double* f, int64_t k, const double* phi, double* x0,
                     double* ur);

/* One preconditioner application s = B r of Pod2gPreconditioner::apply
 * (pod.hpp:264-267 -> Pod2gOperator::cycle pod.hpp:196-207) with the coarse LU
 * already factored.  smoother = OR_SMOOTHER_GS (reference default) or
 * OR_SMOOTHER_JACOBI (SmootherConfig{DampedJacobi, sweeps, omega}). */
typedef struct {
    const or_csr* K;
    int64_t k;
    const double* phi;
    const double* lu;       /* k*k factored */
    const int64_t* perm;    /* k */
    int64_t r1, r2;
    int smoother;
    double omega;
} or_pod2g;

int or_pod2g_setup(or_pod2g* P, const or_csr* K, int64_t k, const double* phi, int64_t r1,
                   int64_t r2, int smoother, double omega, double* lu_storage,
                   int64_t* perm_storage);
int or_pod2g_apply(const or_pod2g* P, const double* r, double* s);

/* krylov.hpp:243-297 pcg_solve with Pod2gPreconditioner (k>0) or the
 * identity preconditioner (k == 0, krylov.hpp:21-25).
 * u0 may be NULL (zero guess).  hist receives the relative residual history
 * (initial entry included), up to hist_cap entries; *hist_len the full length.
 * Returns OR_OK or an error code; *iters/*converged/u are filled in either case
 * with the state reached. */
int or_pcg_pod2g(const or_csr* K, const double* f, int64_t k, const double* phi,
                 const double* u0, double delta, int64_t max_iter, int smoother, double omega,
                 int64_t r1, int64_t r2, double* u, int64_t* iters, int* converged,
                 double* hist, int64_t hist_cap, int64_t* hist_len);

/* Batched convenience for the CPU baseline: instances b = 0..B-1 of a shared
 * pattern (values [B][nnz], f/u0/u [B][n]); nthreads worker threads each take
 * whole instances (the role of parallel_for, core/parallel.hpp:16-43). */
int or_pcg_pod2g_batch(int64_t n, const int64_t* rp, const int64_t* ci, int64_t nnz,
                       const double* values, int64_t B, const double* f, int64_t k,
                       const double* phi, const double* u0, double delta, int64_t max_iter,
                       int smoother, double omega, double* u, int64_t* iters, int* converged,
                       int* status, int nthreads);

/* pod.hpp:224-256 pod2g_solve: the standalone two-grid iteration
 * u <- cycle(f, u) with FORWARD post-smoothing (pod.hpp:196-207,
 * adjoint_post = false), stopped on the true relative residual; GS smoother,
 * r1 / r2 sweeps.  hist as or_pcg_pod2g; *cycles = iterations done. */
int or_pod2g_solve(const or_csr* K, const double* f, int64_t k, const double* phi,
                   const double* u0, double delta, int64_t max_cycles, int64_t r1, int64_t r2,
                   double* u, int64_t* cycles, int* converged, double* hist, int64_t hist_cap,
                   int64_t* hist_len);

/* surrogate.hpp:354-357 predict: x = Phi * denormalize(mlp(normalize(theta))).
 * Mlp::forward surrogate.hpp:62-74 (z = b; z_i += W_ij a_j ascending j; hidden
 * activation tanh (act 0) / relu (act 1), identity output); AffineNormalizer
 * surrogate.hpp:144-157.  widths[0..nlayers]; W = the layers' row-major
 * matrices (widths[l+1] x widths[l]) concatenated; bias likewise.  theta [B][p],
 * x [B][n], phi [n][k] with k == widths[nlayers]. */
int or_surrogate_predict(int nlayers, const int64_t* widths, int act, const double* W,
                         const double* bias, const double* in_mean, const double* in_std,
                         const double* lat_mean, const double* lat_std, int64_t n,
                         const double* phi, int64_t B, const double* theta, double* x);

/* csr_permute.c (test infrastructure, not a restatement): P K P^T with new
 * row i = old row perm[i], columns sorted by new index; nrp n+1, nci/nv nnz */
int or_permute_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* v,
                   const int64_t* perm, int threads, int64_t* nrp, int64_t* nci, double* nv);

#ifdef __cplusplus
}
#endif
#endif
