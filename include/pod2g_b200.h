/*
 * pod2g_b200.h -- C-ABI of the B200-native POD-2G solve path.
 *
 * This is the drop-in boundary for the reference's solve phase
 * (/root/reference/proj/include/pod2g/, cited as file:line below):
 *
 *   reference                                           this ABI
 *   CsrMatrix (core/csr.hpp:14-59)                      p2g_set_pattern + p2g_set_values
 *   PodBasis::phi_r (pod.hpp:19-25)                     p2g_set_basis
 *   Pod2gPreconditioner ctor (pod.hpp:261-263)          p2g_setup   (A_c = Phi^T K Phi + factor)
 *     -> Pod2gOperator ctor (pod.hpp:186-189)
 *     -> reduced_operator (pod.hpp:152-165), DenseLu (core/dense_solve.hpp:15-38)
 *   reduced_solve (pod.hpp:167-179)                     p2g_initial_guess
 *   pcg_solve (krylov.hpp:243-297) + SolveReport        p2g_solve
 *     (core/report.hpp:13-23)
 *   spmv (core/csr.hpp:83-93)                           p2g_spmv        (test hook)
 *   Pod2gPreconditioner::apply (pod.hpp:264-267)        p2g_precond_apply (test hook)
 *   gauss_seidel_sweep[_backward] (smoothers.hpp:26-72) p2g_smooth      (test hook)
 *
 * One handle owns one CUDA device, one stream, one sparsity pattern, one POD
 * basis and a BATCH of B value sets sharing the pattern (the instances the
 * reference runs one per parallel_for slot, core/parallel.hpp:16-43).  A
 * handle is not thread-safe; many handles on many threads/devices are
 * (the reference's reentrancy contract, krylov.hpp:12-13).
 *
 * Host arrays are instance-major, like B separate std::vector<double>:
 * values [B][nnz], vectors [B][n], coarse matrices [B][k][k].  Indices use
 * the reference's size_t (uint64_t); they are range-checked and narrowed to
 * int32 on the device.
 *
 * Errors: every call returns a p2g_status.  P2G_EINVAL mirrors the
 * reference's std::invalid_argument (require(), core/types.hpp:15-17); the
 * per-instance codes of p2g_solve mirror its std::runtime_error cases
 * (krylov.hpp:265-266, 274-275, 287-288, 295; core/dense_solve.hpp:25-26;
 * smoothers.hpp:41-43).  p2g_last_error() holds the message.
 *
 * There is no CPU fallback: without a CUDA device p2g_create fails with
 * P2G_ECUDA.
 */
#ifndef POD2G_B200_H
#define POD2G_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define P2G_ABI_VERSION 2

typedef struct p2g_handle p2g_handle;

typedef enum {
    P2G_OK = 0,
    P2G_EINVAL = 1,      /* invalid argument / dimension mismatch (require)          */
    P2G_EBREAKDOWN = 2,  /* r.s <= 0, p^T K p <= 0, or rs' <= 0 (krylov.hpp:265-288)  */
    P2G_ENONFINITE = 3,  /* non-finite entries in solution (krylov.hpp:295)          */
    P2G_ESINGULAR = 4,   /* coarse operator not SPD / singular (dense_solve.hpp:25)  */
    P2G_EZERODIAG = 5,   /* zero diagonal in a smoother row (smoothers.hpp:41-43)    */
    P2G_ECUDA = 6,       /* CUDA runtime error / no device                           */
    P2G_ENCCL = 7,       /* NCCL error (row-partitioned handles)                      */
    P2G_ESTATE = 8       /* call order violated (e.g. solve before setup)            */
} p2g_status;

typedef enum {
    /* Symmetric Gauss-Seidel in node-colour order: forward sweep over colours
     * 0..C-1, backward over C-1..0, the dofs of one node in ascending
     * (forward) / descending (backward) order.  Identical to the reference's
     * natural-order sweeps (smoothers.hpp:26-72) applied to the
     * colour-permuted system P K P^T -- the stated reordering deviation. */
    P2G_SMOOTHER_GS_MULTICOLOR = 0,
    /* Damped Jacobi, exactly jacobi_sweep (smoothers.hpp:75-87): no reordering. */
    P2G_SMOOTHER_JACOBI = 1
} p2g_smoother;

typedef enum {
    /* t = r - K s with the reference's full row sum (csr.hpp:96-105). */
    P2G_RESIDUAL_FULL = 0,
    /* After ONE forward GS sweep from s = 0, (D+L) s = r holds row by row, so
     * t = r - K s = -U s: only the strictly-upper part of each row is read
     * (half a matrix pass).  Same value up to rounding.  Used only when
     * smoother == GS_MULTICOLOR and r1 == 1; otherwise FULL is used. */
    P2G_RESIDUAL_UPPER = 1
} p2g_residual_form;

typedef enum {
    /* Kp = spmv(K, p) every iteration (krylov.hpp:272), the reference form. */
    P2G_KP_SPMV = 0,
    /* With the GS smoother the backward sweep leaves (D+U) s = r - L s' row by
     * row (s' = the prolongated vector), so K s = r + L (s - s') and
     *   Kp_new = r + L (s - s') + beta Kp:
     * the SpMV and the p update become one half-matrix pass.  Same values up
     * to rounding.  Ignored (SPMV) for the Jacobi smoother. */
    P2G_KP_RECURRENCE = 1
} p2g_kp_update;

typedef struct {
    int32_t smoother;       /* p2g_smoother; reference default GS (smoothers.hpp:10-14)  */
    int32_t pre_sweeps;     /* r1 >= 1 (pod.hpp:186, bench.hpp:122)                      */
    int32_t post_sweeps;    /* r2 >= 1                                                   */
    int32_t residual_form;  /* p2g_residual_form                                         */
    double omega;           /* damped Jacobi weight in (0,1] (smoothers.hpp:79)           */
    int32_t kp_update;      /* p2g_kp_update                                             */
    int32_t reserved;
} p2g_config;

/* Initialise cfg with the defaults: GS_MULTICOLOR, r1 = r2 = 1, RESIDUAL_UPPER,
 * KP_RECURRENCE, omega = 0.5 (2/3, the reference default, is unsafe for these
 * operators: see DESIGN.md). */
void p2g_config_default(p2g_config* cfg);

/* ---- lifetime ---------------------------------------------------------- */
int p2g_create(int device, p2g_handle** out);
int p2g_destroy(p2g_handle* h);
const char* p2g_last_error(const p2g_handle* h);
const char* p2g_status_string(int status);
int p2g_abi_version(void);

/* ---- data -------------------------------------------------------------- */
/* Optional, BEFORE p2g_set_pattern: the number of instances the handle will be
 * solved with (0 = unknown, the default).  The reference builds one
 * Pod2gPreconditioner per instance (bench.hpp:315-330, inside parallel_for,
 * core/parallel.hpp:16-43), so it has no such notion; here the batch shares one
 * pattern analysis, and a large batch on a large pattern (nnz x batch >= 2^29
 * for 2 dofs per node, >= 1.5 x 2^30 otherwise; at least 9 instances) is
 * coloured with the 64-class wavefront colouring instead of the greedy one
 * (fewer PCG iterations, D1).  Results are valid for any later batch
 * size; only the iteration count / speed trade-off depends on the hint. */
int p2g_set_batch_hint(p2g_handle* h, int64_t batch);

/* Square CSR pattern (CsrMatrix::validate invariants, csr.hpp:33-46: offsets
 * non-decreasing from 0 to nnz, columns strictly increasing and < n, every
 * row holding its diagonal).  block_size = dofs per node (rows
 * node*bs .. node*bs+bs-1 belong to one node; 1 = point colouring).  The
 * node graph is coloured greedily in natural order (or by wavefronts, see
 * p2g_set_batch_hint). */
int p2g_set_pattern(p2g_handle* h, int64_t n, const uint64_t* row_offsets,
                    const uint64_t* col_indices, int32_t block_size);

/* B value sets [B][nnz] in the pattern's natural order (host memory).
 * Resets any previous setup. */
int p2g_set_values(p2g_handle* h, int32_t batch, const double* values);
/* Same, from device memory of the handle's device ([B][nnz]). */
int p2g_set_values_device(p2g_handle* h, int32_t batch, const double* d_values);
/* Pipelining for batch streams (the reference's caller loops over batches of
 * instances, bench.hpp:290-330): request the host->device copy of the NEXT
 * batch's values [B][nnz] and return at once.  The copy runs on the handle's
 * copy stream, started by the next p2g_solve right after it has uploaded its
 * right-hand sides, so it overlaps that solve without delaying it.  A later
 * p2g_set_values with the same pointer and batch consumes the copy (device
 * relayout only; it starts the copy itself if no solve did).  The host
 * buffer must stay valid and unchanged (and should be pinned) until then. */
int p2g_prefetch_values(p2g_handle* h, int32_t batch, const double* values);

/* POD basis Phi, n x k row-major (PodBasis::phi_r, pod.hpp:20; rank k).
 * k == 0 disables the coarse correction (pure symmetric smoother). */
int p2g_set_basis(p2g_handle* h, int32_t k, const double* phi);

/* Per-instance setup (Pod2gOperator ctor, pod.hpp:186-189): A_c = Phi^T K Phi
 * and its Cholesky factor.  status (may be NULL) receives B codes
 * (P2G_ESINGULAR for a singular coarse operator, P2G_EZERODIAG for a zero
 * smoother diagonal).  Returns the worst code. */
int p2g_setup(p2g_handle* h, const p2g_config* cfg, int32_t* status);

/* ---- solve ------------------------------------------------------------- */
/* x0 = Phi A_c^{-1} Phi^T b per instance (reduced_solve, pod.hpp:167-179).
 * b, x0: host [B][n]. */
int p2g_initial_guess(p2g_handle* h, const double* b, double* x0);

enum {
    P2G_X0_ZERO = 0,      /* u0 empty => zero (krylov.hpp:247)                  */
    P2G_X0_GIVEN = 1,     /* x0 argument                                        */
    P2G_X0_REDUCED = 2,   /* x0 = reduced_solve(K, b, Phi), computed on device  */
    P2G_X0_SURROGATE = 3  /* x0 = predict(model, theta_b) (p2g_set_surrogate +
                             p2g_set_theta), computed on device                 */
};

/* ---- surrogate warm start ---------------------------------------
 * predict(model, theta) = Phi * denormalize(mlp(normalize(theta)))
 * (surrogate.hpp:354-357), the x0 run_monte_carlo uses (bench.hpp:418-420).
 * The model's linear decoder is the handle's basis (p2g_set_basis); the MLP:
 *   nlayers >= 1 dense layers, widths[0..nlayers] (input p, hidden..., output
 *   = the basis rank k), activation on hidden layers only (Mlp::forward,
 *   surrogate.hpp:62-74): P2G_ACT_TANH / P2G_ACT_RELU;
 *   weights = the row-major W_l (widths[l+1] x widths[l]) concatenated in
 *   layer order, biases likewise -- the order of the reference's weights.bin;
 *   in_mean/in_std [p], lat_mean/lat_std [k]: AffineNormalizer
 *   (surrogate.hpp:144-157).  Widths up to 4096. */
enum { P2G_ACT_TANH = 0, P2G_ACT_RELU = 1 };
int p2g_set_surrogate(p2g_handle* h, int32_t nlayers, const int32_t* widths, int32_t activation,
                      const double* weights, const double* biases, const double* in_mean,
                      const double* in_std, const double* lat_mean, const double* lat_std);
/* parameters theta [B][p] (host) of the instances, for P2G_X0_SURROGATE */
int p2g_set_theta(p2g_handle* h, const double* theta);
/* x [B][n] (host) = predict(model, theta_b) per instance (sets theta too) */
int p2g_surrogate_predict(p2g_handle* h, const double* theta, double* x);

/* pcg_solve per instance (krylov.hpp:243-297) with the POD-2G preconditioner.
 *   b        [B][n]   right-hand sides
 *   x0       [B][n]   initial guesses (x0_mode == P2G_X0_GIVEN), else ignored
 *   tol, max_iter     delta and max_iter of pcg_solve
 *   x        [B][n]   solutions (output)
 *   iters    [B]      SolveReport::cycles
 *   converged[B]      SolveReport::converged
 *   status   [B]      P2G_OK or the error the reference would have thrown
 *   hist     [B][hist_cap] relative residual history incl. the initial entry
 *                     (SolveReport::residual_history); may be NULL
 * Any output pointer may be NULL.  Returns the worst per-instance status. */
int p2g_solve(p2g_handle* h, const double* b, const double* x0, int32_t x0_mode, double tol,
              int64_t max_iter, double* x, int64_t* iters, int32_t* converged, int32_t* status,
              double* hist, int64_t hist_cap);

/* pod2g_solve (pod.hpp:224-256): the standalone POD two-grid iteration
 * u <- cycle(f, u) -- forward GS pre- AND post-smoothing (adjoint_post =
 * false, pod.hpp:196-207; cfg.pre_sweeps / post_sweeps = r1 / r2), coarse
 * correction with A_c from p2g_setup -- until the relative TRUE residual
 * ||f - K u|| / ||f|| <= tol or max_cycles.  Arguments and outputs as
 * p2g_solve (cycles = SolveReport::cycles); needs the GS smoother. */
int p2g_pod2g_solve(p2g_handle* h, const double* b, const double* x0, int32_t x0_mode,
                    double tol, int64_t max_cycles, double* x, int64_t* cycles,
                    int32_t* converged, int32_t* status, double* hist, int64_t hist_cap);

/* Same with b / x0 / x in DEVICE memory ([B][n]); iters/converged/status/hist
 * stay host pointers. */
int p2g_solve_device(p2g_handle* h, const double* d_b, const double* d_x0, int32_t x0_mode,
                     double tol, int64_t max_iter, double* d_x, int64_t* iters,
                     int32_t* converged, int32_t* status, double* hist, int64_t hist_cap);

/* Device time of the last p2g_solve / p2g_solve_device in ms (CUDA events on
 * the handle's stream): [0] = setup-free solve incl. x0, [1] = iteration loop. */
int p2g_last_solve_ms(const p2g_handle* h, double* ms2);

/* ---- test / measurement hooks ---------------------------------------------- */
/* y = K x per instance (spmv, csr.hpp:83-93).  x, y host [B][n]. */
int p2g_spmv(p2g_handle* h, const double* x, double* y);
/* s = B r (Pod2gPreconditioner::apply, pod.hpp:264-267).  host [B][n]. */
int p2g_precond_apply(p2g_handle* h, const double* r, double* s);
/* One smoother sweep in place: direction 0 forward, 1 backward
 * (gauss_seidel_sweep / _backward, smoothers.hpp:26-72, in colour order;
 * jacobi_sweep for the Jacobi smoother).  f, u host [B][n]. */
int p2g_smooth(p2g_handle* h, int32_t direction, const double* f, double* u);
/* Coarse operators A_c [B][k][k] as assembled on the device (before
 * symmetrisation). */
int p2g_coarse_operator(p2g_handle* h, double* Ac);

/* Colour permutation: perm[new] = old (n entries); color_offsets receives
 * ncolors+1 node-row offsets (cap entries at most). */
int p2g_get_permutation(p2g_handle* h, int64_t* perm, int32_t* ncolors, int64_t* color_offsets,
                        int32_t cap);

/* compute_pod's fp64 contractions on the FP64 tensor cores (pod.hpp:81-87 and
 * :120-129), handle-free:
 *   p2g_gram:    G [N][N] (host) = U U^T, the snapshot Gram matrix, U [N][d]
 *                row-major (host, or device with U_on_device = 1);
 *   p2g_combine: Phi [d][r] = U^T W, W [N][r] (host, r <= 64) -- Phi = U Psi
 *                Lambda^{-1/2} with W = Psi Lambda^{-1/2}; Phi is host memory, or
 *                device memory when U_on_device = 1.
 * Deterministic (fixed-order partial sums). */
int p2g_gram(int32_t device, int64_t N, int64_t d, const double* U, int32_t U_on_device, double* G);
int p2g_combine(int32_t device, int64_t N, int64_t d, const double* U, int32_t U_on_device,
                int64_t r, const double* W, double* Phi);

/* Host-only: fnv1a_hash (core/io.hpp:92-99) of a byte payload -- the checksum
 * of the reference's artefacts (weights.bin, vector batches). */
uint64_t p2g_fnv1a64(const void* bytes, int64_t count);

/* Host-only (no device needed): the colouring p2g_set_pattern would use. */
int p2g_analyze_pattern(int64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                        int32_t block_size, int64_t* perm, int32_t* ncolors,
                        int64_t* color_offsets, int32_t cap, char* errbuf, int32_t errcap);

/* Host-only: whether the coloured pattern is node-blocked (every node's
 * block_size rows share one column list of whole neighbour-node blocks, at
 * most 32 neighbour nodes) -- then the node-blocked kernels run.  *blocked =
 * 1 / 0, *nmax = most neighbour nodes of a node (0 if not blocked); returns
 * P2G_OK or P2G_EINVAL for an invalid pattern. */
int p2g_analyze_node_blocking(int64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                              int32_t block_size, int32_t* blocked, int32_t* nmax);

/* Per-kernel-class timing of the iteration loop: the loop body with a CUDA
 * event after every kernel class, captured once as a plain graph and replayed
 * `reps` times on the handle's stream (kernels back to back as in the solve;
 * P2G_PROFILE_EAGER=1: eager launches), on the current state of the last
 * solve (P2G_ESTATE when no solve ran since p2g_setup: a zero state has
 * p'Kp = 0).  ms receives the mean time per iteration of each class, bytes
 * the algorithmic HBM bytes per iteration of each class, names
 * the class names (static). */
#define P2G_NUM_KCLASS 11
int p2g_profile_iteration(p2g_handle* h, int32_t reps, double* ms, double* bytes,
                          const char** names);

/* The handle's CUDA stream (cudaStream_t) -- every kernel of the handle is
 * launched on it; callers time with CUDA events recorded on this stream. */
void* p2g_get_stream(const p2g_handle* h);

/* Test hook.  With P2G_GUARD=1 in the environment (read once, at the first
 * allocation) every handle buffer carries a guard band of a fixed byte
 * pattern on each side; this returns the number of guard bands that changed
 * (out-of-bounds device writes) over all live handles, -1 when guard mode is
 * off, -2 on a CUDA error. */
int p2g_debug_guard_check(void);

/* Kernel launches of one loop iteration, and the running total of every
 * kernel this handle has executed (setup, prologue and graph iterations). */
int p2g_launch_counts(const p2g_handle* h, int64_t* per_iteration, int64_t* total_executed);

/* ---- row-partitioned single system -------------
 * One large system split by contiguous blocks of global rows.  Every rank
 * owns rows [row_bounds[r], row_bounds[r+1]) (multiples of block_size) and
 * keeps ghost copies of the rows its rows couple to.  All ranks use ONE
 * global node colouring (node_colors[g] for every global node g, a proper
 * colouring of the node graph); the multicolour sweeps then equal the
 * single-GPU sweeps in the global colour-major order, with the swept vector's
 * boundary rows exchanged after every colour phase and the scalar partials
 * (p.Kp, ||r||^2, Phi^T t, r.s) summed across ranks.
 *   p2g_part_create_local : all `world` partitions in this process on one
 *                           device (exchange = device copies; for testing and
 *                           single-GPU runs)
 *   p2g_part_create_nccl  : this process is rank `rank` of `world`; exchange
 *                           by NCCL send/recv, sums by NCCL allreduce (uid from
 *                           p2g_nccl_unique_id on one rank, broadcast by the caller)
 * The `rank` argument of the per-partition calls names a hosted partition. */
typedef struct p2g_part p2g_part;
int p2g_nccl_unique_id(void* uid /* 128 bytes */);
int p2g_part_create_local(int device, int world, p2g_part** out);
int p2g_part_create_nccl(int device, int rank, int world, const void* uid, p2g_part** out);
int p2g_part_destroy(p2g_part* p);
const char* p2g_part_last_error(const p2g_part* p);
/* rows [row_bounds[rank], row_bounds[rank+1]) as a CSR with GLOBAL column
 * indices (row_offsets local, n_own+1 entries) */
int p2g_part_set_pattern(p2g_part* p, int rank, int64_t n_global, const int64_t* row_bounds,
                         const uint64_t* row_offsets, const uint64_t* col_indices,
                         int32_t block_size, const int32_t* node_colors);
/* n_own, n_ghost and the global row of every ghost slot (ghost_global may be NULL) */
int p2g_part_ghosts(p2g_part* p, int rank, int64_t* n_own, int64_t* n_ghost,
                    int64_t* ghost_global);
int p2g_part_set_values(p2g_part* p, int rank, int32_t batch, const double* values);
/* phi_own: n_own x k (caller's local row order); phi_ghost: n_ghost x k in
 * p2g_part_ghosts order */
int p2g_part_set_basis(p2g_part* p, int rank, int32_t k, const double* phi_own,
                       const double* phi_ghost);
/* collective over all hosted partitions (and all ranks) */
int p2g_part_setup(p2g_part* p, const p2g_config* cfg, int32_t* status);
/* b, x0, x: one pointer per hosted partition ([B][n_own]); iters / converged
 * / status / hist as p2g_solve (identical on every rank).  x0_mode is
 * P2G_X0_ZERO, P2G_X0_GIVEN or P2G_X0_REDUCED (no surrogate here); anything
 * else is P2G_EINVAL. */
int p2g_part_solve(p2g_part* p, const double* const* b, const double* const* x0, int32_t x0_mode,
                   double tol, int64_t max_iter, double* const* x, int64_t* iters,
                   int32_t* converged, int32_t* status, double* hist, int64_t hist_cap);
int p2g_part_last_solve_ms(const p2g_part* p, double* ms);
/* Kernel launches: per PCG iteration of the captured loop, and the running
 * total over the hosted partitions (graph iterations included); loop_mode =
 * how the last solve's loop ran: 1 conditional-WHILE graph (device-side
 * stopping), 2 captured chunks of 8 iterations with a host poll between
 * chunks, 0 eager (P2G_PART_EAGER=1). */
int p2g_part_launch_counts(const p2g_part* p, int64_t* per_iteration, int64_t* total,
                           int32_t* loop_mode);
/* The stream every hosted partition launches on (cudaStream_t). */
void* p2g_part_get_stream(const p2g_part* p);
/* p2g_profile_iteration for a handle hosting ONE partition (N = 1, or one
 * rank of an NCCL job): eager iterations with CUDA events between kernel
 * classes on the handle's stream; class "halo_allreduce" is the exchange /
 * all-reduce time.  After p2g_part_solve (P2G_ESTATE otherwise). */
int p2g_part_profile_iteration(p2g_part* p, int32_t reps, double* ms, double* bytes,
                               const char** names);
/* Host-only (no device): the partition plan of one rank.  sizes = {n_own,
 * n_ghost, nnz, ncolors}; send_counts / recv_counts ([ncolors][world], zeroed
 * by the caller) accumulate the rows exchanged with each peer per colour. */
int p2g_plan_partition(int rank, int world, const int64_t* row_bounds, int64_t n_global,
                       const uint64_t* row_offsets, const uint64_t* col_indices,
                       int32_t block_size, const int32_t* node_colors, int64_t* sizes,
                       int64_t* ghost_global, int64_t* send_counts, int64_t* recv_counts,
                       char* errbuf, int32_t errcap);

#ifdef __cplusplus
}
#endif
#endif
