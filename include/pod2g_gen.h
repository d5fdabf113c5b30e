/*
 * pod2g_gen.h -- seeded input generator for the BASELINE.json configs.
 *
 * NOT part of the reference boundary: the reference ships only the P1
 * plane-strain `its` and the hex8 Biot problems (problems.hpp:99-344); the
 * benchmark configs need Q4 plane-stress cantilevers and hex8 elasticity with
 * a Karhunen-Loeve lognormal modulus, which this generator provides.  Its
 * conventions follow the reference where one exists:
 *   - Dirichlet dofs removed by row/column elimination, free dofs numbered in
 *     the natural node-major order with components interleaved, exactly as
 *     ConstraintEliminator does (problems.hpp:54-92);
 *   - CSR with strictly increasing columns, explicit zeros kept;
 *   - normals from mt19937_64 raw bits through an inverse normal CDF
 *     (Acklam's rational approximation + one Halley step), the same published
 *     construction as the reference's Rng::normal (core/rng.hpp:12-46).
 */
#ifndef POD2G_GEN_H
#define POD2G_GEN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct p2g_mesh p2g_mesh;

/* dim = 2: Q4 plane stress on [0,Lx]x[0,Ly] with nx x ny square elements
 *          (unit thickness); x = 0 edge clamped; unit traction (0,-1) on x = Lx.
 * dim = 3: hex8 linear elasticity on [0,Lx]x[0,Ly]x[0,Lz], nx x ny x nz cube
 *          elements; x = 0 face clamped; unit traction (0,0,-1) on x = Lx.
 * Elements must be squares / cubes (Lx/nx == Ly/ny [== Lz/nz]). */
int p2g_mesh_create(int32_t dim, int64_t nx, int64_t ny, int64_t nz, double Lx, double Ly,
                    double Lz, double nu, p2g_mesh** out);
void p2g_mesh_destroy(p2g_mesh* m);
int p2g_mesh_info(const p2g_mesh* m, int64_t* n, int64_t* nnz, int64_t* nelem,
                  int32_t* block_size);
int p2g_mesh_pattern(const p2g_mesh* m, uint64_t* row_offsets, uint64_t* col_indices);
/* rows [r0, r1) only (node aligned): rp local (r1-r0+1 entries), global columns */
int p2g_mesh_pattern_range(const p2g_mesh* m, int64_t r0, int64_t r1, uint64_t* row_offsets,
                           uint64_t* col_indices);
/* parity colouring of the free nodes: (ix%2) + 2(iy%2) [+ 4(iz%2)], a proper
 * colouring of the Q4 / hex8 node graph (for the row-partitioned path) */
int p2g_mesh_node_colors(const p2g_mesh* m, int32_t* colors);
/* consistent nodal traction load on the free dofs */
int p2g_mesh_rhs(const p2g_mesh* m, double* f);
/* element stiffness for E = 1 (n_e x n_e, n_e = dim * 2^dim, row-major) */
int p2g_mesh_element_stiffness(const p2g_mesh* m, double* Ke);
/* values[b][nnz] = sum over elements e sharing the entry (ascending e) of
 * E[b][e] * Ke1[local]; nthreads worker threads (<= 0: hardware count). */
int p2g_mesh_assemble(const p2g_mesh* m, int64_t B, const double* E, double* values,
                      int32_t nthreads);
/* The same for the node-aligned free-row range [r0, r1) only (a partition's
 * rows): values[b][nnz_range], nnz_range = row_offsets[r1] - row_offsets[r0]
 * (the p2g_mesh_pattern_range layout).  Identical bits to the full assembly. */
int p2g_mesh_assemble_range(const p2g_mesh* m, int64_t B, const double* E, int64_t r0,
                            int64_t r1, double* values, int32_t nthreads);

/* On-device generation: the B instances K(E_b) written
 * straight into a solver handle whose pattern is this mesh's (p2g_set_pattern
 * with p2g_mesh_pattern), replacing p2g_set_values.  E: [B][nelem] host or
 * device memory.  Same arithmetic as p2g_mesh_assemble (identical bits). */
struct p2g_handle;
struct p2g_part;
int p2g_mesh_assemble_into(const p2g_mesh* m, struct p2g_handle* h, int32_t batch, const double* E,
                           int32_t E_on_device);
/* the same for hosted partition `rank` of a row-partitioned system */
int p2g_part_assemble(struct p2g_part* p, int rank, const p2g_mesh* m, int32_t batch,
                      const double* E, int32_t E_on_device);

/* Lognormal modulus E = exp(g) per element (piecewise constant at element
 * centroids), g = sigma * sum_{m<M} sqrt(lambda_m) phi_m(x) xi_m with the
 * separable squared-exponential covariance exp(-|x-y|^2 / (2 ell^2)):
 * per-axis Nystrom eigenpairs (midpoint rule, `quad` points per axis, cyclic
 * Jacobi), products ranked by eigenvalue, the M largest kept.
 * xi[b][:] are M standard normals from seed seeds[b]; xi may be NULL. */
int p2g_kl_field(const p2g_mesh* m, int32_t M, double sigma, double ell, int32_t quad, int64_t B,
                 const uint64_t* seeds, double* E, double* xi);
/* eigenvalues of the M retained KL modes (descending) */
int p2g_kl_eigenvalues(const p2g_mesh* m, int32_t M, double ell, int32_t quad, double* lambda);
/* count standard normals from mt19937_64(seed) */
int p2g_normal_draws(uint64_t seed, int64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif
