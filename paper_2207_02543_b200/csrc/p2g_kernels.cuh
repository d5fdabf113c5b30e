// p2g_kernels.cuh -- sm_100a kernels of the batched POD-2G PCG solve path.
//
// Data layout in HBM:
//   * rows are in colour-major node order (p2g_pattern.cpp), int32 CSR
//     (rp, ci) shared by all instances, dpos = diagonal position per row;
//   * values  vals[nnz][Bp]   -- the B instances of one nonzero are adjacent,
//     so a warp streams one row with 32*V consecutive doubles per load and
//     the column index is read once for the whole tile (4/B bytes per value);
//   * vectors X[n][Bp]        -- same interleaving, so the x-gathers of a row
//     are also 256/512-byte contiguous;
//   * basis   phi[n][k]       -- PodBasis::phi_r row-major (pod.hpp:20).
//
// Warp tiling (Shape<R,S,W,V>): a warp covers R rows (nodes) x S slot lanes
// per row x W instance lanes, each instance lane owning V instances.
//   B == 1  : R=4,S=8,W=1  (4 rows x 8 slot lanes per warp, 2D and 3D rows)
//   B <= 8  : R=1,S=4,W=8
//   B <= 32 : R=1,S=1,W=32
//   B  > 32 : R=1,S=1,W=32,V=2 (double2 per lane, 64 instances per tile)
// With S == 1 every lane walks its row sequentially in column order with
// separately rounded multiply and add, i.e. exactly the reference's row sums
// (csr.hpp:83-105, smoothers.hpp:26-72); with S > 1 the row is split over
// slot lanes and combined by a fixed xor-shuffle tree.
//
// Node-blocked patterns (FEM vector problems, NodeTab): the sweeps, the upper
// residual and the Kp recurrence walk a node's neighbour NODES instead of
// its rows -- the *_blk kernels (S == 1 shapes: one gather per neighbour node
// for all BS rows, same per-row operation order, bit-identical) and the *_b1
// / *_b1h kernels (B == 1: lane = neighbour node, one node per warp or per
// 16-lane half, rows combined by an xor tree).
//
// All reductions (dot products, Phi^T t) are deterministic: per-block partials
// in a fixed order, then fixed-order warp sums.  No floating-point atomics.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace p2g {

namespace cg = cooperative_groups;

constexpr int kWarps = 8;
constexpr int kBlock = kWarps * 32;
// Reduction-producing kernels run in thread-block clusters of kCluster CTAs:
// the per-CTA partials are combined over DSMEM, so each cluster writes ONE
// partial row.  kCluster = 2 (an SM pair, which always fits): clusters of 8
// leave SM slots idle -- at 2 CTAs/SM only 33 clusters (264 of 296 CTA slots)
// are co-resident, at 1 CTA/SM 15 (120 of 148), ncu launch__cluster_max_active
// -- which cost the hex8 backward sweep 3 % (c4 iteration 15.78 -> 15.61 ms,
// c2 loop 404.1 -> 401.9 us; 4: 15.68 ms / 402.6 us) for 4x the partial rows
// of the per-instance scalar reductions.
#ifndef P2G_KCLUSTER
#define P2G_KCLUSTER 2
#endif
constexpr int kCluster = P2G_KCLUSTER;
#define P2G_CLUSTER __cluster_dims__(kCluster, 1, 1)
// Streaming row kernels are latency bound unless the SM is full: cap them at
// 32 registers so 8 CTAs x 8 warps (100% occupancy) stay resident (the
// difference between 4.4 and 6.3 TB/s for the batched SpMV, tools/spmv_lab.cu).
#ifndef P2G_B1_MINB
#define P2G_B1_MINB 8  // single-instance shapes: CTAs per SM (small spills beat fewer warps)
#endif
#define P2G_ROWK __launch_bounds__(kBlock, Sh::W == 1 ? P2G_B1_MINB : P2G_MINB)
#ifndef P2G_UNROLL
#define P2G_UNROLL 4  // entries of a row in flight per warp (row loops)
#endif
#define P2G_PRAGMA_(x) _Pragma(#x)
#define P2G_PRAGMA(x) P2G_PRAGMA_(x)
#ifndef P2G_MINB
#define P2G_MINB 4
#endif

template <int R_, int S_, int W_, int V_>
struct Shape {
    static constexpr int R = R_, S = S_, W = W_, V = V_, T = W_ * V_;
};
using ShB1a = Shape<4, 8, 1, 1>;
using ShB1b = Shape<1, 32, 1, 1>;
using ShB8 = Shape<1, 4, 8, 1>;
using ShB32 = Shape<1, 1, 32, 1>;
using ShB64 = Shape<1, 1, 32, 2>;

// shape used by kernels that keep k accumulators per lane (restriction,
// K*Phi): one instance per lane to bound registers
template <class Sh>
struct AccShape {
    using type = Sh;
};
template <>
struct AccShape<ShB64> {
    using type = ShB32;
};

struct Mat {
    int n;           // rows
    int bs;          // dofs per node
    const int* rp;   // n+1
    const int* ci;   // nnz
    const int* dpos; // n
    const double* vals;  // [nnz][Bp]
    int Bp;
};

enum : int { ST_OK = 0, ST_EBREAKDOWN = 2, ST_ENONFINITE = 3, ST_ESINGULAR = 4, ST_EZERODIAG = 5 };

struct SolveParams {
    double tol;
    long long max_iter;
    long long hist_cap;
};

// ---------------------------------------------------------------- helpers
template <class Sh>
struct LaneGeo {
    int lane, warp, w, s, r;
    __device__ __forceinline__ LaneGeo() {
        lane = threadIdx.x & 31;
        warp = threadIdx.x >> 5;
        w = lane % Sh::W;
        s = (lane / Sh::W) % Sh::S;
        r = lane / (Sh::W * Sh::S);
    }
};

template <int V>
__device__ __forceinline__ void ldv(double (&d)[V], const double* p) {
    if constexpr (V == 1) {
        d[0] = *p;
    } else {
        const double2 t = *reinterpret_cast<const double2*>(p);
        d[0] = t.x;
        d[1] = t.y;
    }
}
// streamed (evict-first) load for the matrix values: read once per pass
template <int V>
__device__ __forceinline__ void ldv_stream(double (&d)[V], const double* p) {
    if constexpr (V == 1) {
        d[0] = __ldcs(p);
    } else {
        const double2 t = __ldcs(reinterpret_cast<const double2*>(p));
        d[0] = t.x;
        d[1] = t.y;
    }
}
template <int V>
__device__ __forceinline__ void stv(double* p, const double (&d)[V], const bool (&m)[V]) {
    if constexpr (V == 1) {
        if (m[0]) *p = d[0];
    } else {
        if (m[0] && m[1]) {
            *reinterpret_cast<double2*>(p) = make_double2(d[0], d[1]);
        } else {
            if (m[0]) p[0] = d[0];
            if (m[1]) p[1] = d[1];
        }
    }
}

template <class Sh>
__device__ __forceinline__ double slot_sum(double x) {
#pragma unroll
    for (int o = Sh::W; o < Sh::W * Sh::S; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// sum over the (s, r) lanes that share an instance lane w; result in lanes < W
template <class Sh>
__device__ __forceinline__ double inst_sum(double x) {
#pragma unroll
    for (int o = Sh::W; o < 32; o <<= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// acc[v] += sum_{k in [k0,k1), k = k0+s (mod S)} vals[k][b] * X[ci[k]][b]
// (separately rounded multiply and add: the reference's `s += v * x`).
// 64-bit row base, 32-bit offsets inside the row and for the x gathers
// (n * Bp < 2^32 is checked at upload)
// keep the address arithmetic out of 64-bit registers.
template <class Sh>
__device__ __forceinline__ void row_dot(const Mat& A, const double* X, int b0, int k0, int k1,
                                        int s, double (&acc)[Sh::V]) {
    const unsigned Bp = (unsigned)A.Bp;
    const double* Xb = X + b0;
    const double* vb = A.vals + (size_t)k0 * Bp + b0;  // 64-bit row base, 32-bit in-row offsets
P2G_PRAGMA(unroll P2G_UNROLL)
    for (int k = k0 + s; k < k1; k += Sh::S) {
        const unsigned c = (unsigned)__ldg(A.ci + k);
        double a[Sh::V], x[Sh::V];
        ldv_stream<Sh::V>(a, vb + (unsigned)(k - k0) * Bp);
        ldv<Sh::V>(x, Xb + c * Bp);
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) acc[v] = __dadd_rn(acc[v], __dmul_rn(a[v], x[v]));
    }
}

// acc[v] -= vals*X sequentially (gauss_seidel_sweep's `sum -= K_ij u_j`, S == 1 only)
template <class Sh>
__device__ __forceinline__ void row_sub(const Mat& A, const double* X, int b0, int k0, int k1,
                                        double (&acc)[Sh::V]) {
    const unsigned Bp = (unsigned)A.Bp;
    const double* Xb = X + b0;
    const double* vb = A.vals + (size_t)k0 * Bp + b0;
P2G_PRAGMA(unroll P2G_UNROLL)
    for (int k = k0; k < k1; ++k) {
        const unsigned c = (unsigned)__ldg(A.ci + k);
        double a[Sh::V], x[Sh::V];
        ldv_stream<Sh::V>(a, vb + (unsigned)(k - k0) * Bp);
        ldv<Sh::V>(x, Xb + c * Bp);
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) acc[v] = __dsub_rn(acc[v], __dmul_rn(a[v], x[v]));
    }
}

// One Gauss-Seidel row update (smoothers.hpp:31-44):
//   s_i = (f_i - sum_{j != i} K_ij s_j) / K_ii
// upper == false: only the L part is read (first forward sweep from s = 0:
// the U-part entries of s are still zero, and subtracting zeros is exact).
// The L-part values come from xlo, the U-part values from xhi, the result
// goes to s: in place (xlo == xhi == s) for the reference sweeps, or out of
// place for the backward sweep of the Kp recurrence (xlo = s' the
// prolongated vector, xhi = s = the new sweep, D9).
// fo / so (optional) receive f_i and the new s_i on the lanes that store
// them, so a caller's epilogue (the r.s partial) needs no reload.
template <class Sh>
__device__ __forceinline__ void gs_row(const Mat& A, const double* f, const double* xlo,
                                       const double* xhi, double* s, int i, int b0, int lane_s,
                                       bool upper, const bool (&m)[Sh::V], bool any,
                                       double* fo = nullptr, double* so = nullptr) {
    double out[Sh::V];
    if constexpr (Sh::S == 1) {
        if (any) {
            const int kb = __ldg(A.rp + i), kd = __ldg(A.dpos + i), ke = __ldg(A.rp + i + 1);
            double acc[Sh::V], d[Sh::V];
            ldv<Sh::V>(acc, f + (size_t)i * A.Bp + b0);
            if (fo) {
#pragma unroll
                for (int v = 0; v < Sh::V; ++v) fo[v] = acc[v];
            }
            row_sub<Sh>(A, xlo, b0, kb, kd, acc);
            if (upper) row_sub<Sh>(A, xhi, b0, kd + 1, ke, acc);
            ldv<Sh::V>(d, A.vals + (size_t)kd * A.Bp + b0);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) out[v] = __ddiv_rn(acc[v], d[v]);
            stv<Sh::V>(s + (size_t)i * A.Bp + b0, out, m);
            if (so) {
#pragma unroll
                for (int v = 0; v < Sh::V; ++v) so[v] = out[v];
            }
        }
    } else {
        double acc[Sh::V];
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) acc[v] = 0.0;
        int kd = 0;
        if (any) {
            const int kb = __ldg(A.rp + i), ke = __ldg(A.rp + i + 1);
            kd = __ldg(A.dpos + i);
            row_dot<Sh>(A, xlo, b0, kb, kd, lane_s, acc);
            if (upper) row_dot<Sh>(A, xhi, b0, kd + 1, ke, lane_s, acc);
        }
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) acc[v] = slot_sum<Sh>(acc[v]);
        if (any && lane_s == 0) {
            double fi[Sh::V], d[Sh::V];
            ldv<Sh::V>(fi, f + (size_t)i * A.Bp + b0);
            ldv<Sh::V>(d, A.vals + (size_t)kd * A.Bp + b0);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) out[v] = __ddiv_rn(__dsub_rn(fi[v], acc[v]), d[v]);
            stv<Sh::V>(s + (size_t)i * A.Bp + b0, out, m);
            if (fo && so) {
#pragma unroll
                for (int v = 0; v < Sh::V; ++v) {
                    fo[v] = fi[v];
                    so[v] = out[v];
                }
            }
        }
        __syncwarp();  // the next dof of this node reads s_i
    }
}

// Deterministic per-cluster partial: lanes -> warps (fixed order) -> CTA
// total in shared memory -> the cluster's rank-0 CTA sums the kCluster CTA
// totals over DSMEM in rank order and writes (or, ACC, adds to) one row:
//   part[(blockIdx.x / kCluster) * Bp + blockIdx.y * T + t]
template <class Sh>
__device__ __forceinline__ void cluster_partial(double (&acc)[Sh::V], double* part, int Bp,
                                                bool accumulate) {
    __shared__ double sm[kWarps][Sh::T];
    __shared__ double tot[Sh::T];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) acc[v] = inst_sum<Sh>(acc[v]);
    if (lane < Sh::W) {
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) sm[warp][lane * Sh::V + v] = acc[v];
    }
    __syncthreads();
    if (threadIdx.x < Sh::T) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) t += sm[w][threadIdx.x];
        tot[threadIdx.x] = t;
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    if (cl.block_rank() == 0 && threadIdx.x < Sh::T) {
        double t = 0.0;
#pragma unroll
        for (int r = 0; r < kCluster; ++r) t += cl.map_shared_rank(tot, r)[threadIdx.x];
        double* dst = part + (size_t)(blockIdx.x / kCluster) * Bp + blockIdx.y * Sh::T + threadIdx.x;
        *dst = accumulate ? *dst + t : t;
    }
    cl.sync();
}

template <class Sh>
__device__ __forceinline__ void lane_mask(const int* active, int b0, bool (&m)[Sh::V], bool& any) {
    any = false;
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) {
        m[v] = active[b0 + v] != 0;
        any |= m[v];
    }
}

// grid-stride over nodes [nb, ne): node g handled by sub-group r of a warp
#define P2G_NODE_LOOP(Sh, nb, ne, G)                                                         \
    for (int base_ = (nb) + (blockIdx.x * kWarps + (G).warp) * Sh::R; base_ < (ne);        \
         base_ += gridDim.x * kWarps * Sh::R)

// ================================================================ kernels

// y = K x (csr.hpp:83-93) on all rows; DOT: partial of x.y per instance
// (krylov.hpp:272-273: Kp = spmv(K,p); pKp = dot(p, Kp)).
template <class Sh, bool DOT>
__global__ void P2G_CLUSTER P2G_ROWK k_spmv(Mat A, const double* __restrict__ x,
                                                 double* __restrict__ y, const int* active,
                                                 double* part) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double dacc[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) dacc[v] = 0.0;
    const int nn = A.n / A.bs;
    P2G_NODE_LOOP(Sh, 0, nn, G) {
        const int node = base_ + G.r;
        const bool valid = node < nn;
        for (int c = 0; c < A.bs; ++c) {
            const int i = node * A.bs + c;
            double acc[Sh::V];
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = 0.0;
            if (valid && any) row_dot<Sh>(A, x, b0, __ldg(A.rp + i), __ldg(A.rp + i + 1), G.s, acc);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = slot_sum<Sh>(acc[v]);
            if (valid && any && G.s == 0) {
                stv<Sh::V>(y + (size_t)i * A.Bp + b0, acc, m);
                if constexpr (DOT) {
                    double xi[Sh::V];
                    ldv<Sh::V>(xi, x + (size_t)i * A.Bp + b0);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v)
                        dacc[v] = __dadd_rn(dacc[v], __dmul_rn(xi[v], acc[v]));
                }
            }
        }
    }
    if constexpr (DOT) cluster_partial<Sh>(dacc, part, A.Bp, false);
}

enum : int { RES_UPPER = 0, RES_FULL = 1, RES_VECTOR = 2 };

// Residual of the pre-smoothed correction, written to r (the restriction's
// input t, pod.hpp:198-199):
//   RES_FULL : r = f - K u (csr.hpp:96-105: row sum first, then subtract),
//              optional partials of r.r and f.f (||r0||, ||f||, krylov.hpp:252-256)
//   RES_UPPER: r = -U u -- after ONE forward GS sweep from zero,
//              (D + L) u = f row by row, so f - K u = -U u (same value up to
//              rounding, half the matrix traffic: only the strictly upper
//              entries of each row are read)
template <class Sh, int FORM>
__global__ void P2G_CLUSTER P2G_ROWK k_residual(Mat A, const double* __restrict__ f,
                                                     const double* __restrict__ u,
                                                     double* __restrict__ r, const int* active,
                                                     double* part_rr, double* part_ff) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double rr[Sh::V], ff[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) rr[v] = ff[v] = 0.0;
    const int nn = A.n / A.bs;
    P2G_NODE_LOOP(Sh, 0, nn, G) {
        const int node = base_ + G.r;
        const bool valid = node < nn;
        for (int c = 0; c < A.bs; ++c) {
            const int i = node * A.bs + c;
            double acc[Sh::V];
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = 0.0;
            if (valid && any) {
                const int k0 = FORM == RES_UPPER ? __ldg(A.dpos + i) + 1 : __ldg(A.rp + i);
                row_dot<Sh>(A, u, b0, k0, __ldg(A.rp + i + 1), G.s, acc);
            }
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = slot_sum<Sh>(acc[v]);
            if (valid && any && G.s == 0) {
                double ri[Sh::V];
                if constexpr (FORM == RES_UPPER) {
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) ri[v] = -acc[v];
                } else {
                    double fi[Sh::V];
                    ldv<Sh::V>(fi, f + (size_t)i * A.Bp + b0);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) {
                        ri[v] = __dsub_rn(fi[v], acc[v]);
                        rr[v] = __dadd_rn(rr[v], __dmul_rn(ri[v], ri[v]));
                        ff[v] = __dadd_rn(ff[v], __dmul_rn(fi[v], fi[v]));
                    }
                }
                stv<Sh::V>(r + (size_t)i * A.Bp + b0, ri, m);
            }
        }
    }
    if (part_rr) {
        cluster_partial<Sh>(rr, part_rr, A.Bp, false);
        cluster_partial<Sh>(ff, part_ff, A.Bp, false);
    }
}

enum : int { PRE_NONE = 0, PRE_GS = 1, PRE_JACOBI = 2 };

// PCG update fused with the first pre-smoothing step (krylov.hpp:277-279):
//   UPDATE:  u += alpha p ; r += (-alpha) Kp ; partial r.r
//   then     GS: colour-0 nodes' first forward sweep rows (L part only)
//            JACOBI: s_i = omega * r_i / d_i on every row (first sweep from 0,
//            smoothers.hpp:84-85 with u = 0)
template <class Sh, bool UPDATE, int PRE>
__global__ void P2G_CLUSTER P2G_ROWK
    k_update_pre(Mat A, double* __restrict__ u, double* __restrict__ r, const double* __restrict__ p,
                 const double* __restrict__ Kp, double* __restrict__ s, const double* alpha,
                 const int* active, double* part_rr, int color0_nodes, double omega) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double al[Sh::V], rr[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) {
        al[v] = UPDATE ? alpha[b0 + v] : 0.0;
        rr[v] = 0.0;
    }
    const int nn = A.n / A.bs;
    P2G_NODE_LOOP(Sh, 0, nn, G) {
        const int node = base_ + G.r;
        const bool valid = node < nn;
        for (int c = 0; c < A.bs; ++c) {
            const int i = node * A.bs + c;
            if constexpr (UPDATE) {
                if (valid && any && G.s == 0) {
                    double ui[Sh::V], pi[Sh::V], ri[Sh::V], kpi[Sh::V];
                    const size_t o = (size_t)i * A.Bp + b0;
                    ldv<Sh::V>(ui, u + o);
                    ldv<Sh::V>(pi, p + o);
                    ldv<Sh::V>(ri, r + o);
                    ldv<Sh::V>(kpi, Kp + o);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) {
                        ui[v] = __dadd_rn(ui[v], __dmul_rn(al[v], pi[v]));
                        ri[v] = __dadd_rn(ri[v], __dmul_rn(-al[v], kpi[v]));
                        rr[v] = __dadd_rn(rr[v], __dmul_rn(ri[v], ri[v]));
                    }
                    stv<Sh::V>(u + o, ui, m);
                    stv<Sh::V>(r + o, ri, m);
                }
                if constexpr (Sh::S > 1) __syncwarp();
            }
            if constexpr (PRE == PRE_GS) {
                // every lane participates (S > 1 shuffles); only colour-0 rows work
                const bool work = any && valid && node < color0_nodes;
                gs_row<Sh>(A, r, s, s, s, work ? i : 0, b0, G.s, false, m, work);
            } else if constexpr (PRE == PRE_JACOBI) {
                if (valid && any && G.s == 0) {
                    double ri[Sh::V], d[Sh::V], si[Sh::V];
                    const size_t o = (size_t)i * A.Bp + b0;
                    ldv<Sh::V>(ri, r + o);
                    ldv<Sh::V>(d, A.vals + (size_t)__ldg(A.dpos + i) * A.Bp + b0);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v)
                        si[v] = __ddiv_rn(__dmul_rn(omega, ri[v]), d[v]);
                    stv<Sh::V>(s + o, si, m);
                }
            }
        }
    }
    if constexpr (UPDATE) cluster_partial<Sh>(rr, part_rr, A.Bp, false);
}

// Row-parallel PCG update (krylov.hpp:277-278) for the slot-split shapes
// (S > 1, small batches): every lane owns rows, instead of one lane per row
// group as in the fused k_update_pre.  u += alpha p ; r += (-alpha) Kp ;
// cluster partials of r.r.
template <class Sh>
__global__ void P2G_CLUSTER P2G_ROWK k_update_rows(int n, int Bp, double* __restrict__ u,
                                                   double* __restrict__ r,
                                                   const double* __restrict__ p,
                                                   const double* __restrict__ Kp,
                                                   const double* alpha, const int* active,
                                                   double* part_rr) {
    constexpr int W = Sh::W, RL = 32 / Sh::W;
    const int lane = threadIdx.x & 31, w = lane % W, sl = lane / W;
    const int b0 = blockIdx.y * Sh::T + w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double al[Sh::V], rr[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) {
        al[v] = alpha[b0 + v];
        rr[v] = 0.0;
    }
    if (any) {
        for (int i = (blockIdx.x * kWarps + (threadIdx.x >> 5)) * RL + sl; i < n;
             i += gridDim.x * kWarps * RL) {
            const size_t o = (size_t)i * Bp + b0;
            double ui[Sh::V], pi[Sh::V], ri[Sh::V], kpi[Sh::V];
            ldv<Sh::V>(ui, u + o);
            ldv<Sh::V>(pi, p + o);
            ldv<Sh::V>(ri, r + o);
            ldv<Sh::V>(kpi, Kp + o);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) {
                ui[v] = __dadd_rn(ui[v], __dmul_rn(al[v], pi[v]));
                ri[v] = __dadd_rn(ri[v], __dmul_rn(-al[v], kpi[v]));
                rr[v] = __dadd_rn(rr[v], __dmul_rn(ri[v], ri[v]));
            }
            stv<Sh::V>(u + o, ui, m);
            stv<Sh::V>(r + o, ri, m);
        }
    }
    // every lane of an instance holds a partial: reduce over the row lanes
    cluster_partial<Sh>(rr, part_rr, Bp, false);
}

// Forward GS colour phase: nodes [nb, ne) of one colour, dofs ascending.
template <class Sh, bool FIRST>
__global__ void P2G_ROWK k_gs_forward(Mat A, const double* __restrict__ f,
                                                       double* s, const int* active, int nb,
                                                       int ne) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    P2G_NODE_LOOP(Sh, nb, ne, G) {
        const int node = base_ + G.r;
        const bool valid = node < ne;
        for (int c = 0; c < A.bs; ++c)
            gs_row<Sh>(A, f, s, s, s, valid ? node * A.bs + c : 0, b0, G.s, !FIRST, m, any && valid);
    }
}

// Backward GS colour phase: nodes of one colour, dofs descending
// (gauss_seidel_sweep_backward, smoothers.hpp:56-70); LAST: partial of r.s
// over this colour's rows (krylov.hpp:280 rs_new = dot(r, s)).
template <class Sh, bool LAST>
__global__ void P2G_CLUSTER P2G_ROWK k_gs_backward(Mat A, const double* __restrict__ f,
                                                        const double* xlo, double* s,
                                                        const int* active, int nb,
                                                        int ne, double* part_rs, int accumulate) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double rs[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) rs[v] = 0.0;
    P2G_NODE_LOOP(Sh, nb, ne, G) {
        const int node = base_ + G.r;
        const bool valid = node < ne;
        for (int c = A.bs - 1; c >= 0; --c) {
            const int i = valid ? node * A.bs + c : 0;
            if constexpr (LAST) {
                // r.s partial from the row's own f_i and new s_i (no reload)
                double fi[Sh::V], si[Sh::V];
                gs_row<Sh>(A, f, xlo, s, s, i, b0, G.s, true, m, any && valid, fi, si);
                if (valid && any && G.s == 0) {
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) rs[v] = __dadd_rn(rs[v], __dmul_rn(fi[v], si[v]));
                }
            } else {
                gs_row<Sh>(A, f, xlo, s, s, i, b0, G.s, true, m, any && valid);
            }
        }
    }
    if constexpr (LAST) cluster_partial<Sh>(rs, part_rs, A.Bp, accumulate != 0);
}

// Kp recurrence (D9), replacing the SpMV and the p update of the next
// iteration.  After the out-of-place backward sweep, (D + U) s = r - L s'
// row by row (s' = prolongated vector, s = the new sweep), hence
//   K s = r + L (s - s'),   Kp_new = K s + beta Kp = r + L (s - s') + beta Kp,
//   p_new = s + beta p      (krylov.hpp:282),      partial of p_new . Kp_new.
// Only the strictly lower part of each row is read: half a matrix pass.
template <class Sh>
__global__ void P2G_CLUSTER P2G_ROWK k_kp_update(Mat A, const double* __restrict__ r,
                                                 const double* __restrict__ s,
                                                 const double* __restrict__ sp,
                                                 double* __restrict__ Kp, double* __restrict__ p,
                                                 const double* beta, const int* active,
                                                 double* part) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double bt[Sh::V], dacc[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) {
        bt[v] = beta[b0 + v];
        dacc[v] = 0.0;
    }
    const int nn = A.n / A.bs;
    const unsigned Bp = (unsigned)A.Bp;
    P2G_NODE_LOOP(Sh, 0, nn, G) {
        const int node = base_ + G.r;
        const bool valid = node < nn;
        for (int c = 0; c < A.bs; ++c) {
            const int i = node * A.bs + c;
            double acc[Sh::V];
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = 0.0;
            if (valid && any) {
                const int kb = __ldg(A.rp + i), kd = __ldg(A.dpos + i);
                const double* vb = A.vals + (size_t)kb * Bp + b0;
P2G_PRAGMA(unroll P2G_UNROLL)
                for (int k = kb + G.s; k < kd; k += Sh::S) {
                    const unsigned col = (unsigned)__ldg(A.ci + k);
                    double a[Sh::V], x1[Sh::V], x0[Sh::V];
                    ldv_stream<Sh::V>(a, vb + (unsigned)(k - kb) * Bp);
                    ldv<Sh::V>(x1, s + b0 + col * Bp);
                    ldv<Sh::V>(x0, sp + b0 + col * Bp);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v)
                        acc[v] = __dadd_rn(acc[v], __dmul_rn(a[v], __dsub_rn(x1[v], x0[v])));
                }
            }
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = slot_sum<Sh>(acc[v]);
            if (valid && any && G.s == 0) {
                const size_t o = (size_t)i * A.Bp + b0;
                double ri[Sh::V], si[Sh::V], kpi[Sh::V], pi[Sh::V];
                ldv<Sh::V>(ri, r + o);
                ldv<Sh::V>(si, s + o);
                ldv<Sh::V>(kpi, Kp + o);
                ldv<Sh::V>(pi, p + o);
#pragma unroll
                for (int v = 0; v < Sh::V; ++v) {
                    kpi[v] = __dadd_rn(__dadd_rn(ri[v], acc[v]), __dmul_rn(bt[v], kpi[v]));
                    pi[v] = __dadd_rn(si[v], __dmul_rn(bt[v], pi[v]));
                    dacc[v] = __dadd_rn(dacc[v], __dmul_rn(pi[v], kpi[v]));
                }
                stv<Sh::V>(Kp + o, kpi, m);
                stv<Sh::V>(p + o, pi, m);
            }
        }
    }
    cluster_partial<Sh>(dacc, part, A.Bp, false);
}

// Damped Jacobi sweep, out of place (smoothers.hpp:83-86):
//   s_out_i = s_i + omega * (f_i - (K s)_i) / d_i ; LAST: partial of f.s_out
template <class Sh, bool LAST>
__global__ void P2G_CLUSTER P2G_ROWK k_jacobi(Mat A, const double* __restrict__ f,
                                                   const double* __restrict__ s,
                                                   double* __restrict__ s_out, const int* active,
                                                   double omega, double* part_rs) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double rs[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) rs[v] = 0.0;
    const int nn = A.n / A.bs;
    P2G_NODE_LOOP(Sh, 0, nn, G) {
        const int node = base_ + G.r;
        const bool valid = node < nn;
        for (int c = 0; c < A.bs; ++c) {
            const int i = node * A.bs + c;
            double acc[Sh::V];
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = 0.0;
            if (valid && any) row_dot<Sh>(A, s, b0, __ldg(A.rp + i), __ldg(A.rp + i + 1), G.s, acc);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) acc[v] = slot_sum<Sh>(acc[v]);
            if (valid && any && G.s == 0) {
                const size_t o = (size_t)i * A.Bp + b0;
                double fi[Sh::V], si[Sh::V], d[Sh::V], out[Sh::V];
                ldv<Sh::V>(fi, f + o);
                ldv<Sh::V>(si, s + o);
                ldv<Sh::V>(d, A.vals + (size_t)__ldg(A.dpos + i) * A.Bp + b0);
#pragma unroll
                for (int v = 0; v < Sh::V; ++v) {
                    const double res = __dsub_rn(fi[v], acc[v]);
                    out[v] = __dadd_rn(si[v], __ddiv_rn(__dmul_rn(omega, res), d[v]));
                    if (LAST) rs[v] = __dadd_rn(rs[v], __dmul_rn(fi[v], out[v]));
                }
                stv<Sh::V>(s_out + o, out, m);
            }
        }
    }
    if constexpr (LAST) cluster_partial<Sh>(rs, part_rs, A.Bp, false);
}

// ================================================ node-blocked row kernels
// FEM vector problems: every node's BS rows share one column pattern made of
// whole node blocks (checked on the host, p2g_pattern.cpp build_node_table).
// A warp then walks a node's neighbour NODES once for all BS rows:
//   * one x gather (BS consecutive rows of X) serves BS matrix rows,
//   * the neighbour list is one lane-parallel load (lane j = neighbour j,
//     staged in shared memory), prefetched one node ahead,
// so the per-node latency chain shrinks from BS x (row length / unroll)
// dependent ci -> gather rounds to about (neighbours / unroll) rounds.
// Every row still combines its terms in ascending column order with the same
// separately rounded operations, so results are bit-identical to the row
// kernels above (and to the reference's row sums).
// Used for the one-instance-per-lane shapes (S == 1).
// Optional read-only (non-coherent) loads for the node-blocked kernels (RO):
// the values and every x gather are never written by the kernel that reads
// them (other colours' rows, or a row read by the thread that later
// overwrites it), so ld.global.nc may be issued ahead of the kernel's own
// stores.  Measured: it pays only in the Q4 Kp recurrence (c2 93 vs 97 us);
// the sweeps are unchanged (c2) or slower (c4 forward 3.12 vs 2.93 ms).
template <int V, bool RO>
__device__ __forceinline__ void ldv_ro(double (&d)[V], const double* p) {
    if constexpr (!RO) {
        ldv<V>(d, p);
    } else if constexpr (V == 1) {
        d[0] = __ldg(p);
    } else {
        const double2 t = __ldg(reinterpret_cast<const double2*>(p));
        d[0] = t.x;
        d[1] = t.y;
    }
}
template <int V, bool RO>
__device__ __forceinline__ void ldv_vals(double (&d)[V], const double* p) {
    if constexpr (!RO) {
        ldv_stream<V>(d, p);
    } else if constexpr (V == 1) {
        asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(d[0]) : "l"(p));
    } else {
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(d[0]), "=d"(d[1]) : "l"(p));
    }
}

struct NodeTab {
    const int4* info;  // per node {kb0 = first value of row 0, rowlen, pos = own slot, nnb}
    const int* ncol;   // [nodes][nmax] neighbour node ids, ascending
    int nmax;
};

#ifndef P2G_BLK_UNR_L
#define P2G_BLK_UNR_L 1  // neighbour nodes in flight, all-row passes
#endif
#ifndef P2G_BLK_UNR_U
#define P2G_BLK_UNR_U 1  // neighbour nodes in flight, one-row passes, Q4 (c2: 168 vs 172 us at 2)
#endif
#ifndef P2G_BLK_UNR_U_HEX
#define P2G_BLK_UNR_U_HEX 3  // the same for hex8 (c4: 6.30 vs 6.48 ms at 1)
#endif

__device__ __forceinline__ void node_fetch(const NodeTab& T, int node, int lane, int4& inf, int& nc) {
    inf = __ldg(T.info + node);
    nc = lane < T.nmax ? __ldg(T.ncol + (size_t)node * T.nmax + lane) : 0;
}

// acc[c] (-= if SUB else +=) vals(row c, slot j, comp cc) * X[ncol_j*BS + cc]
// for slots j in [j0, j1), rows c in [C0, C1), cc ascending.  DIFF: the
// operand is X - X0 (Kp recurrence).  vb = values of row 0 of the node at
// this lane's instances; nc = the warp's neighbour list in shared memory.
template <class Sh, int BS, int C0, int C1, bool SUB, bool DIFF, int UNR, bool RO = false>
__device__ __forceinline__ void blk_pass(const double* vb, unsigned rowlen, unsigned Bp,
                                         const double* X, const double* X0, const int* nc, int j0,
                                         int j1, double (&acc)[BS][Sh::V]) {
    constexpr int V = Sh::V;
#pragma unroll UNR
    for (int j = j0; j < j1; ++j) {
        const unsigned xo = (unsigned)nc[j] * (unsigned)BS * Bp;
        double x[BS][V];
#pragma unroll
        for (int cc = 0; cc < BS; ++cc) {
            ldv_ro<V, RO>(x[cc], X + xo + cc * Bp);
            if constexpr (DIFF) {
                double x0[V];
                ldv_ro<V, RO>(x0, X0 + xo + cc * Bp);
#pragma unroll
                for (int v = 0; v < V; ++v) x[cc][v] = __dsub_rn(x[cc][v], x0[v]);
            }
        }
#pragma unroll
        for (int c = C0; c < C1; ++c) {
#pragma unroll
            for (int cc = 0; cc < BS; ++cc) {
                double a[V];
                ldv_vals<V, RO>(a, vb + ((unsigned)c * rowlen + (unsigned)(j * BS + cc)) * Bp);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const double pr = __dmul_rn(a[v], x[cc][v]);
                    acc[c][v] = SUB ? __dsub_rn(acc[c][v], pr) : __dadd_rn(acc[c][v], pr);
                }
            }
        }
    }
}

// one row (values at vr = that row's first value): acc -= vals * X over slots [j0, j1)
template <class Sh, int BS, int UNR>
__device__ __forceinline__ void blk_pass_row(const double* vr, unsigned Bp, const double* X,
                                             const int* nc, int j0, int j1, double (&acc)[Sh::V]) {
    constexpr int V = Sh::V;
#pragma unroll UNR
    for (int j = j0; j < j1; ++j) {
        const unsigned xo = (unsigned)nc[j] * (unsigned)BS * Bp;
#pragma unroll
        for (int cc = 0; cc < BS; ++cc) {
            double x[V], a[V];
            ldv_ro<V, false>(x, X + xo + cc * Bp);
            ldv_vals<V, false>(a, vr + (unsigned)(j * BS + cc) * Bp);
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = __dsub_rn(acc[v], __dmul_rn(a[v], x[v]));
        }
    }
}

// node loop with the next node's table entry prefetched; body(node, inf, nc)
#define P2G_BLK_NODE_LOOP(T, nb, ne, ...)                                                    \
    {                                                                                         \
        __shared__ int sh_nc_[kWarps][32];                                                    \
        const int lane_ = threadIdx.x & 31, warp_ = threadIdx.x >> 5;                         \
        const int stride_ = gridDim.x * kWarps;                                               \
        int node_ = (nb) + blockIdx.x * kWarps + warp_;                                       \
        int4 inf_n_ = make_int4(0, 0, 0, 0);                                                  \
        int nc_n_ = 0;                                                                        \
        if (node_ < (ne)) node_fetch(T, node_, lane_, inf_n_, nc_n_);                         \
        for (; node_ < (ne); node_ += stride_) {                                              \
            __syncwarp();                                                                     \
            sh_nc_[warp_][lane_] = nc_n_;                                                     \
            const int4 inf = inf_n_;                                                          \
            __syncwarp();                                                                     \
            if (node_ + stride_ < (ne)) node_fetch(T, node_ + stride_, lane_, inf_n_, nc_n_); \
            const int node = node_;                                                           \
            const int* nc = sh_nc_[warp_];                                                    \
            __VA_ARGS__                                                                       \
        }                                                                                     \
    }

// Forward GS colour phase, first sweep from s = 0 (L part only), all BS rows
// of a node together: lower neighbour nodes, then the node's own lower
// components (new values), then the division (smoothers.hpp:31-44).
#ifndef P2G_FWD_MINB
#define P2G_FWD_MINB P2G_MINB
#endif
#ifndef P2G_FWD_UNR
#define P2G_FWD_UNR P2G_BLK_UNR_L
#endif
// hex8 sweeps: 2 CTAs/SM (128 registers, no spills) beat 4 (64, spilling)
// and 3 -- c4 forward 2.82 / 2.93 / 3.05 ms, backward 6.10 / 6.30 / 6.49 ms
#ifndef P2G_FWD_MINB_HEX
#define P2G_FWD_MINB_HEX 2
#endif
#ifndef P2G_BWD_MINB_HEX
#define P2G_BWD_MINB_HEX 2
#endif
template <class Sh, int BS>
__global__ void __launch_bounds__(kBlock, Sh::W == 1 ? P2G_B1_MINB : (BS == 2 ? P2G_FWD_MINB : P2G_FWD_MINB_HEX))
    k_gs_forward_blk(Mat A, NodeTab T, const double* __restrict__ f, double* s,
                                          const int* active, int nb, int ne) {
    constexpr int V = Sh::V;
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * V;
    bool m[V], any;
    lane_mask<Sh>(active, b0, m, any);
    const unsigned Bp = (unsigned)A.Bp;
    P2G_BLK_NODE_LOOP(T, nb, ne, {
        if (any) {
            const double* vb = A.vals + (size_t)inf.x * Bp + b0;
            const unsigned rl = (unsigned)inf.y, pos = (unsigned)inf.z;
            double* sb = s + (size_t)node * BS * Bp + b0;
            double acc[BS][V];
#pragma unroll
            for (int c = 0; c < BS; ++c) ldv_ro<V, false>(acc[c], f + ((size_t)node * BS + c) * Bp + b0);
            blk_pass<Sh, BS, 0, BS, true, false, P2G_FWD_UNR>(vb, rl, Bp, s + b0, nullptr, nc, 0,
                                                              (int)pos, acc);
            double sn[BS][V];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
#pragma unroll
                for (int cc = 0; cc < c; ++cc) {
                    double a[V];
                    ldv_vals<V, false>(a, vb + (c * rl + pos * BS + cc) * Bp);
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        acc[c][v] = __dsub_rn(acc[c][v], __dmul_rn(a[v], sn[cc][v]));
                }
                double d[V];
                ldv_ro<V, false>(d, vb + (c * rl + pos * BS + c) * Bp);
#pragma unroll
                for (int v = 0; v < V; ++v) sn[c][v] = __ddiv_rn(acc[c][v], d[v]);
                stv<V>(sb + c * Bp, sn[c], m);
            }
        }
    })
}

// Backward GS colour phase (gauss_seidel_sweep_backward, smoothers.hpp:56-70),
// rows of a node descending.  Row c's terms in column order are: lower nodes
// and own components < c (old values, xlo), own components > c (this node's
// new values), upper nodes (new values, s).  Pass 1 runs the lower nodes for
// all rows at once; each row then takes its own pass over the upper nodes
// after the new components it needs (gathers of s hit L1 on the repeat).
// xlo == s: in place; xlo = s' (D9): out of place.  LAST: r.s partial.
template <class Sh, int BS, bool LAST>
__global__ void P2G_CLUSTER
__launch_bounds__(kBlock, Sh::W == 1 ? P2G_B1_MINB : (BS == 2 ? P2G_MINB : P2G_BWD_MINB_HEX)) k_gs_backward_blk(Mat A, NodeTab T, const double* __restrict__ f,
                                                       const double* xlo, double* s,
                                                       const int* active, int nb, int ne,
                                                       double* part_rs, int accumulate) {
    constexpr int V = Sh::V;
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * V;
    bool m[V], any;
    lane_mask<Sh>(active, b0, m, any);
    double rs[V];
#pragma unroll
    for (int v = 0; v < V; ++v) rs[v] = 0.0;
    const unsigned Bp = (unsigned)A.Bp;
    P2G_BLK_NODE_LOOP(T, nb, ne, {
        if (any) {
            const double* vb = A.vals + (size_t)inf.x * Bp + b0;
            const unsigned rl = (unsigned)inf.y, pos = (unsigned)inf.z;
            const int nnb = inf.w;
            const size_t ro = (size_t)node * BS * Bp + b0;
            double acc[BS][V], fi[BS][V];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                ldv_ro<V, false>(fi[c], f + ro + c * Bp);
#pragma unroll
                for (int v = 0; v < V; ++v) acc[c][v] = fi[c][v];
            }
            blk_pass<Sh, BS, 0, BS, true, false, P2G_BLK_UNR_L>(vb, rl, Bp, xlo + b0, nullptr, nc, 0,
                                                                (int)pos, acc);
            // own components below each row (old values)
            if constexpr (BS > 1) {
                double xo[BS - 1][V];
#pragma unroll
                for (int cc = 0; cc < BS - 1; ++cc) ldv_ro<V, false>(xo[cc], xlo + ro + cc * Bp);
#pragma unroll
                for (int c = 1; c < BS; ++c) {
#pragma unroll
                    for (int cc = 0; cc < c; ++cc) {
                        double a[V];
                        ldv_vals<V, false>(a, vb + (c * rl + pos * BS + cc) * Bp);
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            acc[c][v] = __dsub_rn(acc[c][v], __dmul_rn(a[v], xo[cc][v]));
                    }
                }
            }
            double sn[BS][V];
#pragma unroll
            for (int c = BS - 1; c >= 0; --c) {
#pragma unroll
                for (int cc = c + 1; cc < BS; ++cc) {
                    double a[V];
                    ldv_vals<V, false>(a, vb + (c * rl + pos * BS + cc) * Bp);
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        acc[c][v] = __dsub_rn(acc[c][v], __dmul_rn(a[v], sn[cc][v]));
                }
                // one-row pass over the upper nodes
                blk_pass_row<Sh, BS, (BS == 2 ? P2G_BLK_UNR_U : P2G_BLK_UNR_U_HEX)>(
                    vb + c * rl * Bp, Bp, s + b0, nc, (int)pos + 1, nnb, acc[c]);
                double d[V];
                ldv_ro<V, false>(d, vb + (c * rl + pos * BS + c) * Bp);
#pragma unroll
                for (int v = 0; v < V; ++v) sn[c][v] = __ddiv_rn(acc[c][v], d[v]);
                stv<V>(s + ro + c * Bp, sn[c], m);
                if constexpr (LAST) {
#pragma unroll
                    for (int v = 0; v < V; ++v) rs[v] = __dadd_rn(rs[v], __dmul_rn(fi[c][v], sn[c][v]));
                }
            }
        }
    })
    if constexpr (LAST) cluster_partial<Sh>(rs, part_rs, A.Bp, accumulate != 0);
}

// Kp recurrence (D9, see k_kp_update) with node blocking: the L part of all
// BS rows (lower nodes, then own components < c) of s - s'.
// fewer, fatter warps pay here: Q4 (BS = 2) at 2 CTAs/SM with 4 neighbour
// nodes in flight (c2: 96 vs 101 us per iteration); hex8 at 2 CTAs/SM with
// one (c4: 3.40 vs 3.70 ms; 4 nodes in flight spill)
#ifndef P2G_KP_MINB
#define P2G_KP_MINB 2
#endif
#ifndef P2G_KP_UNR
#define P2G_KP_UNR 4
#endif
#ifndef P2G_KP_MINB_HEX
#define P2G_KP_MINB_HEX 2  // hex8, one node in flight, 128 registers: c4 3.40 vs 3.70 ms at 4, 4.55 at 3
#endif
template <class Sh, int BS>
__global__ void P2G_CLUSTER
__launch_bounds__(kBlock, Sh::W == 1 ? P2G_B1_MINB : (BS == 2 ? P2G_KP_MINB : P2G_KP_MINB_HEX)) k_kp_update_blk(Mat A, NodeTab T, const double* __restrict__ r,
                                                     const double* __restrict__ s,
                                                     const double* __restrict__ sp,
                                                     double* __restrict__ Kp, double* __restrict__ p,
                                                     const double* beta, const int* active,
                                                     double* part) {
    constexpr int V = Sh::V;
    constexpr bool KRO = BS == 2;  // read-only loads pay on Q4 only
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * V;
    bool m[V], any;
    lane_mask<Sh>(active, b0, m, any);
    double bt[V], dacc[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        bt[v] = beta[b0 + v];
        dacc[v] = 0.0;
    }
    const unsigned Bp = (unsigned)A.Bp;
    const int nn = A.n / BS;
    P2G_BLK_NODE_LOOP(T, 0, nn, {
        if (any) {
            const double* vb = A.vals + (size_t)inf.x * Bp + b0;
            const unsigned rl = (unsigned)inf.y, pos = (unsigned)inf.z;
            const size_t ro = (size_t)node * BS * Bp + b0;
            double acc[BS][V];
#pragma unroll
            for (int c = 0; c < BS; ++c)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[c][v] = 0.0;
            blk_pass<Sh, BS, 0, BS, false, true, (BS == 2 ? P2G_KP_UNR : P2G_BLK_UNR_L), KRO>(
                vb, rl, Bp, s + b0, sp + b0, nc, 0, (int)pos, acc);
            if constexpr (BS > 1) {
                double xd[BS - 1][V];
#pragma unroll
                for (int cc = 0; cc < BS - 1; ++cc) {
                    double x1[V], x0[V];
                    ldv_ro<V, KRO>(x1, s + ro + cc * Bp);
                    ldv_ro<V, KRO>(x0, sp + ro + cc * Bp);
#pragma unroll
                    for (int v = 0; v < V; ++v) xd[cc][v] = __dsub_rn(x1[v], x0[v]);
                }
#pragma unroll
                for (int c = 1; c < BS; ++c) {
#pragma unroll
                    for (int cc = 0; cc < c; ++cc) {
                        double a[V];
                        ldv_vals<V, KRO>(a, vb + (c * rl + pos * BS + cc) * Bp);
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            acc[c][v] = __dadd_rn(acc[c][v], __dmul_rn(a[v], xd[cc][v]));
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                const size_t o = ro + c * Bp;
                double ri[V], si[V], kpi[V], pi[V];
                ldv_ro<V, KRO>(ri, r + o);
                ldv_ro<V, KRO>(si, s + o);
                ldv_ro<V, KRO>(kpi, Kp + o);
                ldv_ro<V, KRO>(pi, p + o);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    kpi[v] = __dadd_rn(__dadd_rn(ri[v], acc[c][v]), __dmul_rn(bt[v], kpi[v]));
                    pi[v] = __dadd_rn(si[v], __dmul_rn(bt[v], pi[v]));
                    dacc[v] = __dadd_rn(dacc[v], __dmul_rn(pi[v], kpi[v]));
                }
                stv<V>(Kp + o, kpi, m);
                stv<V>(p + o, pi, m);
            }
        }
    })
    cluster_partial<Sh>(dacc, part, A.Bp, false);
}

// Residual after one forward sweep from zero, t = -U u (RES_UPPER, D6), node
// blocked: row c's U part is own components > c, then the upper nodes.
#ifndef P2G_RES_HEX_BLK
#define P2G_RES_HEX_BLK 1  // hex8 upper residual node-blocked at 2 CTAs/SM (c4 2.88 vs 3.21 ms row kernel)
#endif
template <class Sh, int BS>
__global__ void P2G_CLUSTER
__launch_bounds__(kBlock, Sh::W == 1 ? P2G_B1_MINB : (BS == 2 ? P2G_MINB : 2)) k_residual_upper_blk(Mat A, NodeTab T, const double* __restrict__ u,
                                                          double* __restrict__ t,
                                                          const int* active) {
    constexpr int V = Sh::V;
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * V;
    bool m[V], any;
    lane_mask<Sh>(active, b0, m, any);
    const unsigned Bp = (unsigned)A.Bp;
    const int nn = A.n / BS;
    P2G_BLK_NODE_LOOP(T, 0, nn, {
        if (any) {
            const double* vb = A.vals + (size_t)inf.x * Bp + b0;
            const unsigned rl = (unsigned)inf.y, pos = (unsigned)inf.z;
            const int nnb = inf.w;
            const size_t ro = (size_t)node * BS * Bp + b0;
            double acc[BS][V];
#pragma unroll
            for (int c = 0; c < BS; ++c)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[c][v] = 0.0;
            if constexpr (BS > 1) {
                double xo[BS][V];
#pragma unroll
                for (int cc = 1; cc < BS; ++cc) ldv_ro<V, false>(xo[cc], u + ro + cc * Bp);
#pragma unroll
                for (int c = 0; c < BS - 1; ++c) {
#pragma unroll
                    for (int cc = c + 1; cc < BS; ++cc) {
                        double a[V];
                        ldv_vals<V, false>(a, vb + (c * rl + pos * BS + cc) * Bp);
#pragma unroll
                        for (int v = 0; v < V; ++v)
                            acc[c][v] = __dadd_rn(acc[c][v], __dmul_rn(a[v], xo[cc][v]));
                    }
                }
            }
            blk_pass<Sh, BS, 0, BS, false, false, P2G_BLK_UNR_L>(vb, rl, Bp, u + b0, nullptr, nc,
                                                                  (int)pos + 1, nnb, acc);
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                double ti[V];
#pragma unroll
                for (int v = 0; v < V; ++v) ti[v] = -acc[c][v];
                stv<V>(t + ro + c * Bp, ti, m);
            }
        }
    })
}

// ======================= single-instance node-blocked kernels (B = 1)
// One warp per node, lane j = neighbour node j (<= 32): the lane gathers its
// neighbour's BS x values (one contiguous piece) and reads its BS x BS value
// block, so all of a node's rows are summed in ONE round of loads -- no
// row-pointer -> column -> gather chain, and one 4-byte node id per BS*BS
// values instead of a column index per value (B = 1 has no instances to
// amortise index bytes over).  Each row's off-node terms are combined by a
// fixed xor tree, then the node's own BS x BS block is applied in order:
// a rounding-level reassociation, like the slot-split row kernels it
// replaces (tests: <= 1e-12 per sweep, solves +-1 iteration).
#ifndef P2G_B1BLK_MINB
#define P2G_B1BLK_MINB 4  // a whole node's loads in flight per lane need ~60 registers
#endif
#ifndef P2G_B1H_WIDE_MINB
#define P2G_B1H_WIDE_MINB 4  // 128^3: 4 CTAs/SM (small spills) beat 3 (no spills): Kp 0.96 vs 1.03 ms, bwd 1.27 vs 1.33
#endif
__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// lane's contribution to the BS row sums: node slot j of the node whose
// values start at vb (row length rl), x of that neighbour from X
template <int BS>
__device__ __forceinline__ void b1_terms(const double* vb, int rl, int j, const double* X, int col,
                                         double (&p)[BS]) {
    double x[BS];
#pragma unroll
    for (int cc = 0; cc < BS; ++cc) x[cc] = __ldg(X + (size_t)col * BS + cc);
#pragma unroll
    for (int c = 0; c < BS; ++c)
#pragma unroll
        for (int cc = 0; cc < BS; ++cc)
            p[c] = fma(__ldcs(vb + c * rl + j * BS + cc), x[cc], p[c]);
}

// node loop (one node per warp) with the next node's table entry prefetched;
// inf = {kb0, rl, pos, nnb} of `node`, nc = this lane's neighbour id
#define P2G_B1_NODE_LOOP(T, nb, ne, ...)                                                      \
    {                                                                                         \
        const int lane = threadIdx.x & 31;                                                    \
        const int stride_ = gridDim.x * kWarps;                                               \
        int node = (nb) + blockIdx.x * kWarps + (threadIdx.x >> 5);                           \
        int4 inf_n_ = make_int4(0, 0, 0, 0);                                                  \
        int nc_n_ = 0;                                                                        \
        if (node < (ne)) node_fetch(T, node, lane, inf_n_, nc_n_);                            \
        for (; node < (ne); node += stride_) {                                                \
            const int4 inf = inf_n_;                                                          \
            const int nc = nc_n_;                                                             \
            if (node + stride_ < (ne)) node_fetch(T, node + stride_, lane, inf_n_, nc_n_);    \
            __VA_ARGS__                                                                       \
        }                                                                                     \
    }

// the node's own BS x BS block (broadcast loads, issued with the neighbour
// terms so a node costs one round of loads)
template <int BS>
__device__ __forceinline__ void b1_own(const double* vb, int rl, int pos, double (&ob)[BS][BS]) {
#pragma unroll
    for (int c = 0; c < BS; ++c)
#pragma unroll
        for (int cc = 0; cc < BS; ++cc) ob[c][cc] = __ldg(vb + c * rl + pos * BS + cc);
}

// forward GS colour phase, first sweep from zero (L part only)
template <int BS>
__global__ void __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_gs_forward_b1(Mat A, NodeTab T, const double* __restrict__ f, double* s, const int* active,
                    int nb, int ne) {
    if (!active[0]) return;
    P2G_B1_NODE_LOOP(T, nb, ne, {
        const double* vb = A.vals + inf.x;
        const int rl = inf.y, pos = inf.z;
        double ob[BS][BS], fo[BS], p[BS];
        b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            fo[c] = __ldg(f + (size_t)node * BS + c);
            p[c] = 0.0;
        }
        if (lane < pos) b1_terms<BS>(vb, rl, lane, s, nc, p);
#pragma unroll
        for (int c = 0; c < BS; ++c) p[c] = warp_sum(p[c]);
        double sn[BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            double acc = fo[c] - p[c];
#pragma unroll
            for (int cc = 0; cc < c; ++cc) acc -= ob[c][cc] * sn[cc];
            sn[c] = acc / ob[c][c];
        }
#pragma unroll
        for (int c = 0; c < BS; ++c)
            if (lane == c) s[(size_t)node * BS + c] = sn[c];
    })
}

// backward GS colour phase: lower neighbours from xlo, upper from s, in one
// round; own components: below the row from xlo, above it this node's new
// values.  LAST: r.s partial.
template <int BS, bool LAST>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_gs_backward_b1(Mat A, NodeTab T, const double* __restrict__ f, const double* xlo, double* s,
                     const int* active, int nb, int ne, double* part_rs, int accumulate) {
    double rs[1] = {0.0};
    if (active[0]) {
        P2G_B1_NODE_LOOP(T, nb, ne, {
            const double* vb = A.vals + inf.x;
            const int rl = inf.y, pos = inf.z, nnb = inf.w;
            double ob[BS][BS], fo[BS], xo[BS], p[BS];
            b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                fo[c] = __ldg(f + (size_t)node * BS + c);
                xo[c] = __ldg(xlo + (size_t)node * BS + c);
                p[c] = 0.0;
            }
            if (lane < nnb && lane != pos) b1_terms<BS>(vb, rl, lane, lane < pos ? xlo : s, nc, p);
#pragma unroll
            for (int c = 0; c < BS; ++c) p[c] = warp_sum(p[c]);
            double sn[BS];
#pragma unroll
            for (int c = BS - 1; c >= 0; --c) {
                double acc = fo[c] - p[c];
#pragma unroll
                for (int cc = 0; cc < BS; ++cc) {
                    if (cc == c) continue;
                    acc -= ob[c][cc] * (cc < c ? xo[cc] : sn[cc]);
                }
                sn[c] = acc / ob[c][c];
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                if (lane == c) s[(size_t)node * BS + c] = sn[c];
                if (LAST && lane == 0) rs[0] += fo[c] * sn[c];
            }
        })
    }
    if constexpr (LAST) cluster_partial<ShB1a>(rs, part_rs, A.Bp, accumulate != 0);
}

// Kp recurrence (D9): Kp = r + L (s - s') + beta Kp, p = s + beta p, pKp
// partial.  Lane c < BS owns row c's epilogue; its vector loads go out with
// the neighbour terms (every row is read and written by its owner only).
template <int BS>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_kp_update_b1(Mat A, NodeTab T, const double* __restrict__ r, const double* __restrict__ s,
                   const double* __restrict__ sp, double* __restrict__ Kp, double* __restrict__ p,
                   const double* beta, const int* active, double* part) {
    double dacc[1] = {0.0};
    if (active[0]) {
        const double bt = beta[0];
        const int nn = A.n / BS;
        P2G_B1_NODE_LOOP(T, 0, nn, {
            const double* vb = A.vals + inf.x;
            const int rl = inf.y, pos = inf.z;
            const int c_own = lane < BS ? lane : 0;
            const size_t o = (size_t)node * BS + c_own;
            double ob[BS][BS], xd[BS], q[BS];
            b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                xd[c] = __ldg(s + (size_t)node * BS + c) - __ldg(sp + (size_t)node * BS + c);
                q[c] = 0.0;
            }
            const double ri = __ldg(r + o), si = __ldg(s + o), kpo = __ldg(Kp + o), po = __ldg(p + o);
            if (lane < pos) {
                double x[BS];
#pragma unroll
                for (int cc = 0; cc < BS; ++cc)
                    x[cc] = __ldg(s + (size_t)nc * BS + cc) - __ldg(sp + (size_t)nc * BS + cc);
#pragma unroll
                for (int c = 0; c < BS; ++c)
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc)
                        q[c] = fma(__ldcs(vb + c * rl + lane * BS + cc), x[cc], q[c]);
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = warp_sum(q[c]);
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                if (lane != c) continue;
                double acc = q[c];
#pragma unroll
                for (int cc = 0; cc < c; ++cc) acc += ob[c][cc] * xd[cc];
                const double kpi = (ri + acc) + bt * kpo;
                const double pi = si + bt * po;
                Kp[o] = kpi;
                p[o] = pi;
                dacc[0] += pi * kpi;
            }
        })
    }
    cluster_partial<ShB1a>(dacc, part, A.Bp, false);
}

// residual after one forward sweep from zero, t = -U u (D6)
template <int BS>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_residual_upper_b1(Mat A, NodeTab T, const double* __restrict__ u, double* __restrict__ t,
                        const int* active) {
    if (!active[0]) return;
    const int nn = A.n / BS;
    P2G_B1_NODE_LOOP(T, 0, nn, {
        const double* vb = A.vals + inf.x;
        const int rl = inf.y, pos = inf.z, nnb = inf.w;
        double ob[BS][BS], uo[BS], q[BS];
        b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            uo[c] = __ldg(u + (size_t)node * BS + c);
            q[c] = 0.0;
        }
        if (lane > pos && lane < nnb) b1_terms<BS>(vb, rl, lane, u, nc, q);
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = warp_sum(q[c]);
#pragma unroll
        for (int c = 0; c < BS; ++c) {
            if (lane != c) continue;
            double acc = 0.0;
#pragma unroll
            for (int cc = c + 1; cc < BS; ++cc) acc += ob[c][cc] * uo[cc];
            t[(size_t)node * BS + c] = -(acc + q[c]);
        }
    })
}

// Half-pass kernels for wide nodes (hex8: up to 26 lower or upper neighbour
// nodes): TWO nodes per warp, one per 16-lane half, lane l of a half taking
// neighbour slots l and l + 16 -- twice the busy lanes of one node per warp
// when only the lower (or upper) neighbours take part.
__device__ __forceinline__ double half_sum(double x) {
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

// Each half-warp's next node-table entry (info + its two neighbour-id slots)
// is fetched one iteration ahead, so an iteration costs one round of loads
// (values, gathers, own block) instead of table -> ids -> gathers.
#define P2G_B1H_NODE_LOOP(T, nb, ne, ...)                                                      \
    {                                                                                          \
        const int lane = threadIdx.x & 31, hl = lane & 15;                                     \
        const int stride_ = gridDim.x * kWarps * 2;                                            \
        int base_ = (nb) + (blockIdx.x * kWarps + (threadIdx.x >> 5)) * 2;                     \
        int4 inf_n_ = make_int4(0, 0, 0, 0);                                                   \
        int nc0_n_ = 0, nc1_n_ = 0;                                                            \
        auto fetch_ = [&](int b_) {                                                            \
            const int nd_ = b_ + (lane >> 4);                                                  \
            if (nd_ < (ne)) {                                                                  \
                inf_n_ = __ldg(T.info + nd_);                                                  \
                const int* nl_ = T.ncol + (size_t)nd_ * T.nmax;                                \
                nc0_n_ = hl < T.nmax ? __ldg(nl_ + hl) : 0;                                    \
                nc1_n_ = hl + 16 < T.nmax ? __ldg(nl_ + hl + 16) : 0;                          \
            }                                                                                  \
        };                                                                                     \
        if (base_ < (ne)) fetch_(base_);                                                       \
        for (; base_ < (ne); base_ += stride_) {                                               \
            const int node = base_ + (lane >> 4);                                              \
            const bool valid = node < (ne);                                                    \
            const int4 inf = inf_n_;                                                           \
            const int nc0 = nc0_n_, nc1 = nc1_n_;                                              \
            if (base_ + stride_ < (ne)) fetch_(base_ + stride_);                               \
            __VA_ARGS__                                                                        \
        }                                                                                      \
    }

// the value a lane of a node's half-warp stores: row hl's entry of v[BS]
// (predicated selects -- no dynamic register indexing, which would spill the
// array to local memory)
template <int BS>
__device__ __forceinline__ double pick_row(const double (&v)[BS], int hl) {
    double o = v[0];
#pragma unroll
    for (int c = 1; c < BS; ++c) o = hl == c ? v[c] : o;
    return o;
}

// forward sweep from zero, hex8, two nodes per warp (lower neighbours only)
template <int BS>
__global__ void __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_gs_forward_b1h(Mat A, NodeTab T, const double* __restrict__ f, double* s, const int* active,
                     int nb, int ne) {
    if (!active[0]) return;
    P2G_B1H_NODE_LOOP(T, nb, ne, {
        const int nd = node;
        double ob[BS][BS], fo[BS], q[BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = 0.0;
        const double* vb = A.vals + inf.x;
        const int rl = inf.y, pos = inf.z;
        if (valid) {
            b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
            for (int c = 0; c < BS; ++c) fo[c] = __ldg(f + (size_t)nd * BS + c);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = hl + 16 * h;
                if (j < pos) b1_terms<BS>(vb, rl, j, s, h ? nc1 : nc0, q);
            }
        }
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
        if (valid) {
            double sn[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                double acc = fo[c] - q[c];
#pragma unroll
                for (int cc = 0; cc < c; ++cc) acc -= ob[c][cc] * sn[cc];
                sn[c] = acc / ob[c][c];
            }
            if (hl < BS) s[(size_t)nd * BS + hl] = pick_row<BS>(sn, hl);
        }
    })
}

// backward sweep, hex8, two nodes per warp (every neighbour: slots l, l + 16)
template <int BS, bool LAST>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1H_WIDE_MINB)
    k_gs_backward_b1h(Mat A, NodeTab T, const double* __restrict__ f, const double* xlo, double* s,
                      const int* active, int nb, int ne, double* part_rs, int accumulate,
                      double* dlt) {
    double rs[1] = {0.0};
    if (active[0]) {
        P2G_B1H_NODE_LOOP(T, nb, ne, {
            const double* vb = A.vals + inf.x;
            const int rl = inf.y, pos = inf.z, nnb = inf.w;
            double ob[BS][BS], fo[BS], xo[BS], q[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = 0.0;
            if (valid) {
                b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    fo[c] = __ldg(f + (size_t)node * BS + c);
                    xo[c] = __ldg(xlo + (size_t)node * BS + c);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = hl + 16 * h;
                    if (j < nnb && j != pos) b1_terms<BS>(vb, rl, j, j < pos ? xlo : s, h ? nc1 : nc0, q);
                }
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
            if (valid) {
                double sn[BS];
#pragma unroll
                for (int c = BS - 1; c >= 0; --c) {
                    double acc = fo[c] - q[c];
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) {
                        if (cc == c) continue;
                        acc -= ob[c][cc] * (cc < c ? xo[cc] : sn[cc]);
                    }
                    sn[c] = acc / ob[c][c];
                }
                if (hl < BS) {
                    const double sv = pick_row<BS>(sn, hl);
                    s[(size_t)node * BS + hl] = sv;
                    // s - s' of the out-of-place last sweep, for the Kp recurrence's gathers
                    if (dlt) dlt[(size_t)node * BS + hl] = sv - pick_row<BS>(xo, hl);
                }
                if (LAST && hl == 0) {
#pragma unroll
                    for (int c = 0; c < BS; ++c) rs[0] += fo[c] * sn[c];
                }
            }
        })
    }
    if constexpr (LAST) cluster_partial<ShB1a>(rs, part_rs, A.Bp, accumulate != 0);
}

template <int BS>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1H_WIDE_MINB)
    k_kp_update_b1h(Mat A, NodeTab T, const double* __restrict__ r, const double* __restrict__ s,
                    const double* __restrict__ sp, double* __restrict__ Kp, double* __restrict__ p,
                    const double* beta, const int* active, double* part,
                    const double* __restrict__ dlt) {
    double dacc[1] = {0.0};
    if (active[0]) {
        const double bt = beta[0];
        const int nn = A.n / BS;
        P2G_B1H_NODE_LOOP(T, 0, nn, {
            const double* vb = A.vals + inf.x;
            const int rl = inf.y, pos = inf.z;
            double ob[BS][BS], xd[BS], q[BS];
            const int c_own = hl < BS ? hl : 0;
            const size_t o = (size_t)node * BS + c_own;
            double ri = 0, si = 0, kpo = 0, po = 0;
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = 0.0;
            if (valid) {
                b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
                for (int c = 0; c < BS; ++c)
                    xd[c] = dlt ? __ldg(dlt + (size_t)node * BS + c)
                                : __ldg(s + (size_t)node * BS + c) - __ldg(sp + (size_t)node * BS + c);
                ri = __ldg(r + o), si = __ldg(s + o), kpo = __ldg(Kp + o), po = __ldg(p + o);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = hl + 16 * h;
                    if (j < pos) {
                        const int col = h ? nc1 : nc0;
                        double x[BS];
                        // s - s' was stored by the last backward sweep for the owned rows
                        const bool pre = dlt && col * BS < A.n;
#pragma unroll
                        for (int cc = 0; cc < BS; ++cc)
                            x[cc] = pre ? __ldg(dlt + (size_t)col * BS + cc)
                                        : __ldg(s + (size_t)col * BS + cc) - __ldg(sp + (size_t)col * BS + cc);
#pragma unroll
                        for (int c = 0; c < BS; ++c)
#pragma unroll
                            for (int cc = 0; cc < BS; ++cc)
                                q[c] = fma(__ldcs(vb + c * rl + j * BS + cc), x[cc], q[c]);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
            if (valid) {
                double lo[BS];  // every row's L(s - s') term; lane hl < BS keeps row hl's
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    double acc = q[c];
#pragma unroll
                    for (int cc = 0; cc < c; ++cc) acc += ob[c][cc] * xd[cc];
                    lo[c] = acc;
                }
                if (hl < BS) {
                    const double kpi = (ri + pick_row<BS>(lo, hl)) + bt * kpo;
                    const double pi = si + bt * po;
                    Kp[o] = kpi;
                    p[o] = pi;
                    dacc[0] += pi * kpi;
                }
            }
        })
    }
    cluster_partial<ShB1a>(dacc, part, A.Bp, false);
}

template <int BS>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_residual_upper_b1h(Mat A, NodeTab T, const double* __restrict__ u, double* __restrict__ t,
                         const int* active) {
    if (!active[0]) return;
    const int nn = A.n / BS;
    P2G_B1H_NODE_LOOP(T, 0, nn, {
        const double* vb = A.vals + inf.x;
        const int rl = inf.y, pos = inf.z, nnb = inf.w;
        double ob[BS][BS], uo[BS], q[BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = 0.0;
        if (valid) {
            b1_own<BS>(vb, rl, pos, ob);
#pragma unroll
            for (int c = 0; c < BS; ++c) uo[c] = __ldg(u + (size_t)node * BS + c);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = hl + 16 * h;
                if (j > pos && j < nnb) b1_terms<BS>(vb, rl, j, u, h ? nc1 : nc0, q);
            }
        }
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
        if (valid) {
            double tv[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int cc = c + 1; cc < BS; ++cc) acc += ob[c][cc] * uo[cc];
                tv[c] = -(acc + q[c]);
            }
            if (hl < BS) t[(size_t)node * BS + hl] = pick_row<BS>(tv, hl);
        }
    })
}


// Restriction c = Phi^T t (PodBasis::project, pod.hpp:27-35) of a vector
// t[n][Bp] (the residual, or f itself for reduced_solve, pod.hpp:171).
// Lanes: R = 32/W rows x W instance lanes x V instances; each lane keeps the
// k coefficients of its V instances in registers and reads its row of Phi
// with 16-byte vector loads.  Partials: one row per cluster (DSMEM),
// part[cluster][a][b].
template <class Sh, int KMAX>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock) k_restrict_vec(int n, int Bp,
                                                         const double* __restrict__ t,
                                                         const double* __restrict__ phi, int k,
                                                         const int* active, double* part) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    double acc[KMAX][Sh::V];
#pragma unroll
    for (int a = 0; a < KMAX; ++a)
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) acc[a][v] = 0.0;
    const bool keven = (k & 1) == 0;
#pragma unroll 2
    for (int base = (blockIdx.x * kWarps + G.warp) * Sh::R; base < n;
         base += gridDim.x * kWarps * Sh::R) {
        const int i = base + G.r;
        if (i >= n || !any) continue;
        double tv[Sh::V];
        ldv<Sh::V>(tv, t + (size_t)i * Bp + b0);
        const double* ph = phi + (size_t)i * k;
        if (keven) {
#pragma unroll
            for (int a = 0; a < KMAX; a += 2) {
                if (a < k) {
                    const double2 p2 = __ldg(reinterpret_cast<const double2*>(ph + a));
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) {
                        acc[a][v] = fma(p2.x, tv[v], acc[a][v]);
                        acc[a + 1][v] = fma(p2.y, tv[v], acc[a + 1][v]);
                    }
                }
            }
        } else {
#pragma unroll
            for (int a = 0; a < KMAX; ++a) {
                if (a < k) {
                    const double pa = __ldg(ph + a);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) acc[a][v] = fma(pa, tv[v], acc[a][v]);
                }
            }
        }
    }
    // CTA reduction in chunks of 8 coefficients, then the cluster's rank-0
    // CTA sums the kCluster CTA totals over DSMEM: one partial row per cluster
    __shared__ double sm[kWarps][8][Sh::T];
    __shared__ double tot[KMAX][Sh::T];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int a0 = 0; a0 < KMAX; a0 += 8) {
        if (a0 >= k) break;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) {
                const double x = inst_sum<Sh>(acc[a0 + j][v]);
                if (lane < Sh::W) sm[warp][j][lane * Sh::V + v] = x;
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 8 * Sh::T; e += kBlock) {
            const int j = e / Sh::T, bt = e % Sh::T;
            double tt = 0.0;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) tt += sm[w][j][bt];
            tot[a0 + j][bt] = tt;
        }
        __syncthreads();
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    {  // every CTA of the cluster sums its share of the entries (same rank order)
        double* prow = part + (size_t)(blockIdx.x / kCluster) * k * Bp + blockIdx.y * Sh::T;
        for (int e = threadIdx.x + (int)cl.block_rank() * kBlock; e < k * Sh::T; e += kBlock * kCluster) {
            const int a = e / Sh::T, bt = e % Sh::T;
            double tt = 0.0;
#pragma unroll
            for (int r = 0; r < kCluster; ++r) tt += cl.map_shared_rank(&tot[0][0], r)[a * Sh::T + bt];
            prow[(size_t)a * Bp + bt] = tt;
        }
    }
    cl.sync();
}

// Coarse correction (pod.hpp:200): c = sum of the restriction partials
// (fixed order), e = A_c^{-1} c with the LDL^T factor of A_c (L unit lower in
// the strict lower triangle, D on the diagonal; row-major [Bp][k][k]).
// One block per instance.
__global__ void __launch_bounds__(kBlock) k_coarse(int Bp, int k, int nblk, const double* part,
                                                   const double* L, double* e, const int* active) {
    const int b = blockIdx.x;
    if (!active[b]) return;
    __shared__ double c[64];
    __shared__ double Ls[64 * 64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int a = warp; a < k; a += kWarps) {
        double t = 0.0;
#pragma unroll 4
        for (int blk = lane; blk < nblk; blk += 32) t += part[((size_t)blk * k + a) * Bp + b];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) c[a] = t;
    }
    const double* Lb = L + (size_t)b * k * k;
    for (int e2 = threadIdx.x; e2 < k * k; e2 += kBlock) Ls[e2] = Lb[e2];
    __syncthreads();
    if (warp == 0) {
        // forward: L y = c (unit diagonal); lane j owns y_j, y_{j+32}
        double y0 = lane < k ? c[lane] : 0.0, y1 = lane + 32 < k ? c[lane + 32] : 0.0;
        for (int j = 0; j < k; ++j) {
            const double yj = __shfl_sync(0xffffffffu, j < 32 ? y0 : y1, j & 31);
            if (lane > j && lane < k) y0 -= Ls[lane * k + j] * yj;
            if (lane + 32 > j && lane + 32 < k) y1 -= Ls[(lane + 32) * k + j] * yj;
        }
        // z = D^{-1} y
        if (lane < k) y0 /= Ls[lane * k + lane];
        if (lane + 32 < k) y1 /= Ls[(lane + 32) * k + lane + 32];
        // backward: L^T x = z
        for (int j = k - 1; j >= 0; --j) {
            const double xj = __shfl_sync(0xffffffffu, j < 32 ? y0 : y1, j & 31);
            if (lane < j) y0 -= Ls[j * k + lane] * xj;
            if (lane + 32 < j) y1 -= Ls[j * k + lane + 32] * xj;
        }
        if (lane < k) e[(size_t)lane * Bp + b] = y0;
        if (lane + 32 < k) e[(size_t)(lane + 32) * Bp + b] = y1;
    }
}

// Prolongation + add (pod.hpp:201-202: corr = lift(e); u += 1.0 * corr), the
// lift sum in ascending coefficient order like PodBasis::lift (pod.hpp:40-44)
// with fused multiply-adds (rounding-level deviation, D4).
// ASSIGN: s = corr (reduced_solve's lift into a fresh vector, pod.hpp:178).
// Same lane layout as k_restrict_vec; e (k x V) lives in registers.
template <class Sh, int KMAX, bool ASSIGN>
__global__ void __launch_bounds__(kBlock) k_prolong(int n, int Bp, double* s,
                                                    const double* __restrict__ phi, int k,
                                                    const double* __restrict__ e,
                                                    const int* active) {
    LaneGeo<Sh> G;
    const int b0 = blockIdx.y * Sh::T + G.w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    if (!any) return;
    double ev[KMAX][Sh::V];
#pragma unroll
    for (int a = 0; a < KMAX; ++a)
        if (a < k) ldv<Sh::V>(ev[a], e + (size_t)a * Bp + b0);
    const bool keven = (k & 1) == 0;
#pragma unroll 2
    for (int base = (blockIdx.x * kWarps + G.warp) * Sh::R; base < n;
         base += gridDim.x * kWarps * Sh::R) {
        const int i = base + G.r;
        if (i >= n) continue;
        const double* ph = phi + (size_t)i * k;
        double corr[Sh::V];
#pragma unroll
        for (int v = 0; v < Sh::V; ++v) corr[v] = 0.0;
        if (keven) {
#pragma unroll
            for (int a = 0; a < KMAX; a += 2) {
                if (a < k) {
                    const double2 p2 = __ldg(reinterpret_cast<const double2*>(ph + a));
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) {
                        corr[v] = fma(p2.x, ev[a][v], corr[v]);
                        corr[v] = fma(p2.y, ev[a + 1][v], corr[v]);
                    }
                }
            }
        } else {
#pragma unroll
            for (int a = 0; a < KMAX; ++a) {
                if (a < k) {
                    const double pa = __ldg(ph + a);
#pragma unroll
                    for (int v = 0; v < Sh::V; ++v) corr[v] = fma(pa, ev[a][v], corr[v]);
                }
            }
        }
        const size_t o = (size_t)i * Bp + b0;
        if constexpr (!ASSIGN) {
            double si[Sh::V];
            ldv<Sh::V>(si, s + o);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) corr[v] = __dadd_rn(si[v], corr[v]);
        }
        stv<Sh::V>(s + o, corr, m);
    }
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA) helpers for the staged tensor-core restriction /
// prolongation (k_restrict_mma / k_prolong_mma): warp 0 streams each 32-row
// tile of T (or S) and of Phi into one of NS shared-memory stages with
// cp.async.bulk, completion signalled on the stage's mbarrier (expect_tx).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "P2G_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra P2G_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (16-byte aligned addresses, size multiple of 16)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// L2 evict-first policy for streamed-once bulk copies (the matrix values)
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// ================= bulk-copy staged backward GS colour phases (Q4, one instance tile)
// The register-fed node kernels above keep ~2 KB of matrix values in flight
// per warp (one neighbour node), so a node is a chain of ~9 load rounds and a
// short colour phase (c2: ~8k nodes, < 2 nodes per warp) is mostly ramp and
// tail.  Here a warp owns one shared-memory slot and fetches a node's WHOLE
// value block -- BS consecutive rows of one instance tile are contiguous when
// Bp == Sh::T -- with one cp.async.bulk (up to 18 KB, L2 evict-first)
// completing on the warp's mbarrier, while its lanes gather the neighbours' x
// into registers.  A node costs one round trip, and an SM keeps NW x 18 KB
// (144 KB at NW = 8) of values in flight instead of 64 KB.  The row sums run
// from shared memory in exactly the order of k_gs_backward_blk (ascending
// columns, separately rounded multiply / subtract): bit-identical results.
// Reduction partials: one row per CTA (no cluster).
// c2 (per colour phase launch, back to back in a graph): backward sweep 171 ->
// 139 us per iteration; the fixed-length graph loop 439.5 -> 408.8 us per
// iteration (tools/probe_loop.py).  NW = 7..10 are equivalent; at 216 KB of
// slots (NW = 12) the 12 KB of L1 left throttles the gathers (158 us).
// Measured and rejected: two slots per warp with the next node's
// block in flight (the gathers then sit on the critical path: 157-162 us), a
// per-row refill ring (142), a staged forward sweep (87-91 vs 83 us), and the
// whole sweep as one persistent launch with a grid barrier between phases
// (125 us by the per-class events but 410.5 vs 408.8 us in the graph loop).
constexpr int kStgNmax = 9;  // Q4: at most 9 neighbour nodes (own included)
#ifndef P2G_STG_NW_DEFAULT
#define P2G_STG_NW_DEFAULT 8  // warps per CTA of the staged backward phases (0: register-fed kernels)
#endif

template <class Sh, int NW>
struct StgGeo {
    static constexpr int BS = 2;
    static constexpr int SLOT = BS * BS * kStgNmax * Sh::T;  // doubles per warp slot
    static constexpr size_t smem = (size_t)NW * SLOT * sizeof(double);
    static constexpr int minb = NW >= 12 ? 1 : 12 / NW;
};

template <class Sh, int NW>
__device__ __forceinline__ void stg_cta_partial(double (&acc)[Sh::V], double* part, int Bp,
                                                bool accumulate) {
    __shared__ double sm[NW][Sh::T];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) sm[warp][lane * Sh::V + v] = acc[v];
    __syncthreads();
    if (threadIdx.x < Sh::T) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += sm[w][threadIdx.x];
        double* dst = part + (size_t)blockIdx.x * Bp + threadIdx.x;
        *dst = accumulate ? *dst + t : t;
    }
}

template <class Sh, int NW, bool LAST>
__global__ void __launch_bounds__(NW * 32, StgGeo<Sh, NW>::minb)
    k_gs_backward_stg(Mat A, NodeTab T, const double* __restrict__ f, const double* xlo, double* s,
                      const int* active, int nb, int ne, double* part_rs, int accumulate) {
    constexpr int V = Sh::V, BS = 2, TT = Sh::T, SLOT = StgGeo<Sh, NW>::SLOT;
    extern __shared__ __align__(128) double stg_smem[];
    __shared__ uint64_t bars[NW];
    __shared__ int sh_nc[NW][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = lane * V;
    bool m[V], any;
    lane_mask<Sh>(active, b0, m, any);
    double rs[V];
#pragma unroll
    for (int v = 0; v < V; ++v) rs[v] = 0.0;
    double* slot = stg_smem + warp * SLOT;
    uint64_t* bar = &bars[warp];
    if (lane == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    __syncwarp();
    const uint64_t pol = l2_evict_first_policy();
    uint32_t parity = 0;
    // warp-major node order: consecutive nodes on consecutive CTAs, so a
    // partly filled last round leaves every SM equally busy
    const int stride = gridDim.x * NW;
    int node = nb + warp * (int)gridDim.x + (int)blockIdx.x;
    int4 inf_n = make_int4(0, 0, 0, 0);
    int nc_n = 0;
    const bool wany = __any_sync(0xffffffffu, any);  // some instance of the tile is still active
    if (wany && node < ne) node_fetch(T, node, lane, inf_n, nc_n);
    for (; wany && node < ne; node += stride) {
        __syncwarp();  // every lane is done with the slot and the list of the previous node
        sh_nc[warp][lane] = nc_n;
        const int4 inf = inf_n;
        __syncwarp();
        const unsigned rl = (unsigned)inf.y;
        const int pos = inf.z, nnb = inf.w;
        if (lane == 0) {
            // the node's BS rows are one contiguous block of BS * rowlen entries
            const uint32_t bytes = (uint32_t)(BS * rl * TT * sizeof(double));
            mbar_arrive_tx(bar, bytes);
            bulk_g2s_hint(slot, A.vals + (size_t)inf.x * TT, bytes, bar, pol);
        }
        if (node + stride < ne) node_fetch(T, node + stride, lane, inf_n, nc_n);
        const int* nc = sh_nc[warp];
        const size_t ro = (size_t)node * BS * TT + b0;
        // gathers: lower nodes and the node's own old components from xlo,
        // upper nodes (already swept colours) from s
        double x[kStgNmax][BS][V], fi[BS][V];
#pragma unroll
        for (int j = 0; j < kStgNmax; ++j) {
            if (j < nnb) {
                const double* src = (j <= pos ? xlo : s) + (size_t)((unsigned)nc[j] * BS * TT) + b0;
#pragma unroll
                for (int cc = 0; cc < BS; ++cc) ldv<V>(x[j][cc], src + cc * TT);
            }
        }
#pragma unroll
        for (int c = 0; c < BS; ++c) ldv<V>(fi[c], f + ro + c * TT);
        mbar_wait(bar, parity);
        parity ^= 1u;
        double sn[BS][V];
#pragma unroll
        for (int c = BS - 1; c >= 0; --c) {
            double acc[V], d[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                acc[v] = fi[c][v];
                d[v] = 1.0;
            }
            const double* vr = slot + (unsigned)c * rl * TT + b0;
#pragma unroll
            for (int j = 0; j < kStgNmax; ++j) {
                if (j < nnb) {
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) {
                        double a[V];
                        ldv<V>(a, vr + (j * BS + cc) * TT);
                        const bool own = j == pos;
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            // x[pos][.]: old components below c, new ones above (patched
                            // in below); the diagonal entry is kept aside
                            const double nv = __dsub_rn(acc[v], __dmul_rn(a[v], x[j][cc][v]));
                            if (cc == c) {
                                acc[v] = own ? acc[v] : nv;
                                d[v] = own ? a[v] : d[v];
                            } else {
                                acc[v] = nv;
                            }
                        }
                    }
                }
            }
#pragma unroll
            for (int v = 0; v < V; ++v) sn[c][v] = __ddiv_rn(acc[v], d[v]);
            stv<V>(s + ro + c * TT, sn[c], m);
            if (c > 0) {
                // the rows above read this node's new component c
#pragma unroll
                for (int j = 0; j < kStgNmax; ++j)
#pragma unroll
                    for (int v = 0; v < V; ++v) x[j][c][v] = j == pos ? sn[c][v] : x[j][c][v];
            }
            if constexpr (LAST) {
#pragma unroll
                for (int v = 0; v < V; ++v) rs[v] = __dadd_rn(rs[v], __dmul_rn(fi[c][v], sn[c][v]));
            }
        }
    }
    if constexpr (LAST) stg_cta_partial<Sh, NW>(rs, part_rs, A.Bp, accumulate != 0);
}

// ============ bulk-copy staged single-instance hex8 kernels (c5's kernels)
// The two-nodes-per-warp kernels above are bound by L1 wavefronts, not DRAM:
// a lane reads its neighbour slot's 3 x 3 value block with nine 8-byte loads
// at a 24-byte lane stride (every 32-byte sector is requested ~3.5 times:
// ~430 sector requests per node pair) next to ~190 for the x gathers.  The
// staged forms fetch each node's whole value block (BS rows x rowlen, up to
// 1944 contiguous bytes) with ONE cp.async.bulk into the half-warp's
// shared-memory slot -- the copy engine, not the load pipe, moves the matrix --
// and the lanes read their blocks from shared memory (stride of 3 doubles:
// conflict free).  The x gathers and the node's own vector entries are issued
// before the warp waits on its mbarrier.  Lane mapping, fma order and xor tree
// are those of the register-fed kernels: results are bit-identical.
// A node's block starts at an 8-byte aligned value index; the copy starts at
// the 16-byte aligned address at or below it (the values array carries two
// doubles of slack at its end).
constexpr int kB1SlotDoubles = 256;  // per node: 3 * 81 values + alignment slack
#ifndef P2G_B1S_DEFAULT
#define P2G_B1S_DEFAULT 6  // backward sweep and Kp recurrence (128^3: 1265 -> 1153 us, 960 -> 917 us); forward 715 -> 878, residual unchanged
#endif

// terms of neighbour slot j from the staged block vs (row length rl)
template <int BS>
__device__ __forceinline__ void b1s_terms(const double* vs, int rl, int j, const double (&x)[BS],
                                          double (&p)[BS]) {
#pragma unroll
    for (int c = 0; c < BS; ++c)
#pragma unroll
        for (int cc = 0; cc < BS; ++cc) p[c] = fma(vs[c * rl + j * BS + cc], x[cc], p[c]);
}
template <int BS>
__device__ __forceinline__ void b1s_own(const double* vs, int rl, int pos, double (&ob)[BS][BS]) {
#pragma unroll
    for (int c = 0; c < BS; ++c)
#pragma unroll
        for (int cc = 0; cc < BS; ++cc) ob[c][cc] = vs[c * rl + pos * BS + cc];
}

// Node loop of the staged kernels: as P2G_B1H_NODE_LOOP, plus per iteration
// the two bulk copies of the warp's node pair (issued by lane 0 of each half)
// on the warp's mbarrier.  The body gathers first, then calls B1S_WAIT() and
// reads the values through `vs`.
#define P2G_B1S_NODE_LOOP(MODE, BS, A, T, nb, ne, ...)                                              \
    {                                                                                          \
        extern __shared__ __align__(128) double b1s_smem[];                                    \
        __shared__ uint64_t b1s_bars[kWarps];                                                  \
        const int lane = threadIdx.x & 31, hl = lane & 15, warp_ = threadIdx.x >> 5;           \
        double* slot_ = b1s_smem + (warp_ * 2 + (lane >> 4)) * kB1SlotDoubles;                 \
        uint64_t* bar_ = &b1s_bars[warp_];                                                     \
        if (lane == 0) {                                                                       \
            mbar_init(bar_, 1);                                                                \
            mbar_fence_init();                                                                 \
        }                                                                                      \
        __syncwarp();                                                                          \
        const uint64_t pol_ = l2_evict_first_policy();                                         \
        uint32_t par_ = 0;                                                                     \
        const int stride_ = gridDim.x * kWarps * 2;                                            \
        int base_ = (nb) + (blockIdx.x * kWarps + warp_) * 2;                                  \
        int4 inf_n_ = make_int4(0, 0, 0, 0);                                                   \
        int nc0_n_ = 0, nc1_n_ = 0;                                                            \
        auto fetch_ = [&](int b_) {                                                            \
            const int nd_ = b_ + (lane >> 4);                                                  \
            if (nd_ < (ne)) {                                                                  \
                inf_n_ = __ldg(T.info + nd_);                                                  \
                const int* nl_ = T.ncol + (size_t)nd_ * T.nmax;                                \
                nc0_n_ = hl < T.nmax ? __ldg(nl_ + hl) : 0;                                    \
                nc1_n_ = hl + 16 < T.nmax ? __ldg(nl_ + hl + 16) : 0;                          \
            }                                                                                  \
        };                                                                                     \
        if (base_ < (ne)) fetch_(base_);                                                       \
        for (; base_ < (ne); base_ += stride_) {                                               \
            const int node = base_ + (lane >> 4);                                              \
            const bool valid = node < (ne);                                                    \
            const int4 inf = inf_n_;                                                           \
            const int nc0 = nc0_n_, nc1 = nc1_n_;                                              \
            __syncwarp(); /* the previous pair's slot reads are done */                        \
            {                                                                                  \
                /* lane hl < BS copies the part of row hl the kernel reads (MODE 0: lane 0  */ \
                /* copies the whole block; 1: [0, own block]; 2: [own block, row end)),     */ \
                /* widened to 16-byte aligned value indices; same offsets in the slot       */ \
                int e0_ = 0, e1_ = 0;                                                          \
                if (valid && hl < ((MODE) == 0 ? 1 : BS)) {                                    \
                    e0_ = (MODE) == 0 ? 0 : hl * inf.y + ((MODE) == 2 ? inf.z * BS : 0);       \
                    e1_ = (MODE) == 0 ? BS * inf.y                                             \
                                      : hl * inf.y + ((MODE) == 1 ? (inf.z + 1) * BS : inf.y); \
                }                                                                              \
                const int a0_ = (inf.x + e0_) & ~1, a1_ = (inf.x + e1_ + 1) & ~1;              \
                const uint32_t by_ = e1_ > e0_ ? (uint32_t)((a1_ - a0_) * sizeof(double)) : 0u; \
                const uint32_t tot_ = __reduce_add_sync(0xffffffffu, by_);                     \
                if (lane == 0) mbar_arrive_tx(bar_, tot_);                                     \
                __syncwarp();                                                                  \
                if (by_) bulk_g2s_hint(slot_ + (a0_ - (inf.x & ~1)), A.vals + a0_, by_, bar_, pol_); \
            }                                                                                  \
            const double* vs = slot_ + (inf.x & 1);                                            \
            if (base_ + stride_ < (ne)) fetch_(base_ + stride_);                               \
            __VA_ARGS__                                                                        \
        }                                                                                      \
    }
#define B1S_WAIT()              \
    mbar_wait(bar_, par_ & 1u); \
    par_ ^= 1u;

template <int BS>
__global__ void __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_gs_forward_b1s(Mat A, NodeTab T, const double* __restrict__ f, double* s, const int* active,
                     int nb, int ne) {
    if (!active[0]) return;
    P2G_B1S_NODE_LOOP(1, BS, A, T, nb, ne, {
        const int nd = node;
        double ob[BS][BS], fo[BS], q[BS], x[2][BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = 0.0;
        const int rl = inf.y, pos = inf.z;
        if (valid) {
#pragma unroll
            for (int c = 0; c < BS; ++c) fo[c] = __ldg(f + (size_t)nd * BS + c);
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (hl + 16 * h < pos) {
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) x[h][cc] = __ldg(s + (size_t)(h ? nc1 : nc0) * BS + cc);
                }
        }
        B1S_WAIT()
        if (valid) {
            b1s_own<BS>(vs, rl, pos, ob);
#pragma unroll
            for (int h = 0; h < 2; ++h)
                if (hl + 16 * h < pos) b1s_terms<BS>(vs, rl, hl + 16 * h, x[h], q);
        }
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
        if (valid) {
            double sn[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                double acc = fo[c] - q[c];
#pragma unroll
                for (int cc = 0; cc < c; ++cc) acc -= ob[c][cc] * sn[cc];
                sn[c] = acc / ob[c][c];
            }
            if (hl < BS) s[(size_t)nd * BS + hl] = pick_row<BS>(sn, hl);
        }
    })
}

template <int BS, bool LAST>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1H_WIDE_MINB)
    k_gs_backward_b1s(Mat A, NodeTab T, const double* __restrict__ f, const double* xlo, double* s,
                      const int* active, int nb, int ne, double* part_rs, int accumulate,
                      double* dlt) {
    double rs[1] = {0.0};
    if (active[0]) {
        P2G_B1S_NODE_LOOP(0, BS, A, T, nb, ne, {
            const int rl = inf.y, pos = inf.z, nnb = inf.w;
            double ob[BS][BS], fo[BS], xo[BS], q[BS], x[2][BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = 0.0;
            if (valid) {
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    fo[c] = __ldg(f + (size_t)node * BS + c);
                    xo[c] = __ldg(xlo + (size_t)node * BS + c);
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = hl + 16 * h;
                    if (j < nnb && j != pos) {
                        const double* X = j < pos ? xlo : s;
#pragma unroll
                        for (int cc = 0; cc < BS; ++cc) x[h][cc] = __ldg(X + (size_t)(h ? nc1 : nc0) * BS + cc);
                    }
                }
            }
            B1S_WAIT()
            if (valid) {
                b1s_own<BS>(vs, rl, pos, ob);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int j = hl + 16 * h;
                    if (j < nnb && j != pos) b1s_terms<BS>(vs, rl, j, x[h], q);
                }
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
            if (valid) {
                double sn[BS];
#pragma unroll
                for (int c = BS - 1; c >= 0; --c) {
                    double acc = fo[c] - q[c];
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) {
                        if (cc == c) continue;
                        acc -= ob[c][cc] * (cc < c ? xo[cc] : sn[cc]);
                    }
                    sn[c] = acc / ob[c][c];
                }
                if (hl < BS) {
                    const double sv = pick_row<BS>(sn, hl);
                    s[(size_t)node * BS + hl] = sv;
                    // s - s' of the out-of-place last sweep, for the Kp recurrence's gathers
                    if (dlt) dlt[(size_t)node * BS + hl] = sv - pick_row<BS>(xo, hl);
                }
                if (LAST && hl == 0) {
#pragma unroll
                    for (int c = 0; c < BS; ++c) rs[0] += fo[c] * sn[c];
                }
            }
        })
    }
    if constexpr (LAST) cluster_partial<ShB1a>(rs, part_rs, A.Bp, accumulate != 0);
}

template <int BS>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1H_WIDE_MINB)
    k_kp_update_b1s(Mat A, NodeTab T, const double* __restrict__ r, const double* __restrict__ s,
                    const double* __restrict__ sp, double* __restrict__ Kp, double* __restrict__ p,
                    const double* beta, const int* active, double* part,
                    const double* __restrict__ dlt) {
    double dacc[1] = {0.0};
    if (active[0]) {
        const double bt = beta[0];
        const int nn = A.n / BS;
        P2G_B1S_NODE_LOOP(1, BS, A, T, 0, nn, {
            const int rl = inf.y, pos = inf.z;
            double ob[BS][BS], xd[BS], q[BS], x[2][BS];
            const int c_own = hl < BS ? hl : 0;
            const size_t o = (size_t)node * BS + c_own;
            double ri = 0, si = 0, kpo = 0, po = 0;
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = 0.0;
            if (valid) {
#pragma unroll
                for (int c = 0; c < BS; ++c)
                    xd[c] = dlt ? __ldg(dlt + (size_t)node * BS + c)
                                : __ldg(s + (size_t)node * BS + c) - __ldg(sp + (size_t)node * BS + c);
                ri = __ldg(r + o), si = __ldg(s + o), kpo = __ldg(Kp + o), po = __ldg(p + o);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (hl + 16 * h < pos) {
                        const int col = h ? nc1 : nc0;
                        const bool pre = dlt && col * BS < A.n;
#pragma unroll
                        for (int cc = 0; cc < BS; ++cc)
                            x[h][cc] = pre ? __ldg(dlt + (size_t)col * BS + cc)
                                           : __ldg(s + (size_t)col * BS + cc) - __ldg(sp + (size_t)col * BS + cc);
                    }
            }
            B1S_WAIT()
            if (valid) {
                b1s_own<BS>(vs, rl, pos, ob);
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if (hl + 16 * h < pos) b1s_terms<BS>(vs, rl, hl + 16 * h, x[h], q);
            }
#pragma unroll
            for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
            if (valid) {
                double lo[BS];
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    double acc = q[c];
#pragma unroll
                    for (int cc = 0; cc < c; ++cc) acc += ob[c][cc] * xd[cc];
                    lo[c] = acc;
                }
                if (hl < BS) {
                    const double kpi = (ri + pick_row<BS>(lo, hl)) + bt * kpo;
                    const double pi = si + bt * po;
                    Kp[o] = kpi;
                    p[o] = pi;
                    dacc[0] += pi * kpi;
                }
            }
        })
    }
    cluster_partial<ShB1a>(dacc, part, A.Bp, false);
}

template <int BS>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_B1BLK_MINB)
    k_residual_upper_b1s(Mat A, NodeTab T, const double* __restrict__ u, double* __restrict__ t,
                         const int* active) {
    if (!active[0]) return;
    const int nn = A.n / BS;
    P2G_B1S_NODE_LOOP(2, BS, A, T, 0, nn, {
        const int rl = inf.y, pos = inf.z, nnb = inf.w;
        double ob[BS][BS], uo[BS], q[BS], x[2][BS];
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = 0.0;
        if (valid) {
#pragma unroll
            for (int c = 0; c < BS; ++c) uo[c] = __ldg(u + (size_t)node * BS + c);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = hl + 16 * h;
                if (j > pos && j < nnb) {
#pragma unroll
                    for (int cc = 0; cc < BS; ++cc) x[h][cc] = __ldg(u + (size_t)(h ? nc1 : nc0) * BS + cc);
                }
            }
        }
        B1S_WAIT()
        if (valid) {
            b1s_own<BS>(vs, rl, pos, ob);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int j = hl + 16 * h;
                if (j > pos && j < nnb) b1s_terms<BS>(vs, rl, j, x[h], q);
            }
        }
#pragma unroll
        for (int c = 0; c < BS; ++c) q[c] = half_sum(q[c]);
        if (valid) {
            double tv[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int cc = c + 1; cc < BS; ++cc) acc += ob[c][cc] * uo[cc];
                tv[c] = -(acc + q[c]);
            }
            if (hl < BS) t[(size_t)node * BS + hl] = pick_row<BS>(tv, hl);
        }
    })
}

// Row stride (doubles) of the padded Phi copy the tensor-core tiles read:
// k rounded up to 4 (whole k-steps, zero filled), then to 4 mod 8 so both the
// A-fragment pattern of the restriction (row = lane%4, col = lane/4) and of
// the prolongation (row = lane/4, col = lane%4) hit each bank exactly twice
// (two wavefronts, the minimum for 32 x 8 bytes).
__host__ __device__ constexpr int phi_stride(int k) {
    return ((k + 3) / 4 * 4) % 8 == 0 ? (k + 3) / 4 * 4 + 4 : (k + 3) / 4 * 4;
}

// FP64 tensor-core MMA, D(8x8) += A(8x4) B(4x8); fragments (PTX m8n8k4 .f64):
// a = A[lane/4][lane%4], b = B[lane%4][lane/4], d = D[lane/4][2(lane%4) + {0,1}]
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int TB, int KMAX>
struct MmaTile {
    static constexpr int RT = 32, NS = 4;
    static constexpr int TS = TB + 8;  // data-row stride: 8 mod 16 doubles (B fragments)
    static constexpr int KS = phi_stride(KMAX);
    static constexpr int T_DBL = RT * TS;
    static constexpr int STAGE = T_DBL + RT * KS;  // a multiple of 4 doubles (32 bytes)
    static constexpr size_t SMEM = sizeof(double) * (size_t)NS * STAGE + 64;
};

// warp 0 streams tile `tile` into a stage: the RT Phi rows (one contiguous
// copy, stride ks) and, WITH_T, the RT data rows (one copy per row into the
// padded stride TS)
template <int TB, int KMAX, bool WITH_T>
__device__ __forceinline__ void mma_issue(double* stage, uint64_t* bar, int tile, int n, int Bp,
                                          int bt0, const double* data, const double* phit, int ks,
                                          int lane) {
    using MT = MmaTile<TB, KMAX>;
    const int r0 = tile * MT::RT, nr = min(MT::RT, n - r0);
    const uint32_t pbytes = static_cast<uint32_t>(nr * ks) * 8u;
    const uint32_t tbytes = WITH_T ? static_cast<uint32_t>(nr) * TB * 8u : 0u;
    if (lane == 0) mbar_arrive_tx(bar, pbytes + tbytes);
    __syncwarp();
    if (lane == 0) bulk_g2s(stage + MT::T_DBL, phit + (size_t)r0 * ks, pbytes, bar);
    if constexpr (WITH_T)
        if (lane < nr)
            bulk_g2s(stage + lane * MT::TS, data + (size_t)(r0 + lane) * Bp + bt0, TB * 8u, bar);
}

// Restriction C[k][TB] = Phi^T T on the FP64 tensor cores (pod.hpp:33-37,
// the batched form): per 4-row k-step a warp owns one 8-instance n-block and
// every 8-coefficient m-block.  With TB = 32 two warps share an n-block and
// split the k-steps (summed in fixed order).  Persistent CTAs, NS-stage bulk
// pipeline; per-cluster partial rows as before (deterministic).  Rows past n
// contribute zeros; coefficients past k read padding and are not stored.
template <int TB, int KMAX>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock) k_restrict_mma(int n, int Bp,
                                                                     const double* __restrict__ t,
                                                                     const double* __restrict__ phit,
                                                                     int k, int ks, double* part) {
    using MT = MmaTile<TB, KMAX>;
    constexpr int NB = TB / 8, KSPLIT = kWarps / NB, MBX = (KMAX + 7) / 8;
    extern __shared__ __align__(128) double dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)MT::NS * MT::STAGE);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int nb = warp % NB, kpart = warp / NB;
    const int bt0 = blockIdx.y * TB;
    const int ntiles = (n + MT::RT - 1) / MT::RT;
    const int mb = (k + 7) / 8;
    if (threadIdx.x == 0) {
        for (int q = 0; q < MT::NS; ++q) mbar_init(&full[q], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == 0)
        for (int q = 0; q < MT::NS; ++q) {
            const int tile = blockIdx.x + q * gridDim.x;
            if (tile < ntiles)
                mma_issue<TB, KMAX, true>(dsm + (size_t)q * MT::STAGE, &full[q], tile, n, Bp, bt0, t,
                                          phit, ks, lane);
        }
    double c[MBX][2];
#pragma unroll
    for (int m = 0; m < MBX; ++m) c[m][0] = c[m][1] = 0.0;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % MT::NS;
        const double* Ts = dsm + (size_t)st * MT::STAGE;
        const double* Ps = Ts + MT::T_DBL;
        mbar_wait(&full[st], (it / MT::NS) & 1);
        const int nr = min(MT::RT, n - tile * MT::RT);
#pragma unroll
        for (int q = kpart; q < MT::RT / 4; q += KSPLIT) {
            const int row = 4 * q + tg;
            const bool ok = row < nr;
            const double b = ok ? Ts[row * MT::TS + 8 * nb + g] : 0.0;
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                if (m < mb) {
                    const double a = ok ? Ps[row * ks + 8 * m + g] : 0.0;
                    dmma(c[m][0], c[m][1], a, b);
                }
        }
        __syncthreads();  // stage consumed by every warp
        const int nxt = tile + MT::NS * gridDim.x;
        if (warp == 0 && nxt < ntiles)
            mma_issue<TB, KMAX, true>(dsm + (size_t)st * MT::STAGE, &full[st], nxt, n, Bp, bt0, t, phit,
                                      ks, lane);
    }
    // CTA totals [k][TB] (k-split halves summed in fixed order), then the
    // fixed-order cluster sum into this cluster's partial row
    double* tot = dsm;
    double* tot2 = dsm + KMAX * TB;
    if (KSPLIT == 1 || kpart == 0) {
#pragma unroll
        for (int m = 0; m < MBX; ++m)
            if (8 * m + g < k) {
                tot[(8 * m + g) * TB + 8 * nb + 2 * tg] = c[m][0];
                tot[(8 * m + g) * TB + 8 * nb + 2 * tg + 1] = c[m][1];
            }
    } else {
#pragma unroll
        for (int m = 0; m < MBX; ++m)
            if (8 * m + g < k) {
                tot2[(8 * m + g) * TB + 8 * nb + 2 * tg] = c[m][0];
                tot2[(8 * m + g) * TB + 8 * nb + 2 * tg + 1] = c[m][1];
            }
    }
    if constexpr (KSPLIT > 1) {
        __syncthreads();
        for (int q = threadIdx.x; q < k * TB; q += kBlock) tot[q] = tot[q] + tot2[q];
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    {  // every CTA of the cluster sums its share of the entries (same rank order)
        double* prow = part + (size_t)(blockIdx.x / kCluster) * k * Bp + bt0;
        for (int q = threadIdx.x + (int)cl.block_rank() * kBlock; q < k * TB; q += kBlock * kCluster) {
            double tt = 0.0;
#pragma unroll
            for (int r = 0; r < kCluster; ++r) tt += cl.map_shared_rank(tot, r)[q];
            prow[(size_t)(q / TB) * Bp + q % TB] = tt;
        }
    }
    cl.sync();
}

// Prolongation S[rows][TB] (+)= Phi E on the tensor cores (pod.hpp:40-44 +
// 201-202, batched): a warp owns one 8-instance n-block and MPW 8-row
// m-blocks of each 32-row tile; E's B fragments stay in registers; the
// correction is formed first, then added to S (as the reference's
// u += 1.0 * lift(e)).  Masked stores keep inactive instances untouched.
template <int TB, int KMAX, bool ASSIGN>
__global__ void __launch_bounds__(kBlock) k_prolong_mma(int n, int Bp, double* s,
                                                        const double* __restrict__ phit, int k,
                                                        int ks, const double* __restrict__ e,
                                                        const int* active) {
    using MT = MmaTile<TB, KMAX>;
    constexpr int NB = TB / 8, MPW = (MT::RT / 8) * NB / kWarps, KQ = (KMAX + 3) / 4;
    extern __shared__ __align__(128) double dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)MT::NS * MT::STAGE);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int nb = warp % NB, m0 = warp / NB;  // m-blocks m0, m0 + kWarps/NB, ...
    const int bt0 = blockIdx.y * TB;
    const int ntiles = (n + MT::RT - 1) / MT::RT;
    const int kq = (k + 3) / 4;
    if (threadIdx.x == 0) {
        for (int q = 0; q < MT::NS; ++q) mbar_init(&full[q], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == 0)
        for (int q = 0; q < MT::NS; ++q) {
            const int tile = blockIdx.x + q * gridDim.x;
            if (tile < ntiles)
                mma_issue<TB, KMAX, !ASSIGN>(dsm + (size_t)q * MT::STAGE, &full[q], tile, n, Bp, bt0, s,
                                             phit, ks, lane);
        }
    double be[KQ];
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
        const int a = 4 * q + tg;
        be[q] = a < k ? e[(size_t)a * Bp + bt0 + 8 * nb + g] : 0.0;
    }
    const int col = bt0 + 8 * nb + 2 * tg;
    const bool m0a = active[col] != 0, m1a = active[col + 1] != 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % MT::NS;
        const double* Ss = dsm + (size_t)st * MT::STAGE;
        const double* Ps = Ss + MT::T_DBL;
        mbar_wait(&full[st], (it / MT::NS) & 1);
        const int r0 = tile * MT::RT, nr = min(MT::RT, n - r0);
#pragma unroll
        for (int j = 0; j < MPW; ++j) {
            const int mrow = 8 * (m0 + j * (kWarps / NB));
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int q = 0; q < KQ; ++q)
                if (q < kq) dmma(c0, c1, Ps[(mrow + g) * ks + 4 * q + tg], be[q]);
            const int row = mrow + g;
            if (row < nr) {
                double* dst = s + (size_t)(r0 + row) * Bp + col;
                double o0 = c0, o1 = c1;
                if constexpr (!ASSIGN) {
                    o0 = __dadd_rn(Ss[row * MT::TS + 8 * nb + 2 * tg], c0);
                    o1 = __dadd_rn(Ss[row * MT::TS + 8 * nb + 2 * tg + 1], c1);
                }
                if (m0a && m1a)
                    *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
                else {
                    if (m0a) dst[0] = o0;
                    if (m1a) dst[1] = o1;
                }
            }
        }
        __syncthreads();
        const int nxt = tile + MT::NS * gridDim.x;
        if (warp == 0 && nxt < ntiles)
            mma_issue<TB, KMAX, !ASSIGN>(dsm + (size_t)st * MT::STAGE, &full[st], nxt, n, Bp, bt0, s,
                                         phit, ks, lane);
    }
}

// Register-fed tensor-core forms (no shared-memory staging): every fragment
// is loaded straight from global memory -- a B fragment of the restriction
// is 4 rows x 8 consecutive instances (4 x 64 B), a Phi fragment 4 or 8 rows
// of the padded copy (L1 hits across the CTA's warps) -- with U k-steps (or
// m-blocks) of loads issued ahead of their MMAs.
#ifndef P2G_RESTRICT_U
#define P2G_RESTRICT_U 4  // k-steps of T / Phi loads in flight per warp (KMAX <= 24)
#endif
#ifndef P2G_RESTRICT_MINB
#define P2G_RESTRICT_MINB 4
#endif
template <int TB, int KMAX>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, KMAX > 40 ? 2 : P2G_RESTRICT_MINB) k_restrict_reg(int n, int Bp,
                                                                        const double* __restrict__ t,
                                                                        const double* __restrict__ phit,
                                                                        int k, int ks, double* part) {
    constexpr int NB = TB / 8, KSPLIT = kWarps / NB, MBX = (KMAX + 7) / 8;
    constexpr int U = KMAX <= 24 ? P2G_RESTRICT_U : (KMAX <= 40 ? 2 : 1);  // k-steps of loads ahead
    __shared__ double tot[KSPLIT][KMAX * TB];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int nb = warp % NB, kpart = warp / NB;
    const int bt0 = blockIdx.y * TB;
    const int mb = (k + 7) / 8;
    const int nq = (n + 3) / 4;  // 4-row k-steps
    const int wk = blockIdx.x * KSPLIT + kpart, nwk = gridDim.x * KSPLIT;  // workers
    const double* tcol = t + bt0 + 8 * nb + g;
    double c[MBX][2];
#pragma unroll
    for (int m = 0; m < MBX; ++m) c[m][0] = c[m][1] = 0.0;
    for (int q0 = wk; q0 < nq; q0 += U * nwk) {
        double b[U], a[U][MBX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int row = 4 * (q0 + u * nwk) + tg;
            const bool ok = row < n;
            b[u] = ok ? __ldg(tcol + (size_t)row * Bp) : 0.0;
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                a[u][m] = (ok && m < mb) ? __ldg(phit + (size_t)row * ks + 8 * m + g) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                if (m < mb) dmma(c[m][0], c[m][1], a[u][m], b[u]);
    }
#pragma unroll
    for (int m = 0; m < MBX; ++m)
        if (8 * m + g < k) {
            tot[kpart][(8 * m + g) * TB + 8 * nb + 2 * tg] = c[m][0];
            tot[kpart][(8 * m + g) * TB + 8 * nb + 2 * tg + 1] = c[m][1];
        }
    if constexpr (KSPLIT > 1) {
        __syncthreads();
        for (int q = threadIdx.x; q < k * TB; q += kBlock) {
            double x = tot[0][q];
#pragma unroll
            for (int r = 1; r < KSPLIT; ++r) x = x + tot[r][q];
            tot[0][q] = x;
        }
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    {  // every CTA of the cluster sums its share of the entries (same rank order)
        double* prow = part + (size_t)(blockIdx.x / kCluster) * k * Bp + bt0;
        for (int q = threadIdx.x + (int)cl.block_rank() * kBlock; q < k * TB; q += kBlock * kCluster) {
            double tt = 0.0;
#pragma unroll
            for (int r = 0; r < kCluster; ++r) tt += cl.map_shared_rank(&tot[0][0], r)[q];
            prow[(size_t)(q / TB) * Bp + q % TB] = tt;
        }
    }
    cl.sync();
}

// Restriction, wide form: a warp owns a PAIR of 8-instance n-blocks (16
// instances, one 16-byte load per lane per k-step: .x feeds the "even" DMMA
// stream, .y the "odd" one, so both B fragments come from one load) and every
// m-block, with U k-steps of loads in flight -- fewer, fatter loop iterations
// than k_restrict_reg (whose per-iteration latency, not bandwidth, set its
// time: c4 343 k-steps per worker in 172 serial rounds).  Warps of a CTA
// split the k-steps KSPLIT ways; the k-split partials are summed in smem in
// fixed order, then the clusters' partial rows as before (deterministic).
#ifndef P2G_RESTRICT2_MINB
#define P2G_RESTRICT2_MINB 2
#endif
template <int KMAX>
struct Restrict2Cfg {
    static constexpr int MBX = (KMAX + 7) / 8;
    static constexpr int U = KMAX <= 24 ? 8 : (KMAX <= 32 ? 6 : (KMAX <= 40 ? 4 : 2));
};
template <int TB, int KMAX>
__global__ void P2G_CLUSTER __launch_bounds__(kBlock, P2G_RESTRICT2_MINB)
    k_restrict_reg2(int n, int Bp, const double* __restrict__ t, const double* __restrict__ phit,
                    int k, int ks, double* part) {
    constexpr int NP = TB / 16, KSPLIT = kWarps / NP;
    constexpr int MBX = Restrict2Cfg<KMAX>::MBX, U = Restrict2Cfg<KMAX>::U;
    static_assert(TB % 16 == 0 && kWarps % NP == 0, "n-block pairs per CTA");
    extern __shared__ __align__(16) double tot2[];  // [KMAX][TB]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int np = warp % NP, kpart = warp / NP;
    const int bt0 = blockIdx.y * TB;
    const int mb = (k + 7) / 8;
    const int nq = (n + 3) / 4;
    const int wk = blockIdx.x * KSPLIT + kpart, nwk = gridDim.x * KSPLIT;
    const double* tcol = t + bt0 + 16 * np + 2 * g;
    double ce[MBX][2], co[MBX][2];
#pragma unroll
    for (int m = 0; m < MBX; ++m) ce[m][0] = ce[m][1] = co[m][0] = co[m][1] = 0.0;
    for (int q0 = wk; q0 < nq; q0 += U * nwk) {
        double2 b[U];
        double a[U][MBX];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int row = 4 * (q0 + u * nwk) + tg;
            const bool ok = row < n;
            b[u] = ok ? __ldg(reinterpret_cast<const double2*>(tcol + (size_t)row * Bp))
                      : make_double2(0.0, 0.0);
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                a[u][m] = (ok && m < mb) ? __ldg(phit + (size_t)row * ks + 8 * m + g) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                if (m < mb) {
                    dmma(ce[m][0], ce[m][1], a[u][m], b[u].x);
                    dmma(co[m][0], co[m][1], a[u][m], b[u].y);
                }
    }
    // lane holds C[8m + g][instances 16 np + 4 tg + {0 (even .0), 1 (odd .0), 2 (even .1), 3 (odd .1)}]
    for (int kp = KSPLIT - 1; kp >= 0; --kp) {  // fixed-order k-split sum
        if (kpart == kp) {
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                if (8 * m + g < k) {
                    double* d = tot2 + (size_t)(8 * m + g) * TB + 16 * np + 4 * tg;
                    const double v0 = ce[m][0], v1 = co[m][0], v2 = ce[m][1], v3 = co[m][1];
                    if (kp == KSPLIT - 1) {
                        d[0] = v0; d[1] = v1; d[2] = v2; d[3] = v3;
                    } else {
                        d[0] = d[0] + v0; d[1] = d[1] + v1; d[2] = d[2] + v2; d[3] = d[3] + v3;
                    }
                }
        }
        __syncthreads();
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    {  // every CTA of the cluster sums its share of the entries (same rank order)
        double* prow = part + (size_t)(blockIdx.x / kCluster) * k * Bp + bt0;
        for (int q = threadIdx.x + (int)cl.block_rank() * kBlock; q < k * TB; q += kBlock * kCluster) {
            double tt = 0.0;
#pragma unroll
            for (int r = 0; r < kCluster; ++r) tt += cl.map_shared_rank(tot2, r)[q];
            prow[(size_t)(q / TB) * Bp + q % TB] = tt;
        }
    }
    cl.sync();
}

// ---------------------------------------------------------------------------
// Warp-specialised bulk-copy restriction for large systems (c3 / c4 shapes).
// The register-fed kernels keep every warp on the chain global load -> DMMA
// and re-read each Phi row once per 16 instances; the first staged form
// (k_restrict_mma) released its stages with a CTA barrier, which stalled the
// DMMA warps behind the slowest one.  Here:
//  * one PRODUCER warp (warp kWarps) streams RT-row tiles of T (one bulk copy
//    per row into a padded row stride: conflict-free 16-byte fragment reads)
//    and of the padded Phi (one copy) into an NS-stage ring; a stage is handed
//    over by a FULL mbarrier (expect_tx) and handed back by an EMPTY mbarrier
//    on which each consumer warp arrives once -- no CTA-wide barrier in the loop;
//  * 8 CONSUMER warps; a warp owns 32 instances (four 8-instance n-blocks fed
//    by two 16-byte shared loads: .x / .y are the even / odd instances) and
//    every m-block, so a Phi fragment is used four times and the CTA tile
//    spans TBW = 64 / 128 / 256 instances (at TBW = Bp, Phi is read from DRAM
//    once).  Warps split a stage's k-steps KSPLIT = 8 / (TBW / 32) ways.
//  * epilogue as k_restrict_reg2: fixed-order k-split sum in shared memory,
//    fixed-order cluster sum into the cluster's partial row (deterministic).
//  * clusters of kWsCluster = 2 CTAs (an SM pair), not kCluster = 8: with one
//    CTA per SM only 15 clusters of 8 fit the 148 SMs (120 CTAs: ncu
//    launch__cluster_max_active), and this kernel is FP64-tensor-pipe bound
//    (93 % DMMA pipe active), so idle SMs cost time one for one.
constexpr int kWsBlock = kBlock + 32;
constexpr int kWsCluster = 2;
template <int TBW, int KMAX>
struct WsTile {
    static constexpr int NG = TBW / 32, KSPLIT = kWarps / NG;
    static constexpr int QW = 4;                // k-steps per consumer warp and stage
    static constexpr int RT = 4 * QW * KSPLIT;  // rows per stage
    // A stage holds its rows as four QUARTERS of QR consecutive rows; the four
    // rows of a k-step are row q of each quarter (lane%4 picks the quarter).
    // Each quarter is padded by 32 bytes, so the four lanes of a fragment
    // column read different bank groups (data: 16-byte loads; Phi: 8-byte
    // loads, each bank hit twice), and a quarter is ONE bulk copy whenever its
    // rows are contiguous in global memory (Phi always; the data when TBW = Bp).
    static constexpr int QR = RT / 4;
    static constexpr int KS = phi_stride(KMAX);
    static constexpr int QT = QR * TBW + 4;  // data quarter stride (doubles)
    static constexpr int QP = QR * KS + 4;   // Phi quarter stride
    static constexpr int T_DBL = 4 * QT;
    static constexpr int STAGE = T_DBL + 4 * QP;  // doubles (a multiple of 4: 32-byte aligned)
    static constexpr int NSMAX = (227 * 1024 - 256) / (STAGE * 8);
    static constexpr int NS = NSMAX < 4 ? NSMAX : 4;
    static constexpr size_t SMEM = sizeof(double) * (size_t)NS * STAGE + 128;
    static_assert(TBW % 32 == 0 && kWarps % NG == 0 && NS >= 2, "tile geometry");
    static_assert((size_t)KMAX * TBW <= (size_t)NS * STAGE, "epilogue buffer fits the ring");
};
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int TBW, int KMAX, bool MASK>
__device__ __forceinline__ void ws_stage_mma(const double* Ts, const double* Ps, int ks, int mb,
                                             int nr, int ig, int kp, int g, int tg,
                                             double (&acc)[(KMAX + 7) / 8][4][2]) {
    using WT = WsTile<TBW, KMAX>;
    constexpr int MBX = (KMAX + 7) / 8;
#pragma unroll
    for (int j = 0; j < WT::QW; ++j) {
        const int q = kp * WT::QW + j;  // row q of quarter tg
        const bool ok = !MASK || tg * WT::QR + q < nr;
        const double* tr = Ts + tg * WT::QT + q * TBW + 32 * ig + 2 * g;
        double2 b0 = *reinterpret_cast<const double2*>(tr);
        double2 b1 = *reinterpret_cast<const double2*>(tr + 16);
        if (MASK && !ok) b0 = b1 = make_double2(0.0, 0.0);
#pragma unroll
        for (int m = 0; m < MBX; ++m)
            if (m < mb) {
                double a = Ps[tg * WT::QP + q * ks + 8 * m + g];
                if (MASK && !ok) a = 0.0;
                dmma(acc[m][0][0], acc[m][0][1], a, b0.x);
                dmma(acc[m][1][0], acc[m][1][1], a, b0.y);
                dmma(acc[m][2][0], acc[m][2][1], a, b1.x);
                dmma(acc[m][3][0], acc[m][3][1], a, b1.y);
            }
    }
}

template <int TBW, int KMAX>
__global__ void __cluster_dims__(kWsCluster, 1, 1) __launch_bounds__(kWsBlock, 1)
    k_restrict_ws(int n, int Bp, const double* __restrict__ t, const double* __restrict__ phit,
                  int k, int ks, double* part) {
    using WT = WsTile<TBW, KMAX>;
    constexpr int MBX = (KMAX + 7) / 8;
    extern __shared__ __align__(128) double dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)WT::NS * WT::STAGE);
    uint64_t* empty = full + WT::NS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int bt0 = blockIdx.y * TBW;
    const int ntiles = (n + WT::RT - 1) / WT::RT;
    const int mb = (k + 7) / 8;
    if (threadIdx.x == 0) {
        for (int q = 0; q < WT::NS; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int ig = warp % WT::NG, kp = warp / WT::NG;
    double acc[MBX][4][2];
#pragma unroll
    for (int m = 0; m < MBX; ++m)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
    if (warp == kWarps) {  // producer
        const uint64_t pol = l2_evict_first_policy();
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int st = it % WT::NS;
            if (it >= WT::NS) mbar_wait(&empty[st], ((it / WT::NS) - 1) & 1);
            double* stage = dsm + (size_t)st * WT::STAGE;
            const int r0 = tile * WT::RT, nr = min(WT::RT, n - r0);
            if (lane == 0)
                mbar_arrive_tx(&full[st], static_cast<uint32_t>(nr) * (ks + TBW) * 8u);
            __syncwarp();
            if (lane < 4) {  // Phi: one copy per quarter
                const int q0 = lane * WT::QR, qn = min(WT::QR, nr - q0);
                if (qn > 0)
                    bulk_g2s(stage + WT::T_DBL + lane * WT::QP, phit + (size_t)(r0 + q0) * ks,
                             static_cast<uint32_t>(qn * ks) * 8u, &full[st]);
            }
            if (Bp == TBW) {  // contiguous rows: one copy per quarter
                if (lane >= 4 && lane < 8) {
                    const int c = lane - 4, q0 = c * WT::QR, qn = min(WT::QR, nr - q0);
                    if (qn > 0)
                        bulk_g2s_hint(stage + c * WT::QT, t + (size_t)(r0 + q0) * Bp,
                                      static_cast<uint32_t>(qn) * TBW * 8u, &full[st], pol);
                }
            } else {
                for (int r = lane; r < nr; r += 32)
                    bulk_g2s_hint(stage + (r / WT::QR) * WT::QT + (r % WT::QR) * TBW,
                                  t + (size_t)(r0 + r) * Bp + bt0, TBW * 8u, &full[st], pol);
            }
        }
    } else {  // consumers
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int st = it % WT::NS;
            const double* Ts = dsm + (size_t)st * WT::STAGE;
            const double* Ps = Ts + WT::T_DBL;
            mbar_wait(&full[st], (it / WT::NS) & 1);
            const int nr = min(WT::RT, n - tile * WT::RT);
            if (nr == WT::RT)
                ws_stage_mma<TBW, KMAX, false>(Ts, Ps, ks, mb, nr, ig, kp, g, tg, acc);
            else
                ws_stage_mma<TBW, KMAX, true>(Ts, Ps, ks, mb, nr, ig, kp, g, tg, acc);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        }
    }
    __syncthreads();  // every issued stage has been consumed: the ring is free
    // lane holds C[8m + g][32 ig + 16 h + 4 tg + {0 (even .0), 1 (odd .0), 2 (even .1), 3 (odd .1)}]
    double* tot = dsm;  // [k][TBW]
    for (int kq = WT::KSPLIT - 1; kq >= 0; --kq) {  // fixed-order k-split sum
        if (warp < kWarps && kp == kq) {
#pragma unroll
            for (int m = 0; m < MBX; ++m)
                if (8 * m + g < k) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        double* d = tot + (size_t)(8 * m + g) * TBW + 32 * ig + 16 * hh + 4 * tg;
                        const double v0 = acc[m][2 * hh][0], v1 = acc[m][2 * hh + 1][0];
                        const double v2 = acc[m][2 * hh][1], v3 = acc[m][2 * hh + 1][1];
                        if (kq == WT::KSPLIT - 1) {
                            d[0] = v0; d[1] = v1; d[2] = v2; d[3] = v3;
                        } else {
                            d[0] = d[0] + v0; d[1] = d[1] + v1; d[2] = d[2] + v2; d[3] = d[3] + v3;
                        }
                    }
                }
        }
        __syncthreads();
    }
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    {  // every CTA of the cluster sums its share of the entries (same rank order)
        double* prow = part + (size_t)(blockIdx.x / kWsCluster) * k * Bp + bt0;
        for (int q = threadIdx.x + (int)cl.block_rank() * kWsBlock; q < k * TBW; q += kWsBlock * kWsCluster) {
            double tt = 0.0;
#pragma unroll
            for (int r = 0; r < kWsCluster; ++r) tt += cl.map_shared_rank(tot, r)[q];
            prow[(size_t)(q / TBW) * Bp + q % TBW] = tt;
        }
    }
    cl.sync();
}

// Warp-specialised bulk-copy prolongation S (+)= Phi E, the same ring as
// k_restrict_ws: the producer warp streams RT-row tiles of Phi (and, unless
// ASSIGN, of S); a consumer warp owns 32 instances (four 8-instance n-blocks,
// E's B fragments in registers) and MPW 8-row m-blocks of each stage, forms
// the correction, adds it to S (u += 1.0 * lift(e), pod.hpp:201-202) and
// stores straight to global memory (masked for inactive instances).  With
// TBW = Bp a Phi row is read once for the whole batch.
// A stage holds its rows as EIGHTHS of ER consecutive rows; m-block i is row
// i of each eighth (lane/4 picks the eighth), so an eighth is ONE bulk copy
// when its rows are contiguous (Phi always; S when TBW = Bp: 16 copies per
// stage, not one per row -- 512-byte copies are bound by the per-SM TMA
// operation rate).  Eighth strides: S 64 bytes mod 128 (conflict-free 16-byte
// C-fragment reads), Phi 4 doubles mod 16 (each bank hit twice by the 8-byte
// A-fragment reads, the minimum).
template <int TBW, int KMAX>
struct WsPTile {
    static constexpr int NG = TBW / 32, MSPLIT = kWarps / NG;
    static constexpr int MPW = 2;                // m-blocks per consumer warp and stage
    static constexpr int ER = MPW * MSPLIT;      // rows per eighth
    static constexpr int RT = 8 * ER;            // rows per stage
    static constexpr int KS = phi_stride(KMAX);
    static constexpr int ES = ER * TBW + 8;      // S eighth stride (doubles)
    static constexpr int EP = ER * KS + ((4 - ER * KS % 16) + 16) % 16;  // Phi eighth stride
    static constexpr int T_DBL = 8 * ES;
    static constexpr int STAGE = T_DBL + 8 * EP;
    static constexpr int NSMAX = (227 * 1024 - 256) / (STAGE * 8);
    static constexpr int NS = NSMAX < 4 ? NSMAX : 4;
    static constexpr size_t SMEM = sizeof(double) * (size_t)NS * STAGE + 128;
    static_assert(TBW % 32 == 0 && kWarps % NG == 0 && NS >= 2 && EP % 2 == 0, "tile geometry");
};

template <int TBW, int KMAX, bool ASSIGN>
__global__ void __launch_bounds__(kWsBlock, 1)
    k_prolong_ws(int n, int Bp, double* s, const double* __restrict__ phit, int k, int ks,
                 const double* __restrict__ e, const int* active) {
    using WT = WsPTile<TBW, KMAX>;
    constexpr int KQ = (KMAX + 3) / 4;
    extern __shared__ __align__(128) double dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm + (size_t)WT::NS * WT::STAGE);
    uint64_t* empty = full + WT::NS;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int bt0 = blockIdx.y * TBW;
    const int ntiles = (n + WT::RT - 1) / WT::RT;
    const int kq = (k + 3) / 4;
    if (threadIdx.x == 0) {
        for (int q = 0; q < WT::NS; ++q) {
            mbar_init(&full[q], 1);
            mbar_init(&empty[q], kWarps);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == kWarps) {  // producer
        int it = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int st = it % WT::NS;
            if (it >= WT::NS) mbar_wait(&empty[st], ((it / WT::NS) - 1) & 1);
            double* stage = dsm + (size_t)st * WT::STAGE;
            const int r0 = tile * WT::RT, nr = min(WT::RT, n - r0);
            if (lane == 0)
                mbar_arrive_tx(&full[st], static_cast<uint32_t>(nr) * (ks + (ASSIGN ? 0 : TBW)) * 8u);
            __syncwarp();
            if (lane < 8) {  // Phi: one copy per eighth
                const int q0 = lane * WT::ER, qn = min(WT::ER, nr - q0);
                if (qn > 0)
                    bulk_g2s(stage + WT::T_DBL + lane * WT::EP, phit + (size_t)(r0 + q0) * ks,
                             static_cast<uint32_t>(qn * ks) * 8u, &full[st]);
            }
            if constexpr (!ASSIGN) {
                if (Bp == TBW) {  // contiguous rows: one copy per eighth
                    if (lane >= 8 && lane < 16) {
                        const int c = lane - 8, q0 = c * WT::ER, qn = min(WT::ER, nr - q0);
                        if (qn > 0)
                            bulk_g2s(stage + c * WT::ES, s + (size_t)(r0 + q0) * Bp,
                                     static_cast<uint32_t>(qn) * TBW * 8u, &full[st]);
                    }
                } else {
                    for (int r = lane; r < nr; r += 32)
                        bulk_g2s(stage + (r / WT::ER) * WT::ES + (r % WT::ER) * TBW,
                                 s + (size_t)(r0 + r) * Bp + bt0, TBW * 8u, &full[st]);
                }
            }
        }
        return;
    }
    const int ig = warp % WT::NG, mp = warp / WT::NG;
    double be[KQ][4];
    bool act0[4], act1[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int q = 0; q < KQ; ++q) {
            const int a = 4 * q + tg;
            be[q][j] = a < k ? e[(size_t)a * Bp + bt0 + 32 * ig + 8 * j + g] : 0.0;
        }
        const int col = bt0 + 32 * ig + 8 * j + 2 * tg;
        act0[j] = active[col] != 0;
        act1[j] = active[col + 1] != 0;
    }
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % WT::NS;
        const double* Ss = dsm + (size_t)st * WT::STAGE;
        const double* Ps = Ss + WT::T_DBL;
        mbar_wait(&full[st], (it / WT::NS) & 1);
        const int r0 = tile * WT::RT, nr = min(WT::RT, n - r0);
#pragma unroll
        for (int u = 0; u < WT::MPW; ++u) {
            const int i = mp * WT::MPW + u;    // row i of eighth g
            const int row = g * WT::ER + i;    // row within the tile
            double c[4][2];
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j][0] = c[j][1] = 0.0;
#pragma unroll
            for (int q = 0; q < KQ; ++q)
                if (q < kq) {
                    const double a = Ps[g * WT::EP + i * ks + 4 * q + tg];
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma(c[j][0], c[j][1], a, be[q][j]);
                }
            if (row < nr) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int cl = 32 * ig + 8 * j + 2 * tg;
                    double o0 = c[j][0], o1 = c[j][1];
                    if constexpr (!ASSIGN) {
                        const double2 sv =
                            *reinterpret_cast<const double2*>(Ss + g * WT::ES + i * TBW + cl);
                        o0 = __dadd_rn(sv.x, o0);
                        o1 = __dadd_rn(sv.y, o1);
                    }
                    double* dst = s + (size_t)(r0 + row) * Bp + bt0 + cl;
                    if (act0[j] && act1[j])
                        *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
                    else {
                        if (act0[j]) dst[0] = o0;
                        if (act1[j]) dst[1] = o1;
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
}

// the CTA's warps share 8-row m-blocks (NB n-blocks each; with TB = 32 two
// m-blocks per step); U steps of S / Phi loads issued before their MMAs
#ifndef P2G_PROLONG_U_WIDE
#define P2G_PROLONG_U_WIDE 2  // m-blocks in flight for 24 < KMAX <= 40 (c4: 201 vs 241 us at 1)
#endif
#ifndef P2G_PROLONG_MINB_WIDE
#define P2G_PROLONG_MINB_WIDE 3
#endif
#ifndef P2G_PROLONG_U_NARROW
#define P2G_PROLONG_U_NARROW 2  // m-blocks in flight for KMAX <= 24
#endif
#ifndef P2G_PROLONG_MINB_NARROW
#define P2G_PROLONG_MINB_NARROW 4
#endif
template <int TB, int KMAX, bool ASSIGN>
__global__ void __launch_bounds__(kBlock, KMAX > 40 ? 2 : (KMAX > 24 ? P2G_PROLONG_MINB_WIDE : P2G_PROLONG_MINB_NARROW))
    k_prolong_reg(int n, int Bp, double* s, const double* __restrict__ phit, int k, int ks,
                  const double* __restrict__ e, const int* active) {
    constexpr int NB = TB / 8, MSPLIT = kWarps / NB, KQ = (KMAX + 3) / 4;
    constexpr int U = KMAX <= 24 ? P2G_PROLONG_U_NARROW : (KMAX <= 40 ? P2G_PROLONG_U_WIDE : 1);  // m-blocks of loads ahead
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int nb = warp % NB, mpart = warp / NB;
    const int bt0 = blockIdx.y * TB;
    const int kq = (k + 3) / 4;
    double be[KQ];
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
        const int a = 4 * q + tg;
        be[q] = a < k ? e[(size_t)a * Bp + bt0 + 8 * nb + g] : 0.0;
    }
    const int col = bt0 + 8 * nb + 2 * tg;
    const bool m0a = active[col] != 0, m1a = active[col + 1] != 0;
    // the whole warp leaves together (mma.sync needs every lane)
    if (!__any_sync(0xffffffffu, m0a || m1a)) return;
    const int nmb = (n + 7) / 8;
    const int wk = blockIdx.x * MSPLIT + mpart, nwk = gridDim.x * MSPLIT;
    for (int mb0 = wk; mb0 < nmb; mb0 += U * nwk) {
        double a[U][KQ], sv[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int row = 8 * (mb0 + u * nwk) + g;
            const bool ok = row < n;
#pragma unroll
            for (int q = 0; q < KQ; ++q)
                a[u][q] = (ok && q < kq) ? __ldg(phit + (size_t)row * ks + 4 * q + tg) : 0.0;
            sv[u][0] = sv[u][1] = 0.0;
            if (!ASSIGN && ok) {
                const double2 x = *reinterpret_cast<const double2*>(s + (size_t)row * Bp + col);
                sv[u][0] = x.x;
                sv[u][1] = x.y;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double c0 = 0.0, c1 = 0.0;
#pragma unroll
            for (int q = 0; q < KQ; ++q)
                if (q < kq) dmma(c0, c1, a[u][q], be[q]);
            const int row = 8 * (mb0 + u * nwk) + g;
            if (row < n) {
                double* dst = s + (size_t)row * Bp + col;
                const double o0 = ASSIGN ? c0 : __dadd_rn(sv[u][0], c0);
                const double o1 = ASSIGN ? c1 : __dadd_rn(sv[u][1], c1);
                if (m0a && m1a)
                    *reinterpret_cast<double2*>(dst) = make_double2(o0, o1);
                else {
                    if (m0a) dst[0] = o0;
                    if (m1a) dst[1] = o1;
                }
            }
        }
    }
}

// Surrogate latent coordinates (surrogate.hpp:354-357 without the lift):
// e[:, b] = denormalize(mlp(normalize(theta_b))), one CTA per instance.
// Mlp::forward (surrogate.hpp:62-74): z = bias, z_i += W_ij a_j in ascending
// j (separately rounded), activation on hidden layers only; AffineNormalizer
// (surrogate.hpp:150-157).  norm = [in_mean p | in_std p | lat_mean k | lat_std k].
__global__ void __launch_bounds__(kBlock) k_mlp_latent(int nlayers, const int* widths, int act,
                                                       const double* __restrict__ W,
                                                       const double* __restrict__ bias,
                                                       const double* __restrict__ norm,
                                                       const double* __restrict__ theta,
                                                       int wmax, int Bp, double* e) {
    extern __shared__ double mlp_sm[];
    double* a = mlp_sm;
    double* z = mlp_sm + wmax;
    const int b = blockIdx.x;
    const int p = widths[0], k = widths[nlayers];
    for (int j = threadIdx.x; j < p; j += blockDim.x)
        a[j] = __ddiv_rn(__dsub_rn(theta[(size_t)b * p + j], norm[j]), norm[p + j]);
    __syncthreads();
    size_t wo = 0, bo = 0;
    for (int l = 0; l < nlayers; ++l) {
        const int fi = widths[l], fo = widths[l + 1];
        for (int i = threadIdx.x; i < fo; i += blockDim.x) {
            const double* Wi = W + wo + (size_t)i * fi;
            double s = bias[bo + i];
            for (int j = 0; j < fi; ++j) s = __dadd_rn(s, __dmul_rn(Wi[j], a[j]));
            if (l + 1 < nlayers) s = act == 0 ? tanh(s) : fmax(s, 0.0);
            z[i] = s;
        }
        __syncthreads();
        double* t = a;
        a = z;
        z = t;
        wo += (size_t)fo * fi;
        bo += fo;
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x)
        e[(size_t)i * Bp + b] = __dadd_rn(__dmul_rn(a[i], norm[2 * p + k + i]), norm[2 * p + i]);
}

// ---------------------------------------------------------------------------
// compute_pod's contractions (pod.hpp:81-87 Gram, :120-129 Phi = U Psi
// Lambda^{-1/2}) on the FP64 tensor cores.
// Gram G = U U^T, U [N][d] row-major: CTA (x = column chunk, y = macro tile
// (I, J) of 64 x 64 entries, I <= J) stages its two 64-row panels of 32
// columns in shared memory (row stride 36: the fragment pattern row = lane/4,
// col = lane%4 hits each bank twice); warp w accumulates row block w of I
// against the 8 column blocks of J.  Partials [chunk][tile][64][64], reduced
// in fixed order by k_gram_reduce.
constexpr int kGramMT = 64, kGramCW = 32, kGramS = kGramCW + 4;

__global__ void __launch_bounds__(kBlock) k_gram(int N, int64_t d, const double* __restrict__ U,
                                                 const int* __restrict__ tiles, double* part) {
    __shared__ double P[2][kGramMT * kGramS];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int I = tiles[2 * blockIdx.y], J = tiles[2 * blockIdx.y + 1];
    double c[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
    for (int64_t c0 = (int64_t)blockIdx.x * kGramCW; c0 < d; c0 += (int64_t)gridDim.x * kGramCW) {
        for (int q = threadIdx.x; q < 2 * kGramMT * kGramCW; q += kBlock) {
            const int pnl = q / (kGramMT * kGramCW), rem = q % (kGramMT * kGramCW);
            const int row = rem / kGramCW, col = rem % kGramCW;
            const int a = (pnl ? J : I) * kGramMT + row;
            const int64_t cc = c0 + col;
            P[pnl][row * kGramS + col] = (a < N && cc < d) ? __ldg(U + (size_t)a * d + cc) : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < kGramCW / 4; ++ks) {
            const double af = P[0][(8 * warp + g) * kGramS + 4 * ks + tg];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                dmma(c[j][0], c[j][1], af, P[1][(8 * j + g) * kGramS + 4 * ks + tg]);
        }
        __syncthreads();
    }
    double* out = part + ((size_t)blockIdx.x * gridDim.y + blockIdx.y) * kGramMT * kGramMT;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        out[(8 * warp + g) * kGramMT + 8 * j + 2 * tg] = c[j][0];
        out[(8 * warp + g) * kGramMT + 8 * j + 2 * tg + 1] = c[j][1];
    }
}

// G[a][b] (a, b < N) = fixed-order sum over the chunk partials; symmetric fill
__global__ void k_gram_reduce(int N, int nchunks, int ntiles, const int* __restrict__ tiles,
                              const double* __restrict__ part, double* G) {
    const int t = blockIdx.y, I = tiles[2 * t], J = tiles[2 * t + 1];
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < kGramMT * kGramMT;
         q += gridDim.x * blockDim.x) {
        const int a = I * kGramMT + q / kGramMT, b = J * kGramMT + q % kGramMT;
        if (a >= N || b >= N || (I == J && a > b)) continue;
        double s = 0.0;
        for (int ch = 0; ch < nchunks; ++ch) s += part[((size_t)ch * ntiles + t) * kGramMT * kGramMT + q];
        G[(size_t)a * N + b] = s;
        G[(size_t)b * N + a] = s;
    }
}

// Phi[d][r] = U^T W (U [N][d], W [N][r], r <= 64): warp = 8 consecutive rows
// of Phi x all column blocks; A fragment U[a0 + lane%4][i0 + lane/4] (each U
// element read once), B fragments W from L1; k-steps over the N snapshots.
__global__ void __launch_bounds__(kBlock) k_combine(int N, int64_t d, const double* __restrict__ U,
                                                    int r, const double* __restrict__ W,
                                                    double* __restrict__ Phi) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tg = lane & 3;
    const int nb = (r + 7) / 8;
    for (int64_t i0 = ((int64_t)blockIdx.x * kWarps + warp) * 8; i0 < d;
         i0 += (int64_t)gridDim.x * kWarps * 8) {
        double c[8][2];
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j][0] = c[j][1] = 0.0;
        const int64_t i = i0 + g;
        for (int a0 = 0; a0 < N; a0 += 4) {
            const int a = a0 + tg;
            const double af = (a < N && i < d) ? __ldg(U + (size_t)a * d + i) : 0.0;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < nb) {
                    const int col = 8 * j + g;
                    const double bf = (a < N && col < r) ? __ldg(W + (size_t)a * r + col) : 0.0;
                    dmma(c[j][0], c[j][1], af, bf);
                }
        }
        if (i < d) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (j < nb) {
                    const int col = 8 * j + 2 * tg;
                    if (col < r) Phi[(size_t)i * r + col] = c[j][0];
                    if (col + 1 < r) Phi[(size_t)i * r + col + 1] = c[j][1];
                }
        }
    }
}

// shape of the row-local kernels (restriction, prolongation): R = 32/W rows
// per warp, one instance per lane unless k is small enough for two
template <class Sh, int KMAX>
struct LocalShape {
    static constexpr int V = 1;
    using type = Shape<32 / Sh::W, 1, Sh::W, V>;
};

// p = s + beta p (krylov.hpp:282); INIT: p = s (krylov.hpp:263)
template <class Sh, bool INIT>
__global__ void P2G_ROWK k_pupdate(int n, int Bp, const double* __restrict__ s,
                                                    double* __restrict__ p, const double* beta,
                                                    const int* active) {
    const int lane = threadIdx.x & 31, w = lane % Sh::W;
    const int sl = lane / Sh::W;  // remaining lanes stride over rows
    constexpr int RL = 32 / Sh::W;
    const int b0 = blockIdx.y * Sh::T + w * Sh::V;
    bool m[Sh::V], any;
    lane_mask<Sh>(active, b0, m, any);
    if (!any) return;
    double bt[Sh::V];
#pragma unroll
    for (int v = 0; v < Sh::V; ++v) bt[v] = INIT ? 0.0 : beta[b0 + v];
    for (int i = (blockIdx.x * kWarps + (threadIdx.x >> 5)) * RL + sl; i < n;
         i += gridDim.x * kWarps * RL) {
        const size_t o = (size_t)i * Bp + b0;
        double si[Sh::V], pi[Sh::V];
        ldv<Sh::V>(si, s + o);
        if constexpr (!INIT) {
            ldv<Sh::V>(pi, p + o);
#pragma unroll
            for (int v = 0; v < Sh::V; ++v) si[v] = __dadd_rn(si[v], __dmul_rn(bt[v], pi[v]));
        }
        stv<Sh::V>(p + o, si, m);
    }
}

// warp-level fixed-order sum of column b over `rows` partial rows
__device__ __forceinline__ double warp_col_sum(const double* part, int rows, int Bp, int b) {
    const int lane = threadIdx.x & 31;
    double t = 0.0;
#pragma unroll 4
    for (int q = lane; q < rows; q += 32) t += part[(size_t)q * Bp + b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    return t;
}

// alpha = rs_old / pKp with the pKp <= 0 breakdown (krylov.hpp:273-276)
__global__ void k_alpha(int Bp, int nrows, const double* part, const double* rs_old,
                        double* alpha, int* active, int* status) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= Bp) return;
    if (!active[b]) return;
    const double pKp = warp_col_sum(part, nrows, Bp, b);
    if (lane == 0) {
        if (pKp <= 0.0) {
            status[b] = ST_EBREAKDOWN;
            active[b] = 0;
        } else {
            alpha[b] = rs_old[b] / pKp;
        }
    }
}

// End of one PCG iteration (krylov.hpp:280-288): rs_new, beta, k++, rel,
// history, breakdown, convergence, one warp per instance.  The last CTA to
// finish sets the graph's while-condition to "any instance still active"
// (integer atomics only: the flag/ticket are reset by that CTA).
__global__ void __launch_bounds__(256) k_finalize(int Bp, int nrs, const double* part_rs,
                                                  int nrr, const double* part_rr,
                                                  const double* fnorm, double* rs_old,
                                                  double* beta, double* rel, int* iters,
                                                  int* active, int* status, double* hist,
                                                  const SolveParams* prm, unsigned* flag_ticket,
                                                  cudaGraphConditionalHandle cond, int set_cond) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    int any = 0;
    if (b < Bp && active[b]) {
        const double rs_new = warp_col_sum(part_rs, nrs, Bp, b);
        const double rr = warp_col_sum(part_rr, nrr, Bp, b);
        if (lane == 0) {
            const double bt = rs_new / rs_old[b];
            beta[b] = bt;
            rs_old[b] = rs_new;
            const int it = iters[b] + 1;
            iters[b] = it;
            const double fn = fnorm[b];
            const double rn = sqrt(rr);
            const double rl = fn > 0.0 ? rn / fn : rn;  // krylov.hpp:235-237
            rel[b] = rl;
            if (it < prm->hist_cap) hist[(size_t)b * prm->hist_cap + it] = rl;
            if (rs_new <= 0.0 && rl > prm->tol) {
                status[b] = ST_EBREAKDOWN;
                active[b] = 0;
            } else if (!(rl > prm->tol) || it >= prm->max_iter) {
                active[b] = 0;
            } else {
                any = 1;
            }
        }
    }
    any = __syncthreads_or(any);
    if (set_cond && threadIdx.x == 0) {
        if (any) atomicOr(&flag_ticket[0], 1u);
        __threadfence();
        const unsigned t = atomicAdd(&flag_ticket[1], 1u);
        if (t == gridDim.x - 1) {
            const unsigned f = atomicExch(&flag_ticket[0], 0u);
            atomicExch(&flag_ticket[1], 0u);
            cudaGraphSetConditional(cond, f ? 1u : 0u);
        }
    }
}

// End of one pod2g_solve cycle (pod.hpp:243-250): rel from the TRUE residual
// partials, history, cycle count, convergence; graph condition as k_finalize.
__global__ void __launch_bounds__(256) k_cycle_finalize(int Bp, int nrr, const double* part_rr,
                                                        const double* fnorm, double* rel,
                                                        int* iters, int* active, double* hist,
                                                        const SolveParams* prm,
                                                        unsigned* flag_ticket,
                                                        cudaGraphConditionalHandle cond,
                                                        int set_cond) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    int any = 0;
    if (b < Bp && active[b]) {
        const double rr = warp_col_sum(part_rr, nrr, Bp, b);
        if (lane == 0) {
            const int it = iters[b] + 1;
            iters[b] = it;
            const double fn = fnorm[b];
            const double rn = sqrt(rr);
            const double rl = fn > 0.0 ? rn / fn : rn;  // krylov.hpp:235-237
            rel[b] = rl;
            if (it < prm->hist_cap) hist[(size_t)b * prm->hist_cap + it] = rl;
            if (!(rl > prm->tol) || it >= prm->max_iter)
                active[b] = 0;
            else
                any = 1;
        }
    }
    any = __syncthreads_or(any);
    if (set_cond && threadIdx.x == 0) {
        if (any) atomicOr(&flag_ticket[0], 1u);
        __threadfence();
        const unsigned t = atomicAdd(&flag_ticket[1], 1u);
        if (t == gridDim.x - 1) {
            const unsigned f = atomicExch(&flag_ticket[0], 0u);
            atomicExch(&flag_ticket[1], 0u);
            cudaGraphSetConditional(cond, f ? 1u : 0u);
        }
    }
}

// Initial residual bookkeeping (krylov.hpp:252-260): fnorm, rel0, hist[0],
// the loop-entry test.  Instances with a setup error are not entered.
__global__ void k_init_rel(int Bp, int B, int nrows, const double* part_rr, const double* part_ff,
                           double* fnorm, double* rel, int* iters, int* active, int* status,
                           const int* setup_status, double* hist, const SolveParams* prm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= Bp) return;
    const double rr = warp_col_sum(part_rr, nrows, Bp, b);
    const double ff = warp_col_sum(part_ff, nrows, Bp, b);
    if (lane == 0) {
        iters[b] = 0;
        if (b >= B) {
            active[b] = 0;
            status[b] = ST_OK;
            return;
        }
        const double fn = sqrt(ff);
        const double rn = sqrt(rr);
        const double rl = fn > 0.0 ? rn / fn : rn;
        fnorm[b] = fn;
        rel[b] = rl;
        if (prm->hist_cap > 0) hist[(size_t)b * prm->hist_cap] = rl;
        const bool enter = rl > prm->tol && prm->max_iter > 0;
        status[b] = ST_OK;
        if (enter && setup_status[b] != ST_OK) {
            // the reference throws when the preconditioner is first applied
            status[b] = setup_status[b];
            active[b] = 0;
        } else {
            active[b] = enter ? 1 : 0;
        }
    }
}

// rs_old = r.s after the first preconditioner application (krylov.hpp:262-266)
__global__ void k_init_rs(int Bp, int nrows, const double* part_rs, double* rs_old, int* active,
                          int* status) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= Bp || !active[b]) return;
    const double rs = warp_col_sum(part_rs, nrows, Bp, b);
    if (lane == 0) {
        rs_old[b] = rs;
        if (rs <= 0.0) {
            status[b] = ST_EBREAKDOWN;
            active[b] = 0;
        }
    }
}

__global__ void k_set_cond(const int* active, int Bp, cudaGraphConditionalHandle cond) {
    int any = 0;
    for (int b = threadIdx.x; b < Bp; b += blockDim.x) any |= active[b];
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) cudaGraphSetConditional(cond, any ? 1u : 0u);
}

// ================ single-cluster persistent PCG loop (small single systems)
// c1-sized problems (a few thousand dofs, one instance) are latency bound:
// the captured loop runs 15 launches per iteration at ~3.3 us each, and every
// kernel is a chain of 2-3 dependent L2 round trips (~0.5 us each).  Here the
// WHOLE loop (krylov.hpp:267-289 with the Kp recurrence D9 and the POD-2G
// preconditioner, pod.hpp:264-267) runs inside ONE kernel on one thread-block
// cluster of kClSize CTAs:
//   * the phases of an iteration are separated by the hardware cluster
//     barrier (~0.2 us) instead of kernel boundaries, the dot products are
//     combined over distributed shared memory (fixed rank order), and the
//     convergence test never leaves the kernel;
//   * the matrix is SHARED-MEMORY RESIDENT: node q belongs to CTA q % kClSize,
//     which keeps the node's BS x rowlen values and column indices in
//     [entry][slot] layout (conflict free) for the whole solve, so a node's
//     only L2 round trip per phase is ONE round of x gathers, all issued
//     together (the vectors stay in L2: ~0.2 MB);
//   * one THREAD owns a node and walks its rows and their entries in
//     ascending column order with separately rounded multiply / subtract --
//     the reference's own operation order (smoothers.hpp:31-44, 56-70) on the
//     colour-permuted system, without the xor-tree reassociation of the
//     warp-per-node B = 1 kernels.  Reductions are fixed-order (D4).
// Q4-shaped patterns (2 dofs per node, <= 9 neighbour nodes) whose matrix
// fits the cluster's shared memory (<= ~3700 nodes).
constexpr int kClSize = 8;       // CTAs per cluster (portable maximum)
constexpr int kClThreads = 320;  // threads per CTA (204 registers each: a node's 36 gathers stay in flight)
constexpr int kClKmax = 40;      // POD rank limit (coarse vectors and factor in shared memory)
constexpr int kClBS = 2, kClRL = 18;  // dofs per node, entries per row at most

struct ClusterLoop {
    int n, k, ncolors, nrows_pkp, nl;  // nl = node slots per CTA = ceil(nodes / kClSize)
    int color_rows[17];
    const int *rp, *ci, *dpos;
    const double *vals, *phi, *Lfac;  // phi [n][k], Lfac [k][k] (LDL^T, row-major)
    double *u, *r, *p, *Kp, *s, *s2;  // s: forward sweep / prolongated s', s2: backward sweep
    const double* part_pkp;           // pKp partial rows of the prologue's SpMV
    double *rs_old, *rel, *hist, *beta, *alpha;
    const double* fnorm;
    int *iters, *active, *status;
    const SolveParams* prm;
    long long* trace;  // P2G_CLUSTER_TRACE=1: clock64 at the phase boundaries of iteration 2
};
// matrix values + column indices + per-node {row length, own position} + the nodes' Phi rows
inline size_t cluster_loop_smem(int nl, int k) {
    return (size_t)nl * (kClBS * kClRL * (sizeof(double) + sizeof(int)) + 2 * sizeof(int) +
                         kClBS * (size_t)k * sizeof(double)) + 16;
}

struct ClusterShared {
    double warp[kClThreads / 32][2];      // per-warp partials of a block reduction
    double slot[4][2];                    // this CTA's published partials, one slot per reduction point
    double total[2];                      // cluster totals, broadcast inside the CTA
    double prod[8][kClThreads];           // restriction: per-thread products of 8 coefficients
    double cpart[kClKmax];                // this CTA's restriction partial (read over DSMEM)
    double cvec[kClKmax];                 // coarse right-hand side, then the coarse solution e
};

// block-reduce a value (fixed xor tree per warp, warps in order) into this
// CTA's slot; the caller's cluster barrier publishes it
__device__ __forceinline__ void cl_block_reduce(ClusterShared& S, int slot, double a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    a = warp_sum(a);
    if (lane == 0) S.warp[warp][0] = a;
    __syncthreads();
    if (threadIdx.x == 0) {
        double ta = 0.0;
        for (int w = 0; w < kClThreads / 32; ++w) ta += S.warp[w][0];
        S.slot[slot][0] = ta;
    }
}

// after the cluster barrier: sum the CTAs' slots in rank order (same value on every CTA)
__device__ __forceinline__ double cl_gather(cg::cluster_group& cl, ClusterShared& S, int slot) {
    if (threadIdx.x == 0) {
        double ta = 0.0;
        for (int rk = 0; rk < kClSize; ++rk) ta += cl.map_shared_rank(&S.slot[slot][0], rk)[0];
        S.total[0] = ta;
    }
    __syncthreads();
    const double a = S.total[0];
    __syncthreads();
    return a;
}

// Vector loads: plain (weak) loads.  Every vector element read here was
// written before the last cluster barrier (release / acquire at cluster
// scope, which also invalidates L1) or by the reading thread itself.
// (ld.global.cg compiles to LDG.STRONG.GPU here, which the hardware does not
// overlap: a node's 36 gathers then cost 36 serial L2 round trips.)
__device__ __forceinline__ double cl_ld(const double* p) { return *p; }

// one node's view of the shared-memory resident matrix
struct ClNode {
    const double* mv;  // values of entry (c, e) at mv[(c * kClRL + e) * nl]
    const int* mc;     // column indices, same layout
    int nl, rl, dp0;   // slot stride, entries per row, in-row position of the node's own block
};

// x[e] = X[col(c, e)] for the entries e in [e0, e1) of row c (one round of L2 loads)
__device__ __forceinline__ void cl_gather_row(const ClNode& N, int c, int e0, int e1, const double* X,
                                              double (&x)[kClRL]) {
#pragma unroll
    for (int e = 0; e < kClRL; ++e) {
        const bool in = e >= e0 && e < e1;
        const int col = in ? N.mc[(c * kClRL + e) * N.nl] : 0;
        const double v = cl_ld(X + col);  // out-of-range entries read X[0], never used
        x[e] = in ? v : x[e];
    }
}
// sum (-= | +=) a(c, e) * x[e] over e in [e0, e1), ascending, separately rounded
template <bool SUB>
__device__ __forceinline__ double cl_row_sum(const ClNode& N, int c, int e0, int e1,
                                             const double (&x)[kClRL], double sum) {
#pragma unroll
    for (int e = 0; e < kClRL; ++e) {
        if (e >= e0 && e < e1) {
            const double pr = __dmul_rn(N.mv[(c * kClRL + e) * N.nl], x[e]);
            sum = SUB ? __dsub_rn(sum, pr) : __dadd_rn(sum, pr);
        }
    }
    return sum;
}

__global__ void __cluster_dims__(kClSize, 1, 1) __launch_bounds__(kClThreads, 1)
    k_pcg_cluster(ClusterLoop A) {
    constexpr int BS = kClBS, RL = kClRL;
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClusterShared S;
    __shared__ double Ls[kClKmax * kClKmax];
    extern __shared__ __align__(16) unsigned char cl_dyn[];
    const int nl = A.nl;
    double* mv = reinterpret_cast<double*>(cl_dyn);
    int* mc = reinterpret_cast<int*>(mv + (size_t)BS * RL * nl);
    int* meta = mc + (size_t)BS * RL * nl;  // [nl][2] = {row length, own block position}
    // the nodes' Phi rows, [c][a][slot] (8-byte aligned: 2 * nl ints precede it and BS * RL * nl is even)
    double* mphi = reinterpret_cast<double*>(meta + 2 * nl);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int crank = (int)cl.block_rank();
    const int n = A.n, k = A.k, C = A.ncolors;
    const int nn = n / BS;
    const int mine = (nn - crank + kClSize - 1) / kClSize;  // this CTA's nodes: slot * kClSize + crank
    if (!A.active[0]) return;  // uniform over the cluster
    // ---- the CTA's share of the matrix into shared memory, once
    for (int sl = threadIdx.x; sl < mine; sl += kClThreads) {
        const int i0 = (sl * kClSize + crank) * BS;
        const int kb = __ldg(A.rp + i0), rl = __ldg(A.rp + i0 + 1) - kb;
        meta[2 * sl] = rl;
        meta[2 * sl + 1] = __ldg(A.dpos + i0) - kb;
        for (int c = 0; c < BS; ++c)
            for (int e = 0; e < rl; ++e) {
                mv[(c * RL + e) * nl + sl] = __ldg(A.vals + kb + c * rl + e);
                mc[(c * RL + e) * nl + sl] = __ldg(A.ci + kb + c * rl + e);
            }
    }
    for (int sl = threadIdx.x; sl < mine; sl += kClThreads) {
        const int i0 = (sl * kClSize + crank) * BS;
        for (int c = 0; c < BS; ++c)
            for (int a = 0; a < k; ++a) mphi[(c * k + a) * nl + sl] = __ldg(A.phi + (size_t)(i0 + c) * k + a);
    }
    for (int e2 = threadIdx.x; e2 < k * k; e2 += kClThreads) Ls[e2] = A.Lfac[e2];
#define P2G_CL_TRACE(j) \
    if (A.trace && crank == 0 && threadIdx.x == 0 && it == A.iters[0] + 1) A.trace[j] = clock64();
    // pKp of the prologue's SpMV: fixed-order sum of its partial rows
    double pKp = 0.0;
    for (int q = 0; q < A.nrows_pkp; ++q) pKp += A.part_pkp[q];
    double rs_old = A.rs_old[0];
    const double fn = A.fnorm[0];
    const double tol = A.prm->tol;
    const long long max_iter = A.prm->max_iter, hist_cap = A.prm->hist_cap;
    long long it = A.iters[0];
    int status = ST_OK;
    double rl_ = A.rel[0], beta = 0.0, alpha = 0.0;
    __syncthreads();
    // local slot range of the nodes [nb, ne) (node = slot * kClSize + crank)
    auto first_slot = [&](int nb) { return nb > crank ? (nb - crank + kClSize - 1) / kClSize : 0; };
    auto node_of = [&](int sl, ClNode& N) {
        N.mv = mv + sl;
        N.mc = mc + sl;
        N.nl = nl;
        N.rl = meta[2 * sl];
        N.dp0 = meta[2 * sl + 1];
        return (sl * kClSize + crank) * BS;
    };
    for (;;) {
        // ---- alpha (krylov.hpp:273-276)
        if (pKp <= 0.0) {
            status = ST_EBREAKDOWN;
            break;
        }
        alpha = rs_old / pKp;
        P2G_CL_TRACE(44)
        // ---- u += alpha p ; r -= alpha Kp ; r.r ; colour-0 forward rows (own lower components only)
        double rr = 0.0;
        const int c0s = first_slot(A.color_rows[1] / BS);
        for (int sl = threadIdx.x; sl < mine; sl += kClThreads) {
            ClNode N;
            const int i0 = node_of(sl, N);
            double sn[BS];
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                const int i = i0 + c;
                const double ui = __dadd_rn(cl_ld(A.u + i), __dmul_rn(alpha, cl_ld(A.p + i)));
                const double ri = __dadd_rn(cl_ld(A.r + i), __dmul_rn(-alpha, cl_ld(A.Kp + i)));
                rr = __dadd_rn(rr, __dmul_rn(ri, ri));
                A.u[i] = ui;
                A.r[i] = ri;
                if (sl < c0s) {
                    double sum = ri;
#pragma unroll
                    for (int cc = 0; cc < c; ++cc)
                        sum = __dsub_rn(sum, __dmul_rn(N.mv[(c * RL + N.dp0 + cc) * nl], sn[cc]));
                    sn[c] = __ddiv_rn(sum, N.mv[(c * RL + N.dp0 + c) * nl]);
                    A.s[i] = sn[c];
                }
            }
        }
        P2G_CL_TRACE(0)
        cl_block_reduce(S, 0, rr);
        cl.sync();
        P2G_CL_TRACE(1)
        // ---- forward colours 1 .. C-1 (first sweep from zero: L part only)
        for (int col = 1; col < C; ++col) {
            const int sb = first_slot(A.color_rows[col] / BS), se = first_slot(A.color_rows[col + 1] / BS);
            for (int sl = sb + threadIdx.x; sl < se; sl += kClThreads) {
                ClNode N;
                const int i0 = node_of(sl, N);
                double x[BS][RL] = {}, ri[BS], sn[BS];
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    cl_gather_row(N, c, 0, N.dp0, A.s, x[c]);
                    ri[c] = cl_ld(A.r + i0 + c);
                }
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    double sum = cl_row_sum<true>(N, c, 0, N.dp0, x[c], ri[c]);
#pragma unroll
                    for (int cc = 0; cc < c; ++cc)
                        sum = __dsub_rn(sum, __dmul_rn(N.mv[(c * RL + N.dp0 + cc) * nl], sn[cc]));
                    sn[c] = __ddiv_rn(sum, N.mv[(c * RL + N.dp0 + c) * nl]);
                    A.s[i0 + c] = sn[c];
                }
            }
            cl.sync();
        }
        P2G_CL_TRACE(2)
        if (k > 0) {
            // ---- t = -U s (D6) and c = Phi^T t: every thread's products of 8
            // coefficients at a time into shared memory, one warp sums each
            // coefficient over the threads (lane-strided, then a fixed xor tree)
            for (int a = threadIdx.x; a < k; a += kClThreads) S.cpart[a] = 0.0;
            for (int base = 0; base < mine; base += kClThreads) {
                const int sl = base + threadIdx.x;
                const bool ok = sl < mine;
                double t[BS];
#pragma unroll
                for (int c = 0; c < BS; ++c) t[c] = 0.0;
                if (ok) {
                    ClNode N;
                    node_of(sl, N);
                    double x[BS][RL] = {};
#pragma unroll
                    for (int c = 0; c < BS; ++c) cl_gather_row(N, c, N.dp0 + c + 1, N.rl, A.s, x[c]);
#pragma unroll
                    for (int c = 0; c < BS; ++c)
                        t[c] = -cl_row_sum<false>(N, c, N.dp0 + c + 1, N.rl, x[c], 0.0);
                }
                for (int a0 = 0; a0 < k; a0 += 8) {
                    __syncthreads();  // S.prod is free again
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        double v = 0.0;
                        if (ok && a0 + q < k) {
#pragma unroll
                            for (int c = 0; c < BS; ++c)
                                v = __dadd_rn(v, __dmul_rn(mphi[(c * k + a0 + q) * nl + sl], t[c]));
                        }
                        S.prod[q][threadIdx.x] = v;
                    }
                    __syncthreads();
                    if (warp < 8 && a0 + warp < k) {
                        double v = 0.0;
                        for (int q = lane; q < kClThreads; q += 32) v += S.prod[warp][q];
                        v = warp_sum(v);
                        if (lane == 0) S.cpart[a0 + warp] += v;
                    }
                }
            }
            P2G_CL_TRACE(3)
            cl.sync();
            P2G_CL_TRACE(4)
            if (threadIdx.x < k) {
                double tt = 0.0;
                for (int rk = 0; rk < kClSize; ++rk)
                    tt += cl.map_shared_rank(&S.cpart[0], rk)[threadIdx.x];
                S.cvec[threadIdx.x] = tt;
            }
            __syncthreads();
            // e = A_c^{-1} c with the LDL^T factor (k_coarse's substitution order)
            if (warp == 0) {
                double y0 = lane < k ? S.cvec[lane] : 0.0, y1 = lane + 32 < k ? S.cvec[lane + 32] : 0.0;
                for (int j = 0; j < k; ++j) {
                    const double yj = __shfl_sync(0xffffffffu, j < 32 ? y0 : y1, j & 31);
                    if (lane > j && lane < k) y0 -= Ls[lane * k + j] * yj;
                    if (lane + 32 > j && lane + 32 < k) y1 -= Ls[(lane + 32) * k + j] * yj;
                }
                if (lane < k) y0 /= Ls[lane * k + lane];
                if (lane + 32 < k) y1 /= Ls[(lane + 32) * k + lane + 32];
                for (int j = k - 1; j >= 0; --j) {
                    const double xj = __shfl_sync(0xffffffffu, j < 32 ? y0 : y1, j & 31);
                    if (lane < j) y0 -= Ls[j * k + lane] * xj;
                    if (lane + 32 < j) y1 -= Ls[j * k + lane + 32] * xj;
                }
                __syncwarp();
                if (lane < k) S.cvec[lane] = y0;
                if (lane + 32 < k) S.cvec[lane + 32] = y1;
            }
            __syncthreads();
            P2G_CL_TRACE(5)
            // ---- s' = s + Phi e (ascending coefficients, fused multiply-adds: k_prolong)
            for (int sl = threadIdx.x; sl < mine; sl += kClThreads) {
                const int i0 = (sl * kClSize + crank) * BS;
                double si[BS];
#pragma unroll
                for (int c = 0; c < BS; ++c) si[c] = cl_ld(A.s + i0 + c);
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    double corr = 0.0;
                    for (int a = 0; a < k; ++a) corr = fma(mphi[(c * k + a) * nl + sl], S.cvec[a], corr);
                    A.s[i0 + c] = __dadd_rn(si[c], corr);
                }
            }
            P2G_CL_TRACE(6)
            cl.sync();  // also protects S.cpart / S.cvec against the next iteration
            P2G_CL_TRACE(7)
        }
        // ---- backward sweep, out of place (D9): L part from s', U part from the new s2
        double rs = 0.0;
        for (int col = C - 1; col >= 0; --col) {
            const int sb = first_slot(A.color_rows[col] / BS), se = first_slot(A.color_rows[col + 1] / BS);
            for (int sl = sb + threadIdx.x; sl < se; sl += kClThreads) {
                ClNode N;
                const int i0 = node_of(sl, N);
                double x[BS][RL] = {}, ri[BS];
#pragma unroll
                for (int c = 0; c < BS; ++c) {
                    // lower nodes and own components below c: s' ; upper nodes: s2 ; own
                    // components above c are this thread's new values (patched in below)
                    cl_gather_row(N, c, 0, N.dp0 + c, A.s, x[c]);
                    cl_gather_row(N, c, N.dp0 + BS, N.rl, A.s2, x[c]);
                    ri[c] = cl_ld(A.r + i0 + c);
                }
#pragma unroll
                for (int c = BS - 1; c >= 0; --c) {
                    double sum = cl_row_sum<true>(N, c, 0, N.dp0 + c, x[c], ri[c]);
                    sum = cl_row_sum<true>(N, c, N.dp0 + c + 1, N.rl, x[c], sum);
                    const double si = __ddiv_rn(sum, N.mv[(c * RL + N.dp0 + c) * nl]);
                    A.s2[i0 + c] = si;
                    rs = __dadd_rn(rs, __dmul_rn(ri[c], si));
#pragma unroll
                    for (int cr = 0; cr < BS; ++cr) {
                        if (cr < c) {
#pragma unroll
                            for (int e = 0; e < RL; ++e) x[cr][e] = e == N.dp0 + c ? si : x[cr][e];
                        }
                    }
                }
            }
            if (col == 0) cl_block_reduce(S, 1, rs);
            P2G_CL_TRACE(8 + 2 * (C - 1 - col))
            cl.sync();
            P2G_CL_TRACE(9 + 2 * (C - 1 - col))
        }
        // ---- end of the iteration (krylov.hpp:280-288), identical on every thread
        const double rr_t = cl_gather(cl, S, 0);
        const double rs_new = cl_gather(cl, S, 1);
        beta = rs_new / rs_old;
        rs_old = rs_new;
        ++it;
        const double rn = sqrt(rr_t);
        rl_ = fn > 0.0 ? rn / fn : rn;
        if (crank == 0 && threadIdx.x == 0 && it < hist_cap) A.hist[it] = rl_;
        bool done = false;
        if (rs_new <= 0.0 && rl_ > tol) {
            status = ST_EBREAKDOWN;
            done = true;
        } else if (!(rl_ > tol) || it >= max_iter) {
            done = true;
        }
        P2G_CL_TRACE(40)
        if (done) break;
        // ---- Kp = r + L (s2 - s') + beta Kp ; p = s2 + beta p ; p.Kp (D9)
        double dot = 0.0;
        for (int sl = threadIdx.x; sl < mine; sl += kClThreads) {
            ClNode N;
            const int i0 = node_of(sl, N);
#pragma unroll
            for (int c = 0; c < BS; ++c) {
                const int i = i0 + c;
                double x1[RL] = {}, x0[RL] = {};
                cl_gather_row(N, c, 0, N.dp0 + c, A.s2, x1);
                cl_gather_row(N, c, 0, N.dp0 + c, A.s, x0);
                const double ri = cl_ld(A.r + i), kp0 = cl_ld(A.Kp + i), s2i = cl_ld(A.s2 + i),
                             p0 = cl_ld(A.p + i);
#pragma unroll
                for (int e = 0; e < RL; ++e) x1[e] = __dsub_rn(x1[e], x0[e]);
                const double acc = cl_row_sum<false>(N, c, 0, N.dp0 + c, x1, 0.0);
                const double kpi = __dadd_rn(__dadd_rn(ri, acc), __dmul_rn(beta, kp0));
                const double pi = __dadd_rn(s2i, __dmul_rn(beta, p0));
                dot = __dadd_rn(dot, __dmul_rn(pi, kpi));
                A.Kp[i] = kpi;
                A.p[i] = pi;
            }
        }
        P2G_CL_TRACE(41)
        cl_block_reduce(S, 2, dot);
        cl.sync();
        P2G_CL_TRACE(42)
        pKp = cl_gather(cl, S, 2);
        P2G_CL_TRACE(43)
    }
    if (crank == 0 && threadIdx.x == 0) {
        A.rs_old[0] = rs_old;
        A.iters[0] = (int)it;
        A.rel[0] = rl_;
        A.beta[0] = beta;
        A.alpha[0] = alpha;
        A.active[0] = 0;
        if (status != ST_OK) A.status[0] = status;
    }
    cl.sync();  // no CTA exits while its shared memory may still be read
}

// ---------------------------------------------------------------- layout kernels
// dst[new][Bp] (b < B) <- src[b][old] with old = map[new] ; padded columns = pad
__global__ void k_gather_interleave(const double* __restrict__ src, int64_t src_stride, int B,
                                    const int64_t* __restrict__ map, int64_t nnew,
                                    double* __restrict__ dst, int Bp, int b_off, double pad) {
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int bb = blockIdx.y * 32;
    for (int q = ty; q < 32; q += 8) {
        const int b = bb + q;
        const int64_t j = j0 + tx;
        double v = pad;
        if (j < nnew && b < Bp) {
            if (b - b_off >= 0 && b - b_off < B) v = src[(int64_t)(b - b_off) * src_stride + map[j]];
        }
        tile[q][tx] = v;
    }
    __syncthreads();
    for (int q = ty; q < 32; q += 8) {
        const int64_t j = j0 + q;
        const int b = bb + tx;
        if (j < nnew && b < Bp && b - b_off >= 0 && b - b_off < B) dst[j * Bp + b] = tile[tx][q];
    }
}

// dst[b][map[i]] <- src[i][Bp] for b < B (inverse of the above for vectors)
__global__ void k_scatter_deinterleave(const double* __restrict__ src, int Bp, int64_t n,
                                       const int64_t* __restrict__ map, int B,
                                       double* __restrict__ dst) {
    __shared__ double tile[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t i0 = (int64_t)blockIdx.x * 32;
    const int bb = blockIdx.y * 32;
    for (int q = ty; q < 32; q += 8) {
        const int64_t i = i0 + q;
        const int b = bb + tx;
        tile[q][tx] = (i < n && b < Bp) ? src[i * Bp + b] : 0.0;
    }
    __syncthreads();
    for (int q = ty; q < 32; q += 8) {
        const int b = bb + q;
        const int64_t i = i0 + tx;
        if (i < n && b < B) dst[(int64_t)b * n + map[i]] = tile[tx][q];
    }
}

// zero diagonal check (smoothers.hpp:41-43) -> setup status
__global__ void k_check_diag(Mat A, int B, int* status) {
    const int b = blockIdx.y;
    if (b >= B) return;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += gridDim.x * blockDim.x) {
        if (A.vals[(size_t)A.dpos[i] * A.Bp + b] == 0.0) status[b] = ST_EZERODIAG;
    }
}

// non-finite solution check (krylov.hpp:295) for instances without an error
__global__ void k_check_finite(int n, int Bp, const double* u, int* status) {
    const int b = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (!isfinite(u[(size_t)i * Bp + b]) && status[b] == ST_OK) status[b] = ST_ENONFINITE;
    }
}

// ---------------------------------------------------------------- setup kernels
// Y[i][a][bt] = sum_j K_ij Phi[j][a] for the instance chunk [bofs, bofs+Bt)
// (reduced_operator's spmv(K, phi_j), pod.hpp:157, for all k columns at once)
template <class Sh, int KMAX>
__global__ void __launch_bounds__(kBlock) k_spmm_phi(Mat A, const double* __restrict__ phi, int k,
                                                     int bofs, int Bt, double* __restrict__ Y) {
    LaneGeo<Sh> G;
    const int bt = blockIdx.y * Sh::T + G.w;  // V == 1 here
    const int b0 = bofs + bt;
    const int nn = A.n / A.bs;
    P2G_NODE_LOOP(Sh, 0, nn, G) {
        const int node = base_ + G.r;
        const bool valid = node < nn && bt < Bt;
        for (int c = 0; c < A.bs; ++c) {
            const int i = node * A.bs + c;
            double acc[KMAX];
#pragma unroll
            for (int a = 0; a < KMAX; ++a) acc[a] = 0.0;
            if (valid) {
                const int kb = __ldg(A.rp + i), ke = __ldg(A.rp + i + 1);
                for (int q = kb + G.s; q < ke; q += Sh::S) {
                    const int col = __ldg(A.ci + q);
                    const double v = __ldcs(A.vals + (size_t)q * A.Bp + b0);
                    const double* ph = phi + (size_t)col * k;
#pragma unroll
                    for (int a = 0; a < KMAX; ++a)
                        if (a < k) acc[a] = fma(v, __ldg(ph + a), acc[a]);
                }
            }
#pragma unroll
            for (int a = 0; a < KMAX; ++a) acc[a] = slot_sum<Sh>(acc[a]);
            if (valid && G.s == 0) {
                double* y = Y + ((size_t)i * k) * Bt + bt;
#pragma unroll
                for (int a = 0; a < KMAX; ++a)
                    if (a < k) y[(size_t)a * Bt] = acc[a];
            }
        }
    }
}

// part[blk][a][j] = sum_{i in block rows} phi[i][a] * X[i][j], j < ncol
template <int KMAX>
__global__ void __launch_bounds__(kBlock) k_restrict_cols(int n, int ncol, const double* __restrict__ X,
                                                          const double* __restrict__ phi, int k,
                                                          double* part) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int j = blockIdx.y * 32 + lane;
    double acc[KMAX];
#pragma unroll
    for (int a = 0; a < KMAX; ++a) acc[a] = 0.0;
    for (int i = blockIdx.x * kWarps + warp; i < n; i += gridDim.x * kWarps) {
        const double x = j < ncol ? X[(size_t)i * ncol + j] : 0.0;
        const double* ph = phi + (size_t)i * k;
#pragma unroll
        for (int a = 0; a < KMAX; ++a)
            if (a < k) acc[a] = fma(__ldg(ph + a), x, acc[a]);
    }
    __shared__ double sm[kWarps][8][32];
#pragma unroll
    for (int a0 = 0; a0 < KMAX; a0 += 8) {
        if (a0 >= k) break;
#pragma unroll
        for (int q = 0; q < 8; ++q) sm[warp][q][lane] = acc[a0 + q];
        __syncthreads();
        {
            const int q = threadIdx.x / 32, l = threadIdx.x % 32;  // 8 x 32
            const int jj = blockIdx.y * 32 + l;
            if (a0 + q < k && jj < ncol) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) t += sm[w][q][l];
                part[((size_t)blockIdx.x * k + a0 + q) * ncol + jj] = t;
            }
        }
        __syncthreads();
    }
}

// Ac[bofs+bt][a][c] = sum_blk part[blk][a][c*Bt+bt]
__global__ void k_reduce_ac(int nblk, int k, int Bt, int bofs, const double* part, double* Ac) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * (blockDim.x >> 5) + warp;  // (bt, a, c)
    const int total = Bt * k * k;
    if (e >= total) return;
    const int bt = e / (k * k), a = (e / k) % k, c = e % k;
    const int ncol = k * Bt;
    double t = 0.0;
    for (int blk = lane; blk < nblk; blk += 32) t += part[((size_t)blk * k + a) * ncol + c * Bt + bt];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) Ac[((size_t)(bofs + bt) * k + a) * k + c] = t;
}

// Square-root-free Cholesky (LDL^T, no pivoting) of the symmetrised A_c,
// one warp per instance.  Works for any symmetric matrix with nonzero leading
// minors, so an indefinite coarse operator factors like the reference's LU
// and surfaces later as a PCG breakdown; singular (dense_solve.hpp:20,25-26
// analogue) when a pivot |d_j| <= 1e-14 * max|a|.
__global__ void k_cholesky(int B, int k, const double* Ac, double* L, int* status) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int b = blockIdx.x * (blockDim.x >> 5) + warp;
    if (b >= B) return;
    const double* A = Ac + (size_t)b * k * k;
    double* Lb = L + (size_t)b * k * k;
    double mx = 0.0;
    for (int e = lane; e < k * k; e += 32) mx = fmax(mx, fabs(A[e]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const double floor_ = 1e-14 * mx;
    for (int e = lane; e < k * k; e += 32) {
        const int i = e / k, j = e % k;
        Lb[e] = j <= i ? 0.5 * (A[i * k + j] + A[j * k + i]) : 0.0;
    }
    __syncwarp();
    bool bad = false;
    for (int j = 0; j < k; ++j) {
        // d_j = a_jj - sum_q l_jq^2 d_q
        double d = Lb[j * k + j];
        for (int q = 0; q < j; ++q) d -= Lb[j * k + q] * Lb[j * k + q] * Lb[q * k + q];
        if (!(fabs(d) > floor_)) bad = true;
        const double dj = bad ? 1.0 : d;
        __syncwarp();
        for (int i = j + 1 + lane; i < k; i += 32) {
            double v = Lb[i * k + j];
            for (int q = 0; q < j; ++q) v -= Lb[i * k + q] * Lb[j * k + q] * Lb[q * k + q];
            Lb[i * k + j] = v / dj;
        }
        __syncwarp();
        if (lane == 0) Lb[j * k + j] = dj;
        __syncwarp();
    }
    if (lane == 0 && bad && status[b] == ST_OK) status[b] = ST_ESINGULAR;
}

// ---------------------------------------------------------------- generation
// On-device instance generation: the values of a structured
// Q4 / hex8 stiffness matrix K(E) = sum_e E_e K_e^1 written straight into the
// solver's permuted [nnz][Bp] layout.  Each stored entry (node i, comp c;
// node j, comp d) is the sum over the elements shared by nodes i and j in
// ascending element order of E_e * Ke1[a c][b d] -- separately rounded
// multiply and add, exactly the host generator's arithmetic (p2g_mesh.cpp),
// so both produce identical bits.
struct AsmDesc {
    int dim, ned;
    long long nx, ny, nz;        // elements per axis
    long long row_begin;         // first global row of this handle's rows
    long long q_base;            // generator entry index of row_begin
    const double* Ke;            // ned x ned
    const unsigned long long* rpg;  // generator row offsets (global)
};

__device__ __forceinline__ int hex_local(int ox, int oy, int oz) {
    return (oy ? (ox ? 2 : 3) : (ox ? 1 : 0)) + 4 * oz;
}

__global__ void __launch_bounds__(kBlock) k_assemble(Mat A, AsmDesc d, const int64_t* __restrict__ perm,
                                                     const int64_t* __restrict__ vperm,
                                                     const double* __restrict__ Et, int B,
                                                     double* vals) {
    __shared__ double Ks[24 * 24];
    for (int q = threadIdx.x; q < d.ned * d.ned; q += blockDim.x) Ks[q] = d.Ke[q];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long NX = d.nx + 1, NY = d.ny + 1, NZ = d.dim == 3 ? d.nz + 1 : 1;
    for (int i = blockIdx.x * kWarps + warp; i < A.n; i += gridDim.x * kWarps) {
        const long long g = d.row_begin + perm[i];
        const int c = (int)(g % d.dim);
        const long long rn = g / d.dim;
        const long long ix = rn % d.nx + 1, t = rn / d.nx, iy = t % NY, iz = t / NY;
        const long long ax = max(1LL, ix - 1), bx = min(NX - 1, ix + 1);
        const long long ay = max(0LL, iy - 1), by = min(NY - 1, iy + 1);
        const long long az = max(0LL, iz - 1);
        const long long sx = bx - ax + 1, sy = by - ay + 1;
        const long long rowq = (long long)d.rpg[g];
        (void)az;
        const int kb = A.rp[i], len = A.rp[i + 1] - kb;
        for (int p = lane; p < len * B; p += 32) {
            const int k = kb + p / B, b = p % B;
            const long long o = vperm[k] + d.q_base - rowq;
            const long long slot = o / d.dim;
            const int dd = (int)(o % d.dim);
            const long long jx = ax + slot % sx, jy = ay + (slot / sx) % sy;
            const long long jz = d.dim == 3 ? max(0LL, iz - 1) + slot / (sx * sy) : 0;
            const long long ex0 = max(max(ix, jx) - 1, 0LL), ex1 = min(min(ix, jx), d.nx - 1);
            const long long ey0 = max(max(iy, jy) - 1, 0LL), ey1 = min(min(iy, jy), d.ny - 1);
            long long ez0 = 0, ez1 = 0;
            if (d.dim == 3) {
                ez0 = max(max(iz, jz) - 1, 0LL);
                ez1 = min(min(iz, jz), d.nz - 1);
            }
            double v = 0.0;
            for (long long ez = ez0; ez <= ez1; ++ez)
                for (long long ey = ey0; ey <= ey1; ++ey)
                    for (long long ex = ex0; ex <= ex1; ++ex) {
                        const int la = hex_local((int)(ix - ex), (int)(iy - ey), (int)(iz - ez));
                        const int lb = hex_local((int)(jx - ex), (int)(jy - ey), (int)(jz - ez));
                        const long long e = (ez * d.ny + ey) * d.nx + ex;
                        v = __dadd_rn(v, __dmul_rn(Et[e * B + b], Ks[(la * d.dim + c) * d.ned + lb * d.dim + dd]));
                    }
            vals[(size_t)k * A.Bp + b] = v;
        }
    }
}

// Et[e][b] = E[b][e]
__global__ void k_transpose_E(const double* __restrict__ E, int B, long long nelem, double* Et) {
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < nelem * B;
         q += (long long)gridDim.x * blockDim.x) {
        const long long e = q / B;
        const int b = (int)(q % B);
        Et[q] = E[(long long)b * nelem + e];
    }
}

// ---------------------------------------------------------------- partitions
// part[0][j] = sum_{q < nrows} part[q][j] (fixed order, in place): the local
// total of a partial-row buffer before the cross-rank allreduce
__global__ void k_reduce_rows(double* part, int nrows, int ncols) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ncols; j += gridDim.x * blockDim.x) {
        double t = 0.0;
        for (int q = 0; q < nrows; ++q) t += part[(size_t)q * ncols + j];
        part[j] = t;
    }
}

constexpr int kMaxParts = 16;
struct PartPtrs {
    double* p[kMaxParts];
    int* ip[kMaxParts];
};
// emulated allreduce over the in-process partitions: fixed rank order
__global__ void k_sum_parts(PartPtrs pp, int np, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        double t = 0.0;
        for (int q = 0; q < np; ++q) t += pp.p[q][j];
        for (int q = 0; q < np; ++q) pp.p[q][j] = t;
    }
}
__global__ void k_max_parts_int(PartPtrs pp, int np, int n) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        int t = 0;
        for (int q = 0; q < np; ++q) t = max(t, pp.ip[q][j]);
        for (int q = 0; q < np; ++q) pp.ip[q][j] = t;
    }
}
// buf[m][b] = X[rows[m]][b]: pack the boundary rows a peer needs
__global__ void k_pack_rows(const double* __restrict__ X, int Bp, const int* __restrict__ rows,
                            int64_t count, double* __restrict__ buf) {
    const int64_t total = count * Bp;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m = e / Bp;
        const int b = (int)(e % Bp);
        buf[e] = X[(size_t)rows[m] * Bp + b];
    }
}

}  // namespace p2g
