// p2g_mesh.cpp -- structured Q4 / hex8 elasticity generator (include/pod2g_gen.h).
//
// The pattern and the values are built directly row by row (no COO sort):
// on a structured grid the elements shared by a row node and a column node
// are the ex in [max(ix,jx)-1, min(ix,jx)] (same per axis), so every stored
// entry is a sum of at most 2^dim unit-modulus element-stiffness entries
// scaled by the element moduli.  This keeps even the 1e9-nonzero hex8 160^3
// config within a few seconds on the host.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <thread>
#include <vector>

#include "../../include/pod2g_gen.h"
#include "p2g_mesh_desc.h"
#include "p2g_pattern.h"

struct p2g_mesh {
    int dim = 2;
    int64_t nx = 0, ny = 0, nz = 1;   // elements per axis (nz = 1 in 2D)
    double L[3] = {1, 1, 1};
    double h = 1;
    double nu = 0.3;
    int nen = 4;   // nodes per element
    int ned = 8;   // dofs per element
    std::vector<double> Ke;           // ned x ned, E = 1
    int64_t n = 0, nnz = 0, nelem = 0;
    std::vector<uint64_t> rp;         // n+1
};

namespace {

constexpr int P2G_GEN_OK = 0, P2G_GEN_EINVAL = 1;

// local node order: bit 0 -> x, bit 1 -> y, bit 2 -> z offsets, arranged
// counter-clockwise in each z layer: (0,0),(1,0),(1,1),(0,1)
const int kLoc[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0},
                        {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};

int local_index(int dx, int dy, int dz) {
    for (int a = 0; a < 8; ++a)
        if (kLoc[a][0] == dx && kLoc[a][1] == dy && kLoc[a][2] == dz) return a;
    return -1;
}

// Q4 plane stress, square element of side h, 2x2 Gauss; E = 1
void q4_stiffness(double h, double nu, std::vector<double>& Ke) {
    const double c = 1.0 / (1.0 - nu * nu);
    const double D[3][3] = {{c, c * nu, 0}, {c * nu, c, 0}, {0, 0, c * (1.0 - nu) / 2.0}};
    Ke.assign(64, 0.0);
    const double g = 1.0 / std::sqrt(3.0);
    const double detJ = (h / 2.0) * (h / 2.0), inv = 2.0 / h;
    for (int gx = -1; gx <= 1; gx += 2)
        for (int gy = -1; gy <= 1; gy += 2) {
            const double xi = gx * g, eta = gy * g;
            double dN[4][2];
            for (int a = 0; a < 4; ++a) {
                const double sx = 2 * kLoc[a][0] - 1, sy = 2 * kLoc[a][1] - 1;
                dN[a][0] = inv * sx * (1 + sy * eta) / 4.0;
                dN[a][1] = inv * sy * (1 + sx * xi) / 4.0;
            }
            double B[3][8] = {};
            for (int a = 0; a < 4; ++a) {
                B[0][2 * a] = dN[a][0];
                B[1][2 * a + 1] = dN[a][1];
                B[2][2 * a] = dN[a][1];
                B[2][2 * a + 1] = dN[a][0];
            }
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    double s = 0;
                    for (int p = 0; p < 3; ++p)
                        for (int q = 0; q < 3; ++q) s += B[p][i] * D[p][q] * B[q][j];
                    Ke[i * 8 + j] += s * detJ;
                }
        }
}

// hex8 isotropic elasticity, cube of side h, 2x2x2 Gauss; E = 1;
// strains (xx, yy, zz, xy, yz, xz) with engineering shears
void hex8_stiffness(double h, double nu, std::vector<double>& Ke) {
    const double lam = nu / ((1 + nu) * (1 - 2 * nu)), mu = 1.0 / (2 * (1 + nu));
    double D[6][6] = {};
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) D[i][j] = lam + (i == j ? 2 * mu : 0.0);
    D[3][3] = D[4][4] = D[5][5] = mu;
    Ke.assign(24 * 24, 0.0);
    const double g = 1.0 / std::sqrt(3.0);
    const double detJ = (h / 2) * (h / 2) * (h / 2), inv = 2.0 / h;
    for (int gx = -1; gx <= 1; gx += 2)
        for (int gy = -1; gy <= 1; gy += 2)
            for (int gz = -1; gz <= 1; gz += 2) {
                const double p[3] = {gx * g, gy * g, gz * g};
                double dN[8][3];
                for (int a = 0; a < 8; ++a) {
                    double s[3];
                    for (int d = 0; d < 3; ++d) s[d] = 2 * kLoc[a][d] - 1;
                    dN[a][0] = inv * s[0] * (1 + s[1] * p[1]) * (1 + s[2] * p[2]) / 8.0;
                    dN[a][1] = inv * s[1] * (1 + s[0] * p[0]) * (1 + s[2] * p[2]) / 8.0;
                    dN[a][2] = inv * s[2] * (1 + s[0] * p[0]) * (1 + s[1] * p[1]) / 8.0;
                }
                double B[6][24] = {};
                for (int a = 0; a < 8; ++a) {
                    B[0][3 * a] = dN[a][0];
                    B[1][3 * a + 1] = dN[a][1];
                    B[2][3 * a + 2] = dN[a][2];
                    B[3][3 * a] = dN[a][1];
                    B[3][3 * a + 1] = dN[a][0];
                    B[4][3 * a + 1] = dN[a][2];
                    B[4][3 * a + 2] = dN[a][1];
                    B[5][3 * a] = dN[a][2];
                    B[5][3 * a + 2] = dN[a][0];
                }
                for (int i = 0; i < 24; ++i)
                    for (int j = 0; j < 24; ++j) {
                        double s = 0;
                        for (int q = 0; q < 6; ++q) {
                            double t = 0;
                            for (int r = 0; r < 6; ++r) t += D[q][r] * B[r][j];
                            s += B[q][i] * t;
                        }
                        Ke[i * 24 + j] += s * detJ;
                    }
            }
}

struct Grid {
    const p2g_mesh* m;
    int64_t NX, NY, NZ;  // nodes per axis
    // free node (ix >= 1) -> reduced node index
    int64_t rnode(int64_t ix, int64_t iy, int64_t iz) const {
        return (iz * NY + iy) * m->nx + (ix - 1);
    }
    void coords(int64_t rn, int64_t& ix, int64_t& iy, int64_t& iz) const {
        ix = rn % m->nx + 1;
        const int64_t t = rn / m->nx;
        iy = t % NY;
        iz = t / NY;
    }
};

Grid grid_of(const p2g_mesh* m) {
    return Grid{m, m->nx + 1, m->ny + 1, m->dim == 3 ? m->nz + 1 : 1};
}

template <class F>
void parallel_rows(int64_t n, int nthreads, F&& f) {
    if (nthreads <= 0) nthreads = std::max(1u, std::thread::hardware_concurrency());
    nthreads = static_cast<int>(std::min<int64_t>(nthreads, std::max<int64_t>(1, n / 4096)));
    if (nthreads <= 1) {
        f(int64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    const int64_t chunk = (n + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        const int64_t a = t * chunk, b = std::min(n, a + chunk);
        if (a < b) th.emplace_back([&, a, b] { f(a, b); });
    }
    for (auto& x : th) x.join();
}

// neighbour node range along one axis for a node index i in [0, N)
inline void nb_range(int64_t i, int64_t N, int64_t lo_clip, int64_t& a, int64_t& b) {
    a = std::max<int64_t>(lo_clip, i - 1);
    b = std::min<int64_t>(N - 1, i + 1);
}

// ---- normal draws: mt19937_64 raw bits -> (0,1) -> inverse normal CDF
// (Acklam's published rational approximation, refined by one Halley step)
double inv_normal(double p) {
    static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                               -2.759285104469687e+02, 1.383577518672690e+02,
                               -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                               -1.556989798598866e+02, 6.680131188771972e+01,
                               -1.328068155288572e+01};
    static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                               -2.400758277161838e+00, -2.549732539343734e+00,
                               4.374664141464968e+00, 2.938163982698783e+00};
    static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                               2.445134137142996e+00, 3.754408661907416e+00};
    const double lo = 0.02425, hi = 1 - lo;
    double x;
    if (p < lo) {
        const double q = std::sqrt(-2 * std::log(p));
        x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    } else if (p > hi) {
        const double q = std::sqrt(-2 * std::log(1 - p));
        x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    } else {
        const double q = p - 0.5, r = q * q;
        x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
            (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
    }
    const double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;
    const double u = e * std::sqrt(2 * M_PI) * std::exp(x * x / 2);
    return x - u / (1 + x * u / 2);
}

// ---- symmetric eigenpairs by cyclic Jacobi rotations (small, deterministic)
void sym_eig(int n, std::vector<double> A, std::vector<double>& w, std::vector<double>& V) {
    V.assign((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0;
    double fro = 0;
    for (double x : A) fro += x * x;
    const double tol = 1e-15 * std::sqrt(fro);
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += A[(size_t)p * n + q] * A[(size_t)p * n + q];
        if (std::sqrt(2 * off) <= tol) break;
        for (int p = 0; p < n - 1; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A[(size_t)p * n + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double th = (A[(size_t)q * n + q] - A[(size_t)p * n + p]) / (2 * apq);
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1));
                const double cs = 1 / std::sqrt(t * t + 1), sn = t * cs;
                for (int k = 0; k < n; ++k) {
                    const double akp = A[(size_t)k * n + p], akq = A[(size_t)k * n + q];
                    A[(size_t)k * n + p] = cs * akp - sn * akq;
                    A[(size_t)k * n + q] = sn * akp + cs * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const double apk = A[(size_t)p * n + k], aqk = A[(size_t)q * n + k];
                    A[(size_t)p * n + k] = cs * apk - sn * aqk;
                    A[(size_t)q * n + k] = sn * apk + cs * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[(size_t)k * n + p], vkq = V[(size_t)k * n + q];
                    V[(size_t)k * n + p] = cs * vkp - sn * vkq;
                    V[(size_t)k * n + q] = sn * vkp + cs * vkq;
                }
            }
    }
    w.resize(n);
    for (int i = 0; i < n; ++i) w[i] = A[(size_t)i * n + i];
}

// 1D KL modes of exp(-(s-t)^2/(2 ell^2)) on [0, L]: P leading eigenpairs,
// eigenfunctions evaluated (Nystrom extension) at the points `xs`.
void kl_axis(double L, double ell, int quad, int P, const std::vector<double>& xs,
             std::vector<double>& lam, std::vector<double>& phi /*[P][xs]*/) {
    const int Q = quad;
    const double w = L / Q;
    std::vector<double> t(Q), A((size_t)Q * Q);
    for (int q = 0; q < Q; ++q) t[q] = (q + 0.5) * w;
    for (int i = 0; i < Q; ++i)
        for (int j = 0; j < Q; ++j) {
            const double d = t[i] - t[j];
            A[(size_t)i * Q + j] = w * std::exp(-d * d / (2 * ell * ell));
        }
    std::vector<double> ev, V;
    sym_eig(Q, A, ev, V);
    std::vector<int> order(Q);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return ev[a] > ev[b]; });
    P = std::min(P, Q);
    lam.resize(P);
    phi.assign((size_t)P * xs.size(), 0.0);
    for (int p = 0; p < P; ++p) {
        const int c = order[p];
        lam[p] = ev[c];
        // eigenfunction at quadrature points: v_q / sqrt(w); fix the sign with a
        // generic asymmetric weight so it does not depend on the solver
        double sgn = 0;
        for (int q = 0; q < Q; ++q) sgn += V[(size_t)q * Q + c] * (q + 1.0 + 0.1 * q * q);
        const double sg = sgn >= 0 ? 1.0 : -1.0;
        for (size_t e = 0; e < xs.size(); ++e) {
            // Nystrom: phi(x) = (1/lam) sum_q w C(x, t_q) phi(t_q)
            double s = 0;
            for (int q = 0; q < Q; ++q) {
                const double d = xs[e] - t[q];
                s += w * std::exp(-d * d / (2 * ell * ell)) * V[(size_t)q * Q + c] / std::sqrt(w);
            }
            phi[(size_t)p * xs.size() + e] = sg * s / ev[c];
        }
    }
}

struct KL {
    int M = 0;
    std::vector<double> lam;          // M
    std::vector<int> kx, ky, kz;      // per mode axis indices
    std::vector<double> px, py, pz;   // [P][n_axis centroids]
    int P = 0;
    int64_t nx = 0, ny = 0, nz = 1;
};

int build_kl(const p2g_mesh* m, int M, double ell, int quad, KL& kl) {
    if (M < 1 || ell <= 0 || quad < 8) return P2G_GEN_EINVAL;
    const int P = std::min(quad, M);
    kl.P = P;
    kl.M = M;
    kl.nx = m->nx;
    kl.ny = m->ny;
    kl.nz = m->dim == 3 ? m->nz : 1;
    std::vector<double> lx, ly, lz;
    auto cents = [&](int64_t ne, double h) {
        std::vector<double> c(ne);
        for (int64_t e = 0; e < ne; ++e) c[e] = (e + 0.5) * h;
        return c;
    };
    kl_axis(m->L[0], ell, quad, P, cents(m->nx, m->h), lx, kl.px);
    kl_axis(m->L[1], ell, quad, P, cents(m->ny, m->h), ly, kl.py);
    if (m->dim == 3) {
        kl_axis(m->L[2], ell, quad, P, cents(m->nz, m->h), lz, kl.pz);
    } else {
        lz = {1.0};
        kl.pz.assign(1, 1.0);
    }
    struct Cand {
        double l;
        int a, b, c;
    };
    std::vector<Cand> cand;
    for (int a = 0; a < (int)lx.size(); ++a)
        for (int b = 0; b < (int)ly.size(); ++b)
            for (int c = 0; c < (int)lz.size(); ++c) cand.push_back({lx[a] * ly[b] * lz[c], a, b, c});
    std::stable_sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) { return x.l > y.l; });
    if ((int)cand.size() < M) return P2G_GEN_EINVAL;
    kl.lam.resize(M);
    kl.kx.resize(M);
    kl.ky.resize(M);
    kl.kz.resize(M);
    for (int i = 0; i < M; ++i) {
        kl.lam[i] = cand[i].l;
        kl.kx[i] = cand[i].a;
        kl.ky[i] = cand[i].b;
        kl.kz[i] = cand[i].c;
    }
    return P2G_GEN_OK;
}

}  // namespace

namespace p2g {
bool mesh_desc(const p2g_mesh* m, MeshDesc& d) {
    if (!m) return false;
    d.dim = m->dim;
    d.ned = m->ned;
    d.nx = m->nx;
    d.ny = m->ny;
    d.nz = m->nz;
    d.n = m->n;
    d.nnz = m->nnz;
    d.nelem = m->nelem;
    d.Ke = m->Ke.data();
    d.rp = m->rp.data();
    return true;
}
}  // namespace p2g

extern "C" {

int p2g_mesh_create(int32_t dim, int64_t nx, int64_t ny, int64_t nz, double Lx, double Ly,
                    double Lz, double nu, p2g_mesh** out) {
    if (!out) return P2G_GEN_EINVAL;
    *out = nullptr;
    if (dim != 2 && dim != 3) return P2G_GEN_EINVAL;
    if (nx < 1 || ny < 1 || (dim == 3 && nz < 1)) return P2G_GEN_EINVAL;
    if (!(nu >= 0 && nu < 0.5)) return P2G_GEN_EINVAL;
    const double h = Lx / nx;
    if (std::fabs(Ly / ny - h) > 1e-12 * h || (dim == 3 && std::fabs(Lz / nz - h) > 1e-12 * h))
        return P2G_GEN_EINVAL;
    auto* m = new p2g_mesh();
    m->dim = dim;
    m->nx = nx;
    m->ny = ny;
    m->nz = dim == 3 ? nz : 1;
    m->L[0] = Lx;
    m->L[1] = Ly;
    m->L[2] = dim == 3 ? Lz : 1.0;
    m->h = h;
    m->nu = nu;
    m->nen = dim == 2 ? 4 : 8;
    m->ned = dim * m->nen;
    if (dim == 2)
        q4_stiffness(h, nu, m->Ke);
    else
        hex8_stiffness(h, nu, m->Ke);
    // exact symmetry (the quadrature sums round differently for (i,j), (j,i))
    for (int i = 0; i < m->ned; ++i)
        for (int j = i + 1; j < m->ned; ++j) {
            const double v = 0.5 * (m->Ke[i * m->ned + j] + m->Ke[j * m->ned + i]);
            m->Ke[i * m->ned + j] = m->Ke[j * m->ned + i] = v;
        }
    const Grid G = grid_of(m);
    const int64_t nfree_nodes = m->nx * G.NY * G.NZ;
    m->n = nfree_nodes * dim;
    m->nelem = m->nx * m->ny * m->nz;
    m->rp.assign(m->n + 1, 0);
    // row lengths: (# free neighbour nodes) * dim
    for (int64_t rn = 0; rn < nfree_nodes; ++rn) {
        int64_t ix, iy, iz;
        G.coords(rn, ix, iy, iz);
        int64_t ax, bx, ay, by, az, bz;
        nb_range(ix, G.NX, 1, ax, bx);
        nb_range(iy, G.NY, 0, ay, by);
        nb_range(iz, G.NZ, 0, az, bz);
        const int64_t cnt = (bx - ax + 1) * (by - ay + 1) * (bz - az + 1) * dim;
        for (int c = 0; c < dim; ++c) m->rp[rn * dim + c + 1] = cnt;
    }
    for (int64_t i = 0; i < m->n; ++i) m->rp[i + 1] += m->rp[i];
    m->nnz = static_cast<int64_t>(m->rp[m->n]);
    *out = m;
    return P2G_GEN_OK;
}

void p2g_mesh_destroy(p2g_mesh* m) { delete m; }

int p2g_mesh_info(const p2g_mesh* m, int64_t* n, int64_t* nnz, int64_t* nelem, int32_t* bs) {
    if (!m) return P2G_GEN_EINVAL;
    if (n) *n = m->n;
    if (nnz) *nnz = m->nnz;
    if (nelem) *nelem = m->nelem;
    if (bs) *bs = m->dim;
    return P2G_GEN_OK;
}

int p2g_mesh_pattern(const p2g_mesh* m, uint64_t* rp, uint64_t* ci) {
    if (!m || !rp || !ci) return P2G_GEN_EINVAL;
    std::memcpy(rp, m->rp.data(), sizeof(uint64_t) * (m->n + 1));
    const Grid G = grid_of(m);
    const int dim = m->dim;
    parallel_rows(m->n / dim, 0, [&](int64_t r0, int64_t r1) {
        for (int64_t rn = r0; rn < r1; ++rn) {
            int64_t ix, iy, iz;
            G.coords(rn, ix, iy, iz);
            int64_t ax, bx, ay, by, az, bz;
            nb_range(ix, G.NX, 1, ax, bx);
            nb_range(iy, G.NY, 0, ay, by);
            nb_range(iz, G.NZ, 0, az, bz);
            for (int c = 0; c < dim; ++c) {
                uint64_t w = m->rp[rn * dim + c];
                for (int64_t jz = az; jz <= bz; ++jz)
                    for (int64_t jy = ay; jy <= by; ++jy)
                        for (int64_t jx = ax; jx <= bx; ++jx) {
                            const int64_t cn = G.rnode(jx, jy, jz);
                            for (int d = 0; d < dim; ++d) ci[w++] = static_cast<uint64_t>(cn * dim + d);
                        }
            }
        }
    });
    return P2G_GEN_OK;
}

int p2g_mesh_pattern_range(const p2g_mesh* m, int64_t r0, int64_t r1, uint64_t* rp,
                           uint64_t* ci) {
    if (!m || !rp || r0 < 0 || r1 > m->n || r0 > r1 || r0 % m->dim || r1 % m->dim)
        return P2G_GEN_EINVAL;
    const uint64_t base = m->rp[r0];
    for (int64_t i = r0; i <= r1; ++i) rp[i - r0] = m->rp[i] - base;
    if (!ci) return P2G_GEN_OK;
    const Grid G = grid_of(m);
    const int dim = m->dim;
    parallel_rows((r1 - r0) / dim, 0, [&](int64_t a0, int64_t a1) {
        for (int64_t rn = r0 / dim + a0; rn < r0 / dim + a1; ++rn) {
            int64_t ix, iy, iz;
            G.coords(rn, ix, iy, iz);
            int64_t ax, bx, ay, by, az, bz;
            nb_range(ix, G.NX, 1, ax, bx);
            nb_range(iy, G.NY, 0, ay, by);
            nb_range(iz, G.NZ, 0, az, bz);
            for (int c = 0; c < dim; ++c) {
                uint64_t w = m->rp[rn * dim + c] - base;
                for (int64_t jz = az; jz <= bz; ++jz)
                    for (int64_t jy = ay; jy <= by; ++jy)
                        for (int64_t jx = ax; jx <= bx; ++jx) {
                            const int64_t cn = G.rnode(jx, jy, jz);
                            for (int d = 0; d < dim; ++d) ci[w++] = static_cast<uint64_t>(cn * dim + d);
                        }
            }
        }
    });
    return P2G_GEN_OK;
}

int p2g_mesh_node_colors(const p2g_mesh* m, int32_t* colors) {
    if (!m || !colors) return P2G_GEN_EINVAL;
    const Grid G = grid_of(m);
    const int64_t nn = m->n / m->dim;
    // parity classes, processed in the order p2g_set_pattern's colouring would
    // pick (order_colours): class coupling = common neighbours of adjacent
    // nodes, which depends on the parity difference only (Q4: edge 4,
    // diagonal 2; hex8: face 16, edge 10, corner 6)
    const int ncol = m->dim == 3 ? 8 : 4;
    std::vector<double> W((size_t)ncol * ncol, 0.0);
    for (int a = 0; a < ncol; ++a)
        for (int b = 0; b < ncol; ++b) {
            const int bits = __builtin_popcount(a ^ b);
            W[(size_t)a * ncol + b] = bits == 0 ? 0.0
                                      : m->dim == 3 ? (bits == 1 ? 16.0 : bits == 2 ? 10.0 : 6.0)
                                                    : (bits == 1 ? 4.0 : 2.0);
        }
    const std::vector<int32_t> rank = p2g::order_colours(ncol, W);
    for (int64_t rn = 0; rn < nn; ++rn) {
        int64_t ix, iy, iz;
        G.coords(rn, ix, iy, iz);
        colors[rn] = rank[(ix & 1) + 2 * (iy & 1) + (m->dim == 3 ? 4 * (iz & 1) : 0)];
    }
    return P2G_GEN_OK;
}

int p2g_mesh_rhs(const p2g_mesh* m, double* f) {
    if (!m || !f) return P2G_GEN_EINVAL;
    std::fill(f, f + m->n, 0.0);
    const Grid G = grid_of(m);
    const double h = m->h;
    if (m->dim == 2) {
        // unit downward traction on x = Lx: each edge segment gives h/2 to both ends
        for (int64_t ey = 0; ey < m->ny; ++ey)
            for (int64_t dy = 0; dy <= 1; ++dy) f[G.rnode(m->nx, ey + dy, 0) * 2 + 1] += -0.5 * h;
    } else {
        // traction (0,0,-1) on x = Lx: each face quad gives h^2/4 to its 4 nodes
        for (int64_t ez = 0; ez < m->nz; ++ez)
            for (int64_t ey = 0; ey < m->ny; ++ey)
                for (int64_t dz = 0; dz <= 1; ++dz)
                    for (int64_t dy = 0; dy <= 1; ++dy)
                        f[G.rnode(m->nx, ey + dy, ez + dz) * 3 + 2] += -0.25 * h * h;
    }
    return P2G_GEN_OK;
}

int p2g_mesh_element_stiffness(const p2g_mesh* m, double* Ke) {
    if (!m || !Ke) return P2G_GEN_EINVAL;
    std::memcpy(Ke, m->Ke.data(), sizeof(double) * m->Ke.size());
    return P2G_GEN_OK;
}

namespace {
// values of free rows [row0, row1) (node aligned) into values[b][stride],
// entry q of the range at values[b * stride + q - rp[row0]]
int assemble_rows(const p2g_mesh* m, int64_t B, const double* E, int64_t row0, int64_t row1,
                  double* values, int64_t stride, int32_t nthreads) {
    const Grid G = grid_of(m);
    const int dim = m->dim, ned = m->ned;
    const int64_t nx = m->nx, ny = m->ny, nz = m->nz, nnz = stride, nel = m->nelem;
    const int64_t vbase = static_cast<int64_t>(m->rp[row0]);
    parallel_rows((row1 - row0) / dim, nthreads, [&](int64_t a0, int64_t a1) {
        int64_t elist[8];
        int kidx[8][3][3];
        for (int64_t rn = row0 / dim + a0; rn < row0 / dim + a1; ++rn) {
            int64_t ix, iy, iz;
            G.coords(rn, ix, iy, iz);
            int64_t ax, bx, ay, by, az, bz;
            nb_range(ix, G.NX, 1, ax, bx);
            nb_range(iy, G.NY, 0, ay, by);
            nb_range(iz, G.NZ, 0, az, bz);
            int64_t slot = 0;  // column-node position within the row
            for (int64_t jz = az; jz <= bz; ++jz)
                for (int64_t jy = ay; jy <= by; ++jy)
                    for (int64_t jx = ax; jx <= bx; ++jx, ++slot) {
                        // elements shared by nodes i and j, ascending element id
                        int ne = 0;
                        const int64_t ex0 = std::max<int64_t>(std::max(ix, jx) - 1, 0),
                                      ex1 = std::min<int64_t>(std::min(ix, jx), nx - 1);
                        const int64_t ey0 = std::max<int64_t>(std::max(iy, jy) - 1, 0),
                                      ey1 = std::min<int64_t>(std::min(iy, jy), ny - 1);
                        int64_t ez0 = 0, ez1 = 0;
                        if (dim == 3) {
                            ez0 = std::max<int64_t>(std::max(iz, jz) - 1, 0);
                            ez1 = std::min<int64_t>(std::min(iz, jz), nz - 1);
                        }
                        for (int64_t ez = ez0; ez <= ez1; ++ez)
                            for (int64_t ey = ey0; ey <= ey1; ++ey)
                                for (int64_t ex = ex0; ex <= ex1; ++ex) {
                                    const int la = local_index(int(ix - ex), int(iy - ey), int(iz - ez));
                                    const int lb = local_index(int(jx - ex), int(jy - ey), int(jz - ez));
                                    elist[ne] = (ez * ny + ey) * nx + ex;
                                    for (int c = 0; c < dim; ++c)
                                        for (int d = 0; d < dim; ++d)
                                            kidx[ne][c][d] = (la * dim + c) * ned + lb * dim + d;
                                    ++ne;
                                }
                        for (int c = 0; c < dim; ++c) {
                            const int64_t row = rn * dim + c;
                            const int64_t base = static_cast<int64_t>(m->rp[row]) - vbase + slot * dim;
                            for (int d = 0; d < dim; ++d) {
                                for (int64_t b = 0; b < B; ++b) {
                                    const double* Eb = E + b * nel;
                                    double v = 0.0;
                                    for (int q = 0; q < ne; ++q) v += Eb[elist[q]] * m->Ke[kidx[q][c][d]];
                                    values[b * nnz + base + d] = v;
                                }
                            }
                        }
                    }
        }
    });
    return P2G_GEN_OK;
}
}  // namespace

int p2g_mesh_assemble(const p2g_mesh* m, int64_t B, const double* E, double* values,
                      int32_t nthreads) {
    if (!m || !E || !values || B < 1) return P2G_GEN_EINVAL;
    return assemble_rows(m, B, E, 0, m->n, values, m->nnz, nthreads);
}

int p2g_mesh_assemble_range(const p2g_mesh* m, int64_t B, const double* E, int64_t r0,
                            int64_t r1, double* values, int32_t nthreads) {
    if (!m || !E || !values || B < 1 || r0 < 0 || r1 > m->n || r0 > r1 || r0 % m->dim ||
        r1 % m->dim)
        return P2G_GEN_EINVAL;
    const int64_t stride = static_cast<int64_t>(m->rp[r1] - m->rp[r0]);
    if (r0 == r1) return P2G_GEN_OK;
    return assemble_rows(m, B, E, r0, r1, values, stride, nthreads);
}

int p2g_normal_draws(uint64_t seed, int64_t count, double* out) {
    if (!out || count < 0) return P2G_GEN_EINVAL;
    std::mt19937_64 eng(seed);
    for (int64_t i = 0; i < count; ++i) {
        const double u = (static_cast<double>(eng() >> 11) + 0.5) * 0x1.0p-53;
        out[i] = inv_normal(u);
    }
    return P2G_GEN_OK;
}

int p2g_kl_eigenvalues(const p2g_mesh* m, int32_t M, double ell, int32_t quad, double* lambda) {
    if (!m || !lambda) return P2G_GEN_EINVAL;
    KL kl;
    if (build_kl(m, M, ell, quad, kl) != P2G_GEN_OK) return P2G_GEN_EINVAL;
    std::memcpy(lambda, kl.lam.data(), sizeof(double) * M);
    return P2G_GEN_OK;
}

int p2g_kl_field(const p2g_mesh* m, int32_t M, double sigma, double ell, int32_t quad, int64_t B,
                 const uint64_t* seeds, double* E, double* xi) {
    if (!m || !seeds || !E || B < 1) return P2G_GEN_EINVAL;
    KL kl;
    if (build_kl(m, M, ell, quad, kl) != P2G_GEN_OK) return P2G_GEN_EINVAL;
    std::vector<double> xs((size_t)B * M);
    for (int64_t b = 0; b < B; ++b) p2g_normal_draws(seeds[b], M, xs.data() + b * M);
    if (xi) std::memcpy(xi, xs.data(), sizeof(double) * xs.size());
    const int64_t nx = kl.nx, ny = kl.ny, nz = kl.nz;
    const int64_t nel = nx * ny * nz;
    parallel_rows(nel, 0, [&](int64_t e0, int64_t e1) {
        for (int64_t e = e0; e < e1; ++e) {
            const int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
            for (int64_t b = 0; b < B; ++b) {
                double g = 0.0;
                for (int q = 0; q < M; ++q) {
                    const double ph = kl.px[(size_t)kl.kx[q] * nx + ex] *
                                      kl.py[(size_t)kl.ky[q] * ny + ey] *
                                      (m->dim == 3 ? kl.pz[(size_t)kl.kz[q] * nz + ez] : 1.0);
                    g += std::sqrt(kl.lam[q]) * ph * xs[b * M + q];
                }
                E[b * nel + e] = std::exp(sigma * g);
            }
        }
    });
    return P2G_GEN_OK;
}

}  // extern "C"
