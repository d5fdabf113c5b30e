// drop_in_example.cpp -- the reference's call sequence, unchanged except for
// the namespace of the solver entry points:
//   auto T = Pod2gPreconditioner(K, basis, 1, 1);  u = pcg_solve(K, f, T, {}, tol, max_iter)
// The structs below carry the reference's field names (core/csr.hpp:14-59,
// core/types.hpp:20-50, pod.hpp:19-25) so the templated shim reads them the
// same way it reads pod2g::CsrMatrix / pod2g::PodBasis.  Exit code 0 on success.
#include <cmath>
#include <cstdio>
#include <memory>
#include <vector>

#include "../../include/pod2g_b200.hpp"

struct CsrMatrix {
    std::size_t nrows = 0, ncols = 0;
    std::vector<std::size_t> row_offsets, col_indices;
    std::vector<double> values;
};
struct DenseMatrix {
    std::size_t nrows = 0, ncols = 0;
    std::vector<double> data;
};
struct PodBasis {
    DenseMatrix phi_r;
    std::size_t rank = 0;
};

int main() {
    // 2D Laplacian on an m x m grid (5-point), SPD
    const std::size_t m = 48, n = m * m;
    auto K = std::make_shared<CsrMatrix>();
    K->nrows = K->ncols = n;
    K->row_offsets.push_back(0);
    for (std::size_t i = 0; i < n; ++i) {
        const std::size_t x = i % m, y = i / m;
        auto add = [&](std::size_t j, double v) { K->col_indices.push_back(j); K->values.push_back(v); };
        if (y > 0) add(i - m, -1.0);
        if (x > 0) add(i - 1, -1.0);
        add(i, 4.0);
        if (x + 1 < m) add(i + 1, -1.0);
        if (y + 1 < m) add(i + m, -1.0);
        K->row_offsets.push_back(K->values.size());
    }
    // basis: two smooth modes, orthonormalised
    auto basis = std::make_shared<PodBasis>();
    basis->rank = 2;
    basis->phi_r.nrows = n;
    basis->phi_r.ncols = 2;
    basis->phi_r.data.resize(2 * n);
    double n0 = 0, n1 = 0, d = 0;
    for (std::size_t i = 0; i < n; ++i) {
        const double x = (i % m + 1.0) / (m + 1), y = (i / m + 1.0) / (m + 1);
        basis->phi_r.data[2 * i] = std::sin(M_PI * x) * std::sin(M_PI * y);
        basis->phi_r.data[2 * i + 1] = std::sin(2 * M_PI * x) * std::sin(M_PI * y);
    }
    for (std::size_t i = 0; i < n; ++i) n0 += basis->phi_r.data[2 * i] * basis->phi_r.data[2 * i];
    for (std::size_t i = 0; i < n; ++i) basis->phi_r.data[2 * i] /= std::sqrt(n0);
    for (std::size_t i = 0; i < n; ++i) d += basis->phi_r.data[2 * i] * basis->phi_r.data[2 * i + 1];
    for (std::size_t i = 0; i < n; ++i) basis->phi_r.data[2 * i + 1] -= d * basis->phi_r.data[2 * i];
    for (std::size_t i = 0; i < n; ++i) n1 += basis->phi_r.data[2 * i + 1] * basis->phi_r.data[2 * i + 1];
    for (std::size_t i = 0; i < n; ++i) basis->phi_r.data[2 * i + 1] /= std::sqrt(n1);
    std::vector<double> f(n, 1.0);

    using namespace pod2g_b200;
    Pod2gPreconditioner<CsrMatrix, PodBasis> T(K, basis, 1, 1);
    auto [u, rep] = pcg_solve(*K, f, T, {}, 1e-10, 5000);
    // true residual
    double rn = 0, fn = 0;
    for (std::size_t i = 0; i < n; ++i) {
        double s = 0;
        for (std::size_t k = K->row_offsets[i]; k < K->row_offsets[i + 1]; ++k)
            s += K->values[k] * u[K->col_indices[k]];
        rn += (f[i] - s) * (f[i] - s);
        fn += f[i] * f[i];
    }
    const double rel = std::sqrt(rn / fn);
    std::printf("pcg_solve(pod2g on GPU): converged=%d cycles=%zu history=%zu true_rel=%.3e name=%s\n",
                rep.converged, rep.cycles, rep.residual_history.size(), rel, T.name().c_str());
    auto x0 = reduced_solve(*K, f, *basis);
    bool threw = false;
    try {
        pcg_solve(*K, std::vector<double>(n + 1, 1.0), T, {}, 1e-8, 10);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    return (rep.converged && rel < 2e-10 && x0.size() == n && threw) ? 0 : 1;
}
