// pod2g_b200.hpp -- header-only C++ shim over the C-ABI (pod2g_b200.h) with
// the reference's solver interface, so reference-style callers swap in the
// GPU path with a namespace change:
//
//   reference (/root/reference/proj/include/pod2g/)          this shim
//   Pod2gPreconditioner(K, basis, r1, r2)  pod.hpp:261-263    pod2g_b200::Pod2gPreconditioner
//   Preconditioner::apply(r, s) / name()   krylov.hpp:14-19   same
//   pcg_solve(K, f, T, u0, delta, max_iter) krylov.hpp:243-297 pod2g_b200::pcg_solve
//   reduced_solve(K, f, basis)             pod.hpp:167-179    pod2g_b200::reduced_solve
//   SolveReport                            core/report.hpp     pod2g_b200::SolveReport
//
// The matrix and basis types are template parameters read by field name
// (CsrMatrix::nrows/row_offsets/col_indices/values, PodBasis::phi_r.{nrows,
// data}/rank), i.e. exactly the reference's own structs work unchanged.
// Errors keep the reference's exception split: std::invalid_argument for
// P2G_EINVAL (require(), core/types.hpp:15-17), std::runtime_error otherwise.
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pod2g_b200.h"

namespace pod2g_b200 {

struct SolveReport {
    bool converged = false;
    std::size_t cycles = 0;
    std::vector<double> residual_history;
    double wall_time_s = 0.0;
    double final_residual() const {
        return residual_history.empty() ? 0.0 / 0.0 : residual_history.back();
    }
};

inline void throw_status(int st, const std::string& msg) {
    if (st == P2G_OK) return;
    if (st == P2G_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// RAII owner of one handle.
class Handle {
public:
    explicit Handle(int device = 0) {
        p2g_handle* h = nullptr;
        const int st = p2g_create(device, &h);
        if (st != P2G_OK) throw std::runtime_error("p2g_create: no usable CUDA device");
        h_.reset(h);
    }
    p2g_handle* get() const { return h_.get(); }
    void check(int st, const char* what) const {
        if (st != P2G_OK) throw_status(st, std::string(what) + ": " + p2g_last_error(h_.get()));
    }

private:
    struct Del {
        void operator()(p2g_handle* h) const { p2g_destroy(h); }
    };
    std::unique_ptr<p2g_handle, Del> h_;
};

template <class Csr>
inline void upload_pattern(const Handle& h, const Csr& K, int block_size) {
    if (K.nrows != K.ncols) throw std::invalid_argument("pod2g_b200: matrix not square");
    std::vector<uint64_t> rp(K.row_offsets.begin(), K.row_offsets.end());
    std::vector<uint64_t> ci(K.col_indices.begin(), K.col_indices.end());
    h.check(p2g_set_pattern(h.get(), static_cast<int64_t>(K.nrows), rp.data(), ci.data(),
                            block_size),
            "set_pattern");
}

// Pod2gPreconditioner (pod.hpp:259-274) on the GPU.  The constructor builds
// A_c = Phi^T K Phi and its factor (Pod2gOperator ctor, pod.hpp:186-189).
// The smoother runs in node-colour order (D1); block_size = dofs
// per node of the caller's numbering (1 = point colouring).
template <class Csr, class Basis>
class Pod2gPreconditioner {
public:
    Pod2gPreconditioner(std::shared_ptr<const Csr> K, std::shared_ptr<const Basis> basis,
                        std::size_t r1 = 1, std::size_t r2 = 1, int block_size = 1,
                        int device = 0)
        : K_(std::move(K)), basis_(std::move(basis)), h_(device) {
        upload_pattern(h_, *K_, block_size);
        h_.check(p2g_set_values(h_.get(), 1, K_->values.data()), "set_values");
        if (basis_->phi_r.nrows != K_->nrows)
            throw std::invalid_argument("Pod2gPreconditioner: basis dimension mismatch");
        h_.check(p2g_set_basis(h_.get(), static_cast<int32_t>(basis_->rank),
                               basis_->phi_r.data.data()),
                 "set_basis");
        p2g_config cfg;
        p2g_config_default(&cfg);
        cfg.pre_sweeps = static_cast<int32_t>(r1);
        cfg.post_sweeps = static_cast<int32_t>(r2);
        int32_t st = P2G_OK;
        const int rc = p2g_setup(h_.get(), &cfg, &st);
        if (rc == P2G_EINVAL || rc == P2G_ECUDA || rc == P2G_ESTATE) h_.check(rc, "setup");
        if (st == P2G_ESINGULAR)
            throw std::runtime_error("DenseLu: matrix is singular to working precision");
        setup_status_ = st;
    }

    void apply(const std::vector<double>& r, std::vector<double>& s) const {
        if (setup_status_ == P2G_EZERODIAG) throw std::runtime_error("gauss_seidel_sweep: zero diagonal");
        if (r.size() != K_->nrows) throw std::invalid_argument("Pod2gPreconditioner: size mismatch");
        s.resize(r.size());
        h_.check(p2g_precond_apply(h_.get(), r.data(), s.data()), "precond_apply");
    }
    std::string name() const { return "pod2g"; }

    const Csr& matrix() const { return *K_; }
    p2g_handle* handle() const { return h_.get(); }

private:
    std::shared_ptr<const Csr> K_;
    std::shared_ptr<const Basis> basis_;
    Handle h_;
    int32_t setup_status_ = P2G_OK;
};

// pcg_solve (krylov.hpp:243-297) with the GPU preconditioner built on K.
template <class Csr, class Basis>
std::pair<std::vector<double>, SolveReport> pcg_solve(const Csr& K, const std::vector<double>& f,
                                                      const Pod2gPreconditioner<Csr, Basis>& T,
                                                      std::vector<double> u0, double delta,
                                                      std::size_t max_iter) {
    if (K.nrows != K.ncols || f.size() != K.nrows)
        throw std::invalid_argument("pcg_solve: dimension mismatch");
    if (!u0.empty() && u0.size() != K.nrows)
        throw std::invalid_argument("pcg_solve: initial guess dimension mismatch");
    if (&T.matrix() != &K)
        throw std::invalid_argument("pcg_solve: preconditioner built on another matrix");
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<double> u(K.nrows);
    const int64_t cap = static_cast<int64_t>(max_iter) + 1;
    std::vector<double> hist(static_cast<std::size_t>(cap));
    int64_t it = 0;
    int32_t conv = 0, st = 0;
    const int rc = p2g_solve(T.handle(), f.data(), u0.empty() ? nullptr : u0.data(),
                             u0.empty() ? P2G_X0_ZERO : P2G_X0_GIVEN, delta,
                             static_cast<int64_t>(max_iter), u.data(), &it, &conv, &st,
                             hist.data(), cap);
    if (rc == P2G_EINVAL || rc == P2G_ECUDA || rc == P2G_ESTATE)
        throw_status(rc, std::string("pcg_solve: ") + p2g_last_error(T.handle()));
    switch (st) {
        case P2G_OK: break;
        case P2G_EBREAKDOWN:
            throw std::runtime_error("pcg_solve: breakdown (matrix or preconditioner not SPD)");
        case P2G_ENONFINITE: throw std::runtime_error("pcg_solve: non-finite entries in solution");
        case P2G_ESINGULAR: throw std::runtime_error("DenseLu: matrix is singular to working precision");
        case P2G_EZERODIAG: throw std::runtime_error("gauss_seidel_sweep: zero diagonal");
        default: throw std::runtime_error("pcg_solve: failed");
    }
    SolveReport rep;
    rep.converged = conv != 0;
    rep.cycles = static_cast<std::size_t>(it);
    rep.residual_history.assign(hist.begin(), hist.begin() + std::min<int64_t>(it + 1, cap));
    rep.wall_time_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return {std::move(u), std::move(rep)};
}

// reduced_solve (pod.hpp:167-179): x0 = Phi (Phi^T K Phi)^{-1} Phi^T f.
template <class Csr, class Basis>
std::vector<double> reduced_solve(const Csr& K, const std::vector<double>& f, const Basis& basis,
                                  int device = 0) {
    if (f.size() != K.nrows) throw std::invalid_argument("reduced_solve: dimension mismatch");
    Handle h(device);
    upload_pattern(h, K, 1);
    h.check(p2g_set_values(h.get(), 1, K.values.data()), "set_values");
    h.check(p2g_set_basis(h.get(), static_cast<int32_t>(basis.rank), basis.phi_r.data.data()),
            "set_basis");
    int32_t st = P2G_OK;
    const int rc = p2g_setup(h.get(), nullptr, &st);
    if (rc == P2G_EINVAL || rc == P2G_ECUDA || rc == P2G_ESTATE) h.check(rc, "setup");
    if (st == P2G_ESINGULAR)
        throw std::runtime_error("reduced_solve: reduced operator is singular for this basis");
    std::vector<double> x0(K.nrows);
    h.check(p2g_initial_guess(h.get(), f.data(), x0.data()), "initial_guess");
    return x0;
}

// Batched drop-in for the reference's per-instance loop (bench.hpp:290-330):
// B matrices sharing one pattern (values only differ) solved together.
template <class Csr, class Basis>
std::vector<std::pair<std::vector<double>, SolveReport>> pcg_solve_batch(
    const std::vector<const Csr*>& Ks, const std::vector<std::vector<double>>& fs,
    const Basis& basis, double delta, std::size_t max_iter, bool reduced_x0 = true,
    int block_size = 1, int device = 0) {
    if (Ks.empty() || Ks.size() != fs.size())
        throw std::invalid_argument("pcg_solve_batch: empty or mismatched batch");
    const std::size_t n = Ks[0]->nrows, nnz = Ks[0]->values.size(), B = Ks.size();
    Handle h(device);
    h.check(p2g_set_batch_hint(h.get(), static_cast<int64_t>(B)), "set_batch_hint");
    upload_pattern(h, *Ks[0], block_size);
    std::vector<double> vals(B * nnz), F(B * n);
    for (std::size_t b = 0; b < B; ++b) {
        if (Ks[b]->values.size() != nnz || fs[b].size() != n)
            throw std::invalid_argument("pcg_solve_batch: instances must share the pattern");
        std::copy(Ks[b]->values.begin(), Ks[b]->values.end(), vals.begin() + b * nnz);
        std::copy(fs[b].begin(), fs[b].end(), F.begin() + b * n);
    }
    h.check(p2g_set_values(h.get(), static_cast<int32_t>(B), vals.data()), "set_values");
    h.check(p2g_set_basis(h.get(), static_cast<int32_t>(basis.rank), basis.phi_r.data.data()),
            "set_basis");
    std::vector<int32_t> sst(B);
    const int src = p2g_setup(h.get(), nullptr, sst.data());
    if (src == P2G_EINVAL || src == P2G_ECUDA || src == P2G_ESTATE) h.check(src, "setup");
    const int64_t cap = static_cast<int64_t>(max_iter) + 1;
    std::vector<double> X(B * n), hist(B * static_cast<std::size_t>(cap));
    std::vector<int64_t> it(B);
    std::vector<int32_t> conv(B), st(B);
    const auto t0 = std::chrono::steady_clock::now();
    const int rc = p2g_solve(h.get(), F.data(), nullptr, reduced_x0 ? P2G_X0_REDUCED : P2G_X0_ZERO,
                             delta, static_cast<int64_t>(max_iter), X.data(), it.data(),
                             conv.data(), st.data(), hist.data(), cap);
    // per-instance statuses come back in st[]; a call-level failure (EINVAL, ECUDA e.g. OOM,
    // ESTATE) leaves X unwritten and must not pass as an all-zero "solution"
    if (rc == P2G_EINVAL || rc == P2G_ECUDA || rc == P2G_ESTATE) h.check(rc, "pcg_solve_batch");
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<std::pair<std::vector<double>, SolveReport>> out;
    for (std::size_t b = 0; b < B; ++b) {
        if (st[b] != P2G_OK)
            throw std::runtime_error("pcg_solve_batch: instance " + std::to_string(b) + ": " +
                                     p2g_status_string(st[b]));
        SolveReport rep;
        rep.converged = conv[b] != 0;
        rep.cycles = static_cast<std::size_t>(it[b]);
        const double* hb = hist.data() + b * static_cast<std::size_t>(cap);
        rep.residual_history.assign(hb, hb + std::min<int64_t>(it[b] + 1, cap));
        rep.wall_time_s = wall;
        out.emplace_back(std::vector<double>(X.begin() + b * n, X.begin() + (b + 1) * n),
                         std::move(rep));
    }
    return out;
}

}  // namespace pod2g_b200
