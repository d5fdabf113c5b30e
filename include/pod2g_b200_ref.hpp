// pod2g_b200_ref.hpp -- the GPU POD-2G preconditioner as a plug-in of the
// REFERENCE's own solver interface: a subclass of pod2g::Preconditioner
// (/root/reference/proj/include/pod2g/krylov.hpp:14-19) with the constructor
// of pod2g::Pod2gPreconditioner (pod.hpp:259-263).  The reference's own
// pcg_solve (krylov.hpp:243-297, IterationTrace included), run_pcg_benchmark's
// "pod-2g" branch (bench.hpp:315-317) and run_monte_carlo (bench.hpp:418-420)
// take it unchanged; a maintainer's swap is the one class name
// (INTEGRATION.md).
//
// Requires the reference headers on the include path (-I proj/include, plus
// the nlohmann/json directory they include) and links libpod2g_b200.so.
//
// Contract (krylov.hpp:12-13): a fixed SPD operator, immutable after
// construction.  apply() is const and may be called from several threads on
// one instance: calls on one instance are serialised (one device handle);
// separate instances run concurrently (one handle, stream and device buffer
// set each), which is how parallel_for uses it (bench.hpp:290-330).
//
// Errors keep the reference's exception types: a singular coarse operator
// throws std::runtime_error from the constructor (DenseLu, dense_solve.hpp:
// 25-26); a zero smoother diagonal throws from apply (smoothers.hpp:41-43);
// dimension mismatches throw std::invalid_argument (require, types.hpp:15-17).
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "pod2g/krylov.hpp"
#include "pod2g/pod.hpp"
#include "pod2g_b200.h"

namespace pod2g_b200 {

class RefPod2gPreconditioner final : public pod2g::Preconditioner {
public:
    // Same arguments as pod2g::Pod2gPreconditioner (pod.hpp:261-263); the
    // trailing ones are the GPU's: dofs per node of the caller's numbering
    // (node colouring, D1; 1 = point colouring) and the device.
    RefPod2gPreconditioner(std::shared_ptr<const pod2g::CsrMatrix> K,
                           std::shared_ptr<const pod2g::PodBasis> basis, pod2g::index_t r1 = 1,
                           pod2g::index_t r2 = 1, int block_size = 1, int device = 0)
        : K_(std::move(K)), basis_(std::move(basis)) {
        pod2g::require(K_ && basis_, "RefPod2gPreconditioner: null matrix or basis");
        pod2g::require(K_->nrows == K_->ncols, "RefPod2gPreconditioner: matrix not square");
        pod2g::require(basis_->phi_r.nrows == K_->nrows,
                       "RefPod2gPreconditioner: basis dimension mismatch");
        p2g_handle* h = nullptr;
        if (p2g_create(device, &h) != P2G_OK)
            throw std::runtime_error("RefPod2gPreconditioner: no usable CUDA device");
        h_.reset(h);
        std::vector<uint64_t> rp(K_->row_offsets.begin(), K_->row_offsets.end());
        std::vector<uint64_t> ci(K_->col_indices.begin(), K_->col_indices.end());
        check(p2g_set_pattern(h, static_cast<int64_t>(K_->nrows), rp.data(), ci.data(), block_size),
              "set_pattern");
        check(p2g_set_values(h, 1, K_->values.data()), "set_values");
        check(p2g_set_basis(h, static_cast<int32_t>(basis_->rank), basis_->phi_r.data.data()),
              "set_basis");
        p2g_config cfg;
        p2g_config_default(&cfg);
        cfg.pre_sweeps = static_cast<int32_t>(r1);
        cfg.post_sweeps = static_cast<int32_t>(r2);
        int32_t st = P2G_OK;
        const int rc = p2g_setup(h, &cfg, &st);
        if (rc == P2G_EINVAL || rc == P2G_ECUDA || rc == P2G_ESTATE) check(rc, "setup");
        if (st == P2G_ESINGULAR)
            throw std::runtime_error("DenseLu: matrix is singular to working precision");
        setup_status_ = st;
    }

    // s = B r (pod.hpp:264-267: s := 0; cycle(r, s, adjoint_post = true))
    void apply(const pod2g::Vector& r, pod2g::Vector& s) const override {
        pod2g::require(r.size() == K_->nrows, "RefPod2gPreconditioner: size mismatch");
        if (setup_status_ == P2G_EZERODIAG)
            throw std::runtime_error("gauss_seidel_sweep: zero diagonal");
        s.resize(r.size());
        std::lock_guard<std::mutex> lock(mu_);
        check(p2g_precond_apply(h_.get(), r.data(), s.data()), "precond_apply");
    }

    std::string name() const override { return "pod2g"; }

    p2g_handle* handle() const { return h_.get(); }

private:
    void check(int st, const char* what) const {
        if (st == P2G_OK) return;
        const std::string msg = std::string("RefPod2gPreconditioner ") + what + ": " +
                                p2g_last_error(h_.get());
        if (st == P2G_EINVAL) throw std::invalid_argument(msg);
        throw std::runtime_error(msg);
    }
    struct Del {
        void operator()(p2g_handle* h) const { p2g_destroy(h); }
    };
    std::shared_ptr<const pod2g::CsrMatrix> K_;
    std::shared_ptr<const pod2g::PodBasis> basis_;
    std::unique_ptr<p2g_handle, Del> h_;
    int32_t setup_status_ = P2G_OK;
    mutable std::mutex mu_;
};

}  // namespace pod2g_b200
