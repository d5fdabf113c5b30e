// ref_plugin_test.cpp -- the GPU preconditioner inside the REFERENCE's own
// code, compiled against the unmodified reference headers
// (/root/reference/proj/include; built by `make -C oracle plugin` into
// oracle/_ref/, run by tests/test_gpu_api.py on the GPU box).
//
//  A. pod2g::pcg_solve (krylov.hpp:243-297, with an IterationTrace) driven by
//     pod2g_b200::RefPod2gPreconditioner : pod2g::Preconditioner, against the
//     same reference pcg_solve with the reference's Pod2gPreconditioner on the
//     colour-permuted system P K P^T (the GPU smoother's exact reference
//     equivalent, D1): iterations within 1, residual histories
//     within 1e-6, solution at matched iterations within 1e-8.
//  B. run_pcg_benchmark's "pod-2g" branch (bench.hpp:315-317, parallel_for
//     over 2 jobs) and run_monte_carlo (bench.hpp:418-420, surrogate warm
//     start) with the plug-in swapped in by the one class name, the bench
//     code itself untouched (the alias below stands in for a maintainer's
//     one-line edit); compared with the stock natural-order results.
//  C. The templated shim (include/pod2g_b200.hpp) on the real pod2g::CsrMatrix
//     / pod2g::PodBasis: pod2g_b200::pcg_solve and reduced_solve.
// Exit code 0 on success.
#include <cmath>
#include <cstdio>
#include <numeric>

#include "pod2g/pod.hpp"

#include "../../include/pod2g_b200_ref.hpp"
#include "../../include/pod2g_b200.hpp"

namespace pod2g {
using Pod2gPreconditionerGpu = pod2g_b200::RefPod2gPreconditioner;
}
#define Pod2gPreconditioner Pod2gPreconditionerGpu
#include "pod2g/bench.hpp"
#undef Pod2gPreconditioner

using namespace pod2g;

static int failures = 0;
#define CHECK(cond, ...)                         \
    do {                                         \
        if (!(cond)) {                           \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);            \
            std::printf("\n");                   \
            ++failures;                          \
        }                                        \
    } while (0)

static double rel_diff(const Vector& a, const Vector& b) {
    double num = 0, den = 0;
    for (index_t i = 0; i < a.size(); ++i) {
        num += (a[i] - b[i]) * (a[i] - b[i]);
        den += b[i] * b[i];
    }
    return std::sqrt(num / den);
}

// P K P^T: new row i = old row perm[i], columns ascending in the new numbering
static CsrMatrix permute(const CsrMatrix& K, const std::vector<int64_t>& perm) {
    const index_t n = K.nrows;
    std::vector<index_t> iperm(n);
    for (index_t i = 0; i < n; ++i) iperm[perm[i]] = i;
    CsrMatrix P(n, n);
    for (index_t i = 0; i < n; ++i) {
        const index_t o = perm[i];
        std::vector<std::pair<index_t, double>> row;
        for (index_t q = K.row_offsets[o]; q < K.row_offsets[o + 1]; ++q)
            row.emplace_back(iperm[K.col_indices[q]], K.values[q]);
        std::sort(row.begin(), row.end());
        for (auto& e : row) {
            P.col_indices.push_back(e.first);
            P.values.push_back(e.second);
        }
        P.row_offsets[i + 1] = P.col_indices.size();
    }
    P.symmetric_hint = K.symmetric_hint;
    return P;
}

int main() {
    const ParametricProblem prob = make_its_problem(16);
    OfflineConfig oc;
    oc.n_snapshots = 40;
    oc.training.epochs = 30;
    oc.jobs = 4;
    const OfflineArtifacts art = run_offline(prob, oc);
    // A and C: a richer coarse space than the 0.9999-energy basis (rank 1 here)
    auto basis = std::make_shared<const PodBasis>(
        compute_pod(art.snapshots.solutions, RankTarget{8}));
    std::printf("its16: offline basis rank %zu; A/C basis rank %zu\n", (size_t)art.basis.rank,
                (size_t)basis->rank);

    // ---------------------------------------------------------------- A
    {
        Rng sampler(11);
        const AssembledSystem sys = prob.assemble(sample_lognormal(prob.parameters, sampler));
        auto K = std::make_shared<const CsrMatrix>(sys.K);
        const pod2g_b200::RefPod2gPreconditioner gpu(K, basis, 1, 1);
        const Preconditioner& T = gpu;  // used through the reference's interface only
        const index_t n = K->nrows;
        std::vector<int64_t> perm(n);
        int32_t ncol = 0;
        std::vector<int64_t> offs(65);
        CHECK(p2g_get_permutation(gpu.handle(), perm.data(), &ncol, offs.data(), 64) == P2G_OK,
              "permutation");
        auto PK = std::make_shared<const CsrMatrix>(permute(*K, perm));
        auto PB = std::make_shared<PodBasis>(*basis);
        for (index_t i = 0; i < n; ++i)
            for (index_t a = 0; a < basis->rank; ++a)
                PB->phi_r.data[i * basis->rank + a] = basis->phi_r.data[perm[i] * basis->rank + a];
        Vector Pf(n);
        for (index_t i = 0; i < n; ++i) Pf[i] = sys.f[perm[i]];
        const Pod2gPreconditioner stock(PK, PB, 1, 1);  // the reference's own class
        IterationTrace trace;
        auto [u_g, rep_g] = pcg_solve(*K, sys.f, T, {}, 1e-8, 5000, &trace);
        auto [u_r, rep_r] = pcg_solve(*PK, Pf, stock, {}, 1e-8, 5000);
        CHECK(rep_g.converged && rep_r.converged, "converged %d %d", rep_g.converged, rep_r.converged);
        const long dk = (long)rep_g.cycles - (long)rep_r.cycles;
        CHECK(std::labs(dk) <= 1, "iterations gpu %zu ref %zu", (size_t)rep_g.cycles,
              (size_t)rep_r.cycles);
        const index_t m = std::min(rep_g.residual_history.size(), rep_r.residual_history.size());
        double hmax = 0;
        for (index_t i = 0; i < m; ++i)
            hmax = std::max(hmax, std::fabs(rep_g.residual_history[i] - rep_r.residual_history[i]) /
                                      rep_r.residual_history[i]);
        CHECK(hmax <= 1e-6, "history rel diff %.3e", hmax);
        CHECK(!trace.residuals.empty() && trace.residuals[0].size() == n, "trace");
        // matched iteration count
        const index_t it = rep_g.cycles;
        auto [u_gm, r1] = pcg_solve(*K, sys.f, T, {}, 0.0, it);
        auto [u_rm, r2] = pcg_solve(*PK, Pf, stock, {}, 0.0, it);
        Vector u_back(n);
        for (index_t i = 0; i < n; ++i) u_back[i] = u_gm[perm[i]];
        const double ex = rel_diff(u_back, u_rm);
        CHECK(ex <= 1e-8, "matched-iteration x rel diff %.3e", ex);
        // natural order (the reference default) beside it
        const Pod2gPreconditioner natural(K, basis, 1, 1);
        auto [u_n, rep_n] = pcg_solve(*K, sys.f, natural, {}, 1e-8, 5000);
        std::printf("A: reference pcg_solve + GPU plug-in: %zu iterations (reference on P K P^T: "
                    "%zu, natural order: %zu); history %.1e, matched x %.1e\n",
                    (size_t)rep_g.cycles, (size_t)rep_r.cycles, (size_t)rep_n.cycles, hmax, ex);
    }

    // ---------------------------------------------------------------- B
    {
        BenchmarkConfig cfg;
        cfg.tolerances = {1e-6, 1e-8};
        cfg.n_test = 6;
        cfg.jobs = 2;
        const BenchmarkResult res = run_pcg_benchmark(prob, art, cfg, {"pod-2g"}, "pod-2g");
        // stock natural-order counts of the same samples (bench.hpp:275-279 sampler)
        Rng sampler(cfg.seed);
        std::vector<double> stock(cfg.n_test);
        auto art_basis = std::make_shared<const PodBasis>(art.basis);
        for (index_t i = 0; i < cfg.n_test; ++i) {
            const AssembledSystem sys = prob.assemble(sample_lognormal(prob.parameters, sampler));
            auto K = std::make_shared<const CsrMatrix>(sys.K);
            const Pod2gPreconditioner natural(K, art_basis, 1, 1);
            stock[i] = (double)pcg_solve(sys.K, sys.f, natural, {}, 1e-8, 5000).second.cycles;
        }
        const double stock_mean = std::accumulate(stock.begin(), stock.end(), 0.0) / cfg.n_test;
        for (const auto& c : res.cells) {
            CHECK(c.failures == 0, "run_pcg_benchmark %s eps %g: %zu failures", c.solver.c_str(),
                  c.epsilon, (size_t)c.failures);
            for (index_t i = 0; i < cfg.n_test; ++i)
                CHECK(c.final_residuals[i] <= c.epsilon, "final residual %g", c.final_residuals[i]);
        }
        const BenchmarkCell* c8 = res.find("pod-2g", 1e-8);
        CHECK(c8 && c8->mean_cycles >= 0.9 * stock_mean && c8->mean_cycles <= 1.6 * stock_mean,
              "pod-2g mean cycles %g vs natural %g", c8 ? c8->mean_cycles : -1.0, stock_mean);
        std::printf("B: run_pcg_benchmark pod-2g (GPU plug-in, 2 jobs): mean cycles %.1f at 1e-8 "
                    "(stock natural order %.1f), 0 failures\n", c8 ? c8->mean_cycles : -1.0,
                    stock_mean);

        const index_t n_mc = 100;
        const MonteCarloResult mc = run_monte_carlo(prob, art, n_mc, 99, 1e-6, 2);
        Rng s2(99);
        double ref_mean = 0;
        for (index_t i = 0; i < n_mc; ++i) {
            const Vector th = sample_lognormal(prob.parameters, s2);
            const AssembledSystem sys = prob.assemble(th);
            auto K = std::make_shared<const CsrMatrix>(sys.K);
            const Pod2gPreconditioner natural(K, art_basis, 1, 1);
            auto [u, rep] = pcg_solve(sys.K, sys.f, natural, predict(art.model, th), 1e-6, 100000);
            ref_mean += detail::extract_qoi(prob, sys, u) / n_mc;
        }
        const double dq = std::fabs(mc.mean - ref_mean) / std::fabs(ref_mean);
        CHECK(dq <= 1e-4, "run_monte_carlo mean QoI %.10g vs stock %.10g", mc.mean, ref_mean);
        std::printf("B: run_monte_carlo (GPU plug-in, surrogate warm start, 100 samples): mean QoI "
                    "%.8g (stock %.8g, rel %.1e)\n", mc.mean, ref_mean, dq);
    }

    // ---------------------------------------------------------------- C
    {
        Rng sampler(5);
        const AssembledSystem sys = prob.assemble(sample_lognormal(prob.parameters, sampler));
        auto K = std::make_shared<const CsrMatrix>(sys.K);
        const pod2g_b200::Pod2gPreconditioner<CsrMatrix, PodBasis> T(K, basis, 1, 1);
        auto [u, rep] = pod2g_b200::pcg_solve(*K, sys.f, T, {}, 1e-8, 5000);
        Vector r;
        residual(*K, sys.f, u, r);
        const double rel = norm2(r) / norm2(sys.f);
        CHECK(rep.converged && rel <= 1.01e-8, "shim pcg_solve rel %g", rel);
        const Vector x0 = pod2g_b200::reduced_solve(*K, sys.f, *basis);
        const Vector x0_ref = reduced_solve(*K, sys.f, *basis).first;
        const double dx = rel_diff(x0, x0_ref);
        CHECK(dx <= 1e-10, "shim reduced_solve %.3e", dx);
        std::printf("C: shim on pod2g::CsrMatrix/PodBasis: %zu iterations, true rel %.2e; "
                    "reduced_solve %.1e\n", (size_t)rep.cycles, rel, dx);
    }
    std::printf(failures ? "ref_plugin_test: %d FAILURES\n" : "ref_plugin_test: ok\n", failures);
    return failures ? 1 : 0;
}
