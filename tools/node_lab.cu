// node_lab.cu -- library row kernels vs node-blocked kernels on the c2 layout:
// time one SpMV and one backward / forward GS colour phase, check bitwise equality.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include "../include/pod2g_b200.h"
#include "../include/pod2g_gen.h"
#include "../paper_2207_02543_b200/csrc/p2g_kernels.cuh"
using namespace p2g;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

template <class F> float timeit(F f, int reps = 20) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); CK(cudaDeviceSynchronize());
    cudaEventRecord(a); for (int r = 0; r < reps; ++r) f(); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}

int main(int argc, char** argv) {
    const int dim = argc > 1 ? atoi(argv[1]) : 2;
    const int nx = argc > 2 ? atoi(argv[2]) : 256;
    const int Bp = argc > 3 ? atoi(argv[3]) : 64;
    p2g_mesh* mm;
    if (dim == 2) p2g_mesh_create(2, nx, nx / 2, 1, 2.0, 1.0, 1.0, 0.3, &mm);
    else p2g_mesh_create(3, nx, nx, nx, 1.0, 1.0, 1.0, 0.3, &mm);
    int64_t n, nnz, ne; int32_t bs;
    p2g_mesh_info(mm, &n, &nnz, &ne, &bs);
    std::vector<uint64_t> rp(n + 1), ci(nnz);
    p2g_mesh_pattern(mm, rp.data(), ci.data());
    std::vector<int64_t> perm(n), offs(65); int32_t nc; char err[256];
    p2g_analyze_pattern(n, rp.data(), ci.data(), bs, perm.data(), &nc, offs.data(), 65, err, 256);
    std::vector<int64_t> iperm(n);
    for (int64_t i = 0; i < n; ++i) iperm[perm[i]] = i;
    std::vector<int> prp(n + 1, 0), pci(nnz), dpos(n);
    for (int64_t i = 0; i < n; ++i) {
        std::vector<int> cols;
        for (uint64_t k = rp[perm[i]]; k < rp[perm[i] + 1]; ++k) cols.push_back((int)iperm[ci[k]]);
        std::sort(cols.begin(), cols.end());
        for (size_t q = 0; q < cols.size(); ++q) { pci[prp[i] + q] = cols[q]; if (cols[q] == i) dpos[i] = prp[i] + (int)q; }
        prp[i + 1] = prp[i] + (int)cols.size();
    }
    printf("dim=%d n=%ld nnz=%ld colours=%d Bp=%d\n", dim, (long)n, (long)nnz, nc, Bp);
    int *d_rp, *d_ci, *d_dp, *d_act; double *d_v, *d_x, *d_y, *d_y2, *d_f, *d_part;
    CK(cudaMalloc(&d_rp, 4 * (n + 1))); CK(cudaMalloc(&d_ci, 4 * nnz)); CK(cudaMalloc(&d_dp, 4 * n));
    CK(cudaMalloc(&d_act, 4 * Bp)); CK(cudaMalloc(&d_v, 8 * nnz * Bp));
    for (double** p : {&d_x, &d_y, &d_y2, &d_f}) CK(cudaMalloc(p, 8 * n * Bp));
    CK(cudaMalloc(&d_part, 8 * 4096 * Bp));
    CK(cudaMemcpy(d_rp, prp.data(), 4 * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, pci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_dp, dpos.data(), 4 * n, cudaMemcpyHostToDevice));
    std::vector<int> act(Bp, 1); CK(cudaMemcpy(d_act, act.data(), 4 * Bp, cudaMemcpyHostToDevice));
    {
        std::mt19937_64 g(1);
        std::vector<double> h(nnz * Bp);
        for (auto& v : h) v = 0.1 + (g() >> 11) * 0x1.0p-53;
        for (int64_t i = 0; i < n; ++i) for (int b = 0; b < Bp; ++b) h[(size_t)dpos[i] * Bp + b] += 40.0;
        CK(cudaMemcpy(d_v, h.data(), 8 * h.size(), cudaMemcpyHostToDevice));
        std::vector<double> hx(n * Bp);
        for (auto& v : hx) v = (g() >> 11) * 0x1.0p-53;
        CK(cudaMemcpy(d_x, hx.data(), 8 * hx.size(), cudaMemcpyHostToDevice));
        for (auto& v : hx) v = (g() >> 11) * 0x1.0p-53;
        CK(cudaMemcpy(d_f, hx.data(), 8 * hx.size(), cudaMemcpyHostToDevice));
    }
    Mat A{(int)n, bs, d_rp, d_ci, d_dp, d_v, Bp};
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double spmv_bytes = 8.0 * nnz * Bp + 4.0 * nnz + 4.0 * (n + 1) + 16.0 * n * Bp;
    auto cmp = [&](const char* what) {
        std::vector<double> a(n * Bp), b(n * Bp);
        CK(cudaMemcpy(a.data(), d_y, 8 * a.size(), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(b.data(), d_y2, 8 * b.size(), cudaMemcpyDeviceToHost));
        size_t diff = 0; for (size_t i = 0; i < a.size(); ++i) diff += a[i] != b[i];
        printf("   %s: %zu differing entries\n", what, diff);
    };
    const int nn = (int)(n / bs);
    auto G = [&](int units, int rows_per_block, int cap_per_sm) {
        int g = std::min((units + rows_per_block - 1) / rows_per_block, sms * cap_per_sm);
        return (g + 7) / 8 * 8;
    };
    using S64 = ShB64;
    using S32 = ShB32;
#define REPORT(name, ms, bytes) printf("%-44s %8.1f us %7.0f GB/s\n", name, (ms) * 1e3, (bytes) / ((ms) * 1e-3) / 1e9)
    // ---- SpMV
    {
        float ms = timeit([&] { k_spmv<S64, true><<<dim3(G(nn, 8, 8), Bp / 64), 256>>>(A, d_x, d_y, d_act, d_part); });
        REPORT("row spmv V2", ms, spmv_bytes);
#define SPN(SH, CH, MB) { float t = timeit([&] { k_spmv_node<SH, 2, CH, true, MB><<<dim3(G(nn, 8, 8), Bp / SH::T), 256>>>(A, d_x, d_y2, d_act, d_part); }); \
        char nm[80]; snprintf(nm, 80, "node spmv T%d CH%d minb%d", SH::T, CH, MB); REPORT(nm, t, spmv_bytes); cmp("spmv"); }
        if (bs == 2) { SPN(S64, 4, 8) SPN(S64, 4, 4) SPN(S64, 8, 4) SPN(S32, 4, 8) SPN(S32, 8, 8) SPN(S32, 8, 4) }
    }
    // ---- backward GS phase on the largest colour (in place: reset s each run)
    {
        const int c = 0;
        const int nb = (int)(offs[c] / bs), ne2 = (int)(offs[c + 1] / bs);
        const double bytes = (double)(prp[offs[c + 1]] - prp[offs[c]]) * 8.0 * Bp + 24.0 * (ne2 - nb) * bs * Bp;
        auto reset = [&](double* s) { CK(cudaMemcpy(s, d_x, 8 * n * Bp, cudaMemcpyDeviceToDevice)); };
        reset(d_y);
        float ms = timeit([&] { k_gs_backward<S64, true><<<dim3(G(ne2 - nb, 8, 8), Bp / 64), 256>>>(A, d_f, d_y, d_act, nb, ne2, d_part, 0); }, 1);
        reset(d_y);
        k_gs_backward<S64, true><<<dim3(G(ne2 - nb, 8, 8), Bp / 64), 256>>>(A, d_f, d_y, d_act, nb, ne2, d_part, 0);
        ms = timeit([&] { k_gs_backward<S64, true><<<dim3(G(ne2 - nb, 8, 8), Bp / 64), 256>>>(A, d_f, d_y, d_act, nb, ne2, d_part, 0); });
        reset(d_y);
        k_gs_backward<S64, true><<<dim3(G(ne2 - nb, 8, 8), Bp / 64), 256>>>(A, d_f, d_y, d_act, nb, ne2, d_part, 0);
        REPORT("row gs_backward phase V2", ms, bytes);
#define GSN(SH, CH, MB, MODE) { \
        auto run = [&] { k_gs_node<SH, 2, CH, MODE, true, MB><<<dim3(G(ne2 - nb, 8, 8), Bp / SH::T), 256>>>(A, d_f, d_y2, d_act, nb, ne2, d_part, 0); }; \
        float t = timeit(run); reset(d_y2); run(); CK(cudaDeviceSynchronize()); \
        char nm[80]; snprintf(nm, 80, "node gs mode%d T%d CH%d minb%d", MODE, SH::T, CH, MB); REPORT(nm, t, bytes); if (MODE == 2) cmp("gs_bwd"); }
        if (bs == 2) { GSN(S64, 4, 8, 2) GSN(S64, 4, 4, 2) GSN(S64, 8, 4, 2) GSN(S32, 4, 8, 2) GSN(S32, 8, 8, 2) GSN(S32, 8, 4, 2) }
        // forward first sweep on colour 2
        const int c2 = 2;
        const int nb2 = (int)(offs[c2] / bs), ne3 = (int)(offs[c2 + 1] / bs);
        const double fb = (double)(prp[offs[c2 + 1]] - prp[offs[c2]]) * 4.0 * Bp + 24.0 * (ne3 - nb2) * bs * Bp;
        reset(d_y); reset(d_y2);
        auto rowf = [&] { k_gs_forward<S64, true><<<dim3(G(ne3 - nb2, 8, 8), Bp / 64), 256>>>(A, d_f, d_y, d_act, nb2, ne3); };
        float t = timeit(rowf); REPORT("row gs_forward first phase V2", t, fb);
#define GSF(SH, CH, MB) { auto run = [&] { k_gs_node<SH, 2, CH, 0, false, MB><<<dim3(G(ne3 - nb2, 8, 8), Bp / SH::T), 256>>>(A, d_f, d_y2, d_act, nb2, ne3, d_part, 0); }; \
        float t2 = timeit(run); char nm[80]; snprintf(nm, 80, "node gs first T%d CH%d minb%d", SH::T, CH, MB); REPORT(nm, t2, fb); cmp("gs_fwd_first"); }
        if (bs == 2) { GSF(S64, 4, 8) GSF(S64, 8, 4) GSF(S32, 8, 8) GSF(S32, 8, 4) }
    }
    return 0;
}
