// spmv_lab.cu -- microbenchmark of batched SpMV variants on the c2 layout
// ([nnz][64] values, [n][64] vectors, colour-permuted Q4 pattern).
// Build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//   -o tools/spmv_lab tools/spmv_lab.cu -Lpaper_2207_02543_b200 -lpod2g_b200 \
//   -Xlinker -rpath,$PWD/paper_2207_02543_b200
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#include "../include/pod2g_b200.h"
#include "../include/pod2g_gen.h"

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e = (x);                                                         \
        if (e != cudaSuccess) {                                                      \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));         \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

constexpr int BP = 64;

__device__ __forceinline__ double2 ld_na(const double* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ double2 ld_cs(const double* p) { return __ldcs((const double2*)p); }
__device__ __forceinline__ double2 ld_x(const double* p) { return *(const double2*)p; }

// V0: one row per warp, lanes = 32 x double2 instances, unroll 4 (the library's loop)
template <int MODE>
__global__ void __launch_bounds__(256) sp_v0(int n, const int* rp, const int* ci, const double* vals,
                                             const double* x, double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = lane * 2;
    for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
        double a0 = 0, a1 = 0;
        const int kb = rp[i], ke = rp[i + 1];
#pragma unroll 4
        for (int k = kb; k < ke; ++k) {
            const int c = __ldg(ci + k);
            const double2 a = MODE == 0 ? ld_cs(vals + (size_t)k * BP + b0) : ld_na(vals + (size_t)k * BP + b0);
            const double2 xx = ld_x(x + (size_t)c * BP + b0);
            a0 += a.x * xx.x;
            a1 += a.y * xx.y;
        }
        *(double2*)(y + (size_t)i * BP + b0) = make_double2(a0, a1);
    }
}

// V3: node-blocked (bs = 2): both rows of a node share the column list, x
// loaded once per entry; values of both rows loaded together.
template <int MODE, int UNR>
__global__ void __launch_bounds__(256) sp_node(int nn, const int* rp, const int* ci, const double* vals,
                                               const double* x, double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = lane * 2;
    for (int a = blockIdx.x * 8 + warp; a < nn; a += gridDim.x * 8) {
        const int i0 = 2 * a;
        const int kb0 = rp[i0], kb1 = rp[i0 + 1], ke1 = rp[i0 + 2];
        const int len = kb1 - kb0;  // == ke1 - kb1
        double r00 = 0, r01 = 0, r10 = 0, r11 = 0;
#pragma unroll UNR
        for (int j = 0; j < len; ++j) {
            const int c = __ldg(ci + kb0 + j);
            const double2 v0 = MODE == 0 ? ld_cs(vals + (size_t)(kb0 + j) * BP + b0) : ld_na(vals + (size_t)(kb0 + j) * BP + b0);
            const double2 v1 = MODE == 0 ? ld_cs(vals + (size_t)(kb1 + j) * BP + b0) : ld_na(vals + (size_t)(kb1 + j) * BP + b0);
            const double2 xx = ld_x(x + (size_t)c * BP + b0);
            r00 += v0.x * xx.x;
            r01 += v0.y * xx.y;
            r10 += v1.x * xx.x;
            r11 += v1.y * xx.y;
        }
        *(double2*)(y + (size_t)i0 * BP + b0) = make_double2(r00, r01);
        *(double2*)(y + (size_t)(i0 + 1) * BP + b0) = make_double2(r10, r11);
    }
}

// V4: node-blocked + lane-cooperative column preload
template <int MODE>
__global__ void __launch_bounds__(256) sp_node_pre(int nn, const int* rp, const int* ci,
                                                   const double* vals, const double* x, double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = lane * 2;
    for (int a = blockIdx.x * 8 + warp; a < nn; a += gridDim.x * 8) {
        const int i0 = 2 * a;
        const int kb0 = rp[i0], kb1 = rp[i0 + 1];
        const int len = kb1 - kb0;
        const int myc = lane < len ? __ldg(ci + kb0 + lane) : 0;
        double r00 = 0, r01 = 0, r10 = 0, r11 = 0;
        for (int j0 = 0; j0 < len; j0 += 6) {
            double2 v0[6], v1[6], xx[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                const int c = __shfl_sync(0xffffffffu, myc, (j0 + q) & 31);
                if (j0 + q < len) {
                    v0[q] = MODE == 0 ? ld_cs(vals + (size_t)(kb0 + j0 + q) * BP + b0) : ld_na(vals + (size_t)(kb0 + j0 + q) * BP + b0);
                    v1[q] = MODE == 0 ? ld_cs(vals + (size_t)(kb1 + j0 + q) * BP + b0) : ld_na(vals + (size_t)(kb1 + j0 + q) * BP + b0);
                    xx[q] = ld_x(x + (size_t)c * BP + b0);
                }
            }
#pragma unroll
            for (int q = 0; q < 6; ++q)
                if (j0 + q < len) {
                    r00 += v0[q].x * xx[q].x;
                    r01 += v0[q].y * xx[q].y;
                    r10 += v1[q].x * xx[q].x;
                    r11 += v1[q].y * xx[q].y;
                }
        }
        *(double2*)(y + (size_t)i0 * BP + b0) = make_double2(r00, r01);
        *(double2*)(y + (size_t)(i0 + 1) * BP + b0) = make_double2(r10, r11);
    }
}

// V2: one instance per lane (two 32-wide tiles)
__global__ void __launch_bounds__(256) sp_v1lane(int n, const int* rp, const int* ci, const double* vals,
                                                 const double* x, double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = blockIdx.y * 32 + lane;
    for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
        double acc = 0;
        const int kb = rp[i], ke = rp[i + 1];
#pragma unroll 4
        for (int k = kb; k < ke; ++k) {
            const int c = __ldg(ci + k);
            acc += __ldcs(vals + (size_t)k * BP + b) * x[(size_t)c * BP + b];
        }
        y[(size_t)i * BP + b] = acc;
    }
}

__global__ void copy_k(const double2* a, double2* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}

template <class F>
float timeit(F f, int reps = 20) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const int nx = argc > 1 ? atoi(argv[1]) : 256, ny = nx / 2;
    p2g_mesh* m;
    p2g_mesh_create(2, nx, ny, 1, 2.0, 1.0, 1.0, 0.3, &m);
    int64_t n, nnz, ne;
    int32_t bs;
    p2g_mesh_info(m, &n, &nnz, &ne, &bs);
    std::vector<uint64_t> rp(n + 1), ci(nnz);
    p2g_mesh_pattern(m, rp.data(), ci.data());
    std::vector<int64_t> perm(n), offs(65);
    int32_t nc;
    char err[256];
    p2g_analyze_pattern(n, rp.data(), ci.data(), bs, perm.data(), &nc, offs.data(), 65, err, 256);
    std::vector<int64_t> iperm(n);
    for (int64_t i = 0; i < n; ++i) iperm[perm[i]] = i;
    std::vector<int> prp(n + 1, 0), pci(nnz);
    for (int64_t i = 0; i < n; ++i) {
        const int64_t o = perm[i];
        std::vector<int> cols;
        for (uint64_t k = rp[o]; k < rp[o + 1]; ++k) cols.push_back((int)iperm[ci[k]]);
        std::sort(cols.begin(), cols.end());
        std::copy(cols.begin(), cols.end(), pci.begin() + prp[i]);
        prp[i + 1] = prp[i] + (int)cols.size();
    }
    printf("n=%ld nnz=%ld colours=%d\n", (long)n, (long)nnz, nc);
    int *d_rp, *d_ci;
    double *d_v, *d_x, *d_y;
    CK(cudaMalloc(&d_rp, sizeof(int) * (n + 1)));
    CK(cudaMalloc(&d_ci, sizeof(int) * nnz));
    CK(cudaMalloc(&d_v, sizeof(double) * nnz * BP));
    CK(cudaMalloc(&d_x, sizeof(double) * n * BP));
    CK(cudaMalloc(&d_y, sizeof(double) * n * BP));
    CK(cudaMemcpy(d_rp, prp.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d_ci, pci.data(), sizeof(int) * nnz, cudaMemcpyHostToDevice));
    {
        std::vector<double> h(nnz * BP);
        std::mt19937_64 g(1);
        for (auto& v : h) v = (g() >> 11) * 0x1.0p-53;
        CK(cudaMemcpy(d_v, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice));
        std::vector<double> hx(n * BP);
        for (auto& v : hx) v = (g() >> 11) * 0x1.0p-53;
        CK(cudaMemcpy(d_x, hx.data(), sizeof(double) * hx.size(), cudaMemcpyHostToDevice));
    }
    const double bytes = 8.0 * nnz * BP + 4.0 * nnz + 4.0 * (n + 1) + 16.0 * n * BP;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto report = [&](const char* name, float ms) {
        printf("%-34s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    };
    {
        size_t cn = nnz * BP / 2;
        float ms = timeit([&] { copy_k<<<sms * 8, 256>>>((double2*)d_v, (double2*)d_y, std::min(cn, (size_t)n * BP / 2)); });
        printf("copy (n*64 doubles) %8.1f us %7.0f GB/s\n", ms * 1e3, 16.0 * n * BP / (ms * 1e-3) / 1e9);
    }
    for (int occ : {4, 6, 8, 16}) {
        char nm[64];
        const int g = sms * occ;
        snprintf(nm, 64, "v0 cs grid=%d", g);
        report(nm, timeit([&] { sp_v0<0><<<g, 256>>>(n, d_rp, d_ci, d_v, d_x, d_y); }));
        snprintf(nm, 64, "v0 noalloc grid=%d", g);
        report(nm, timeit([&] { sp_v0<1><<<g, 256>>>(n, d_rp, d_ci, d_v, d_x, d_y); }));
        snprintf(nm, 64, "node u4 cs grid=%d", g);
        report(nm, timeit([&] { sp_node<0, 4><<<g, 256>>>(n / 2, d_rp, d_ci, d_v, d_x, d_y); }));
        snprintf(nm, 64, "node u4 noalloc grid=%d", g);
        report(nm, timeit([&] { sp_node<1, 4><<<g, 256>>>(n / 2, d_rp, d_ci, d_v, d_x, d_y); }));
        snprintf(nm, 64, "node u8 noalloc grid=%d", g);
        report(nm, timeit([&] { sp_node<1, 8><<<g, 256>>>(n / 2, d_rp, d_ci, d_v, d_x, d_y); }));
        snprintf(nm, 64, "node pre noalloc grid=%d", g);
        report(nm, timeit([&] { sp_node_pre<1><<<g, 256>>>(n / 2, d_rp, d_ci, d_v, d_x, d_y); }));
        snprintf(nm, 64, "v1lane grid=%dx2", g);
        report(nm, timeit([&] { sp_v1lane<<<dim3(g, 2), 256>>>(n, d_rp, d_ci, d_v, d_x, d_y); }));
    }
    {
        const int g = (int)((n / 2 + 7) / 8);
        report("node u4 noalloc full grid", timeit([&] { sp_node<1, 4><<<g, 256>>>(n / 2, d_rp, d_ci, d_v, d_x, d_y); }));
        report("v0 noalloc full grid", timeit([&] { sp_v0<1><<<(int)((n + 7) / 8), 256>>>(n, d_rp, d_ci, d_v, d_x, d_y); }));
    }
    return 0;
}
