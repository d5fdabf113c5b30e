// row_lab.cu -- register budget vs memory-level parallelism for the batched
// row loops: SpMV variants over (V instances/lane, unroll, min CTAs/SM,
// column preload).  Same data as spmv_lab (c2 layout, Bp = 64).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>
#include "../include/pod2g_b200.h"
#include "../include/pod2g_gen.h"
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
constexpr int BP = 64;

template <int V> struct VT;
template <> struct VT<1> { using T = double; };
template <> struct VT<2> { using T = double2; };
__device__ __forceinline__ double ld_cs1(const double* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_cs2(const double* p) { return __ldcs((const double2*)p); }

// plain: ci -> x dependency per entry, unroll UNR
template <int V, int UNR, int MINB>
__global__ void __launch_bounds__(256, MINB) sp_plain(int n, const int* rp, const int* ci, const double* vals,
                                                      const double* x, double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = blockIdx.y * 32 * V + lane * V;
    for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
        double a0 = 0, a1 = 0;
        const int kb = rp[i], ke = rp[i + 1];
#pragma unroll UNR
        for (int k = kb; k < ke; ++k) {
            const unsigned c = (unsigned)__ldg(ci + k);
            if constexpr (V == 2) {
                const double2 a = ld_cs2(vals + (unsigned)k * BP + b0);
                const double2 xx = *(const double2*)(x + c * BP + b0);
                a0 += a.x * xx.x; a1 += a.y * xx.y;
            } else {
                a0 += ld_cs1(vals + (unsigned)k * BP + b0) * x[c * BP + b0];
            }
        }
        if constexpr (V == 2) *(double2*)(y + (size_t)i * BP + b0) = make_double2(a0, a1);
        else y[(size_t)i * BP + b0] = a0;
    }
}

// preloaded columns (lane-cooperative + shfl), CH entries in flight
template <int V, int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) sp_pre(int n, const int* rp, const int* ci, const double* vals,
                                                    const double* x, double* y) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b0 = blockIdx.y * 32 * V + lane * V;
    for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
        double a0 = 0, a1 = 0;
        const int kb = rp[i], ke = rp[i + 1];
        for (int base = kb; base < ke; base += 32) {
            const int cnt = min(32, ke - base);
            const int myc = lane < cnt ? __ldg(ci + base + lane) : 0;
            for (int j0 = 0; j0 < cnt; j0 += CH) {
                typename VT<V>::T a[CH], xx[CH];
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    const unsigned c = (unsigned)__shfl_sync(0xffffffffu, myc, (j0 + q) & 31);
                    if (j0 + q < cnt) {
                        if constexpr (V == 2) {
                            a[q] = ld_cs2(vals + (unsigned)(base + j0 + q) * BP + b0);
                            xx[q] = *(const double2*)(x + c * BP + b0);
                        } else {
                            a[q] = ld_cs1(vals + (unsigned)(base + j0 + q) * BP + b0);
                            xx[q] = x[c * BP + b0];
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < CH; ++q)
                    if (j0 + q < cnt) {
                        if constexpr (V == 2) { a0 += a[q].x * xx[q].x; a1 += a[q].y * xx[q].y; }
                        else a0 += a[q] * xx[q];
                    }
            }
        }
        if constexpr (V == 2) *(double2*)(y + (size_t)i * BP + b0) = make_double2(a0, a1);
        else y[(size_t)i * BP + b0] = a0;
    }
}

template <class F> float timeit(F f, int reps = 20) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    f(); CK(cudaDeviceSynchronize()); cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); return ms / reps;
}

int main() {
    p2g_mesh* m; p2g_mesh_create(2, 256, 128, 1, 2.0, 1.0, 1.0, 0.3, &m);
    int64_t n, nnz, ne; int32_t bs; p2g_mesh_info(m, &n, &nnz, &ne, &bs);
    std::vector<uint64_t> rp(n + 1), ci(nnz); p2g_mesh_pattern(m, rp.data(), ci.data());
    std::vector<int64_t> perm(n), offs(65); int32_t nc; char err[256];
    p2g_analyze_pattern(n, rp.data(), ci.data(), bs, perm.data(), &nc, offs.data(), 65, err, 256);
    std::vector<int64_t> iperm(n); for (int64_t i = 0; i < n; ++i) iperm[perm[i]] = i;
    std::vector<int> prp(n + 1, 0), pci(nnz);
    for (int64_t i = 0; i < n; ++i) { std::vector<int> cols; for (uint64_t k = rp[perm[i]]; k < rp[perm[i] + 1]; ++k) cols.push_back((int)iperm[ci[k]]);
        std::sort(cols.begin(), cols.end()); std::copy(cols.begin(), cols.end(), pci.begin() + prp[i]); prp[i + 1] = prp[i] + (int)cols.size(); }
    int *d_rp, *d_ci; double *d_v, *d_x, *d_y;
    CK(cudaMalloc(&d_rp, 4 * (n + 1))); CK(cudaMalloc(&d_ci, 4 * nnz)); CK(cudaMalloc(&d_v, 8 * nnz * BP));
    CK(cudaMalloc(&d_x, 8 * n * BP)); CK(cudaMalloc(&d_y, 8 * n * BP));
    CK(cudaMemcpy(d_rp, prp.data(), 4 * (n + 1), cudaMemcpyHostToDevice)); CK(cudaMemcpy(d_ci, pci.data(), 4 * nnz, cudaMemcpyHostToDevice));
    CK(cudaMemset(d_v, 0, 8 * nnz * BP)); CK(cudaMemset(d_x, 0, 8 * n * BP));
    const double bytes = 8.0 * nnz * BP + 4.0 * nnz + 4.0 * (n + 1) + 16.0 * n * BP;
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
#define RUN(name, KERN, V, MINB) { int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, KERN, 256, 0); \
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, KERN); dim3 g(sms * occ, 2 / V); \
    float ms = timeit([&] { KERN<<<g, 256>>>((int)n, d_rp, d_ci, d_v, d_x, d_y); }); \
    printf("%-28s regs %3d occ %d  %7.1f us %6.0f GB/s\n", name, fa.numRegs, occ, ms * 1e3, bytes / (ms * 1e-3) / 1e9); }
    RUN("plain V2 u4 minb8", (sp_plain<2, 4, 8>), 2, 8)
    RUN("plain V2 u4 minb4", (sp_plain<2, 4, 4>), 2, 4)
    RUN("plain V2 u8 minb4", (sp_plain<2, 8, 4>), 2, 4)
    RUN("plain V2 u8 minb6", (sp_plain<2, 8, 6>), 2, 6)
    RUN("plain V1 u4 minb8", (sp_plain<1, 4, 8>), 1, 8)
    RUN("plain V1 u8 minb8", (sp_plain<1, 8, 8>), 1, 8)
    RUN("plain V1 u8 minb4", (sp_plain<1, 8, 4>), 1, 4)
    RUN("pre V2 ch4 minb8", (sp_pre<2, 4, 8>), 2, 8)
    RUN("pre V2 ch8 minb4", (sp_pre<2, 8, 4>), 2, 4)
    RUN("pre V2 ch6 minb6", (sp_pre<2, 6, 6>), 2, 6)
    RUN("pre V2 ch4 minb6", (sp_pre<2, 4, 6>), 2, 6)
    RUN("pre V1 ch8 minb8", (sp_pre<1, 8, 8>), 1, 8)
    RUN("pre V1 ch6 minb8", (sp_pre<1, 6, 8>), 1, 8)
    RUN("pre V1 ch16 minb4", (sp_pre<1, 16, 4>), 1, 4)
    RUN("pre V1 ch12 minb6", (sp_pre<1, 12, 6>), 1, 6)
    return 0;
}
