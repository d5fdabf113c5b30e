// p2g_solver.cu -- host orchestration and the C-ABI (include/pod2g_b200.h) of
// the batched POD-2G PCG solve path on B200 (sm_100a).
//
// One PCG iteration (krylov.hpp:272-286 with Pod2gPreconditioner::apply,
// pod.hpp:264-267 -> Pod2gOperator::cycle, pod.hpp:196-207) is the kernel
// sequence
//   spmv+dot | alpha | update+pre-smooth(colour 0) | fwd colours 1..C-1 |
//   residual+restrict | coarse solve | prolong | bwd colours C-1..0 (+r.s) |
//   finalize (beta, rel, history, convergence) | p-update
// captured once into a CUDA graph whose body sits in a conditional WHILE node:
// the loop runs entirely on the device until every instance has converged,
// broken down or hit max_iter (the finalize kernel sets the condition).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pod2g_b200.h"
#include "p2g_kernels.cuh"
#include "p2g_pattern.h"
#include "p2g_partition.h"
#include "p2g_mesh_desc.h"
#include "../../include/pod2g_gen.h"

#include <dlfcn.h>
#include <mutex>
#include <unordered_map>
#include <nccl.h>

using namespace p2g;

namespace {

enum Kclass {
    KC_SPMV = 0,
    KC_UPDATE,
    KC_FWD,
    KC_RESTRICT,
    KC_COARSE,
    KC_PROLONG,
    KC_BWD,
    KC_REDUCE,
    KC_PUPDATE,
    KC_RESID,
    KC_COMM
};
// one class per kernel family of the loop body (gs_forward / gs_backward: the
// colour-phase launches of one sweep; scalar_reduce: k_alpha + k_finalize)
const char* kKclassNames[P2G_NUM_KCLASS] = {"spmv_dot", "update_presmooth", "gs_forward",
                                            "restrict", "coarse_solve", "prolong",
                                            "gs_backward", "scalar_reduce", "p_update",
                                            "residual", "halo_allreduce"};

enum ShapeId { SH_B1A = 0, SH_B1B, SH_B8, SH_B32, SH_B64 };

}  // namespace

struct p2g_handle {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    std::string err;

    // pattern
    ColouredPattern pat;
    bool have_pattern = false;
    int64_t n_ghost = 0;         // partitioned handles: ghost rows after the owned ones
    bool own_stream = true;
    int *d_rp = nullptr, *d_ci = nullptr, *d_dpos = nullptr;
    int64_t *d_vperm = nullptr, *d_perm = nullptr;
    // node-blocked view (build_node_table); node_blk == false: row kernels only
    bool node_blk = false;
    int nmax = 0;
    int4* d_ninfo = nullptr;
    int* d_ncol = nullptr;

    // batch
    int B = 0, Bp = 0, shape = SH_B64;
    double* d_vals = nullptr;
    bool have_values = false;

    // basis
    int k = -1;
    double* d_phi = nullptr;   // [rows][k]
    double* d_phit = nullptr;  // [rows][phi_ks], zero padded (tensor-core tiles, phi_stride)
    int phi_ks = 0;

    // surrogate warm start (p2g_set_surrogate): MLP on the device
    int sg_layers = 0, sg_act = 0, sg_wmax = 0;
    std::vector<int> sg_widths;
    int* d_sg_widths = nullptr;
    double *d_sg_W = nullptr, *d_sg_b = nullptr, *d_sg_norm = nullptr, *d_theta = nullptr;
    bool theta_set = false;

    // vectors [n][Bp]
    double *d_u = nullptr, *d_r = nullptr, *d_s = nullptr, *d_s2 = nullptr, *d_p = nullptr,
           *d_Kp = nullptr, *d_b = nullptr, *d_t = nullptr;
    // per-instance
    double *d_alpha = nullptr, *d_beta = nullptr, *d_rsold = nullptr, *d_fnorm = nullptr,
           *d_rel = nullptr, *d_e = nullptr, *d_L = nullptr, *d_Ac = nullptr;
    int *d_active = nullptr, *d_iters = nullptr, *d_status = nullptr, *d_setup_status = nullptr,
        *d_all = nullptr;
    double* d_hist = nullptr;
    SolveParams* d_prm = nullptr;
    unsigned* d_flag_ticket = nullptr;  // [any-active flag, CTA ticket] of k_finalize
    // partials
    int nb_cap = 0;
    double *d_part_dot = nullptr, *d_part_rr = nullptr, *d_part_ff = nullptr,
           *d_part_rs = nullptr, *d_part_c = nullptr;
    int part_rs_rows = 0;
    // staging
    double* d_stage = nullptr;
    size_t stage_bytes = 0;
    // p2g_prefetch_values: next batch's values copied on a side stream
    cudaStream_t cstream = nullptr;
    cudaEvent_t pref_ev = nullptr;
    double* d_pref = nullptr;
    size_t pref_cap = 0;
    const double* pref_host = nullptr;
    int pref_B = 0;
    bool pref_started = false;  // deferred until the next solve has uploaded its b

    // setup
    p2g_config cfg{};
    bool setup_done = false;
    bool has_state = false;  // a solve ran since the last setup (Krylov state valid)
    double* s_final = nullptr;  // buffer holding B r after the post-smoother
    double* s_prol = nullptr;   // prolongated s' (Kp recurrence)
    int64_t batch_hint = 0;  // p2g_set_batch_hint: the batch the handle will be used with (0: unknown)
    const double* dlt_of = nullptr;  // the sweep output whose s - s' the last backward sweep left in d_t

    // graph
    cudaGraphExec_t loop_exec = nullptr;
    std::vector<uint64_t> graph_key;  // what the captured graph baked in
    cudaGraphConditionalHandle cond = 0;
    // the pod2g_solve cycle loop (p2g_pod2g_solve): its own graph and condition
    cudaGraphExec_t cyc_exec = nullptr;
    std::vector<uint64_t> cyc_key;
    cudaGraphConditionalHandle cyc_cond = 0;
    int64_t launches_per_cycle = 0;

    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<std::pair<const void*, int>> occ_cache;
    std::vector<std::pair<void*, size_t>> caps;  // ensure() capacities
    double *d_Y = nullptr, *d_part_ac = nullptr;  // setup workspaces
    double last_ms[2] = {0, 0};
    int64_t launches_per_iter = 0, launches_last_solve = 0, launch_counter = 0;
    int64_t launches_executed = 0;  // every kernel this handle ran (graph iterations included)
    bool capturing = false;
    // profiling
    bool profiling = false;
    static constexpr int kMaxKev = 192;  // > 15 + 2 x 64 colour phases
    cudaEvent_t kev[kMaxKev];
    int kev_n = 0;
    int kev_class[kMaxKev];
};

namespace {

#define CU(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            h->err = std::string(#call) + ": " + cudaGetErrorString(e_);                  \
            return static_cast<int>(P2G_ECUDA);                                          \
        }                                                                                 \
    } while (0)

#define REQ(cond, code, msg)           \
    do {                                \
        if (!(cond)) {                  \
            h->err = (msg);             \
            return static_cast<int>(code); \
        }                               \
    } while (0)

#define TRY(expr)                       \
    do {                                \
        int st_ = (expr);               \
        if (st_ != P2G_OK) return st_;  \
    } while (0)

// ---- guard bands (P2G_GUARD=1, debugging / tests): every handle buffer gets
// kGuardBytes of a fixed byte pattern on each side; p2g_debug_guard_check()
// reports buffers whose bands changed, i.e. out-of-bounds device writes.
// (compute-sanitizer is not available on the GPU pool this was built on.)
constexpr size_t kGuardBytes = 256;
constexpr unsigned char kGuardByte = 0xA5;
struct GuardRegistry {
    std::mutex mu;
    std::unordered_map<void*, size_t> bytes;  // user pointer -> user bytes
};
GuardRegistry& guards() {
    static GuardRegistry g;
    return g;
}
bool guard_mode() {
    static const bool on = [] {
        const char* v = std::getenv("P2G_GUARD");
        return v && v[0] == '1';
    }();
    return on;
}

template <class T>
void dfree(T*& p) {
    if (p) {
        void* raw = p;
        if (guard_mode()) {
            std::lock_guard<std::mutex> lk(guards().mu);
            auto it = guards().bytes.find((void*)p);
            if (it != guards().bytes.end()) {
                raw = (unsigned char*)(void*)p - kGuardBytes;
                guards().bytes.erase(it);
            }
        }
        cudaFree(raw);
    }
    p = nullptr;
}

template <class T>
int dalloc(p2g_handle* h, T*& p, size_t count) {
    dfree(p);
    if (count == 0) count = 1;
    if (!guard_mode()) {
        CU(cudaMalloc(&p, count * sizeof(T)));
        return P2G_OK;
    }
    const size_t bytes = count * sizeof(T);
    unsigned char* raw = nullptr;
    CU(cudaMalloc(&raw, bytes + 2 * kGuardBytes));
    CU(cudaMemset(raw, kGuardByte, kGuardBytes));
    CU(cudaMemset(raw + kGuardBytes + bytes, kGuardByte, kGuardBytes));
    p = reinterpret_cast<T*>(raw + kGuardBytes);
    std::lock_guard<std::mutex> lk(guards().mu);
    guards().bytes[(void*)p] = bytes;
    return P2G_OK;
}

// grow-only workspace: reallocates only when `count` exceeds the capacity
// (no cudaMalloc/cudaFree on the per-batch path once sizes are stable)
template <class T>
int ensure(p2g_handle* h, T*& p, size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    for (auto& c : h->caps)
        if (c.first == (void*)&p) {
            if (p && c.second >= bytes) return P2G_OK;
            TRY(dalloc(h, p, std::max<size_t>(count, 1)));
            c.second = bytes;
            return P2G_OK;
        }
    TRY(dalloc(h, p, std::max<size_t>(count, 1)));
    h->caps.emplace_back((void*)&p, bytes);
    return P2G_OK;
}

constexpr int kProlongTmaRows = 1 << 18;  // rows from which k_prolong_mma is used when k_prolong_ws is off
// the warp-specialised prolongation (k_prolong_ws) from this many rows on: c2
// (66,048 rows) 16.4 vs 18.5 us, c4 173 vs 190 us, c3 725 vs 969 us
constexpr int kProlongWsRows = 1 << 16;

// the wide tensor-core restriction (k_restrict_reg2); P2G_RESTRICT_WIDE=0
// selects k_restrict_reg (A/B)
// the warp-specialised bulk-copy restriction (k_restrict_ws) from this many
// rows on (P2G_RESTRICT_WS=0 disables it, =1 forces it at any size); c2
// (66,048 rows): 16.4 vs 18.8 us, c4 119 vs 152 us, c3 534 vs 1091 us
constexpr int kRestrictWsRows = 1 << 16;
int restrict_ws_mode() {
    const char* v = std::getenv("P2G_RESTRICT_WS");
    return v ? (v[0] == '0' ? 0 : 2) : 1;
}

int prolong_ws_mode() {  // k_prolong_ws, same convention (P2G_PROLONG_WS)
    const char* v = std::getenv("P2G_PROLONG_WS");
    return v ? (v[0] == '0' ? 0 : 2) : 1;
}

bool restrict_wide() {
    static const bool w = [] {
        const char* v = std::getenv("P2G_RESTRICT_WIDE");
        return !(v && v[0] == '0');
    }();
    return w;
}

template <int KM>
struct KTag {};

int kbucket(int k) {
    if (k <= 8) return 8;
    if (k <= 16) return 16;
    if (k <= 24) return 24;
    if (k <= 32) return 32;
    if (k <= 40) return 40;
    return 64;
}

#define KSWITCH(kv, ...)                                            \
    switch (kbucket(kv)) {                                          \
        case 8: { constexpr int KM = 8; __VA_ARGS__; } break;      \
        case 16: { constexpr int KM = 16; __VA_ARGS__; } break;    \
        case 24: { constexpr int KM = 24; __VA_ARGS__; } break;    \
        case 32: { constexpr int KM = 32; __VA_ARGS__; } break;    \
        case 40: { constexpr int KM = 40; __VA_ARGS__; } break;    \
        default: { constexpr int KM = 64; __VA_ARGS__; } break;    \
    }

// upload Phi ([rows][k], already in local row order) and its padded copy
int upload_phi(p2g_handle* h, const std::vector<double>& phi, int64_t rows, int k) {
    TRY(ensure(h, h->d_phi, phi.size() + 2));  // +2: 16-byte rounded bulk tile copies
    CU(cudaMemcpy(h->d_phi, phi.data(), sizeof(double) * phi.size(), cudaMemcpyHostToDevice));
    const int ks = phi_stride(std::max(k, 1));
    std::vector<double> pt((size_t)rows * ks, 0.0);
    for (int64_t i = 0; i < rows; ++i)
        for (int a = 0; a < k; ++a) pt[i * ks + a] = phi[i * k + a];
    TRY(ensure(h, h->d_phit, pt.size()));
    CU(cudaMemcpy(h->d_phit, pt.data(), sizeof(double) * pt.size(), cudaMemcpyHostToDevice));
    h->phi_ks = ks;
    return P2G_OK;
}

bool kp_recurrence(const p2g_handle* h) {
    return h->cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR && h->cfg.kp_update == P2G_KP_RECURRENCE;
}

Mat mat_of(p2g_handle* h) {
    Mat A;
    A.n = static_cast<int>(h->pat.n);
    A.bs = h->pat.bs;
    A.rp = h->d_rp;
    A.ci = h->d_ci;
    A.dpos = h->d_dpos;
    A.vals = h->d_vals;
    A.Bp = h->Bp;
    return A;
}

// p2g_profile_iteration: close the current timing interval (everything
// issued on the stream since the previous mark) and charge it to `kclass`
// (inside a stream capture the record becomes an external event-record node)
cudaError_t prof_record(p2g_handle* h, cudaEvent_t e, cudaStream_t st) {
    return h->capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                        : cudaEventRecord(e, st);
}

void prof_mark(p2g_handle* h, int kclass) {
    if (h->profiling && h->kev_n < p2g_handle::kMaxKev - 1) {
        h->kev_class[h->kev_n] = kclass;
        prof_record(h, h->kev[h->kev_n + 1], h->stream);
        ++h->kev_n;
    }
}

void count_launch(p2g_handle* h, int kclass) {
    ++h->launch_counter;
    if (!h->capturing) ++h->launches_executed;
    prof_mark(h, kclass);
}

// grid for a node-range kernel: one wave of resident blocks at most
// cluster == true: grid.x rounded up to a multiple of kCluster (the kernel
// carries __cluster_dims__), one partial row per cluster
// Resident CTAs per kernel (one full wave), cached per function.  For the
// cluster kernels this is the number of co-resident CLUSTERS x kCluster, so
// the grid never spills into a partial second wave.
int resident_ctas(p2g_handle* h, const void* fn, bool cluster, size_t smem = 0, int block = kBlock,
                  int csize = kCluster) {
    for (auto& e : h->occ_cache)
        if (e.first == fn) return e.second;
    int ctas = 0;
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cluster) {
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3(csize * 1024, 1, 1);
        lc.blockDim = dim3(block, 1, 1);
        lc.dynamicSmemBytes = smem;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, fn, &lc) != cudaSuccess || ncl <= 0) {
            cudaGetLastError();
            ncl = h->num_sms / csize;
        }
        ctas = ncl * csize;
    } else {
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, block, smem);
        ctas = std::max(occ, 1) * h->num_sms;
    }
    h->occ_cache.emplace_back(fn, ctas);
    return ctas;
}

template <class Sh>
dim3 node_grid(p2g_handle* h, int64_t units, const void* fn, bool cluster = false) {
    const int64_t need = (units + kWarps * Sh::R - 1) / (kWarps * Sh::R);
    int64_t gx = std::min<int64_t>(need, resident_ctas(h, fn, cluster));
    gx = std::max<int64_t>(gx, 1);
    gx = std::min<int64_t>(gx, h->nb_cap);
    if (cluster) gx = (gx + kCluster - 1) / kCluster * kCluster;
    return dim3(static_cast<unsigned>(gx), static_cast<unsigned>(h->Bp / Sh::T));
}

// ----------------------------------------------------------------------------
// Shape-specialised launch sequence
template <class Sh>
struct Run {
    using ASh = typename AccShape<Sh>::type;

    static int nnodes(p2g_handle* h) { return static_cast<int>(h->pat.n / h->pat.bs); }

    // node-blocked kernels: one-instance-per-lane shapes on node-blocked patterns
    static bool blk(const p2g_handle* h) { return Sh::S == 1 && h->node_blk; }
    static NodeTab ntab(const p2g_handle* h) { return NodeTab{h->d_ninfo, h->d_ncol, h->nmax}; }
    // single-instance node-blocked kernels (one warp per node)
    static bool blk1(const p2g_handle* h) {
        return Sh::W == 1 && h->node_blk && !std::getenv("P2G_NO_NODEBLK1");
    }
    // the half-pass kernels (Kp recurrence, upper residual) leave most lanes
    // idle on hex8 (one lane per lower / upper neighbour): row kernels there
    // (128^3: 1.26 vs 2.05 ms and 1.33 vs 1.85 ms); blocked on Q4
    static bool blk1_half(const p2g_handle* h) { return blk1(h) && h->pat.bs == 2; }
    // hex8: two nodes per warp (16-lane halves) for the half passes
    static bool blk1_hw(const p2g_handle* h) {
        return blk1(h) && h->pat.bs == 3 && !std::getenv("P2G_NO_B1H");
    }
    // bulk-copy staged two-nodes-per-warp kernels (k_*_b1s): P2G_B1S = bit mask
    // {1 forward, 2 backward, 4 Kp recurrence, 8 upper residual}
    static constexpr size_t kB1sSmem = (size_t)kWarps * 2 * kB1SlotDoubles * sizeof(double);
    static bool blk1_stg(const p2g_handle* h, int bit) {
        if (!blk1_hw(h) || h->nmax * h->pat.bs * h->pat.bs + 2 > kB1SlotDoubles) return false;
        const char* e = std::getenv("P2G_B1S");
        const int mask = e ? std::atoi(e) : P2G_B1S_DEFAULT;
        return (mask & bit) != 0;
    }
    static dim3 blk1_grid(p2g_handle* h, int64_t nodes, const void* fn, bool cluster, size_t smem = 0) {
        const int64_t need = (nodes + kWarps - 1) / kWarps;
        int64_t gx = std::min<int64_t>(need, resident_ctas(h, fn, cluster, smem));
        gx = std::min<int64_t>(std::max<int64_t>(gx, 1), h->nb_cap);
        if (cluster) gx = (gx + kCluster - 1) / kCluster * kCluster;
        return dim3(static_cast<unsigned>(gx), 1);
    }
#define P2G_BS_SWITCH(bs, ...)          \
    if ((bs) == 2) {                    \
        constexpr int BS = 2;           \
        __VA_ARGS__                     \
    } else {                            \
        constexpr int BS = 3;           \
        __VA_ARGS__                     \
    }

    // the two producers of pKp partials (k_spmv<DOT>, k_kp_update) share one
    // grid so k_alpha always reduces the same number of partial rows
    static dim3 dot_grid(p2g_handle* h) {
        const dim3 a = node_grid<Sh>(h, nnodes(h), (const void*)k_spmv<Sh, true>, true);
        const void* kp = (const void*)k_kp_update<Sh>;
        if constexpr (Sh::S == 1) {
            if (blk(h)) kp = h->pat.bs == 2 ? (const void*)k_kp_update_blk<Sh, 2>
                                            : (const void*)k_kp_update_blk<Sh, 3>;
        }
        if constexpr (Sh::W == 1) {
            if (blk1_hw(h)) {
                const bool stg = blk1_stg(h, 4);
                kp = stg ? (const void*)k_kp_update_b1s<3> : (const void*)k_kp_update_b1h<3>;
                const dim3 b1 = blk1_grid(h, (nnodes(h) + 1) / 2, kp, true, stg ? kB1sSmem : 0);
                return a.x <= b1.x ? a : b1;
            }
            if (blk1_half(h)) {
                kp = h->pat.bs == 2 ? (const void*)k_kp_update_b1<2> : (const void*)k_kp_update_b1<3>;
                const dim3 b1 = blk1_grid(h, nnodes(h), kp, true);
                return a.x <= b1.x ? a : b1;
            }
        }
        const dim3 b = node_grid<Sh>(h, nnodes(h), kp, true);
        return a.x <= b.x ? a : b;
    }

    static int spmv(p2g_handle* h, const double* x, double* y, bool dot, int* nb_out) {
        Mat A = mat_of(h);
        if (dot) {
            auto fn = k_spmv<Sh, true>;
            dim3 g = dot_grid(h);
            fn<<<g, kBlock, 0, h->stream>>>(A, x, y, h->d_active, h->d_part_dot);
            if (nb_out) *nb_out = g.x / kCluster;
        } else {
            auto fn = k_spmv<Sh, false>;
            dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
            fn<<<g, kBlock, 0, h->stream>>>(A, x, y, h->d_active, nullptr);
        }
        count_launch(h, KC_SPMV);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    static int residual(p2g_handle* h, const double* f, const double* u, double* r, int* nb_out) {
        Mat A = mat_of(h);
        auto fn = k_residual<Sh, RES_FULL>;
        dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
        fn<<<g, kBlock, 0, h->stream>>>(A, f, u, r, h->d_active, h->d_part_rr, h->d_part_ff);
        *nb_out = g.x / kCluster;
        count_launch(h, KC_SPMV);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // pre-smoothing (+ optional PCG update) ; returns the row count of the rr partials
    static int update_pre(p2g_handle* h, bool update, const double* f_r, int* nb_rr) {
        if constexpr (Sh::S > 1) {
            // slot-split rows: a row-parallel update kernel, then colour 0 as a
            // regular forward phase (GS) -- the fused kernel would leave all
            // but one lane of each row group idle on the vector update
            if (update) {
                auto fn = k_update_rows<Sh>;
                const int n = static_cast<int>(h->pat.n);
                constexpr int RL = 32 / Sh::W;
                const int64_t need = (n + kWarps * RL - 1) / (kWarps * RL);
                int64_t gx = std::min<int64_t>(need, resident_ctas(h, (const void*)fn, true));
                gx = std::min<int64_t>(std::max<int64_t>(gx, 1), h->nb_cap);
                gx = (gx + kCluster - 1) / kCluster * kCluster;
                dim3 g((unsigned)gx, (unsigned)(h->Bp / Sh::T));
                fn<<<g, kBlock, 0, h->stream>>>(n, h->Bp, h->d_u, h->d_r, h->d_p, h->d_Kp,
                                                h->d_alpha, h->d_active, h->d_part_rr);
                if (nb_rr) *nb_rr = g.x / kCluster;
                count_launch(h, KC_UPDATE);
                CU(cudaGetLastError());
            }
            const double* rr = update ? h->d_r : f_r;
            if (h->cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR) return gs_forward(h, rr, h->d_s, 0, true);
        }
        Mat A = mat_of(h);
        const int pre = h->cfg.smoother == P2G_SMOOTHER_JACOBI ? PRE_JACOBI : PRE_GS;
        const int c0 = static_cast<int>(h->pat.color_rows[1] / h->pat.bs);
        double* r = update ? h->d_r : const_cast<double*>(f_r);
#define P2G_UP(U, P)                                                                         \
    {                                                                                        \
        auto fn = k_update_pre<Sh, U, P>;                                                    \
        dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);                         \
        fn<<<g, kBlock, 0, h->stream>>>(A, h->d_u, r, h->d_p, h->d_Kp, h->d_s, h->d_alpha,   \
                                        h->d_active, h->d_part_rr, c0, h->cfg.omega);        \
        if (U && nb_rr) *nb_rr = g.x / kCluster;                                             \
    }
        if (update && Sh::S == 1) {
            if (pre == PRE_GS) P2G_UP(true, PRE_GS) else P2G_UP(true, PRE_JACOBI)
        } else {
            if (pre == PRE_GS) P2G_UP(false, PRE_GS) else P2G_UP(false, PRE_JACOBI)
        }
#undef P2G_UP
        count_launch(h, KC_UPDATE);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // Bulk-copy staged backward colour phases (k_gs_backward_stg): Q4
    // node-blocked patterns with the whole batch in one instance tile.
    // P2G_STG_NW = warps per CTA (4, 6, 7, 8, 9, 10, 12; 0 = register-fed kernels).
    static int stg_nw(const p2g_handle* h) {
        if constexpr (Sh::S != 1 || Sh::T < 32) return 0;
        if (!h->node_blk || h->pat.bs != 2 || h->nmax > kStgNmax || h->Bp != Sh::T) return 0;
        const char* e = std::getenv("P2G_STG_NW");
        const int v = e ? std::atoi(e) : P2G_STG_NW_DEFAULT;
        return (v == 4 || v == 6 || v == 7 || v == 8 || v == 9 || v == 10 || v == 12) ? v : 0;
    }
    template <int NW>
    static dim3 stg_grid(p2g_handle* h, int64_t nodes, const void* fn) {
        int ctas = 0;
        for (auto& e : h->occ_cache)
            if (e.first == fn) ctas = e.second;
        if (!ctas) {
            const size_t smem = StgGeo<Sh, NW>::smem;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            int occ = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, NW * 32, smem);
            ctas = std::max(occ, 1) * h->num_sms;
            h->occ_cache.emplace_back(fn, ctas);
        }
        const int64_t need = (nodes + NW - 1) / NW;
        int64_t gx = std::min<int64_t>(std::max<int64_t>(std::min<int64_t>(need, ctas), 1), h->nb_cap);
        return dim3(static_cast<unsigned>(gx), 1);
    }
#define P2G_NW_CASE(nw, ...) \
    case nw: { constexpr int NW = nw; __VA_ARGS__ } break;
#define P2G_NW_SWITCH(code, ...)               \
    switch (code) {                            \
        P2G_NW_CASE(4, __VA_ARGS__)            \
        P2G_NW_CASE(6, __VA_ARGS__)            \
        P2G_NW_CASE(7, __VA_ARGS__)            \
        P2G_NW_CASE(9, __VA_ARGS__)            \
        P2G_NW_CASE(10, __VA_ARGS__)           \
        P2G_NW_CASE(12, __VA_ARGS__)           \
        default: { constexpr int NW = 8; __VA_ARGS__ } break; \
    }

    static int gs_forward(p2g_handle* h, const double* f, double* s, int c, bool first) {
        Mat A = mat_of(h);
        const int nb = static_cast<int>(h->pat.color_rows[c] / h->pat.bs);
        const int ne = static_cast<int>(h->pat.color_rows[c + 1] / h->pat.bs);
        if (ne <= nb) return P2G_OK;
        if constexpr (Sh::W == 1) {
            if (first && blk1_hw(h)) {
                const bool stg = blk1_stg(h, 1);
                auto fn = stg ? k_gs_forward_b1s<3> : k_gs_forward_b1h<3>;
                const size_t smem = stg ? kB1sSmem : 0;
                dim3 g = blk1_grid(h, (ne - nb + 1) / 2, (const void*)fn, false, smem);
                fn<<<g, kBlock, smem, h->stream>>>(A, ntab(h), f, s, h->d_active, nb, ne);
                count_launch(h, KC_FWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
            if (first && blk1(h)) {
                P2G_BS_SWITCH(h->pat.bs, {
                    auto fn = k_gs_forward_b1<BS>;
                    dim3 g = blk1_grid(h, ne - nb, (const void*)fn, false);
                    fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), f, s, h->d_active, nb, ne);
                })
                count_launch(h, KC_FWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
        }
        if constexpr (Sh::S == 1) {
            if (first && blk(h)) {
                P2G_BS_SWITCH(h->pat.bs, {
                    auto fn = k_gs_forward_blk<Sh, BS>;
                    dim3 g = node_grid<Sh>(h, ne - nb, (const void*)fn);
                    fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), f, s, h->d_active, nb, ne);
                })
                count_launch(h, KC_FWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
        }
        if (first) {
            auto fn = k_gs_forward<Sh, true>;
            dim3 g = node_grid<Sh>(h, ne - nb, (const void*)fn);
            fn<<<g, kBlock, 0, h->stream>>>(A, f, s, h->d_active, nb, ne);
        } else {
            auto fn = k_gs_forward<Sh, false>;
            dim3 g = node_grid<Sh>(h, ne - nb, (const void*)fn);
            fn<<<g, kBlock, 0, h->stream>>>(A, f, s, h->d_active, nb, ne);
        }
        count_launch(h, KC_FWD);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // one backward colour phase; every phase of a sweep uses the same grid
    // (the largest colour's) so the LAST sweep's r.s partials accumulate into
    // the same rows phase after phase (first phase writes, later ones add)
    static int gs_backward(p2g_handle* h, const double* f, const double* xlo, double* s, int c,
                           bool last, int* rs_rows, bool first_phase) {
        Mat A = mat_of(h);
        const int nb = static_cast<int>(h->pat.color_rows[c] / h->pat.bs);
        const int ne = static_cast<int>(h->pat.color_rows[c + 1] / h->pat.bs);
        int64_t maxc = 1;
        for (int q = 0; q < h->pat.ncolors; ++q)
            maxc = std::max<int64_t>(maxc, (h->pat.color_rows[q + 1] - h->pat.color_rows[q]) / h->pat.bs);
        if constexpr (Sh::W == 1) {
            if (blk1_hw(h) && !std::getenv("P2G_NO_B1H_BWD")) {
                const bool stg = blk1_stg(h, 2);
                auto fn = stg ? (last ? k_gs_backward_b1s<3, true> : k_gs_backward_b1s<3, false>)
                              : (last ? k_gs_backward_b1h<3, true> : k_gs_backward_b1h<3, false>);
                const size_t smem = stg ? kB1sSmem : 0;
                dim3 g = blk1_grid(h, (maxc + 1) / 2, (const void*)fn, true, smem);
                // out-of-place last sweep (D9): also store s - s' for the recurrence's gathers
                // (d_t is free between the restriction and the next residual)
                const bool dl = last && xlo != s && h->d_t && !std::getenv("P2G_NO_DLT");
                h->dlt_of = dl ? s : (h->dlt_of == s ? nullptr : h->dlt_of);
                fn<<<g, kBlock, smem, h->stream>>>(A, ntab(h), f, xlo, s, h->d_active, nb, ne,
                                                last ? h->d_part_rs : nullptr, first_phase ? 0 : 1,
                                                dl ? h->d_t : nullptr);
                if (last) *rs_rows = g.x / kCluster;
                count_launch(h, KC_BWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
            if (blk1(h)) {
                P2G_BS_SWITCH(h->pat.bs, {
                    auto fn = last ? k_gs_backward_b1<BS, true> : k_gs_backward_b1<BS, false>;
                    dim3 g = blk1_grid(h, maxc, (const void*)fn, true);
                    fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), f, xlo, s, h->d_active, nb, ne,
                                                    last ? h->d_part_rs : nullptr,
                                                    first_phase ? 0 : 1);
                    if (last) *rs_rows = g.x / kCluster;
                })
                count_launch(h, KC_BWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
        }
        if constexpr (Sh::S == 1 && Sh::T >= 32) {
            if (stg_nw(h) > 0) {
                P2G_NW_SWITCH(stg_nw(h), {
                    if (last) {
                        auto fn = k_gs_backward_stg<Sh, NW, true>;
                        dim3 g = stg_grid<NW>(h, maxc, (const void*)fn);
                        fn<<<g, NW * 32, StgGeo<Sh, NW>::smem, h->stream>>>(
                            A, ntab(h), f, xlo, s, h->d_active, nb, ne, h->d_part_rs, first_phase ? 0 : 1);
                        *rs_rows = g.x;
                    } else {
                        auto fn = k_gs_backward_stg<Sh, NW, false>;
                        dim3 g = stg_grid<NW>(h, maxc, (const void*)fn);
                        fn<<<g, NW * 32, StgGeo<Sh, NW>::smem, h->stream>>>(
                            A, ntab(h), f, xlo, s, h->d_active, nb, ne, nullptr, 0);
                    }
                })
                count_launch(h, KC_BWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
        }
        if constexpr (Sh::S == 1) {
            if (blk(h)) {
                P2G_BS_SWITCH(h->pat.bs, {
                    if (last) {
                        auto fn = k_gs_backward_blk<Sh, BS, true>;
                        dim3 g = node_grid<Sh>(h, maxc, (const void*)fn, true);
                        fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), f, xlo, s, h->d_active, nb, ne,
                                                        h->d_part_rs, first_phase ? 0 : 1);
                        *rs_rows = g.x / kCluster;
                    } else {
                        auto fn = k_gs_backward_blk<Sh, BS, false>;
                        dim3 g = node_grid<Sh>(h, maxc, (const void*)fn, true);
                        fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), f, xlo, s, h->d_active, nb, ne,
                                                        nullptr, 0);
                    }
                })
                count_launch(h, KC_BWD);
                CU(cudaGetLastError());
                return P2G_OK;
            }
        }
        if (last) {
            auto fn = k_gs_backward<Sh, true>;
            dim3 g = node_grid<Sh>(h, maxc, (const void*)fn, true);
            fn<<<g, kBlock, 0, h->stream>>>(A, f, xlo, s, h->d_active, nb, ne, h->d_part_rs,
                                            first_phase ? 0 : 1);
            *rs_rows = g.x / kCluster;
        } else {
            auto fn = k_gs_backward<Sh, false>;
            dim3 g = node_grid<Sh>(h, maxc, (const void*)fn, true);
            fn<<<g, kBlock, 0, h->stream>>>(A, f, xlo, s, h->d_active, nb, ne, nullptr, 0);
        }
        count_launch(h, KC_BWD);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // Kp / p / pKp by the recurrence (D9); returns the partial row count
    static int kp_update(p2g_handle* h, const double* s_new, const double* s_prol, int* nb_out) {
        Mat A = mat_of(h);
        dim3 g = dot_grid(h);
        bool done = false;
        if constexpr (Sh::W == 1) {
            if (blk1_hw(h)) {
                const double* dlt = h->dlt_of == s_new ? h->d_t : nullptr;
                if (blk1_stg(h, 4))
                    k_kp_update_b1s<3><<<g, kBlock, kB1sSmem, h->stream>>>(
                        A, ntab(h), h->d_r, s_new, s_prol, h->d_Kp, h->d_p, h->d_beta, h->d_active,
                        h->d_part_dot, dlt);
                else
                    k_kp_update_b1h<3><<<g, kBlock, 0, h->stream>>>(A, ntab(h), h->d_r, s_new, s_prol,
                                                                     h->d_Kp, h->d_p, h->d_beta,
                                                                     h->d_active, h->d_part_dot, dlt);
                done = true;
            } else if (blk1_half(h)) {
                P2G_BS_SWITCH(h->pat.bs, {
                    k_kp_update_b1<BS><<<g, kBlock, 0, h->stream>>>(
                        A, ntab(h), h->d_r, s_new, s_prol, h->d_Kp, h->d_p, h->d_beta, h->d_active,
                        h->d_part_dot);
                })
                done = true;
            }
        }
        if constexpr (Sh::S == 1) {
            if (blk(h)) {
                P2G_BS_SWITCH(h->pat.bs, {
                    k_kp_update_blk<Sh, BS><<<g, kBlock, 0, h->stream>>>(
                        A, ntab(h), h->d_r, s_new, s_prol, h->d_Kp, h->d_p, h->d_beta, h->d_active,
                        h->d_part_dot);
                })
                done = true;
            }
        }
        if (!done)
            k_kp_update<Sh><<<g, kBlock, 0, h->stream>>>(A, h->d_r, s_new, s_prol, h->d_Kp, h->d_p,
                                                         h->d_beta, h->d_active, h->d_part_dot);
        if (nb_out) *nb_out = g.x / kCluster;
        count_launch(h, KC_SPMV);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    static int kp_rows(p2g_handle* h) { return dot_grid(h).x / kCluster; }

    static int jacobi(p2g_handle* h, const double* f, const double* s, double* s_out, bool last,
                      int* rs_rows, int kclass) {
        Mat A = mat_of(h);
        if (last) {
            auto fn = k_jacobi<Sh, true>;
            dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
            fn<<<g, kBlock, 0, h->stream>>>(A, f, s, s_out, h->d_active, h->cfg.omega,
                                            h->d_part_rs);
            *rs_rows = g.x / kCluster;
        } else {
            auto fn = k_jacobi<Sh, false>;
            dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
            fn<<<g, kBlock, 0, h->stream>>>(A, f, s, s_out, h->d_active, h->cfg.omega, nullptr);
        }
        count_launch(h, kclass);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    template <int TBW, int KM>
    static int restrict_ws(p2g_handle* h, const double* t, int* nb_out, KTag<KM>) {
        using WT = WsTile<TBW, KM>;
        auto fn = k_restrict_ws<TBW, KM>;
        const int n = static_cast<int>(h->pat.n);
        const int64_t need = (n + WT::RT - 1) / WT::RT;
        const int64_t tiles = h->Bp / TBW;
        int64_t gx = std::min<int64_t>(
            need, std::max<int64_t>(resident_ctas(h, (const void*)fn, true, WT::SMEM, kWsBlock, kWsCluster) / tiles,
                                    kWsCluster));
        gx = std::min<int64_t>(std::max<int64_t>(gx, 1), (int64_t)h->nb_cap * kWsCluster);
        gx = (gx + kWsCluster - 1) / kWsCluster * kWsCluster;
        dim3 g((unsigned)gx, (unsigned)tiles);
        fn<<<g, kWsBlock, WT::SMEM, h->stream>>>(n, h->Bp, t, h->d_phit, h->k, h->phi_ks, h->d_part_c);
        *nb_out = g.x / kWsCluster;
        return P2G_OK;
    }

    // c = Phi^T t with t = FORM(f, s) (RES_VECTOR: t = f).  The residual goes
    // to its own buffer d_t (Kp must survive the iteration for the recurrence).
    static int restrict_(p2g_handle* h, int form, const double* f, const double* s, int* nb_out) {
        Mat A = mat_of(h);
        const double* t = f;
        if (form != RES_VECTOR) {
            double* tb = h->d_t;
            bool done = false;
            if constexpr (Sh::W == 1) {
                if (form == RES_UPPER && blk1_hw(h)) {
                    const bool stg = blk1_stg(h, 8);
                    auto fn = stg ? k_residual_upper_b1s<3> : k_residual_upper_b1h<3>;
                    const size_t smem = stg ? kB1sSmem : 0;
                    dim3 g = blk1_grid(h, (nnodes(h) + 1) / 2, (const void*)fn, true, smem);
                    fn<<<g, kBlock, smem, h->stream>>>(A, ntab(h), s, tb, h->d_active);
                    done = true;
                } else if (form == RES_UPPER && blk1_half(h)) {
                    P2G_BS_SWITCH(h->pat.bs, {
                        auto fn = k_residual_upper_b1<BS>;
                        dim3 g = blk1_grid(h, nnodes(h), (const void*)fn, true);
                        fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), s, tb, h->d_active);
                    })
                    done = true;
                }
            }
            if constexpr (Sh::S == 1) {
                if (form == RES_UPPER && blk(h) && (h->pat.bs == 2 || P2G_RES_HEX_BLK)) {
                    P2G_BS_SWITCH(h->pat.bs, {
                        auto fn = k_residual_upper_blk<Sh, BS>;
                        dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
                        fn<<<g, kBlock, 0, h->stream>>>(A, ntab(h), s, tb, h->d_active);
                    })
                    done = true;
                }
            }
            if (done) {
            } else if (form == RES_UPPER) {
                auto fn = k_residual<Sh, RES_UPPER>;
                dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
                fn<<<g, kBlock, 0, h->stream>>>(A, f, s, tb, h->d_active, nullptr, nullptr);
            } else {
                auto fn = k_residual<Sh, RES_FULL>;
                dim3 g = node_grid<Sh>(h, nnodes(h), (const void*)fn, true);
                fn<<<g, kBlock, 0, h->stream>>>(A, f, s, tb, h->d_active, nullptr, nullptr);
            }
            count_launch(h, KC_RESID);
            t = tb;
        }
        const int k = h->k;
        const int n = static_cast<int>(h->pat.n);
        if constexpr (Sh::S == 1) {  // batched tiles: tensor-core restriction
            constexpr int TB = Sh::T;
            const int wsm = restrict_ws_mode();
            if (h->Bp % 64 == 0 && std::getenv("P2G_TMA") == nullptr &&
                (wsm == 2 || (wsm == 1 && n >= kRestrictWsRows))) {
                KSWITCH(k, {
                    if (h->Bp % 256 == 0) restrict_ws<256>(h, t, nb_out, KTag<KM>{});
                    else if (h->Bp % 128 == 0) restrict_ws<128>(h, t, nb_out, KTag<KM>{});
                    else restrict_ws<64>(h, t, nb_out, KTag<KM>{});
                });
                count_launch(h, KC_RESTRICT);
                CU(cudaGetLastError());
                return P2G_OK;
            }
            KSWITCH(k, {
                const bool tma = std::getenv("P2G_TMA") != nullptr;
                const bool wide = TB % 16 == 0 && !tma && restrict_wide();
                auto fn = tma ? k_restrict_mma<TB, KM>
                              : (wide ? k_restrict_reg2<(TB % 16 == 0 ? TB : 16), KM>
                                      : k_restrict_reg<TB, KM>);
                const size_t smem = tma ? MmaTile<TB, KM>::SMEM
                                        : (wide ? sizeof(double) * KM * TB : 0);
                const int64_t need = (n + 127) / 128;
                // every instance tile (grid.y) co-resident in ONE wave, marching over
                // the same rows together: a Phi row read from DRAM serves every tile
                // from L2 (one wave per tile re-streamed Phi once per tile)
                const int64_t tiles = h->Bp / TB;
                int64_t gx = std::min<int64_t>(
                    need, std::max<int64_t>(resident_ctas(h, (const void*)fn, true, smem) / tiles, kCluster));
                gx = std::min<int64_t>(std::max<int64_t>(gx, 1), h->nb_cap);
                gx = (gx + kCluster - 1) / kCluster * kCluster;
                dim3 g((unsigned)gx, (unsigned)(h->Bp / TB));
                fn<<<g, kBlock, smem, h->stream>>>(n, h->Bp, t, h->d_phit, k, h->phi_ks, h->d_part_c);
                *nb_out = g.x / kCluster;
            });
            count_launch(h, KC_RESTRICT);
            CU(cudaGetLastError());
            return P2G_OK;
        }
        KSWITCH(k, {
            using LSh = typename LocalShape<Sh, KM>::type;
            auto fn = k_restrict_vec<LSh, KM>;
            const int64_t need = (n + kWarps * LSh::R - 1) / (kWarps * LSh::R);
            int64_t gx = std::min<int64_t>(need, resident_ctas(h, (const void*)fn, true));
            gx = std::min<int64_t>(std::max<int64_t>(gx, 1), h->nb_cap);
            gx = (gx + kCluster - 1) / kCluster * kCluster;
            dim3 g((unsigned)gx, (unsigned)(h->Bp / LSh::T));
            fn<<<g, kBlock, 0, h->stream>>>(n, h->Bp, t, h->d_phi, k, h->d_active, h->d_part_c);
            *nb_out = g.x / kCluster;
        });
        count_launch(h, KC_RESTRICT);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    static int coarse(p2g_handle* h, int nblk) {
        k_coarse<<<h->Bp, kBlock, 0, h->stream>>>(h->Bp, h->k, nblk, h->d_part_c, h->d_L, h->d_e,
                                                   h->d_active);
        count_launch(h, KC_COARSE);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    template <int TBW, int KM>
    static void prolong_ws(p2g_handle* h, double* s, int n, bool assign, KTag<KM>) {
        using WT = WsPTile<TBW, KM>;
        auto fn = assign ? k_prolong_ws<TBW, KM, true> : k_prolong_ws<TBW, KM, false>;
        const int64_t need = (n + WT::RT - 1) / WT::RT;
        const int64_t tiles = h->Bp / TBW;
        int64_t gx = std::min<int64_t>(
            need, std::max<int64_t>(resident_ctas(h, (const void*)fn, false, WT::SMEM, kWsBlock) / tiles, 1));
        dim3 g((unsigned)std::max<int64_t>(gx, 1), (unsigned)tiles);
        fn<<<g, kWsBlock, WT::SMEM, h->stream>>>(n, h->Bp, s, h->d_phit, h->k, h->phi_ks, h->d_e,
                                                 h->d_active);
    }

    static int prolong(p2g_handle* h, double* s, bool assign) {
        const int k = h->k;
        const int n = static_cast<int>(h->pat.n + h->n_ghost);  // ghosts too (partitioned)
        if constexpr (Sh::S == 1) {  // batched tiles: bulk-copy pipelined prolongation
            constexpr int TB = Sh::T;
            const int wsm = prolong_ws_mode();
            if (h->Bp % 64 == 0 && std::getenv("P2G_TMA") == nullptr &&
                (wsm == 2 || (wsm == 1 && n >= kProlongWsRows))) {
                KSWITCH(k, {
                    if (h->Bp % 256 == 0) prolong_ws<256>(h, s, n, assign, KTag<KM>{});
                    else if (h->Bp % 128 == 0) prolong_ws<128>(h, s, n, assign, KTag<KM>{});
                    else prolong_ws<64>(h, s, n, assign, KTag<KM>{});
                });
                count_launch(h, KC_PROLONG);
                CU(cudaGetLastError());
                return P2G_OK;
            }
            KSWITCH(k, {
                // the TMA-staged (bulk copy + mbarrier) form pays on large systems
                // (c3 975 vs 1100 us, c4 190 vs 201), not on c2 (21 vs 18.5 us)
                const bool tma = std::getenv("P2G_TMA") != nullptr || n >= kProlongTmaRows;
                auto fn = tma ? (assign ? k_prolong_mma<TB, KM, true> : k_prolong_mma<TB, KM, false>)
                              : (assign ? k_prolong_reg<TB, KM, true> : k_prolong_reg<TB, KM, false>);
                const size_t smem = tma ? MmaTile<TB, KM>::SMEM : 0;
                const int64_t need = (n + 31) / 32;
                const int64_t tiles = h->Bp / TB;  // all tiles in one wave (Phi rows shared via L2)
                int64_t gx = std::min<int64_t>(
                    need, std::max<int64_t>(resident_ctas(h, (const void*)fn, false, smem) / tiles, 1));
                dim3 g((unsigned)std::max<int64_t>(gx, 1), (unsigned)(h->Bp / TB));
                fn<<<g, kBlock, smem, h->stream>>>(n, h->Bp, s, h->d_phit, k, h->phi_ks, h->d_e,
                                                   h->d_active);
            });
            count_launch(h, KC_PROLONG);
            CU(cudaGetLastError());
            return P2G_OK;
        }
        KSWITCH(k, {
            using LSh = typename LocalShape<Sh, KM>::type;
            auto fn = assign ? k_prolong<LSh, KM, true> : k_prolong<LSh, KM, false>;
            const int64_t need = (n + kWarps * LSh::R - 1) / (kWarps * LSh::R);
            int64_t gx = std::min<int64_t>(need, resident_ctas(h, (const void*)fn, false));
            dim3 g((unsigned)std::max<int64_t>(gx, 1), (unsigned)(h->Bp / LSh::T));
            fn<<<g, kBlock, 0, h->stream>>>(n, h->Bp, s, h->d_phi, k, h->d_e, h->d_active);
        });
        count_launch(h, KC_PROLONG);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    static int pupdate(p2g_handle* h, const double* s, bool init) {
        const int n = static_cast<int>(h->pat.n);
        constexpr int RL = 32 / Sh::W;
        const int64_t need = (n + kWarps * RL - 1) / (kWarps * RL);
        dim3 g(static_cast<unsigned>(std::min<int64_t>(need, (int64_t)h->num_sms * 8)),
               h->Bp / Sh::T);
        if (init)
            k_pupdate<Sh, true><<<g, kBlock, 0, h->stream>>>(n, h->Bp, s, h->d_p, h->d_beta,
                                                             h->d_active);
        else
            k_pupdate<Sh, false><<<g, kBlock, 0, h->stream>>>(n, h->Bp, s, h->d_p, h->d_beta,
                                                              h->d_active);
        count_launch(h, KC_PUPDATE);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // s = B r, B the POD-2G preconditioner (pod.hpp:264-267).  When `update`,
    // the PCG update of u and r precedes it in the same kernel (r = d_r).
    // *rs_rows receives the number of r.s partial rows written (post-smoother).
    static int precond(p2g_handle* h, bool update, const double* r, int* nb_rr, int* rs_rows) {
        const p2g_config& cfg = h->cfg;
        const int C = h->pat.ncolors;
        const double* rr = update ? h->d_r : r;
        double* cur = h->d_s;
        TRY(update_pre(h, update, rr, nb_rr));
        if (cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR) {
            for (int c = 1; c < C; ++c) TRY(gs_forward(h, rr, cur, c, true));
            for (int sw = 1; sw < cfg.pre_sweeps; ++sw)
                for (int c = 0; c < C; ++c) TRY(gs_forward(h, rr, cur, c, false));
        } else {
            for (int sw = 1; sw < cfg.pre_sweeps; ++sw) {
                double* nxt = cur == h->d_s ? h->d_s2 : h->d_s;
                int dummy = 0;
                TRY(jacobi(h, rr, cur, nxt, false, &dummy, KC_FWD));
                cur = nxt;
            }
        }
        if (h->k > 0) {
            const bool upper = cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR && cfg.pre_sweeps == 1 &&
                               cfg.residual_form == P2G_RESIDUAL_UPPER;
            int nbc = 0;
            TRY(restrict_(h, upper ? RES_UPPER : RES_FULL, rr, cur, &nbc));
            TRY(coarse(h, nbc));
            TRY(prolong(h, cur, false));
        }
        int rs_row = 0;
        if (cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR) {
            for (int sw = 0; sw < cfg.post_sweeps; ++sw) {
                const bool last = sw + 1 == cfg.post_sweeps;
                // the recurrence needs s' (the prolongated vector) intact: the
                // LAST backward sweep reads its L part from s' and writes d_s2
                const bool oop = last && kp_recurrence(h);
                double* out = oop ? h->d_s2 : cur;
                for (int c = C - 1; c >= 0; --c)
                    TRY(gs_backward(h, rr, cur, out, c, last, &rs_row, c == C - 1));
                if (oop) {
                    h->s_prol = cur;
                    cur = out;
                }
            }
        } else {
            for (int sw = 0; sw < cfg.post_sweeps; ++sw) {
                const bool last = sw + 1 == cfg.post_sweeps;
                double* nxt = cur == h->d_s ? h->d_s2 : h->d_s;
                TRY(jacobi(h, rr, cur, nxt, last, &rs_row, KC_BWD));
                cur = nxt;
            }
        }
        h->s_final = cur;
        if (rs_rows) *rs_rows = rs_row;
        return P2G_OK;
    }

    // one PCG iteration (krylov.hpp:272-288).  Reference form: SpMV first,
    // p update last.  Recurrence form (D9): the body starts at alpha (pKp
    // partials of the previous kp_update / prologue SpMV) and ends with the
    // half-pass kp_update that produces Kp, p and pKp for the next iteration.
    static int iteration(p2g_handle* h, bool in_graph) {
        int nb_dot = 0, nb_rr = 0, rs_rows = 0;
        const bool rec = kp_recurrence(h);
        if (rec)
            nb_dot = kp_rows(h);
        else
            TRY(spmv(h, h->d_p, h->d_Kp, true, &nb_dot));
        const int wb = 8;  // warps per block for the per-instance reducers
        k_alpha<<<(h->Bp + wb - 1) / wb, wb * 32, 0, h->stream>>>(h->Bp, nb_dot, h->d_part_dot,
                                                                  h->d_rsold, h->d_alpha,
                                                                  h->d_active, h->d_status);
        count_launch(h, KC_REDUCE);
        TRY(precond(h, true, nullptr, &nb_rr, &rs_rows));
        k_finalize<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(
            h->Bp, rs_rows, h->d_part_rs, nb_rr, h->d_part_rr, h->d_fnorm, h->d_rsold, h->d_beta,
            h->d_rel, h->d_iters, h->d_active, h->d_status, h->d_hist, h->d_prm, h->d_flag_ticket,
            h->cond, in_graph ? 1 : 0);
        count_launch(h, KC_REDUCE);
        if (rec)
            TRY(kp_update(h, h->s_final, h->s_prol, nullptr));
        else
            TRY(pupdate(h, h->s_final, false));
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // One pod2g_solve cycle (pod.hpp:243-250: op.cycle(f, u); r = f - K u):
    // r1 forward sweeps on u (full rows), t = f - K u, coarse correction,
    // r2 FORWARD sweeps (adjoint_post = false, pod.hpp:196-207), the true
    // residual with its norm partials, bookkeeping.
    static int cycle(p2g_handle* h, bool in_graph) {
        const int C = h->pat.ncolors;
        for (int sw = 0; sw < h->cfg.pre_sweeps; ++sw)
            for (int c = 0; c < C; ++c) TRY(gs_forward(h, h->d_b, h->d_u, c, false));
        if (h->k > 0) {
            int nbc = 0;
            TRY(restrict_(h, RES_FULL, h->d_b, h->d_u, &nbc));
            TRY(coarse(h, nbc));
            TRY(prolong(h, h->d_u, false));
        }
        for (int sw = 0; sw < h->cfg.post_sweeps; ++sw)
            for (int c = 0; c < C; ++c) TRY(gs_forward(h, h->d_b, h->d_u, c, false));
        int nb = 0;
        TRY(residual(h, h->d_b, h->d_u, h->d_r, &nb));
        k_cycle_finalize<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(
            h->Bp, nb, h->d_part_rr, h->d_fnorm, h->d_rel, h->d_iters, h->d_active, h->d_hist,
            h->d_prm, h->d_flag_ticket, h->cyc_cond, in_graph ? 1 : 0);
        count_launch(h, KC_REDUCE);
        CU(cudaGetLastError());
        return P2G_OK;
    }

    // ---- setup: A_c = Phi^T K Phi per instance, then Cholesky
    static int coarse_setup(p2g_handle* h, bool factor = true) {
        const int k = h->k;
        const int n = static_cast<int>(h->pat.n);
        Mat A = mat_of(h);
        using MSh = ASh;  // one instance per lane
        // instance chunk so that Y = n*k*Bt doubles stays below ~4 GiB
        int Bt = h->Bp;
        while (Bt > MSh::T && (size_t)n * k * Bt * 8 > ((size_t)4 << 30)) Bt /= 2;
        Bt = std::max(Bt, MSh::T);
        const int ncol = k * Bt;
        int occ_blocks = h->num_sms * 2;
        const size_t part_count = (size_t)occ_blocks * k * ncol;
        TRY(ensure(h, h->d_Y, (size_t)n * k * Bt));
        TRY(ensure(h, h->d_part_ac, part_count));
        double* Y = h->d_Y;
        double* part = h->d_part_ac;
        int st = P2G_OK;
        for (int bofs = 0; bofs < h->Bp && st == P2G_OK; bofs += Bt) {
            KSWITCH(k, {
                auto fn = k_spmm_phi<MSh, KM>;
                int occ = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, kBlock, 0);
                occ = std::max(occ, 1);
                const int64_t need = (n / h->pat.bs + kWarps * MSh::R - 1) / (kWarps * MSh::R);
                dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)h->num_sms * occ)),
                       (unsigned)((Bt + MSh::T - 1) / MSh::T));
                fn<<<g, kBlock, 0, h->stream>>>(A, h->d_phi, k, bofs, Bt, Y); ++h->launches_executed;
                // Phi^T Y: the restriction's DMMA kernel with Y's k*Bt columns as
                // the "instances" (row stride ncol), one partial row per cluster
                // (the [blk][a][ncol] layout k_reduce_ac reads); the CUDA-core
                // k_restrict_cols remains for column counts off the 32 grid
                int nblk = 0;
                if (ncol % 32 == 0 && !std::getenv("P2G_AC_CUDACORE")) {
                    auto launch = [&](auto fr, int TB) {
                        const int64_t need = (n + 127) / 128;
                        int64_t gx = std::min<int64_t>(need, resident_ctas(h, (const void*)fr, true));
                        gx = std::min<int64_t>(std::max<int64_t>(gx, 1), occ_blocks);
                        gx = std::max<int64_t>(gx / kCluster, 1) * kCluster;
                        dim3 g2((unsigned)gx, (unsigned)(ncol / TB));
                        fr<<<g2, kBlock, 0, h->stream>>>(n, ncol, Y, h->d_phit, k, h->phi_ks, part);
                        nblk = (int)(gx / kCluster);
                    };
                    if (ncol % 64 == 0) launch(k_restrict_reg<64, KM>, 64);
                    else launch(k_restrict_reg<32, KM>, 32);
                } else {
                    auto fr = k_restrict_cols<KM>;
                    dim3 g2((unsigned)std::min<int64_t>(occ_blocks, (n + kWarps - 1) / kWarps),
                            (unsigned)((ncol + 31) / 32));
                    fr<<<g2, kBlock, 0, h->stream>>>(n, ncol, Y, h->d_phi, k, part);
                    nblk = (int)g2.x;
                }
                ++h->launches_executed;
                const int total = Bt * k * k;
                k_reduce_ac<<<(total + 7) / 8, 256, 0, h->stream>>>(nblk, k, Bt, bofs, part, h->d_Ac); ++h->launches_executed;
            });
            if (cudaGetLastError() != cudaSuccess) st = P2G_ECUDA;
        }
        cudaStreamSynchronize(h->stream);
        if (st != P2G_OK) {
            h->err = "coarse_setup: kernel launch failed";
            return st;
        }
        if (!factor) return P2G_OK;
        k_cholesky<<<(h->B + 7) / 8, 256, 0, h->stream>>>(h->B, k, h->d_Ac, h->d_L,
                                                          h->d_setup_status); ++h->launches_executed;
        CU(cudaGetLastError());
        return P2G_OK;
    }
};

template <class F>
int dispatch(p2g_handle* h, F&& f) {
    switch (h->shape) {
        case SH_B1A: return f(Run<ShB1a>{});
        case SH_B1B: return f(Run<ShB1b>{});
        case SH_B8: return f(Run<ShB8>{});
        case SH_B32: return f(Run<ShB32>{});
        default: return f(Run<ShB64>{});
    }
}

// ---------------------------------------------------------------- layout helpers
// host [B][len] (natural order) -> device [len][Bp] (permuted by map)
int upload_interleaved(p2g_handle* h, const double* src_host, const double* src_dev, int64_t len,
                       const int64_t* d_map, double* dst) {
    const int B = h->B;
    // instance chunk that fits the staging buffer
    if (src_dev) {
        dim3 g((unsigned)((len + 31) / 32), (unsigned)((h->Bp + 31) / 32));
        k_gather_interleave<<<g, 256, 0, h->stream>>>(src_dev, len, B, d_map, len, dst, h->Bp, 0,
                                                      0.0); ++h->launches_executed;
        CU(cudaGetLastError());
        return P2G_OK;
    }
    const size_t per = (size_t)len * sizeof(double);
    size_t want = std::min<size_t>((size_t)B * per, (size_t)1 << 31);
    want = std::max(want, per);
    if (h->stage_bytes < want) {
        dfree(h->d_stage);
        CU(cudaMalloc(&h->d_stage, want));
        h->stage_bytes = want;
    }
    const int chunk = static_cast<int>(std::max<size_t>(1, h->stage_bytes / per));
    for (int b0 = 0; b0 < B; b0 += chunk) {
        const int nb = std::min(chunk, B - b0);
        CU(cudaMemcpyAsync(h->d_stage, src_host + (size_t)b0 * len, (size_t)nb * per,
                           cudaMemcpyHostToDevice, h->stream));
        // rows of this chunk: columns [b0, b0+nb)
        dim3 g((unsigned)((len + 31) / 32), (unsigned)((h->Bp + 31) / 32));
        k_gather_interleave<<<g, 256, 0, h->stream>>>(h->d_stage, len, nb, d_map, len, dst, h->Bp,
                                                      b0, 0.0); ++h->launches_executed;
        CU(cudaGetLastError());
        CU(cudaStreamSynchronize(h->stream));  // staging buffer reuse
    }
    return P2G_OK;
}

int download_interleaved(p2g_handle* h, const double* src, double* dst_host, double* dst_dev) {
    const int64_t n = h->pat.n;
    dim3 g((unsigned)((n + 31) / 32), (unsigned)((h->Bp + 31) / 32));
    if (dst_dev) {
        k_scatter_deinterleave<<<g, 256, 0, h->stream>>>(src, h->Bp, n, h->d_perm, h->B, dst_dev); ++h->launches_executed;
        CU(cudaGetLastError());
        return P2G_OK;
    }
    const size_t bytes = (size_t)h->B * n * sizeof(double);
    if (h->stage_bytes < bytes) {
        dfree(h->d_stage);
        CU(cudaMalloc(&h->d_stage, bytes));
        h->stage_bytes = bytes;
    }
    k_scatter_deinterleave<<<g, 256, 0, h->stream>>>(src, h->Bp, n, h->d_perm, h->B, h->d_stage); ++h->launches_executed;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(dst_host, h->d_stage, bytes, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return P2G_OK;
}

void destroy_graph(p2g_handle* h) {
    if (h->loop_exec) cudaGraphExecDestroy(h->loop_exec);
    h->loop_exec = nullptr;
    if (h->cyc_exec) cudaGraphExecDestroy(h->cyc_exec);
    h->cyc_exec = nullptr;
}

int alloc_batch(p2g_handle* h) {
    const size_t nv = (size_t)(h->pat.n + h->n_ghost) * h->Bp;
    // two doubles of slack: the staged B = 1 kernels copy whole 16-byte pairs
    TRY(dalloc(h, h->d_vals, (size_t)h->pat.nnz * h->Bp + 2));
    CU(cudaMemsetAsync(h->d_vals, 0, (size_t)h->pat.nnz * h->Bp * sizeof(double), h->stream));
    for (double** p : {&h->d_u, &h->d_r, &h->d_s, &h->d_s2, &h->d_p, &h->d_Kp, &h->d_b, &h->d_t}) {
        TRY(dalloc(h, *p, nv));
        CU(cudaMemsetAsync(*p, 0, nv * sizeof(double), h->stream));
    }
    for (double** p : {&h->d_alpha, &h->d_beta, &h->d_rsold, &h->d_fnorm, &h->d_rel})
        TRY(dalloc(h, *p, h->Bp));
    for (int** p : {&h->d_active, &h->d_iters, &h->d_status, &h->d_setup_status, &h->d_all})
        TRY(dalloc(h, *p, h->Bp));
    std::vector<int> ones(h->Bp, 0);
    for (int b = 0; b < h->B; ++b) ones[b] = 1;
    CU(cudaMemcpy(h->d_all, ones.data(), sizeof(int) * h->Bp, cudaMemcpyHostToDevice));
    // partials: up to nb_cap blocks per kernel
    h->nb_cap = h->num_sms * 8;
    TRY(dalloc(h, h->d_part_dot, (size_t)h->nb_cap * h->Bp));
    TRY(dalloc(h, h->d_part_rr, (size_t)h->nb_cap * h->Bp));
    TRY(dalloc(h, h->d_part_ff, (size_t)h->nb_cap * h->Bp));
    h->part_rs_rows = h->nb_cap * std::max(1, h->pat.ncolors);
    TRY(dalloc(h, h->d_part_rs, (size_t)h->part_rs_rows * h->Bp));
    return P2G_OK;
}

int choose_shape(p2g_handle* h, int B) {
    if (B == 1) {
        h->shape = SH_B1A;  // 4 rows x 8 slots per warp (more rows in flight than a warp per row)
        const char* b1 = std::getenv("P2G_B1_SHAPE");  // tuning knob: "b" = a warp per row
        if (b1 && b1[0] == 'b') h->shape = SH_B1B;
        h->Bp = 1;
    } else if (B <= 8) {
        h->shape = SH_B8;
        h->Bp = 8;
    } else if (B <= 32) {
        h->shape = SH_B32;
        h->Bp = 32;
    } else {
        h->shape = SH_B64;
        h->Bp = (B + 63) / 64 * 64;
    }
    // tuning knob: P2G_WIDE=0 runs large batches with one instance per lane
    // (32-wide tiles) instead of double2 lanes (64-wide tiles)
    if (h->shape == SH_B64) {
        const char* w = std::getenv("P2G_WIDE");
        if (w && w[0] == '0') h->shape = SH_B32;
    }
    return P2G_OK;
}

int set_values_impl(p2g_handle* h, int32_t batch, const double* host, const double* dev,
                    bool upload = true) {
    REQ(h->have_pattern, P2G_ESTATE, "p2g_set_values: pattern not set");
    REQ(batch >= 1, P2G_EINVAL, "p2g_set_values: batch must be >= 1");
    REQ(!upload || host || dev, P2G_EINVAL, "p2g_set_values: null values");
    
    h->setup_done = false;
    const int oldBp = h->Bp;
    const int oldB = h->B;
    const int64_t bp_est = batch <= 32 ? (batch == 1 ? 1 : (batch <= 8 ? 8 : 32)) : (batch + 63) / 64 * 64;
    REQ((uint64_t)h->pat.n * (uint64_t)bp_est < ((uint64_t)1 << 32), P2G_EINVAL,
        "p2g_set_values: n * batch exceeds 2^32 vector elements (split the batch)");
    h->B = batch;
    choose_shape(h, batch);
    if (h->Bp != oldBp || oldB != batch || !h->d_vals) TRY(alloc_batch(h));
    if (h->k >= 0) {
        TRY(ensure(h, h->d_e, (size_t)std::max(h->k, 1) * h->Bp));
        TRY(ensure(h, h->d_L, (size_t)std::max(h->k * h->k, 1) * h->Bp));
        TRY(ensure(h, h->d_Ac, (size_t)std::max(h->k * h->k, 1) * h->Bp));
        TRY(ensure(h, h->d_part_c, (size_t)h->nb_cap * std::max(h->k, 1) * h->Bp));
    }
    if (host || dev) TRY(upload_interleaved(h, host, dev, h->pat.nnz, h->d_vperm, h->d_vals));
    CU(cudaStreamSynchronize(h->stream));
    h->have_values = true;
    return P2G_OK;
}

// values generated on the device from a structured mesh
int assemble_impl(p2g_handle* h, const p2g_mesh* m, int32_t batch, const double* E,
                  int64_t row_begin, bool E_on_device) {
    MeshDesc md;
    REQ(mesh_desc(m, md), P2G_EINVAL, "assemble: null mesh");
    REQ(h->have_pattern, P2G_ESTATE, "assemble: pattern not set");
    REQ(E && batch >= 1, P2G_EINVAL, "assemble: null moduli");
    TRY(set_values_impl(h, batch, nullptr, nullptr, false));
    // device copies of Ke, the generator row offsets, the moduli
    double* dKe = nullptr;
    unsigned long long* drp = nullptr;
    double *dE = nullptr, *dEt = nullptr;
    const size_t ne = (size_t)md.nelem * batch;
    CU(cudaMalloc(&dKe, sizeof(double) * md.ned * md.ned));
    CU(cudaMalloc(&drp, sizeof(unsigned long long) * (md.n + 1)));
    CU(cudaMalloc(&dEt, sizeof(double) * ne));
    CU(cudaMemcpyAsync(dKe, md.Ke, sizeof(double) * md.ned * md.ned, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(drp, md.rp, sizeof(unsigned long long) * (md.n + 1), cudaMemcpyHostToDevice,
                       h->stream));
    const double* Esrc = E;
    if (!E_on_device) {
        CU(cudaMalloc(&dE, sizeof(double) * ne));
        CU(cudaMemcpyAsync(dE, E, sizeof(double) * ne, cudaMemcpyHostToDevice, h->stream));
        Esrc = dE;
    }
    k_transpose_E<<<4096, 256, 0, h->stream>>>(Esrc, batch, md.nelem, dEt);
    AsmDesc d;
    d.dim = md.dim;
    d.ned = md.ned;
    d.nx = md.nx;
    d.ny = md.ny;
    d.nz = md.nz;
    d.row_begin = row_begin;
    d.q_base = (long long)md.rp[row_begin];
    d.Ke = dKe;
    d.rpg = drp;
    Mat A = mat_of(h);
    const int64_t need = (h->pat.n + kWarps - 1) / kWarps;
    k_assemble<<<(unsigned)std::min<int64_t>(need, (int64_t)h->num_sms * 8), kBlock, 0, h->stream>>>(
        A, d, h->d_perm, h->d_vperm, dEt, batch, h->d_vals);
    h->launches_executed += 2;
    const cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(h->stream);
    cudaFree(dKe);
    cudaFree(drp);
    cudaFree(dEt);
    if (dE) cudaFree(dE);
    CU(e);
    return P2G_OK;
}

std::vector<uint64_t> graph_key_of(p2g_handle* h) {
    auto u = [](const void* p) { return (uint64_t)(uintptr_t)p; };
    return {u(h->d_vals), u(h->d_phi), u(h->d_phit), u(h->d_e), u(h->d_L), u(h->d_part_c), u(h->d_u), u(h->d_r),
            u(h->d_s), u(h->d_s2), u(h->d_p), u(h->d_Kp), u(h->d_t), u(h->d_hist), (uint64_t)h->Bp,
            (uint64_t)h->B, (uint64_t)h->k, (uint64_t)h->shape, (uint64_t)h->cfg.smoother,
            (uint64_t)h->cfg.pre_sweeps, (uint64_t)h->cfg.post_sweeps,
            (uint64_t)h->cfg.residual_form, (uint64_t)std::llround(h->cfg.omega * 1e15),
            (uint64_t)h->cfg.kp_update};
}

// cycle == false: the PCG iteration loop; true: the pod2g_solve cycle loop
int build_loop_graph(p2g_handle* h, bool cycle = false) {
    cudaGraphExec_t& exec = cycle ? h->cyc_exec : h->loop_exec;
    if (exec) cudaGraphExecDestroy(exec);
    exec = nullptr;
    cudaGraph_t outer = nullptr;
    CU(cudaGraphCreate(&outer, 0));
    cudaGraphConditionalHandle cond;
    CU(cudaGraphConditionalHandleCreate(&cond, outer, 0, 0));
    (cycle ? h->cyc_cond : h->cond) = cond;
    // upstream kernel: condition := any instance active
    cudaKernelNodeParams kp = {};
    int Bp = h->Bp;
    int* act = h->d_active;
    void* args[] = {&act, &Bp, &cond};
    kp.func = (void*)k_set_cond;
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(256);
    kp.sharedMemBytes = 0;
    kp.kernelParams = args;
    cudaGraphNode_t setn;
    CU(cudaGraphAddKernelNode(&setn, outer, nullptr, 0, &kp));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CU(cudaGraphAddNode(&wnode, outer, &setn, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CU(cudaStreamBeginCaptureToGraph(h->stream, body, nullptr, nullptr, 0,
                                     cudaStreamCaptureModeRelaxed));
    const int64_t before = h->launch_counter;
    h->capturing = true;
    int st = dispatch(h, [&](auto R) -> int {
        return cycle ? decltype(R)::cycle(h, true) : decltype(R)::iteration(h, true);
    });
    h->capturing = false;
    cudaGraph_t captured = nullptr;
    cudaError_t ce = cudaStreamEndCapture(h->stream, &captured);
    if (st != P2G_OK) {
        cudaGraphDestroy(outer);
        return st;
    }
    if (ce != cudaSuccess) {
        cudaGraphDestroy(outer);
        h->err = std::string("graph capture: ") + cudaGetErrorString(ce);
        return P2G_ECUDA;
    }
    (cycle ? h->launches_per_cycle : h->launches_per_iter) = h->launch_counter - before;
    (cycle ? h->cyc_key : h->graph_key) = graph_key_of(h);
    cudaError_t ie = cudaGraphInstantiate(&exec, outer, 0);
    cudaGraphDestroy(outer);
    if (ie != cudaSuccess) {
        h->err = std::string("graph instantiate: ") + cudaGetErrorString(ie);
        return P2G_ECUDA;
    }
    return P2G_OK;
}

// u = predict(model, theta_b) per instance: MLP latent coordinates into the
// coarse-coefficient buffer, then the prolongation in assign mode (lift)
int surrogate_x0(p2g_handle* h, double* u) {
    const size_t smem = sizeof(double) * 2 * (size_t)h->sg_wmax;
    if (smem > 48 * 1024)
        CU(cudaFuncSetAttribute(k_mlp_latent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
    k_mlp_latent<<<h->B, kBlock, smem, h->stream>>>(h->sg_layers, h->d_sg_widths, h->sg_act,
                                                    h->d_sg_W, h->d_sg_b, h->d_sg_norm,
                                                    h->d_theta, h->sg_wmax, h->Bp, h->d_e);
    ++h->launches_executed;
    CU(cudaGetLastError());
    return dispatch(h, [&](auto R) -> int { return decltype(R)::prolong(h, u, true); });
}

bool eager_loop() {
    static const bool e = [] {
        const char* v = std::getenv("P2G_EAGER_LOOP");
        return v && v[0] == '1';
    }();
    return e;
}

// Single-cluster persistent loop (k_pcg_cluster): one instance, default
// configuration (multicolour GS, one pre / post sweep, upper residual, Kp
// recurrence), Q4-shaped pattern whose matrix fits the cluster's shared memory.
// P2G_CLUSTER_NNZ = largest nnz taken.  OFF by default (0): measured on c1 at
// 55 us per iteration against 51 us for the captured loop -- a phase costs one
// global round trip (~1 us under the cluster barrier's release) plus the
// barrier (~0.9 us), no less than a kernel boundary inside a graph
// (P2G_CLUSTER_TRACE=1 prints the phase clock, c1).
bool cluster_loop_ok(const p2g_handle* h) {
    const char* e = std::getenv("P2G_CLUSTER_NNZ");
    const long long lim = e ? std::atoll(e) : 0;
    const int nl = static_cast<int>((h->pat.n / 2 + kClSize - 1) / kClSize);
    return h->B == 1 && h->Bp == 1 && lim > 0 && (long long)h->pat.nnz <= lim && kp_recurrence(h) &&
           h->cfg.pre_sweeps == 1 && h->cfg.post_sweeps == 1 &&
           h->cfg.residual_form == P2G_RESIDUAL_UPPER && h->k <= kClKmax && h->pat.ncolors <= 16 &&
           h->pat.ncolors >= 1 && h->node_blk && h->pat.bs == kClBS && h->nmax * kClBS <= kClRL &&
           cluster_loop_smem(nl, h->k) <= 200 * 1024;
}

// cycle == false: pcg_solve (krylov.hpp:243-297) with the POD-2G preconditioner;
// cycle == true: pod2g_solve (pod.hpp:224-256), iters = cycles
// start a requested prefetch copy (p2g_prefetch_values) on the copy stream
int start_prefetch(p2g_handle* h) {
    if (!h->pref_host || h->pref_started) return P2G_OK;
    const size_t bytes = (size_t)h->pref_B * h->pat.nnz * sizeof(double);
    CU(cudaMemcpyAsync(h->d_pref, h->pref_host, bytes, cudaMemcpyHostToDevice, h->cstream));
    CU(cudaEventRecord(h->pref_ev, h->cstream));
    h->pref_started = true;
    return P2G_OK;
}

int solve_impl(p2g_handle* h, const double* b_host, const double* b_dev, const double* x0_host,
               const double* x0_dev, int32_t x0_mode, double tol, int64_t max_iter,
               double* x_host, double* x_dev, int64_t* iters, int32_t* converged, int32_t* status,
               double* hist, int64_t hist_cap, bool cycle = false) {
    REQ(h->setup_done, P2G_ESTATE, "p2g_solve: p2g_setup not called");
    REQ(!cycle || h->cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR, P2G_EINVAL,
        "p2g_pod2g_solve: the standalone iteration uses the Gauss-Seidel smoother (pod.hpp:227)");
    REQ(b_host || b_dev, P2G_EINVAL, "p2g_solve: null right-hand side");
    REQ(x0_mode >= 0 && x0_mode <= 3, P2G_EINVAL, "p2g_solve: bad x0_mode");
    REQ(x0_mode != P2G_X0_SURROGATE || (h->sg_layers > 0 && h->theta_set),
        P2G_ESTATE, "p2g_solve: surrogate x0 needs p2g_set_surrogate and p2g_set_theta");
    REQ(x0_mode != P2G_X0_SURROGATE || h->sg_widths.back() == h->k, P2G_EINVAL,
        "predict: surrogate output width differs from the basis rank");
    REQ(x0_mode != P2G_X0_GIVEN || x0_host || x0_dev, P2G_EINVAL, "p2g_solve: null x0");
    REQ(x0_mode != P2G_X0_REDUCED || h->k > 0, P2G_EINVAL,
        "p2g_solve: reduced initial guess needs a basis");
    REQ(max_iter >= 0 && hist_cap >= 0, P2G_EINVAL, "p2g_solve: negative max_iter/hist_cap");
    const int64_t cap_dev = std::max<int64_t>(hist_cap, 1);
    // sized by bytes (ensure), so a later, larger batch on the same handle regrows it
    TRY(ensure(h, h->d_hist, (size_t)cap_dev * h->Bp));
    if (cycle) {
        if (!h->cyc_exec || h->cyc_key != graph_key_of(h)) TRY(build_loop_graph(h, true));
    } else if (!h->loop_exec || h->graph_key != graph_key_of(h)) {
        TRY(build_loop_graph(h));
    }
    const int64_t lc0 = h->launches_executed;
    h->has_state = !cycle;
    SolveParams prm{tol, (long long)max_iter, (long long)hist_cap};
    CU(cudaMemcpyAsync(h->d_prm, &prm, sizeof(prm), cudaMemcpyHostToDevice, h->stream));

    // inputs: b, x0 (H2D inside the caller's timed region for e2e)
    CU(cudaEventRecord(h->ev[0], h->stream));
    TRY(upload_interleaved(h, b_host, b_dev, h->pat.n, h->d_perm, h->d_b));
    TRY(start_prefetch(h));  // the next batch's values follow b over the link
    CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                       h->stream));
    int st = dispatch(h, [&](auto R) -> int {
        using Rn = decltype(R);
        if (x0_mode == P2G_X0_GIVEN) {
            TRY(upload_interleaved(h, x0_host, x0_dev, h->pat.n, h->d_perm, h->d_u));
        } else if (x0_mode == P2G_X0_REDUCED) {
            int nbc = 0;
            TRY(Rn::restrict_(h, RES_VECTOR, h->d_b, nullptr, &nbc));
            TRY(Rn::coarse(h, nbc));
            TRY(Rn::prolong(h, h->d_u, true));
        } else if (x0_mode == P2G_X0_SURROGATE) {
            TRY(surrogate_x0(h, h->d_u));
        } else {
            CU(cudaMemsetAsync(h->d_u, 0, (size_t)h->pat.n * h->Bp * sizeof(double), h->stream));
        }
        int nb = 0;
        TRY(Rn::residual(h, h->d_b, h->d_u, h->d_r, &nb));
        k_init_rel<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(
            h->Bp, h->B, nb, h->d_part_rr, h->d_part_ff, h->d_fnorm, h->d_rel, h->d_iters,
            h->d_active, h->d_status, h->d_setup_status, h->d_hist, h->d_prm);
        count_launch(h, KC_REDUCE);
        if (cycle) return P2G_OK;  // pod2g_solve: u, r, rel and the history entry 0 only
        // s = T r0 ; rs_old = r.s ; p = s   (krylov.hpp:262-266)
        int rs_rows = 0;
        TRY(Rn::precond(h, false, h->d_r, nullptr, &rs_rows));
        k_init_rs<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(h->Bp, rs_rows, h->d_part_rs,
                                                           h->d_rsold, h->d_active, h->d_status);
        count_launch(h, KC_REDUCE);
        TRY(Rn::pupdate(h, h->s_final, true));
        if (kp_recurrence(h)) TRY(Rn::spmv(h, h->d_p, h->d_Kp, true, nullptr));  // Kp_0, pKp_0
        return P2G_OK;
    });
    if (st != P2G_OK) return st;
    CU(cudaEventRecord(h->ev[1], h->stream));
    int64_t eager_iters = -1;
    bool cluster_loop = false;
    if (eager_loop()) {
        // profiling aid (P2G_EAGER_LOOP=1): the same loop body launched eagerly so
        // ncu lists every kernel (it does not descend into the conditional-WHILE
        // graph body); the host polls the active flags every 16 iterations --
        // surplus iterations are fully masked no-ops
        std::vector<int> act(h->Bp);
        for (eager_iters = 0;; ++eager_iters) {
            if (eager_iters % 16 == 0) {
                CU(cudaMemcpyAsync(act.data(), h->d_active, sizeof(int) * h->Bp,
                                   cudaMemcpyDeviceToHost, h->stream));
                CU(cudaStreamSynchronize(h->stream));
                if (std::none_of(act.begin(), act.end(), [](int a) { return a != 0; })) break;
            }
            TRY(dispatch(h, [&](auto R) -> int {
                return cycle ? decltype(R)::cycle(h, false) : decltype(R)::iteration(h, false);
            }));
        }
    } else if (!cycle && cluster_loop_ok(h)) {
        // small single system: the whole loop in one kernel on one cluster
        ClusterLoop A;
        A.n = static_cast<int>(h->pat.n);
        A.nl = static_cast<int>((h->pat.n / kClBS + kClSize - 1) / kClSize);
        A.k = h->k;
        A.ncolors = h->pat.ncolors;
        A.nrows_pkp = dispatch(h, [&](auto R) -> int { return decltype(R)::kp_rows(h); });
        for (int c = 0; c <= h->pat.ncolors; ++c) A.color_rows[c] = static_cast<int>(h->pat.color_rows[c]);
        A.rp = h->d_rp;
        A.ci = h->d_ci;
        A.dpos = h->d_dpos;
        A.vals = h->d_vals;
        A.phi = h->d_phi;
        A.Lfac = h->d_L;
        A.u = h->d_u;
        A.r = h->d_r;
        A.p = h->d_p;
        A.Kp = h->d_Kp;
        A.s = h->d_s;
        A.s2 = h->d_s2;
        A.part_pkp = h->d_part_dot;
        A.rs_old = h->d_rsold;
        A.rel = h->d_rel;
        A.hist = h->d_hist;
        A.beta = h->d_beta;
        A.alpha = h->d_alpha;
        A.fnorm = h->d_fnorm;
        A.iters = h->d_iters;
        A.active = h->d_active;
        A.status = h->d_status;
        A.prm = h->d_prm;
        const size_t smem = cluster_loop_smem(A.nl, A.k);
        CU(cudaFuncSetAttribute(k_pcg_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        A.trace = nullptr;
        const bool trace = std::getenv("P2G_CLUSTER_TRACE") != nullptr;
        if (trace) {
            CU(cudaMalloc(&A.trace, 64 * sizeof(long long)));
            CU(cudaMemset(A.trace, 0, 64 * sizeof(long long)));
        }
        k_pcg_cluster<<<kClSize, kClThreads, smem, h->stream>>>(A);
        if (trace) {
            long long tr[64];
            CU(cudaStreamSynchronize(h->stream));
            CU(cudaMemcpy(tr, A.trace, sizeof(tr), cudaMemcpyDeviceToHost));
            cudaFree(A.trace);
            std::fprintf(stderr, "k_pcg_cluster trace (cycles since the iteration's alpha):");
            for (int j = 0; j < 44; ++j)
                if (tr[j]) std::fprintf(stderr, " [%d]%lld", j, tr[j] - tr[44]);
            std::fprintf(stderr, "\n");
        }
        CU(cudaGetLastError());
        h->s_prol = h->d_s;
        h->s_final = h->d_s2;
        cluster_loop = true;
    } else {
        CU(cudaGraphLaunch(cycle ? h->cyc_exec : h->loop_exec, h->stream));
    }
    CU(cudaEventRecord(h->ev[2], h->stream));
    {
        const dim3 g((unsigned)std::min<int64_t>((h->pat.n + 255) / 256, 1024), h->B);
        k_check_finite<<<g, 256, 0, h->stream>>>(static_cast<int>(h->pat.n), h->Bp, h->d_u,
                                                  h->d_status); ++h->launches_executed;
        CU(cudaGetLastError());
    }
    if (x_host || x_dev) TRY(download_interleaved(h, h->d_u, x_host, x_dev));
    CU(cudaEventRecord(h->ev[3], h->stream));
    CU(cudaStreamSynchronize(h->stream));
    std::vector<int> it(h->Bp), stt(h->Bp);
    std::vector<double> rel(h->Bp);
    CU(cudaMemcpy(it.data(), h->d_iters, sizeof(int) * h->Bp, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(stt.data(), h->d_status, sizeof(int) * h->Bp, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(rel.data(), h->d_rel, sizeof(double) * h->Bp, cudaMemcpyDeviceToHost));
    int worst = P2G_OK;
    for (int b = 0; b < h->B; ++b) {
        if (iters) iters[b] = it[b];
        if (converged) converged[b] = rel[b] <= tol ? 1 : 0;
        if (status) status[b] = stt[b];
        if (stt[b] != P2G_OK) worst = stt[b];
    }
    if (hist && hist_cap > 0) {
        CU(cudaMemcpy(hist, h->d_hist, sizeof(double) * hist_cap * h->B,
                      cudaMemcpyDeviceToHost));
        for (int b = 0; b < h->B; ++b) {
            const int64_t len = std::min<int64_t>(it[b] + 1, hist_cap);
            for (int64_t q = len; q < hist_cap; ++q) hist[b * hist_cap + q] = NAN;
        }
    }
    float ms_all = 0, ms_loop = 0;
    cudaEventElapsedTime(&ms_all, h->ev[0], h->ev[3]);
    cudaEventElapsedTime(&ms_loop, h->ev[1], h->ev[2]);
    h->last_ms[0] = ms_all;
    h->last_ms[1] = ms_loop;
    int64_t maxit = 0;
    for (int b = 0; b < h->B; ++b) maxit = std::max<int64_t>(maxit, it[b]);
    if (cluster_loop)
        h->launches_executed += 1;
    else if (eager_iters < 0)
        h->launches_executed +=
            1 /*set_cond*/ + maxit * (cycle ? h->launches_per_cycle : h->launches_per_iter);
    h->launches_last_solve = h->launches_executed - lc0;
    if (worst != P2G_OK) h->err = "p2g_solve: at least one instance failed (see status)";
    return worst;
}

}  // namespace

namespace {
struct DevScratch {  // handle-free entry points: own stream and buffers
    cudaStream_t st = nullptr;
    std::vector<void*> bufs;
    ~DevScratch() {
        for (void* p : bufs) cudaFree(p);
        if (st) cudaStreamDestroy(st);
    }
    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        if (cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) return nullptr;
        bufs.push_back(p);
        return static_cast<T*>(p);
    }
};
}  // namespace

// ============================================================================ C-ABI
extern "C" {

void p2g_config_default(p2g_config* cfg) {
    if (!cfg) return;
    cfg->smoother = P2G_SMOOTHER_GS_MULTICOLOR;
    cfg->pre_sweeps = 1;
    cfg->post_sweeps = 1;
    cfg->residual_form = P2G_RESIDUAL_UPPER;
    cfg->omega = 0.5;
    cfg->kp_update = P2G_KP_RECURRENCE;
    cfg->reserved = 0;
}

int p2g_abi_version(void) { return P2G_ABI_VERSION; }

const char* p2g_status_string(int s) {
    switch (s) {
        case P2G_OK: return "ok";
        case P2G_EINVAL: return "invalid argument";
        case P2G_EBREAKDOWN: return "PCG breakdown (preconditioner or matrix not SPD)";
        case P2G_ENONFINITE: return "non-finite entries in solution";
        case P2G_ESINGULAR: return "coarse operator singular";
        case P2G_EZERODIAG: return "zero diagonal";
        case P2G_ECUDA: return "CUDA error";
        case P2G_ENCCL: return "NCCL error";
        case P2G_ESTATE: return "call order violated";
        default: return "unknown";
    }
}

int p2g_create(int device, p2g_handle** out) {
    if (!out) return P2G_EINVAL;
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return P2G_ECUDA;
    if (device < 0 || device >= ndev) return P2G_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return P2G_ECUDA;
    p2g_handle* h = new p2g_handle();
    h->device = device;
    cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete h;
        return P2G_ECUDA;
    }
    for (auto& e : h->ev) cudaEventCreate(&e);
    for (auto& e : h->kev) cudaEventCreate(&e);
    if (cudaMalloc(&h->d_prm, sizeof(SolveParams)) != cudaSuccess ||
        cudaMalloc(&h->d_flag_ticket, 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemset(h->d_flag_ticket, 0, 2 * sizeof(unsigned)) != cudaSuccess) {
        delete h;
        return P2G_ECUDA;
    }
    p2g_config_default(&h->cfg);
    *out = h;
    return P2G_OK;
}

int p2g_destroy(p2g_handle* h) {
    if (!h) return P2G_EINVAL;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    if (h->cstream) {
        cudaStreamSynchronize(h->cstream);
        cudaStreamDestroy(h->cstream);
        cudaEventDestroy(h->pref_ev);
    }
    dfree(h->d_pref);
    destroy_graph(h);
    dfree(h->d_rp);
    dfree(h->d_ci);
    dfree(h->d_dpos);
    dfree(h->d_vperm);
    dfree(h->d_ninfo);
    dfree(h->d_ncol);
    dfree(h->d_perm);
    dfree(h->d_vals);
    dfree(h->d_phi);
    dfree(h->d_phit);
    dfree(h->d_sg_widths);
    dfree(h->d_sg_W);
    dfree(h->d_sg_b);
    dfree(h->d_sg_norm);
    dfree(h->d_theta);
    for (double** p : {&h->d_u, &h->d_r, &h->d_s, &h->d_s2, &h->d_p, &h->d_Kp, &h->d_b, &h->d_t, &h->d_alpha,
                       &h->d_beta, &h->d_rsold, &h->d_fnorm, &h->d_rel, &h->d_e, &h->d_L, &h->d_Ac,
                       &h->d_hist, &h->d_part_dot, &h->d_part_rr, &h->d_part_ff, &h->d_part_rs,
                       &h->d_part_c, &h->d_stage})
        dfree(*p);
    for (int** p : {&h->d_active, &h->d_iters, &h->d_status, &h->d_setup_status, &h->d_all})
        dfree(*p);
    dfree(h->d_prm);
    dfree(h->d_flag_ticket);
    dfree(h->d_Y);
    dfree(h->d_part_ac);
    for (auto& e : h->ev) cudaEventDestroy(e);
    for (auto& e : h->kev) cudaEventDestroy(e);
    if (h->own_stream) cudaStreamDestroy(h->stream);
    delete h;
    return P2G_OK;
}

const char* p2g_last_error(const p2g_handle* h) { return h ? h->err.c_str() : "null handle"; }

// node-blocked kernels (NodeTab): batched one-instance-per-lane shapes, bs 2 / 3
// (P2G_NO_NODEBLK=1 keeps the row kernels, for A/B measurements)
int upload_node_table(p2g_handle* h) {
    h->node_blk = false;
    h->nmax = 0;
    const int bs = h->pat.bs;
    if ((bs != 2 && bs != 3) || std::getenv("P2G_NO_NODEBLK")) return P2G_OK;
    std::vector<int32_t> info, ncol;
    int nmax = 0;
    if (!build_node_table(h->pat.n, bs, h->pat.rp, h->pat.ci, h->pat.dpos, info, ncol, nmax))
        return P2G_OK;
    TRY(dalloc(h, h->d_ninfo, info.size() / 4));
    TRY(dalloc(h, h->d_ncol, ncol.size()));
    CU(cudaMemcpy(h->d_ninfo, info.data(), sizeof(int32_t) * info.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_ncol, ncol.data(), sizeof(int32_t) * ncol.size(), cudaMemcpyHostToDevice));
    h->nmax = nmax;
    h->node_blk = true;
    return P2G_OK;
}

int p2g_set_batch_hint(p2g_handle* h, int64_t batch) {
    if (!h || batch < 0) return P2G_EINVAL;
    h->batch_hint = batch;
    return P2G_OK;
}

// Colouring policy (D1).  P2G_WAVE_COLOURS decides when set (-1:
// build_coloured_pattern reads it).  Otherwise the 64-class wavefront colouring
// is used when the caller announced a batch (p2g_set_batch_hint) large enough
// that an iteration lasts several ms: there its 11-17 % fewer iterations
// outweigh its 120 extra colour phases per iteration (~3 us each) and its less
// local gathers.  Measured (solves/s, work = nnz x batch):
//   Q4 (2 dofs per node): c3 mesh x 256 / 128 / 64 / 32 instances (4.8e9 ..
//     6.0e8) +7.7 / +6.0 / +12.5 / +13.8 %; c2 (7.5e7) -10..-50 %  -> 2^29
//   hex8 (3 dofs per node; neighbours spread over 14 classes, not 6): c4 mesh
//     x 64 / 32 (4.0e9 / 2.0e9) +5.6 / +5.0 %, x 16 / 8 (1.0e9 / 5.0e8)
//     -2.9 / -4.3 %  -> 1.5 x 2^30
// P2G_WAVE_MIN_WORK overrides the threshold.
static int wave_colours_for(const p2g_handle* h, int64_t n, const uint64_t* row_offsets,
                            int block_size) {
    if (std::getenv("P2G_WAVE_COLOURS")) return -1;
    if (h->batch_hint < 9 || n <= 0 || !row_offsets) return 0;  // lane-per-instance batches only
    double min_work = block_size == 2 ? 536870912.0 : 1610612736.0;
    if (const char* v = std::getenv("P2G_WAVE_MIN_WORK")) min_work = std::atof(v);
    const double work = (double)row_offsets[n] * (double)h->batch_hint;
    return work >= min_work ? 64 : 0;
}

int p2g_set_pattern(p2g_handle* h, int64_t n, const uint64_t* row_offsets,
                    const uint64_t* col_indices, int32_t block_size) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    ColouredPattern pat;
    const std::string msg = build_coloured_pattern(n, row_offsets, col_indices, block_size, pat,
                                                   wave_colours_for(h, n, row_offsets, block_size));
    REQ(msg.empty(), P2G_EINVAL, msg);
    destroy_graph(h);
    if (h->cstream) CU(cudaStreamSynchronize(h->cstream));
    h->pref_host = nullptr;  // a prefetch sized for the old pattern is void
    h->pat = std::move(pat);
    h->have_pattern = true;
    h->have_values = false;
    h->setup_done = false;
    h->B = 0;
    h->Bp = 0;
    h->k = -1;
    dfree(h->d_vals);
    TRY(dalloc(h, h->d_rp, h->pat.rp.size()));
    TRY(dalloc(h, h->d_ci, h->pat.ci.size()));
    TRY(dalloc(h, h->d_dpos, h->pat.dpos.size()));
    TRY(dalloc(h, h->d_vperm, h->pat.vperm.size()));
    TRY(dalloc(h, h->d_perm, h->pat.perm.size()));
    CU(cudaMemcpy(h->d_rp, h->pat.rp.data(), sizeof(int) * h->pat.rp.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_ci, h->pat.ci.data(), sizeof(int) * h->pat.ci.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_dpos, h->pat.dpos.data(), sizeof(int) * h->pat.dpos.size(),
                  cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_vperm, h->pat.vperm.data(), sizeof(int64_t) * h->pat.vperm.size(),
                  cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_perm, h->pat.perm.data(), sizeof(int64_t) * h->pat.perm.size(),
                  cudaMemcpyHostToDevice));
    return upload_node_table(h);
}


int p2g_set_values(p2g_handle* h, int32_t batch, const double* values) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    if (values && values == h->pref_host && batch == h->pref_B) {
        // consume the prefetched copy: the relayout waits for it on the stream
        TRY(start_prefetch(h));
        h->pref_host = nullptr;
        CU(cudaStreamWaitEvent(h->stream, h->pref_ev, 0));
        return set_values_impl(h, batch, nullptr, h->d_pref);
    }
    return set_values_impl(h, batch, values, nullptr);
}

int p2g_prefetch_values(p2g_handle* h, int32_t batch, const double* values) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->have_pattern, P2G_ESTATE, "p2g_prefetch_values: pattern not set");
    REQ(batch >= 1 && values, P2G_EINVAL, "p2g_prefetch_values: null values");
    if (!h->cstream) {
        CU(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&h->pref_ev, cudaEventDisableTiming));
    }
    const size_t bytes = (size_t)batch * h->pat.nnz * sizeof(double);
    if (h->pref_cap < bytes) {
        CU(cudaEventSynchronize(h->pref_ev));  // an earlier prefetch may still be copying
        // the solve stream may still read the old buffer (a consumed prefetch)
        CU(cudaStreamSynchronize(h->stream));
        dfree(h->d_pref);
        CU(cudaMalloc(&h->d_pref, bytes));
        h->pref_cap = bytes;
    }
    // d_pref is free: p2g_set_values synchronises its stream after the relayout
    // of a consumed prefetch, and successive prefetches are ordered on cstream.
    // The copy itself starts once the next solve has uploaded its right-hand
    // sides (solve_impl), so it does not delay them on the host link; a
    // p2g_set_values that comes first starts it.
    if (h->pref_host && h->pref_started) CU(cudaEventSynchronize(h->pref_ev));
    h->pref_host = values;
    h->pref_B = batch;
    h->pref_started = false;
    return P2G_OK;
}

int p2g_set_values_device(p2g_handle* h, int32_t batch, const double* d_values) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    return set_values_impl(h, batch, nullptr, d_values);
}

int p2g_set_basis(p2g_handle* h, int32_t k, const double* phi) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->have_pattern, P2G_ESTATE, "p2g_set_basis: pattern not set");
    REQ(k >= 0 && k <= 64, P2G_EINVAL, "p2g_set_basis: rank must lie in [0, 64]");
    REQ(k == 0 || phi, P2G_EINVAL, "p2g_set_basis: null basis");
    
    h->setup_done = false;
    h->k = k;
    const int64_t n = h->pat.n;
    std::vector<double> perm_phi((size_t)n * std::max(k, 1), 0.0);
    for (int64_t i = 0; i < n; ++i)
        for (int a = 0; a < k; ++a) perm_phi[i * k + a] = phi[h->pat.perm[i] * k + a];
    TRY(upload_phi(h, perm_phi, n, k));
    if (h->Bp > 0) {
        TRY(ensure(h, h->d_e, (size_t)std::max(k, 1) * h->Bp));
        TRY(ensure(h, h->d_L, (size_t)std::max(k * k, 1) * h->Bp));
        TRY(ensure(h, h->d_Ac, (size_t)std::max(k * k, 1) * h->Bp));
        TRY(ensure(h, h->d_part_c, (size_t)h->nb_cap * std::max(k, 1) * h->Bp));
    }
    return P2G_OK;
}

int p2g_setup(p2g_handle* h, const p2g_config* cfg, int32_t* status) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->have_values, P2G_ESTATE, "p2g_setup: values not set");
    REQ(h->k >= 0, P2G_ESTATE, "p2g_setup: basis not set");
    p2g_config c;
    if (cfg) c = *cfg; else p2g_config_default(&c);
    REQ(c.smoother == P2G_SMOOTHER_GS_MULTICOLOR || c.smoother == P2G_SMOOTHER_JACOBI, P2G_EINVAL,
        "p2g_setup: unknown smoother");
    REQ(c.pre_sweeps >= 1 && c.post_sweeps >= 1 && c.pre_sweeps <= 16 && c.post_sweeps <= 16,
        P2G_EINVAL, "p2g_setup: sweeps must lie in [1,16]");
    REQ(c.smoother != P2G_SMOOTHER_JACOBI || (c.omega > 0.0 && c.omega <= 1.0), P2G_EINVAL,
        "jacobi_sweep: omega outside (0,1]");
    REQ(c.residual_form == P2G_RESIDUAL_FULL || c.residual_form == P2G_RESIDUAL_UPPER, P2G_EINVAL,
        "p2g_setup: unknown residual form");
    REQ(c.kp_update == P2G_KP_SPMV || c.kp_update == P2G_KP_RECURRENCE, P2G_EINVAL,
        "p2g_setup: unknown kp_update");
    
    h->cfg = c;
    CU(cudaMemsetAsync(h->d_setup_status, 0, sizeof(int) * h->Bp, h->stream));
    {
        Mat A = mat_of(h);
        dim3 g(std::max(1, std::min(1024, (int)((h->pat.n + 255) / 256))), h->B);
        k_check_diag<<<g, 256, 0, h->stream>>>(A, h->B, h->d_setup_status); ++h->launches_executed;
        CU(cudaGetLastError());
    }
    if (h->k > 0) TRY(dispatch(h, [&](auto R) -> int { return decltype(R)::coarse_setup(h); }));
    CU(cudaStreamSynchronize(h->stream));
    std::vector<int> st(h->Bp);
    CU(cudaMemcpy(st.data(), h->d_setup_status, sizeof(int) * h->Bp, cudaMemcpyDeviceToHost));
    int worst = P2G_OK;
    for (int b = 0; b < h->B; ++b) {
        if (status) status[b] = st[b];
        if (st[b] != P2G_OK) worst = st[b];
    }
    h->setup_done = true;
    h->has_state = false;
    if (worst != P2G_OK) h->err = "p2g_setup: at least one instance failed (see status)";
    return worst;
}

int p2g_initial_guess(p2g_handle* h, const double* b, double* x0) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->setup_done, P2G_ESTATE, "p2g_initial_guess: p2g_setup not called");
    REQ(h->k > 0, P2G_EINVAL, "reduced_solve: basis has rank 0");
    REQ(b && x0, P2G_EINVAL, "p2g_initial_guess: null argument");
    TRY(upload_interleaved(h, b, nullptr, h->pat.n, h->d_perm, h->d_b));
    CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                       h->stream));
    TRY(dispatch(h, [&](auto R) -> int {
        using Rn = decltype(R);
        int nbc = 0;
        TRY(Rn::restrict_(h, RES_VECTOR, h->d_b, nullptr, &nbc));
        TRY(Rn::coarse(h, nbc));
        TRY(Rn::prolong(h, h->d_u, true));
        return P2G_OK;
    }));
    TRY(download_interleaved(h, h->d_u, x0, nullptr));
    return P2G_OK;
}

// ---- compute_pod's contractions on the device -------------------

int p2g_gram(int32_t device, int64_t N, int64_t d, const double* U, int32_t U_on_device, double* G) {
    if (N < 1 || d < 1 || !U || !G) return P2G_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return P2G_ECUDA;
    DevScratch S;
    if (cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking) != cudaSuccess) return P2G_ECUDA;
    const double* dU = U;
    if (!U_on_device) {
        double* t = S.alloc<double>((size_t)N * d);
        if (!t || cudaMemcpyAsync(t, U, sizeof(double) * N * d, cudaMemcpyHostToDevice, S.st))
            return P2G_ECUDA;
        dU = t;
    }
    const int NM = (int)((N + kGramMT - 1) / kGramMT);
    std::vector<int> tiles;
    for (int I = 0; I < NM; ++I)
        for (int J = I; J < NM; ++J) tiles.push_back(I), tiles.push_back(J);
    const int ntiles = (int)tiles.size() / 2;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t chunks = (d + kGramCW - 1) / kGramCW;
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(chunks, (int64_t)4 * sms / ntiles));
    int* dT = S.alloc<int>(tiles.size());
    double* part = S.alloc<double>((size_t)gx * ntiles * kGramMT * kGramMT);
    double* dG = S.alloc<double>((size_t)N * N);
    if (!dT || !part || !dG) return P2G_ECUDA;
    if (cudaMemcpyAsync(dT, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice, S.st))
        return P2G_ECUDA;
    k_gram<<<dim3(gx, ntiles), kBlock, 0, S.st>>>((int)N, d, dU, dT, part);
    k_gram_reduce<<<dim3(16, ntiles), 256, 0, S.st>>>((int)N, gx, ntiles, dT, part, dG);
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpyAsync(G, dG, sizeof(double) * N * N, cudaMemcpyDeviceToHost, S.st) ||
        cudaStreamSynchronize(S.st))
        return P2G_ECUDA;
    return P2G_OK;
}

int p2g_combine(int32_t device, int64_t N, int64_t d, const double* U, int32_t U_on_device,
                int64_t r, const double* W, double* Phi) {
    if (N < 1 || d < 1 || r < 1 || r > 64 || !U || !W || !Phi) return P2G_EINVAL;
    if (cudaSetDevice(device) != cudaSuccess) return P2G_ECUDA;
    DevScratch S;
    if (cudaStreamCreateWithFlags(&S.st, cudaStreamNonBlocking) != cudaSuccess) return P2G_ECUDA;
    const double* dU = U;
    if (!U_on_device) {
        double* t = S.alloc<double>((size_t)N * d);
        if (!t || cudaMemcpyAsync(t, U, sizeof(double) * N * d, cudaMemcpyHostToDevice, S.st))
            return P2G_ECUDA;
        dU = t;
    }
    double* dW = S.alloc<double>((size_t)N * r);
    double* dP = U_on_device ? Phi : S.alloc<double>((size_t)d * r);
    if (!dW || !dP || cudaMemcpyAsync(dW, W, sizeof(double) * N * r, cudaMemcpyHostToDevice, S.st))
        return P2G_ECUDA;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const int64_t need = (d + 8 * kWarps - 1) / (8 * kWarps);
    const int gx = (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)8 * sms));
    k_combine<<<gx, kBlock, 0, S.st>>>((int)N, d, dU, (int)r, dW, dP);
    if (cudaGetLastError() != cudaSuccess) return P2G_ECUDA;
    if (!U_on_device &&
        cudaMemcpyAsync(Phi, dP, sizeof(double) * d * r, cudaMemcpyDeviceToHost, S.st))
        return P2G_ECUDA;
    return cudaStreamSynchronize(S.st) == cudaSuccess ? P2G_OK : P2G_ECUDA;
}

uint64_t p2g_fnv1a64(const void* bytes, int64_t count) {
    const unsigned char* c = static_cast<const unsigned char*>(bytes);
    uint64_t hsh = 1469598103934665603ull;
    for (int64_t i = 0; i < count; ++i) {
        hsh ^= c[i];
        hsh *= 1099511628211ull;
    }
    return hsh;
}

int p2g_set_surrogate(p2g_handle* h, int32_t nlayers, const int32_t* widths, int32_t activation,
                      const double* weights, const double* biases, const double* in_mean,
                      const double* in_std, const double* lat_mean, const double* lat_std) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(nlayers >= 1 && widths, P2G_EINVAL, "Mlp: at least input and output layers required");
    REQ(weights && biases && in_mean && in_std && lat_mean && lat_std, P2G_EINVAL,
        "p2g_set_surrogate: null argument");
    REQ(activation == P2G_ACT_TANH || activation == P2G_ACT_RELU, P2G_EINVAL,
        "p2g_set_surrogate: unknown activation");
    size_t nw = 0, nb = 0;
    int wmax = 0;
    for (int l = 0; l <= nlayers; ++l) {
        REQ(widths[l] >= 1 && widths[l] <= 4096, P2G_EINVAL, "p2g_set_surrogate: widths in [1, 4096]");
        wmax = std::max(wmax, (int)widths[l]);
        if (l < nlayers) {
            nw += (size_t)widths[l] * widths[l + 1];
            nb += widths[l + 1];
        }
    }
    const int p = widths[0], k = widths[nlayers];
    std::vector<double> norm;
    norm.insert(norm.end(), in_mean, in_mean + p);
    norm.insert(norm.end(), in_std, in_std + p);
    norm.insert(norm.end(), lat_mean, lat_mean + k);
    norm.insert(norm.end(), lat_std, lat_std + k);
    TRY(ensure(h, h->d_sg_widths, (size_t)nlayers + 1));
    TRY(ensure(h, h->d_sg_W, nw));
    TRY(ensure(h, h->d_sg_b, nb));
    TRY(ensure(h, h->d_sg_norm, norm.size()));
    CU(cudaMemcpy(h->d_sg_widths, widths, sizeof(int) * (nlayers + 1), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_sg_W, weights, sizeof(double) * nw, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_sg_b, biases, sizeof(double) * nb, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_sg_norm, norm.data(), sizeof(double) * norm.size(), cudaMemcpyHostToDevice));
    h->sg_layers = nlayers;
    h->sg_act = activation;
    h->sg_wmax = wmax;
    h->sg_widths.assign(widths, widths + nlayers + 1);
    h->theta_set = false;
    return P2G_OK;
}

int p2g_set_theta(p2g_handle* h, const double* theta) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->sg_layers > 0, P2G_ESTATE, "p2g_set_theta: p2g_set_surrogate not called");
    REQ(h->B > 0, P2G_ESTATE, "p2g_set_theta: values not set (batch size unknown)");
    REQ(theta, P2G_EINVAL, "p2g_set_theta: null theta");
    const size_t cnt = (size_t)h->B * h->sg_widths[0];
    TRY(ensure(h, h->d_theta, cnt));
    CU(cudaMemcpy(h->d_theta, theta, sizeof(double) * cnt, cudaMemcpyHostToDevice));
    h->theta_set = true;
    return P2G_OK;
}

int p2g_surrogate_predict(p2g_handle* h, const double* theta, double* x) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(x, P2G_EINVAL, "p2g_surrogate_predict: null output");
    TRY(p2g_set_theta(h, theta));
    REQ(h->k > 0 && h->sg_widths.back() == h->k, P2G_EINVAL,
        "predict: surrogate output width differs from the basis rank");
    REQ(h->d_e, P2G_ESTATE, "p2g_surrogate_predict: basis / values not set");
    CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                       h->stream));
    TRY(surrogate_x0(h, h->d_u));
    TRY(download_interleaved(h, h->d_u, x, nullptr));
    return P2G_OK;
}

int p2g_solve(p2g_handle* h, const double* b, const double* x0, int32_t x0_mode, double tol,
              int64_t max_iter, double* x, int64_t* iters, int32_t* converged, int32_t* status,
              double* hist, int64_t hist_cap) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    return solve_impl(h, b, nullptr, x0, nullptr, x0_mode, tol, max_iter, x, nullptr, iters,
                      converged, status, hist, hist_cap);
}

int p2g_pod2g_solve(p2g_handle* h, const double* b, const double* x0, int32_t x0_mode,
                    double tol, int64_t max_cycles, double* x, int64_t* cycles,
                    int32_t* converged, int32_t* status, double* hist, int64_t hist_cap) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    return solve_impl(h, b, nullptr, x0, nullptr, x0_mode, tol, max_cycles, x, nullptr, cycles,
                      converged, status, hist, hist_cap, true);
}

int p2g_solve_device(p2g_handle* h, const double* d_b, const double* d_x0, int32_t x0_mode,
                     double tol, int64_t max_iter, double* d_x, int64_t* iters,
                     int32_t* converged, int32_t* status, double* hist, int64_t hist_cap) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    return solve_impl(h, nullptr, d_b, nullptr, d_x0, x0_mode, tol, max_iter, nullptr, d_x, iters,
                      converged, status, hist, hist_cap);
}

int p2g_last_solve_ms(const p2g_handle* h, double* ms2) {
    if (!h || !ms2) return P2G_EINVAL;
    ms2[0] = h->last_ms[0];
    ms2[1] = h->last_ms[1];
    return P2G_OK;
}

int p2g_spmv(p2g_handle* h, const double* x, double* y) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->have_values, P2G_ESTATE, "p2g_spmv: values not set");
    REQ(x && y, P2G_EINVAL, "p2g_spmv: null argument");
    TRY(upload_interleaved(h, x, nullptr, h->pat.n, h->d_perm, h->d_p));
    CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                       h->stream));
    TRY(dispatch(h, [&](auto R) -> int { return decltype(R)::spmv(h, h->d_p, h->d_Kp, false, nullptr); }));
    TRY(download_interleaved(h, h->d_Kp, y, nullptr));
    return P2G_OK;
}

int p2g_precond_apply(p2g_handle* h, const double* r, double* s) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->setup_done, P2G_ESTATE, "p2g_precond_apply: p2g_setup not called");
    REQ(r && s, P2G_EINVAL, "p2g_precond_apply: null argument");
    TRY(upload_interleaved(h, r, nullptr, h->pat.n, h->d_perm, h->d_r));
    CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                       h->stream));
    TRY(dispatch(h, [&](auto R) -> int { return decltype(R)::precond(h, false, h->d_r, nullptr, nullptr); }));
    TRY(download_interleaved(h, h->s_final, s, nullptr));
    return P2G_OK;
}

int p2g_smooth(p2g_handle* h, int32_t direction, const double* f, double* u) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->have_values, P2G_ESTATE, "p2g_smooth: values not set");
    REQ(f && u, P2G_EINVAL, "p2g_smooth: null argument");
    REQ(direction == 0 || direction == 1, P2G_EINVAL, "p2g_smooth: direction must be 0 or 1");
    TRY(upload_interleaved(h, f, nullptr, h->pat.n, h->d_perm, h->d_r));
    TRY(upload_interleaved(h, u, nullptr, h->pat.n, h->d_perm, h->d_s));
    CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                       h->stream));
    double* out = h->d_s;
    TRY(dispatch(h, [&](auto R) -> int {
        using Rn = decltype(R);
        const int C = h->pat.ncolors;
        if (h->cfg.smoother == P2G_SMOOTHER_JACOBI) {
            int dummy = 0;
            TRY(Rn::jacobi(h, h->d_r, h->d_s, h->d_s2, false, &dummy, KC_FWD));
            out = h->d_s2;
        } else if (direction == 0) {
            for (int c = 0; c < C; ++c) TRY(Rn::gs_forward(h, h->d_r, h->d_s, c, false));
        } else {
            int row = 0;
            for (int c = C - 1; c >= 0; --c)
                TRY(Rn::gs_backward(h, h->d_r, h->d_s, h->d_s, c, false, &row, c == C - 1));
        }
        return P2G_OK;
    }));
    TRY(download_interleaved(h, out, u, nullptr));
    return P2G_OK;
}

int p2g_coarse_operator(p2g_handle* h, double* Ac) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->setup_done && h->k > 0, P2G_ESTATE, "p2g_coarse_operator: no coarse operator");
    REQ(Ac, P2G_EINVAL, "p2g_coarse_operator: null argument");
    CU(cudaMemcpy(Ac, h->d_Ac, sizeof(double) * h->k * h->k * h->B, cudaMemcpyDeviceToHost));
    return P2G_OK;
}

int p2g_get_permutation(p2g_handle* h, int64_t* perm, int32_t* ncolors, int64_t* color_offsets,
                        int32_t cap) {
    if (!h) return P2G_EINVAL;
    REQ(h->have_pattern, P2G_ESTATE, "p2g_get_permutation: pattern not set");
    if (perm) std::memcpy(perm, h->pat.perm.data(), sizeof(int64_t) * h->pat.n);
    if (ncolors) *ncolors = h->pat.ncolors;
    if (color_offsets)
        for (int c = 0; c <= h->pat.ncolors && c < cap; ++c) color_offsets[c] = h->pat.color_rows[c];
    return P2G_OK;
}

int p2g_analyze_pattern(int64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                        int32_t block_size, int64_t* perm, int32_t* ncolors,
                        int64_t* color_offsets, int32_t cap, char* errbuf, int32_t errcap) {
    ColouredPattern pat;
    const std::string msg = build_coloured_pattern(n, row_offsets, col_indices, block_size, pat);
    if (!msg.empty()) {
        if (errbuf && errcap > 0) {
            std::strncpy(errbuf, msg.c_str(), errcap - 1);
            errbuf[errcap - 1] = 0;
        }
        return P2G_EINVAL;
    }
    if (perm) std::memcpy(perm, pat.perm.data(), sizeof(int64_t) * n);
    if (ncolors) *ncolors = pat.ncolors;
    if (color_offsets)
        for (int c = 0; c <= pat.ncolors && c < cap; ++c) color_offsets[c] = pat.color_rows[c];
    return P2G_OK;
}

int p2g_analyze_node_blocking(int64_t n, const uint64_t* row_offsets, const uint64_t* col_indices,
                              int32_t block_size, int32_t* blocked, int32_t* nmax) {
    ColouredPattern pat;
    if (!build_coloured_pattern(n, row_offsets, col_indices, block_size, pat).empty())
        return P2G_EINVAL;
    std::vector<int32_t> info, ncol;
    int nm = 0;
    const bool ok = build_node_table(pat.n, pat.bs, pat.rp, pat.ci, pat.dpos, info, ncol, nm);
    if (blocked) *blocked = ok ? 1 : 0;
    if (nmax) *nmax = ok ? nm : 0;
    return P2G_OK;
}

// algorithmic HBM bytes per iteration of each kernel class (DESIGN.md,
// SURVEY.md 8(d)) for the handle's current pattern / batch / basis / config
static void class_bytes(const p2g_handle* h, double* by) {
    for (int q = 0; q < P2G_NUM_KCLASS; ++q) by[q] = 0.0;
    const double n = (double)h->pat.n, z = (double)h->pat.nnz, Bp = (double)h->B;
    const double k = (double)std::max(h->k, 0);
    const double Mv = 8.0 * z * Bp;                // values, one pass
    const double C = h->pat.ncolors;
    // lower/upper halves of the values (strict), diagonal
    const double zl = 0.5 * (z - n);
    // index bytes, shared by the batch: CSR column indices + row pointers, or
    // -- node-blocked patterns, whose kernels read no column index -- the
    // node table (16 B per node) and one 4 B neighbour id per bs x bs block
    const double bs = std::max(h->pat.bs, 1), nodes = n / bs;
    const double idx = h->node_blk ? 4.0 * z / (bs * bs) + 16.0 * nodes : 4.0 * z + 4.0 * (n + 1);
    const double idx_half = h->node_blk ? 4.0 * (zl + n) / (bs * bs) + 16.0 * nodes
                                        : 4.0 * zl + 4.0 * n;
    const bool gs = h->cfg.smoother == P2G_SMOOTHER_GS_MULTICOLOR;
    by[KC_SPMV] = kp_recurrence(h) ? 8.0 * zl * Bp + idx_half + 64.0 * n * Bp
                                   : Mv + idx + 16.0 * n * Bp;  // L vals | vals, x once, y
    by[KC_UPDATE] = 48.0 * n * Bp + (gs ? 0.0 : 24.0 * n * Bp);  // u,p,r,Kp r/w (+ s,d for Jacobi)
    by[KC_FWD] = gs ? (8.0 * (zl + n) * Bp + idx_half + 24.0 * n * Bp * (C - 1) / C) : 0.0;
    // residual: upper form t = -U s (U values, s read, t written); full form
    // t = r - K s (all values, r and s read, t written)
    by[KC_RESID] = gs && h->cfg.residual_form == P2G_RESIDUAL_UPPER && h->cfg.pre_sweeps == 1
                       ? 8.0 * zl * Bp + idx_half + 16.0 * n * Bp
                       : Mv + idx + 24.0 * n * Bp;
    by[KC_RESTRICT] = 8.0 * n * Bp + 8.0 * n * k;  // t read, Phi read once
    by[KC_COARSE] = 0.0;
    by[KC_PROLONG] = 16.0 * n * Bp + 8.0 * n * k;
    by[KC_BWD] = Mv + idx + 24.0 * n * Bp;
    by[KC_REDUCE] = 0.0;
    by[KC_PUPDATE] = kp_recurrence(h) ? 0.0 : 24.0 * n * Bp;
    if (h->k == 0) by[KC_RESID] = by[KC_RESTRICT] = by[KC_PROLONG] = 0.0;
}

int p2g_profile_iteration(p2g_handle* h, int32_t reps, double* ms, double* bytes,
                          const char** names) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    REQ(h->setup_done, P2G_ESTATE, "p2g_profile_iteration: p2g_setup not called");
    REQ(reps >= 1, P2G_EINVAL, "p2g_profile_iteration: reps >= 1");
    // a zero Krylov state has p'Kp = 0: every instance would stop as a breakdown
    REQ(h->has_state, P2G_ESTATE, "p2g_profile_iteration: run p2g_solve first (Krylov state)");
    std::vector<double> acc(P2G_NUM_KCLASS, 0.0);
    // every instance active for the whole replay: no convergence or max_iter
    // exit inside the profiled iterations (state is scratch)
    {
        SolveParams prm{0.0, (long long)1 << 62, 0};
        CU(cudaMemcpyAsync(h->d_prm, &prm, sizeof(prm), cudaMemcpyHostToDevice, h->stream));
    }
    // The loop body with a CUDA event after every kernel class, captured as a
    // plain graph and replayed: kernels follow each other as in the solve's
    // graph (no host launch gap between them), and the event-record nodes time
    // each class on the device.  P2G_PROFILE_EAGER=1: eager launches instead.
    const char* pe = std::getenv("P2G_PROFILE_EAGER");
    const bool eager = pe && pe[0] == '1';
    auto body = [&]() -> int {
        h->profiling = true;
        h->kev_n = 0;
        CU(prof_record(h, h->kev[0], h->stream));
        const int st = dispatch(h, [&](auto R) -> int { return decltype(R)::iteration(h, false); });
        h->profiling = false;
        return st;
    };
    cudaGraphExec_t ge = nullptr;
    if (!eager) {
        CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
        h->capturing = true;
        const int st = body();
        h->capturing = false;
        cudaGraph_t g = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
        TRY(st);
        CU(ce);
        const cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
        cudaGraphDestroy(g);
        CU(ie);
    }
    struct ExecGuard {
        cudaGraphExec_t e;
        ~ExecGuard() { if (e) cudaGraphExecDestroy(e); }
    } guard{ge};
    for (int rep = 0; rep < reps; ++rep) {
        CU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                           h->stream));
        if (kp_recurrence(h)) {
            // the body starts at alpha: refresh Kp and the pKp partials first
            TRY(dispatch(h, [&](auto R) -> int { return decltype(R)::spmv(h, h->d_p, h->d_Kp, true, nullptr); }));
        }
        if (ge) {
            CU(cudaGraphLaunch(ge, h->stream));
        } else {
            TRY(body());
        }
        CU(cudaStreamSynchronize(h->stream));
        for (int q = 0; q < h->kev_n; ++q) {
            float t = 0;
            cudaEventElapsedTime(&t, h->kev[q], h->kev[q + 1]);
            acc[h->kev_class[q]] += t;
        }
    }
    double by[P2G_NUM_KCLASS] = {0};
    class_bytes(h, by);
    for (int q = 0; q < P2G_NUM_KCLASS; ++q) {
        if (ms) ms[q] = acc[q] / reps;
        if (bytes) bytes[q] = by[q];
        if (names) names[q] = kKclassNames[q];
    }
    return P2G_OK;
}

void* p2g_get_stream(const p2g_handle* h) { return h ? (void*)h->stream : nullptr; }

int p2g_debug_guard_check(void) {
    if (!guard_mode()) return -1;
    if (cudaDeviceSynchronize() != cudaSuccess) return -2;
    std::lock_guard<std::mutex> lk(guards().mu);
    int bad = 0;
    std::vector<unsigned char> band(kGuardBytes);
    for (const auto& [p, bytes] : guards().bytes) {
        const unsigned char* u = static_cast<const unsigned char*>(p);
        for (const unsigned char* b : {u - kGuardBytes, u + bytes}) {
            if (cudaMemcpy(band.data(), b, kGuardBytes, cudaMemcpyDeviceToHost) != cudaSuccess)
                return -2;
            for (unsigned char c : band)
                if (c != kGuardByte) {
                    ++bad;
                    break;
                }
        }
    }
    return bad;
}

int p2g_launch_counts(const p2g_handle* h, int64_t* per_iteration, int64_t* last_solve_total) {
    if (!h) return P2G_EINVAL;
    if (per_iteration) *per_iteration = h->launches_per_iter;
    if (last_solve_total) *last_solve_total = h->launches_executed;
    return P2G_OK;
}

}  // extern "C"

// ============================================================================
// Row-partitioned single-system path
//
// A p2g_part holds the partitions this process hosts: every rank of the job
// for the in-process (emulated) transport, or exactly one rank for NCCL.
// Each partition is an ordinary handle whose pattern is its owned rows (in
// the global colour-major order) plus ghost rows; the same kernels run on the
// owned rows and read ghosts through local column indices.  Per iteration the
// exchange steps are: the swept vector after every forward and backward
// colour phase (only that colour's boundary rows move), and allreduces of
// the scalar partials (pKp; ||r||^2; Phi^T t; r.s).  The prolongation is
// applied to ghost rows locally (ghost rows of Phi are stored; e is
// replicated), so s' needs no exchange.
// ============================================================================
namespace {

struct NcclApi {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    bool load(std::string& err) {
        if (lib) return true;
        lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            err = "dlopen(libnccl.so.2) failed";
            return false;
        }
#define P2G_SYM(f, name) f = reinterpret_cast<decltype(f)>(dlsym(lib, name)); if (!f) { err = std::string("missing ") + name; return false; }
        P2G_SYM(GetUniqueId, "ncclGetUniqueId")
        P2G_SYM(CommInitRank, "ncclCommInitRank")
        P2G_SYM(CommDestroy, "ncclCommDestroy")
        P2G_SYM(AllReduce, "ncclAllReduce")
        P2G_SYM(Send, "ncclSend")
        P2G_SYM(Recv, "ncclRecv")
        P2G_SYM(GroupStart, "ncclGroupStart")
        P2G_SYM(GroupEnd, "ncclGroupEnd")
        P2G_SYM(GetErrorString, "ncclGetErrorString")
#undef P2G_SYM
        return true;
    }
};
NcclApi g_nccl;

struct PartLocal {
    int rank = 0;
    p2g_handle* h = nullptr;
    PartitionPlan plan;
    // device send lists: all colours, then one block per colour
    int* d_rows = nullptr;
    std::vector<int64_t> all_off;                 // per send_all message
    std::vector<std::vector<int64_t>> col_off;    // [colour][message]
    int64_t rows_all = 0;
    std::vector<int64_t> col_base;                // first entry of colour c in d_rows
    double* d_sendbuf = nullptr;
    size_t sendbuf_elems = 0;
};

}  // namespace

struct p2g_part {
    int device = 0;
    int world = 1;
    bool use_nccl = false;
    ncclComm_t comm = nullptr;
    cudaStream_t stream = nullptr;
    std::vector<PartLocal> parts;
    std::string err;
    int B = 0;
    bool setup_done = false;
    double last_ms = 0;
    int64_t iters_host = 0;
    // the captured loop (build_part_graph): mode 1 = conditional WHILE node
    // (device-side stopping, no host round trip), mode 2 = a chunk of
    // kChunk iterations replayed until the host sees no active instance
    cudaGraphExec_t loop_exec = nullptr;
    int graph_mode = 0;
    std::vector<uint64_t> graph_key;
    cudaGraphConditionalHandle cond = 0;
    bool capturing = false;
    int64_t launches_per_iter = 0;
};

namespace {

#define PCU(call)                                                                       \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            P->err = std::string(#call) + ": " + cudaGetErrorString(e_);                \
            return static_cast<int>(P2G_ECUDA);                                         \
        }                                                                               \
    } while (0)
#define PNC(call)                                                                       \
    do {                                                                                \
        ncclResult_t r_ = (call);                                                       \
        if (r_ != ncclSuccess) {                                                        \
            P->err = std::string(#call) + ": " + g_nccl.GetErrorString(r_);             \
            return static_cast<int>(P2G_ENCCL);                                         \
        }                                                                               \
    } while (0)
#define PTRY(expr)                                                                      \
    do {                                                                                \
        int st_ = (expr);                                                               \
        if (st_ != P2G_OK) {                                                            \
            if (P->err.empty()) P->err = "partition step failed";                       \
            return st_;                                                                 \
        }                                                                               \
    } while (0)

PartLocal* local_of(p2g_part* P, int rank) {
    for (auto& L : P->parts)
        if (L.rank == rank) return &L;
    return nullptr;
}

// send the boundary rows of `vec` (member of the handle) of one colour
// (colour < 0: all ghosts) into the peers' ghost rows
int part_exchange(p2g_part* P, double* p2g_handle::*vec, int colour) {
    for (auto& L : P->parts) {
        p2g_handle* h = L.h;
        const int64_t base = colour < 0 ? 0 : L.col_base[colour];
        const int64_t cnt = colour < 0 ? L.rows_all : L.col_base[colour + 1] - L.col_base[colour];
        if (cnt == 0) continue;
        const int64_t total = cnt * h->Bp;
        const int grid = (int)std::min<int64_t>((total + 255) / 256, 4096);
        k_pack_rows<<<grid, 256, 0, P->stream>>>(h->*vec, h->Bp, L.d_rows + base, cnt, L.d_sendbuf);
        count_launch(h, KC_COMM);
        PCU(cudaGetLastError());
    }
    if (!P->use_nccl) {
        for (auto& L : P->parts) {  // receive side
            const auto& recvs = colour < 0 ? L.plan.recv_all : L.plan.recv_c[colour];
            for (const auto& rm : recvs) {
                PartLocal* S = local_of(P, rm.peer);
                if (!S) {
                    P->err = "partition: peer not hosted in this process";
                    return P2G_ESTATE;
                }
                const auto& sends = colour < 0 ? S->plan.send_all : S->plan.send_c[colour];
                const auto& offs = colour < 0 ? S->all_off : S->col_off[colour];
                int64_t off = -1, cnt = 0;
                for (size_t q = 0; q < sends.size(); ++q)
                    if (sends[q].peer == L.rank) {
                        off = offs[q];
                        cnt = sends[q].count;
                    }
                if (off < 0 || cnt != rm.count) {
                    P->err = "partition: send/receive lists disagree (pattern not symmetric?)";
                    return P2G_EINVAL;
                }
                const int Bp = L.h->Bp;
                PCU(cudaMemcpyAsync((L.h->*vec) + (size_t)rm.ghost_off * Bp,
                                    S->d_sendbuf + (size_t)off * Bp, sizeof(double) * cnt * Bp,
                                    cudaMemcpyDeviceToDevice, P->stream));
            }
        }
        prof_mark(P->parts[0].h, KC_COMM);
        return P2G_OK;
    }
    PartLocal& L = P->parts[0];
    const int Bp = L.h->Bp;
    const auto& sends = colour < 0 ? L.plan.send_all : L.plan.send_c[colour];
    const auto& offs = colour < 0 ? L.all_off : L.col_off[colour];
    const auto& recvs = colour < 0 ? L.plan.recv_all : L.plan.recv_c[colour];
    PNC(g_nccl.GroupStart());
    for (size_t q = 0; q < sends.size(); ++q)
        PNC(g_nccl.Send(L.d_sendbuf + (size_t)offs[q] * Bp, sends[q].count * Bp, ncclFloat64,
                        sends[q].peer, P->comm, P->stream));
    for (const auto& rm : recvs)
        PNC(g_nccl.Recv((L.h->*vec) + (size_t)rm.ghost_off * Bp, rm.count * Bp, ncclFloat64, rm.peer,
                        P->comm, P->stream));
    PNC(g_nccl.GroupEnd());
    prof_mark(L.h, KC_COMM);
    return P2G_OK;
}

// reduce each partition's partial rows to row 0, then sum row 0 across ranks
int part_allreduce(p2g_part* P, double* p2g_handle::*buf, int nrows, int ncols) {
    for (auto& L : P->parts) {
        if (nrows > 1) {
            k_reduce_rows<<<(ncols + 255) / 256, 256, 0, P->stream>>>(L.h->*buf, nrows, ncols);
            count_launch(L.h, KC_COMM);
        }
    }
    if (P->world == 1) return P2G_OK;
    if (!P->use_nccl) {
        PartPtrs pp{};
        for (size_t q = 0; q < P->parts.size(); ++q) pp.p[q] = P->parts[q].h->*buf;
        k_sum_parts<<<(ncols + 255) / 256, 256, 0, P->stream>>>(pp, (int)P->parts.size(), ncols);
        count_launch(P->parts[0].h, KC_COMM);
        PCU(cudaGetLastError());
        return P2G_OK;
    }
    double* b = P->parts[0].h->*buf;
    PNC(g_nccl.AllReduce(b, b, ncols, ncclFloat64, ncclSum, P->comm, P->stream));
    prof_mark(P->parts[0].h, KC_COMM);
    return P2G_OK;
}

int part_allmax_int(p2g_part* P, int* p2g_handle::*buf, int n) {
    if (P->world == 1) return P2G_OK;
    if (!P->use_nccl) {
        PartPtrs pp{};
        for (size_t q = 0; q < P->parts.size(); ++q) pp.ip[q] = P->parts[q].h->*buf;
        k_max_parts_int<<<(n + 255) / 256, 256, 0, P->stream>>>(pp, (int)P->parts.size(), n);
        PCU(cudaGetLastError());
        return P2G_OK;
    }
    int* b = P->parts[0].h->*buf;
    PNC(g_nccl.AllReduce(b, b, n, ncclInt32, ncclMax, P->comm, P->stream));
    return P2G_OK;
}

template <class F>
int for_parts(p2g_part* P, F&& f) {
    for (auto& L : P->parts) {
        const int st = f(L.h);
        if (st != P2G_OK) {
            if (P->err.empty()) P->err = L.h->err;
            return st;
        }
    }
    return P2G_OK;
}

template <class Sh>
struct PartRun {
    using R = Run<Sh>;

    // s = B r on every partition (update: the PCG update of u, r first);
    // returns the partial-row counts of ||r||^2 (update only) and r.s
    static int precond(p2g_part* P, bool update, int* nb_rr, int* rs_rows) {
        const int C = P->parts[0].h->pat.ncolors;
        const bool rec = kp_recurrence(P->parts[0].h);
        const bool upper = P->parts[0].h->cfg.residual_form == P2G_RESIDUAL_UPPER;
        PTRY(for_parts(P, [&](p2g_handle* h) { return R::update_pre(h, update, h->d_r, nb_rr); }));
        PTRY(part_exchange(P, &p2g_handle::d_s, 0));
        for (int c = 1; c < C; ++c) {
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::gs_forward(h, h->d_r, h->d_s, c, true); }));
            PTRY(part_exchange(P, &p2g_handle::d_s, c));
        }
        int nbc = 0;
        if (P->parts[0].h->k > 0) {
            PTRY(for_parts(P, [&](p2g_handle* h) {
                return R::restrict_(h, upper ? RES_UPPER : RES_FULL, h->d_r, h->d_s, &nbc);
            }));
            const int kk = P->parts[0].h->k, Bp = P->parts[0].h->Bp;
            PTRY(part_allreduce(P, &p2g_handle::d_part_c, nbc, kk * Bp));
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::coarse(h, 1); }));
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::prolong(h, h->d_s, false); }));
        }
        double* p2g_handle::*out = rec ? &p2g_handle::d_s2 : &p2g_handle::d_s;
        for (int c = C - 1; c >= 0; --c) {
            PTRY(for_parts(P, [&](p2g_handle* h) {
                return R::gs_backward(h, h->d_r, h->d_s, h->*out, c, true, rs_rows, c == C - 1);
            }));
            PTRY(part_exchange(P, out, c));
        }
        for (auto& L : P->parts) {
            L.h->s_final = L.h->*out;
            L.h->s_prol = L.h->d_s;
        }
        return P2G_OK;
    }

    static int iteration(p2g_part* P) {
        p2g_handle* h0 = P->parts[0].h;
        const bool rec = kp_recurrence(h0);
        const int Bp = h0->Bp;
        int nb_dot = R::kp_rows(h0), nb_rr = 0, rs_rows = 0;
        if (!rec) {
            PTRY(part_exchange(P, &p2g_handle::d_p, -1));
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::spmv(h, h->d_p, h->d_Kp, true, &nb_dot); }));
        }
        PTRY(part_allreduce(P, &p2g_handle::d_part_dot, nb_dot, Bp));
        PTRY(for_parts(P, [&](p2g_handle* h) {
            k_alpha<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(h->Bp, 1, h->d_part_dot, h->d_rsold,
                                                           h->d_alpha, h->d_active, h->d_status);
            count_launch(h, KC_REDUCE);
            return P2G_OK;
        }));
        PTRY(precond(P, true, &nb_rr, &rs_rows));
        PTRY(part_allreduce(P, &p2g_handle::d_part_rr, nb_rr, Bp));
        PTRY(part_allreduce(P, &p2g_handle::d_part_rs, rs_rows, Bp));
        PTRY(for_parts(P, [&](p2g_handle* h) {
            // every partition holds the same (all-reduced) per-instance state;
            // partition 0 drives the WHILE condition of the captured loop
            const int set_cond = P->capturing && P->graph_mode == 1 && h == P->parts[0].h;
            k_finalize<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(
                h->Bp, 1, h->d_part_rs, 1, h->d_part_rr, h->d_fnorm, h->d_rsold, h->d_beta,
                h->d_rel, h->d_iters, h->d_active, h->d_status, h->d_hist, h->d_prm,
                h->d_flag_ticket, set_cond ? P->cond : h->cond, set_cond);
            count_launch(h, KC_REDUCE);
            return P2G_OK;
        }));
        if (rec)
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::kp_update(h, h->s_final, h->s_prol, nullptr); }));
        else
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::pupdate(h, h->s_final, false); }));
        return P2G_OK;
    }

    static int setup(p2g_part* P) {
        // A_c per partition (owned rows; ghost rows of Phi for K Phi), summed
        // over ranks, then factored identically everywhere
        p2g_handle* h0 = P->parts[0].h;
        if (h0->k > 0) {
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::coarse_setup(h, false); }));
            PTRY(part_allreduce(P, &p2g_handle::d_Ac, 1, h0->k * h0->k * h0->Bp));
            PTRY(for_parts(P, [&](p2g_handle* h) {
                k_cholesky<<<(h->B + 7) / 8, 256, 0, h->stream>>>(h->B, h->k, h->d_Ac, h->d_L,
                                                                  h->d_setup_status);
                ++h->launches_executed;
                return P2G_OK;
            }));
        }
        return P2G_OK;
    }

    static int prologue(p2g_part* P, int x0_mode) {
        p2g_handle* h0 = P->parts[0].h;
        const int Bp = h0->Bp;
        if (x0_mode == P2G_X0_REDUCED) {
            int nbc = 0;
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::restrict_(h, RES_VECTOR, h->d_b, nullptr, &nbc); }));
            PTRY(part_allreduce(P, &p2g_handle::d_part_c, nbc, h0->k * Bp));
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::coarse(h, 1); }));
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::prolong(h, h->d_u, true); }));
        } else if (x0_mode == P2G_X0_GIVEN) {
            PTRY(part_exchange(P, &p2g_handle::d_u, -1));
        }
        int nb = 0;
        PTRY(for_parts(P, [&](p2g_handle* h) { return R::residual(h, h->d_b, h->d_u, h->d_r, &nb); }));
        PTRY(part_allreduce(P, &p2g_handle::d_part_rr, nb, Bp));
        PTRY(part_allreduce(P, &p2g_handle::d_part_ff, nb, Bp));
        PTRY(for_parts(P, [&](p2g_handle* h) {
            k_init_rel<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(
                h->Bp, h->B, 1, h->d_part_rr, h->d_part_ff, h->d_fnorm, h->d_rel, h->d_iters,
                h->d_active, h->d_status, h->d_setup_status, h->d_hist, h->d_prm);
            count_launch(h, KC_REDUCE);
            return P2G_OK;
        }));
        int rs_rows = 0;
        PTRY(precond(P, false, nullptr, &rs_rows));
        PTRY(part_allreduce(P, &p2g_handle::d_part_rs, rs_rows, Bp));
        PTRY(for_parts(P, [&](p2g_handle* h) {
            k_init_rs<<<(h->Bp + 7) / 8, 256, 0, h->stream>>>(h->Bp, 1, h->d_part_rs, h->d_rsold,
                                                              h->d_active, h->d_status);
            count_launch(h, KC_REDUCE);
            return R::pupdate(h, h->s_final, true);
        }));
        if (kp_recurrence(h0)) {
            PTRY(part_exchange(P, &p2g_handle::d_p, -1));
            PTRY(for_parts(P, [&](p2g_handle* h) { return R::spmv(h, h->d_p, h->d_Kp, true, nullptr); }));
        }
        return P2G_OK;
    }
};

template <class F>
int pdispatch(p2g_part* P, F&& f) {
    switch (P->parts[0].h->shape) {
        case SH_B1A: return f(PartRun<ShB1a>{});
        case SH_B1B: return f(PartRun<ShB1b>{});
        case SH_B8: return f(PartRun<ShB8>{});
        case SH_B32: return f(PartRun<ShB32>{});
        default: return f(PartRun<ShB64>{});
    }
}

constexpr int kPartChunk = 8;  // iterations per replay in graph mode 2 / the eager loop

std::vector<uint64_t> part_graph_key(p2g_part* P) {
    std::vector<uint64_t> key;
    for (auto& L : P->parts) {
        const auto k = graph_key_of(L.h);
        key.insert(key.end(), k.begin(), k.end());
        key.push_back((uint64_t)(uintptr_t)L.d_sendbuf);
        key.push_back((uint64_t)(uintptr_t)L.d_rows);
    }
    return key;
}

void destroy_part_graph(p2g_part* P) {
    if (P->loop_exec) cudaGraphExecDestroy(P->loop_exec);
    P->loop_exec = nullptr;
    P->graph_mode = 0;
}

// Capture one PCG iteration of every hosted partition (kernels, halo copies /
// NCCL send-recv, all-reduces) as the body of a conditional WHILE node whose
// condition partition 0's k_finalize sets (mode 1).  If the body cannot be
// captured or instantiated that way (e.g. a transport whose operations are
// not allowed inside a conditional body), capture kPartChunk iterations as a
// plain graph instead (mode 2).  Returns P2G_OK with graph_mode 0 when neither
// works: the eager loop then runs (P2G_PART_EAGER=1 forces it).
int build_part_graph(p2g_part* P) {
    destroy_part_graph(P);
    const char* ev = std::getenv("P2G_PART_EAGER");
    if (ev && ev[0] == '1') return P2G_OK;
    p2g_handle* h0 = P->parts[0].h;
    for (int mode = 1; mode <= 2; ++mode) {
        cudaGraph_t outer = nullptr, body = nullptr;
        if (cudaGraphCreate(&outer, 0) != cudaSuccess) break;
        if (mode == 1) {
            cudaGraphConditionalHandle cond;
            if (cudaGraphConditionalHandleCreate(&cond, outer, 0, 0) != cudaSuccess) {
                cudaGraphDestroy(outer);
                continue;
            }
            P->cond = cond;
            cudaKernelNodeParams kp = {};
            int Bp = h0->Bp;
            int* act = h0->d_active;
            void* args[] = {&act, &Bp, &cond};
            kp.func = (void*)k_set_cond;
            kp.gridDim = dim3(1);
            kp.blockDim = dim3(256);
            kp.kernelParams = args;
            cudaGraphNode_t setn, wnode;
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = cond;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            if (cudaGraphAddKernelNode(&setn, outer, nullptr, 0, &kp) != cudaSuccess ||
                cudaGraphAddNode(&wnode, outer, &setn, 1, &cp) != cudaSuccess) {
                cudaGraphDestroy(outer);
                continue;
            }
            body = cp.conditional.phGraph_out[0];
        } else {
            body = outer;
        }
        if (cudaStreamBeginCaptureToGraph(P->stream, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed) != cudaSuccess) {
            cudaGraphDestroy(outer);
            cudaGetLastError();
            continue;
        }
        P->capturing = true;
        P->graph_mode = mode;
        int64_t before = 0;
        for (auto& L : P->parts) {
            L.h->capturing = true;
            before += L.h->launch_counter;
        }
        int st = P2G_OK;
        const int reps = mode == 1 ? 1 : kPartChunk;
        for (int q = 0; q < reps && st == P2G_OK; ++q)
            st = pdispatch(P, [&](auto R) -> int { return decltype(R)::iteration(P); });
        int64_t after = 0;
        for (auto& L : P->parts) {
            L.h->capturing = false;
            after += L.h->launch_counter;
        }
        P->capturing = false;
        cudaGraph_t captured = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(P->stream, &captured);
        cudaGetLastError();
        if (st != P2G_OK || ce != cudaSuccess) {
            cudaGraphDestroy(outer);
            P->graph_mode = 0;
            P->err.clear();
            if (st != P2G_OK && st != P2G_ECUDA && st != P2G_ENCCL) return st;
            continue;
        }
        cudaGraphExec_t exec = nullptr;
        const cudaError_t ie = cudaGraphInstantiate(&exec, outer, 0);
        cudaGraphDestroy(outer);
        if (ie != cudaSuccess) {
            cudaGetLastError();
            P->graph_mode = 0;
            continue;
        }
        P->loop_exec = exec;
        P->launches_per_iter = (after - before) / reps;
        P->graph_key = part_graph_key(P);
        return P2G_OK;
    }
    P->graph_mode = 0;
    return P2G_OK;
}

int part_new(int device, int world, p2g_part** out) {
    p2g_part* P = new p2g_part();
    P->device = device;
    P->world = world;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete P;
        return P2G_ECUDA;
    }
    *out = P;
    return P2G_OK;
}

int part_add_local(p2g_part* P, int rank) {
    PartLocal L;
    L.rank = rank;
    const int st = p2g_create(P->device, &L.h);
    if (st != P2G_OK) return st;
    cudaStreamDestroy(L.h->stream);  // every partition of the process shares one stream
    L.h->stream = P->stream;
    L.h->own_stream = false;
    P->parts.push_back(std::move(L));
    return P2G_OK;
}

}  // namespace

extern "C" {

int p2g_nccl_unique_id(void* uid) {
    std::string err;
    if (!uid || !g_nccl.load(err)) return P2G_ENCCL;
    ncclUniqueId id;
    if (g_nccl.GetUniqueId(&id) != ncclSuccess) return P2G_ENCCL;
    std::memcpy(uid, &id, sizeof(id));
    return P2G_OK;
}

int p2g_part_create_local(int device, int world, p2g_part** out) {
    if (!out || world < 1 || world > kMaxParts) return P2G_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return P2G_ECUDA;
    p2g_part* P = nullptr;
    int st = part_new(device, world, &P);
    if (st != P2G_OK) return st;
    for (int r = 0; r < world && st == P2G_OK; ++r) st = part_add_local(P, r);
    if (st != P2G_OK) {
        p2g_part_destroy(P);
        return st;
    }
    *out = P;
    return P2G_OK;
}

int p2g_part_create_nccl(int device, int rank, int world, const void* uid, p2g_part** out) {
    if (!out || !uid || world < 1 || rank < 0 || rank >= world) return P2G_EINVAL;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return P2G_ECUDA;
    std::string err;
    if (!g_nccl.load(err)) return P2G_ENCCL;
    p2g_part* P = nullptr;
    int st = part_new(device, world, &P);
    if (st != P2G_OK) return st;
    P->use_nccl = true;
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    if (g_nccl.CommInitRank(&P->comm, world, id, rank) != ncclSuccess) {
        p2g_part_destroy(P);
        return P2G_ENCCL;
    }
    st = part_add_local(P, rank);
    if (st != P2G_OK) {
        p2g_part_destroy(P);
        return st;
    }
    *out = P;
    return P2G_OK;
}

int p2g_part_destroy(p2g_part* P) {
    if (!P) return P2G_EINVAL;
    cudaSetDevice(P->device);
    cudaStreamSynchronize(P->stream);
    destroy_part_graph(P);
    for (auto& L : P->parts) {
        if (L.d_rows) cudaFree(L.d_rows);
        if (L.d_sendbuf) cudaFree(L.d_sendbuf);
        if (L.h) p2g_destroy(L.h);
    }
    if (P->comm) g_nccl.CommDestroy(P->comm);
    cudaStreamDestroy(P->stream);
    delete P;
    return P2G_OK;
}

const char* p2g_part_last_error(const p2g_part* P) { return P ? P->err.c_str() : "null"; }

int p2g_part_set_pattern(p2g_part* P, int rank, int64_t n_global, const int64_t* row_bounds,
                         const uint64_t* row_offsets, const uint64_t* col_indices,
                         int32_t block_size, const int32_t* node_colors) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    destroy_part_graph(P);
    PartLocal* L = local_of(P, rank);
    if (!L) {
        P->err = "p2g_part_set_pattern: rank not hosted by this handle";
        return P2G_EINVAL;
    }
    PartitionPlan plan;
    const std::string msg = build_partition_plan(rank, P->world, row_bounds, n_global, row_offsets,
                                                 col_indices, block_size, node_colors, plan);
    if (!msg.empty()) {
        P->err = msg;
        return P2G_EINVAL;
    }
    p2g_handle* h = L->h;
    destroy_graph(h);
    // the partition's local pattern: owned rows colour-major, ghosts appended
    ColouredPattern& pat = h->pat;
    pat = ColouredPattern();
    pat.n = plan.n_own;
    pat.nnz = plan.nnz;
    pat.bs = plan.bs;
    pat.ncolors = plan.ncolors;
    pat.color_rows = plan.color_rows;
    pat.perm.resize(plan.n_own);
    for (int64_t i = 0; i < plan.n_own; ++i) pat.perm[i] = plan.own_global[i] - plan.row_begin;
    pat.rp = plan.rp;
    pat.ci = plan.ci;
    pat.dpos = plan.dpos;
    pat.vperm = plan.vperm;
    h->n_ghost = plan.n_ghost;
    h->have_pattern = true;
    h->have_values = false;
    h->setup_done = false;
    h->B = 0;
    h->Bp = 0;
    h->k = -1;
    dfree(h->d_vals);
    auto up = [&](auto*& d, const auto& v) -> int {
        using T = std::remove_reference_t<decltype(*d)>;
        TRY(dalloc(h, d, v.size()));
        CU(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
        return P2G_OK;
    };
    if (up(h->d_rp, pat.rp) || up(h->d_ci, pat.ci) || up(h->d_dpos, pat.dpos) ||
        up(h->d_vperm, pat.vperm) || up(h->d_perm, pat.perm) || upload_node_table(h)) {
        P->err = h->err;
        return P2G_ECUDA;
    }
    // device send lists
    std::vector<int32_t> rows;
    L->all_off.clear();
    for (const auto& m : plan.send_all) {
        L->all_off.push_back((int64_t)rows.size());
        rows.insert(rows.end(), m.rows.begin(), m.rows.end());
    }
    L->rows_all = (int64_t)rows.size();
    L->col_base.assign(plan.ncolors + 1, 0);
    L->col_off.assign(plan.ncolors, {});
    for (int c = 0; c < plan.ncolors; ++c) {
        L->col_base[c] = (int64_t)rows.size();
        int64_t rel = 0;
        for (const auto& m : plan.send_c[c]) {
            L->col_off[c].push_back(rel);
            rows.insert(rows.end(), m.rows.begin(), m.rows.end());
            rel += m.count;
        }
    }
    L->col_base[plan.ncolors] = (int64_t)rows.size();
    if (L->d_rows) cudaFree(L->d_rows);
    L->d_rows = nullptr;
    PCU(cudaMalloc(&L->d_rows, sizeof(int32_t) * std::max<size_t>(rows.size(), 1)));
    PCU(cudaMemcpy(L->d_rows, rows.data(), sizeof(int32_t) * rows.size(), cudaMemcpyHostToDevice));
    L->plan = std::move(plan);
    P->setup_done = false;
    return P2G_OK;
}

int p2g_part_ghosts(p2g_part* P, int rank, int64_t* n_own, int64_t* n_ghost, int64_t* ghost_global) {
    if (!P) return P2G_EINVAL;
    PartLocal* L = local_of(P, rank);
    if (!L) return P2G_EINVAL;
    if (n_own) *n_own = L->plan.n_own;
    if (n_ghost) *n_ghost = L->plan.n_ghost;
    if (ghost_global)
        std::memcpy(ghost_global, L->plan.ghost_global.data(), sizeof(int64_t) * L->plan.n_ghost);
    return P2G_OK;
}

int p2g_part_set_values(p2g_part* P, int rank, int32_t batch, const double* values) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    PartLocal* L = local_of(P, rank);
    if (!L) return P2G_EINVAL;
    const int st = set_values_impl(L->h, batch, values, nullptr);
    if (st != P2G_OK) {
        P->err = L->h->err;
        return st;
    }
    const size_t need = (size_t)std::max<int64_t>(L->rows_all, 1) * L->h->Bp;
    if (L->sendbuf_elems < need) {
        if (L->d_sendbuf) cudaFree(L->d_sendbuf);
        PCU(cudaMalloc(&L->d_sendbuf, sizeof(double) * need));
        L->sendbuf_elems = need;
    }
    P->B = batch;
    P->setup_done = false;
    return P2G_OK;
}

int p2g_part_set_basis(p2g_part* P, int rank, int32_t k, const double* phi_own,
                       const double* phi_ghost) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    PartLocal* L = local_of(P, rank);
    if (!L) return P2G_EINVAL;
    p2g_handle* h = L->h;
    if (k < 1 || k > 64 || !phi_own || (L->plan.n_ghost > 0 && !phi_ghost)) {
        P->err = "p2g_part_set_basis: rank in [1,64] and both row blocks required";
        return P2G_EINVAL;
    }
    const int64_t n = h->pat.n, ng = h->n_ghost;
    std::vector<double> phi((size_t)(n + ng) * k);
    for (int64_t i = 0; i < n; ++i)
        for (int a = 0; a < k; ++a) phi[i * k + a] = phi_own[h->pat.perm[i] * k + a];
    for (int64_t j = 0; j < ng; ++j)
        for (int a = 0; a < k; ++a) phi[(n + j) * k + a] = phi_ghost[j * k + a];
    h->k = k;
    if (upload_phi(h, phi, n + ng, k) != P2G_OK) return P2G_ECUDA;
    if (h->Bp > 0) {
        if (ensure(h, h->d_e, (size_t)k * h->Bp) || ensure(h, h->d_L, (size_t)k * k * h->Bp) ||
            ensure(h, h->d_Ac, (size_t)k * k * h->Bp) ||
            ensure(h, h->d_part_c, (size_t)h->nb_cap * k * h->Bp))
            return P2G_ECUDA;
    }
    P->setup_done = false;
    return P2G_OK;
}

int p2g_part_setup(p2g_part* P, const p2g_config* cfg, int32_t* status) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    p2g_config c;
    if (cfg) c = *cfg; else p2g_config_default(&c);
    destroy_part_graph(P);
    if (c.smoother != P2G_SMOOTHER_GS_MULTICOLOR || c.pre_sweeps != 1 || c.post_sweeps != 1) {
        P->err = "p2g_part_setup: the partitioned path runs the multicolour GS smoother with r1 = r2 = 1";
        return P2G_EINVAL;
    }
    for (auto& L : P->parts) {
        if (!L.h->have_values || L.h->k < 1 || L.h->B != P->B) {
            P->err = "p2g_part_setup: every hosted partition needs pattern, values and basis";
            return P2G_ESTATE;
        }
        L.h->cfg = c;
        PCU(cudaMemsetAsync(L.h->d_setup_status, 0, sizeof(int) * L.h->Bp, P->stream));
        Mat A = mat_of(L.h);
        dim3 g(std::max(1, std::min(1024, (int)((L.h->pat.n + 255) / 256))), L.h->B);
        k_check_diag<<<g, 256, 0, P->stream>>>(A, L.h->B, L.h->d_setup_status);
    }
    PTRY(pdispatch(P, [&](auto R) -> int { return decltype(R)::setup(P); }));
    PTRY(part_allmax_int(P, &p2g_handle::d_setup_status, P->parts[0].h->Bp));
    PCU(cudaStreamSynchronize(P->stream));
    std::vector<int> st(P->parts[0].h->Bp);
    PCU(cudaMemcpy(st.data(), P->parts[0].h->d_setup_status, sizeof(int) * st.size(),
                   cudaMemcpyDeviceToHost));
    int worst = P2G_OK;
    for (int b = 0; b < P->B; ++b) {
        if (status) status[b] = st[b];
        if (st[b] != P2G_OK) worst = st[b];
    }
    for (auto& L : P->parts) L.h->setup_done = true;
    P->setup_done = true;
    return worst;
}

// b / x: one pointer per hosted partition (in hosted order = rank order for
// the in-process group), each [B][n_own] in the caller's local row order.
int p2g_part_solve(p2g_part* P, const double* const* b, const double* const* x0, int32_t x0_mode,
                   double tol, int64_t max_iter, double* const* x, int64_t* iters,
                   int32_t* converged, int32_t* status, double* hist, int64_t hist_cap) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    if (!P->setup_done) {
        P->err = "p2g_part_solve: p2g_part_setup not called";
        return P2G_ESTATE;
    }
    if (!b || (x0_mode == P2G_X0_GIVEN && !x0) || max_iter < 0 || hist_cap < 0) {
        P->err = "p2g_part_solve: bad arguments";
        return P2G_EINVAL;
    }
    if (x0_mode != P2G_X0_ZERO && x0_mode != P2G_X0_GIVEN && x0_mode != P2G_X0_REDUCED) {
        P->err = "p2g_part_solve: x0_mode must be ZERO, GIVEN or REDUCED (no surrogate on the "
                 "partitioned path)";
        return P2G_EINVAL;
    }
    const int64_t cap_dev = std::max<int64_t>(hist_cap, 1);
    struct Events {  // destroyed on every exit path
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        Events() { cudaEventCreate(&e0); cudaEventCreate(&e1); }
        ~Events() { cudaEventDestroy(e0); cudaEventDestroy(e1); }
    } ev;
    cudaEvent_t e0 = ev.e0, e1 = ev.e1;
    cudaEventRecord(e0, P->stream);
    for (size_t q = 0; q < P->parts.size(); ++q) {
        p2g_handle* h = P->parts[q].h;
        if (ensure(h, h->d_hist, (size_t)cap_dev * h->Bp) != P2G_OK) {
            P->err = h->err;
            return P2G_ECUDA;
        }
        SolveParams prm{tol, (long long)max_iter, (long long)hist_cap};
        PCU(cudaMemcpyAsync(h->d_prm, &prm, sizeof(prm), cudaMemcpyHostToDevice, P->stream));
        if (upload_interleaved(h, b[q], nullptr, h->pat.n, h->d_perm, h->d_b) != P2G_OK) {
            P->err = h->err;
            return P2G_ECUDA;
        }
        if (x0_mode == P2G_X0_GIVEN &&
            upload_interleaved(h, x0[q], nullptr, h->pat.n, h->d_perm, h->d_u) != P2G_OK) {
            P->err = h->err;
            return P2G_ECUDA;
        }
        if (x0_mode == P2G_X0_ZERO)
            PCU(cudaMemsetAsync(h->d_u, 0, (size_t)(h->pat.n + h->n_ghost) * h->Bp * sizeof(double),
                                P->stream));
        PCU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                            P->stream));
    }
    if (!P->loop_exec || P->graph_key != part_graph_key(P)) PTRY(build_part_graph(P));
    PTRY(pdispatch(P, [&](auto R) -> int { return decltype(R)::prologue(P, x0_mode); }));
    // instances deactivate on the device (exact stopping: iteration counts,
    // history and solution equal those of independent solves)
    const int Bp = P->parts[0].h->Bp;
    int64_t replays = 0;
    if (P->graph_mode == 1) {
        // the whole loop on the device: conditional WHILE node
        PCU(cudaGraphLaunch(P->loop_exec, P->stream));
    } else {
        // chunks of kPartChunk iterations (captured, or eager), the host
        // polling "any active" between chunks
        int64_t done = 0;
        std::vector<int> act(Bp);
        for (;;) {
            PCU(cudaMemcpyAsync(act.data(), P->parts[0].h->d_active, sizeof(int) * Bp,
                                cudaMemcpyDeviceToHost, P->stream));
            PCU(cudaStreamSynchronize(P->stream));
            bool any = false;
            for (int v : act) any |= v != 0;
            if (!any || done >= max_iter) break;
            if (P->graph_mode == 2) {
                PCU(cudaGraphLaunch(P->loop_exec, P->stream));
                ++replays;
            } else {
                for (int q = 0; q < kPartChunk; ++q)
                    PTRY(pdispatch(P, [&](auto R) -> int { return decltype(R)::iteration(P); }));
            }
            done += kPartChunk;
        }
    }
    for (auto& L : P->parts) {
        p2g_handle* h = L.h;
        const dim3 g((unsigned)std::min<int64_t>((h->pat.n + 255) / 256, 1024), h->B);
        k_check_finite<<<g, 256, 0, P->stream>>>(static_cast<int>(h->pat.n), h->Bp, h->d_u,
                                                  h->d_status);
    }
    PTRY(part_allmax_int(P, &p2g_handle::d_status, Bp));
    if (P->graph_mode == 2) {
        P->parts[0].h->launches_executed += replays * kPartChunk * P->launches_per_iter;
    }
    for (size_t q = 0; q < P->parts.size(); ++q)
        if (x && x[q] && download_interleaved(P->parts[q].h, P->parts[q].h->d_u, x[q], nullptr) != P2G_OK) {
            P->err = P->parts[q].h->err;
            return P2G_ECUDA;
        }
    cudaEventRecord(e1, P->stream);
    PCU(cudaStreamSynchronize(P->stream));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    P->last_ms = ms;
    p2g_handle* h = P->parts[0].h;
    std::vector<int> it(Bp), stt(Bp);
    std::vector<double> rel(Bp);
    PCU(cudaMemcpy(it.data(), h->d_iters, sizeof(int) * Bp, cudaMemcpyDeviceToHost));
    PCU(cudaMemcpy(stt.data(), h->d_status, sizeof(int) * Bp, cudaMemcpyDeviceToHost));
    PCU(cudaMemcpy(rel.data(), h->d_rel, sizeof(double) * Bp, cudaMemcpyDeviceToHost));
    if (P->graph_mode == 1) {  // set_cond + one body per iteration of the slowest instance
        int maxit = 0;
        for (int bb = 0; bb < P->B; ++bb) maxit = std::max(maxit, it[bb]);
        P->parts[0].h->launches_executed += 1 + (int64_t)maxit * P->launches_per_iter;
    }
    int worst = P2G_OK;
    for (int bb = 0; bb < P->B; ++bb) {
        if (iters) iters[bb] = it[bb];
        if (converged) converged[bb] = rel[bb] <= tol ? 1 : 0;
        if (status) status[bb] = stt[bb];
        if (stt[bb] != P2G_OK) worst = stt[bb];
    }
    if (hist && hist_cap > 0) {
        PCU(cudaMemcpy(hist, h->d_hist, sizeof(double) * hist_cap * P->B, cudaMemcpyDeviceToHost));
        for (int bb = 0; bb < P->B; ++bb)
            for (int64_t q = std::min<int64_t>(it[bb] + 1, hist_cap); q < hist_cap; ++q)
                hist[bb * hist_cap + q] = NAN;
    }
    return worst;
}

int p2g_part_last_solve_ms(const p2g_part* P, double* ms) {
    if (!P || !ms) return P2G_EINVAL;
    *ms = P->last_ms;
    return P2G_OK;
}

void* p2g_part_get_stream(const p2g_part* P) { return P ? (void*)P->stream : nullptr; }

int p2g_part_launch_counts(const p2g_part* P, int64_t* per_iteration, int64_t* total,
                           int32_t* loop_mode) {
    if (!P) return P2G_EINVAL;
    int64_t t = 0;
    for (const auto& L : P->parts) t += L.h->launches_executed;
    if (per_iteration) *per_iteration = P->launches_per_iter;
    if (total) *total = t;
    if (loop_mode) *loop_mode = P->graph_mode;
    return P2G_OK;
}

int p2g_part_profile_iteration(p2g_part* P, int32_t reps, double* ms, double* bytes,
                               const char** names) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    if (P->parts.size() != 1 || !P->setup_done || reps < 1) {
        P->err = "p2g_part_profile_iteration: one hosted partition, after p2g_part_solve, reps >= 1";
        return P2G_ESTATE;
    }
    p2g_handle* h = P->parts[0].h;
    std::vector<double> acc(P2G_NUM_KCLASS, 0.0);
    SolveParams prm{0.0, (long long)1 << 62, 0};
    PCU(cudaMemcpyAsync(h->d_prm, &prm, sizeof(prm), cudaMemcpyHostToDevice, P->stream));
    for (int rep = 0; rep < reps; ++rep) {
        PCU(cudaMemcpyAsync(h->d_active, h->d_all, sizeof(int) * h->Bp, cudaMemcpyDeviceToDevice,
                            P->stream));
        if (kp_recurrence(h)) {  // refresh Kp and the pKp partials (the body starts at alpha)
            PTRY(part_exchange(P, &p2g_handle::d_p, -1));
            PTRY(pdispatch(P, [&](auto R) -> int {
                using Rn = typename decltype(R)::R;
                return Rn::spmv(h, h->d_p, h->d_Kp, true, nullptr);
            }));
        }
        // as p2g_profile_iteration: the body captured with its event nodes and
        // replayed as a graph (P2G_PROFILE_EAGER=1: eager)
        const char* pe = std::getenv("P2G_PROFILE_EAGER");
        const bool eager = pe && pe[0] == '1';
        auto body = [&]() -> int {
            h->profiling = true;
            h->kev_n = 0;
            PCU(prof_record(h, h->kev[0], P->stream));
            const int st = pdispatch(P, [&](auto R) -> int { return decltype(R)::iteration(P); });
            h->profiling = false;
            return st;
        };
        if (eager) {
            PTRY(body());
        } else {
            PCU(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeRelaxed));
            h->capturing = true;
            const int st = body();
            h->capturing = false;
            cudaGraph_t g = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(P->stream, &g);
            PTRY(st);
            PCU(ce);
            cudaGraphExec_t ge = nullptr;
            const cudaError_t ie = cudaGraphInstantiate(&ge, g, 0);
            cudaGraphDestroy(g);
            PCU(ie);
            const cudaError_t le = cudaGraphLaunch(ge, P->stream);
            cudaStreamSynchronize(P->stream);
            cudaGraphExecDestroy(ge);
            PCU(le);
        }
        PCU(cudaStreamSynchronize(P->stream));
        for (int q = 0; q < h->kev_n; ++q) {
            float t = 0;
            cudaEventElapsedTime(&t, h->kev[q], h->kev[q + 1]);
            acc[h->kev_class[q]] += t;
        }
    }
    double by[P2G_NUM_KCLASS];
    class_bytes(h, by);
    for (int q = 0; q < P2G_NUM_KCLASS; ++q) {
        if (ms) ms[q] = acc[q] / reps;
        if (bytes) bytes[q] = by[q];
        if (names) names[q] = kKclassNames[q];
    }
    return P2G_OK;
}

}  // extern "C"

extern "C" int p2g_plan_partition(int rank, int world, const int64_t* row_bounds, int64_t n_global,
                                  const uint64_t* row_offsets, const uint64_t* col_indices,
                                  int32_t block_size, const int32_t* node_colors, int64_t* sizes,
                                  int64_t* ghost_global, int64_t* send_counts, int64_t* recv_counts,
                                  char* errbuf, int32_t errcap) {
    PartitionPlan plan;
    const std::string msg = build_partition_plan(rank, world, row_bounds, n_global, row_offsets,
                                                 col_indices, block_size, node_colors, plan);
    if (!msg.empty()) {
        if (errbuf && errcap > 0) {
            std::strncpy(errbuf, msg.c_str(), errcap - 1);
            errbuf[errcap - 1] = 0;
        }
        return P2G_EINVAL;
    }
    if (sizes) {
        sizes[0] = plan.n_own;
        sizes[1] = plan.n_ghost;
        sizes[2] = plan.nnz;
        sizes[3] = plan.ncolors;
    }
    if (ghost_global)
        std::memcpy(ghost_global, plan.ghost_global.data(), sizeof(int64_t) * plan.n_ghost);
    for (int c = 0; c < plan.ncolors; ++c) {
        if (send_counts)
            for (const auto& m : plan.send_c[c]) send_counts[c * world + m.peer] += m.count;
        if (recv_counts)
            for (const auto& m : plan.recv_c[c]) recv_counts[c * world + m.peer] += m.count;
    }
    return P2G_OK;
}

extern "C" int p2g_mesh_assemble_into(const p2g_mesh* m, p2g_handle* h, int32_t batch,
                                      const double* E, int32_t E_on_device) {
    if (!h) return P2G_EINVAL;
    CU(cudaSetDevice(h->device));
    MeshDesc md;
    REQ(mesh_desc(m, md) && md.n == h->pat.n + 0 && md.nnz == h->pat.nnz, P2G_EINVAL,
        "p2g_mesh_assemble_into: the handle's pattern is not this mesh's");
    return assemble_impl(h, m, batch, E, 0, E_on_device != 0);
}

extern "C" int p2g_part_assemble(p2g_part* P, int rank, const p2g_mesh* m, int32_t batch,
                                 const double* E, int32_t E_on_device) {
    if (!P) return P2G_EINVAL;
    PCU(cudaSetDevice(P->device));
    PartLocal* L = local_of(P, rank);
    if (!L) return P2G_EINVAL;
    MeshDesc md;
    if (!mesh_desc(m, md) || md.n != L->plan.n_global) {
        P->err = "p2g_part_assemble: mesh does not match the partitioned system";
        return P2G_EINVAL;
    }
    const int st = assemble_impl(L->h, m, batch, E, L->plan.row_begin, E_on_device != 0);
    if (st != P2G_OK) {
        P->err = L->h->err;
        return st;
    }
    const size_t need = (size_t)std::max<int64_t>(L->rows_all, 1) * L->h->Bp;
    if (L->sendbuf_elems < need) {
        if (L->d_sendbuf) cudaFree(L->d_sendbuf);
        PCU(cudaMalloc(&L->d_sendbuf, sizeof(double) * need));
        L->sendbuf_elems = need;
    }
    P->B = batch;
    P->setup_done = false;
    return P2G_OK;
}
