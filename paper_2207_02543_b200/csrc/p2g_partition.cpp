// p2g_partition.cpp -- see p2g_partition.h.
//
// Cost: O(nnz) plus per-row sorts, spread over the host's threads; no
// per-entry map lookups (the c5 rank plan, 12.4 M rows / 1e9 entries, is
// built in seconds).
#include "p2g_partition.h"

#include <algorithm>
#include <numeric>
#include <thread>

namespace p2g {

namespace {

template <class F>
void parallel_ranges(int64_t n, F&& f) {
    int nt = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    nt = static_cast<int>(std::min<int64_t>(nt, std::max<int64_t>(1, n / 16384)));
    if (nt <= 1) {
        f(0, int64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) {
        const int64_t a = n * t / nt, b = n * (t + 1) / nt;
        th.emplace_back([&f, t, a, b] { f(t, a, b); });
    }
    for (auto& x : th) x.join();
}

}  // namespace

std::string build_partition_plan(int rank, int world, const int64_t* bounds, int64_t n_global,
                                 const uint64_t* rp, const uint64_t* ci, int bs,
                                 const int32_t* color, PartitionPlan& P) {
    if (world < 1 || rank < 0 || rank >= world) return "partition: bad rank / world";
    if (bs < 1 || n_global <= 0 || n_global % bs) return "partition: bad n_global / block_size";
    if (!bounds || !rp || !ci || !color) return "partition: null argument";
    if (bounds[0] != 0 || bounds[world] != n_global) return "partition: row_bounds must span [0, n)";
    for (int q = 0; q < world; ++q)
        if (bounds[q] > bounds[q + 1] || bounds[q] % bs) return "partition: bad row_bounds";
    const int64_t r0 = bounds[rank], r1 = bounds[rank + 1], n_own = r1 - r0;
    const int64_t nn_global = n_global / bs;
    int ncol = 0;
    for (int64_t g = 0; g < nn_global; ++g) {
        if (color[g] < 0 || color[g] >= 64) return "partition: node colours must lie in [0, 64)";
        ncol = std::max(ncol, color[g] + 1);
    }
    // global colour-major key of every node: (colour, node) -> position
    std::vector<int64_t> cstart(ncol + 1, 0);
    for (int64_t g = 0; g < nn_global; ++g) ++cstart[color[g] + 1];
    for (int c = 0; c < ncol; ++c) cstart[c + 1] += cstart[c];
    std::vector<int64_t> nkey(nn_global);
    {
        std::vector<int64_t> pos(cstart.begin(), cstart.end() - 1);
        for (int64_t g = 0; g < nn_global; ++g) nkey[g] = pos[color[g]]++;
    }
    auto key = [&](int64_t grow) { return nkey[grow / bs] * bs + grow % bs; };
    auto owner = [&](int64_t grow) {
        return static_cast<int>(std::upper_bound(bounds, bounds + world + 1, grow) - bounds - 1);
    };

    // validate rows (parallel); collect the off-block rows each thread sees
    const int nth = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::string> terr(nth);
    std::vector<std::vector<int64_t>> toff(nth);
    parallel_ranges(n_own, [&](int t, int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            bool diag = false;
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int64_t c = static_cast<int64_t>(ci[k]);
                if (c < 0 || c >= n_global) {
                    terr[t] = "csr: column index out of range";
                    return;
                }
                if (k > rp[i] && !(ci[k - 1] < ci[k])) {
                    terr[t] = "csr: columns not strictly increasing";
                    return;
                }
                if (c == r0 + i) diag = true;
                if (c < r0 || c >= r1) toff[t].push_back(c - c % bs);  // the ghost's node
            }
            if (!diag) {
                terr[t] = "partition: row without a stored diagonal";
                return;
            }
        }
    });
    for (const auto& e : terr)
        if (!e.empty()) return e;
    // ghosts are whole nodes
    std::vector<int64_t> gnodes;
    for (auto& v : toff) gnodes.insert(gnodes.end(), v.begin(), v.end());
    std::sort(gnodes.begin(), gnodes.end());
    gnodes.erase(std::unique(gnodes.begin(), gnodes.end()), gnodes.end());

    P = PartitionPlan();
    P.rank = rank;
    P.world = world;
    P.bs = bs;
    P.ncolors = ncol;
    P.n_global = n_global;
    P.row_begin = r0;
    P.row_end = r1;
    P.n_own = n_own;
    // owned rows colour-major by global key: within a colour the key grows
    // with the node id, so a stable counting sort of the owned nodes by colour
    std::vector<int64_t> own(n_own);
    {
        std::vector<int64_t> cpos(ncol + 1, 0);
        for (int64_t g = r0; g < r1; g += bs) ++cpos[color[g / bs] + 1];
        for (int c = 0; c < ncol; ++c) cpos[c + 1] += cpos[c];
        for (int64_t g = r0; g < r1; g += bs) {
            int64_t& p = cpos[color[g / bs]];
            for (int cc = 0; cc < bs; ++cc) own[p * bs + cc] = g + cc;
            ++p;
        }
    }
    P.own_global = own;
    P.color_rows.assign(ncol + 1, 0);
    for (int64_t g : own) ++P.color_rows[color[g / bs] + 1];
    for (int c = 0; c < ncol; ++c) P.color_rows[c + 1] += P.color_rows[c];
    // ghosts ordered by (owner, colour, key)
    std::vector<int64_t> gh;
    gh.reserve(gnodes.size() * bs);
    for (int64_t g : gnodes)
        for (int cc = 0; cc < bs; ++cc) gh.push_back(g + cc);
    std::stable_sort(gh.begin(), gh.end(), [&](int64_t a, int64_t b) {
        const int oa = owner(a), ob = owner(b);
        if (oa != ob) return oa < ob;
        return key(a) < key(b);
    });
    P.ghost_global = gh;
    P.n_ghost = static_cast<int64_t>(gh.size());
    // global row -> local index: owned rows by table, ghosts by binary search
    std::vector<int32_t> own_local(n_own);
    for (int64_t li = 0; li < n_own; ++li) own_local[own[li] - r0] = static_cast<int32_t>(li);
    std::vector<std::pair<int64_t, int32_t>> gsorted(P.n_ghost);
    for (int64_t j = 0; j < P.n_ghost; ++j) gsorted[j] = {gh[j], static_cast<int32_t>(n_own + j)};
    std::sort(gsorted.begin(), gsorted.end());
    auto local_of = [&](int64_t c) -> int32_t {
        if (c >= r0 && c < r1) return own_local[c - r0];
        auto it = std::lower_bound(gsorted.begin(), gsorted.end(), std::make_pair(c, INT32_MIN));
        return it->second;
    };
    // local CSR, entries in global key order (rows in parallel)
    P.rp.assign(n_own + 1, 0);
    for (int64_t li = 0; li < n_own; ++li) {
        const int64_t i = own[li] - r0;
        P.rp[li + 1] = P.rp[li] + static_cast<int32_t>(rp[i + 1] - rp[i]);
    }
    P.nnz = P.rp[n_own];
    P.ci.resize(P.nnz);
    P.vperm.resize(P.nnz);
    P.dpos.resize(n_own);
    parallel_ranges(n_own, [&](int, int64_t a, int64_t b) {
        std::vector<std::pair<int64_t, int64_t>> row;
        for (int64_t li = a; li < b; ++li) {
            const int64_t g = own[li], i = g - r0;
            row.clear();
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k)
                row.emplace_back(key((int64_t)ci[k]), (int64_t)k);
            std::sort(row.begin(), row.end());
            int64_t o = P.rp[li];
            for (const auto& [kk, k] : row) {
                const int64_t c = static_cast<int64_t>(ci[k]);
                if (c == g) P.dpos[li] = static_cast<int32_t>(o);
                P.ci[o] = local_of(c);
                P.vperm[o] = k;
                ++o;
            }
        }
    });
    // receive messages: ghost slots per (peer, colour) -- contiguous by construction
    P.recv_c.assign(ncol, {});
    P.send_c.assign(ncol, {});
    for (int64_t j = 0; j < P.n_ghost;) {
        const int o = owner(gh[j]);
        const int64_t j0 = j;
        while (j < P.n_ghost && owner(gh[j]) == o) ++j;
        PartMsg all;
        all.peer = o;
        all.ghost_off = n_own + j0;
        all.count = j - j0;
        P.recv_all.push_back(all);
        for (int64_t q = j0; q < j;) {
            const int c = color[gh[q] / bs];
            const int64_t q0 = q;
            while (q < j && color[gh[q] / bs] == c) ++q;
            PartMsg m;
            m.peer = o;
            m.ghost_off = n_own + q0;
            m.count = q - q0;
            P.recv_c[c].push_back(m);
        }
    }
    // send messages: my rows that are ghosts on peer q = my rows coupled to a
    // row of q (structural symmetry, checked by the peers' receive counts);
    // whole nodes, in the receiver's ghost order (colour, key).  Only rows
    // with an off-block column matter: the owned boundary rows.
    std::vector<std::vector<std::pair<int, int64_t>>> tsend(nth);
    parallel_ranges(n_own, [&](int t, int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            const int64_t g = r0 + i;
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int64_t c = static_cast<int64_t>(ci[k]);
                if (c < r0 || c >= r1)
                    for (int cc = 0; cc < bs; ++cc) tsend[t].emplace_back(owner(c), g - g % bs + cc);
            }
        }
    });
    std::vector<std::pair<int, int64_t>> sends;
    for (auto& v : tsend) sends.insert(sends.end(), v.begin(), v.end());
    std::sort(sends.begin(), sends.end(), [&](const auto& x, const auto& y) {
        if (x.first != y.first) return x.first < y.first;
        return key(x.second) < key(y.second);
    });
    sends.erase(std::unique(sends.begin(), sends.end()), sends.end());
    for (size_t s = 0; s < sends.size();) {
        const int q = sends[s].first;
        std::vector<int64_t> v;
        while (s < sends.size() && sends[s].first == q) v.push_back(sends[s++].second);
        PartMsg all;
        all.peer = q;
        for (int64_t g : v) all.rows.push_back(local_of(g));
        all.count = static_cast<int64_t>(all.rows.size());
        P.send_all.push_back(all);
        for (size_t a = 0; a < v.size();) {
            const int c = color[v[a] / bs];
            PartMsg m;
            m.peer = q;
            while (a < v.size() && color[v[a] / bs] == c) m.rows.push_back(local_of(v[a++]));
            m.count = static_cast<int64_t>(m.rows.size());
            P.send_c[c].push_back(m);
        }
    }
    return "";
}

}  // namespace p2g
