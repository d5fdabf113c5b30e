// p2g_partition.cpp -- see p2g_partition.h.
#include "p2g_partition.h"

#include <algorithm>
#include <map>
#include <numeric>

namespace p2g {

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

    // validate rows, collect ghosts
    std::map<int64_t, int> ghost_owner;  // global row -> owner
    for (int64_t i = 0; i < n_own; ++i) {
        bool diag = false;
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t c = static_cast<int64_t>(ci[k]);
            if (c < 0 || c >= n_global) return "csr: column index out of range";
            if (k > rp[i] && !(ci[k - 1] < ci[k])) return "csr: columns not strictly increasing";
            if (c == r0 + i) diag = true;
            if (c < r0 || c >= r1) ghost_owner[c] = owner(c);
        }
        if (!diag) return "partition: row without a stored diagonal";
    }
    // ghosts are whole nodes: a ghost row's node-mates are ghosts too
    {
        std::vector<int64_t> extra;
        for (const auto& [g, o] : ghost_owner)
            for (int c = 0; c < bs; ++c) extra.push_back(g - g % bs + c);
        for (int64_t g : extra) ghost_owner[g] = owner(g);
    }
    P = PartitionPlan();
    P.rank = rank;
    P.world = world;
    P.bs = bs;
    P.ncolors = ncol;
    P.n_global = n_global;
    P.row_begin = r0;
    P.row_end = r1;
    P.n_own = n_own;
    // owned rows colour-major (by global key)
    std::vector<int64_t> own(n_own);
    std::iota(own.begin(), own.end(), r0);
    std::stable_sort(own.begin(), own.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
    P.own_global = own;
    P.color_rows.assign(ncol + 1, 0);
    for (int64_t g : own) ++P.color_rows[color[g / bs] + 1];
    for (int c = 0; c < ncol; ++c) P.color_rows[c + 1] += P.color_rows[c];
    // ghosts ordered by (owner, colour, key)
    std::vector<int64_t> gh;
    for (const auto& [g, o] : ghost_owner) gh.push_back(g);
    std::stable_sort(gh.begin(), gh.end(), [&](int64_t a, int64_t b) {
        const int oa = owner(a), ob = owner(b);
        if (oa != ob) return oa < ob;
        return key(a) < key(b);
    });
    P.ghost_global = gh;
    P.n_ghost = static_cast<int64_t>(gh.size());
    std::map<int64_t, int32_t> local_of;  // global row -> local index
    for (int64_t i = 0; i < n_own; ++i) local_of[own[i]] = static_cast<int32_t>(i);
    for (int64_t j = 0; j < P.n_ghost; ++j) local_of[gh[j]] = static_cast<int32_t>(n_own + j);
    // local CSR, entries in global key order
    P.rp.assign(n_own + 1, 0);
    std::vector<std::pair<int64_t, int64_t>> row;
    for (int64_t li = 0; li < n_own; ++li) {
        const int64_t g = own[li], i = g - r0;
        row.clear();
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) row.emplace_back(key((int64_t)ci[k]), (int64_t)k);
        std::sort(row.begin(), row.end());
        for (const auto& [kk, k] : row) {
            const int64_t c = static_cast<int64_t>(ci[k]);
            if (c == g) P.dpos.push_back(static_cast<int32_t>(P.ci.size()));
            P.ci.push_back(local_of.at(c));
            P.vperm.push_back(k);
        }
        P.rp[li + 1] = static_cast<int32_t>(P.ci.size());
    }
    P.nnz = static_cast<int64_t>(P.ci.size());
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
    // whole nodes, in the receiver's ghost order (colour, key)
    std::map<int, std::vector<int64_t>> to_peer;
    for (int64_t li = 0; li < n_own; ++li) {
        const int64_t g = own[li], i = g - r0;
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int64_t c = static_cast<int64_t>(ci[k]);
            if (c < r0 || c >= r1)
                for (int cc = 0; cc < bs; ++cc) to_peer[owner(c)].push_back(g - g % bs + cc);
        }
    }
    for (auto& [q, v] : to_peer) {
        std::sort(v.begin(), v.end(), [&](int64_t a, int64_t b) { return key(a) < key(b); });
        v.erase(std::unique(v.begin(), v.end()), v.end());
        PartMsg all;
        all.peer = q;
        for (int64_t g : v) all.rows.push_back(local_of.at(g));
        all.count = static_cast<int64_t>(all.rows.size());
        P.send_all.push_back(all);
        for (size_t a = 0; a < v.size();) {
            const int c = color[v[a] / bs];
            PartMsg m;
            m.peer = q;
            while (a < v.size() && color[v[a] / bs] == c) m.rows.push_back(local_of.at(v[a++]));
            m.count = static_cast<int64_t>(m.rows.size());
            P.send_c[c].push_back(m);
        }
    }
    return "";
}

}  // namespace p2g
