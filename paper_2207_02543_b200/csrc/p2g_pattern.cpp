// p2g_pattern.cpp -- see p2g_pattern.h.
//
// Colouring: nodes (groups of bs consecutive rows) are coloured greedily in
// natural node order, each node taking the smallest colour unused by its
// already-coloured neighbours.  On the structured Q4 / hex8 meshes of the
// benchmark configs this yields the 2^d parity colouring (4 colours in 2D,
// 8 in 3D).  The new numbering is sorted by (colour, node, component), so
//  * the rows of one colour are contiguous,
//  * a node's dofs stay adjacent and in order,
//  * in every row the entries with smaller new index (L part) precede the
//    diagonal, which precedes the U part -- the layout the forward sweep
//    (L only) and the upper-form residual (U only) exploit.
// Natural-order Gauss-Seidel (smoothers.hpp:26-72) on the permuted system is
// exactly what the GPU's colour-phase sweeps compute.
#include "p2g_pattern.h"

#include <algorithm>
#include <cstdlib>
#include <numeric>
#include <string>

namespace p2g {

std::vector<int32_t> order_colours(int ncol, const std::vector<double>& W) {
    std::vector<int32_t> seq(ncol), best;
    std::iota(seq.begin(), seq.end(), 0);
    auto cost = [&](const std::vector<int32_t>& q) {
        double c = 0.0;
        for (int t = 0; t + 1 < ncol; ++t) c += W[(size_t)q[t] * ncol + q[t + 1]];
        return c;
    };
    if (ncol <= 9) {
        double bc = 0.0;
        do {
            const double c = cost(seq);
            if (best.empty() || c < bc) bc = c, best = seq;
        } while (std::next_permutation(seq.begin(), seq.end()));
    } else {
        std::vector<char> used(ncol, 0);
        best.push_back(0);
        used[0] = 1;
        for (int t = 1; t < ncol; ++t) {
            int nxt = -1;
            for (int c = 0; c < ncol; ++c)
                if (!used[c] && (nxt < 0 || W[(size_t)best.back() * ncol + c] <
                                                W[(size_t)best.back() * ncol + nxt]))
                    nxt = c;
            best.push_back(nxt);
            used[nxt] = 1;
        }
    }
    std::vector<int32_t> rank(ncol);
    for (int t = 0; t < ncol; ++t) rank[best[t]] = t;
    return rank;
}

std::string build_coloured_pattern(int64_t n, const uint64_t* rp, const uint64_t* ci, int bs,
                                   ColouredPattern& out, int wave_colours) {
    if (n <= 0) return "p2g_set_pattern: n must be positive";
    if (bs < 1 || bs > 8) return "p2g_set_pattern: block_size outside [1,8]";
    if (n % bs != 0) return "p2g_set_pattern: n not a multiple of block_size";
    if (!rp || !ci) return "p2g_set_pattern: null array";
    // core/csr.hpp:33-46
    if (rp[0] != 0) return "csr: row_offsets[0] != 0";
    for (int64_t i = 0; i < n; ++i)
        if (rp[i] > rp[i + 1]) return "csr: decreasing row_offsets";
    const uint64_t nnz = rp[n];
    if (nnz > static_cast<uint64_t>(INT32_MAX))
        return "p2g_set_pattern: nnz exceeds the int32 device index range";
    if (static_cast<uint64_t>(n) > static_cast<uint64_t>(INT32_MAX))
        return "p2g_set_pattern: n exceeds the int32 device index range";
    std::vector<int32_t> dpos_old(n, -1);
    for (int64_t i = 0; i < n; ++i) {
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] >= static_cast<uint64_t>(n)) return "csr: column index out of range";
            if (k > rp[i] && !(ci[k - 1] < ci[k])) return "csr: columns not strictly increasing";
            if (ci[k] == static_cast<uint64_t>(i)) dpos_old[i] = static_cast<int32_t>(k);
        }
        if (dpos_old[i] < 0)
            return "p2g_set_pattern: row " + std::to_string(i) +
                   " has no stored diagonal (smoothers.hpp:41-43 zero diagonal)";
    }

    const int64_t nn = n / bs;
    // node adjacency (CSR over nodes, deduplicated)
    std::vector<int64_t> nadj_off(nn + 1, 0);
    std::vector<int64_t> nadj;
    {
        std::vector<int64_t> tmp;
        for (int64_t a = 0; a < nn; ++a) {
            tmp.clear();
            for (int c = 0; c < bs; ++c) {
                const int64_t i = a * bs + c;
                for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                    const int64_t b = static_cast<int64_t>(ci[k]) / bs;
                    if (b != a) tmp.push_back(b);
                }
            }
            std::sort(tmp.begin(), tmp.end());
            tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
            nadj.insert(nadj.end(), tmp.begin(), tmp.end());
            nadj_off[a + 1] = static_cast<int64_t>(nadj.size());
        }
    }
    // structural symmetry of the node graph: required for the colouring to be
    // a valid independent-set partition in both sweep directions
    for (int64_t a = 0; a < nn; ++a)
        for (int64_t q = nadj_off[a]; q < nadj_off[a + 1]; ++q) {
            const int64_t b = nadj[q];
            if (!std::binary_search(nadj.begin() + nadj_off[b], nadj.begin() + nadj_off[b + 1], a))
                return "p2g_set_pattern: pattern is not structurally symmetric";
        }

    std::vector<int32_t> color(nn, -1);
    int ncol = 0;
    std::vector<int64_t> mark(64, -1);
    for (int64_t a = 0; a < nn; ++a) {
        for (int64_t q = nadj_off[a]; q < nadj_off[a + 1]; ++q) {
            const int32_t c = color[nadj[q]];
            if (c >= 0) {
                if (c >= static_cast<int32_t>(mark.size())) mark.resize(c + 1, -1);
                mark[c] = a;
            }
        }
        int32_t c = 0;
        while (c < static_cast<int32_t>(mark.size()) && mark[c] == a) ++c;
        if (c >= static_cast<int32_t>(mark.size())) mark.resize(c + 1, -1);
        color[a] = c;
        ncol = std::max(ncol, c + 1);
    }
    if (ncol > 64) return "p2g_set_pattern: more than 64 node colours";

    // wavefront colouring (wave_colours = C; P2G_WAVE_COLOURS=C): colour = level mod C
    // with level = the node's level in natural-order Gauss-Seidel's dependency
    // DAG, classes run in level order -- as C grows, natural order.
    bool wave = false;
    if (wave_colours < 0) {
        const char* w = std::getenv("P2G_WAVE_COLOURS");
        wave_colours = w ? std::atoi(w) : 0;
    }
    {
        const int C = wave_colours;
        if (C >= 2 && C <= 64) {
            std::vector<int64_t> lev(nn, 0);
            for (int64_t a = 0; a < nn; ++a)
                for (int64_t q = nadj_off[a]; q < nadj_off[a + 1] && nadj[q] < a; ++q)
                    lev[a] = std::max(lev[a], lev[nadj[q]] + 1);
            bool ok = true;
            for (int64_t a = 0; a < nn && ok; ++a)
                for (int64_t q = nadj_off[a]; q < nadj_off[a + 1]; ++q)
                    if (lev[a] % C == lev[nadj[q]] % C) { ok = false; break; }
            if (ok) {
                int64_t mx = 0;
                for (int64_t a = 0; a < nn; ++a) {
                    color[a] = static_cast<int32_t>(lev[a] % C);
                    mx = std::max(mx, lev[a]);
                }
                ncol = static_cast<int>(std::min<int64_t>(C, mx + 1));
                wave = true;
            }
        }
    }

    if (!wave)  // class coupling: the mean strength of the adjacent node pairs between two
    // classes, strength = common neighbours (pattern-only: Q4 edge / diagonal
    // neighbours share 4 / 2, hex8 face / edge / corner neighbours 16 / 10 /
    // 6); sampled on large graphs
    {
        std::vector<double> W((size_t)ncol * ncol, 0.0), P((size_t)ncol * ncol, 0.0);
        const int64_t stride = std::max<int64_t>(1, nn / 200000);
        for (int64_t a = 0; a < nn; a += stride)
            for (int64_t q = nadj_off[a]; q < nadj_off[a + 1]; ++q) {
                const int64_t b = nadj[q];
                int64_t common = 0;
                for (int64_t x = nadj_off[a], y = nadj_off[b]; x < nadj_off[a + 1] && y < nadj_off[b + 1];) {
                    if (nadj[x] < nadj[y]) ++x;
                    else if (nadj[y] < nadj[x]) ++y;
                    else ++common, ++x, ++y;
                }
                W[(size_t)color[a] * ncol + color[b]] += static_cast<double>(common);
                P[(size_t)color[a] * ncol + color[b]] += 1.0;
            }
        for (int x = 0; x < ncol; ++x)
            for (int y = x + 1; y < ncol; ++y) {
                const double w = W[(size_t)x * ncol + y] + W[(size_t)y * ncol + x];
                const double c = P[(size_t)x * ncol + y] + P[(size_t)y * ncol + x];
                W[(size_t)x * ncol + y] = W[(size_t)y * ncol + x] = c > 0 ? w / c : 0.0;
            }
        const std::vector<int32_t> rank = order_colours(ncol, W);
        for (int64_t a = 0; a < nn; ++a) color[a] = rank[color[a]];
    }

    // counting sort of nodes by colour (stable in node index)
    std::vector<int64_t> cnt(ncol + 1, 0);
    for (int64_t a = 0; a < nn; ++a) ++cnt[color[a] + 1];
    for (int c = 0; c < ncol; ++c) cnt[c + 1] += cnt[c];
    std::vector<int64_t> node_new_order(nn);
    {
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t a = 0; a < nn; ++a) node_new_order[pos[color[a]]++] = a;
    }
    out.n = n;
    out.nnz = static_cast<int64_t>(nnz);
    out.bs = bs;
    out.ncolors = ncol;
    out.color_rows.assign(ncol + 1, 0);
    for (int c = 0; c <= ncol; ++c) out.color_rows[c] = cnt[c] * bs;
    out.perm.resize(n);
    out.iperm.resize(n);
    for (int64_t na = 0; na < nn; ++na)
        for (int c = 0; c < bs; ++c) {
            const int64_t newi = na * bs + c, oldi = node_new_order[na] * bs + c;
            out.perm[newi] = oldi;
            out.iperm[oldi] = newi;
        }

    out.rp.assign(n + 1, 0);
    out.ci.resize(nnz);
    out.vperm.resize(nnz);
    out.dpos.resize(n);
    std::vector<std::pair<int32_t, int64_t>> row;
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t o = out.perm[i];
        row.clear();
        for (uint64_t k = rp[o]; k < rp[o + 1]; ++k)
            row.emplace_back(static_cast<int32_t>(out.iperm[ci[k]]), static_cast<int64_t>(k));
        std::sort(row.begin(), row.end());
        for (const auto& [c, k] : row) {
            if (c == i) out.dpos[i] = static_cast<int32_t>(w);
            out.ci[w] = c;
            out.vperm[w] = k;
            ++w;
        }
        out.rp[i + 1] = static_cast<int32_t>(w);
    }
    return "";
}

bool build_node_table(int64_t n, int bs, const std::vector<int32_t>& rp,
                      const std::vector<int32_t>& ci, const std::vector<int32_t>& dpos,
                      std::vector<int32_t>& info, std::vector<int32_t>& ncol, int& nmax) {
    info.clear();
    ncol.clear();
    nmax = 0;
    if (bs < 1 || n % bs != 0) return false;
    const int64_t nn = n / bs;
    for (int64_t a = 0; a < nn; ++a) {
        const int64_t r0 = a * bs;
        const int32_t len = rp[r0 + 1] - rp[r0];
        if (len <= 0 || len % bs != 0 || len / bs > 32) return false;
        nmax = std::max(nmax, len / bs);
    }
    info.resize(4 * nn);
    ncol.assign(nn * nmax, 0);
    for (int64_t a = 0; a < nn; ++a) {
        const int64_t r0 = a * bs;
        const int32_t kb = rp[r0], len = rp[r0 + 1] - rp[r0], nnb = len / bs;
        int32_t pos = -1;
        for (int32_t j = 0; j < nnb; ++j) {
            const int32_t c0 = ci[kb + j * bs];
            if (c0 % bs != 0) return false;
            if (c0 == r0) pos = j;
            ncol[a * nmax + j] = c0 / bs;
            for (int c = 0; c < bs; ++c) {
                const int64_t kc = kb + (int64_t)c * len;
                if (rp[r0 + c + 1] - rp[r0 + c] != len || rp[r0 + c] != kc) return false;
                for (int cc = 0; cc < bs; ++cc)
                    if (ci[kc + j * bs + cc] != c0 + cc) return false;
            }
        }
        if (pos < 0) return false;
        for (int c = 0; c < bs; ++c)
            if (dpos[r0 + c] != kb + (int64_t)c * len + pos * bs + c) return false;
        info[4 * a + 0] = kb;
        info[4 * a + 1] = len;
        info[4 * a + 2] = pos;
        info[4 * a + 3] = nnb;
    }
    return true;
}

}  // namespace p2g
