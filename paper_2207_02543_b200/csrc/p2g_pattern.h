// p2g_pattern.h -- host-side pattern analysis for the B200 POD-2G path:
// validation (CsrMatrix::validate, core/csr.hpp:33-46), greedy node colouring
// and the colour-major permutation the multicolour smoother runs in.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace p2g {

struct ColouredPattern {
    int64_t n = 0, nnz = 0;
    int bs = 1;                           // dofs per node
    int ncolors = 0;
    std::vector<int64_t> perm;            // new row -> old row
    std::vector<int64_t> iperm;           // old row -> new row
    std::vector<int64_t> color_rows;      // ncolors+1 row offsets (new numbering)
    std::vector<int32_t> rp;              // new CSR row offsets (n+1)
    std::vector<int32_t> ci;              // new CSR columns (sorted ascending)
    std::vector<int32_t> dpos;            // new: position of the diagonal in each row
    std::vector<int64_t> vperm;           // new nnz position -> old nnz position
};

// Processing order of ncol colour classes given their coupling W (ncol x ncol,
// symmetric): the sequence minimising the total coupling between consecutive
// classes (exhaustive for ncol <= 9, nearest-neighbour chain beyond; the
// lexicographically first minimum).  Returns rank[c] = position of class c.
// Rationale (D1): weakly coupled classes run back to back, strongly
// coupled ones in different phases -- red-black-like on the strong couplings,
// which cuts the multicolour iteration count by 13-15 % on the Q4 / hex8
// benchmark meshes.
std::vector<int32_t> order_colours(int ncol, const std::vector<double>& W);

// Returns "" on success, else the require()-style message.  Validates the
// reference invariants, the presence of every diagonal, the int32 range, the
// node blocking (n % bs == 0) and structural symmetry of the node graph.
// wave_colours: C >= 2 selects the wavefront colouring (colour = level in
// natural-order GS's dependency DAG mod C; D1) when it is a proper
// colouring of this graph, 0 the greedy colouring, -1 reads P2G_WAVE_COLOURS.
std::string build_coloured_pattern(int64_t n, const uint64_t* row_offsets,
                                   const uint64_t* col_indices, int bs, ColouredPattern& out,
                                   int wave_colours = -1);

// Node-blocked view of a (coloured) local pattern for the node-blocked row
// kernels (NodeTab, p2g_kernels.cuh).  Returns false unless every node's bs
// rows share one ascending column list made of whole node blocks
// (bs consecutive columns starting at a multiple of bs) with at most 32
// neighbour nodes.  info[4a..4a+3] = {first value of row 0 of node a, row
// length, slot of node a in its own list, neighbour count}; ncol[a*nmax + j]
// = neighbour node j of node a (column / bs).  Columns may point past the
// owned rows (ghost nodes of a partitioned handle).
bool build_node_table(int64_t n, int bs, const std::vector<int32_t>& rp,
                      const std::vector<int32_t>& ci, const std::vector<int32_t>& dpos,
                      std::vector<int32_t>& info, std::vector<int32_t>& ncol, int& nmax);

}  // namespace p2g
