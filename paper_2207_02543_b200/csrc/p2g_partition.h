// p2g_partition.h -- host-side plan of the row-partitioned single-system path
// (SURVEY 8(e), config c5): each rank owns a contiguous block of global rows
// (z-slabs for the node-major structured meshes) plus ghost copies of the
// neighbouring rows its rows couple to.
//
// Ordering.  All ranks use one GLOBAL node colouring.  Every local row keeps
// its entries sorted by the global colour-major key (colour, node, component)
// -- exactly the order of the single-GPU colour-permuted system -- so the L
// part (smaller key), the diagonal and the U part stay contiguous and every
// row sum is computed in the same order as on one GPU (bit-identical sweeps;
// only the cross-rank dot / restriction sums differ in association).
//
// Local numbering: owned rows colour-major [0, n_own), then ghost rows
// [n_own, n_own + n_ghost) ordered by (owner rank, colour, global row), so the
// ghosts a peer sends for one colour are contiguous, and so are all of them.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace p2g {

struct PartMsg {
    int peer = -1;
    std::vector<int32_t> rows;  // send: local owned rows, in the receiver's ghost order
    int64_t ghost_off = 0;      // recv: first ghost slot (local row index)
    int64_t count = 0;          // rows in the message
};

struct PartitionPlan {
    int rank = 0, world = 1, bs = 1, ncolors = 0;
    int64_t n_global = 0, row_begin = 0, row_end = 0;
    int64_t n_own = 0, n_ghost = 0, nnz = 0;
    std::vector<int64_t> color_rows;   // ncolors+1 owned-row offsets (local, colour-major)
    std::vector<int64_t> own_global;   // local owned row -> global row
    std::vector<int64_t> ghost_global; // ghost slot -> global row
    std::vector<int32_t> rp, ci, dpos; // local CSR (columns local, entries in global key order)
    std::vector<int64_t> vperm;        // local entry -> entry of the caller's local CSR
    // per colour: messages to / from each peer; plus the all-colour messages
    std::vector<std::vector<PartMsg>> send_c, recv_c;
    std::vector<PartMsg> send_all, recv_all;
};

// rows [row_begin, row_end) of a square pattern of n_global rows, given as a
// local CSR with GLOBAL column indices (size_t, sorted per row); row_bounds
// (world+1, multiples of bs) says which rank owns which rows; node_colors[g]
// is the colour of global node g (n_global / bs entries) -- a proper
// colouring of the node graph.  Returns "" or a require()-style message.
std::string build_partition_plan(int rank, int world, const int64_t* row_bounds, int64_t n_global,
                                 const uint64_t* row_offsets, const uint64_t* col_indices, int bs,
                                 const int32_t* node_colors, PartitionPlan& out);

}  // namespace p2g
