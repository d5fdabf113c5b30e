// p2g_mesh_desc.h -- what the device-side assembly needs to know about a
// structured generator mesh (p2g_mesh is opaque outside p2g_mesh.cpp).
#pragma once
#include <cstdint>

struct p2g_mesh;

namespace p2g {
struct MeshDesc {
    int dim = 2, ned = 8;
    int64_t nx = 0, ny = 0, nz = 1;  // elements per axis
    int64_t n = 0, nnz = 0, nelem = 0;
    const double* Ke = nullptr;      // ned x ned, E = 1
    const uint64_t* rp = nullptr;    // host row offsets of the generator CSR (n+1)
};
bool mesh_desc(const p2g_mesh* m, MeshDesc& d);
}  // namespace p2g
