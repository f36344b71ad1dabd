// Host-side icosahedral hierarchy for the CUDA path (setup only, untimed).
// Independent of oracle/: cells carry their own vertex triples and children's
// neighbours are derived structurally from the parent's (see mesh.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace hmg {

struct HostLevel {
    int ref = 0;
    int64_t n = 0;                 // cells = 20 * 4^ref
    std::vector<double> vtx;       // [n][3][3] vertex coordinates of each cell, counter-clockwise
    std::vector<int32_t> nbr;      // [n][3] cell across edge (v_j, v_{j+1})
    std::vector<double> area;      // [n]
    std::vector<double> len;       // [n][3]
    std::vector<double> cd;        // [n][3]
};

// Builds levels 0..fine_ref (index = ref).  Geometry per DESIGN.md reading R2.
std::vector<HostLevel> build_icosahedral_levels(int fine_ref);

}  // namespace hmg
