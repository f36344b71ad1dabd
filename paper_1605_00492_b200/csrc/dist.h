// Horizontal domain decomposition of the icosahedral hierarchy (
// the paper's MPI decomposition with PyOP2 halo exchanges).
//
// Rank r of P owns the ref-2 cells [r*320/P, (r+1)*320/P); because the
// children of cell p are 4p..4p+3, it then owns the contiguous global range
// [r*n/P, (r+1)*n/P) on every level ref >= 2, so restriction and
// prolongation are rank-local and only neighbour gathers cross ranks.
// Levels ref <= gather_ref are replicated on every rank (the coarse gather).
#pragma once
#include <cstdint>
#include <vector>

namespace hmg {

struct PeerPlan {
    int rank = 0;
    std::vector<int32_t> send_local;  // my owned cells (local index) that the peer holds in its halo, by global id
    int64_t recv_offset = 0;          // first halo slot (relative to n_own) filled from this peer
    int64_t recv_count = 0;
};

struct LevelPlan {
    int ref = 0;
    int64_t n_global = 0;
    int64_t off = 0;                  // global id of local cell 0
    int64_t n_own = 0;
    std::vector<int64_t> halo_gid;    // halo cells, grouped by owner rank, ascending global id
    std::vector<int32_t> nbr_local;   // [n_own][3] neighbours in local numbering
    std::vector<PeerPlan> peers;      // ascending rank
    int64_t n_halo() const { return (int64_t)halo_gid.size(); }
    // local index of global cell g (owned or halo), -1 if not present
    int64_t local_of(int64_t g) const;
};

// Plan of one distributed level from the global neighbour table [n][3].
// Valid for ref >= 2 and nranks dividing 320.
LevelPlan plan_level(int ref, const std::vector<int32_t>& nbr_global, int rank, int nranks);

}  // namespace hmg
