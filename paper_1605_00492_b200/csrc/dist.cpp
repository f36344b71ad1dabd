// Partition plans for the distributed hierarchy (see dist.h).
#include "dist.h"

#include <algorithm>
#include <stdexcept>

namespace hmg {

int64_t LevelPlan::local_of(int64_t g) const {
    if (g >= off && g < off + n_own) return g - off;
    // halo: grouped by owner rank, ascending gid within a group; owner ranges are
    // ascending in gid too, so the whole list is ascending
    auto it = std::lower_bound(halo_gid.begin(), halo_gid.end(), g);
    if (it != halo_gid.end() && *it == g) return n_own + (it - halo_gid.begin());
    return -1;
}

LevelPlan plan_level(int ref, const std::vector<int32_t>& nbr, int rank, int nranks) {
    if (nranks < 1 || 320 % nranks != 0) throw std::invalid_argument("nranks must divide 320");
    if (ref < 2 && nranks > 1) throw std::invalid_argument("distributed levels need ref >= 2");
    LevelPlan P;
    P.ref = ref;
    P.n_global = (int64_t)(nbr.size() / 3);
    const int64_t per = P.n_global / nranks;
    P.off = (int64_t)rank * per;
    P.n_own = per;
    auto owner = [&](int64_t g) { return (int)(g / per); };
    // halo: neighbours outside the owned range
    std::vector<int64_t> halo;
    for (int64_t c = P.off; c < P.off + P.n_own; ++c)
        for (int j = 0; j < 3; ++j) {
            const int64_t o = nbr[c * 3 + j];
            if (o < P.off || o >= P.off + P.n_own) halo.push_back(o);
        }
    std::sort(halo.begin(), halo.end());
    halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
    P.halo_gid = halo;   // ascending gid == grouped by owner (owner ranges are ascending)
    // local neighbour table
    P.nbr_local.resize(P.n_own * 3);
    for (int64_t c = 0; c < P.n_own; ++c)
        for (int j = 0; j < 3; ++j) P.nbr_local[c * 3 + j] = (int32_t)P.local_of(nbr[(P.off + c) * 3 + j]);
    // receive side: contiguous halo runs per owner
    for (int64_t i = 0; i < (int64_t)halo.size();) {
        const int q = owner(halo[i]);
        int64_t e = i;
        while (e < (int64_t)halo.size() && owner(halo[e]) == q) ++e;
        PeerPlan pp;
        pp.rank = q;
        pp.recv_offset = i;
        pp.recv_count = e - i;
        P.peers.push_back(pp);
        i = e;
    }
    // send side: my owned cells adjacent to a cell of peer q, ascending gid
    // (adjacency is symmetric, so this is exactly q's halo run from me)
    for (PeerPlan& pp : P.peers) {
        const int q = pp.rank;
        for (int64_t c = P.off; c < P.off + P.n_own; ++c) {
            bool adj = false;
            for (int j = 0; j < 3; ++j) adj = adj || owner(nbr[c * 3 + j]) == q;
            if (adj) pp.send_local.push_back((int32_t)(c - P.off));
        }
    }
    return P;
}

}  // namespace hmg
