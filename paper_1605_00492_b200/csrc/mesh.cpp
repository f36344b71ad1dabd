// Icosahedral mesh hierarchy for the CUDA path: MeshHierarchy of
// UnitIcosahedralSphereMesh, built without a vertex
// table.  Each cell stores its three vertex coordinates; refinement splits it
// into 4p+0 = (a, m_ab, m_ca), 4p+1 = (m_ab, b, m_bc), 4p+2 = (m_ca, m_bc, c),
// 4p+3 = (m_ab, m_bc, m_ca) (reading R1), and the children's
// neighbour slots follow structurally from the parent's:
//   * corner child i lies on parent edges i and i+2 (mod 3) at the same slot
//     index; across parent edge e = (v_e, v_e+1) with neighbour q whose slot
//     s points back, the corner child at v_e meets q's child 4q+(s+1)%3 and
//     the corner child at v_e+1 meets 4q+s;
//   * corner child i's remaining slot (i+1)%3 faces the centre child 4p+3;
//   * the centre child's slot j faces corner child 4p+(j+1)%3.
// Midpoints m = normalise((a + b) * 0.5) are recomputed by both cells sharing
// an edge; a + b is commutative in IEEE arithmetic, so both get the same bits.
// Compile with -ffp-contract=off: geometry must be bitwise reproducible.
#include "mesh.h"

#include <cmath>
#include <stdexcept>

namespace hmg {
namespace {

inline void normalise3(double* v) {
    double r = std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]);
    v[0] = v[0] / r;
    v[1] = v[1] / r;
    v[2] = v[2] / r;
}

// The 12 vertices (0, +-1, +-phi), (+-1, +-phi, 0), (+-phi, 0, +-1) in the order
// of reading R1, and the 20 faces: every triple of mutually adjacent vertices
// in lexicographic order, oriented counter-clockwise seen from outside.
const int kBaseFaces[20][3] = {
    {0, 8, 2},  {0, 2, 9},  {0, 6, 4},  {0, 4, 8},  {0, 9, 6},  {1, 3, 10}, {1, 11, 3},
    {1, 4, 6},  {1, 10, 4}, {1, 6, 11}, {2, 5, 7},  {2, 8, 5},  {2, 7, 9},  {3, 7, 5},
    {3, 5, 10}, {3, 11, 7}, {4, 10, 8}, {5, 8, 10}, {6, 9, 11}, {7, 11, 9}};

void base_vertices(double v[12][3]) {
    const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
    int i = 0;
    for (int s1 : {-1, 1})
        for (int s2 : {-1, 1}) { v[i][0] = 0.0; v[i][1] = s1; v[i][2] = s2 * phi; ++i; }
    for (int s1 : {-1, 1})
        for (int s2 : {-1, 1}) { v[i][0] = s1; v[i][1] = s2 * phi; v[i][2] = 0.0; ++i; }
    for (int s1 : {-1, 1})
        for (int s2 : {-1, 1}) { v[i][0] = s2 * phi; v[i][1] = 0.0; v[i][2] = s1; ++i; }
    for (int k = 0; k < 12; ++k) normalise3(v[k]);
}

HostLevel base_level() {
    HostLevel L;
    L.ref = 0;
    L.n = 20;
    double v[12][3];
    base_vertices(v);
    L.vtx.resize(20 * 9);
    for (int c = 0; c < 20; ++c)
        for (int j = 0; j < 3; ++j)
            for (int d = 0; d < 3; ++d) L.vtx[c * 9 + j * 3 + d] = v[kBaseFaces[c][j]][d];
    // neighbour across edge (a, b) = the face holding the directed edge (b, a)
    L.nbr.assign(60, -1);
    for (int c = 0; c < 20; ++c)
        for (int j = 0; j < 3; ++j) {
            int a = kBaseFaces[c][j], b = kBaseFaces[c][(j + 1) % 3];
            for (int o = 0; o < 20; ++o)
                for (int i = 0; i < 3; ++i)
                    if (kBaseFaces[o][i] == b && kBaseFaces[o][(i + 1) % 3] == a) L.nbr[c * 3 + j] = o;
        }
    for (int x : L.nbr)
        if (x < 0) throw std::runtime_error("base icosahedron: open edge");
    return L;
}

HostLevel refine(const HostLevel& P) {
    HostLevel C;
    C.ref = P.ref + 1;
    C.n = P.n * 4;
    C.vtx.resize(C.n * 9);
    C.nbr.resize(C.n * 3);
    for (int64_t p = 0; p < P.n; ++p) {
        const double* a = &P.vtx[p * 9 + 0];
        const double* b = &P.vtx[p * 9 + 3];
        const double* c = &P.vtx[p * 9 + 6];
        double mab[3], mbc[3], mca[3];
        for (int d = 0; d < 3; ++d) {
            mab[d] = (a[d] + b[d]) * 0.5;
            mbc[d] = (b[d] + c[d]) * 0.5;
            mca[d] = (c[d] + a[d]) * 0.5;
        }
        normalise3(mab);
        normalise3(mbc);
        normalise3(mca);
        const double* tri[4][3] = {{a, mab, mca}, {mab, b, mbc}, {mca, mbc, c}, {mab, mbc, mca}};
        for (int k = 0; k < 4; ++k)
            for (int j = 0; j < 3; ++j)
                for (int d = 0; d < 3; ++d) C.vtx[(4 * p + k) * 9 + j * 3 + d] = tri[k][j][d];
        // structural neighbours
        int32_t* N = &C.nbr[4 * p * 3];
        for (int e = 0; e < 3; ++e) {
            int32_t q = P.nbr[p * 3 + e];
            int s = -1;
            for (int i = 0; i < 3; ++i)
                if (P.nbr[q * 3 + i] == (int32_t)p) s = i;
            if (s < 0) throw std::runtime_error("asymmetric neighbour table");
            // corner child at v_e (child e) and at v_{e+1} (child (e+1)%3), both at slot e
            N[e * 3 + e] = 4 * q + (s + 1) % 3;
            N[((e + 1) % 3) * 3 + e] = 4 * q + s;
        }
        for (int i = 0; i < 3; ++i) N[i * 3 + (i + 1) % 3] = (int32_t)(4 * p + 3);
        for (int j = 0; j < 3; ++j) N[3 * 3 + j] = (int32_t)(4 * p + (j + 1) % 3);
    }
    return C;
}

// Reading R2: area = 0.5 |(v1-v0) x (v2-v0)|, centroid ((v0+v1)+v2)/3,
// len_j = |v_{j+1} - v_j|, cd_j = |cen - cen_{N_j}|, |d| = sqrt((dx*dx+dy*dy)+dz*dz).
void geometry(HostLevel& L) {
    const int64_t n = L.n;
    L.area.resize(n);
    L.len.resize(n * 3);
    L.cd.resize(n * 3);
    std::vector<double> cen(n * 3);
    for (int64_t c = 0; c < n; ++c) {
        const double* v0 = &L.vtx[c * 9];
        const double* v1 = v0 + 3;
        const double* v2 = v0 + 6;
        double e1x = v1[0] - v0[0], e1y = v1[1] - v0[1], e1z = v1[2] - v0[2];
        double e2x = v2[0] - v0[0], e2y = v2[1] - v0[1], e2z = v2[2] - v0[2];
        double cx = e1y * e2z - e1z * e2y;
        double cy = e1z * e2x - e1x * e2z;
        double cz = e1x * e2y - e1y * e2x;
        L.area[c] = 0.5 * std::sqrt((cx * cx + cy * cy) + cz * cz);
        for (int d = 0; d < 3; ++d) cen[c * 3 + d] = ((v0[d] + v1[d]) + v2[d]) / 3.0;
        for (int j = 0; j < 3; ++j) {
            const double* p = v0 + 3 * j;
            const double* q = v0 + 3 * ((j + 1) % 3);
            double dx = q[0] - p[0], dy = q[1] - p[1], dz = q[2] - p[2];
            L.len[c * 3 + j] = std::sqrt((dx * dx + dy * dy) + dz * dz);
        }
    }
    for (int64_t c = 0; c < n; ++c)
        for (int j = 0; j < 3; ++j) {
            int64_t o = L.nbr[c * 3 + j];
            double dx = cen[c * 3] - cen[o * 3];
            double dy = cen[c * 3 + 1] - cen[o * 3 + 1];
            double dz = cen[c * 3 + 2] - cen[o * 3 + 2];
            L.cd[c * 3 + j] = std::sqrt((dx * dx + dy * dy) + dz * dz);
        }
}

}  // namespace

std::vector<HostLevel> build_icosahedral_levels(int fine_ref) {
    std::vector<HostLevel> levels;
    levels.reserve(fine_ref + 1);
    levels.push_back(base_level());
    for (int r = 1; r <= fine_ref; ++r) levels.push_back(refine(levels.back()));
    for (auto& L : levels) geometry(L);
    return levels;
}

}  // namespace hmg
