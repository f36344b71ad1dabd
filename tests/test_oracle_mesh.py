"""Pins P1/P2 of the oracle's mesh and geometry (readings R1, R2).

The icosahedral hierarchy is the paper's MeshHierarchy(UnitIcosahedralSphereMesh)
(P:234-235).  Values checked here come from the mathematics of the
icosahedron, not from the oracle: Euler's formula, the closed-form geometry of
the regular icosahedron inscribed in the unit sphere, and the midpoint
refinement rule (children ordered 4*parent+k, BASELINE.json C0).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def h5():
    nz = 1
    lam = np.ones((nz, 20 * 4 ** 5))
    h = oracle.Hierarchy(5, 0, nz, 0.01, 1e-4, lam)
    yield h
    h.close()


@pytest.mark.parametrize("ref", range(0, 6))
def test_counts_and_euler(h5, ref):
    """P1: F = 20*4^r, V = 10*4^r + 2, E = 30*4^r, V - E + F = 2."""
    L = h5.level(ref)
    F = L["faces"].shape[0]
    V = L["verts"].shape[0]
    edges = {tuple(sorted((int(f[j]), int(f[(j + 1) % 3])))) for f in L["faces"] for j in range(3)}
    assert F == 20 * 4 ** ref
    assert V == 10 * 4 ** ref + 2
    assert len(edges) == 30 * 4 ** ref
    assert V - len(edges) + F == 2


@pytest.mark.parametrize("ref", range(0, 6))
def test_neighbours_share_edges_and_are_symmetric(h5, ref):
    """P1: each slot j names the cell across edge (v_j, v_{j+1}); relation symmetric."""
    L = h5.level(ref)
    f, N = L["faces"], L["nbr"]
    n = f.shape[0]
    for c in range(n):
        assert len(set(N[c])) == 3 and c not in N[c]
        for j in range(3):
            o = N[c, j]
            a, b = f[c, j], f[c, (j + 1) % 3]
            # the neighbour holds the same edge in reverse orientation
            jo = [i for i in range(3) if N[o, i] == c]
            assert len(jo) == 1
            assert (f[o, jo[0]], f[o, (jo[0] + 1) % 3]) == (b, a)


def test_vertices_on_unit_sphere(h5):
    for ref in range(6):
        v = h5.level(ref)["verts"]
        assert np.max(np.abs(np.linalg.norm(v, axis=1) - 1.0)) < 4e-16


def test_ref0_closed_forms(h5):
    """P2: regular icosahedron in the unit sphere: edge = 1/sin(2 pi/5),
    area = sqrt(3)/4 edge^2, |centroid| = inradius, centroid distance
    2 |cen| sin(theta/2) with cos(theta) = sqrt(5)/3, len/cd = 3/phi."""
    L = h5.level(0)
    edge = 1.0 / math.sin(2 * math.pi / 5)
    area = math.sqrt(3) / 4 * edge ** 2
    phi = (1 + math.sqrt(5)) / 2
    inr = math.sqrt((7 + 3 * math.sqrt(5)) / 6) / math.sqrt((5 + math.sqrt(5)) / 2)  # r_in/r_circ of icosahedron
    theta = math.acos(math.sqrt(5) / 3)
    cd = 2 * inr * math.sin(theta / 2)
    assert np.allclose(L["len"], edge, rtol=1e-14, atol=0)
    assert np.allclose(L["area"], area, rtol=1e-14, atol=0)
    assert np.allclose(L["cd"], cd, rtol=1e-13, atol=0)
    assert np.allclose(L["len"] / L["cd"], 3 / phi, rtol=1e-13, atol=0)
    # cross-check the published constants quoted in the survey
    assert abs(edge - 1.0514622242) < 1e-10 and abs(area - 0.4787270692) < 1e-10
    assert abs(inr - 0.7946544723) < 1e-10 and abs(cd - 0.5671005389) < 1e-10


def test_ref0_faces_golden(h5):
    """Base face table (orientation rule of reading R1) vs committed fixture."""
    with open(os.path.join(GOLDEN, "ico_ref0_faces.json")) as fh:
        g = json.load(fh)
    assert h5.level(0)["faces"].tolist() == g["faces"]


def test_faces_counter_clockwise_from_outside(h5):
    for ref in range(6):
        L = h5.level(ref)
        v, f = L["verts"], L["faces"]
        a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
        assert np.all(np.einsum("ij,ij->i", np.cross(b - a, c - a), a + b + c) > 0)


@pytest.mark.parametrize("ref", range(1, 6))
def test_child_ordering(h5, ref):
    """Children of p are 4p+k: child k<3 holds parent vertex k, child 3 the
    three edge midpoints; midpoints are normalised (va+vb)/2 (reading R1/R8)."""
    P, C = h5.level(ref - 1), h5.level(ref)
    pv, pf = P["verts"], P["faces"]
    cv, cf = C["verts"], C["faces"]
    assert np.array_equal(cv[: pv.shape[0]], pv)
    for p in range(pf.shape[0]):
        a, b, c = (pv[i] for i in pf[p])
        mids = []
        for x, y in ((a, b), (b, c), (c, a)):
            m = (x + y) * 0.5
            mids.append(m / np.linalg.norm(m))
        mab, mbc, mca = mids
        expect = [(a, mab, mca), (mab, b, mbc), (mca, mbc, c), (mab, mbc, mca)]
        for k in range(4):
            got = cv[cf[4 * p + k]]
            assert np.allclose(got, np.array(expect[k]), rtol=0, atol=1e-15)


def test_area_heron_and_total(h5):
    """Area against Heron's formula from the edge lengths; the total area of
    the chordal polyhedron increases towards 4 pi under refinement."""
    prev = 0.0
    for ref in range(6):
        L = h5.level(ref)
        a, b, c = L["len"][:, 0], L["len"][:, 1], L["len"][:, 2]
        s = (a + b + c) / 2
        heron = np.sqrt(s * (s - a) * (s - b) * (s - c))
        assert np.allclose(L["area"], heron, rtol=1e-10, atol=0)
        tot = L["area"].sum()
        assert prev < tot < 4 * math.pi
        prev = tot
    assert 4 * math.pi - prev < 4 * math.pi * 1e-3


def test_edge_lengths_match_vertices_and_symmetry(h5):
    """len_j = |v_{j+1} - v_j| and the centroid distances are bitwise
    symmetric across each shared edge (the difference flips sign exactly)."""
    for ref in range(4):
        L = h5.level(ref)
        v, f, N = L["verts"], L["faces"], L["nbr"]
        for j in range(3):
            d = v[f[:, (j + 1) % 3]] - v[f[:, j]]
            assert np.allclose(L["len"][:, j], np.linalg.norm(d, axis=1), rtol=1e-15, atol=0)
        for c in range(f.shape[0]):
            for j in range(3):
                o = N[c, j]
                jo = list(N[o]).index(c)
                assert L["len"][c, j] == L["len"][o, jo]
                assert L["cd"][c, j] == L["cd"][o, jo]


def test_ref0_faces_lexicographic(h5):
    """Reading R1: faces are the adjacent triples i<j<k in lexicographic order,
    each stored as (i,j,k) or (i,k,j)."""
    f = h5.level(0)["faces"]
    keys = [tuple(sorted(t)) for t in f.tolist()]
    assert all(t[0] == s[0] for t, s in zip(f.tolist(), keys))
    assert keys == sorted(keys) and len(set(keys)) == 20
