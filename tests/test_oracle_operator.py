"""Pins P3/P4 of the oracle's coefficients, assembly and apply (readings R3-R5).

H^ = M3 + w_c^2 (Dh Minv Dh^T + Dz Minv Dz^T / (1+w_N^2)) (Eq. 8)
with DG0 pressure and lumped two-point couplings is diag(vol) plus a weighted
graph Laplacian; the checks below follow from that structure alone.
"""
import math

import numpy as np
import pytest
import scipy.linalg

import hmg_inputs as hi
import oracle
from dense import helmholtz_sparse

EPS = np.finfo(np.float64).eps


def _back_slot(nbr, c, j):
    o = nbr[c, j]
    return o, list(nbr[o]).index(c)


def test_symmetry_bitwise_and_m_matrix(c0_oracle):
    """P4: A_ij == A_ji bitwise; D > 0, off-diagonals <= 0 (M-matrix signs)."""
    cfg, h, lam, b = c0_oracle
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        L = h.level(ref)
        nbr, H = L["nbr"], L["H"]
        n = nbr.shape[0]
        for c in range(n):
            for j in range(3):
                o, jo = _back_slot(nbr, c, j)
                assert np.array_equal(H[j, :, c], H[jo, :, o])
        assert np.all(L["D"] > 0)
        assert np.all(H < 0) and np.all(L["U"][:-1] < 0) and np.all(L["U"][-1] == 0)
        A = helmholtz_sparse(L, cfg.nz)
        assert (A != A.T).nnz == 0


@pytest.mark.parametrize("cfgname", ["C0", "C1"])
def test_row_sum_identity(cfgname):
    """P4 / reading R10: H^ 1 = vol (the couplings form a Laplacian; no lateral
    boundary on the sphere and u.n = 0 at top and bottom)."""
    cfg = hi.CONFIGS[cfgname]
    if cfgname == "C1":
        cfg = hi.Config("C1s", 3, 2, 16, 0.01, 1e-4)
    lam, _ = hi.make_inputs(cfg)
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam)
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        L = h.level(ref)
        ones = np.ones(h.shape(ref))
        y = h.apply(ref, ones)
        vol = L["area"] * (cfg.thickness / cfg.nz)
        assert np.max(np.abs(y - vol[None, :])) <= 8 * EPS * L["D"].max()
    h.close()


def test_apply_equals_sparse_matvec(c0_oracle):
    """Loop-form apply (O5) equals the assembled-matrix product."""
    cfg, h, lam, b = c0_oracle
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        L = h.level(ref)
        x = hi.uniform_vector(h.shape(ref), 7 + ref)
        y = h.apply(ref, x)
        A = helmholtz_sparse(L, cfg.nz)
        ref_y = (A @ x.reshape(-1)).reshape(x.shape)
        assert np.max(np.abs(y - ref_y)) <= 1e-14 * np.max(np.abs(ref_y))


def test_spd_and_spectrum_bounds(c0_oracle):
    """P4: dense eigvalsh on C0: SPD, lambda_min >= min vol, lambda_max <= 2 max D."""
    cfg, h, lam, b = c0_oracle
    L = h.level(cfg.fine_ref)
    A = helmholtz_sparse(L, cfg.nz).toarray()
    ev = np.linalg.eigvalsh(A)
    vol = L["area"] * (cfg.thickness / cfg.nz)
    assert ev[0] >= vol.min() * (1 - 1e-10)
    assert ev[-1] <= 2 * L["D"].max()


def test_coefficient_coarsening(c0_oracle):
    """Reading R3: coarse lam = mean of the four children in the same layer;
    the mean over the sphere is preserved."""
    cfg, h, lam, b = c0_oracle
    for ref in range(cfg.fine_ref, cfg.coarsest_ref, -1):
        f, c = h.level(ref)["lam"], h.level(ref - 1)["lam"]
        assert np.allclose(c, f.reshape(cfg.nz, -1, 4).mean(axis=2), rtol=1e-15, atol=0)
        assert abs(c.mean() - f.mean()) < 1e-14


def test_couplings_from_geometry(c0_oracle):
    """Reading R4 in matrix form: off-diagonal entries are minus the
    two-point fluxes w2*|edge|*dz*lamf/cd (horizontal) and w2*area*lamf/dz
    (vertical), lamf the arithmetic face mean."""
    cfg, h, lam, b = c0_oracle
    dz = cfg.thickness / cfg.nz
    L = h.level(cfg.fine_ref)
    nbr = L["nbr"]
    lamf_h = 0.5 * (L["lam"][:, :, None] + L["lam"][:, nbr])        # [nz][n][3]
    Hc = cfg.w2 * L["len"][None] * dz * lamf_h / L["cd"][None]
    assert np.allclose(-L["H"].transpose(1, 2, 0), Hc, rtol=4 * EPS, atol=0)
    lamf_v = 0.5 * (L["lam"][:-1] + L["lam"][1:])
    assert np.allclose(-L["U"][:-1], cfg.w2 * L["area"][None] * lamf_v / dz, rtol=4 * EPS, atol=0)


def _dodecahedron_spectrum():
    s5 = math.sqrt(5)
    return np.sort([3.0] + [s5] * 3 + [1.0] * 5 + [0.0] * 4 + [-2.0] * 4 + [-s5] * 3)


def test_ref0_closed_form_spectrum():
    """P3: with lam = 1 at ref 0 the horizontal graph is the dodecahedron
    graph and H^ = T - Hc*A_dodec with T = (vol+3Hc)I + V*L_path; cosine
    modes (x) graph eigenvectors are eigenvectors of H^ and T with closed-form
    eigenvalues.  Geometry values are the closed forms of test_ref0_closed_forms."""
    nz, t, w2 = 8, 0.01, 1e-4
    h = oracle.Hierarchy(0, 0, nz, t, w2, np.ones((nz, 20)))
    L = h.level(0)
    A = np.zeros((20, 20))
    for c in range(20):
        for j in range(3):
            A[c, L["nbr"][c, j]] = 1.0
    ev, evec = np.linalg.eigh(A)
    assert np.allclose(ev, _dodecahedron_spectrum(), atol=1e-13)
    edge = 1.0 / math.sin(2 * math.pi / 5)
    area = math.sqrt(3) / 4 * edge ** 2
    phi = (1 + math.sqrt(5)) / 2
    dz = t / nz
    vol = area * dz
    Hc = w2 * dz * (3 / phi)            # w2 * len * dz / cd with len/cd = 3/phi
    V = w2 * area / dz
    k = np.arange(nz)
    for m in range(nz):
        cosm = np.cos(math.pi * m * (k + 0.5) / nz)
        tau = vol + 3 * Hc + V * (2 - 2 * math.cos(math.pi * m / nz))
        for jj in (0, 5, 19):
            v = cosm[:, None] * evec[:, jj][None, :]
            lam_ = tau - Hc * ev[jj]
            assert np.allclose(h.apply(0, v), lam_ * v, rtol=0, atol=1e-12 * lam_)
            # T^{-1} via the Thomas solve: one undamped zero-guess sweep with the
            # horizontal bands removed from H^ is exactly T^{-1}
            u1 = h.sweep(0, v, None, 1, 1.0)         # u = T^{-1} v  (omega = 1)
            assert np.allclose(u1, v / tau, rtol=0, atol=1e-12 / tau)
            # s damped sweeps from zero: u_s = (1 - (1 - w lam/tau)^s)/lam * v
            for s in (2, 5):
                us = h.sweep(0, v, None, s, 0.8)
                expect = (1 - (1 - 0.8 * lam_ / tau) ** s) / lam_
                assert np.allclose(us, expect * v, rtol=0, atol=1e-11 * abs(expect))
    h.close()


@pytest.mark.parametrize("omega_n", [0.0, 1.0])
def test_diagonal_reforms_from_couplings_bitwise(omega_n):
    """The identity the streamed GPU kernels rely on (DESIGN 7.7): with the
    stored U_k = -V_up,k and H_j = -(coupling j), the assembled diagonal is,
    bit for bit, ((((vol - U_{k-1}) - U_k) - H0) - H1) - H2 with vol = area * dz
    (the k > 0 / k < nz - 1 terms dropped at the ends): V_dn at layer k is the
    same expression as V_up at layer k - 1, and x + (-y) is x - y in IEEE
    arithmetic.  Also with buoyancy (reading R24), on every level."""
    cfg = hi.Config("dref", 3, 0, 9, 0.01, 1e-3)
    lam, _ = hi.make_inputs(cfg)
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, omega_n=omega_n)
    dz = cfg.thickness / cfg.nz
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        L = h.level(ref)
        U, H = L["U"], L["H"]
        vol = L["area"] * dz
        for k in range(cfg.nz):
            d = vol.copy()
            if k > 0:
                d = d - U[k - 1]
            if k < cfg.nz - 1:
                d = d - U[k]
            d = d - H[0, k]
            d = d - H[1, k]
            d = d - H[2, k]
            assert np.array_equal(d, L["D"][k]), f"ref {ref} layer {k}"
    h.close()
