"""Pins of the oracle's NEXT-4 mixed velocity-pressure system (readings R15-R20).

A = [[M2, -omega D^T], [omega D, M3]] (Eq. 5, omega_N = 0,
omega = sqrt(w2)), lowest order: RT0 horizontal fluxes, P1-in-the-vertical
fluxes, DG0 pressure.  What fixes each part independently of the oracle's own
formulas:
  * the edge table is a pairing of the mesh's neighbour slots;
  * D is the discrete divergence: net outward flux, so the sum over all cells
    of D U vanishes (every face shared by two cells, no flux through top and
    bottom), and D^T is its adjoint;
  * the lumped Schur complement M3 + omega^2 D L^-1 D^T equals BASELINE's
    operator H^ (the hot path, pinned in test_oracle_operator.py);
  * the RT0 Gram matrices reproduce constant vector fields exactly
    (u0 = sum_j F_j psi_j with F_j the outward fluxes of u0 through the edges,
    so F^T G F = |T| |u0|^2);
  * the P1 vertical mass integrates the hat functions exactly (row sums);
  * GMRES minimises the residual over its Krylov space (checked against an
    independent least-squares solve), and its reported residual is the true one.
"""
import numpy as np
import pytest

import hmg_inputs as hi
import oracle

EPS = np.finfo(np.float64).eps


@pytest.fixture(scope="module")
def c0(c0_oracle):
    cfg, h, lam, b = c0_oracle
    return cfg, h, lam, h.level(cfg.fine_ref)


def _rand(shape, seed):
    return hi.uniform_vector(shape, seed)


def test_edge_table_pairs_neighbour_slots(c0):
    cfg, h, lam, L = c0
    ec, es, ce = h.mixed_edges()
    nbr = L["nbr"]
    n = nbr.shape[0]
    assert ec.shape[0] == 3 * n // 2
    assert np.all(ec[:, 0] < ec[:, 1])
    assert np.all(nbr[ec[:, 0], es[:, 0]] == ec[:, 1])
    assert np.all(nbr[ec[:, 1], es[:, 1]] == ec[:, 0])
    for e, (a, b) in enumerate(ec):
        assert ce[a, es[e, 0]] == e and ce[b, es[e, 1]] == e
    assert np.all(np.sort(ce.ravel()) == np.repeat(np.arange(ec.shape[0]), 2))
    # reading R16: ordered by lower cell, then its slot
    key = ec[:, 0].astype(np.int64) * 3 + es[:, 0]
    assert np.all(np.diff(key) > 0)


def test_divergence_theorem_and_adjoint(c0):
    cfg, h, lam, L = c0
    ne, N = h.mixed_sizes()
    nz, n = cfg.nz, L["nbr"].shape[0]
    Uh, Uz, P = _rand((nz, ne), 1), _rand((nz - 1, n), 2), _rand((nz, n), 3)
    d = h.mixed_part("div", Uh, Uz)
    assert abs(d.sum()) <= 64 * EPS * np.abs(Uh).sum()
    th, tz = h.mixed_part("divT", P=P)
    lhs = np.dot(d.ravel(), P.ravel())
    rhs = np.dot(th.ravel(), Uh.ravel()) + np.dot(tz.ravel(), Uz.ravel())
    assert abs(lhs - rhs) <= 1e-13 * (np.abs(d).sum() + np.abs(th).sum())
    # constant pressure has no gradient; top/bottom carry no flux
    th1, tz1 = h.mixed_part("divT", P=np.ones((nz, n)))
    assert np.all(th1 == 0) and np.all(tz1 == 0)


def test_lumped_schur_complement_is_the_helmholtz_operator(c0):
    """M3 P + omega^2 D (L^-1 (D^T P)) == H^ P (reading R19): the mixed system's
    lumped Schur complement is BASELINE's operator, to rounding."""
    cfg, h, lam, L = c0
    nz, n = cfg.nz, L["nbr"].shape[0]
    for seed in (4, 5):
        P = _rand((nz, n), seed)
        th, tz = h.mixed_part("divT", P=P)
        lh, lz = h.mixed_part("lumped_inv", th, tz)
        s = (L["area"] * h.thickness / nz)[None, :] * P + cfg.w2 * h.mixed_part("div", lh, lz)
        ref = h.apply(cfg.fine_ref, P)
        assert np.max(np.abs(s - ref)) <= 64 * EPS * np.max(np.abs(ref))


def test_rt0_gram_reproduces_constant_fields(c0):
    cfg, h, lam, L = c0
    G = h.mixed_part("gram")
    V, F = L["verts"], L["faces"]
    rng = np.random.default_rng(7)
    for c in range(F.shape[0]):
        Pv = V[F[c]]
        nrm = np.cross(Pv[1] - Pv[0], Pv[2] - Pv[0])
        area = 0.5 * np.linalg.norm(nrm)
        nhat = nrm / np.linalg.norm(nrm)
        assert np.dot(nhat, Pv.mean(axis=0)) > 0            # counter-clockwise from outside
        u0 = rng.standard_normal(3)
        u0 = u0 - np.dot(u0, nhat) * nhat                    # tangent to the cell's plane
        flux = np.array([np.dot(u0, np.cross(Pv[(j + 1) % 3] - Pv[j], nhat)) for j in range(3)])
        assert abs(flux.sum()) <= 1e-14 * np.abs(flux).sum()   # constant field is divergence-free
        assert np.allclose(G[c], G[c].T, rtol=0, atol=1e-15 * np.abs(G[c]).max())
        assert flux @ G[c] @ flux == pytest.approx(area * np.dot(u0, u0), rel=1e-12)
        assert np.all(np.linalg.eigvalsh(G[c]) > 0)


def test_vertical_mass_integrates_hats(c0):
    """Row sums of the P1 vertical mass: int hat_i / (area lam) over the two
    layers of interface i = (dz/2) (1/(area lam_lo) + 1/(area lam_hi)); interfaces
    next to the top or bottom lose the absent neighbour's dz/6 term."""
    cfg, h, lam, L = c0
    ne, _ = h.mixed_sizes()
    nz, n = cfg.nz, L["nbr"].shape[0]
    dz = h.thickness / nz
    _, yz = h.mixed_part("mass", np.zeros((nz, ne)), np.ones((nz - 1, n)))
    A = L["area"][None, :]
    lo, hi_ = A * L["lam"][:-1], A * L["lam"][1:]
    want = (dz / 2) * (1 / lo + 1 / hi_)
    want[0] -= (dz / 6) / lo[0]
    want[-1] -= (dz / 6) / hi_[-1]
    assert np.allclose(yz, want, rtol=1e-14, atol=0)


def test_mass_symmetric_positive_definite(c0):
    cfg, h, lam, L = c0
    ne, _ = h.mixed_sizes()
    nz, n = cfg.nz, L["nbr"].shape[0]
    x = (_rand((nz, ne), 11), _rand((nz - 1, n), 12))
    y = (_rand((nz, ne), 13), _rand((nz - 1, n), 14))
    Mx, My = h.mixed_part("mass", *x), h.mixed_part("mass", *y)
    a = sum(np.dot(p.ravel(), q.ravel()) for p, q in zip(Mx, y))
    b = sum(np.dot(p.ravel(), q.ravel()) for p, q in zip(x, My))
    assert abs(a - b) <= 1e-13 * abs(a)
    assert sum(np.dot(p.ravel(), q.ravel()) for p, q in zip(Mx, x)) > 0


def test_apply_block_structure(c0):
    cfg, h, lam, L = c0
    ne, N = h.mixed_sizes()
    nz, n = cfg.nz, L["nbr"].shape[0]
    x = _rand(N, 21)
    Uh, Uz, P = h.mixed_split(x)
    y = h.mixed_apply(x)
    yh, yz, yp = h.mixed_split(y)
    om = np.sqrt(cfg.w2)
    mh, mz = h.mixed_part("mass", Uh, Uz)
    th, tz = h.mixed_part("divT", P=P)
    vol = (L["area"] * h.thickness / nz)[None, :]
    assert np.allclose(yh, mh - om * th, rtol=0, atol=8 * EPS * np.abs(mh).max())
    assert np.allclose(yz, mz - om * tz, rtol=0, atol=8 * EPS * np.abs(mz).max())
    assert np.allclose(yp, om * h.mixed_part("div", Uh, Uz) + vol * P, rtol=0, atol=8 * EPS * np.abs(yp).max())


def _tiny():
    cfg = hi.Config("tiny", 0, 0, 2, 0.01, 1e-4)
    lam, b = hi.make_inputs(cfg, seed=3)
    return cfg, oracle.Hierarchy(0, 0, 2, 0.01, 1e-4, lam)


def _dense(f, N):
    return np.stack([f(np.eye(N)[i]) for i in range(N)], axis=1)


def test_gmres_minimises_the_residual_over_the_krylov_space():
    """Unpreconditioned GMRES on a 120-unknown system: after j steps the
    residual is min ||F - A x|| over x in K_j(A, F) (an independent dense
    least-squares solve); the reported relres is the true residual."""
    cfg, h = _tiny()
    ne, N = h.mixed_sizes()
    A = _dense(h.mixed_apply, N)
    F = hi.uniform_vector(N, 31)
    x, it, rel, hist, st = h.mixed_gmres(F, rtol=1e-10, restart=40, maxit=40, precond="none")
    assert it == 40
    assert np.linalg.norm(F - A @ x) / np.linalg.norm(F) == pytest.approx(rel, rel=1e-8)
    K = np.empty((N, 0))
    v = F / np.linalg.norm(F)
    for j in range(1, 13):
        K = np.column_stack([K, v])
        Q, _ = np.linalg.qr(K)
        K = Q
        y, *_ = np.linalg.lstsq(A @ K, F, rcond=None)
        best = np.linalg.norm(F - A @ K @ y) / np.linalg.norm(F)
        assert hist[j] == pytest.approx(best, rel=1e-8, abs=1e-14)
        v = A @ K[:, -1]
    h.close()


def test_gmres_right_preconditioned_minimises_over_preconditioned_space():
    """Right preconditioning: x_j = M^-1 t with t in K_j(A M^-1, F) minimising
    ||F - A M^-1 t||; M^-1 = the Schur-complement preconditioner (dense)."""
    cfg, h = _tiny()
    ne, N = h.mixed_sizes()
    A = _dense(h.mixed_apply, N)
    Minv = _dense(lambda f: h.mixed_precond(f), N)
    B = A @ Minv
    F = hi.uniform_vector(N, 32)
    x, it, rel, hist, st = h.mixed_gmres(F, rtol=1e-12, restart=30, maxit=60)
    assert st == 0
    K = np.empty((N, 0))
    v = F / np.linalg.norm(F)
    for j in range(1, min(it, 8) + 1):
        K, _ = np.linalg.qr(np.column_stack([K, v]))
        y, *_ = np.linalg.lstsq(B @ K, F, rcond=None)
        assert hist[j] == pytest.approx(np.linalg.norm(F - B @ K @ y) / np.linalg.norm(F), rel=1e-7, abs=1e-14)
        v = B @ K[:, -1]
    assert np.linalg.norm(F - A @ x) / np.linalg.norm(F) == pytest.approx(rel, rel=1e-6)
    h.close()


def test_schur_preconditioner_factorisation(c0):
    """Eq. 6 with the lumped mass: M^-1 = [[1, w L^-1 D^T], [0, 1]] diag(L^-1, V)
    [[1, 0], [-w D L^-1, 1]], V = the V-cycle (dense on the pressure space)."""
    cfg, h = _tiny()
    ne, N = h.mixed_sizes()
    nz, n = 2, 20
    om = np.sqrt(1e-4)
    nu = nz * ne + (nz - 1) * n

    def split_u(u):
        return u[: nz * ne].reshape(nz, ne), u[nz * ne:].reshape(nz - 1, n)

    Linv = _dense(lambda u: np.concatenate([a.ravel() for a in h.mixed_part("lumped_inv", *split_u(u))]), nu)
    D = _dense(lambda u: h.mixed_part("div", *split_u(u)).ravel(), nu)
    Vc = _dense(lambda p: h.vcycle(p.reshape(nz, n)).ravel(), nz * n)
    np_ = nz * n
    Lo = np.block([[np.eye(nu), np.zeros((nu, np_))], [-om * D @ Linv, np.eye(np_)]])
    Mid = np.block([[Linv, np.zeros((nu, np_))], [np.zeros((np_, nu)), Vc]])
    Up = np.block([[np.eye(nu), om * Linv @ D.T], [np.zeros((np_, nu)), np.eye(np_)]])
    f = hi.uniform_vector(N, 41)
    assert np.allclose(h.mixed_precond(f), Up @ Mid @ Lo @ f, rtol=0, atol=1e-12 * np.abs(Up @ Mid @ Lo @ f).max())
    h.close()


def test_gmres_c0_converges_like_the_paper(c0):
    """C0 with the Schur + V(2,2) preconditioner reaches 1e-5 in ~10 GMRES
    iterations (the paper's LO: 10 outer iterations, P:899-905 -- context
    only, different mesh and workload) and the returned x meets the tolerance."""
    cfg, h, lam, L = c0
    ne, N = h.mixed_sizes()
    F = hi.uniform_vector(N, 51)
    x, it, rel, hist, st = h.mixed_gmres(F, rtol=1e-5)
    assert st == 0 and 3 <= it <= 30
    r = F - h.mixed_apply(x)
    assert np.linalg.norm(r) / np.linalg.norm(F) == pytest.approx(rel, rel=1e-10)
    assert rel <= 1e-5
    _, it0, _, _, st0 = h.mixed_gmres(F, rtol=1e-5, maxit=60, precond="none")
    assert st0 != 0 or it0 > 3 * it


@pytest.mark.parametrize("gs_passes", [1, 2], ids=["CGS", "CGS2"])
def test_gmres_both_gram_schmidt_variants_minimise(gs_passes):
    """On a small, well-conditioned case one and two Gram-Schmidt passes both
    give the least-squares-minimal residual history (checked against an
    independent dense solve): the variant only matters once orthogonality is
    lost (next test)."""
    cfg, h = _tiny()
    ne, N = h.mixed_sizes()
    A = _dense(h.mixed_apply, N)
    Minv = _dense(lambda f: h.mixed_precond(f), N)
    B = A @ Minv
    F = hi.uniform_vector(N, 33)
    x, it, rel, hist, st = h.mixed_gmres(F, rtol=1e-10, restart=30, maxit=60, gs_passes=gs_passes)
    assert st == 0
    K = np.empty((N, 0))
    v = F / np.linalg.norm(F)
    for j in range(1, min(it, 6) + 1):
        K, _ = np.linalg.qr(np.column_stack([K, v]))
        y, *_ = np.linalg.lstsq(B @ K, F, rcond=None)
        assert hist[j] == pytest.approx(np.linalg.norm(F - B @ K @ y) / np.linalg.norm(F), rel=1e-7, abs=1e-14)
        v = B @ K[:, -1]
    h.close()


def test_gmres_cgs_loses_orthogonality_cgs2_keeps_it():
    """Why reading R20 departs from PETSc's default (one classical Gram-Schmidt
    pass, most likely what the paper's GMRES(30) ran): on the
    anisotropic problems one pass loses the Arnoldi basis' orthogonality --
    the loss of CGS grows like eps * kappa^2 of the Krylov matrix -- while two
    passes keep it at the rounding level ("twice is enough": ||I - V^T V|| =
    O(eps), independent of kappa).  Measured on the oracle alone, no GPU
    involved: C2c's anisotropy at ref 4 x 64 and C2b's at ref 3 x 16; at ref 5 x
    64 (C2b) CGS's basis is ~1e-1 from orthogonal (13 s, not run here)."""
    for name, ref, nz, loss_cgs in (("C2c", 4, 64, 1e-3), ("C2b", 3, 16, 1e-7)):
        c = hi.CONFIGS[name]
        cfg = hi.Config("orth", ref, 0, nz, c.thickness, c.w2)
        lam, _ = hi.make_inputs(cfg)
        h = oracle.Hierarchy(ref, 0, nz, cfg.thickness, cfg.w2, lam)
        _, N = h.mixed_sizes()
        F = hi.uniform_vector(N, 65)
        _, it1, rel1, _, st1, orth1 = h.mixed_gmres(F, rtol=1e-5, gs_passes=1, orth=True)
        _, it2, rel2, _, st2, orth2 = h.mixed_gmres(F, rtol=1e-5, gs_passes=2, orth=True)
        assert st1 == 0 and st2 == 0
        assert orth2 <= 1000 * EPS, (name, orth2)
        assert orth1 >= loss_cgs, (name, orth1)
        h.close()


@pytest.mark.parametrize("omega_n", [0.5, 1.0, 3.0])
def test_buoyancy_scales_the_vertical_terms(c0, omega_n):
    """Reading R24 (Eq. 5; Eq. 8): with buoyancy eliminated,
    M~2 = M2h (+) (1 + omega_N^2) M2z, so the vertical velocity mass is scaled by
    1 + omega_N^2 -- exactly, the horizontal one untouched -- and the pressure
    operator's vertical couplings are divided by it (exactly: the same quotient
    divided once more), the horizontal ones and the pressure mass untouched."""
    cfg, h0, lam, L0 = c0
    sn = 1.0 + omega_n * omega_n
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, omega_n=omega_n)
    for ref in range(cfg.coarsest_ref, cfg.fine_ref + 1):
        A, B = h0.level(ref), h.level(ref)
        assert np.array_equal(B["U"], A["U"] / sn)
        assert np.array_equal(B["H"], A["H"])
        # diagonal: volume + the scaled vertical + the horizontal couplings, in R4's order
        nz, n = cfg.nz, A["area"].shape[0]
        vol = A["area"] * (cfg.thickness / nz)
        vup = -B["U"]
        d = np.tile(vol, (nz, 1))
        d[1:] = d[1:] + vup[:-1]
        d[:-1] = d[:-1] + vup[:-1]
        for j in range(3):
            d = d - A["H"][j]
        assert np.array_equal(B["D"], d)
    _, N = h.mixed_sizes()
    x = hi.uniform_vector(N, 91)
    ne = h.mixed_sizes()[0]
    Uh, Uz, P = h.mixed_split(x)
    mh0, mz0 = h0.mixed_part("mass", Uh, Uz)
    mh, mz = h.mixed_part("mass", Uh, Uz)
    assert np.array_equal(mh, mh0) and np.array_equal(mz, mz0 * sn)
    lh0, lz0 = h0.mixed_part("lumped_inv", Uh, Uz)
    lh, lz = h.mixed_part("lumped_inv", Uh, Uz)
    assert np.array_equal(lh, lh0)
    assert np.max(np.abs(lz - lz0 / sn)) <= 2 * EPS * np.max(np.abs(lz0 / sn))
    h.close()


@pytest.mark.parametrize("omega_n", [0.5, 2.0])
def test_buoyant_lumped_schur_complement_is_the_helmholtz_operator(c0, omega_n):
    """With buoyancy the lumped Schur complement M3 + omega^2 D L~^-1 D^T of the
    mixed system is the hierarchy's operator H^(omega_N) of Eq. 8 -- the two
    are computed by different code (mixed system vs band assembly) -- and
    GMRES(30) with the Schur preconditioner converges in a few iterations."""
    cfg, h0, lam, L = c0
    h = oracle.Hierarchy(cfg.fine_ref, cfg.coarsest_ref, cfg.nz, cfg.thickness, cfg.w2, lam, omega_n=omega_n)
    nz, n = cfg.nz, L["nbr"].shape[0]
    for seed in (4, 5):
        P = _rand((nz, n), seed)
        th, tz = h.mixed_part("divT", P=P)
        lh, lz = h.mixed_part("lumped_inv", th, tz)
        s = (L["area"] * h.thickness / nz)[None, :] * P + cfg.w2 * h.mixed_part("div", lh, lz)
        ref = h.apply(cfg.fine_ref, P)
        assert np.max(np.abs(s - ref)) <= 64 * EPS * np.max(np.abs(ref))
    _, N = h.mixed_sizes()
    F = hi.uniform_vector(N, 51)
    x, it, rel, hist, st = h.mixed_gmres(F, rtol=1e-5)
    assert st == 0 and it <= 30 and rel <= 1e-5
    assert np.linalg.norm(F - h.mixed_apply(x)) / np.linalg.norm(F) == pytest.approx(rel, rel=1e-10)
    h.close()
