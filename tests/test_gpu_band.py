"""NEXT-3 core on the GPU == oracle (oracle/band_oracle.c), through the C-ABI
(hmg_band_factor / hmg_band_solve / hmg_band_apply / hmg_p_restrict /
hmg_p_prolong_add).

The kernels run LAPACK's algorithms (dgbtf2 / dgbtrs) and the
paper's banded product in the oracle's operation order with no
contraction, per grid column, so every result is BITWISE the oracle's: the
pivot rows (an integer decision taken in the same precision on both sides),
the LU factors, the solutions, the products and the DG1 <-> DG0 transfers
(P:645-648).  Shapes: the NLO column operator (m = 384, kl = ku = 13,
P:1099-1106) and small / asymmetric / degenerate bands; column counts that
span several tiles with a ragged tail (also past ld, 128-column solve tiles); at full size (81,920 columns,
BASELINE-scale NLO problem N2) sampled columns against the oracle.
"""
import numpy as np
import pytest

import hmg_inputs as hi
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1605_00492_b200 import HmgError, band_apply, band_factor, band_solve, p_prolong_add, p_restrict  # noqa: E402


def ld_of(ncol):
    return (ncol + 31) // 32 * 32


def oracle_column(ab, c):
    """Column c of the batched LU storage [m][ldab][ld] -> oracle layout [ldab][m]."""
    return np.ascontiguousarray(ab[:, :, c].T)


SHAPES = [(384, 13, 13, 100), (384, 13, 13, 200), (48, 13, 13, 70), (13, 13, 13, 33), (5, 13, 13, 40), (1, 13, 13, 32),
          (64, 1, 1, 97), (40, 3, 5, 65), (30, 5, 2, 31), (17, 0, 0, 40), (7, 2, 2, 64)]


@pytest.mark.parametrize("m,kl,ku,ncol", SHAPES)
def test_factor_solve_bitwise(m, kl, ku, ncol):
    ld = ld_of(ncol)
    ab = hi.band_lu_storage(ncol, m, kl, ku, seed=m + 7 * kl + ku, ld=ld)
    b = hi.uniform_vector((m, ld), 3)
    b[:, ncol:] = 0.0
    abd = torch.from_numpy(ab).cuda()
    ipd = torch.zeros((m, ld), dtype=torch.int32, device="cuda")
    assert band_factor(abd, ipd, ncol, kl, ku) == -1
    bd = torch.from_numpy(b).cuda()
    xd = torch.zeros_like(bd)
    band_solve(abd, ipd, bd, xd, ncol, kl, ku)
    lu, ip, x = abd.cpu().numpy(), ipd.cpu().numpy(), xd.cpu().numpy()
    for c in range(ncol):
        lu_o, ip_o, info = oracle.gbtrf(oracle_column(ab, c), kl, ku)
        assert info == 0
        assert np.array_equal(ip[:, c], ip_o), c
        assert np.array_equal(lu[:, :, c].T, lu_o), c
        x_o = oracle.gbtrs(lu_o, kl, ku, ip_o, b[:, c])
        assert np.array_equal(x[:, c], x_o), c
    # padding columns are never written
    assert np.all(x[:, ncol:] == 0.0)


@pytest.mark.parametrize("m,kl,ku,ncol", [(384, 13, 13, 100), (48, 13, 13, 70), (5, 13, 13, 40), (64, 1, 1, 97),
                                          (40, 3, 5, 65), (30, 5, 2, 31), (17, 0, 0, 40)])
def test_apply_bitwise(m, kl, ku, ncol):
    ld = ld_of(ncol)
    ar = hi.band_row_storage(ncol, m, kl, ku, seed=11 + m, ld=ld)
    x = hi.uniform_vector((m, ld), 4)
    y = band_apply(torch.from_numpy(ar).cuda(), torch.from_numpy(x).cuda(),
                   torch.zeros((m, ld), dtype=torch.float64, device="cuda"), ncol, kl, ku).cpu().numpy()
    for c in range(ncol):
        assert np.array_equal(y[:, c], oracle.gbmv(np.ascontiguousarray(ar[:, :, c]), kl, ku, x[:, c])), c
    assert np.all(y[:, ncol:] == 0.0)


def test_singular_column_reported():
    """An identically zero matrix column in grid column 37: LAPACK's info > 0,
    here HMG_ERR_SINGULAR_COLUMN naming column 37; the factorisation is still
    completed and equal to the oracle's (as dgbtrf's)."""
    m, kl, ku, ncol = 48, 13, 13, 70
    ld = ld_of(ncol)
    ab = hi.band_lu_storage(ncol, m, kl, ku, seed=5, ld=ld)
    ab[20, :, 37] = 0.0                       # matrix column 20 of grid column 37
    abd = torch.from_numpy(ab).cuda()
    ipd = torch.zeros((m, ld), dtype=torch.int32, device="cuda")
    with pytest.raises(HmgError, match="singular column: column 37"):
        band_factor(abd, ipd, ncol, kl, ku)
    lu_o, ip_o, info = oracle.gbtrf(oracle_column(ab, 37), kl, ku)
    assert info > 0
    assert np.array_equal(abd.cpu().numpy()[:, :, 37].T, lu_o)
    assert np.array_equal(ipd.cpu().numpy()[:, 37], ip_o)


def test_band_argument_errors():
    t = torch.zeros((8, 40, 32), dtype=torch.float64, device="cuda")
    ip = torch.zeros((8, 32), dtype=torch.int32, device="cuda")
    with pytest.raises(HmgError, match="kl, ku"):
        band_factor(torch.zeros((8, 13, 32), dtype=torch.float64, device="cuda"), ip, 10, 4, 4)
    with pytest.raises(HmgError, match="ld"):
        band_factor(torch.zeros((8, 40, 20), dtype=torch.float64, device="cuda"),
                    torch.zeros((8, 20), dtype=torch.int32, device="cuda"), 20, 13, 13)
    v = torch.zeros((8, 32), dtype=torch.float64, device="cuda")
    with pytest.raises(HmgError, match="x: must not alias b"):
        band_solve(t, ip, v, v, 10, 13, 13)
    with pytest.raises(TypeError):
        band_factor(t, ip.to(torch.int64), 10, 13, 13)


@pytest.mark.parametrize("ncol,nz", [(100, 9), (32, 1), (5, 64)])
def test_p_transfers_bitwise(ncol, nz):
    ld = ld_of(ncol)
    r1 = hi.uniform_vector((6 * nz, ld), 21)
    u0 = hi.uniform_vector((nz, ld), 22)
    u1 = hi.uniform_vector((6 * nz, ld), 23)
    b0 = p_restrict(torch.from_numpy(r1).cuda(), torch.zeros((nz, ld), dtype=torch.float64, device="cuda"),
                    ncol).cpu().numpy()
    # oracle layout: [ncol][6 nz] and [ncol][nz] (column-contiguous)
    b0_o = oracle.p_restrict(np.ascontiguousarray(r1[:, :ncol].T))
    assert np.array_equal(b0[:, :ncol], b0_o.T)
    got = p_prolong_add(torch.from_numpy(u0).cuda(), torch.from_numpy(u1).cuda(), ncol).cpu().numpy()
    ref = oracle.p_prolong_add(np.ascontiguousarray(u0[:, :ncol].T), np.ascontiguousarray(u1[:, :ncol].T))
    assert np.array_equal(got[:, :ncol], ref.T)
    assert np.array_equal(got[:, ncol:], u1[:, ncol:])


@pytest.mark.slow
def test_full_size_nlo_sampled_columns():
    """The B200-sized NLO problem N2 (ref 6 x 64 layers: 81,920 columns x 384
    rows, kl = ku = 13; 10 GB of LU storage) in the launch configuration
    bench.py times: factor and solve, 40 sampled columns (first, last, tile
    boundaries, random) bitwise equal to the oracle."""
    ref, nz = hi.NLO_CONFIGS["N2"]
    ncol, m, kl, ku = 20 * 4 ** ref, 6 * nz, 13, 13
    ld = ld_of(ncol)
    ab = hi.band_lu_storage(ncol, m, kl, ku, seed=2, ld=ld)
    b = hi.uniform_vector((m, ld), 31)
    abd = torch.from_numpy(ab).cuda()
    ipd = torch.zeros((m, ld), dtype=torch.int32, device="cuda")
    band_factor(abd, ipd, ncol, kl, ku)
    xd = band_solve(abd, ipd, torch.from_numpy(b).cuda(), torch.zeros((m, ld), dtype=torch.float64, device="cuda"),
                    ncol, kl, ku)
    rng = np.random.default_rng(0)
    cols = sorted({0, 1, 31, 32, 33, ncol - 1, ncol - 32, *rng.integers(0, ncol, 33).tolist()})
    idx = torch.tensor(cols, device="cuda")
    lu = abd[:, :, idx].cpu().numpy()
    ip = ipd[:, idx].cpu().numpy()
    x = xd[:, idx].cpu().numpy()
    for q, c in enumerate(cols):
        lu_o, ip_o, info = oracle.gbtrf(oracle_column(ab, c), kl, ku)
        assert np.array_equal(ip[:, q], ip_o) and np.array_equal(lu[:, :, q].T, lu_o), c
        assert np.array_equal(x[:, q], oracle.gbtrs(lu_o, kl, ku, ip_o, b[:, c])), c
