"""Seeded synthetic inputs and workload shapes (shared by oracle tests and the CUDA path).

This module holds NO method arithmetic: only the configuration table of
BASELINE.json (C0-C4) and the seeded random draws of
DESIGN.md reading R11 (numpy PCG64, ``default_rng(seed)``; lam drawn first,
uniform [0.9, 1.1]; then the right-hand side, uniform (-1, 1); for C1 then x
and u the same way).  All arrays are fp64, layer-major ``[nz][n]``.

The paper's own workload (81,920 cells = ref 6 x 64 layers) is a
synthetic gravity-wave step whose right-hand side it does not print; no public
dataset is involved.  White-noise right-hand sides excite every mode.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def ncells(ref: int) -> int:
    """Icosahedral cells at refinement ``ref``: 20 * 4**ref."""
    return 20 * 4 ** ref


@dataclass(frozen=True)
class Config:
    name: str
    fine_ref: int
    coarsest_ref: int
    nz: int
    thickness: float
    w2: float
    seed: int = 0

    @property
    def n(self) -> int:
        return ncells(self.fine_ref)

    @property
    def ndofs(self) -> int:
        return self.n * self.nz


# BASELINE.json configs; C2 carries the three anisotropy settings.
CONFIGS = {
    "C0": Config("C0", 2, 0, 8, 0.01, 1e-4),
    "C1": Config("C1", 5, 4, 64, 0.01, 1e-4),
    "C2a": Config("C2a", 7, 0, 64, 0.01, 1e-4),
    "C2b": Config("C2b", 7, 0, 64, 0.001, 1e-5),
    "C2c": Config("C2c", 7, 0, 64, 1e-4, 1e-6),
    "C4": Config("C4", 8, 0, 128, 0.001, 1e-5),
}


def make_inputs(cfg: Config, seed: int | None = None, extra: int = 0):
    """Return (lam, b, *extras): lam ~ U[0.9,1.1], b ~ U(-1,1), then ``extra``
    more U(-1,1) vectors (C1 uses 2: x, u).  Shapes [nz][n], fp64."""
    rng = np.random.default_rng(cfg.seed if seed is None else seed)
    shape = (cfg.nz, cfg.n)
    lam = rng.uniform(0.9, 1.1, shape)
    out = [lam, rng.uniform(-1.0, 1.0, shape)]
    for _ in range(extra):
        out.append(rng.uniform(-1.0, 1.0, shape))
    return tuple(out)


def uniform_vector(shape, seed: int) -> np.ndarray:
    """An extra seeded U(-1,1) vector (test vectors, not part of a config)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, shape)


# ---- NEXT-3 core inputs: batched banded column matrices ----------------------
# The NLO column operator: m = 6 nz rows, kl = ku = 13.  Its
# entries depend on the BDFM1 velocity mass the paper does not print (DESIGN.md
# R21), so the banded solver is driven by seeded random band matrices of that
# shape: entries U(-1, 1) inside the band (not diagonally dominant, so partial
# pivoting really interchanges rows), zero outside and in the fill-in rows.
NLO_CONFIGS = {
    # name: (fine ref, layers) -> ncol = 20 * 4**ref columns, m = 6 * layers rows
    "N0": (2, 8),     # tiny: 320 columns x 48 rows
    "N1": (4, 64),    # the paper's NLO mesh (5,120 cells x 64 layers): m = 384
    "N2": (6, 64),    # a B200-sized NLO problem: 81,920 columns x 384 rows = 31.5M DG1 dofs
}


def band_lu_storage(ncol: int, m: int, kl: int, ku: int, seed: int, ld: int | None = None) -> np.ndarray:
    """Seeded band matrices in the batched LAPACK LU layout [m][2kl+ku+1][ld]
    (A(i, j) at [j][kl+ku+i-j][c]; columns c >= ncol and entries outside the
    band zero)."""
    ld = ncol if ld is None else ld
    ldab = 2 * kl + ku + 1
    rng = np.random.default_rng(seed)
    ab = np.zeros((m, ldab, ld))
    ab[:, kl:, :ncol] = rng.uniform(-1.0, 1.0, (m, kl + ku + 1, ncol))
    r = np.arange(kl, ldab)
    j = np.arange(m)
    i = j[:, None] + r[None, :] - (kl + ku)          # matrix row of each band slot
    ab[:, kl:, :][(i < 0) | (i >= m)] = 0.0
    return ab


def band_row_storage(ncol: int, m: int, kl: int, ku: int, seed: int, ld: int | None = None) -> np.ndarray:
    """Seeded band matrices in the paper's row-wise layout [m][kl+ku+1][ld]
    (A(i, j) at [i][kl+j-i][c]; slots with j outside [0, m) zero)."""
    ld = ncol if ld is None else ld
    bw = kl + ku + 1
    rng = np.random.default_rng(seed)
    ar = np.zeros((m, bw, ld))
    ar[:, :, :ncol] = rng.uniform(-1.0, 1.0, (m, bw, ncol))
    i = np.arange(m)
    j = i[:, None] + np.arange(bw)[None, :] - kl
    ar[(j < 0) | (j >= m)] = 0.0
    return ar
