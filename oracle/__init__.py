"""CPU oracle for the pressure Helmholtz multigrid path of arXiv:1605.00492.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this package.  The product package ``paper_1605_00492_b200`` never imports it
and shares no code with it; the only module both sides use is ``hmg_inputs``
(seeded random inputs, no method arithmetic).

The arithmetic lives in ``hmg_oracle.c`` (plain C, fp64, ``-O2
-ffp-contract=off``), which follows DESIGN.md's readings R1-R12 (and R15-R20 for the NEXT-4 mixed
system) of the paper
step by step; this module is ctypes marshalling only.  Arrays are numpy fp64,
layer-major ``[nz][n]`` (C order), ``n = 20 * 4**ref`` cells.

Parity status: every function is pinned by tests in ``tests/test_oracle_*.py``
(see DESIGN.md "Oracle pins"); the convergence-factor check (P10) has no
printed value in the paper to compare with and is "parity unpinned" in
absolute value.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hmg_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "band_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the oracle shared library (gcc).  Returns its path."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *_SRCS, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64p = ctypes.POINTER(ctypes.c_int64)
            lib.ora_build.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_double, P, ctypes.POINTER(P)]
            lib.ora_build_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, P, ctypes.POINTER(P)]
            lib.ora_free.argtypes = [P]
            lib.ora_free.restype = None
            lib.ora_ncells.argtypes = [P, ctypes.c_int]
            lib.ora_ncells.restype = ctypes.c_int64
            lib.ora_nverts.argtypes = [P, ctypes.c_int]
            lib.ora_nverts.restype = ctypes.c_int64
            lib.ora_export_level.argtypes = [P, ctypes.c_int] + [P] * 10
            lib.ora_set_bands.argtypes = [P, ctypes.c_int, P, P, P]
            lib.ora_apply.argtypes = [P, ctypes.c_int, P, P]
            lib.ora_thomas.argtypes = [ctypes.c_int, P, P, P, P]
            lib.ora_sweep.argtypes = [P, ctypes.c_int, P, P, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_int, i64p]
            lib.ora_residual.argtypes = [P, ctypes.c_int, P, P, P]
            lib.ora_restrict.argtypes = [P, ctypes.c_int, P, P]
            lib.ora_prolong_add.argtypes = [P, ctypes.c_int, P, P]
            lib.ora_vcycle.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, P, P]
            lib.ora_pcg.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_double, P, P, ctypes.c_double, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), P]
            lib.ora_mixed_nedges.argtypes = [P]
            lib.ora_mixed_nedges.restype = ctypes.c_int64
            lib.ora_mixed_size.argtypes = [P]
            lib.ora_mixed_size.restype = ctypes.c_int64
            lib.ora_mixed_edges.argtypes = [P, P, P, P]
            lib.ora_mixed_part.argtypes = [P, ctypes.c_int, P, P, P, P, P, P]
            lib.ora_mixed_apply.argtypes = [P, P, P]
            lib.ora_mixed_precond.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_double, P, P]
            lib.ora_mixed_gmres.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                            ctypes.c_int, P, P, ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_double), P, ctypes.POINTER(ctypes.c_double)]
            lib.ora_last_error.restype = ctypes.c_char_p
            lib.ora_set_threads.argtypes = [ctypes.c_int]
            lib.ora_set_threads.restype = None
            # NEXT-3 core (band_oracle.c)
            lib.ora_gbtrf.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P]
            lib.ora_gbtrs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P, P, P]
            lib.ora_gbtrs.restype = None
            lib.ora_gbmv.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P]
            lib.ora_gbmv.restype = None
            lib.ora_p_restrict.argtypes = [ctypes.c_int64, ctypes.c_int, P, P]
            lib.ora_p_restrict.restype = None
            lib.ora_p_prolong_add.argtypes = [ctypes.c_int64, ctypes.c_int, P, P]
            lib.ora_p_prolong_add.restype = None
            _lib = lib
    return _lib


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's column loops (results are independent of it)."""
    _load().ora_set_threads(int(n))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


SINGULAR = 4
NOT_CONVERGED = 5


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(code: int):
    if code != 0:
        raise OracleError(code, _load().ora_last_error().decode())


def thomas(D, U, r) -> np.ndarray:
    """O6 Thomas solve of one column: diag D[nz], off-diagonal U[nz] (U[k]
    couples k and k+1), rhs r[nz]."""
    D, U, r = _f64(D), _f64(U), _f64(r)
    out = np.empty_like(r)
    _check(_load().ora_thomas(len(D), _ptr(D), _ptr(U), _ptr(r), _ptr(out)))
    return out


class Hierarchy:
    """Oracle hierarchy ref ``fine_ref`` -> ``coarsest_ref`` (O1-O4)."""

    def __init__(self, fine_ref: int, coarsest_ref: int, nz: int, thickness: float, w2: float, lam,
                 omega_n: float = 0.0):
        """omega_n: the buoyancy term omega_N = (dt/2) N of Eq. 5 (reading R24);
        0 = BASELINE's operator."""
        lib = _load()
        self.fine_ref, self.coarsest_ref, self.nz = fine_ref, coarsest_ref, nz
        self.thickness, self.w2, self.omega_n = thickness, w2, omega_n
        lam = _f64(lam)
        h = ctypes.c_void_p()
        _check(lib.ora_build_ex(fine_ref, coarsest_ref, nz, thickness, w2, omega_n, _ptr(lam), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _load().ora_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def n(self, ref: int) -> int:
        return int(_load().ora_ncells(self._h, ref))

    def shape(self, ref: int):
        return (self.nz, self.n(ref))

    def level(self, ref: int) -> dict:
        """Export topology, geometry, coefficients and bands of one level."""
        lib = _load()
        n, nz = self.n(ref), self.nz
        nv = int(lib.ora_nverts(self._h, ref))
        out = dict(
            verts=np.empty((nv, 3)), faces=np.empty((n, 3), np.int32), nbr=np.empty((n, 3), np.int32),
            area=np.empty(n), len=np.empty((n, 3)), cd=np.empty((n, 3)), lam=np.empty((nz, n)),
            D=np.empty((nz, n)), U=np.empty((nz, n)), H=np.empty((3, nz, n)))
        _check(lib.ora_export_level(self._h, ref, *[_ptr(out[k]) for k in
                                                    ("verts", "faces", "nbr", "area", "len", "cd", "lam", "D", "U", "H")]))
        return out

    def set_bands(self, ref: int, D=None, U=None, H=None):
        D = None if D is None else _f64(D)
        U = None if U is None else _f64(U)
        H = None if H is None else _f64(H)
        _check(_load().ora_set_bands(self._h, ref, _ptr(D), _ptr(U), _ptr(H)))

    def apply(self, ref: int, x) -> np.ndarray:
        x = _f64(x)
        y = np.empty_like(x)
        _check(_load().ora_apply(self._h, ref, _ptr(x), _ptr(y)))
        return y

    def residual(self, ref: int, b, u) -> np.ndarray:
        b, u = _f64(b), _f64(u)
        r = np.empty_like(b)
        _check(_load().ora_residual(self._h, ref, _ptr(b), _ptr(u), _ptr(r)))
        return r

    def sweep(self, ref: int, b, u=None, nsweeps: int = 1, omega: float = 0.8) -> np.ndarray:
        """O7: ``nsweeps`` damped line-Jacobi sweeps; u=None is the zero guess."""
        b = _f64(b)
        zero = u is None
        u = np.zeros_like(b) if zero else _f64(u).copy()
        bad = ctypes.c_int64(-1)
        _check(_load().ora_sweep(self._h, ref, _ptr(b), _ptr(u), nsweeps, omega, int(zero), ctypes.byref(bad)))
        return u

    def restrict(self, fine_ref: int, r) -> np.ndarray:
        r = _f64(r)
        bc = np.empty((self.nz, self.n(fine_ref - 1)))
        _check(_load().ora_restrict(self._h, fine_ref, _ptr(r), _ptr(bc)))
        return bc

    def prolong_add(self, fine_ref: int, uc, uf) -> np.ndarray:
        uc, uf = _f64(uc), _f64(uf).copy()
        _check(_load().ora_prolong_add(self._h, fine_ref, _ptr(uc), _ptr(uf)))
        return uf

    def vcycle(self, b, nu_pre=2, nu_post=2, n_coarse=20, omega=0.8) -> np.ndarray:
        b = _f64(b)
        z = np.empty_like(b)
        _check(_load().ora_vcycle(self._h, nu_pre, nu_post, n_coarse, omega, _ptr(b), _ptr(z)))
        return z

    def pcg(self, b, rtol=1e-8, maxit=200, precond="vcycle", nu_pre=2, nu_post=2, n_coarse=20,
            omega=0.8, raise_on_fail=False):
        """O10 PCG.  Returns (x, iters, relres, history, status)."""
        kind = {"none": 0, "vcycle": 1, "single": 2}[precond]
        b = _f64(b)
        x = np.empty_like(b)
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        hist = np.zeros(maxit + 1)
        code = _load().ora_pcg(self._h, kind, nu_pre, nu_post, n_coarse, omega, _ptr(b), _ptr(x),
                               rtol, maxit, ctypes.byref(it), ctypes.byref(rr), _ptr(hist))
        if code not in (0, NOT_CONVERGED) or (raise_on_fail and code):
            _check(code)
        return x, it.value, rr.value, hist[: it.value + 1], code

    # ---- NEXT-4: mixed velocity-pressure system (readings R15-R20) ----
    def mixed_sizes(self):
        """(ne, N): fine-level edge count and the mixed vector length
        nz*ne + (nz-1)*n + nz*n (blocks [U_h | U_z | P])."""
        lib = _load()
        return int(lib.ora_mixed_nedges(self._h)), int(lib.ora_mixed_size(self._h))

    def mixed_split(self, x):
        """Views (U_h [nz][ne], U_z [nz-1][n], P [nz][n]) of a mixed vector."""
        ne, _ = self.mixed_sizes()
        nz, n = self.nz, self.n(self.fine_ref)
        a, b = nz * ne, nz * ne + (nz - 1) * n
        return x[:a].reshape(nz, ne), x[a:b].reshape(nz - 1, n), x[b:].reshape(nz, n)

    def mixed_edges(self):
        """Edge table (reading R16): ec [ne][2] cells (a < b), es [ne][2]
        slots, ce [n][3] edge across each slot."""
        ne, _ = self.mixed_sizes()
        n = self.n(self.fine_ref)
        ec, es, ce = np.empty((ne, 2), np.int32), np.empty((ne, 2), np.int32), np.empty((n, 3), np.int32)
        _check(_load().ora_mixed_edges(self._h, _ptr(ec), _ptr(es), _ptr(ce)))
        return ec, es, ce

    def mixed_part(self, which: str, Uh=None, Uz=None, P=None):
        """One operator of the mixed system: 'div' (U -> p), 'divT' (P -> U),
        'mass' (M2), 'lumped_inv' (L^-1), 'gram' (RT0 Gram matrices [n][3][3])."""
        ne, _ = self.mixed_sizes()
        nz, n = self.nz, self.n(self.fine_ref)
        code = {"div": 0, "divT": 1, "mass": 2, "lumped_inv": 3, "gram": 4}[which]
        Uh = None if Uh is None else _f64(Uh)
        Uz = None if Uz is None else _f64(Uz)
        P = None if P is None else _f64(P)
        yh = np.zeros((n, 3, 3)) if which == "gram" else np.zeros((nz, ne))
        yz, yp = np.zeros((max(nz - 1, 0), n)), np.zeros((nz, n))
        _check(_load().ora_mixed_part(self._h, code, _ptr(Uh), _ptr(Uz), _ptr(P), _ptr(yh), _ptr(yz), _ptr(yp)))
        if which == "div":
            return yp
        if which == "gram":
            return yh
        return yh, yz

    def mixed_apply(self, x) -> np.ndarray:
        """y = A x, A = [[M2, -omega D^T], [omega D, M3]], omega = sqrt(w2)."""
        x = _f64(x)
        y = np.empty_like(x)
        _check(_load().ora_mixed_apply(self._h, _ptr(x), _ptr(y)))
        return y

    def mixed_precond(self, f, precond="schur", nu_pre=2, nu_post=2, n_coarse=20, omega=0.8) -> np.ndarray:
        """Schur-complement preconditioner (Eq. 6, lumped mass, one V-cycle)."""
        f = _f64(f)
        x = np.empty_like(f)
        kind = {"none": 0, "schur": 1}[precond]
        _check(_load().ora_mixed_precond(self._h, kind, nu_pre, nu_post, n_coarse, omega, _ptr(f), _ptr(x)))
        return x

    def mixed_gmres(self, F, rtol=1e-5, restart=30, maxit=300, precond="schur", nu_pre=2, nu_post=2, n_coarse=20,
                    omega=0.8, gs_passes=2, orth=False):
        """Right-preconditioned GMRES(restart), x0 = 0, classical Gram-Schmidt
        applied ``gs_passes`` times per Arnoldi step (1 = CGS, PETSc's default;
        2 = CGS2, reading R20).  Returns (x, iters, relres, history, status), plus
        the basis' worst orthogonality error max|<v_a, v_b> - delta_ab| over all
        cycles when ``orth``."""
        F = _f64(F)
        x = np.empty_like(F)
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        oe = ctypes.c_double(0.0)
        hist = np.zeros(maxit + 1)
        kind = {"none": 0, "schur": 1}[precond]
        code = _load().ora_mixed_gmres(self._h, kind, nu_pre, nu_post, n_coarse, omega, restart, rtol, maxit,
                                       gs_passes, _ptr(F), _ptr(x), ctypes.byref(it), ctypes.byref(rr), _ptr(hist),
                                       ctypes.byref(oe) if orth else None)
        if code not in (0, NOT_CONVERGED):
            _check(code)
        out = (x, it.value, rr.value, hist[: it.value + 1], code)
        return out + (oe.value,) if orth else out


# ---- NEXT-3 core: per-column banded LU (dgbtrf / dgbtrs) and DG1 <-> DG0 ----
def gbtrf(ab, kl: int, ku: int):
    """dgbtrf (unblocked dgbtf2 order) of ONE m x m banded matrix in LAPACK band
    storage ``ab`` [ldab][m] (ldab >= 2 kl + ku + 1, A(i, j) = ab[kl + ku + i - j, j]).
    Returns (lu [ldab][m], ipiv [m] 0-based int32, info)."""
    a = np.asfortranarray(ab, dtype=np.float64)          # column j contiguous, as LAPACK
    ldab, m = a.shape
    flat = np.ascontiguousarray(a.T)                      # [m][ldab]
    ipiv = np.zeros(m, np.int32)
    info = _load().ora_gbtrf(m, kl, ku, _ptr(flat), ldab, _ptr(ipiv))
    return flat.T.copy(), ipiv, int(info)


def gbtrs(lu, kl: int, ku: int, ipiv, b) -> np.ndarray:
    """dgbtrs ('N', one right-hand side) from gbtrf's factors."""
    ldab, m = lu.shape
    flat = np.ascontiguousarray(np.asarray(lu, dtype=np.float64).T)
    ip = np.ascontiguousarray(ipiv, dtype=np.int32)
    b = _f64(b)
    x = np.empty_like(b)
    _load().ora_gbtrs(m, kl, ku, _ptr(flat), ldab, _ptr(ip), _ptr(b), _ptr(x))
    return x


def gbmv(ab_rows, kl: int, ku: int, x) -> np.ndarray:
    """y = A x, the paper's row-wise band storage ab_rows [m][kl + ku + 1]."""
    a = _f64(ab_rows)
    m = a.shape[0]
    assert a.shape[1] == kl + ku + 1
    x = _f64(x)
    y = np.empty(m)
    _load().ora_gbmv(m, kl, ku, _ptr(a), _ptr(x), _ptr(y))
    return y


def p_restrict(r1) -> np.ndarray:
    """DG1 -> DG0: r1 [ncol][6 nz] -> b0 [ncol][nz], the 6 nodal values summed."""
    r1 = _f64(r1)
    ncol, m = r1.shape
    b0 = np.empty((ncol, m // 6))
    _load().ora_p_restrict(ncol, m // 6, _ptr(r1), _ptr(b0))
    return b0


def p_prolong_add(u0, u1) -> np.ndarray:
    """u1 + P u0: every nodal value of cell k gets the cell's DG0 value."""
    u0, u1 = _f64(u0), _f64(u1).copy()
    ncol, nz = u0.shape
    _load().ora_p_prolong_add(ncol, nz, _ptr(u0), _ptr(u1))
    return u1
