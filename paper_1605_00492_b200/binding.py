"""ctypes binding of the C-ABI in include/hmg.h (argument marshalling only).

Device vectors are torch float64 CUDA tensors of shape (nlayers, ld) (layer-
major, see ``Hierarchy.level_info``); host vectors are numpy float64 arrays of
shape (nlayers, ncells).  Calls are enqueued on torch's current CUDA stream.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libhmg.so")
_lib = None

STATUS = {0: "HMG_OK", 1: "HMG_ERR_INVALID_ARG", 2: "HMG_ERR_CUDA", 3: "HMG_ERR_NCCL",
          4: "HMG_ERR_SINGULAR_COLUMN", 5: "HMG_ERR_NOT_CONVERGED", 6: "HMG_ERR_OOM"}


class HmgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nccl_id", ctypes.c_void_p),
                ("gather_ref", ctypes.c_int)]


class _Params(ctypes.Structure):
    _fields_ = [("nu_pre", ctypes.c_int), ("nu_post", ctypes.c_int), ("n_coarse", ctypes.c_int),
                ("omega", ctypes.c_double)]


@dataclass(frozen=True)
class MGParams:
    """V-cycle parameters; defaults are BASELINE.json's V(2,2), 20 coarse sweeps, omega 0.8."""
    nu_pre: int = 2
    nu_post: int = 2
    n_coarse: int = 20
    omega: float = 0.8

    def c(self) -> _Params:
        return _Params(self.nu_pre, self.nu_post, self.n_coarse, self.omega)


def lib_path() -> str:
    return _LIB_PATH


def load_library():
    """Load libhmg.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"CUDA library {_LIB_PATH} not built: run __graft_entry__.build() "
                          "(python -m paper_1605_00492_b200.build)")
    lib = ctypes.CDLL(_LIB_PATH)
    P, I, D, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64
    pI, pD, pI64 = ctypes.POINTER(I), ctypes.POINTER(D), ctypes.POINTER(I64)
    pP = ctypes.POINTER(_Params)
    sig = {
        "hmg_build_hierarchy": [I, I, I, D, D, P, I, ctypes.POINTER(P)],
        "hmg_free_hierarchy": [P],
        "hmg_level_info": [P, I, pI64, pI64],
        "hmg_apply_helmholtz": [P, I, P, P, P],
        "hmg_line_smooth": [P, I, P, P, I, D, I, P],
        "hmg_restrict": [P, I, P, P, P],
        "hmg_residual_restrict": [P, I, P, P, P, P],
        "hmg_prolong_add": [P, I, P, P, P],
        "hmg_vcycle": [P, pP, P, P, P],
        "hmg_pcg_solve": [P, pP, P, P, D, I, pI, pD, P],
        "hmg_pcg_solve_host": [P, pP, P, P, D, I, pI, pD, P],
        "hmg_pcg_solve_host_batch": [P, pP, I, P, P, D, I, pI, pD, P],
        "hmg_pcg_solve_single_level": [P, I, D, P, P, D, I, pI, pD, P],
        "hmg_export_level": [P, I, P, P, P, P],
        "hmg_selftest_div": [P, P, P, P, I64, P],
        "hmg_profile_begin": [P],
        "hmg_profile_end": [P],
        "hmg_profile_select": [P, I, I],
        "hmg_profile_query": [P, I, I, pI64, pD],
        "hmg_build_hierarchy_dist": [I, I, I, D, D, P, I, P, ctypes.POINTER(P)],
        "hmg_build_hierarchy_ex": [I, I, I, D, D, D, P, I, P, ctypes.POINTER(P)],
        "hmg_nccl_unique_id": [P],
        "hmg_partition_plan": [I, I, I, I, pI64, pI64, pI64, pI, pI64, P, P, P, P, P, P, P],
        "hmg_mixed_layout": [P, pI64, pI64, pI64, pI64, pI64],
        "hmg_edge_store": [P, I, pI],
        "hmg_mixed_export_edges": [P, P, P],
        "hmg_mixed_apply": [P, P, P, P],
        "hmg_mixed_precond": [P, pP, P, P, P],
        "hmg_mixed_gmres": [P, pP, P, P, D, I, I, I, pI, pD, P],
        "hmg_pcg_history": [P, P, I, pI],
        "hmg_band_factor": [I64, I, I, I, P, I64, P, pI64, P],
        "hmg_band_solve": [I64, I, I, I, P, I64, P, P, P, P],
        "hmg_band_apply": [I64, I, I, I, P, I64, P, P, P],
        "hmg_p_restrict": [I64, I, P, I64, P, P],
        "hmg_p_prolong_add": [I64, I, P, I64, P, P],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.hmg_launch_count.argtypes = [P]
    lib.hmg_launch_count.restype = I64
    lib.hmg_last_error.argtypes = []
    lib.hmg_last_error.restype = ctypes.c_char_p
    _lib = lib
    return lib


def _check(code: int, allow=()):
    if code != 0 and code not in allow:
        raise HmgError(code, load_library().hmg_last_error().decode())
    return code


def _stream():
    import torch
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dptr(t, name: str):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous float64 CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


def _tptr(t, name: str, dtype_name: str):
    import torch
    dt = {"float64": torch.float64, "int32": torch.int32}[dtype_name]
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dt or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous {dtype_name} CUDA tensor")
    return ctypes.c_void_p(t.data_ptr())


# ---- NEXT-3 core: batched per-column banded algebra (include/hmg.h hmg_band_*) ----
def band_factor(ab, ipiv, ncol: int, kl: int, ku: int) -> int:
    """In-place LU (dgbtrf) of every column: ab [m][2kl+ku+1][ld] float64,
    ipiv [m][ld] int32 (CUDA tensors).  Raises HmgError (HMG_ERR_SINGULAR_COLUMN)
    naming the first column with a zero pivot (the factorisation is completed)."""
    m, ldab, ld = ab.shape
    assert ldab == 2 * kl + ku + 1 and tuple(ipiv.shape) == (m, ld)
    sing = ctypes.c_int64(-1)
    _check(load_library().hmg_band_factor(ncol, m, kl, ku, _tptr(ab, "ab", "float64"), ld,
                                          _tptr(ipiv, "ipiv", "int32"), ctypes.byref(sing), _stream()))
    return sing.value


def band_solve(ab, ipiv, b, x, ncol: int, kl: int, ku: int):
    """x = A^-1 b per column (dgbtrs) from band_factor's output; b, x [m][ld]."""
    m, ldab, ld = ab.shape
    _check(load_library().hmg_band_solve(ncol, m, kl, ku, _tptr(ab, "ab", "float64"), ld,
                                         _tptr(ipiv, "ipiv", "int32"), _tptr(b, "b", "float64"),
                                         _tptr(x, "x", "float64"), _stream()))
    return x


def band_apply(ar, x, y, ncol: int, kl: int, ku: int):
    """y = A x per column, ar [m][kl+ku+1][ld] the paper's row-wise band storage."""
    m, bw, ld = ar.shape
    assert bw == kl + ku + 1
    _check(load_library().hmg_band_apply(ncol, m, kl, ku, _tptr(ar, "ar", "float64"), ld,
                                         _tptr(x, "x", "float64"), _tptr(y, "y", "float64"), _stream()))
    return y


def p_restrict(r1, b0, ncol: int):
    """DG1 -> DG0: b0 [nz][ld] = sum of the 6 nodal values, r1 [6 nz][ld]."""
    nz, ld = b0.shape
    _check(load_library().hmg_p_restrict(ncol, nz, _tptr(r1, "r1", "float64"), ld, _tptr(b0, "b0", "float64"),
                                         _stream()))
    return b0


def p_prolong_add(u0, u1, ncol: int):
    """DG0 -> DG1: u1 [6 nz][ld] += the cell value on each of its 6 nodes."""
    nz, ld = u0.shape
    _check(load_library().hmg_p_prolong_add(ncol, nz, _tptr(u0, "u0", "float64"), ld, _tptr(u1, "u1", "float64"),
                                            _stream()))
    return u1


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) for hmg_build_hierarchy_dist; call on rank 0 and broadcast."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().hmg_nccl_unique_id(buf))
    return buf.raw


def partition_plan(fine_ref: int, ref: int, rank: int, nranks: int) -> dict:
    """Host-only partition plan of one level for one rank (hmg_partition_plan)."""
    lib = load_library()
    off, n_own, n_halo, send_total = (ctypes.c_int64() for _ in range(4))
    npeers = ctypes.c_int()
    _check(lib.hmg_partition_plan(fine_ref, ref, rank, nranks, ctypes.byref(off), ctypes.byref(n_own),
                                  ctypes.byref(n_halo), ctypes.byref(npeers), ctypes.byref(send_total),
                                  *([None] * 7)))
    halo = np.empty(n_halo.value, np.int64)
    nbr = np.empty((n_own.value, 3), np.int32)
    prank = np.empty(npeers.value, np.int32)
    scount, roff, rcount = (np.empty(npeers.value, np.int64) for _ in range(3))
    slocal = np.empty(send_total.value, np.int32)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    _check(lib.hmg_partition_plan(fine_ref, ref, rank, nranks, None, None, None, None, None, ptr(halo), ptr(nbr),
                                  ptr(prank), ptr(scount), ptr(roff), ptr(rcount), ptr(slocal)))
    peers, pos = [], 0
    for i in range(npeers.value):
        peers.append(dict(rank=int(prank[i]), send_local=slocal[pos:pos + scount[i]].copy(),
                          recv_offset=int(roff[i]), recv_count=int(rcount[i])))
        pos += int(scount[i])
    return dict(off=off.value, n_own=n_own.value, halo_gid=halo, nbr_local=nbr, peers=peers)


def selftest_div(a, b):
    """(fast, ref) device tensors: the sweep kernel's division vs the '/' operator."""
    import torch
    fast, ref = torch.empty_like(a), torch.empty_like(a)
    _check(load_library().hmg_selftest_div(_dptr(a, "a"), _dptr(b, "b"), _dptr(fast, "fast"), _dptr(ref, "ref"),
                                           a.numel(), _stream()))
    return fast, ref


class Hierarchy:
    """Device hierarchy ref ``fine_ref`` -> ``coarsest_ref`` (hmg_build_hierarchy)."""

    def __init__(self, fine_ref: int, coarsest_ref: int, nlayers: int, thickness: float, w2: float,
                 lam, device: int = 0, dist=None, omega_n: float = 0.0):
        """dist = (rank, nranks, nccl_id_bytes, gather_ref) for one rank of a
        distributed hierarchy; lam is then this rank's owned part of the finest
        level when gather_ref < fine_ref.  omega_n: the buoyancy term of Eq. 5
        (hmg_build_hierarchy_ex; 0 = BASELINE's operator)."""
        lib = load_library()
        lam = np.ascontiguousarray(np.asarray(lam, dtype=np.float64))
        n = 20 * 4 ** fine_ref if 0 <= fine_ref <= 10 else 0
        if dist is not None and dist[3] < fine_ref:
            n //= max(int(dist[1]), 1)                # this rank's owned part of the finest level
        if lam.size != nlayers * n:
            raise ValueError(f"lam: expected {nlayers} x {n} values, got shape {lam.shape}")
        h = ctypes.c_void_p()
        if dist is None and omega_n == 0.0:
            _check(lib.hmg_build_hierarchy(fine_ref, coarsest_ref, nlayers, thickness, w2,
                                           lam.ctypes.data_as(ctypes.c_void_p), device, ctypes.byref(h)))
        elif dist is None:
            _check(lib.hmg_build_hierarchy_ex(fine_ref, coarsest_ref, nlayers, thickness, w2, omega_n,
                                              lam.ctypes.data_as(ctypes.c_void_p), device, None, ctypes.byref(h)))
        else:
            rank, nranks, nid, gref = dist
            self._nid = ctypes.create_string_buffer(bytes(nid), 128)
            d = _Dist(rank, nranks, ctypes.cast(self._nid, ctypes.c_void_p), gref)
            _check(lib.hmg_build_hierarchy_ex(fine_ref, coarsest_ref, nlayers, thickness, w2, omega_n,
                                              lam.ctypes.data_as(ctypes.c_void_p), device, ctypes.byref(d),
                                              ctypes.byref(h)))
        self.dist = dist
        self._h = h
        self.fine_ref, self.coarsest_ref, self.nz = fine_ref, coarsest_ref, nlayers
        self.thickness, self.w2, self.device, self.omega_n = thickness, w2, device, omega_n

    def close(self):
        if getattr(self, "_h", None):
            load_library().hmg_free_hierarchy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- shapes and tensors -------------------------------------------------
    def level_info(self, ref: int):
        n, ld = ctypes.c_int64(), ctypes.c_int64()
        _check(load_library().hmg_level_info(self._h, ref, ctypes.byref(n), ctypes.byref(ld)))
        return n.value, ld.value

    def empty(self, ref: int):
        import torch
        _, ld = self.level_info(ref)
        return torch.zeros((self.nz, ld), dtype=torch.float64, device=f"cuda:{self.device}")

    def to_device(self, ref: int, a):
        """numpy [nz][n] -> padded CUDA tensor [nz][ld]."""
        import torch
        n, ld = self.level_info(ref)
        t = self.empty(ref)
        t[:, :n] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(t.device)
        return t

    def to_host(self, ref: int, t) -> np.ndarray:
        n, _ = self.level_info(ref)
        return t[:, :n].cpu().numpy().copy()

    @property
    def launches(self) -> int:
        return int(load_library().hmg_launch_count(self._h))

    # -- the C-ABI calls -----------------------------------------------------
    def apply_helmholtz(self, ref: int, x, y=None):
        y = self.empty(ref) if y is None else y
        _check(load_library().hmg_apply_helmholtz(self._h, ref, _dptr(x, "x"), _dptr(y, "y"), _stream()))
        return y

    def line_smooth(self, ref: int, b, u, nsweeps: int = 1, omega: float = 0.8, u_is_zero: bool = False):
        _check(load_library().hmg_line_smooth(self._h, ref, _dptr(b, "b"), _dptr(u, "u"), nsweeps, omega,
                                              int(u_is_zero), _stream()))
        return u

    def restrict(self, fine_ref: int, r_f, b_c=None):
        b_c = self.empty(fine_ref - 1) if b_c is None else b_c
        _check(load_library().hmg_restrict(self._h, fine_ref, _dptr(r_f, "r_f"), _dptr(b_c, "b_c"), _stream()))
        return b_c

    def residual_restrict(self, fine_ref: int, b, u, b_c=None):
        b_c = self.empty(fine_ref - 1) if b_c is None else b_c
        _check(load_library().hmg_residual_restrict(self._h, fine_ref, _dptr(b, "b"), _dptr(u, "u"),
                                                    _dptr(b_c, "b_c"), _stream()))
        return b_c

    def prolong_add(self, fine_ref: int, u_c, u_f):
        _check(load_library().hmg_prolong_add(self._h, fine_ref, _dptr(u_c, "u_c"), _dptr(u_f, "u_f"), _stream()))
        return u_f

    def vcycle(self, b, z=None, params: MGParams = MGParams()):
        z = self.empty(self.fine_ref) if z is None else z
        p = params.c()
        _check(load_library().hmg_vcycle(self._h, ctypes.byref(p), _dptr(b, "b"), _dptr(z, "z"), _stream()))
        return z

    def pcg_solve(self, b, x=None, rtol: float = 1e-8, maxit: int = 200, params: MGParams = MGParams()):
        """Returns (x, iters, relres, status_name)."""
        x = self.empty(self.fine_ref) if x is None else x
        p = params.c()
        it, rr = ctypes.c_int(0), ctypes.c_double(0.0)
        code = _check(load_library().hmg_pcg_solve(self._h, ctypes.byref(p), _dptr(b, "b"), _dptr(x, "x"), rtol,
                                                   maxit, ctypes.byref(it), ctypes.byref(rr), _stream()),
                      allow=(5,))
        return x, it.value, rr.value, STATUS[code]

    def pcg_history(self) -> np.ndarray:
        """||r_k|| / ||b||, k = 0 .. iters, of the last PCG solve (hmg_pcg_history)."""
        n = ctypes.c_int(0)
        _check(load_library().hmg_pcg_history(self._h, None, 0, ctypes.byref(n)))
        out = np.zeros(n.value)
        _check(load_library().hmg_pcg_history(self._h, out.ctypes.data_as(ctypes.c_void_p), n.value,
                                              ctypes.byref(n)))
        return out

    def pcg_solve_single_level(self, b, x=None, nsweeps: int = 2, omega: float = 0.8, rtol: float = 1e-8,
                               maxit: int = 500):
        x = self.empty(self.fine_ref) if x is None else x
        it, rr = ctypes.c_int(0), ctypes.c_double(0.0)
        code = _check(load_library().hmg_pcg_solve_single_level(self._h, nsweeps, omega, _dptr(b, "b"),
                                                                _dptr(x, "x"), rtol, maxit, ctypes.byref(it),
                                                                ctypes.byref(rr), _stream()), allow=(5,))
        return x, it.value, rr.value, STATUS[code]

    def pcg_solve_host(self, b: np.ndarray, x: np.ndarray | None = None, rtol: float = 1e-8, maxit: int = 200,
                       params: MGParams = MGParams()):
        """End-to-end entry point: host arrays [nz][n] in and out."""
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty_like(b) if x is None else x
        p = params.c()
        it, rr = ctypes.c_int(0), ctypes.c_double(0.0)
        code = _check(load_library().hmg_pcg_solve_host(self._h, ctypes.byref(p), b.ctypes.data_as(ctypes.c_void_p),
                                                        x.ctypes.data_as(ctypes.c_void_p), rtol, maxit,
                                                        ctypes.byref(it), ctypes.byref(rr), _stream()), allow=(5,))
        return x, it.value, rr.value, STATUS[code]

    def pcg_solve_host_batch(self, bs, xs, rtol: float = 1e-8, maxit: int = 200,
                             params: MGParams = MGParams()):
        """Pipelined end-to-end solves of several right-hand sides: host arrays
        bs[i] -> xs[i], each [nz][n] float64 C-contiguous (page-locked for the
        copy/compute overlap).  Returns (iters list, relres list, status)."""
        k = len(bs)
        if len(xs) != k:
            raise ValueError("bs and xs must have the same length")
        for a in list(bs) + list(xs):
            if a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError("host buffers must be C-contiguous float64")
        bp = (ctypes.c_void_p * max(k, 1))(*[a.ctypes.data for a in bs])
        xp = (ctypes.c_void_p * max(k, 1))(*[a.ctypes.data for a in xs])
        it = (ctypes.c_int * max(k, 1))()
        rr = (ctypes.c_double * max(k, 1))()
        p = params.c()
        code = _check(load_library().hmg_pcg_solve_host_batch(self._h, ctypes.byref(p), k, bp, xp, rtol, maxit,
                                                              it, rr, _stream()), allow=(5,))
        return list(it)[:k], list(rr)[:k], STATUS[code]

    # -- diagnostics -----------------------------------------------------------
    KERNEL_CLASSES = {"apply": 0, "sweep_zero": 1, "sweep": 2, "sweep_prolong": 3, "resid_restrict": 4,
                      "restrict": 5, "prolong": 6, "vector": 7, "coarse_tail": 8, "apply_pupdate": 9,
                      "mixed": 10}

    def profile_begin(self):
        _check(load_library().hmg_profile_begin(self._h))

    def profile_select(self, kernel_class: str | None = None, ref: int = -1):
        """Record only one kernel class on one level (None: all)."""
        cls = -1 if kernel_class is None else self.KERNEL_CLASSES[kernel_class]
        _check(load_library().hmg_profile_select(self._h, cls, ref))

    def profile_end(self):
        _check(load_library().hmg_profile_end(self._h))

    def profile_query(self, kernel_class: str, ref: int = -1):
        """(launch count, total ms) of one kernel class recorded since profile_begin."""
        n, ms = ctypes.c_int64(), ctypes.c_double()
        _check(load_library().hmg_profile_query(self._h, self.KERNEL_CLASSES[kernel_class], ref, ctypes.byref(n),
                                                ctypes.byref(ms)))
        return n.value, ms.value

    def edge_store(self, ref: int) -> dict:
        """Which kernels of level ``ref`` read the edge-deduplicated coupling store."""
        k = ctypes.c_int(0)
        _check(load_library().hmg_edge_store(self._h, ref, ctypes.byref(k)))
        return {"sweep": bool(k.value & 1), "apply": bool(k.value & 2), "resid_restrict": bool(k.value & 4)}

    # -- NEXT-4: mixed velocity-pressure system (include/hmg.h hmg_mixed_*) ----
    def mixed_layout(self) -> dict:
        """ne, ldh, off_z, off_p, ntot of the mixed vectors [U_h | U_z | P]."""
        v = [ctypes.c_int64() for _ in range(5)]
        _check(load_library().hmg_mixed_layout(self._h, *[ctypes.byref(x) for x in v]))
        return dict(zip(("ne", "ldh", "off_z", "off_p", "ntot"), (x.value for x in v)))

    def mixed_edges(self):
        """(ec [ne][2], ce [n][3]) host int32 arrays."""
        lay = self.mixed_layout()
        n, _ = self.level_info(self.fine_ref)
        ec, ce = np.empty((lay["ne"], 2), np.int32), np.empty((n, 3), np.int32)
        _check(load_library().hmg_mixed_export_edges(self._h, ec.ctypes.data_as(ctypes.c_void_p),
                                                     ce.ctypes.data_as(ctypes.c_void_p)))
        return ec, ce

    def mixed_to_device(self, x: np.ndarray):
        """Oracle-layout mixed vector (nz*ne | (nz-1)*n | nz*n) -> padded device vector."""
        import torch
        lay = self.mixed_layout()
        n, ld = self.level_info(self.fine_ref)
        nz, ne = self.nz, lay["ne"]
        t = torch.zeros(lay["ntot"], dtype=torch.float64, device=f"cuda:{self.device}")
        a, b = nz * ne, nz * ne + (nz - 1) * n
        x = np.ascontiguousarray(x, dtype=np.float64)
        t[: lay["off_z"]].view(nz, lay["ldh"])[:, :ne] = torch.from_numpy(x[:a].reshape(nz, ne))
        if nz > 1:
            t[lay["off_z"]: lay["off_p"]].view(nz - 1, ld)[:, :n] = torch.from_numpy(x[a:b].reshape(nz - 1, n))
        t[lay["off_p"]:].view(nz, ld)[:, :n] = torch.from_numpy(x[b:].reshape(nz, n))
        return t

    def mixed_to_host(self, t) -> np.ndarray:
        lay = self.mixed_layout()
        n, ld = self.level_info(self.fine_ref)
        nz, ne = self.nz, lay["ne"]
        parts = [t[: lay["off_z"]].view(nz, lay["ldh"])[:, :ne]]
        if nz > 1:
            parts.append(t[lay["off_z"]: lay["off_p"]].view(nz - 1, ld)[:, :n])
        parts.append(t[lay["off_p"]:].view(nz, ld)[:, :n])
        return np.concatenate([p.cpu().numpy().ravel() for p in parts])

    def mixed_empty(self):
        import torch
        return torch.zeros(self.mixed_layout()["ntot"], dtype=torch.float64, device=f"cuda:{self.device}")

    def mixed_apply(self, x, y=None):
        y = self.mixed_empty() if y is None else y
        _check(load_library().hmg_mixed_apply(self._h, _dptr(x, "x"), _dptr(y, "y"), _stream()))
        return y

    def mixed_precond(self, f, x=None, params: MGParams | None = MGParams()):
        x = self.mixed_empty() if x is None else x
        p = None if params is None else params.c()
        _check(load_library().hmg_mixed_precond(self._h, None if p is None else ctypes.byref(p), _dptr(f, "f"),
                                                _dptr(x, "x"), _stream()))
        return x

    def mixed_gmres(self, F, X=None, rtol: float = 1e-5, restart: int = 30, maxit: int = 300,
                    params: MGParams | None = MGParams(), gs_passes: int = 2):
        """gs_passes: 1 = CGS, 2 = CGS2.  Returns (X, iters, relres, status_name)."""
        X = self.mixed_empty() if X is None else X
        p = None if params is None else params.c()
        it, rr = ctypes.c_int(0), ctypes.c_double(0.0)
        code = _check(load_library().hmg_mixed_gmres(self._h, None if p is None else ctypes.byref(p), _dptr(F, "F"),
                                                     _dptr(X, "X"), rtol, restart, maxit, gs_passes, ctypes.byref(it),
                                                     ctypes.byref(rr), _stream()), allow=(5,))
        return X, it.value, rr.value, STATUS[code]

    def export_level(self, ref: int) -> dict:
        n, _ = self.level_info(ref)
        nz = self.nz
        nbr = np.empty((n, 3), np.int32)
        geom = np.empty((7, n))
        bands = np.empty((5, nz, n))
        lam = np.empty((nz, n))
        _check(load_library().hmg_export_level(self._h, ref, nbr.ctypes.data_as(ctypes.c_void_p),
                                               geom.ctypes.data_as(ctypes.c_void_p),
                                               bands.ctypes.data_as(ctypes.c_void_p),
                                               lam.ctypes.data_as(ctypes.c_void_p)))
        return dict(nbr=nbr, area=geom[0], len=geom[1:4].T.copy(), cd=geom[4:7].T.copy(), lam=lam,
                    D=bands[0], U=bands[1], H=bands[2:5])
