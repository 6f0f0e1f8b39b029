"""CPU oracle for the GMAF hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2511_06824_b200``) never imports it, and this package
never imports the product: both consume plain arrays produced by
``gmaf_inputs``.

The arithmetic lives in ``gmaf_oracle.c`` (plain C11, FP64, single thread,
``-O2 -ffp-contract=off``); this module only compiles it and marshals numpy
arrays through ctypes.  Every function cites the PAPER.md passage it follows
(see ``gmaf_oracle.h``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gmaf_oracle.c")
_HDR = os.path.join(_HERE, "gmaf_oracle.h")
LIB_PATH = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID_ARG, E_INVALID_MESH, E_MESH_TOO_COARSE = 0, -1, -2, -3
E_NONPOSITIVE_THICKNESS, E_BREAKDOWN, E_NO_CONVERGENCE = -4, -5, -6
PRECOND = {"none": 0, "jacobi": 1, "assor2": 2, "assor1": 3, "ssor": 4}
COUPLING = {"coupled": 0, "lockstep": 1}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math)."""
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < newest:
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
               "-shared", "-o", LIB_PATH + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class _Grid(C.Structure):
    _fields_ = [("n_theta", C.c_int32), ("n_y", C.c_int32), ("R_k", C.c_double), ("R_c", C.c_double),
                ("mu", C.c_double), ("h_min", C.c_double), ("tex_n_theta", C.c_int32),
                ("tex_n_y", C.c_int32), ("tex_band_rows", C.c_int32), ("tex_fill_num", C.c_int32),
                ("tex_fill_den", C.c_int32), ("tex_depth", C.c_double)]


class _Cond(C.Structure):
    _fields_ = [("e", C.c_double * 4), ("edot", C.c_double * 4), ("L_F", C.c_double),
                ("U_theta", C.c_double), ("U_y", C.c_double), ("p_in", C.c_double),
                ("p_out", C.c_double)]


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("rel_residual", C.c_double), ("true_rel_residual", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        D = C.POINTER(C.c_double)
        _lib.orc_thickness.argtypes = [C.POINTER(_Grid), C.POINTER(_Cond), D, D, D]
        _lib.orc_assemble.argtypes = [C.POINTER(_Grid), C.POINTER(_Cond), D, D, D, D]
        _lib.orc_check_grid.argtypes = [C.POINTER(_Grid)]
        _lib.orc_texture_mask.argtypes = [C.POINTER(_Grid), C.c_int32, C.c_int32]
        _lib.orc_spmv.argtypes = [C.c_int32, C.c_int32, D, D, D, D, D]
        _lib.orc_spmv.restype = None
        _lib.orc_precond_apply.argtypes = [C.c_int32, C.c_int32, D, D, D, C.c_int32, C.c_double, D, D]
        _lib.orc_precond_apply.restype = None
        _lib.orc_assor2_dense.argtypes = [C.c_int32, C.c_int32, D, D, D, C.c_double, D]
        _lib.orc_expand_dense.argtypes = [C.c_int32, C.c_int32, D, D, D, D]
        _lib.orc_cholesky_solve.argtypes = [C.c_int32, D, D, D]
        _lib.orc_pcg_joint.argtypes = [C.c_int32, C.c_int32, C.c_int32, D, D, D, D, D, C.c_double,
                                       C.c_double, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(_Stats), D, D]
        _lib.orc_pcg_joint_sr.argtypes = _lib.orc_pcg_joint.argtypes
        _lib.orc_pcg_async.argtypes = [C.c_int32, C.c_int32, C.c_int32, D, D, D, D, D, C.c_double,
                                       C.c_double, C.c_int32, C.c_int32, C.POINTER(C.c_int32),
                                       C.POINTER(_Stats)]
        _lib.orc_wrench.argtypes = [C.POINTER(_Grid), C.POINTER(_Cond), D, D]
        _lib.orc_sr_set_restart_threshold.argtypes = [C.c_double]
        _lib.orc_sr_set_restart_threshold.restype = None
        _lib.orc_sr_restarts.restype = C.c_int32
    return _lib


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _grid(g: dict) -> _Grid:
    return _Grid(int(g["n_theta"]), int(g["n_y"]), g["R_k"], g["R_c"], g["mu"], g["h_min"],
                 int(g.get("tex_n_theta", 0)), int(g.get("tex_n_y", 0)),
                 int(g.get("tex_band_rows", 0)), int(g.get("tex_fill_num", 1)),
                 int(g.get("tex_fill_den", 2)), g.get("tex_depth", 0.0))


def _cond(c) -> _Cond:
    c = np.asarray(c, dtype=np.float64).reshape(13)
    out = _Cond()
    for q in range(4):
        out.e[q] = c[q]
        out.edot[q] = c[4 + q]
    out.L_F, out.U_theta, out.U_y, out.p_in, out.p_out = (float(x) for x in c[8:13])
    return out


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle status {code} {msg}")
        self.code = code


def check_grid(g: dict) -> int:
    return lib().orc_check_grid(C.byref(_grid(g)))


def texture_mask(g: dict) -> np.ndarray:
    """T(i,j) for rows j=-1..n_y, shape (n_y+2, n_theta)."""
    gg = _grid(g)
    out = np.zeros((g["n_y"] + 2, g["n_theta"]), dtype=np.int8)
    for j in range(-1, g["n_y"] + 1):
        for i in range(g["n_theta"]):
            out[j + 1, i] = lib().orc_texture_mask(C.byref(gg), i, j)
    return out


def thickness(g: dict, cond):
    """h, dh/dt on rows -1..n_y, each (n_y+2, n_theta)."""
    nt, ny = g["n_theta"], g["n_y"]
    h = np.empty((ny + 2, nt))
    hd = np.empty((ny + 2, nt))
    bad = np.zeros(3)
    rc = lib().orc_thickness(C.byref(_grid(g)), C.byref(_cond(cond)), _ptr(h), _ptr(hd), _ptr(bad))
    if rc != OK:
        raise OracleError(rc, f"bad node i={bad[0]:.0f} j={bad[1]:.0f} h={bad[2]:.3e}")
    return h, hd


def assemble(g: dict, cond):
    """A_P, A_E, A_N, S for one condition, each (n_y, n_theta)."""
    nt, ny = g["n_theta"], g["n_y"]
    AP, AE, AN, S = (np.empty((ny, nt)) for _ in range(4))
    rc = lib().orc_assemble(C.byref(_grid(g)), C.byref(_cond(cond)), _ptr(AP), _ptr(AE), _ptr(AN), _ptr(S))
    if rc != OK:
        raise OracleError(rc)
    return AP, AE, AN, S


def assemble_joint(g: dict, conds):
    """Bands for K conditions stacked [K][n_y][n_theta] (Eq. 3.8 layout)."""
    parts = [assemble(g, c) for c in np.asarray(conds).reshape(-1, 13)]
    return tuple(np.ascontiguousarray(np.stack([p[q] for p in parts])) for q in range(4))


def spmv(AP, AE, AN, x):
    ny, nt = AP.shape
    y = np.empty_like(x)
    lib().orc_spmv(nt, ny, _ptr(AP), _ptr(AE), _ptr(AN), _ptr(np.ascontiguousarray(x)), _ptr(y))
    return y


def precond_apply(AP, AE, AN, r, precond="assor2", omega=1.8):
    ny, nt = AP.shape
    z = np.empty_like(r)
    lib().orc_precond_apply(nt, ny, _ptr(AP), _ptr(AE), _ptr(AN), PRECOND[precond], omega,
                            _ptr(np.ascontiguousarray(r)), _ptr(z))
    return z


def expand_dense(AP, AE, AN):
    ny, nt = AP.shape
    n = nt * ny
    A = np.empty((n, n))
    rc = lib().orc_expand_dense(nt, ny, _ptr(AP), _ptr(AE), _ptr(AN), _ptr(A))
    if rc != OK:
        raise OracleError(rc)
    return A


def assor2_dense(AP, AE, AN, omega):
    ny, nt = AP.shape
    n = nt * ny
    M = np.empty((n, n))
    rc = lib().orc_assor2_dense(nt, ny, _ptr(AP), _ptr(AE), _ptr(AN), omega, _ptr(M))
    if rc != OK:
        raise OracleError(rc)
    return M


def cholesky_solve(A, b):
    A = np.array(A, dtype=np.float64, order="C")
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    x = np.empty_like(b)
    rc = lib().orc_cholesky_solve(A.shape[0], _ptr(A), _ptr(b), _ptr(x))
    if rc != OK:
        raise OracleError(rc)
    return x


@dataclass
class SolveResult:
    p: np.ndarray
    iterations: int
    converged: bool
    status: int
    rel_residual: float
    true_rel_residual: float
    history: np.ndarray | None
    cond_rel: np.ndarray


def pcg_joint(AP, AE, AN, S, tol=1e-10, omega=1.8, precond="assor2", coupling="coupled",
              max_iter=100000, p0=None, history=False, schedule="table1") -> SolveResult:
    """O7: joint PCG over K stacked conditions (arrays [K][n_y][n_theta] or [n_y][n_theta]).
    schedule="table1": Table 1 with two reductions per iteration; "single": the same
    method with one (gamma, delta, r.r) reduction per iteration (orc_pcg_joint_sr)."""
    squeeze = AP.ndim == 2
    if squeeze:
        AP, AE, AN, S = (x[None] for x in (AP, AE, AN, S))
    K, ny, nt = AP.shape
    p = np.zeros((K, ny, nt)) if p0 is None else np.array(p0, dtype=np.float64).reshape(K, ny, nt)
    hist = np.zeros(max_iter + 1) if history else None
    cond_rel = np.zeros(K)
    st = _Stats()
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (AP, AE, AN, S)]
    fn = lib().orc_pcg_joint if schedule == "table1" else lib().orc_pcg_joint_sr
    rc = fn(nt, ny, K, *(_ptr(a) for a in arrs), _ptr(p), tol, omega,
                             PRECOND[precond], COUPLING[coupling], max_iter, int(p0 is not None),
                             C.byref(st), _ptr(hist), _ptr(cond_rel))
    if hist is not None:
        hist = hist[: st.iterations + 1]
    return SolveResult(p[0] if squeeze else p, st.iterations, bool(st.converged), rc,
                       st.rel_residual, st.true_rel_residual, hist, cond_rel)


def sr_restart_threshold(thresh: float) -> None:
    """Test hook of the single-reduction restart branch (R-A32): restart when the alpha
    denominator <= thresh * delta' (0 = the method itself)."""
    lib().orc_sr_set_restart_threshold(float(thresh))


def sr_restarts() -> int:
    """Restarts taken by the last single-reduction solve."""
    return int(lib().orc_sr_restarts())


def pcg_async(AP, AE, AN, S, tol=1e-10, omega=1.8, precond="assor2", max_iter=100000):
    K, ny, nt = AP.shape
    p = np.zeros((K, ny, nt))
    iters = (C.c_int32 * K)()
    st = _Stats()
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (AP, AE, AN, S)]
    rc = lib().orc_pcg_async(nt, ny, K, *(_ptr(a) for a in arrs), _ptr(p), tol, omega,
                             PRECOND[precond], max_iter, iters, C.byref(st))
    return p, np.array(list(iters)), rc


def wrench(g: dict, cond, p) -> np.ndarray:
    """O8: 12-vector [Fp_xyz, Mp_xyz, Fs_xyz, Ms_xyz] for one condition."""
    w = np.empty(12)
    pp = np.ascontiguousarray(p, dtype=np.float64).reshape(g["n_y"], g["n_theta"])
    rc = lib().orc_wrench(C.byref(_grid(g)), C.byref(_cond(cond)), _ptr(pp), _ptr(w))
    if rc != OK:
        raise OracleError(rc)
    return w


def joint_step(g: dict, conds, tol=1e-10, omega=1.8, precond="assor2", coupling="coupled",
               max_iter=100000):
    """One Picard-step joint analysis (GMAF steps I-III): assemble all K
    conditions, solve the joint system, integrate the K wrenches."""
    conds = np.asarray(conds, dtype=np.float64).reshape(-1, 13)
    AP, AE, AN, S = assemble_joint(g, conds)
    res = pcg_joint(AP, AE, AN, S, tol=tol, omega=omega, precond=precond, coupling=coupling,
                    max_iter=max_iter)
    W = np.stack([wrench(g, conds[k], res.p[k]) for k in range(conds.shape[0])])
    return res, W
