"""paper_2511_06824_b200 -- B200-native hot path of GMAF (arXiv 2511.06824).

Thin ctypes binding of ``libgmaf.so`` (C ABI in ``include/gmaf.h``).  This module
only marshals arguments: every step of the path (thickness, assembly, PCG-ASSOR,
quadrature) runs in the library's sm_100a kernels.  PyTorch is used for the device
workspace and the CUDA stream only.  There is no CPU fallback: if the library is not
built or no CUDA device is present, the calls raise.

Low-level functions carry the ABI names (``gmaf_create``, ``gmaf_thickness``,
``gmaf_assemble``, ``gmaf_solve``, ``gmaf_integrate``, ...); ``JointSolver`` wraps
them for one Picard step of K working conditions (GMAF steps I-III).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgmaf.so")   # the in-tree product library, nothing else

STATUS = {0: "OK", -1: "INVALID_ARG", -2: "INVALID_MESH", -3: "MESH_TOO_COARSE",
          -4: "NONPOSITIVE_THICKNESS", -5: "BREAKDOWN", -6: "NO_CONVERGENCE", -7: "STATE",
          -8: "WORKSPACE", -9: "CUDA", -10: "NCCL", -11: "SINGULAR"}
PRECOND = {"none": 0, "jacobi": 1, "assor2": 2, "assor1": 3}
COUPLING = {"coupled": 0, "lockstep": 1, "async": 2}
FIELD = {"p": 0, "h": 1, "hdot": 2, "AP": 3, "AE": 4, "AN": 5, "S": 6, "r": 7}


class gmaf_grid(C.Structure):
    _fields_ = [("n_theta", C.c_int32), ("n_y", C.c_int32), ("R_k", C.c_double), ("R_c", C.c_double),
                ("mu", C.c_double), ("h_min", C.c_double), ("tex_n_theta", C.c_int32),
                ("tex_n_y", C.c_int32), ("tex_band_rows", C.c_int32), ("tex_fill_num", C.c_int32),
                ("tex_fill_den", C.c_int32), ("tex_depth", C.c_double)]


class gmaf_condition(C.Structure):
    _fields_ = [("e", C.c_double * 4), ("edot", C.c_double * 4), ("L_F", C.c_double),
                ("U_theta", C.c_double), ("U_y", C.c_double), ("p_in", C.c_double),
                ("p_out", C.c_double)]


class gmaf_dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("shard", C.c_int32)]


class gmaf_solve_stats(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("status", C.c_int32),
                ("precond", C.c_int32), ("schedule", C.c_int32), ("pad", C.c_int32),
                ("rel_residual", C.c_double),
                ("true_rel_residual", C.c_double), ("solve_ms", C.c_double)]


class gmaf_kernel_timing(C.Structure):
    _fields_ = [("name", C.c_char * 24), ("launches", C.c_int64), ("total_ms", C.c_double),
                ("bytes_per_launch", C.c_double)]


class gmaf_tiles(C.Structure):
    _fields_ = [("tw", C.c_int32), ("th", C.c_int32), ("n_strips", C.c_int32), ("n_chunks", C.c_int32),
                ("n_ctas", C.c_int32), ("schedule", C.c_int32), ("persistent", C.c_int32), ("pad", C.c_int32)]


class gmaf_pump(C.Structure):
    _fields_ = [("m_k", C.c_double), ("m_G", C.c_double), ("R_b", C.c_double), ("beta", C.c_double),
                ("omega_s", C.c_double), ("R_k", C.c_double)]


class gmaf_picard_iterate(C.Structure):
    _fields_ = [("F", C.c_double * 4), ("F_oil", C.c_double * 4), ("F_ext", C.c_double * 4),
                ("F_inertial", C.c_double * 4), ("J_e", C.c_double * 16), ("J_edot", C.c_double * 16),
                ("e_next", C.c_double * 4), ("edot_next", C.c_double * 4), ("wrench", C.c_double * 12),
                ("pcg_iterations", C.c_int32), ("pad", C.c_int32)]


PICARD_SCHEME = {"simplified": 0, "general": 1}

_SCHED_NAME = {0: "table1", 1: "single"}


class GmafError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"gmaf {STATUS.get(code, code)} ({code}): {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load libgmaf.so (in-tree).  Raises if it is missing -- no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.gmaf_workspace_bytes.restype = C.c_size_t
        L.gmaf_workspace_bytes.argtypes = [C.POINTER(gmaf_grid), C.c_int32, C.POINTER(gmaf_dist)]
        L.gmaf_workspace_bytes_m.restype = C.c_size_t
        L.gmaf_workspace_bytes_m.argtypes = [C.POINTER(gmaf_grid), C.c_int32, C.c_int32, C.POINTER(gmaf_dist)]
        L.gmaf_create.argtypes = [C.POINTER(gmaf_grid), C.c_int32, C.POINTER(gmaf_dist), P, C.c_size_t, P,
                                  C.POINTER(P)]
        L.gmaf_destroy.argtypes = [P]
        L.gmaf_thickness.argtypes = [P, C.POINTER(gmaf_condition)]
        L.gmaf_assemble.argtypes = [P]
        L.gmaf_solve.argtypes = [P, C.c_double, C.c_double, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                 C.POINTER(gmaf_solve_stats), C.POINTER(C.c_double)]
        L.gmaf_solve_fixed.argtypes = [P, C.c_double, C.c_int32, C.c_int32, C.POINTER(gmaf_solve_stats)]
        L.gmaf_integrate.argtypes = [P, C.POINTER(C.c_double)]
        L.gmaf_get.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
        L.gmaf_field_ptr.argtypes = [P, C.c_int32, C.c_int32, C.POINTER(P)]
        L.gmaf_kernel_times.argtypes = [P, C.POINTER(gmaf_kernel_timing), C.c_int32, C.POINTER(C.c_int32)]
        L.gmaf_reset_kernel_times.argtypes = [P]
        L.gmaf_set_schedule.argtypes = [P, C.c_int32]
        L.gmaf_nccl_unique_id.argtypes = [P]
        L.gmaf_cond_iterations.argtypes = [P, C.POINTER(C.c_int32)]
        L.gmaf_general_forces.argtypes = [C.POINTER(gmaf_pump), C.POINTER(gmaf_condition), C.c_double,
                                          C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
        L.gmaf_picard_iteration.argtypes = [P, C.POINTER(gmaf_pump), C.POINTER(gmaf_condition), C.c_double,
                                            C.c_double, C.c_int32, C.c_double, C.c_double, C.c_double,
                                            C.c_double, C.c_int32, C.c_int32, C.POINTER(gmaf_picard_iterate)]
        L.gmaf_picard_step.argtypes = [P, C.POINTER(gmaf_pump), C.POINTER(gmaf_condition), C.c_double,
                                       C.c_double, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_int32,
                                       C.c_double, C.c_double, C.c_int32, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int32)]
        L.gmaf_p2p_handle.argtypes = [P, P]
        L.gmaf_p2p_connect.argtypes = [P, P]
        L.gmaf_slab.argtypes = [P, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.gmaf_tile_config.argtypes = [P, C.POINTER(gmaf_tiles)]
        L.gmaf_cta_arrivals.argtypes = [P, C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_int32)]
        L.gmaf_slab_rows.argtypes = [C.c_int32, C.c_int32, C.c_int32] + [C.POINTER(C.c_int32)] * 4
        L.gmaf_last_error.restype = C.c_char_p
        L.gmaf_last_error.argtypes = [P]
        L.gmaf_version.restype = C.c_char_p
        for name in ("gmaf_create", "gmaf_destroy", "gmaf_thickness", "gmaf_assemble", "gmaf_solve",
                     "gmaf_solve_fixed", "gmaf_integrate", "gmaf_get", "gmaf_field_ptr",
                     "gmaf_kernel_times", "gmaf_reset_kernel_times", "gmaf_set_schedule",
                     "gmaf_nccl_unique_id", "gmaf_cond_iterations", "gmaf_general_forces",
                     "gmaf_picard_iteration", "gmaf_picard_step", "gmaf_p2p_handle", "gmaf_p2p_connect",
                     "gmaf_slab", "gmaf_slab_rows", "gmaf_tile_config", "gmaf_cta_arrivals"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


ABI_SYMBOLS = ("gmaf_workspace_bytes", "gmaf_workspace_bytes_m", "gmaf_create", "gmaf_destroy", "gmaf_thickness", "gmaf_assemble",
               "gmaf_solve", "gmaf_solve_fixed", "gmaf_integrate", "gmaf_get", "gmaf_field_ptr",
               "gmaf_kernel_times", "gmaf_reset_kernel_times", "gmaf_set_schedule", "gmaf_nccl_unique_id",
               "gmaf_cond_iterations", "gmaf_general_forces", "gmaf_picard_iteration", "gmaf_picard_step",
               "gmaf_p2p_handle", "gmaf_p2p_connect", "gmaf_slab", "gmaf_slab_rows", "gmaf_tile_config",
               "gmaf_cta_arrivals", "gmaf_last_error", "gmaf_version")
SCHEDULE = {"table1": 0, "single": 1}


def make_grid(g: dict) -> gmaf_grid:
    return gmaf_grid(int(g["n_theta"]), int(g["n_y"]), g["R_k"], g["R_c"], g["mu"], g["h_min"],
                     int(g.get("tex_n_theta", 0)), int(g.get("tex_n_y", 0)), int(g.get("tex_band_rows", 0)),
                     int(g.get("tex_fill_num", 1)), int(g.get("tex_fill_den", 2)), g.get("tex_depth", 0.0))


def make_conditions(conds) -> C.Array:
    conds = np.asarray(conds, dtype=np.float64).reshape(-1, 13)
    arr = (gmaf_condition * conds.shape[0])()
    for k, c in enumerate(conds):
        for q in range(4):
            arr[k].e[q] = c[q]
            arr[k].edot[q] = c[4 + q]
        arr[k].L_F, arr[k].U_theta, arr[k].U_y, arr[k].p_in, arr[k].p_out = (float(x) for x in c[8:13])
    return arr


def make_pump(pump: dict) -> gmaf_pump:
    """gmaf_pump from a dict with m_k, m_G, R_b, beta (rad), omega_s (rad/s), R_k."""
    return gmaf_pump(pump["m_k"], pump["m_G"], pump["R_b"], pump["beta"], pump["omega_s"], pump["R_k"])


def general_forces(pump: dict, cond, phi: float, wrench12=None):
    """Generalized forces (Eq. 2.11) of one state: (F_oil, F_ext, F_inertial) as numpy 4-vectors
    (F_oil is None without a wrench).  DESIGN.md R-A28..R-A30; host only."""
    c = make_conditions(np.asarray(cond, dtype=np.float64).reshape(1, 13))
    fo, fe, fi = (C.c_double * 4)(), (C.c_double * 4)(), (C.c_double * 4)()
    w = None
    if wrench12 is not None:
        w = (C.c_double * 12)(*np.asarray(wrench12, dtype=np.float64).ravel())
    code = lib().gmaf_general_forces(C.byref(make_pump(pump)), c, float(phi), w, fo if w is not None else None,
                                     fe, fi)
    _check(None, code)
    return (np.array(fo[:]) if w is not None else None), np.array(fe[:]), np.array(fi[:])


def _check(ctx, code: int):
    if code != 0:
        msg = lib().gmaf_last_error(ctx).decode()   # NULL ctx: the last failed create
        raise GmafError(code, msg)


# ---- ABI-named thin wrappers ------------------------------------------------------------

def gmaf_nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (make it on rank 0, broadcast it to the others)."""
    buf = (C.c_char * 128)()
    _check(None, lib().gmaf_nccl_unique_id(buf))
    return bytes(buf)


SHARD = {"conditions": 1, "rows": 2}   # peer-to-peer modes (include/gmaf.h GMAF_SHARD_*_P2P)


def make_dist(rank: int, world: int, uid: bytes | None, p2p: bool = False, shard: str = "conditions"):
    if p2p:   # peer-to-peer sharding: no NCCL id (connect with p2p_connect)
        return gmaf_dist(int(rank), int(world), None, SHARD[shard]), None
    if uid is None:
        return None, None
    keep = C.create_string_buffer(uid, 128)
    return gmaf_dist(int(rank), int(world), C.cast(keep, C.c_void_p), 0), keep


def gmaf_slab_rows(n_y: int, world: int, rank: int) -> tuple[int, int, int, int]:
    """Row slab of `rank` (include/gmaf.h gmaf_slab_rows): own rows (y0, y1), stored rows (yb, ye)."""
    v = [C.c_int32() for _ in range(4)]
    _check(None, lib().gmaf_slab_rows(int(n_y), int(world), int(rank), *(C.byref(x) for x in v)))
    return tuple(int(x.value) for x in v)


def gmaf_workspace_bytes(grid: gmaf_grid, K: int, dist: gmaf_dist | None = None) -> int:
    return int(lib().gmaf_workspace_bytes(C.byref(grid), int(K), C.byref(dist) if dist else None))


def gmaf_workspace_bytes_m(grid: gmaf_grid, K: int, max_matrices: int, dist: gmaf_dist | None = None) -> int:
    return int(lib().gmaf_workspace_bytes_m(C.byref(grid), int(K), int(max_matrices),
                                            C.byref(dist) if dist else None))


def gmaf_create(grid: gmaf_grid, K: int, d_workspace: int, ws_bytes: int, stream: int,
                dist: gmaf_dist | None = None) -> C.c_void_p:
    ctx = C.c_void_p()
    _check(None, lib().gmaf_create(C.byref(grid), int(K), C.byref(dist) if dist else None,
                                   C.c_void_p(d_workspace), ws_bytes, C.c_void_p(stream), C.byref(ctx)))
    return ctx


def gmaf_thickness(ctx, conds_arr) -> None:
    _check(ctx, lib().gmaf_thickness(ctx, conds_arr))


def gmaf_assemble(ctx) -> None:
    _check(ctx, lib().gmaf_assemble(ctx))


def gmaf_solve(ctx, tol, omega, precond, coupling, max_iter, warm, K):
    st = gmaf_solve_stats()
    cr = (C.c_double * K)()
    code = lib().gmaf_solve(ctx, float(tol), float(omega), int(precond), int(coupling), int(max_iter),
                            int(warm), C.byref(st), cr)
    return code, st, np.array(list(cr))


def gmaf_integrate(ctx, K) -> np.ndarray:
    w = np.empty(K * 12)
    _check(ctx, lib().gmaf_integrate(ctx, w.ctypes.data_as(C.POINTER(C.c_double))))
    return w.reshape(K, 12)


def gmaf_destroy(ctx) -> None:
    lib().gmaf_destroy(ctx)


@dataclass
class SolveStats:
    schedule: str
    iterations: int
    converged: bool
    status: int
    rel_residual: float
    true_rel_residual: float
    solve_ms: float
    cond_rel: np.ndarray


class JointSolver:
    """One context: K working conditions on one mesh (Eq. 3.7 joint system)."""

    def __init__(self, grid: dict, K: int, device: int | str = 0, stream=None, rank: int = 0,
                 world: int = 1, nccl_uid: bytes | None = None, p2p: bool = False, shard: str = "conditions",
                 max_matrices: int | None = None):
        """K = total conditions.  With nccl_uid the K conditions are sharded over `world` ranks
        (condition sharding with one NCCL allgather per iteration, include/gmaf.h gmaf_dist); with
        p2p=True they are sharded peer to peer (the gathers fused into the iteration kernel over
        IPC-mapped peer memory) -- call p2p_handle() / p2p_connect() before the first solve, or
        paper_2511_06824_b200.dist.connect_p2p(solver).  shard="rows" (implies p2p) splits the rows
        of all K conditions into contiguous slabs instead (GMAF_SHARD_ROWS_P2P): get() then fills
        only this rank's rows [y0, y1) = self.slab."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("JointSolver needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.grid_dict = dict(grid)
        self.grid = make_grid(grid)
        self.K = int(K)
        self.n_theta, self.n_y = int(grid["n_theta"]), int(grid["n_y"])
        if shard == "rows":
            p2p = True
        self.shard = shard
        self.dist, self._uid_buf = make_dist(rank, world, nccl_uid, p2p=p2p and world >= 1, shard=shard)
        self.rank, self.world = int(rank), int(world)
        # max_matrices: distinct coefficient sets to store (the 9 FD conditions of one state need 5;
        # None = K, the worst case)
        nbytes = (gmaf_workspace_bytes(self.grid, self.K, self.dist) if max_matrices is None else
                  gmaf_workspace_bytes_m(self.grid, self.K, int(max_matrices), self.dist))
        if nbytes == 0:
            raise GmafError(-1, "invalid grid for workspace sizing")
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            # 256-byte alignment: torch's caching allocator returns >= 512-byte aligned blocks
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.ctx = gmaf_create(self.grid, self.K, self.workspace.data_ptr(), nbytes, self.stream.cuda_stream,
                               self.dist)
        y0, y1 = C.c_int32(), C.c_int32()
        _check(self.ctx, lib().gmaf_slab(self.ctx, C.byref(y0), C.byref(y1)))
        self.slab = (int(y0.value), int(y1.value))   # own rows (all rows unless shard="rows")

    def p2p_handle(self) -> bytes:
        """This rank's 64-byte CUDA IPC handle of its exchange buffer (peer-to-peer mode)."""
        buf = (C.c_char * 64)()
        _check(self.ctx, lib().gmaf_p2p_handle(self.ctx, buf))
        return bytes(buf)

    def p2p_connect(self, handles: list[bytes]):
        """Open every rank's exchange buffer (handles in rank order, world x 64 bytes)."""
        blob = b"".join(handles)
        assert len(blob) == 64 * self.world
        _check(self.ctx, lib().gmaf_p2p_connect(self.ctx, C.create_string_buffer(blob, len(blob))))

    def close(self):
        if getattr(self, "ctx", None):
            gmaf_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- the hot path ------------------------------------------------------------------
    def thickness(self, conds) -> None:
        conds = np.asarray(conds, dtype=np.float64).reshape(-1, 13)
        if conds.shape[0] != self.K:
            raise ValueError(f"expected {self.K} conditions, got {conds.shape[0]}")
        gmaf_thickness(self.ctx, make_conditions(conds))

    def assemble(self) -> None:
        gmaf_assemble(self.ctx)

    def solve(self, tol=1e-10, omega=1.8, precond="assor2", coupling="coupled", max_iter=200000,
              warm=False, raise_on_error=True) -> SolveStats:
        code, st, cr = gmaf_solve(self.ctx, tol, omega, PRECOND[precond], COUPLING[coupling], max_iter,
                                  warm, self.K)
        if code != 0 and raise_on_error:
            _check(self.ctx, code)
        return SolveStats(_SCHED_NAME[st.schedule], st.iterations, bool(st.converged), st.status,
                          st.rel_residual, st.true_rel_residual, st.solve_ms, cr)

    def solve_fixed(self, n_iter: int, omega=1.6, precond="assor2") -> SolveStats:
        st = gmaf_solve_stats()
        _check(self.ctx, lib().gmaf_solve_fixed(self.ctx, float(omega), PRECOND[precond], int(n_iter),
                                                 C.byref(st)))
        return SolveStats(_SCHED_NAME[st.schedule], st.iterations, bool(st.converged), st.status,
                          st.rel_residual, st.true_rel_residual, st.solve_ms, np.zeros(self.K))

    def tile_config(self) -> dict:
        """Launch configuration of the iteration kernel (include/gmaf.h gmaf_tile_config)."""
        t = gmaf_tiles()
        _check(self.ctx, lib().gmaf_tile_config(self.ctx, C.byref(t)))
        return {"tw": t.tw, "th": t.th, "n_strips": t.n_strips, "n_chunks": t.n_chunks, "n_ctas": t.n_ctas,
                "schedule": _SCHED_NAME[t.schedule], "persistent": bool(t.persistent)}

    def cta_arrivals(self) -> np.ndarray:
        """[iteration][CTA] %globaltimer ns of each CTA's arrival at the persistent kernel's grid
        barrier (first 32 iterations of the last solve; needs GMAF_DIAG at create; else empty)."""
        t = self.tile_config()
        n = 32 * t["n_ctas"]
        buf = (C.c_uint64 * n)()
        cnt = C.c_int32()
        _check(self.ctx, lib().gmaf_cta_arrivals(self.ctx, buf, n, C.byref(cnt)))
        return np.array(list(buf)[: cnt.value], dtype=np.uint64).reshape(-1, t["n_ctas"]) if cnt.value else \
            np.zeros((0, t["n_ctas"]), dtype=np.uint64)

    def cond_iterations(self) -> np.ndarray:
        """Per-condition iteration counts of the last solve (the freeze iteration under 'async')."""
        out = (C.c_int32 * self.K)()
        _check(self.ctx, lib().gmaf_cond_iterations(self.ctx, out))
        return np.array(list(out))

    def set_schedule(self, schedule: str) -> None:
        """'single' (one kernel + one reduction per iteration, default) or 'table1'."""
        _check(self.ctx, lib().gmaf_set_schedule(self.ctx, SCHEDULE[schedule]))

    def integrate(self) -> np.ndarray:
        return gmaf_integrate(self.ctx, self.K)

    def step(self, conds, tol=1e-10, omega=1.8, precond="assor2", coupling="coupled",
             max_iter=200000, warm=False):
        """One joint Picard-step analysis: thickness -> assemble -> solve -> integrate."""
        self.thickness(conds)
        self.assemble()
        st = self.solve(tol=tol, omega=omega, precond=precond, coupling=coupling, max_iter=max_iter,
                        warm=warm)
        return st, self.integrate()

    # -- Picard driver (Sec. 2.3; include/gmaf.h) ----------------------------------------
    def picard_iteration(self, pump: dict, state, phi: float, dt: float, scheme="general", de=1e-9,
                         dedot=1e-8, tol=1e-10, omega=1.6, max_iter=200000, warm=False) -> dict:
        """One Picard iteration around `state` (13 numbers: e, edot, L_F, U_theta, U_y, p_in,
        p_out): the 9 joint solves, general forces, FD Jacobians and the update."""
        c = make_conditions(np.asarray(state, dtype=np.float64).reshape(1, 13))
        it = gmaf_picard_iterate()
        _check(self.ctx, lib().gmaf_picard_iteration(self.ctx, C.byref(make_pump(pump)), c, float(phi),
                                                     float(dt), PICARD_SCHEME[scheme], float(de), float(dedot),
                                                     float(tol), float(omega), int(max_iter), int(bool(warm)),
                                                     C.byref(it)))
        return dict(F=np.array(it.F[:]), F_oil=np.array(it.F_oil[:]), F_ext=np.array(it.F_ext[:]),
                    F_inertial=np.array(it.F_inertial[:]), J_e=np.array(it.J_e[:]).reshape(4, 4),
                    J_edot=np.array(it.J_edot[:]).reshape(4, 4), e_next=np.array(it.e_next[:]),
                    edot_next=np.array(it.edot_next[:]), wrench=np.array(it.wrench[:]),
                    pcg_iterations=int(it.pcg_iterations))

    def picard_step(self, pump: dict, state, phi: float, dt: float, scheme="general", de=1e-9, dedot=1e-8,
                    eps_dyn=1e-3, max_picard=20, tol=1e-10, omega=1.6, max_iter=200000,
                    raise_on_error=True):
        """One time step of the Picard march from (e_l, edot_l) with the load case of t_l + dt.
        Returns (new state (13,), n_picard, residual, pcg_iterations, status)."""
        c = make_conditions(np.asarray(state, dtype=np.float64).reshape(1, 13))
        n, res, pcg = C.c_int32(), C.c_double(), C.c_int32()
        code = lib().gmaf_picard_step(self.ctx, C.byref(make_pump(pump)), c, float(phi), float(dt),
                                      PICARD_SCHEME[scheme], float(de), float(dedot), float(eps_dyn),
                                      int(max_picard), float(tol), float(omega), int(max_iter), C.byref(n),
                                      C.byref(res), C.byref(pcg))
        if raise_on_error and code != 0:
            _check(self.ctx, code)
        new = np.array(list(c[0].e) + list(c[0].edot) + [c[0].L_F, c[0].U_theta, c[0].U_y, c[0].p_in,
                                                         c[0].p_out])
        return new, int(n.value), float(res.value), int(pcg.value), code

    # -- readback ----------------------------------------------------------------------
    def get(self, field: str, k: int) -> np.ndarray:
        rows = self.n_y + 2 if field in ("h", "hdot") else self.n_y
        out = np.zeros((rows, self.n_theta))   # a row slab fills only its own rows
        _check(self.ctx, lib().gmaf_get(self.ctx, FIELD[field], int(k),
                                        out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def field_tensor(self, field: str, k: int):
        """Zero-copy torch view of a device field of condition k."""
        ptr = C.c_void_p()
        _check(self.ctx, lib().gmaf_field_ptr(self.ctx, FIELD[field], int(k), C.byref(ptr)))
        base = self.workspace.data_ptr()
        off = (ptr.value - base) // 8
        rows = self.slab[1] - self.slab[0]   # own rows (all rows unless shard="rows")
        n = self.n_theta * rows
        return self.workspace.view(self.torch.float64)[off:off + n].view(rows, self.n_theta)

    def kernel_times(self) -> list[dict]:
        arr = (gmaf_kernel_timing * 16)()
        cnt = C.c_int32()
        _check(self.ctx, lib().gmaf_kernel_times(self.ctx, arr, 16, C.byref(cnt)))
        return [dict(name=arr[i].name.decode(), launches=int(arr[i].launches), total_ms=arr[i].total_ms,
                     bytes_per_launch=arr[i].bytes_per_launch) for i in range(cnt.value)]

    def reset_kernel_times(self) -> None:
        _check(self.ctx, lib().gmaf_reset_kernel_times(self.ctx))
