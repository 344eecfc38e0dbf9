"""Thin ctypes binding of the C ABI in include/diffreg.h (argument marshalling only).

Every function here forwards to the CUDA library `libdiffreg.so`; no step of the hot path runs in
Python.  Fields are torch tensors (CUDA, or CPU for the host-buffer entry points), float32 by default
or float64 for DR_FP64 contexts, shaped (N3, N2, N1) for scalars and (3, N3, N2, N1) for vectors.
Importing this module never falls back to anything: if the library is missing or cannot be loaded,
`lib()` raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# DR_CHECK=1 selects the bounds-checked debug build (paper_1608_03630_b200/build.py with DR_CHECK=1)
LIB_PATH = os.path.join(_PKG, "libdiffreg_check.so" if os.environ.get("DR_CHECK", "0") == "1" else "libdiffreg.so")
if os.environ.get("DR_LIB_VARIANT"):  # A/B builds of the same sources (build.py --variant NAME -D...)
    LIB_PATH = os.path.join(_PKG, f"libdiffreg_{os.environ['DR_LIB_VARIANT']}.so")

DR_OK, DR_ERR_ARG, DR_ERR_GRID, DR_ERR_PARAM, DR_ERR_ORDER, DR_ERR_CUDA, DR_ERR_NCCL, DR_ERR_OOM, \
    DR_ERR_NONFINITE, DR_ERR_PLAN = range(10)
DR_REG_H1, DR_REG_H2 = 1, 2
DR_ISOCHORIC, DR_FP64, DR_FULL_NEWTON, DR_CHECK_FINITE = 1, 2, 4, 8
DR_OP_GRAD, DR_OP_DIV, DR_OP_REG, DR_OP_PRECOND, DR_OP_LERAY = range(5)
(DR_FIELD_STATE, DR_FIELD_STATE_GRAD, DR_FIELD_ADJOINT, DR_FIELD_INC_STATE, DR_FIELD_INC_ADJOINT,
 DR_FIELD_BTILDE, DR_FIELD_MULTIPLIER, DR_FIELD_VELOCITY) = range(8)

# every symbol include/diffreg.h declares (checked by tests/test_abi.py)
EXPORTS = ["dr_workspace_bytes", "dr_create", "dr_destroy", "dr_set_images", "dr_set_velocity",
           "dr_forward_solve", "dr_adjoint_solve", "dr_hessian_matvec", "dr_precond_apply", "dr_sync",
           "dr_last_error", "dr_status_string", "dr_op_spectral", "dr_op_interp", "dr_get_departure",
           "dr_get_field", "dr_profile_enable", "dr_profile_reset", "dr_profile_only", "dr_profile_count", "dr_profile_entry",
           "dr_nccl_get_unique_id", "dr_comm_create_nccl", "dr_hub_create", "dr_hub_destroy",
           "dr_comm_create_loopback", "dr_comm_destroy", "dr_slab", "dr_workspace_bytes_dist", "dr_create_dist",
           "dr_gradient", "dr_objective", "dr_pcg", "dr_deformation", "dr_solve", "dr_comm_selftest",
           "dr_peer_export", "dr_peer_import"]


class dr_config(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32 * 3), ("nt", ctypes.c_int32), ("reg", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("beta", ctypes.c_double), ("ghost_lo", ctypes.c_int32),
                ("ghost_hi", ctypes.c_int32)]


class dr_solve_opts(ctypes.Structure):
    _fields_ = [("gtol", ctypes.c_double), ("max_newton", ctypes.c_int32), ("max_krylov", ctypes.c_int32),
                ("c1", ctypes.c_double), ("shrink", ctypes.c_double), ("max_backtracks", ctypes.c_int32)]


class dr_solve_report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("matvecs", ctypes.c_int32), ("reason", ctypes.c_int32),
                ("J0", ctypes.c_double), ("J", ctypes.c_double), ("g0", ctypes.c_double), ("g", ctypes.c_double),
                ("history", ctypes.POINTER(ctypes.c_double)), ("history_len", ctypes.c_int32)]


SOLVE_REASONS = {0: "converged", 1: "max_newton", 2: "line_search_failed"}


class DiffRegError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libdiffreg.so (raises if absent: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run __graft_entry__.build() or paper_1608_03630_b200/build.py")
        if "DR_NCCL_LIB" not in os.environ:  # torch's bundled NCCL for the multi-GPU communicator (dlopen'ed lazily)
            try:
                import nvidia.nccl as _nccl
                cand = os.path.join(list(_nccl.__path__)[0], "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["DR_NCCL_LIB"] = cand
            except ImportError:
                pass
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        L.dr_workspace_bytes.argtypes = [ctypes.POINTER(dr_config)]
        L.dr_workspace_bytes.restype = ctypes.c_size_t
        L.dr_create.argtypes = [ctypes.POINTER(dr_config), vp, ctypes.c_size_t, vp, ctypes.POINTER(vp)]
        for name, args in [("dr_destroy", [vp]), ("dr_set_images", [vp, vp, vp]), ("dr_set_velocity", [vp, vp]),
                           ("dr_forward_solve", [vp, vp]), ("dr_adjoint_solve", [vp, vp]),
                           ("dr_hessian_matvec", [vp, vp, vp]), ("dr_precond_apply", [vp, vp, vp]),
                           ("dr_sync", [vp]), ("dr_op_spectral", [vp, i32, vp, vp]),
                           ("dr_op_interp", [vp, vp, i64, vp, vp]), ("dr_get_departure", [vp, i32, vp]),
                           ("dr_get_field", [vp, i32, i32, vp]), ("dr_profile_enable", [vp, i32]),
                           ("dr_profile_reset", [vp]),
                           ("dr_profile_only", [vp, ctypes.c_char_p]),
                           ("dr_profile_count", [vp, ctypes.POINTER(i32), ctypes.POINTER(i64)]),
                           ("dr_profile_entry", [vp, i32, ctypes.c_char_p, i32, ctypes.POINTER(i64),
                                                 ctypes.POINTER(ctypes.c_double)])]:
            getattr(L, name).argtypes = args
            getattr(L, name).restype = ctypes.c_int
        L.dr_create.restype = ctypes.c_int
        L.dr_workspace_bytes_dist.argtypes = [ctypes.POINTER(dr_config), i32]
        L.dr_workspace_bytes_dist.restype = ctypes.c_size_t
        L.dr_create_dist.argtypes = [ctypes.POINTER(dr_config), vp, vp, ctypes.c_size_t, vp, ctypes.POINTER(vp)]
        L.dr_create_dist.restype = ctypes.c_int
        for name, args in [("dr_comm_selftest", [vp, vp, ctypes.POINTER(i32)]),
                           ("dr_deformation", [vp, vp, vp, ctypes.POINTER(ctypes.c_double),
                                               ctypes.POINTER(ctypes.c_double)]),
                           ("dr_solve", [vp, vp, ctypes.POINTER(dr_solve_opts), ctypes.POINTER(dr_solve_report)]),
                           ("dr_pcg", [vp, vp, vp, ctypes.c_double, i32, ctypes.POINTER(i32),
                                       ctypes.POINTER(ctypes.c_double)]),
                           ("dr_gradient", [vp, vp]),
                           ("dr_peer_export", [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]),
                           ("dr_peer_import", [vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]),
                           ("dr_objective", [vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
                           ("dr_nccl_get_unique_id", [ctypes.c_char_p]),
                           ("dr_comm_create_nccl", [ctypes.c_char_p, i32, i32, ctypes.POINTER(vp)]),
                           ("dr_hub_create", [i32, ctypes.POINTER(vp)]), ("dr_hub_destroy", [vp]),
                           ("dr_comm_create_loopback", [vp, i32, ctypes.POINTER(vp)]), ("dr_comm_destroy", [vp]),
                           ("dr_slab", [ctypes.POINTER(dr_config), i32, i32, ctypes.POINTER(i32),
                                        ctypes.POINTER(i32)])]:
            getattr(L, name).argtypes = args
            getattr(L, name).restype = ctypes.c_int
        L.dr_last_error.argtypes = [vp]
        L.dr_last_error.restype = ctypes.c_char_p
        L.dr_status_string.argtypes = [ctypes.c_int]
        L.dr_status_string.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


@dataclass
class Config:
    n: tuple  # (N1, N2, N3)
    nt: int = 4
    reg: int = DR_REG_H2
    beta: float = 1e-2
    isochoric: bool = False
    fp64: bool = False
    newton: bool = False  # NEXT-3: full-Newton Hessian (default Gauss-Newton)
    ghost_lo: int = 0  # slab ghost planes (multi-GPU; 0 -> library default 4 / 5)
    ghost_hi: int = 0
    check_finite: bool = False  # DR_CHECK_FINITE: NaN / Inf inputs -> DR_ERR_NONFINITE (synchronising scan)

    def c(self) -> dr_config:
        n = (self.n,) * 3 if isinstance(self.n, int) else tuple(self.n)
        flags = (DR_ISOCHORIC if self.isochoric else 0) | (DR_FP64 if self.fp64 else 0) | \
            (DR_FULL_NEWTON if self.newton else 0) | (DR_CHECK_FINITE if self.check_finite else 0)
        cfg = dr_config()
        cfg.n[:] = list(n)
        cfg.nt, cfg.reg, cfg.flags, cfg.beta = self.nt, self.reg, flags, self.beta
        cfg.ghost_lo, cfg.ghost_hi = self.ghost_lo, self.ghost_hi
        return cfg

    @property
    def dtype(self):
        return torch.float64 if self.fp64 else torch.float32

    @property
    def shape(self):
        n = (self.n,) * 3 if isinstance(self.n, int) else tuple(self.n)
        return (n[2], n[1], n[0])


def dr_workspace_bytes(cfg: Config) -> int:
    c = cfg.c()
    return int(lib().dr_workspace_bytes(ctypes.byref(c)))


def dr_workspace_bytes_dist(cfg: Config, nranks: int) -> int:
    c = cfg.c()
    return int(lib().dr_workspace_bytes_dist(ctypes.byref(c), nranks))


def dr_slab(cfg: Config, nranks: int, rank: int) -> tuple[int, int]:
    """(z0, nz): the x3 planes [z0, z0 + nz) rank `rank` of `nranks` owns (host-only, no GPU)."""
    c = cfg.c()
    z0, nz = ctypes.c_int(), ctypes.c_int()
    st = lib().dr_slab(ctypes.byref(c), nranks, rank, ctypes.byref(z0), ctypes.byref(nz))
    if st != DR_OK:
        raise DiffRegError(st, lib().dr_status_string(st).decode())
    return z0.value, nz.value


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().dr_nccl_get_unique_id(buf)
    if st != DR_OK:
        raise DiffRegError(st, lib().dr_status_string(st).decode())
    return buf.raw


class Comm:
    """A communicator of the slab path: NCCL (one process per GPU) or loopback (virtual ranks of one
    process, see Hub).  Must outlive the contexts that use it."""

    def __init__(self, handle, rank: int, size: int, keep=None):
        self.h, self.rank, self.size, self._keep = handle, rank, size, keep

    @classmethod
    def nccl(cls, uid: bytes, rank: int, size: int) -> "Comm":
        h = ctypes.c_void_p()
        st = lib().dr_comm_create_nccl(uid, rank, size, ctypes.byref(h))
        if st != DR_OK:
            raise DiffRegError(st, lib().dr_status_string(st).decode())
        return cls(h, rank, size)

    def selftest(self, stream=None) -> bool:
        """All-to-all of rank-stamped chunks through the library's exchange path (collective)."""
        s = stream if stream is not None else torch.cuda.current_stream()
        ok = ctypes.c_int()
        st = lib().dr_comm_selftest(self.h, ctypes.c_void_p(s.cuda_stream), ctypes.byref(ok))
        if st != DR_OK:
            raise DiffRegError(st, lib().dr_status_string(st).decode())
        return bool(ok.value)

    def close(self):
        if getattr(self, "h", None):
            lib().dr_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Hub:
    """P virtual ranks in one process on one GPU (testing the slab path without P GPUs): each rank's
    context must be driven from its own host thread on its own stream."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        st = lib().dr_hub_create(nranks, ctypes.byref(h))
        if st != DR_OK:
            raise DiffRegError(st, "dr_hub_create")
        self.h, self.size = h, nranks

    def comm(self, rank: int) -> Comm:
        h = ctypes.c_void_p()
        st = lib().dr_comm_create_loopback(self.h, rank, ctypes.byref(h))
        if st != DR_OK:
            raise DiffRegError(st, "dr_comm_create_loopback")
        return Comm(h, rank, self.size, keep=self)

    def close(self):
        if getattr(self, "h", None):
            lib().dr_hub_destroy(self.h)
            self.h = None


class Context:
    """One dr_ctx: owns its workspace tensor (torch device memory) and uses the given CUDA stream.
    With `comm` the context is one rank of the slab decomposition and every field is its x3 slab."""

    def __init__(self, cfg: Config, device="cuda", stream: torch.cuda.Stream | None = None, comm: Comm | None = None):
        self.cfg = cfg
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.comm = comm
        self.nranks = comm.size if comm is not None else 1
        self.rank = comm.rank if comm is not None else 0
        self.z0, self.nz = dr_slab(cfg, self.nranks, self.rank)
        nbytes = dr_workspace_bytes_dist(cfg, self.nranks)
        if nbytes == 0:
            raise DiffRegError(DR_ERR_PARAM, f"invalid config {cfg} for {self.nranks} ranks")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        c = cfg.c()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):  # dr_create binds the context to the current device
            st = lib().dr_create_dist(ctypes.byref(c), comm.h if comm is not None else None, _ptr(self.workspace),
                                      nbytes, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if st != DR_OK:
            raise DiffRegError(st, lib().dr_status_string(st).decode())
        self.h = h

    def _check(self, st):
        if st != DR_OK:
            raise DiffRegError(st, lib().dr_last_error(self.h).decode())

    # fused ghost exchange (DR_PEER_GHOSTS=1, include/diffreg.h dr_peer_export): the CUDA IPC mapping of
    # the neighbours' workspaces for one process per GPU; loopback ranks need nothing
    def peer_export(self) -> tuple[bytes, int]:
        buf = ctypes.create_string_buffer(64)
        off = ctypes.c_uint64()
        self._check(lib().dr_peer_export(self.h, buf, ctypes.byref(off)))
        return buf.raw, off.value

    def peer_import(self, handles: list[bytes], offsets: list[int]):
        assert len(handles) == len(offsets) == self.nranks and all(len(h) == 64 for h in handles)
        arr = (ctypes.c_uint64 * self.nranks)(*offsets)
        self._check(lib().dr_peer_import(self.h, b"".join(handles), arr))

    def close(self):
        if getattr(self, "h", None):
            lib().dr_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # allocation helpers (on the context device; the rank's slab)
    @property
    def shape(self):
        n3, n2, n1 = self.cfg.shape
        return (self.nz, n2, n1)

    def scalar(self, device=None):
        return torch.empty(self.shape, dtype=self.cfg.dtype, device=device or self.device)

    def vector(self, device=None):
        return torch.empty((3,) + self.shape, dtype=self.cfg.dtype, device=device or self.device)

    def _buf(self, t, kind, what, host_ok=True):
        """Pointer of a field argument after checking what the library cannot (it sees only the pointer):
        a contiguous tensor of the context dtype with the rank's scalar (kind "s") / vector ("v") numel,
        on the context's device (or the host, where the C ABI stages host buffers).  ValueError otherwise."""
        if t is None:
            return None
        if not isinstance(t, torch.Tensor):
            raise ValueError(f"{what}: expected a torch.Tensor, got {type(t).__name__}")
        n = (3 if kind == "v" else 1) * self.nz * self.cfg.shape[1] * self.cfg.shape[2]
        if t.dtype != self.cfg.dtype:
            raise ValueError(f"{what}: dtype {t.dtype}, the context computes in {self.cfg.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what}: must be contiguous")
        if kind != "any" and t.numel() != n:
            raise ValueError(f"{what}: {t.numel()} elements, expected {n} ({'vector' if kind == 'v' else 'scalar'} "
                             f"field of the slab {self.shape})")
        if t.device.type == "cuda":
            if t.device.index != self.device.index and not (t.device.index is None or self.device.index is None):
                raise ValueError(f"{what}: on {t.device}, the context is on {self.device}")
        elif not (host_ok and t.device.type == "cpu"):
            raise ValueError(f"{what}: unsupported device {t.device}")
        return _ptr(t)

    def _in(self, t, kind="v", what="input"):
        return self._buf(t, kind, what)

    def _out(self, t, kind="v", what="output"):
        return self._buf(t, kind, what)

    # ---- main path (same names as the C ABI) ----
    def set_images(self, rho_T, rho_R):
        self._check(lib().dr_set_images(self.h, self._in(rho_T, "s", "rho_T"), self._in(rho_R, "s", "rho_R")))

    def set_velocity(self, v):
        self._check(lib().dr_set_velocity(self.h, self._in(v, "v", "v")))

    def forward_solve(self, rho1_out=None):
        self._check(lib().dr_forward_solve(self.h, self._out(rho1_out, "s", "rho1_out")))
        return rho1_out

    def adjoint_solve(self, lambda0_out=None):
        self._check(lib().dr_adjoint_solve(self.h, self._out(lambda0_out, "s", "lambda0_out")))
        return lambda0_out

    def hessian_matvec(self, vt, Hvt=None):
        if Hvt is None:
            Hvt = self.vector(vt.device)
        self._check(lib().dr_hessian_matvec(self.h, self._in(vt, "v", "vt"), self._out(Hvt, "v", "Hvt")))
        return Hvt

    def precond_apply(self, r, z=None):
        if z is None:
            z = self.vector(r.device)
        self._check(lib().dr_precond_apply(self.h, self._in(r, "v", "r"), self._out(z, "v", "z")))
        return z

    def sync(self):
        self._check(lib().dr_sync(self.h))

    # ---- NEXT-1: gradient and objective ----
    def gradient(self, g=None):
        if g is None:
            g = self.vector()
        self._check(lib().dr_gradient(self.h, self._out(g, "v", "g")))
        return g

    def pcg(self, g, eta: float, maxit: int, dv=None):
        """Newton step dv with H dv ~ -g (|r| <= eta |g|); returns (dv, iterations, |r| / |g|)."""
        if dv is None:
            dv = self.vector(g.device)
        it, rr = ctypes.c_int(), ctypes.c_double()
        self._check(lib().dr_pcg(self.h, self._in(g, "v", "g"), self._out(dv, "v", "dv"), eta, maxit, ctypes.byref(it),
                                 ctypes.byref(rr)))
        return dv, it.value, rr.value

    def deformation(self, want_u=True, want_det=True):
        """(u_1 = y_1 - x or None, det grad y_1 or None, det min, det max)."""
        u = self.vector() if want_u else None
        det = self.scalar() if want_det else None
        lo, hi = ctypes.c_double(), ctypes.c_double()
        self._check(lib().dr_deformation(self.h, self._out(u, "v", "u"), self._out(det, "s", "det"), ctypes.byref(lo),
                                         ctypes.byref(hi)))
        return u, det, lo.value, hi.value

    def solve(self, v, gtol=1e-2, max_newton=50, max_krylov=100, c1=1e-4, shrink=0.5, max_backtracks=20):
        """Armijo (G)N-Krylov registration from the device velocity v (updated in place).
        Returns (report dict, history rows [(J, |g|/|g0|, pcg matvecs, alpha, cumulative matvecs)])."""
        o = dr_solve_opts(gtol, max_newton, max_krylov, c1, shrink, max_backtracks)
        hist = (ctypes.c_double * (5 * max(1, max_newton)))()
        r = dr_solve_report()
        r.history = hist
        r.history_len = max_newton
        self._check(lib().dr_solve(self.h, self._buf(v, "v", "v", host_ok=False), ctypes.byref(o), ctypes.byref(r)))
        rows = [tuple(hist[5 * i:5 * i + 5]) for i in range(min(r.iterations, max_newton))]
        rep = {"iterations": r.iterations, "matvecs": r.matvecs, "reason": SOLVE_REASONS.get(r.reason, r.reason),
               "J0": r.J0, "J": r.J, "g0": r.g0, "g": r.g}
        return rep, rows

    def objective(self):
        """(J, misfit) as Python floats (collective with slabs)."""
        J, m = ctypes.c_double(), ctypes.c_double()
        self._check(lib().dr_objective(self.h, ctypes.byref(J), ctypes.byref(m)))
        return J.value, m.value

    # ---- tracing ----
    def profile_enable(self, on: bool = True):
        self._check(lib().dr_profile_enable(self.h, int(bool(on))))

    def profile_reset(self):
        self._check(lib().dr_profile_reset(self.h))

    def profile_only(self, tag=None):
        """Time only the launches tagged `tag` (None: all)."""
        self._check(lib().dr_profile_only(self.h, tag.encode() if tag else None))

    def profile(self):
        """({tag: (launches, total_ms)}, total kernel launches since the last reset)."""
        n = ctypes.c_int()
        tot = ctypes.c_int64()
        self._check(lib().dr_profile_count(self.h, ctypes.byref(n), ctypes.byref(tot)))
        out = {}
        for i in range(n.value):
            name = ctypes.create_string_buffer(64)
            k = ctypes.c_int64()
            ms = ctypes.c_double()
            self._check(lib().dr_profile_entry(self.h, i, name, 64, ctypes.byref(k), ctypes.byref(ms)))
            out[name.value.decode()] = (k.value, ms.value)
        return out, tot.value

    # ---- test hooks ----
    def op_spectral(self, op: int, x, out=None):
        if out is None:
            out = self.vector() if op in (DR_OP_GRAD, DR_OP_REG, DR_OP_PRECOND, DR_OP_LERAY) else self.scalar()
        vin = op in (DR_OP_DIV, DR_OP_REG, DR_OP_PRECOND, DR_OP_LERAY)
        vout = op in (DR_OP_GRAD, DR_OP_REG, DR_OP_PRECOND, DR_OP_LERAY)
        self._check(lib().dr_op_spectral(self.h, op, self._buf(x, "v" if vin else "s", "x", False),
                                         self._buf(out, "v" if vout else "s", "out", False)))
        return out

    def op_interp(self, f, s, out=None):
        s = s.contiguous()
        npts = s.shape[-1]
        if out is None:
            out = torch.empty(npts, dtype=self.cfg.dtype, device=self.device)
        if out.numel() != npts or s.numel() != 3 * npts:
            raise ValueError("op_interp: s must be (3, npts) and out (npts,)")
        self._check(lib().dr_op_interp(self.h, self._buf(f, "s", "f", False), npts, self._buf(s, "any", "s", False),
                                       self._buf(out, "any", "out", False)))
        return out

    def get_departure(self, sigma: int):
        out = self.vector()
        self._check(lib().dr_get_departure(self.h, sigma, self._out(out, "v", "out")))
        return out

    def get_field(self, which: int, j: int = 0):
        vec = which in (DR_FIELD_STATE_GRAD, DR_FIELD_BTILDE, DR_FIELD_VELOCITY)
        out = self.vector() if vec else self.scalar()
        self._check(lib().dr_get_field(self.h, which, j, self._out(out, "v" if vec else "s", "out")))
        return out


def _make_current(fn):
    """Run a Context method with the context's device current: the library launches on the current
    device, and a process may drive contexts on several GPUs."""
    import functools

    @functools.wraps(fn)
    def w(self, *a, **k):
        if self.device.type == "cuda" and self.device.index is not None:
            with torch.cuda.device(self.device):
                return fn(self, *a, **k)
        return fn(self, *a, **k)
    return w


for _name, _fn in list(vars(Context).items()):
    if callable(_fn) and not _name.startswith("_") and _name not in ("scalar", "vector", "close"):
        setattr(Context, _name, _make_current(_fn))
