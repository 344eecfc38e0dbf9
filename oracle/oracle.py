"""fp64 CPU ORACLE of the Gauss-Newton Hessian matvec (arXiv 1608.03630) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this module.  It shares no code with the CUDA product path and never imports it.

Primitives (FFT, spectral symbols, tricubic interpolation, RK2 departure points) live in the
plain C file oracle/oracle.c; the solves below compose them step by step in the paper's order
and notation (readings A1-A18 are listed in DESIGN.md).  All arrays are
float64 numpy arrays, scalars shaped (N3, N2, N1) and vectors (3, N3, N2, N1), x1 fastest.

Parity status: every function here is pinned by tests/test_oracle_pins.py except the general-v
matvec, which has no closed form ("parity unpinned" for general non-constant v: it is pinned
only indirectly, by the constant-v closed forms P12, the v=0 closed form P11 and the
convergence trends P8/P13/P14 -- see DESIGN.md §Parity).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -fopenmp, fp64, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER(ctypes.c_double)
        i, d, i64 = ctypes.c_int, ctypes.c_double, ctypes.c_int64
        L.or_spectral_scalar.argtypes = [i, i, i, i, P, P]
        L.or_grad.argtypes = [i, i, i, P, P]
        L.or_div.argtypes = [i, i, i, P, P]
        L.or_reg_apply.argtypes = [i, i, i, i, d, P, P]
        L.or_leray.argtypes = [i, i, i, P, P]
        L.or_precond.argtypes = [i, i, i, i, d, i, P, P]
        L.or_interp.argtypes = [i, i, i, P, i64, P, P, P, P]
        L.or_sl_gather.argtypes = [i, i, i, P, P, P]
        L.or_departure.argtypes = [i, i, i, i, i, P, P]
        L.or_fft3.argtypes = [i, i, i, ctypes.c_void_p, i]
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _n(a: np.ndarray):
    """(N1, N2, N3) of a scalar (N3,N2,N1) or vector (3,N3,N2,N1) array."""
    s = a.shape[-3:]
    return s[2], s[1], s[0]


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP thread count of the C primitives (timing protocol only; results do not depend on it)."""
    lib().or_set_num_threads(int(n))


# ------------------------------------------------------------------ grid (D0, D1)

def h(n):
    return tuple(2.0 * math.pi / N for N in n)


def inner(a: np.ndarray, b: np.ndarray) -> float:
    """<a,b> = h1 h2 h3 sum_i a_i b_i (D1; SPEC S:L53 discrete L2 inner product of P:L115)."""
    n = _n(a)
    hh = h(n)
    return float(hh[0] * hh[1] * hh[2] * np.sum(a * b))


# ------------------------------------------------------------------ spectral operators (D2, D3)

KIND = {"dx1": 0, "dx2": 1, "dx3": 2, "lap": 3, "biharm": 4}


def fft3(a: np.ndarray, sign: int) -> np.ndarray:
    """Unnormalised 3-D DFT of a complex (N3,N2,N1) array; sign=-1 forward, +1 inverse (D2)."""
    out = np.ascontiguousarray(a, dtype=np.complex128).copy()
    n1, n2, n3 = _n(out)
    lib().or_fft3(n1, n2, n3, out.ctypes.data, sign)
    return out


def spectral_scalar(kind: str, f: np.ndarray) -> np.ndarray:
    f = _c(f)
    out = np.empty_like(f)
    lib().or_spectral_scalar(*_n(f), KIND[kind], _p(f), _p(out))
    return out


def grad(f: np.ndarray) -> np.ndarray:
    """grad f via i k' (D3)."""
    f = _c(f)
    out = np.empty((3,) + f.shape)
    lib().or_grad(*_n(f), _p(f), _p(out))
    return out


def div(u: np.ndarray) -> np.ndarray:
    u = _c(u)
    out = np.empty(u.shape[1:])
    lib().or_div(*_n(u), _p(u), _p(out))
    return out


def reg_apply(u: np.ndarray, reg: int, beta: float) -> np.ndarray:
    """beta*A u, A = -Lap (reg=1, H1) or Lap^2 (reg=2, H2); Eq. 4, Eq. 5e."""
    u = _c(u)
    out = np.empty_like(u)
    lib().or_reg_apply(*_n(u), reg, beta, _p(u), _p(out))
    return out


def leray(u: np.ndarray) -> np.ndarray:
    """Leray projection I - grad Lap^{-1} div (Eq. 4)."""
    u = _c(u)
    out = np.empty_like(u)
    lib().or_leray(*_n(u), _p(u), _p(out))
    return out


def precond(r: np.ndarray, reg: int, beta: float, iso: bool) -> np.ndarray:
    """(beta A)^{-1} with a_hat(0)=1, then Leray if isochoric (§III-A; D13)."""
    r = _c(r)
    out = np.empty_like(r)
    lib().or_precond(*_n(r), reg, beta, int(bool(iso)), _p(r), _p(out))
    return out


# ------------------------------------------------------------------ interpolation and characteristics

def interp(f: np.ndarray, s: np.ndarray) -> np.ndarray:
    """Tricubic Lagrange interpolation of f at cell coordinates s (3, npts) (D4)."""
    f = _c(f)
    s = _c(s).reshape(3, -1)
    s1, s2, s3 = (_c(s[a]) for a in range(3))
    out = np.empty(s.shape[1])
    lib().or_interp(*_n(f), _p(f), s.shape[1], _p(s1), _p(s2), _p(s3), _p(out))
    return out


def sl_gather(f: np.ndarray, d: np.ndarray) -> np.ndarray:
    """out_i = I[f](i - d_i): one semi-Lagrangian interpolation at the departure points (D6)."""
    f = _c(f)
    d = _c(d)
    out = np.empty_like(f)
    lib().or_sl_gather(*_n(f), _p(f), _p(d), _p(out))
    return out


def departure(v: np.ndarray, nt: int, sigma: int) -> np.ndarray:
    """RK2 departure displacements d^sigma (cell units) for velocity sigma*v (Eq. 6; D5)."""
    v = _c(v)
    d = np.empty_like(v)
    lib().or_departure(*_n(v), nt, sigma, _p(v), _p(d))
    return d


# ------------------------------------------------------------------ transport solves (Eq. 7 literally)

def sl_step(nu: np.ndarray, d: np.ndarray, dt: float, f_at_X=None, f_at_x=None) -> np.ndarray:
    """One RK2 semi-Lagrangian step, Eq. 7, in order:
         nu0(X) = nu(X, 0)
         f0(X)  = f(nu0(X), X)
         nu*(x) = nu0(X) + dt f0(X)
         f*(x)  = f(nu*(x), x)
         nu(x, dt) = nu0(X) + dt/2 (f0(X) + f*(x))
    f_at_X(nu0X) returns f0(X); f_at_x(nu_star) returns f*(x).  With f == 0 this is nu0(X).
    """
    nu0X = sl_gather(nu, d)
    if f_at_X is None:
        return nu0X
    f0X = f_at_X(nu0X)
    nu_star = nu0X + dt * f0X
    f_star = f_at_x(nu_star)
    return nu0X + 0.5 * dt * (f0X + f_star)


def state_solve(rho_T: np.ndarray, d_plus: np.ndarray, nt: int) -> list[np.ndarray]:
    """State, Eqs. 2b-2c with f == 0 (D6): rho_{j+1} = I[rho_j](s+); all n_t+1 slices kept."""
    rho = [_c(rho_T)]
    for _ in range(nt):
        rho.append(sl_step(rho[-1], d_plus, 1.0 / nt))
    return rho


def adjoint_like_solve(nu_final: np.ndarray, d_minus: np.ndarray, Dv, nt: int) -> list[np.ndarray]:
    """Backward transport -d_t nu - div(v nu) = 0 solved forward in tau = 1 - t with -v, i.e.
    d_tau nu + (-v).grad nu = nu div v (D7).  The source f(nu, x) = nu * div v(x); by Eq. 7 and
    P:L275 ("interpolations for the f terms that depend on X") f0(X) = nu0(X) * I[div v](X)
    (reading A11).  Dv = None means div v == 0 (isochoric: pure advection).
    Returns slices indexed by t: out[k] ~ nu(t_k), k = 0..nt, out[nt] = nu_final."""
    dt = 1.0 / nt
    out = [None] * (nt + 1)
    out[nt] = _c(nu_final)
    if Dv is None:
        for k in range(nt, 0, -1):
            out[k - 1] = sl_step(out[k], d_minus, dt)
    else:
        Dbar = sl_gather(Dv, d_minus)  # div v at X (one interpolation, reused: v is stationary)
        for k in range(nt, 0, -1):
            out[k - 1] = sl_step(out[k], d_minus, dt,
                                 f_at_X=lambda nu0X: nu0X * Dbar,
                                 f_at_x=lambda nus: nus * Dv)
    return out


def inc_state_solve(vt: np.ndarray, G: list[np.ndarray], d_plus: np.ndarray, nt: int) -> list[np.ndarray]:
    """Incremental state, Eqs. 5a-5b via Algorithm 2, D9:
      line 1  rt0(X) = rt(X, t_j)                       (reading A8: rho-tilde)
      line 2-3 f0(x) = -vt(x).grad rho(x, t_j)          (G_j, cached per velocity)
      line 4  f0(X) by interpolation
      line 5  predictor rt*(x) = rt0(X) + dt f0(X)
      line 6-7 f*(x) = -vt(x).grad rho(x, t_{j+1})      (reading A9: the stored next state slice)
      line 8  rt(x, t_{j+1}) = rt0(X) + dt/2 (f0(X) + f*(x))
    rt(0) = 0 (Eq. 5b).  Returns all slices rt_0..rt_nt."""
    dt = 1.0 / nt
    f = [-(vt[0] * Gj[0] + vt[1] * Gj[1] + vt[2] * Gj[2]) for Gj in G]
    rt = [np.zeros_like(f[0])]
    for j in range(nt):
        f0X = sl_gather(f[j], d_plus)
        rt.append(sl_step(rt[j], d_plus, dt, f_at_X=lambda _nu0X, f0X=f0X: f0X,
                          f_at_x=lambda _nus, j=j: f[j + 1]))
    return rt


def inc_adjoint_newton_solve(rt1: np.ndarray, lam: list[np.ndarray], vt: np.ndarray, d_minus: np.ndarray, Dv,
                             nt: int) -> list[np.ndarray]:
    """Full-Newton incremental adjoint, Eq. 5c with the lambda term kept (NEXT-3):
      -d_t lt - div(lt v + lam vt) = 0,  lt(1) = -rt(1)  (Eq. 5d).
    In tau = 1 - t with -v: d_tau lt + (-v).grad lt = lt div v + s, s(t) = div(lam(t) vt)
    (spectral div, D3).  Eq. 7 with the f terms that depend on X interpolated (reading A11):
      f0(X) = nu0(X) I[div v](X) + I[s(t_k)](X)     (old level t_k, at the departure point)
      f*(x) = nu*(x) div v(x) + s(x, t_{k-1})       (new level, at the grid point)
    Dv = None: div v == 0 (isochoric), the first terms vanish."""
    dt = 1.0 / nt
    s = [div(lam[k] * vt) for k in range(nt + 1)]
    out = [None] * (nt + 1)
    out[nt] = -_c(rt1)
    Dbar = None if Dv is None else sl_gather(Dv, d_minus)
    for k in range(nt, 0, -1):
        sX = sl_gather(s[k], d_minus)
        if Dv is None:
            fX = (lambda nu0X, sX=sX: sX)
            fx = (lambda nus, k=k: s[k - 1])
        else:
            fX = (lambda nu0X, sX=sX: nu0X * Dbar + sX)
            fx = (lambda nus, k=k: nus * Dv + s[k - 1])
        out[k - 1] = sl_step(out[k], d_minus, dt, f_at_X=fX, f_at_x=fx)
    return out


def quadrature(lam: list[np.ndarray], G: list[np.ndarray], nt: int) -> np.ndarray:
    """b = int_0^1 lam grad rho dt by the trapezoidal rule on t_j = j dt (reading A12)."""
    dt = 1.0 / nt
    b = np.zeros_like(G[0])
    for j in range(nt + 1):
        w = 0.5 if j in (0, nt) else 1.0
        b += (dt * w) * lam[j] * G[j]
    return b


# ------------------------------------------------------------------ the registration problem

@dataclass
class Problem:
    rho_T: np.ndarray
    rho_R: np.ndarray
    nt: int = 4
    reg: int = 2            # 1: H1 (A = -Lap), 2: H2 (A = Lap^2)
    beta: float = 1e-2
    iso: bool = False       # isochoric variant (Leray-projected)


@dataclass
class VelocityState:
    """Everything computed once per velocity (points constructed "only when the velocity
    field changes"), plus the state solve and the cached state gradients G_j = grad rho_j."""
    v: np.ndarray
    d_plus: np.ndarray
    d_minus: np.ndarray
    Dv: np.ndarray | None
    rho: list = field(default_factory=list)
    G: list = field(default_factory=list)


def set_velocity(prob: Problem, v: np.ndarray) -> VelocityState:
    """Departure points for +v and -v (Eq. 6), div v for the adjoint source (non-isochoric),
    then the forward (state) solve and its gradients."""
    v = _c(v)
    if prob.iso:
        v = leray(v)  # keep v in the div-free subspace
    st = VelocityState(v=v, d_plus=departure(v, prob.nt, +1), d_minus=departure(v, prob.nt, -1),
                       Dv=None if prob.iso else div(v))
    st.rho = state_solve(prob.rho_T, st.d_plus, prob.nt)
    st.G = [grad(r) for r in st.rho]
    return st


def adjoint_solve(prob: Problem, st: VelocityState) -> list[np.ndarray]:
    """Adjoint, Eq. 3: lam(1) = rho_R - rho(1) (D8)."""
    return adjoint_like_solve(prob.rho_R - st.rho[-1], st.d_minus, st.Dv, prob.nt)


def hessian_matvec(prob: Problem, st: VelocityState, vt: np.ndarray, parts: bool = False, newton: bool = False,
                   lam=None):
    """Hessian matvec (Eqs. 5a-5e):
      rho-tilde by Algorithm 2, lam-tilde(1) = -rho-tilde(1) (Eq. 5d), backward incremental adjoint,
      b-tilde = int lam-tilde grad rho dt [+ int lam grad rho-tilde dt], H vt = beta A vt + P b-tilde
      (P = Leray if isochoric, else I).  Gauss-Newton (default): the two lambda terms dropped.
      newton=True (NEXT-3): both kept -- div(lam vt) in Eq. 5c and lam grad rho-tilde in b-tilde; needs
      the adjoint slices `lam` (computed by adjoint_solve when not given)."""
    vt = _c(vt)
    nt = prob.nt
    rt = inc_state_solve(vt, st.G, st.d_plus, nt)
    if newton:
        if lam is None:
            lam = adjoint_solve(prob, st)
        lt = inc_adjoint_newton_solve(rt[nt], lam, vt, st.d_minus, st.Dv, nt)
        bt = quadrature(lt, st.G, nt) + quadrature(lam, [grad(r) for r in rt], nt)
    else:
        lt = adjoint_like_solve(-rt[nt], st.d_minus, st.Dv, nt)
        bt = quadrature(lt, st.G, nt)
    reg_term = reg_apply(vt, prob.reg, prob.beta)
    data_term = leray(bt) if prob.iso else bt
    Hv = reg_term + data_term
    if parts:
        return Hv, {"reg": reg_term, "data": data_term, "btilde": bt, "rho_tilde": rt, "lam_tilde": lt}
    return Hv


def gradient(prob: Problem, st: VelocityState, lam=None) -> np.ndarray:
    """Reduced gradient g = beta A v + P b, b = int lam grad rho dt (Eq. 4; D14)."""
    if lam is None:
        lam = adjoint_solve(prob, st)
    b = quadrature(lam, st.G, prob.nt)
    return reg_apply(st.v, prob.reg, prob.beta) + (leray(b) if prob.iso else b)


def objective(prob: Problem, st: VelocityState) -> float:
    """J = 1/2 <rho(1) - rho_R, rho(1) - rho_R> + beta/2 <v, A v> (Eq. 2a; D14)."""
    r = st.rho[-1] - prob.rho_R
    return 0.5 * inner(r, r) + 0.5 * inner(st.v, reg_apply(st.v, prob.reg, prob.beta))


# ------------------------------------------------------------------ NEXT-2: inexact PCG

def forcing(gnorm: float, g0norm: float) -> float:
    """Quadratic forcing (Eisenstat-Walker): eta = min(0.5, |g| / |g_0|), so the
    Newton-system residual is <= eta |g| ~ |g|^2 / |g_0| (reading A22 in DESIGN.md)."""
    return min(0.5, gnorm / g0norm)


def pcg(prob: Problem, st: VelocityState, g: np.ndarray, eta: float, maxit: int):
    """Preconditioned CG on H dv = -g from dv = 0 (PCG, preconditioner (beta A)^-1, inexact
    with relative tolerance eta on the residual |r| <= eta |g|).  Norms and inner products are the
    discrete L2 ones (D1).  Returns (dv, iterations, |r| / |g|)."""
    g = _c(g)
    dv = np.zeros_like(g)
    r = -g
    gnorm = math.sqrt(inner(g, g))
    z = precond(r, prob.reg, prob.beta, prob.iso)
    p = z.copy()
    rz = inner(r, z)
    it = 0
    rnorm = gnorm
    while it < maxit and rnorm > eta * gnorm:
        q = hessian_matvec(prob, st, p)
        alpha = rz / inner(p, q)
        dv = dv + alpha * p
        r = r - alpha * q
        it += 1
        rnorm = math.sqrt(inner(r, r))
        if rnorm <= eta * gnorm:
            break
        z = precond(r, prob.reg, prob.beta, prob.iso)
        rz_new = inner(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return dv, it, rnorm / gnorm


# ------------------------------------------------------------------ NEXT-4: deformation map, det grad y

def deformation(v: np.ndarray, d_plus: np.ndarray, nt: int) -> np.ndarray:
    """Displacement u_1 = y_1 - x of the deformation map, Eq. 1: d_t y + v.grad y = 0,
    y(0) = x.  With y = x + u (u periodic): d_t u + v.grad u = -v, u(0) = 0, solved by Eq. 7 with the
    source f = -v (stationary, independent of u): f0(X) = I[-v](X), f*(x) = -v(x)."""
    v = _c(v)
    dt = 1.0 / nt
    u = np.zeros_like(v)
    fX = np.stack([sl_gather(-v[a], d_plus) for a in range(3)])
    for _ in range(nt):
        u = np.stack([sl_step(u[a], d_plus, dt, f_at_X=lambda _n, a=a: fX[a], f_at_x=lambda _n, a=a: -v[a])
                      for a in range(3)])
    return u


def det_grad_y(u: np.ndarray) -> np.ndarray:
    """det(grad y_1) = det(I + grad u_1) pointwise (Fig. 7 caption), grad by D3."""
    J = np.empty((3, 3) + u.shape[1:])
    for a in range(3):
        ga = grad(u[a])
        for b in range(3):
            J[a, b] = ga[b] + (1.0 if a == b else 0.0)
    return (J[0, 0] * (J[1, 1] * J[2, 2] - J[1, 2] * J[2, 1]) - J[0, 1] * (J[1, 0] * J[2, 2] - J[1, 2] * J[2, 0]) +
            J[0, 2] * (J[1, 0] * J[2, 1] - J[1, 1] * J[2, 0]))


# ------------------------------------------------------------------ NEXT-4: Armijo Gauss-Newton-Krylov

def solve(prob: Problem, v0: np.ndarray, gtol: float = 1e-2, max_newton: int = 50, max_krylov: int = 100,
          c1: float = 1e-4, shrink: float = 0.5, max_backtracks: int = 20, newton: bool = False):
    """Inexact (Gauss-)Newton-Krylov with Armijo line search:
      g_k = g(v_k); stop when |g_k| <= gtol |g_0|;  PCG on H dv = -g_k with eta = forcing(|g_k|, |g_0|);
      alpha = 1, shrink until J(v_k + alpha dv) <= J(v_k) + c1 alpha <g_k, dv>;  v_{k+1} = v_k + alpha dv.
    Returns (v, history, reason): history rows (J, |g|/|g0|, pcg iterations, alpha, cumulative matvecs)."""
    v = _c(v0).copy()
    st = set_velocity(prob, v)
    J = objective(prob, st)
    g = gradient(prob, st)
    g0 = math.sqrt(inner(g, g))
    hist, matvecs, reason = [], 0, "max_newton"
    for _ in range(max_newton):
        gn = math.sqrt(inner(g, g))
        if gn <= gtol * g0:
            reason = "converged"
            break
        lam = adjoint_solve(prob, st) if newton else None
        dv, it, _ = _pcg_op(prob, st, g, forcing(gn, g0), max_krylov, newton, lam)
        matvecs += it
        slope = inner(g, dv)
        alpha, accepted = 1.0, False
        for _ in range(max_backtracks + 1):
            st_try = set_velocity(prob, v + alpha * dv)
            J_try = objective(prob, st_try)
            if J_try <= J + c1 * alpha * slope:
                accepted = True
                break
            alpha *= shrink
        if not accepted:
            reason = "line_search_failed"
            break
        v = v + alpha * dv
        st, J = st_try, J_try
        g = gradient(prob, st)
        hist.append((J, math.sqrt(inner(g, g)) / g0, it, alpha, matvecs))
    else:
        if math.sqrt(inner(g, g)) <= gtol * g0:
            reason = "converged"
    return v, hist, reason


def _pcg_op(prob, st, g, eta, maxit, newton, lam):
    """pcg() with the (Gauss-)Newton matvec of the current linearisation."""
    if not newton:
        return pcg(prob, st, g, eta, maxit)
    g = _c(g)
    dv = np.zeros_like(g)
    r = -g
    gnorm = math.sqrt(inner(g, g))
    z = precond(r, prob.reg, prob.beta, prob.iso)
    p = z.copy()
    rz = inner(r, z)
    it, rnorm = 0, gnorm
    while it < maxit and rnorm > eta * gnorm:
        q = hessian_matvec(prob, st, p, newton=True, lam=lam)
        alpha = rz / inner(p, q)
        dv = dv + alpha * p
        r = r - alpha * q
        it += 1
        rnorm = math.sqrt(inner(r, r))
        if rnorm <= eta * gnorm:
            break
        z = precond(r, prob.reg, prob.beta, prob.iso)
        rz_new = inner(r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return dv, it, rnorm / gnorm
