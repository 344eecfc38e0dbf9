"""Pins of the fp64 oracle against what the paper and the mathematics fix.

None of these tests compares the oracle with itself: each checks a closed form, an invariant, an
independent library routine (numpy.fft / numpy.linalg), brute force on tiny inputs, or a
convergence rate, chosen so that a dropped term, a wrong sign / index or a transposed operand in
the oracle fails at least one of them.
"""
import math
import os

import numpy as np
import pytest

import synth
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def coords(n):
    return [a.numpy() for a in synth.grid_coords(n)]


def full(x, n):
    N1, N2, N3 = (n, n, n) if isinstance(n, int) else n
    return np.broadcast_to(x, (N3, N2, N1)).copy()


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


# ------------------------------------------------------------------ P1 spectral closed forms

def test_p1_grad_lap_biharm_rhoT():
    """rho_T = 1/2 - sum cos(2x_a)/6: grad, Laplacian, biharmonic in closed form."""
    n = 32
    rho = synth.rho_t_paper(n).numpy()
    x1, x2, x3 = coords(n)
    g = O.grad(rho)
    np.testing.assert_allclose(g[0], full(np.sin(2 * x1) / 3, n), atol=1e-13)
    np.testing.assert_allclose(g[1], full(np.sin(2 * x2) / 3, n), atol=1e-13)
    np.testing.assert_allclose(g[2], full(np.sin(2 * x3) / 3, n), atol=1e-13)
    s = full(np.cos(2 * x1) + np.cos(2 * x2) + np.cos(2 * x3), n)
    np.testing.assert_allclose(O.spectral_scalar("lap", rho), (2.0 / 3.0) * s, atol=1e-12)
    np.testing.assert_allclose(O.spectral_scalar("biharm", rho), -(8.0 / 3.0) * s, atol=1e-10)


def test_p1_div_closed_forms():
    n = 32
    x1, x2, x3 = coords(n)
    # BASELINE config-1 field is divergence-free; v* has div = -2 sin x1 sin x2 + cos x1 cos x3
    assert np.abs(O.div(synth.v_cfg1(n).numpy())).max() < 1e-13
    dv = O.div(synth.v_star(n).numpy())
    np.testing.assert_allclose(dv, full(-2 * np.sin(x1) * np.sin(x2) + np.cos(x1) * np.cos(x3), n), atol=1e-13)


def test_p1_anisotropic_grid_and_product_mode():
    n = (32, 16, 8)
    x1, x2, x3 = coords(n)
    f = full(np.sin(2 * x1) * np.cos(3 * x2) * np.cos(x3), n)
    g = O.grad(f)
    np.testing.assert_allclose(g[0], full(2 * np.cos(2 * x1) * np.cos(3 * x2) * np.cos(x3), n), atol=1e-12)
    np.testing.assert_allclose(g[1], full(-3 * np.sin(2 * x1) * np.sin(3 * x2) * np.cos(x3), n), atol=1e-12)
    np.testing.assert_allclose(g[2], full(-np.sin(2 * x1) * np.cos(3 * x2) * np.sin(x3), n), atol=1e-12)


def test_p1_spectral_examples_golden():
    """Single-mode symbol values (tests/golden/spectral_examples.txt)."""
    n = 16
    x1, _, _ = coords(n)
    for line in open(os.path.join(GOLD, "spectral_examples.txt")):
        if line.startswith("#") or not line.strip():
            continue
        op, beta, k, amp_in, amp_out = line.split()
        beta, k, amp_in, amp_out = float(beta), int(k), float(amp_in), float(amp_out)
        u = np.zeros((3, n, n, n))
        u[0] = full(amp_in * np.sin(k * x1), n)
        out = O.reg_apply(u, 2, beta) if op == "biharmonic" else O.precond(u, 2, beta, False)
        np.testing.assert_allclose(out[0], full(amp_out * np.sin(k * x1), n), atol=1e-12)
        assert np.abs(out[1:]).max() < 1e-14


def test_p1_h1_regulariser():
    n = 16
    x1, x2, _ = coords(n)
    u = np.zeros((3, n, n, n))
    u[1] = full(np.sin(2 * x1) * np.cos(x2), n)  # |k|^2 = 5
    out = O.reg_apply(u, 1, 0.5)
    np.testing.assert_allclose(out[1], 0.5 * 5 * u[1], atol=1e-12)


# ------------------------------------------------------------------ P2 FFT vs an independent library

@pytest.mark.parametrize("shape", [(8, 8, 8), (16, 8, 32), (6, 10, 4)])
def test_p2_fft_matches_numpy(shape):
    rng = np.random.default_rng(3)
    a = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
    np.testing.assert_allclose(O.fft3(a, -1), np.fft.fftn(a), atol=1e-12 * a.size)
    np.testing.assert_allclose(O.fft3(a, +1), np.fft.ifftn(a) * a.size, atol=1e-12 * a.size)


def test_p2_nyquist_conventions():
    """Reading A2: odd-order symbols zero the Nyquist mode, even-order symbols keep it."""
    n = 16
    x1, _, _ = coords(n)
    f = full(np.cos(8 * x1), n)  # pure Nyquist mode along x1: (-1)^i1
    assert np.abs(O.spectral_scalar("dx1", f)).max() < 1e-13
    np.testing.assert_allclose(O.spectral_scalar("lap", f), -64.0 * f, atol=1e-11)


# ------------------------------------------------------------------ P3 operator identities

def test_p3_identities_white_noise():
    n = 16
    rng = np.random.default_rng(5)
    f = rng.standard_normal((n, n, n))
    u = rng.standard_normal((3, n, n, n))
    gf = O.grad(f)
    # <grad f, u> = -<f, div u>   (periodic integration by parts)
    lhs, rhs = O.inner(gf, u), -O.inner(f, O.div(u))
    assert abs(lhs - rhs) < 1e-11 * (abs(lhs) + 1)
    Lu = O.leray(u)
    assert np.abs(O.div(Lu)).max() < 1e-11                     # div o L = 0
    assert rel(O.leray(Lu), Lu) < 1e-13                        # L^2 = L
    assert np.abs(O.leray(gf)).max() < 1e-11 * np.abs(gf).max()  # L grad f = 0
    w = synth.smooth_vec(7, n, kmax=4, divfree=True).numpy()
    assert rel(O.leray(w), w) < 1e-13                          # L u = u for div-free u
    # L is an orthogonal projector: <L u, u - L u> = 0
    assert abs(O.inner(Lu, u - Lu)) < 1e-10


# ------------------------------------------------------------------ P4 preconditioner

@pytest.mark.parametrize("reg", [1, 2])
def test_p4_preconditioner_inverts_regulariser(reg):
    n = 16
    beta = 0.37
    u = synth.smooth_vec(11, n, kmax=6).numpy()
    u -= u.mean(axis=(1, 2, 3), keepdims=True)
    assert rel(O.precond(O.reg_apply(u, reg, beta), reg, beta, False), u) < 1e-12
    c = np.ones((3, n, n, n)) * np.array([1.0, -2.0, 3.0])[:, None, None, None]
    np.testing.assert_allclose(O.precond(c, reg, beta, False), c / beta, atol=1e-12)


def test_p4_isochoric_preconditioner_is_projected():
    n = 16
    r = synth.smooth_vec(12, n, kmax=6).numpy()
    z = O.precond(r, 2, 1e-2, True)
    assert np.abs(O.div(z)).max() < 1e-9 * np.abs(z).max()
    assert rel(z, O.leray(O.precond(r, 2, 1e-2, False))) < 1e-13


# ------------------------------------------------------------------ P5 interpolation

def test_p5_node_exact_and_constants():
    n = (8, 16, 12)
    rng = np.random.default_rng(1)
    f = rng.standard_normal((12, 16, 8))
    i3, i2, i1 = np.meshgrid(np.arange(12), np.arange(16), np.arange(8), indexing="ij")
    s = np.stack([i1.ravel(), i2.ravel(), i3.ravel()]).astype(np.float64)
    assert np.array_equal(O.interp(f, s), f.ravel())  # bitwise: t = 0 picks one node with weight 1
    # periodic images of nodes are nodes too
    s2 = s + np.array([[8.0], [-16.0], [24.0]])
    assert np.array_equal(O.interp(f, s2), f.ravel())
    c = np.full((12, 16, 8), 2.5)
    pts = rng.uniform(-20, 20, (3, 500))
    np.testing.assert_allclose(O.interp(c, pts), 2.5, atol=1e-14)


def test_p5_reproduces_tensor_cubics_without_wrap():
    N = 16
    rng = np.random.default_rng(2)
    i = np.arange(N, dtype=np.float64)
    cf = [rng.standard_normal(4) for _ in range(3)]
    p = [np.polyval(cf[a], i / N) for a in range(3)]
    f = p[2][:, None, None] * p[1][None, :, None] * p[0][None, None, :]
    pts = rng.uniform(1.0, N - 3.0, (3, 400))  # stencil q-1..q+2 stays inside [0, N)
    ref = np.ones(400)
    for a in range(3):
        ref *= np.polyval(cf[a], pts[a] / N)
    np.testing.assert_allclose(O.interp(f, pts), ref, rtol=1e-11, atol=1e-11)


def test_p5_brute_force_vandermonde():
    """The 64-node tricubic interpolant equals the unique polynomial in span{x^l y^m z^n, l,m,n<=3}
    through the 4x4x4 stencil (numpy.linalg solve), on a tiny random grid."""
    N = 6
    rng = np.random.default_rng(4)
    f = rng.standard_normal((N, N, N))
    for _ in range(20):
        s = rng.uniform(0, N, 3)
        q = np.floor(s).astype(int)
        nodes = [(a, b, c) for c in range(-1, 3) for b in range(-1, 3) for a in range(-1, 3)]
        V = np.array([[(a ** l) * (b ** m) * (c ** k) for k in range(4) for m in range(4) for l in range(4)]
                      for a, b, c in nodes], dtype=np.float64)
        vals = np.array([f[(q[2] + c) % N, (q[1] + b) % N, (q[0] + a) % N] for a, b, c in nodes])
        coef = np.linalg.solve(V, vals)
        t = s - q
        mono = np.array([(t[0] ** l) * (t[1] ** m) * (t[2] ** k) for k in range(4) for m in range(4) for l in range(4)])
        assert abs(O.interp(f, s.reshape(3, 1))[0] - mono @ coef) < 1e-10


def test_p5_fourth_order_convergence():
    rng = np.random.default_rng(6)
    errs = []
    for N in (16, 32, 64, 128):
        x1, x2, x3 = coords(N)
        f = np.sin(x3) * np.sin(x2) * np.sin(x1)
        X = rng.uniform(0, 2 * np.pi, (3, 4000))
        s = X / (2 * np.pi / N)
        ex = np.sin(X[0]) * np.sin(X[1]) * np.sin(X[2])
        errs.append(np.abs(O.interp(f, s) - ex).max())
    order = math.log2(errs[-2] / errs[-1])
    assert order >= 3.7, errs


# ------------------------------------------------------------------ P6 constant velocity = Fourier multiplier

def _G_multiplier(N, d):
    """Amplification factor of one gather at constant displacement d (cells) along one axis:
    sum_m w_m(t) e^{i k (floor(-d)+m) 2pi/N}, m = -1..2 (Lagrange weights written from their node
    definition: w_m(t) = prod_{j != m} (t - j)/(m - j))."""
    e = -d
    fl = math.floor(e)
    t = e - fl
    k = np.fft.fftfreq(N, 1.0 / N)
    G = np.zeros(N, dtype=np.complex128)
    for m in range(-1, 3):
        w = 1.0
        for j in range(-1, 3):
            if j != m:
                w *= (t - j) / (m - j)
        G += w * np.exp(1j * k * (fl + m) * 2 * np.pi / N)
    return G


def test_p6_constant_velocity_transport_is_multiplier():
    n = 16
    nt = 3
    c = np.array([0.37, -0.81, 0.55])
    v = np.ones((3, n, n, n)) * c[:, None, None, None]
    d = O.departure(v, nt, +1)
    hh = 2 * np.pi / n
    np.testing.assert_allclose(d, v * (1.0 / nt) / hh, rtol=1e-15, atol=0)  # P7: d = dt c / h
    rho = O.state_solve(synth.blobs(3, n, kcut=6).numpy(), d, nt)
    G1, G2, G3 = (_G_multiplier(n, c[a] / nt / hh) for a in range(3))
    G = G3[:, None, None] * G2[None, :, None] * G1[None, None, :]
    ref = np.fft.ifftn(G ** nt * np.fft.fftn(rho[0])).real
    assert np.abs(rho[-1] - ref).max() < 1e-13


def test_p6_integer_shift_is_roll():
    n = 16
    nt = 2
    cells = np.array([1, -2, 3])  # per step
    hh = 2 * np.pi / n
    v = np.ones((3, n, n, n)) * (cells * hh * nt)[:, None, None, None]
    rho0 = np.random.default_rng(8).standard_normal((n, n, n))
    rho = O.state_solve(rho0, O.departure(v, nt, +1), nt)
    ref = np.roll(rho0, shift=(nt * cells[2], nt * cells[1], nt * cells[0]), axis=(0, 1, 2))
    assert np.array_equal(rho[-1], ref)


# ------------------------------------------------------------------ P7 departure points

def test_p7_zero_velocity_and_hand_example():
    n = 16
    assert np.array_equal(O.departure(np.zeros((3, n, n, n)), 4, 1), np.zeros((3, n, n, n)))
    kv = {}
    for line in open(os.path.join(GOLD, "departure_hand_example.txt")):
        if line.startswith("#") or not line.strip():
            continue
        k, *vals = line.split()
        kv[k] = [float(x) for x in vals]
    N, nt = int(kv["N"][0]), int(kv["nt"][0])
    i1, i2, i3 = (int(x) for x in kv["node"])
    _, x2, _ = coords(N)
    v = np.zeros((3, N, N, N))
    v[0] = full(np.sin(x2), N)
    d = O.departure(v, nt, +1) * (2 * np.pi / N)  # cells -> length
    assert abs(d[0, i3, i2, i1] - kv["disp_x1"][0]) < 1e-15
    assert abs(d[1, i3, i2, i1] - kv["disp_x2"][0]) < 1e-15
    assert abs(d[2, i3, i2, i1] - kv["disp_x3"][0]) < 1e-15


def _v_cfg1_analytic(X):
    x1, x2, x3 = X
    return np.stack([0.5 * np.sin(x3) * np.cos(x2) * np.sin(x2),
                     0.5 * np.sin(x1) * np.cos(x3) * np.sin(x3),
                     0.5 * np.sin(x2) * np.cos(x1) * np.sin(x1)])


def _v_star_analytic(X):
    x1, x2, x3 = X
    return np.stack([np.cos(x1) * np.sin(x2), np.cos(x2) * np.sin(x1), np.cos(x1) * np.sin(x3)])


def _grid_points(N):
    x1, x2, x3 = coords(N)
    return np.stack([full(x1, N), full(x2, N), full(x3, N)])


@pytest.mark.parametrize("vfun,gen", [(_v_cfg1_analytic, synth.v_cfg1), (_v_star_analytic, synth.v_star)])
def test_p7_departure_converges_to_analytic_rk2(vfun, gen):
    nt = 4
    dt = 1.0 / nt
    errs = []
    for N in (16, 32, 64, 128):
        X = _grid_points(N)
        vx = vfun(X)
        d_exact = 0.5 * dt * (vx + vfun(X - dt * vx)) / (2 * np.pi / N)
        d = O.departure(gen(N).numpy(), nt, +1)
        errs.append(np.abs(d - d_exact).max() * (2 * np.pi / N))
    assert math.log2(errs[-2] / errs[-1]) >= 3.5, errs


# ------------------------------------------------------------------ P8 transport

def test_p8_zero_velocity_identity_and_stability():
    n = 16
    rho0 = np.random.default_rng(9).standard_normal((n, n, n))
    rho = O.state_solve(rho0, O.departure(np.zeros((3, n, n, n)), 4, 1), 4)
    assert all(np.array_equal(r, rho0) for r in rho)
    # unconditional stability at CFL > 1: v* on 64^3, n_t = 4 (~1.3 cells/step ... )
    N = 64
    rT = synth.rho_t_paper(N).numpy()
    rho = O.state_solve(rT, O.departure(synth.v_star(N).numpy() * 4, 4, 1), 4)
    lo, hi = rT.min(), rT.max()
    for r in rho:
        assert np.isfinite(r).all()
        assert r.min() >= lo - 0.05 * (hi - lo) and r.max() <= hi + 0.05 * (hi - lo)


def test_p8_transport_converges_to_composed_rk2_map():
    nt = 4
    dt = 1.0 / nt
    errs = []
    for N in (32, 64, 128):
        X = _grid_points(N)
        Y = X.copy()
        for _ in range(nt):  # rho_nt(x) = rho_T(Phi^nt(x)), Phi = analytic-v RK2 departure map
            vY = _v_cfg1_analytic(Y)
            Y = Y - 0.5 * dt * (vY + _v_cfg1_analytic(Y - dt * vY))
        ref = (np.sin(Y[0]) ** 2 + np.sin(Y[1]) ** 2 + np.sin(Y[2]) ** 2) / 3
        rho = O.state_solve(synth.rho_t_paper(N).numpy(), O.departure(synth.v_cfg1(N).numpy(), nt, 1), nt)
        errs.append(np.abs(rho[-1] - ref).max())
    assert math.log2(errs[-2] / errs[-1]) >= 3.3, errs


# ------------------------------------------------------------------ P9/P10 incremental solves, special cases

def _problem(n, nt=4, reg=2, beta=1e-2, iso=False, rhoR=None):
    rT = synth.blobs(21, n, kcut=n // 3).numpy()
    return O.Problem(rho_T=rT, rho_R=rT.copy() if rhoR is None else rhoR, nt=nt, reg=reg, beta=beta, iso=iso)


def test_p9_p10_special_cases():
    n = 16
    prob = _problem(n)
    st = O.set_velocity(prob, np.zeros((3, n, n, n)))
    vt = synth.smooth_vec(1, n, kmax=4).numpy()
    rt = O.inc_state_solve(vt, st.G, st.d_plus, prob.nt)
    # v = 0: rho-tilde(1) = -vt . grad rho_T exactly (trapezoid of a constant source)
    np.testing.assert_allclose(rt[-1], -(vt * st.G[0]).sum(0), atol=1e-14)
    # vt = 0: rho-tilde == 0
    assert all(np.array_equal(r, 0 * r) for r in O.inc_state_solve(0 * vt, st.G, st.d_plus, prob.nt))
    # v = 0: the GN incremental adjoint is the identity in time
    lt = O.adjoint_like_solve(rt[-1], st.d_minus, st.Dv, prob.nt)
    assert all(np.array_equal(l, rt[-1]) for l in lt)
    # m == 1 path (div-free v) transports a constant exactly
    st2 = O.set_velocity(_problem(n, iso=True), synth.v_cfg1(n).numpy())
    lt = O.adjoint_like_solve(np.full((n, n, n), -1.5), st2.d_minus, st2.Dv, 4)
    assert all(np.abs(l + 1.5).max() < 1e-14 for l in lt)


def test_p10_adjoint_source_literal_eq7_equals_multiplier():
    """Eq. 7 with f = nu div v, applied literally, equals nu0(X) * m with
    m = 1 + dt/2 (Dbar + D + dt Dbar D) -- the rearrangement the GPU uses."""
    n = 16
    nt = 4
    v = synth.v_star(n).numpy()
    dm = O.departure(v, nt, -1)
    D = O.div(v)
    Db = O.sl_gather(D, dm)
    m = 1 + 0.5 / nt * (Db + D + Db * D / nt)
    lam = synth.blobs(4, n, kcut=5).numpy()
    out = O.adjoint_like_solve(lam, dm, D, nt)
    np.testing.assert_allclose(out[nt - 1], m * O.sl_gather(lam, dm), rtol=1e-13, atol=1e-14)


# ------------------------------------------------------------------ P11/P12 matvec closed forms

def test_p11_matvec_at_zero_velocity():
    n = 16
    for iso in (False, True):
        prob = _problem(n, iso=iso)
        st = O.set_velocity(prob, np.zeros((3, n, n, n)))
        vt = synth.smooth_vec(2, n, kmax=4).numpy()
        G0 = O.grad(prob.rho_T)
        data = (vt * G0).sum(0) * G0
        ref = O.reg_apply(vt, prob.reg, prob.beta) + (O.leray(data) if iso else data)
        assert rel(O.hessian_matvec(prob, st, vt), ref) < 1e-13


def _const_v_problem(n, nt, c, reg=2):
    prob = _problem(n, nt=nt, reg=reg)
    v = np.ones((3, n, n, n)) * np.asarray(c)[:, None, None, None]
    return prob, O.set_velocity(prob, v)


@pytest.mark.parametrize("c", [(0.37, -0.81, 0.55), (1.0, 0.0, 0.0)])
def test_p12_constant_velocity_symmetry_and_energy(c):
    n, nt = 16, 4
    prob, st = _const_v_problem(n, nt, c)
    x = synth.smooth_vec(30, n, kmax=5).numpy()
    y = synth.smooth_vec(31, n, kmax=5).numpy()
    Hx, px = O.hessian_matvec(prob, st, x, parts=True)
    Hy = O.hessian_matvec(prob, st, y)
    sym = abs(O.inner(Hx, y) - O.inner(x, Hy)) / (abs(O.inner(Hx, y)) + 1e-300)
    assert sym < 1e-12
    e_lhs = O.inner(x, Hx)
    e_rhs = O.inner(x, px["reg"]) + O.inner(px["rho_tilde"][-1], px["rho_tilde"][-1])
    assert abs(e_lhs - e_rhs) < 1e-12 * abs(e_lhs)


def test_p12_constant_velocity_fft_only_reference_path():
    """Independent numpy.fft implementation of the whole GN matvec at constant v, where every
    semi-Lagrangian gather is the Fourier multiplier of its constant displacement."""
    n, nt = 16, 4
    c = np.array([0.37, -0.81, 0.55])
    prob, st = _const_v_problem(n, nt, c, reg=1)
    hh = 2 * np.pi / n
    dt = 1.0 / nt
    # departure displacements in cells for +v and -v
    dp = c * dt / hh
    Gp = [_G_multiplier(n, dp[a]) for a in range(3)]
    Gm = [_G_multiplier(n, -dp[a]) for a in range(3)]
    Pp = Gp[2][:, None, None] * Gp[1][None, :, None] * Gp[0][None, None, :]
    Pm = Gm[2][:, None, None] * Gm[1][None, :, None] * Gm[0][None, None, :]
    k = np.fft.fftfreq(n, 1.0 / n)
    kp = np.where(np.abs(k) < n / 2, k, 0.0)
    K = np.meshgrid(k, k, k, indexing="ij")  # (k3, k2, k1) order
    KP = np.meshgrid(kp, kp, kp, indexing="ij")
    kk = K[0] ** 2 + K[1] ** 2 + K[2] ** 2
    F, iF = np.fft.fftn, lambda a: np.fft.ifftn(a).real
    rho_hat = [F(prob.rho_T)]
    for _ in range(nt):
        rho_hat.append(Pp * rho_hat[-1])
    Gr = [np.stack([iF(1j * KP[2] * r), iF(1j * KP[1] * r), iF(1j * KP[0] * r)]) for r in rho_hat]
    vt = synth.smooth_vec(5, n, kmax=5).numpy()
    f = [-(vt * g).sum(0) for g in Gr]
    rt = np.zeros((n, n, n))
    for j in range(nt):
        rt = iF(Pp * F(rt)) + 0.5 * dt * (iF(Pp * F(f[j])) + f[j + 1])
    lt = [None] * (nt + 1)
    lt[nt] = -rt
    for kk_ in range(nt, 0, -1):
        lt[kk_ - 1] = iF(Pm * F(lt[kk_]))
    bt = sum((0.5 if j in (0, nt) else 1.0) * dt * lt[j] * Gr[j] for j in range(nt + 1))
    reg = np.stack([iF(prob.beta * kk * F(vt[a])) for a in range(3)])
    ref = reg + bt
    Hv, parts = O.hessian_matvec(prob, st, vt, parts=True)
    assert rel(parts["data"], bt) < 1e-12
    assert rel(Hv, ref) < 1e-13


# ------------------------------------------------------------------ P13/P14 general v: discretisation-error trends

def _gn_defects(n, nt, v_gen, reg=1):
    """Zero-residual problem (rho_R = rho(1)[v], reading A13, so GN == Newton); returns the data-term
    symmetry defect |<Hx,y>-<x,Hy>|/sqrt(<Hx,x><Hy,y>), the energy-identity defect
    |<x,Hx> - |rho~(1)|^2|/<x,Hx> and the FD-of-gradient defect |FD - H x|/|H x| (data term)."""
    rT = synth.rho_t_paper(n).numpy()
    prob0 = O.Problem(rho_T=rT, rho_R=rT, nt=nt, reg=reg, beta=1e-2)
    v = v_gen(n).numpy()
    st = O.set_velocity(prob0, v)
    prob = O.Problem(rho_T=rT, rho_R=st.rho[-1].copy(), nt=nt, reg=reg, beta=1e-2)
    st = O.set_velocity(prob, v)
    x = synth.smooth_vec(40, n, kmax=3).numpy()
    y = synth.smooth_vec(41, n, kmax=3).numpy()
    _, px = O.hessian_matvec(prob, st, x, parts=True)
    _, py = O.hessian_matvec(prob, st, y, parts=True)
    scale = math.sqrt(O.inner(px["data"], x) * O.inner(py["data"], y))
    sym = abs(O.inner(px["data"], y) - O.inner(x, py["data"])) / scale
    ex = O.inner(x, px["data"])
    energy = abs(ex - O.inner(px["rho_tilde"][-1], px["rho_tilde"][-1])) / ex
    eps = 1e-4
    gp = O.gradient(prob, O.set_velocity(prob, v + eps * x))
    gm = O.gradient(prob, O.set_velocity(prob, v - eps * x))
    fd = (gp - gm) / (2 * eps) - O.reg_apply(x, reg, prob.beta)
    return sym, energy, rel(fd, px["data"])


def test_p13_p14_trends_decrease_under_refinement():
    """General v (v*, not div-free): symmetry, energy identity and FD-of-gradient hold only to
    discretisation error; all three must shrink when N and n_t are refined."""
    d = [_gn_defects(n, nt, synth.v_star) for n, nt in ((16, 4), (32, 4), (64, 8))]
    for a, b in zip(d[:-1], d[1:]):
        assert all(y < x for x, y in zip(a, b)), d
    assert d[-1][0] < 1e-3 and d[-1][1] < 1e-3 and d[-1][2] < 1e-2, d


@pytest.mark.parametrize("n", [8, (16, 8, 12)])
def test_objective_absolute_closed_forms(n):
    """J of Eq. 2a in absolute value, so the D1 weight h1 h2 h3 of `inner` is pinned (a
    1/M weight would fail): both cases are trigonometric polynomials whose grid sums are exact for N >= 8.
    (a) rho_T = G1 = (sin^2 x1 + sin^2 x2 + sin^2 x3)/3, rho_R = 0, v = 0 (identity transport, P8):
        J = 1/2 int rho_T^2 = (2 pi)^3 (1/4 + 3/72) / 2 = 7 (2 pi)^3 / 48.
    (b) v = (sin 2 x2, 0, 0), H2 (A = Delta^2: Delta^2 sin 2x2 = 16 sin 2x2), constant images (the
        constant is transported exactly, misfit 0): J = beta/2 * 16 int sin^2 2x2 = 4 beta (2 pi)^3."""
    N1, N2, N3 = (n, n, n) if isinstance(n, int) else n
    x1, x2, x3 = coords(n)
    rT = full((np.sin(x1) ** 2 + np.sin(x2) ** 2 + np.sin(x3) ** 2) / 3, n)
    prob = O.Problem(rho_T=rT, rho_R=np.zeros_like(rT), nt=4, reg=2, beta=1e-2)
    J = O.objective(prob, O.set_velocity(prob, np.zeros((3,) + rT.shape)))
    assert abs(J - 7 * (2 * math.pi) ** 3 / 48) < 1e-12 * J
    beta = 0.37
    c = np.full_like(rT, 0.25)
    v = np.zeros((3,) + rT.shape)
    v[0] = full(np.sin(2 * x2), n)
    for nt in (1, 3):
        prob = O.Problem(rho_T=c, rho_R=c.copy(), nt=nt, reg=2, beta=beta)
        J = O.objective(prob, O.set_velocity(prob, v))
        assert abs(J - 4 * beta * (2 * math.pi) ** 3) < 1e-12 * J, (nt, J)
    # H1 (A = -Delta: -Delta sin 2x2 = 4 sin 2x2): J = beta/2 * 4 * (2 pi)^3 / 2 = beta (2 pi)^3
    prob = O.Problem(rho_T=c, rho_R=c.copy(), nt=2, reg=1, beta=beta)
    J = O.objective(prob, O.set_velocity(prob, v))
    assert abs(J - beta * (2 * math.pi) ** 3) < 1e-12 * J


def test_gradient_matches_fd_of_objective():
    """<g, vt> against a centred difference of J (SPEC acceptance 5 idea): optimize-then-discretize,
    so agreement is to discretisation error only, shrinking under refinement."""
    defects = []
    for n, nt in ((16, 4), (32, 8)):
        prob = O.Problem(rho_T=synth.rho_t_paper(n).numpy(), rho_R=synth.blobs(8, n, kcut=5).numpy() * 0.3,
                         nt=nt, reg=2, beta=1e-2)
        v = 0.3 * synth.smooth_vec(9, n, kmax=3).numpy()
        vt = synth.smooth_vec(10, n, kmax=3).numpy()
        g = O.gradient(prob, O.set_velocity(prob, v))
        eps = 1e-4
        fd = (O.objective(prob, O.set_velocity(prob, v + eps * vt)) -
              O.objective(prob, O.set_velocity(prob, v - eps * vt))) / (2 * eps)
        defects.append(abs(O.inner(g, vt) - fd) / abs(fd))
    assert defects[1] < defects[0] and defects[1] < 4e-3, defects


# ------------------------------------------------------------------ NEXT-2: PCG against a dense solve

def test_pcg_matches_dense_solve_at_constant_velocity():
    """At constant v the discrete GN Hessian is exactly symmetric (P12) and positive definite, so PCG
    run to a tight tolerance must reproduce numpy.linalg.solve of the dense matrix H, assembled column
    by column from the oracle matvec on a 4^3 grid (192 unknowns); the forcing rule is checked too."""
    n, nt = 4, 2
    prob, st = _const_v_problem(n, nt, (0.37, -0.81, 0.55))
    N = 3 * n ** 3
    H = np.empty((N, N))
    for j in range(N):
        e = np.zeros(N)
        e[j] = 1.0
        H[:, j] = O.hessian_matvec(prob, st, e.reshape(3, n, n, n)).ravel()
    assert np.abs(H - H.T).max() < 1e-12 * np.abs(H).max()
    assert np.linalg.eigvalsh(0.5 * (H + H.T)).min() > 0
    g = synth.smooth_vec(40, n, kmax=1).numpy()
    dv_ref = np.linalg.solve(H, -g.ravel()).reshape(g.shape)
    dv, it, rr = O.pcg(prob, st, g, 1e-12, 500)
    assert rr <= 1e-12 and it <= N
    assert rel(dv, dv_ref) < 1e-9
    # inexact solve: the returned residual really is below eta |g|
    dv2, it2, rr2 = O.pcg(prob, st, g, 0.1, 500)
    res = O.hessian_matvec(prob, st, dv2) + g
    assert math.sqrt(O.inner(res, res)) <= 0.1 * math.sqrt(O.inner(g, g)) * (1 + 1e-9) and it2 < it
    assert abs(rr2 - math.sqrt(O.inner(res, res) / O.inner(g, g))) < 1e-9
    assert O.forcing(1.0, 1.0) == 0.5 and O.forcing(0.01, 1.0) == 0.01


# ------------------------------------------------------------------ NEXT-3: full-Newton Hessian

def _newton_fd_defects(n, nt, iso=False):
    """|FD of the gradient - H vt| / |FD| for the full-Newton and the Gauss-Newton matvec at a
    problem with a large residual (rho_R unrelated to rho_T), where the lambda terms matter."""
    prob = O.Problem(rho_T=synth.rho_t_paper(n).numpy(), rho_R=synth.blobs(8, n, kcut=5).numpy() * 0.3,
                     nt=nt, reg=1, beta=1e-2, iso=iso)
    v = 0.3 * synth.smooth_vec(9, n, kmax=3, divfree=iso).numpy()
    vt = synth.smooth_vec(10, n, kmax=3, divfree=iso).numpy()
    st = O.set_velocity(prob, v)
    eps = 1e-4
    fd = (O.gradient(prob, O.set_velocity(prob, v + eps * vt)) -
          O.gradient(prob, O.set_velocity(prob, v - eps * vt))) / (2 * eps)
    Hn = O.hessian_matvec(prob, st, vt, newton=True)
    Hg = O.hessian_matvec(prob, st, vt)
    nf = math.sqrt(O.inner(fd, fd))
    return (math.sqrt(O.inner(fd - Hn, fd - Hn)) / nf, math.sqrt(O.inner(fd - Hg, fd - Hg)) / nf)


def test_newton_hessian_matches_fd_of_gradient():
    """NEXT-3 pin (Eq. 5c with div(lam vt), b~ with lam grad rho~): the full-Newton
    matvec approximates the derivative of the gradient to discretisation error, clearly better than
    Gauss-Newton at a large residual, and the defect shrinks under refinement."""
    dn16, dg16 = _newton_fd_defects(16, 4)
    dn32, dg32 = _newton_fd_defects(32, 8)
    assert dn16 < 0.5 * dg16 and dn32 < 0.2 * dg32, (dn16, dg16, dn32, dg32)
    assert dn32 < dn16 and dn32 < 2e-2, (dn16, dn32)


def test_newton_equals_gauss_newton_at_zero_adjoint():
    """lam == 0 (zero residual, rho_R = rho(1)) makes the two lambda terms vanish: Newton == GN exactly
    (reading A13); the isochoric branch (no div v source) likewise."""
    for iso in (False, True):
        n, nt = 16, 4
        v = 0.4 * synth.smooth_vec(11, n, kmax=3, divfree=iso).numpy()
        prob = O.Problem(rho_T=synth.rho_t_paper(n).numpy(), rho_R=synth.rho_t_paper(n).numpy(), nt=nt, reg=2,
                         beta=1e-2, iso=iso)
        st = O.set_velocity(prob, v)
        prob.rho_R = st.rho[-1].copy()
        vt = synth.smooth_vec(12, n, kmax=3).numpy()
        a = O.hessian_matvec(prob, st, vt, newton=True)
        b = O.hessian_matvec(prob, st, vt)
        assert np.array_equal(a, b) or rel(a, b) < 1e-15


# ------------------------------------------------------------------ NEXT-4: deformation map and solver

def test_deformation_special_cases():
    """Eq. 1: v = 0 gives y_1 = x (u = 0, det = 1, bitwise); constant v = c gives y_1 = x - c exactly
    (a constant source transported at constant displacement), det = 1; a divergence-free v preserves
    volume up to discretisation error, which shrinks under refinement."""
    n, nt = 16, 4
    z = np.zeros((3, n, n, n))
    u = O.deformation(z, O.departure(z, nt, +1), nt)
    assert np.array_equal(u, z) and np.array_equal(O.det_grad_y(u), np.ones((n, n, n)))
    c = np.array([0.37, -0.81, 0.55])
    vc = np.ones((3, n, n, n)) * c[:, None, None, None]
    u = O.deformation(vc, O.departure(vc, nt, +1), nt)
    assert np.abs(u + vc).max() < 1e-13
    assert np.abs(O.det_grad_y(u) - 1).max() < 1e-12
    errs = []
    for n, nt in ((16, 4), (32, 8)):
        v = 0.5 * synth.v_cfg1(n).numpy()  # divergence-free (BJ config 1's field)
        u = O.deformation(v, O.departure(v, nt, +1), nt)
        errs.append(np.abs(O.det_grad_y(u) - 1).max())
    assert errs[1] < errs[0] < 0.05, errs


def test_solver_reduces_gradient_on_synthetic_problem():
    """NEXT-4 on the paper's synthetic problem: rho_T = (sin^2 x1 + sin^2 x2 + sin^2 x3)/3,
    rho_R = rho_T transported by v*; GN-Krylov with Armijo reaches g_tol = 1e-2, J decreases
    monotonically, every accepted step satisfies the Armijo condition, det grad y_1 > 0."""
    n, nt = 16, 4
    rT = synth.rho_t_paper(n).numpy()
    vstar = synth.v_star(n).numpy()
    prob0 = O.Problem(rho_T=rT, rho_R=rT, nt=nt, reg=2, beta=1e-2)
    rR = O.set_velocity(prob0, vstar).rho[-1]
    prob = O.Problem(rho_T=rT, rho_R=rR, nt=nt, reg=2, beta=1e-2)
    J0 = O.objective(prob, O.set_velocity(prob, np.zeros_like(vstar)))
    v, hist, reason = O.solve(prob, np.zeros_like(vstar), gtol=1e-2, max_newton=20)
    assert reason == "converged" and hist[-1][1] <= 1e-2
    Js = [J0] + [h[0] for h in hist]
    assert all(b < a for a, b in zip(Js[:-1], Js[1:]))
    st = O.set_velocity(prob, v)
    assert O.det_grad_y(O.deformation(v, st.d_plus, nt)).min() > 0
