"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Bars (BASELINE.json north_star): relative L2 <= 1e-5 per operator and <= 1e-4 per Hessian matvec for
the fp32 build; the data term P b~ is checked on its own as well (SURVEY P16'), since beta A vt
dominates |H vt| for H2.  The fp64 build (DR_FP64, BASELINE config 1) is held to 1e-12 / 1e-11.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

TOL32_OP, TOL32_MV = 1e-5, 1e-4
TOL64_OP, TOL64_MV = 1e-12, 1e-11


@pytest.fixture(scope="module")
def dr():
    from paper_1608_03630_b200 import build
    build.build()
    import paper_1608_03630_b200 as m
    m.lib()
    return m


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def np64(t):
    return t.detach().to("cpu", torch.float64).numpy()


def prep(x, fp64):
    """Round once to the GPU dtype; the oracle gets the rounded values."""
    g = x if fp64 else synth.round32(x)
    return g.contiguous(), synth.promote64(g)


def tols(fp64):
    return (TOL64_OP, TOL64_MV) if fp64 else (TOL32_OP, TOL32_MV)


def amp_tol(tol, shape, reg, beta, u64, Au64, fp64):
    """Tolerance of an amplifying operator (beta A, a(k) = |k|^(2 reg)) in fp64: both sides' FFT rounding
    (~eps |u| spread over every mode) is multiplied by a(k) up to the grid's largest |k|, while the signal
    is amplified only by its own modes'.  Relative error ~ eps * rms_k a(k) / (|A u| / |u|): on 1024-long
    lines with |k| <= 4 probes that is ~1e-8 for H2, far above 1e-12 (reading A20's conditioning argument,
    in fp64).  fp32 contexts run these forward passes in fp64 too, so their 1e-5 bar is unaffected."""
    if not fp64:
        return tol
    k = np.meshgrid(*[np.fft.fftfreq(N, 1.0 / N) for N in shape], indexing="ij")
    a = (k[0] ** 2 + k[1] ** 2 + k[2] ** 2) ** reg
    rms_a = float(np.sqrt(np.mean(a.astype(np.float64) ** 2)))
    eff = np.linalg.norm(Au64) / (beta * np.linalg.norm(u64))
    return max(tol, 32 * 2.0 ** -53 * rms_a / eff)


# ------------------------------------------------------------------ spectral operators

@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("n", [(32, 16, 64), (64, 64, 64), (8, 4, 16)])
def test_spectral_ops(dr, n, fp64):
    tol = tols(fp64)[0]
    for reg in (1, 2):
        cfg = dr.Config(n=n, nt=2, reg=reg, beta=0.37, fp64=fp64)
        ctx = dr.Context(cfg)
        f, f64 = prep(synth.blobs(5, n, kcut=min(n) // 3), fp64)
        u, u64 = prep(synth.smooth_vec(6, n, kmax=min(n) // 3), fp64)
        f, u = f.cuda(), u.cuda()
        assert rel(np64(ctx.op_spectral(dr.DR_OP_GRAD, f)), O.grad(f64)) < tol
        assert rel(np64(ctx.op_spectral(dr.DR_OP_DIV, u)), O.div(u64)) < tol
        assert rel(np64(ctx.op_spectral(dr.DR_OP_REG, u)), O.reg_apply(u64, reg, 0.37)) < tol
        assert rel(np64(ctx.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, False)) < tol
        assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, u)), O.leray(u64)) < tol
        ci = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37, fp64=fp64, isochoric=True))
        assert rel(np64(ci.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, True)) < tol


# FFT line lengths 128 (radix plan 16 x 8), 512 (16 x 16 x 2) and 1024 (16 x 16 x 4) on each axis, on
# anisotropic grids the oracle finishes in seconds (BJ configs 4-5 run 512- and 1024-long lines)
LONG_GRIDS = [(1024, 16, 16), (16, 1024, 16), (16, 16, 1024), (128, 32, 64), (512, 16, 32)]


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("n", LONG_GRIDS, ids=["x".join(map(str, g)) for g in LONG_GRIDS])
def test_spectral_ops_long_lines(dr, n, fp64):
    """grad, div, beta A (H1, H2), (beta A)^-1 (isochoric and not) and the Leray projection with long
    lines on every axis, in both precisions; the inputs carry modes up to |k| = min(n)/3 on every axis."""
    tol = tols(fp64)[0]
    kc = min(n) // 3
    f, f64 = prep(synth.blobs(5, n, kcut=kc), fp64)
    u, u64 = prep(synth.smooth_vec(6, n, kmax=kc), fp64)
    f, u = f.cuda(), u.cuda()
    for reg in (1, 2):
        ctx = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37, fp64=fp64))
        if reg == 1:
            assert rel(np64(ctx.op_spectral(dr.DR_OP_GRAD, f)), O.grad(f64)) < tol
            assert rel(np64(ctx.op_spectral(dr.DR_OP_DIV, u)), O.div(u64)) < tol
            assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, u)), O.leray(u64)) < tol
        Au = O.reg_apply(u64, reg, 0.37)
        assert rel(np64(ctx.op_spectral(dr.DR_OP_REG, u)), Au) < amp_tol(tol, u64.shape[1:], reg, 0.37, u64, Au, fp64)
        assert rel(np64(ctx.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, False)) < tol
        ci = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37, fp64=fp64, isochoric=True))
        assert rel(np64(ci.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, True)) < tol


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("iso", [False, True])
@pytest.mark.parametrize("n", LONG_GRIDS, ids=["x".join(map(str, g)) for g in LONG_GRIDS])
def test_matvec_long_lines(dr, n, iso, fp64):
    """One GN matvec per mode on the long-line grids (the isochoric data term goes through the x3
    middle pass KIND 6, the non-isochoric one through the staged row passes with b~ added)."""
    top, tmv = tols(fp64)
    kc = min(n) // 3
    nt = 2
    ctx = dr.Context(dr.Config(n=n, nt=nt, reg=2, beta=1e-2, isochoric=iso, fp64=fp64))
    rT, rT64 = prep(synth.blobs(11, n, kcut=kc), fp64)
    rR, rR64 = prep(synth.blobs(12, n, kcut=kc), fp64)
    v, v64 = prep(synth.smooth_vec(9, n, kmax=min(kc, 4), divfree=iso, cells_per_step=1.5, nt=nt), fp64)
    ctx.set_images(rT.cuda(), rR.cuda())
    ctx.set_velocity(v.cuda())
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=2, beta=1e-2, iso=iso)
    vt, vt64 = prep(synth.smooth_vec(21, n, kmax=min(kc, 4), divfree=iso), fp64)
    check_matvec(dr, ctx, prob, v64, vt, vt64, fp64, iso)


# extents that are not powers of two (one rank; Bluestein passes, M = 16 .. 1024): the paper's own
# grid is 256 x 300 x 256; SURVEY §8(b) admits any even N >= 4
BLUE_GRIDS = [(8, 6, 8), (16, 12, 8), (32, 24, 16), (16, 300, 16), (32, 510, 8),
              # x3 (Bluestein middle passes and x3 derivatives), and both axes at once
              (8, 8, 6), (16, 8, 12), (16, 16, 24), (8, 16, 300), (16, 12, 20),
              # x1 (Bluestein half-length row transforms, N1 % 4 == 0), and all three axes
              (12, 8, 8), (20, 16, 8), (300, 8, 16), (12, 12, 20)]


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("n", BLUE_GRIDS, ids=["x".join(map(str, g)) for g in BLUE_GRIDS])
def test_spectral_ops_non_pow2_x2(dr, n, fp64):
    """grad, div, beta A (H1, H2), (beta A)^-1 (isochoric and not) and the Leray projection on grids whose
    N1, N2 and / or N3 is not a power of two, against the oracle (whose non-power-of-two lines are plain
    DFT sums)."""
    tol = tols(fp64)[0]
    kc = max(1, min(n) // 3)
    f, f64 = prep(synth.blobs(5, n, kcut=kc), fp64)
    u, u64 = prep(synth.smooth_vec(6, n, kmax=kc), fp64)
    f, u = f.cuda(), u.cuda()
    for reg in (1, 2):
        ctx = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37, fp64=fp64))
        if reg == 1:
            assert rel(np64(ctx.op_spectral(dr.DR_OP_GRAD, f)), O.grad(f64)) < tol
            assert rel(np64(ctx.op_spectral(dr.DR_OP_DIV, u)), O.div(u64)) < tol
            assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, u)), O.leray(u64)) < tol
        Au = O.reg_apply(u64, reg, 0.37)
        assert rel(np64(ctx.op_spectral(dr.DR_OP_REG, u)), Au) < amp_tol(tol, u64.shape[1:], reg, 0.37, u64, Au, fp64)
        assert rel(np64(ctx.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, False)) < tol
        ci = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37, fp64=fp64, isochoric=True))
        assert rel(np64(ci.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, True)) < tol


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("iso", [False, True])
@pytest.mark.parametrize("n", BLUE_GRIDS[1:4] + BLUE_GRIDS[6:], ids=["x".join(map(str, g)) for g in BLUE_GRIDS[1:4] + BLUE_GRIDS[6:]])
def test_matvec_non_pow2_x2(dr, n, iso, fp64):
    """Setup, forward solve and one GN matvec per mode with non-power-of-two extents (ragged
    gather tiles, periodic wrap by remainder, Bluestein x2 / x3 passes in the gradients, the tail, the
    data term and the preconditioner)."""
    kc = max(1, min(n) // 3)
    nt = 2
    ctx = dr.Context(dr.Config(n=n, nt=nt, reg=2, beta=1e-2, isochoric=iso, fp64=fp64))
    rT, rT64 = prep(synth.blobs(11, n, kcut=kc), fp64)
    rR, rR64 = prep(synth.blobs(12, n, kcut=kc), fp64)
    v, v64 = prep(synth.smooth_vec(9, n, kmax=min(kc, 3), divfree=iso, cells_per_step=1.5, nt=nt), fp64)
    ctx.set_images(rT.cuda(), rR.cuda())
    ctx.set_velocity(v.cuda())
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=2, beta=1e-2, iso=iso)
    vt, vt64 = prep(synth.smooth_vec(21, n, kmax=min(kc, 3), divfree=iso), fp64)
    check_matvec(dr, ctx, prob, v64, vt, vt64, fp64, iso)


@pytest.mark.parametrize("fp64", [False, True])
def test_spectral_white_noise_nyquist(dr, fp64):
    """White noise carries Nyquist content: both sides must zero it in odd symbols (reading A2)."""
    n = (16, 32, 8)
    tol = tols(fp64)[0]
    ctx = dr.Context(dr.Config(n=n, nt=2, fp64=fp64))
    g = torch.Generator().manual_seed(3)
    f, f64 = prep(torch.randn((8, 32, 16), generator=g, dtype=torch.float64), fp64)
    u, u64 = prep(torch.randn((3, 8, 32, 16), generator=g, dtype=torch.float64), fp64)
    assert rel(np64(ctx.op_spectral(dr.DR_OP_GRAD, f.cuda())), O.grad(f64)) < tol
    assert rel(np64(ctx.op_spectral(dr.DR_OP_DIV, u.cuda())), O.div(u64)) < tol
    assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, u.cuda())), O.leray(u64)) < tol
    assert rel(np64(ctx.op_spectral(dr.DR_OP_REG, u.cuda())), O.reg_apply(u64, 2, 1e-2)) < tol


@pytest.mark.parametrize("fp64", [False, True])
def test_spectral_unaligned_input_same_bits(dr, fp64):
    """Device inputs and outputs that are not 16-byte aligned (the kernels' bulk copies and vector
    loads need 16 bytes) are staged through the workspace: same bits as aligned buffers, no fault."""
    n = (64, 32, 16)
    ctx = dr.Context(dr.Config(n=n, nt=2, reg=2, beta=0.37, fp64=fp64))
    u, _ = prep(synth.smooth_vec(6, n, kmax=5), fp64)
    u = u.cuda()
    buf = torch.empty(u.numel() + 1, dtype=u.dtype, device=u.device)
    ua = buf[1:].view(u.shape)  # 4 / 8 bytes past a 256-byte allocation boundary
    ua.copy_(u)
    assert ua.data_ptr() % 16 != 0
    obuf = torch.empty_like(buf)
    oa = obuf[1:].view(u.shape)  # unaligned output as well
    for op in (dr.DR_OP_REG, dr.DR_OP_PRECOND, dr.DR_OP_GRAD):
        x, xa = (u[0].contiguous(), buf[1:1 + u[0].numel()].view(u[0].shape)) if op == dr.DR_OP_GRAD else (u, ua)
        assert torch.equal(ctx.op_spectral(op, x), ctx.op_spectral(op, xa, out=oa)), op
    # main path: the matvec with an unaligned input and output
    ctx.set_images(*(prep(synth.blobs(s_, n, kcut=8), fp64)[0].cuda() for s_ in (1, 2)))
    ctx.set_velocity(prep(synth.smooth_vec(3, n, kmax=4, cells_per_step=1.5, nt=2), fp64)[0].cuda())
    ctx.forward_solve()
    assert torch.equal(ctx.hessian_matvec(u), ctx.hessian_matvec(ua, Hvt=oa))


# ------------------------------------------------------------------ interpolation

@pytest.mark.parametrize("fp64", [False, True])
def test_interp_points(dr, fp64):
    n = (32, 16, 64)
    ctx = dr.Context(dr.Config(n=n, nt=2, fp64=fp64))
    f, f64 = prep(synth.blobs(7, n, kcut=6), fp64)
    rng = np.random.default_rng(0)
    s = np.concatenate([rng.uniform(-40, 100, (3, 5000)),
                        np.array([[0, 31, 5], [0, 15, 3], [0, 63, 7]], dtype=np.float64)], axis=1)  # + exact nodes
    st = torch.tensor(s, dtype=torch.float64 if fp64 else torch.float32)
    out = np64(ctx.op_interp(f.cuda(), st.cuda()))
    ref = O.interp(f64, synth.promote64(st))
    assert rel(out, ref) < tols(fp64)[0]
    # node exactness: t = 0 reproduces the node value exactly
    fv = np64(f)
    assert out[-3] == fv[0, 0, 0] and out[-2] == fv[63, 15, 31] and out[-1] == fv[7, 3, 5]
    # empty input is a no-op
    ctx.op_interp(f.cuda(), torch.zeros((3, 0), dtype=f.dtype, device="cuda"))


# ------------------------------------------------------------------ transport, departure points, state/adjoint

CASES = [
    # name, n, nt, velocity generator, iso
    ("cfg1", 32, 4, lambda n: synth.v_cfg1(n), True),
    ("vstar64", 64, 8, lambda n: synth.v_star(n), False),
    ("smooth_aniso", (64, 32, 16), 4, lambda n: synth.smooth_vec(9, n, kmax=4, cells_per_step=2.0, nt=4), False),
    # large displacement (~9 cells/step): boxes exceed the shared-memory capacity -> global fallback tiles
    ("stress", 64, 4, lambda n: synth.smooth_vec(10, n, kmax=6, cells_per_step=9.0, nt=4), False),
]


def setup_case(dr, name, n, nt, vgen, iso, fp64, reg=2, beta=1e-2):
    cfg = dr.Config(n=n, nt=nt, reg=reg, beta=beta, isochoric=iso, fp64=fp64)
    ctx = dr.Context(cfg)
    rT, rT64 = prep(synth.blobs(11, n, kcut=10) if name != "cfg1" else synth.rho_t_paper(n), fp64)
    rR, rR64 = prep(synth.blobs(12, n, kcut=10), fp64)
    v, v64 = prep(vgen(n), fp64)
    ctx.set_images(rT.cuda(), rR.cuda())
    ctx.set_velocity(v.cuda())
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=reg, beta=beta, iso=iso)
    return ctx, prob, v64


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_departure_state_adjoint(dr, case, fp64):
    name, n, nt, vgen, iso = case
    tol = tols(fp64)[0]
    ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, fp64)
    st = O.set_velocity(prob, v64)
    if iso:
        assert rel(np64(ctx.get_field(dr.DR_FIELD_VELOCITY)), st.v) < tol
    assert rel(np64(ctx.get_departure(+1)), st.d_plus) < tol
    assert rel(np64(ctx.get_departure(-1)), st.d_minus) < tol
    if not iso:
        Db = O.sl_gather(st.Dv, st.d_minus)
        m_ref = 1 + 0.5 / nt * (Db + st.Dv + Db * st.Dv / nt)
        assert rel(np64(ctx.get_field(dr.DR_FIELD_MULTIPLIER)) - 1, m_ref - 1) < 10 * tol
    ctx.forward_solve()
    for j in range(nt + 1):
        assert rel(np64(ctx.get_field(dr.DR_FIELD_STATE, j)), st.rho[j]) < tol, j
        assert rel(np64(ctx.get_field(dr.DR_FIELD_STATE_GRAD, j)), st.G[j]) < tol, j
    ctx.adjoint_solve()
    lam = O.adjoint_solve(prob, st)
    for j in range(nt + 1):
        assert rel(np64(ctx.get_field(dr.DR_FIELD_ADJOINT, j)), lam[j]) < tol, j


def test_departure_single_step_on_gpu_inputs(dr):
    """Exact per-step parity: oracle interpolation of the GPU's own rho_j at the GPU's departure points
    reproduces the GPU's rho_{j+1} (isolates the gather kernel from accumulated rounding)."""
    ctx, prob, v64 = setup_case(dr, "stress", 64, 4, CASES[3][3], False, False)
    ctx.forward_solve()
    d = np64(ctx.get_departure(+1))
    for j in range(4):
        rj = np64(ctx.get_field(dr.DR_FIELD_STATE, j))
        ref = O.sl_gather(rj, d)
        assert rel(np64(ctx.get_field(dr.DR_FIELD_STATE, j + 1)), ref) < 1e-6


# ------------------------------------------------------------------ Hessian matvec

def check_matvec(dr, ctx, prob, v64, vt, vt64, fp64, iso):
    top, tmv = tols(fp64)
    st = O.set_velocity(prob, v64)
    ctx.forward_solve()
    Hv = np64(ctx.hessian_matvec(vt.cuda()))
    ref, parts = O.hessian_matvec(prob, st, vt64, parts=True)
    # per term (SURVEY P16'): the data term P b~ on its own, then beta A vt, then the sum
    bt_gpu = ctx.get_field(dr.DR_FIELD_BTILDE)
    bt = np64(bt_gpu)
    assert rel(bt, parts["btilde"]) < tmv
    if iso:
        assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, bt_gpu)), parts["data"]) < tmv
    assert rel(np64(ctx.get_field(dr.DR_FIELD_INC_STATE)), parts["rho_tilde"][-1]) < tmv
    for j in range(prob.nt + 1):
        assert rel(np64(ctx.get_field(dr.DR_FIELD_INC_ADJOINT, j)), parts["lam_tilde"][j]) < tmv, j
    reg = np64(ctx.op_spectral(dr.DR_OP_REG, vt.cuda()))
    shape = vt64.shape[1:]
    atol = amp_tol(top, shape, prob.reg, prob.beta, vt64, parts["reg"], fp64)
    assert rel(reg, parts["reg"]) < atol
    assert rel(Hv, ref) < max(tmv, atol)
    return Hv


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("zero_residual", [True, False])
def test_matvec_config2(dr, zero_residual, fp64):
    """BASELINE config 2: 64^3, nt = 8, H1, beta = 1e-2, v* (div v != 0 -> multiplier path), random smooth
    vt (|k| <= 8, unit RMS); rho_R = rho(1)[v] (zero residual, GN == Newton; reading A13) or rho_R = rho_T."""
    n, nt = 64, 8
    cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H1, beta=1e-2, fp64=fp64)
    ctx = dr.Context(cfg)
    rT, rT64 = prep(synth.rho_t_paper(n), fp64)
    v, v64 = prep(synth.v_star(n), fp64)
    ctx.set_images(rT.cuda(), rT.cuda())
    ctx.set_velocity(v.cuda())
    if zero_residual:
        rho1 = ctx.forward_solve(torch.empty_like(rT).cuda())
        rR, rR64 = rho1.cpu().contiguous(), synth.promote64(rho1.cpu())
        ctx.set_images(rT.cuda(), rho1)
    else:
        rR, rR64 = rT, rT64
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=1, beta=1e-2)
    vt, vt64 = prep(synth.smooth_vec(2, n, kmax=8), fp64)
    check_matvec(dr, ctx, prob, v64, vt, vt64, fp64, False)


@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_matvec_cases(dr, case, fp64):
    name, n, nt, vgen, iso = case
    ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, fp64)
    vt, vt64 = prep(synth.smooth_vec(21, n, kmax=6, divfree=iso), fp64)
    check_matvec(dr, ctx, prob, v64, vt, vt64, fp64, iso)


@pytest.mark.parametrize("iso", [False, True])
def test_precond_apply(dr, iso):
    n = (32, 64, 16)
    ctx = dr.Context(dr.Config(n=n, nt=2, reg=2, beta=1e-2, isochoric=iso))
    r, r64 = prep(synth.smooth_vec(31, n, kmax=8), False)
    z = np64(ctx.precond_apply(r.cuda()))
    assert rel(z, O.precond(r64, 2, 1e-2, iso)) < TOL32_OP
    # in-place (r and z may alias)
    rc = r.cuda().clone()
    ctx.precond_apply(rc, rc)
    assert rel(np64(rc), z) < 1e-7


# ------------------------------------------------------------------ ABI behaviour on the GPU

def test_host_buffers_match_device_buffers(dr):
    n, nt = 32, 4
    ctx = dr.Context(dr.Config(n=n, nt=nt))
    rT = synth.round32(synth.blobs(1, n, kcut=8))
    v = synth.round32(synth.smooth_vec(2, n, kmax=4, cells_per_step=1.0, nt=nt))
    vt = synth.round32(synth.smooth_vec(3, n, kmax=4))
    ctx.set_images(rT, rT)  # host pointers
    ctx.set_velocity(v.pin_memory())
    ctx.forward_solve()
    h_host = ctx.hessian_matvec(vt.pin_memory(), torch.empty_like(vt).pin_memory())
    h_pageable = ctx.hessian_matvec(vt, torch.empty_like(vt))
    h_dev = ctx.hessian_matvec(vt.cuda()).cpu()
    assert torch.equal(h_host, h_dev) and torch.equal(h_pageable, h_dev)
    z_host = ctx.precond_apply(vt, torch.empty_like(vt))
    assert torch.equal(z_host, ctx.precond_apply(vt.cuda()).cpu())


def test_profiler_tag_filter(dr):
    """dr_profile_only(tag): only that tag's launches are timed; the launch counter still counts all."""
    n = (32, 16, 64)
    ctx, prob, v64 = setup_case(dr, "smooth_aniso", n, 4, lambda n_: synth.smooth_vec(9, n_, kmax=4, cells_per_step=2.0, nt=4),
                                False, False)
    ctx.forward_solve()
    vt = synth.round32(synth.smooth_vec(21, n, kmax=5)).contiguous().cuda()
    for only in (None, "sl_inc_adjoint_q2"):
        ctx.profile_reset()
        ctx.profile_only(only)
        ctx.profile_enable(True)
        ctx.hessian_matvec(vt)
        prof, launches = ctx.profile()
        ctx.profile_enable(False)
        if only is None:
            assert {"sl_inc_state", "sl_inc_state_b", "sl_inc_adjoint_q2", "inc_init"} <= set(prof)
            assert sum(k for k, _ in prof.values()) == launches
            full = launches
        else:
            assert set(prof) == {only} and prof[only][0] == 4 and prof[only][1] > 0
            assert launches == full
    ctx.profile_only(None)


def test_call_order_and_argument_errors(dr):
    n = 16
    ctx = dr.Context(dr.Config(n=n, nt=2))
    vt = torch.zeros((3, n, n, n), device="cuda")
    with pytest.raises(dr.DiffRegError) as e:
        ctx.hessian_matvec(vt)
    assert e.value.status == dr.DR_ERR_ORDER
    with pytest.raises(dr.DiffRegError) as e:
        ctx.forward_solve()
    assert e.value.status == dr.DR_ERR_ORDER
    with pytest.raises(dr.DiffRegError) as e:
        ctx.adjoint_solve()
    assert e.value.status == dr.DR_ERR_ORDER
    f = torch.zeros((n, n, n), device="cuda")
    ctx.set_images(f, f)
    ctx.set_velocity(vt)
    ctx.forward_solve()
    with pytest.raises(dr.DiffRegError) as e:
        ctx.hessian_matvec(vt, vt)  # aliasing
    assert e.value.status == dr.DR_ERR_ARG
    # zero velocity, zero probe: H 0 = 0 exactly
    assert torch.count_nonzero(ctx.hessian_matvec(vt)) == 0
    ctx.set_velocity(vt)  # invalidates the state
    with pytest.raises(dr.DiffRegError) as e:
        ctx.hessian_matvec(vt)
    assert e.value.status == dr.DR_ERR_ORDER


def test_matvec_linearity_and_determinism(dr):
    """H is linear in vt.  The data term (b~) is checked tightly; the full H vt only to 1e-4 because the
    fp32 rounding of the input 2x - 3y itself is amplified by the H2 symbol |k|^4 (DESIGN.md,
    "fp32 conditioning of the regulariser")."""
    n, nt = 32, 4
    ctx = dr.Context(dr.Config(n=n, nt=nt))
    rT = synth.round32(synth.blobs(1, n, kcut=8)).cuda()
    ctx.set_images(rT, rT)
    ctx.set_velocity(synth.round32(synth.smooth_vec(2, n, kmax=4, cells_per_step=1.5, nt=nt)).cuda())
    ctx.forward_solve()
    x = synth.round32(synth.smooth_vec(3, n, kmax=4)).cuda()
    y = synth.round32(synth.smooth_vec(4, n, kmax=4)).cuda()
    hx = ctx.hessian_matvec(x)
    bx = ctx.get_field(dr.DR_FIELD_BTILDE)
    hy = ctx.hessian_matvec(y)
    by = ctx.get_field(dr.DR_FIELD_BTILDE)
    h = ctx.hessian_matvec((2 * x - 3 * y).contiguous())
    b = ctx.get_field(dr.DR_FIELD_BTILDE)
    assert rel(np64(b), np64(2 * bx - 3 * by)) < 1e-5
    assert rel(np64(h), np64(2 * hx - 3 * hy)) < 1e-4
    assert torch.equal(ctx.hessian_matvec(x), hx)  # bitwise deterministic


# ------------------------------------------------------------------ NEXT-1: gradient and objective

@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("case", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_gradient_objective(dr, case, fp64):
    """g = beta A v + P b, b = int lambda grad rho (Eq. 4) and J (Eq. 2a) against the oracle's D14."""
    name, n, nt, vgen, iso = case
    top, tmv = tols(fp64)
    ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, fp64)
    st = O.set_velocity(prob, v64)
    ctx.forward_solve()
    g = np64(ctx.gradient())
    gref = O.gradient(prob, st)
    # fp64: beta A v amplifies FFT rounding (~1e-16) by |k|^4 up to (32 sqrt 3)^4 ~ 1e7 against the
    # |k|^4 ~ 4 of v*'s own modes (reading A20's conditioning, in fp64), so 1e-10 rather than 1e-11
    assert rel(g, gref) < (1e-10 if fp64 else tmv)
    J, mis = ctx.objective()
    Jref = O.objective(prob, st)
    r = st.rho[-1] - prob.rho_R
    assert abs(mis - 0.5 * O.inner(r, r)) <= (1e-12 if fp64 else 1e-5) * abs(0.5 * O.inner(r, r))
    assert abs(J - Jref) <= (1e-12 if fp64 else 1e-5) * abs(Jref)


@pytest.mark.parametrize("fp64", [False, True])
def test_objective_absolute_closed_forms(dr, fp64):
    """The GPU's J (Eq. 2a) against closed forms, not only against the oracle's J:
    rho_T = G1, rho_R = 0, v = 0 gives J = 7 (2 pi)^3 / 48; constant images with v = (sin 2x2, 0, 0)
    and H2 give J = 4 beta (2 pi)^3 (both exact on the grid for N >= 8)."""
    n = (16, 8, 32)
    tol = 1e-12 if fp64 else 1e-6
    x1, x2, x3 = synth.grid_coords(n)
    rT = ((torch.sin(x1) ** 2 + torch.sin(x2) ** 2 + torch.sin(x3) ** 2) / 3).expand(32, 8, 16)
    dt_ = torch.float64 if fp64 else torch.float32
    ctx = dr.Context(dr.Config(n=n, nt=4, reg=2, beta=1e-2, fp64=fp64))
    ctx.set_images(rT.to(dt_).contiguous().cuda(), torch.zeros_like(rT, dtype=dt_).cuda())
    ctx.set_velocity(torch.zeros((3, 32, 8, 16), dtype=dt_, device="cuda"))
    ctx.forward_solve()
    J, mis = ctx.objective()
    assert abs(J - 7 * (2 * np.pi) ** 3 / 48) < tol * J and J == mis
    beta = 0.37
    ctx = dr.Context(dr.Config(n=n, nt=3, reg=2, beta=beta, fp64=fp64))
    c = torch.full((32, 8, 16), 0.25, dtype=dt_, device="cuda")
    ctx.set_images(c, c.clone())
    v = torch.zeros((3, 32, 8, 16), dtype=torch.float64)
    v[0] = torch.sin(2 * x2).expand(32, 8, 16)
    ctx.set_velocity(v.to(dt_).contiguous().cuda())
    ctx.forward_solve()
    J, mis = ctx.objective()
    assert abs(J - 4 * beta * (2 * np.pi) ** 3) < tol * J and abs(mis) < tol * J


# ------------------------------------------------------------------ NEXT-2: PCG

@pytest.mark.parametrize("case", [CASES[1], CASES[0]], ids=["vstar64", "cfg1"])
def test_pcg_against_oracle(dr, case):
    """Fixed iteration count (eta = 0): the GPU's fp32 PCG iterate follows the fp64 oracle's PCG; the
    inexact solve's residual, re-evaluated with the ORACLE's matvec, is below eta |g| (+ fp32 slack)."""
    name, n, nt, vgen, iso = case
    ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
    st = O.set_velocity(prob, v64)
    ctx.forward_solve()
    # isochoric problems live in the divergence-free subspace (the preconditioner projects), so their
    # right-hand sides -- gradients -- are divergence-free
    g, g64 = prep(synth.smooth_vec(41, n, kmax=6, divfree=iso), False)
    dv, it, rr = ctx.pcg(g.cuda(), 0.0, 3)
    ref, it_ref, rr_ref = O.pcg(prob, st, g64, 0.0, 3)
    assert it == it_ref == 3
    assert rel(np64(dv), ref) < 1e-4
    assert abs(rr - rr_ref) < 1e-3 * rr_ref
    eta = 0.05
    dv, it, rr = ctx.pcg(g.cuda(), eta, 50)
    res = O.hessian_matvec(prob, st, np64(dv)) + g64
    assert rr <= eta and 0 < it < 50
    assert np.sqrt(O.inner(res, res) / O.inner(g64, g64)) < eta + 1e-4


# ------------------------------------------------------------------ NEXT-3: full-Newton matvec

@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("case", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_full_newton_matvec(dr, case, fp64):
    """DR_FULL_NEWTON: Eq. 5c with div(lam vt) and b~ with lam grad rho~ against the
    oracle's full-Newton matvec; the images differ (rho_R unrelated to rho(1)), so lambda != 0."""
    name, n, nt, vgen, iso = case
    top, tmv = tols(fp64)
    cfg = dr.Config(n=n, nt=nt, reg=2, beta=1e-2, isochoric=iso, fp64=fp64, newton=True)
    ctx = dr.Context(cfg)
    rT, rT64 = prep(synth.blobs(11, n, kcut=10) if name != "cfg1" else synth.rho_t_paper(n), fp64)
    rR, rR64 = prep(synth.blobs(12, n, kcut=10), fp64)
    v, v64 = prep(vgen(n), fp64)
    vt, vt64 = prep(synth.smooth_vec(13, n, kmax=4, divfree=iso), fp64)
    ctx.set_images(rT.cuda(), rR.cuda())
    ctx.set_velocity(v.cuda())
    ctx.forward_solve()
    Hv = np64(ctx.hessian_matvec(vt.cuda()))
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=2, beta=1e-2, iso=iso)
    st = O.set_velocity(prob, v64)
    ref, parts = O.hessian_matvec(prob, st, vt64, parts=True, newton=True)
    assert rel(np64(ctx.get_field(dr.DR_FIELD_BTILDE)), parts["btilde"]) < tmv
    assert rel(Hv, ref) < tmv
    # and it differs from Gauss-Newton by much more than the tolerance
    gn = O.hessian_matvec(prob, st, vt64)
    assert rel(gn, ref) > 100 * tmv


# ------------------------------------------------------------------ NEXT-4: deformation map and solver

@pytest.mark.parametrize("fp64", [False, True])
@pytest.mark.parametrize("case", CASES[:3], ids=[c[0] for c in CASES[:3]])
def test_deformation_map(dr, case, fp64):
    """u_1 = y_1 - x (Eq. 1) and det grad y_1 (Fig. 7 caption) against the oracle."""
    name, n, nt, vgen, iso = case
    top, tmv = tols(fp64)
    ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, fp64)
    st = O.set_velocity(prob, v64)
    u, det, lo, hi = ctx.deformation()
    uref = O.deformation(st.v, st.d_plus, nt)
    dref = O.det_grad_y(uref)
    assert rel(np64(u), uref) < top
    # det is stored in the field precision: near-volume-preserving maps (det - 1 ~ 1e-4) are compared
    # absolutely, not through the relative error of det - 1
    assert rel(np64(det), dref) < top and np.abs(np64(det) - dref).max() < 10 * top
    assert abs(lo - dref.min()) < 10 * top and abs(hi - dref.max()) < 10 * top


@pytest.mark.parametrize("newton", [False, True])
def test_solver_on_synthetic_problem(dr, newton):
    """The paper's synthetic problem at 16^3, n_t = 4, H2, beta = 1e-2, g_tol = 1e-2:
    the GPU's Armijo (G)N-Krylov run follows the fp64 oracle's run iteration by iteration."""
    n, nt = 16, 4
    rT, rT64 = prep(synth.rho_t_paper(n), False)
    vs, vs64 = prep(synth.v_star(n), False)
    prob0 = O.Problem(rho_T=rT64, rho_R=rT64, nt=nt, reg=2, beta=1e-2)
    rR64 = O.set_velocity(prob0, vs64).rho[-1]
    rR, rR64 = prep(torch.from_numpy(rR64), False)
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=2, beta=1e-2)
    vref, hist_ref, reason_ref = O.solve(prob, np.zeros_like(vs64), gtol=1e-2, max_newton=20, newton=newton)
    ctx = dr.Context(dr.Config(n=n, nt=nt, reg=2, beta=1e-2, newton=newton))
    ctx.set_images(rT.cuda(), rR.cuda())
    v = torch.zeros((3, n, n, n), dtype=torch.float32, device="cuda")
    rep, hist = ctx.solve(v, gtol=1e-2, max_newton=20)
    assert rep["reason"] == reason_ref == "converged"
    assert rep["iterations"] == len(hist_ref) and [h[2] for h in hist] == [h[2] for h in hist_ref]
    for a, b in zip(hist, hist_ref):
        assert abs(a[0] - b[0]) < 1e-4 * abs(b[0]) and abs(a[1] - b[1]) < 1e-3 and a[3] == b[3]
    assert rel(np64(v), vref) < 1e-3
    _, det, lo, hi = ctx.deformation(want_u=False)
    assert lo > 0


def test_overlap_stream_matvec_same_bits(dr, monkeypatch):
    """DR_OVERLAP=1 (beta A vt on a second stream concurrent with the transport sweeps) runs the same
    kernels on the same data: bit-identical H vt."""
    n = (32, 16, 64)
    out = []
    for ov in ("0", "1"):
        monkeypatch.setenv("DR_OVERLAP", ov)  # read at dr_create
        ctx, prob, v64 = setup_case(dr, "smooth_aniso", n, 4, lambda n_: synth.smooth_vec(9, n_, kmax=4, cells_per_step=2.0, nt=4),
                                    False, False)
        ctx.forward_solve()
        vt = synth.round32(synth.smooth_vec(21, n, kmax=5)).contiguous().cuda()
        out.append(ctx.hessian_matvec(vt))
    assert torch.equal(out[0], out[1])


def test_tma_middle_same_bits(dr, monkeypatch):
    """The preconditioner's fp32 x3 middle pass through tensor-map TMA tiles (256 planes) against the
    one-tile-per-CTA pass: same arithmetic, bit-identical z."""
    n = (64, 32, 256)
    u = synth.round32(synth.smooth_vec(6, n, kmax=5)).contiguous().cuda()
    out = []
    for tm in ("0", "1"):
        monkeypatch.setenv("DR_TMA_MIDDLE", tm)  # read at dr_create
        ctx = dr.Context(dr.Config(n=n, nt=2, reg=2, beta=0.37))
        out.append(ctx.precond_apply(u))
    assert torch.equal(out[0], out[1])


def test_pcg_graph_matches_host_loop(dr, monkeypatch):
    """The CUDA-graph PCG iteration (device scalars, captured once per context) reproduces the host-scalar
    loop bit for bit, including a second solve that replays the cached graph."""
    name, n, nt, vgen, iso = CASES[1]
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("DR_GRAPHS", mode)
        ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
        ctx.forward_solve()
        g, _ = prep(synth.smooth_vec(41, n, kmax=6), False)
        a = ctx.pcg(g.cuda(), 0.05, 20)
        b = ctx.pcg((2 * g).contiguous().cuda(), 0.05, 20)
        outs[mode] = (a, b)
    for (da, ia, ra), (db, ib, rb) in zip(outs["1"], outs["0"]):
        assert ia == ib and ra == rb and torch.equal(da, db)


def test_pcg_graph_with_overlap_stream(dr, monkeypatch):
    """DR_OVERLAP=1 inside the captured PCG iteration: the matvec forks beta A vt onto the aux stream
    and joins back into the capture stream (it used to join into the context stream, which
    broke the capture).  Same bits as the serial matvec, and the cached graph replays."""
    name, n, nt, vgen, iso = CASES[2]
    outs = {}
    for ov in ("0", "1"):
        monkeypatch.setenv("DR_OVERLAP", ov)
        monkeypatch.setenv("DR_GRAPHS", "1")
        ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
        ctx.forward_solve()
        g, _ = prep(synth.smooth_vec(41, n, kmax=6), False)
        outs[ov] = (ctx.pcg(g.cuda(), 0.05, 20), ctx.pcg((2 * g).contiguous().cuda(), 0.05, 20))
    for (da, ia, ra), (db, ib, rb) in zip(outs["0"], outs["1"]):
        assert ia == ib and ra == rb and torch.equal(da, db)


def test_window_gather_same_bits_as_pair_path(dr, monkeypatch):
    """The sliding-window fp32 gather (k_sl_window) against the pair path (k_sl_gather, DR_WINDOW=0) on
    every transport of the hot path (departure points, multiplier, state, adjoint, matvec): the zero-
    padded weights add exact zeros and the non-zero terms are summed in the same order, so the bits
    agree.  The stress case (9 cells/step) mixes window warps, pair-path warps and global tiles."""
    for case in (CASES[1], CASES[2], CASES[3]):
        name, n, nt, vgen, iso = case
        res = {}
        for w in ("0", "1"):
            monkeypatch.setenv("DR_WINDOW", w)
            ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
            ctx.forward_solve()
            ctx.adjoint_solve()
            vt = synth.round32(synth.smooth_vec(21, n, kmax=5)).contiguous().cuda()
            res[w] = [ctx.get_departure(1), ctx.get_departure(-1), ctx.get_field(dr.DR_FIELD_MULTIPLIER),
                      ctx.get_field(dr.DR_FIELD_STATE, nt), ctx.get_field(dr.DR_FIELD_ADJOINT, 0),
                      ctx.hessian_matvec(vt), ctx.get_field(dr.DR_FIELD_BTILDE)]
        for a, b in zip(res["0"], res["1"]):
            assert torch.equal(a, b), name


def test_call_graphs_match_eager(dr, monkeypatch):
    """dr_hessian_matvec / dr_precond_apply replayed from the context's cached CUDA graphs (default) give
    the bits of eager execution (DR_GRAPHS=0): the first call (capture + launch), replays, a second
    argument pair, and a new velocity (one rank: the same graphs replayed -- they read the velocity's
    products from fixed workspace slots).  The profiler's per-kernel launch counts agree (its events are
    record nodes retargeted at every replay)."""
    name, n, nt, vgen, iso = CASES[2]
    res, prof = {}, {}
    for mode in ("0", "1"):
        monkeypatch.setenv("DR_GRAPHS", mode)
        ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
        ctx.forward_solve()
        vts = [synth.round32(synth.smooth_vec(21 + i, n, kmax=5)).contiguous().cuda() for i in range(2)]
        Hs = [torch.empty_like(vts[0]) for _ in range(2)]
        Zs = [torch.empty_like(vts[0]) for _ in range(2)]
        out = []
        for rep in range(3):
            for i in range(2):
                ctx.hessian_matvec(vts[i], Hs[i])
                ctx.precond_apply(Hs[i], Zs[i])
                out += [Hs[i].clone(), Zs[i].clone()]
        ctx.set_velocity(synth.round32(synth.smooth_vec(9, n, kmax=4, cells_per_step=1.0, nt=nt)).contiguous().cuda())
        ctx.forward_solve()
        for i in range(2):
            ctx.hessian_matvec(vts[i], Hs[i])
            ctx.precond_apply(Hs[i], Zs[i])
            out += [Hs[i].clone(), Zs[i].clone()]
        ctx.profile_reset()
        ctx.profile_enable(True)
        for i in range(2):
            ctx.hessian_matvec(vts[i], Hs[i])
            ctx.precond_apply(Hs[i], Zs[i])
        torch.cuda.synchronize()
        p, launches = ctx.profile()
        ctx.profile_enable(False)
        out += [Hs[0].clone(), Zs[1].clone()]
        res[mode] = out
        prof[mode] = ({t: k for t, (k, ms) in p.items()}, launches)
        assert all(ms > 0 for t, (k, ms) in p.items()), p
    for a, b in zip(res["0"], res["1"]):
        assert torch.equal(a, b)
    assert prof["0"] == prof["1"]


# N1 = N2 = 256 planes take the fused x1/x2 cluster transforms (plane2d.cuh) in fp32 contexts; n3 = 32
# (96 plane items) is not a multiple of the resident cluster count, so clusters finish on different planes
PLANE_GRIDS = [(256, 256, 8), (256, 256, 32)]


@pytest.mark.parametrize("n", PLANE_GRIDS, ids=["x".join(map(str, g)) for g in PLANE_GRIDS])
def test_plane2d_spectral_ops(dr, n, monkeypatch):
    """(DR_PLANE2D=1, opt-in: measured slower than the per-axis passes) grad, div, beta A (H1, H2), (beta A)^-1 (isochoric and not), Leray through the fused plane
    transforms against the oracle, with modes up to |k| = 80 along x1/x2 (and n3/3 along x3) and white
    noise with Nyquist content; the profiler shows the fused kernels ran."""
    monkeypatch.setenv("DR_PLANE2D", "1")
    tol = TOL32_OP
    f, f64 = prep(synth.blobs(5, n, kcut=80), False)
    u, u64 = prep(synth.smooth_vec(6, n, kmax=min(n) // 3), False)
    f, u = f.cuda(), u.cuda()
    for reg in (1, 2):
        ctx = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37))
        ctx.profile_reset()
        ctx.profile_enable(True)
        if reg == 1:
            assert rel(np64(ctx.op_spectral(dr.DR_OP_GRAD, f)), O.grad(f64)) < tol
            assert rel(np64(ctx.op_spectral(dr.DR_OP_DIV, u)), O.div(u64)) < tol
            assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, u)), O.leray(u64)) < tol
        assert rel(np64(ctx.op_spectral(dr.DR_OP_REG, u)), O.reg_apply(u64, reg, 0.37)) < tol
        assert rel(np64(ctx.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, False)) < tol
        torch.cuda.synchronize()
        p, _ = ctx.profile()
        assert any(t.startswith("plane_fwd") for t in p) and any(t.startswith("plane_inv") for t in p), p
        ci = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=0.37, isochoric=True))
        assert rel(np64(ci.op_spectral(dr.DR_OP_PRECOND, u)), O.precond(u64, reg, 0.37, True)) < tol
    w = torch.from_numpy(np.random.default_rng(3).standard_normal((3,) + tuple(n)[::-1]))
    w, w64 = prep(w, False)
    ctx = dr.Context(dr.Config(n=n, nt=2, reg=1, beta=0.37))
    assert rel(np64(ctx.op_spectral(dr.DR_OP_PRECOND, w.cuda())), O.precond(w64, 1, 0.37, False)) < tol
    assert rel(np64(ctx.op_spectral(dr.DR_OP_LERAY, w.cuda())), O.leray(w64)) < tol


@pytest.mark.parametrize("iso", [False, True])
def test_plane2d_matvec(dr, iso, monkeypatch):
    """(DR_PLANE2D=1) One GN matvec through the fused plane transforms (non-isochoric: the three components batched,
    b~ added in the inverse kernel's epilogue; isochoric: the KIND-6 path per component)."""
    monkeypatch.setenv("DR_PLANE2D", "1")
    n, nt = (256, 256, 8), 2
    ctx = dr.Context(dr.Config(n=n, nt=nt, reg=2, beta=1e-2, isochoric=iso))
    rT, rT64 = prep(synth.blobs(11, n, kcut=2), False)
    rR, rR64 = prep(synth.blobs(12, n, kcut=2), False)
    v, v64 = prep(synth.smooth_vec(9, n, kmax=2, divfree=iso, cells_per_step=1.5, nt=nt), False)
    ctx.set_images(rT.cuda(), rR.cuda())
    ctx.set_velocity(v.cuda())
    prob = O.Problem(rho_T=rT64, rho_R=rR64, nt=nt, reg=2, beta=1e-2, iso=iso)
    vt, vt64 = prep(synth.smooth_vec(21, n, kmax=2, divfree=iso), False)
    check_matvec(dr, ctx, prob, v64, vt, vt64, False, iso)


def test_plane2d_close_to_axis_passes(dr, monkeypatch):
    """The fused plane transforms against the per-axis passes (DR_PLANE2D=0) on the same inputs: the
    same transforms up to the rounding of the two-real-in-one split of columns 0 and N1/2."""
    n = (256, 256, 16)
    u = synth.round32(synth.smooth_vec(6, n, kmax=40)).contiguous().cuda()
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("DR_PLANE2D", mode)  # (the per-axis passes are the default)
        ctx = dr.Context(dr.Config(n=n, nt=2, reg=2, beta=0.37))
        out[mode] = [np64(ctx.op_spectral(k, u)) for k in (dr.DR_OP_REG, dr.DR_OP_PRECOND, dr.DR_OP_LERAY)]
    for a, b in zip(out["0"], out["1"]):
        assert rel(a, b) < 2e-6


@pytest.mark.parametrize("ring", ["4", "8"])
def test_ring_chunks_same_bits(dr, monkeypatch, ring):
    """x1/x2 pass pairs run per plane chunk through the scratch ring (DR_RING) give the bits of the
    whole-field passes: the same line transforms, only their order and the intermediate's address change
    (beta A, (beta A)^-1 and a matvec with b~ added in the c2r)."""
    name, n, nt, vgen, iso = CASES[1]
    out = {}
    for mode in ("0", ring):
        monkeypatch.setenv("DR_RING", mode)
        ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
        ctx.forward_solve()
        vt = synth.round32(synth.smooth_vec(21, n, kmax=5)).contiguous().cuda()
        out[mode] = [ctx.op_spectral(dr.DR_OP_REG, vt), ctx.op_spectral(dr.DR_OP_PRECOND, vt), ctx.hessian_matvec(vt)]
    for a, b in zip(out["0"], out[ring]):
        assert torch.equal(a, b)


def test_pairs_gather_same_bits_as_pair_path(dr, monkeypatch):
    """The shared-plane pair gather (k_sl_pairs, DR_PAIRS=1, opt-in: measured slower)
    against the default pair path on every transport of the hot path: the zero x3 weights add exact
    zeros and the non-zero terms are summed in the same order, deferred pairs use the same two-pointer
    arithmetic, so the bits agree.  The stress case mixes deferred pairs and global-memory tiles."""
    for case in (CASES[1], CASES[2], CASES[3]):
        name, n, nt, vgen, iso = case
        res = {}
        for w in ("0", "1"):
            monkeypatch.setenv("DR_PAIRS", w)
            ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
            ctx.forward_solve()
            ctx.adjoint_solve()
            vt = synth.round32(synth.smooth_vec(21, n, kmax=5)).contiguous().cuda()
            res[w] = [ctx.get_departure(1), ctx.get_departure(-1), ctx.get_field(dr.DR_FIELD_MULTIPLIER),
                      ctx.get_field(dr.DR_FIELD_STATE, nt), ctx.get_field(dr.DR_FIELD_ADJOINT, 0),
                      ctx.hessian_matvec(vt), ctx.get_field(dr.DR_FIELD_BTILDE)]
        for a, b in zip(res["0"], res["1"]):
            assert torch.equal(a, b), name


def test_gather_tma_staging_same_bits(dr, monkeypatch):
    """Gather boxes staged by the TMA engine (default: k_sl_gather_tma, tiles whose planned box does not
    wrap) against cp.async staging only (DR_GATHER_TMA=0): the same values land in the same shared-memory
    layout, so every transport of the hot path gives the same bits (the stress case mixes TMA tiles,
    wrapping cp.async tiles and global-memory tiles)."""
    for case in (CASES[1], CASES[2], CASES[3]):
        name, n, nt, vgen, iso = case
        res = {}
        for w in ("0", "1"):
            monkeypatch.setenv("DR_GATHER_TMA", w)
            ctx, prob, v64 = setup_case(dr, name, n, nt, vgen, iso, False)
            ctx.forward_solve()
            ctx.adjoint_solve()
            vt = synth.round32(synth.smooth_vec(21, n, kmax=5)).contiguous().cuda()
            res[w] = [ctx.get_departure(1), ctx.get_departure(-1), ctx.get_field(dr.DR_FIELD_MULTIPLIER),
                      ctx.get_field(dr.DR_FIELD_STATE, nt), ctx.get_field(dr.DR_FIELD_ADJOINT, 0),
                      ctx.hessian_matvec(vt), ctx.get_field(dr.DR_FIELD_BTILDE)]
        for a, b in zip(res["0"], res["1"]):
            assert torch.equal(a, b), name


@pytest.mark.parametrize("fp64", [False, True])
def test_nonfinite_inputs_rejected(dr, fp64):
    """DR_CHECK_FINITE (SURVEY §8(b) DR_ERR_NONFINITE): a NaN or Inf in an image, the velocity, a matvec
    probe or a preconditioner input -- device or host buffer -- returns DR_ERR_NONFINITE before any
    work; finite inputs give the bits of an unchecked context."""
    n = 16
    cfg = dr.Config(n=n, nt=2, fp64=fp64, check_finite=True)
    dt = torch.float64 if fp64 else torch.float32
    ctx = dr.Context(cfg)
    ref = dr.Context(dr.Config(n=n, nt=2, fp64=fp64))
    f = synth.blobs(1, n, kcut=4).to(dt).cuda()
    v = synth.smooth_vec(2, n, kmax=3, cells_per_step=1.0, nt=2).to(dt).cuda()
    vt = synth.smooth_vec(3, n, kmax=3).to(dt).cuda()

    def bad(x, val, host=False):
        y = x.clone()
        y.view(-1)[y.numel() // 3] = val
        return y.cpu() if host else y

    for val in (float("nan"), float("inf")):
        for host in (False, True):
            with pytest.raises(dr.DiffRegError) as e:
                ctx.set_images(bad(f, val, host), f.cpu() if host else f)
            assert e.value.status == dr.DR_ERR_NONFINITE
            with pytest.raises(dr.DiffRegError) as e:
                ctx.set_velocity(bad(v, val, host))
            assert e.value.status == dr.DR_ERR_NONFINITE
    for c in (ctx, ref):
        c.set_images(f, f)
        c.set_velocity(v)
        c.forward_solve()
    with pytest.raises(dr.DiffRegError) as e:
        ctx.hessian_matvec(bad(vt, float("nan")))
    assert e.value.status == dr.DR_ERR_NONFINITE
    with pytest.raises(dr.DiffRegError) as e:
        ctx.precond_apply(bad(vt, float("-inf")))
    assert e.value.status == dr.DR_ERR_NONFINITE
    assert torch.equal(ctx.hessian_matvec(vt), ref.hessian_matvec(vt))
    assert torch.equal(ctx.precond_apply(vt), ref.precond_apply(vt))
