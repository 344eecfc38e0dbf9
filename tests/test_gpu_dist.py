"""Slab decomposition on one GPU: P virtual ranks in one process (loopback communicator,
one host thread + one stream per rank) against the single-rank library on the same inputs.

Pins: the per-point arithmetic of every gather, FFT line, symbol and quadrature is the
same on slabs as on the whole grid, so departure points, states, adjoints, gradients, the Hessian
matvec and the preconditioner must agree bit for bit; a loose 1e-6 relative bound is asserted as well
in case a future pass reorders a sum.  The single-rank path itself is held to the oracle by
test_gpu_parity.py."""
import threading

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dr():
    from paper_1608_03630_b200 import build
    build.build()
    import paper_1608_03630_b200 as m
    m.lib()
    return m


def rel(a, b):
    a = a.double().cpu().numpy().ravel()
    b = b.double().cpu().numpy().ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def run_ranks(P, fn):
    """fn(rank) on P threads; re-raises the first failure."""
    out, err = [None] * P, []

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def pipeline(ctx, rT, rR, v, vt):
    """The library's full hot path on one context; returns every observable it exposes."""
    dr = pytest.importorskip("paper_1608_03630_b200")
    F = dr.diffreg
    ctx.set_images(rT, rR)
    ctx.set_velocity(v)
    res = {"d+": ctx.get_departure(+1), "d-": ctx.get_departure(-1), "vel": ctx.get_field(F.DR_FIELD_VELOCITY)}
    if not ctx.cfg.isochoric:
        res["m"] = ctx.get_field(F.DR_FIELD_MULTIPLIER)
    ctx.forward_solve()
    nt = ctx.cfg.nt
    for j in range(nt + 1):
        res[f"rho{j}"] = ctx.get_field(F.DR_FIELD_STATE, j)
        res[f"G{j}"] = ctx.get_field(F.DR_FIELD_STATE_GRAD, j)
    ctx.adjoint_solve()
    res["lam0"] = ctx.get_field(F.DR_FIELD_ADJOINT, 0)
    res["Hv"] = ctx.hessian_matvec(vt)
    res["bt"] = ctx.get_field(F.DR_FIELD_BTILDE)
    res["z"] = ctx.precond_apply(vt)
    res["reg"] = ctx.op_spectral(F.DR_OP_REG, vt)
    res["leray"] = ctx.op_spectral(F.DR_OP_LERAY, vt)
    res["div"] = ctx.op_spectral(F.DR_OP_DIV, vt)
    res["grad"] = ctx.gradient()
    J, mis = ctx.objective()
    dv, it, rr = ctx.pcg(vt, 0.0, 2)
    res["pcg"] = dv
    u, det, lo, hi = ctx.deformation()
    res["u"], res["det"] = u, det
    ctx.sync()
    out = {k: t.clone() for k, t in res.items()}
    out["_J"] = (J, mis)
    return out


CASES = [
    # n, nt, iso, velocity (max displacement must stay within the 4/5 ghost planes along x3)
    # [, full Newton]
    ((32, 32, 32), 4, False, lambda n: synth.smooth_vec(9, n, kmax=4, cells_per_step=2.0, nt=4)),
    ((64, 32, 16), 2, True, lambda n: synth.smooth_vec(5, n, kmax=3, cells_per_step=1.5, nt=2, divfree=True)),
    ((16, 64, 32), 4, False, lambda n: synth.v_star(n)),
    ((32, 32, 32), 2, False, lambda n: synth.smooth_vec(14, n, kmax=4, cells_per_step=1.5, nt=2), True),
    ((32, 16, 32), 2, True, lambda n: synth.smooth_vec(15, n, kmax=3, cells_per_step=1.5, nt=2, divfree=True), True),
]


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_slabs_match_single_rank(dr, P, case):
    n, nt, iso, vgen = CASES[case][:4]
    newton = len(CASES[case]) > 4 and CASES[case][4]
    D = dr.dist
    cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2, isochoric=iso, newton=newton)
    if dr.diffreg.dr_workspace_bytes_dist(cfg, P) == 0:
        pytest.skip("grid not divisible into P slabs")
    rT = synth.round32(synth.blobs(11, n, kcut=6)).cuda()
    rR = synth.round32(synth.blobs(12, n, kcut=6)).cuda()
    v = synth.round32(vgen(n)).cuda()
    vt = synth.round32(synth.smooth_vec(13, n, kmax=4)).cuda()
    ref = pipeline(dr.Context(cfg), rT, rR, v, vt)

    hub = dr.diffreg.Hub(P)
    comms = [hub.comm(r) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [dr.Context(cfg, stream=streams[r], comm=comms[r]) for r in range(P)]
    torch.cuda.synchronize()
    sl = lambda x, r: D.slab_of(x, cfg, P, r)  # noqa: E731
    ins = [(sl(rT, r), sl(rR, r), sl(v, r), sl(vt, r)) for r in range(P)]
    torch.cuda.synchronize()

    def rank(r):
        with torch.cuda.stream(streams[r]):
            out = pipeline(ctxs[r], *ins[r])
        streams[r].synchronize()
        return out

    outs = run_ranks(P, rank)
    for o in outs:  # the objective is a collective: every rank holds the same sum (rank-order partials)
        assert o["_J"] == outs[0]["_J"]
        assert abs(o["_J"][0] - ref["_J"][0]) <= 1e-12 * abs(ref["_J"][0])
        assert abs(o["_J"][1] - ref["_J"][1]) <= 1e-12 * abs(ref["_J"][1]) + 1e-300
    for k, full in ref.items():
        if k == "_J":
            continue
        got = D.assemble([o[k] for o in outs])
        assert got.shape == full.shape, k
        assert rel(got, full) < 1e-6, (k, rel(got, full))
        if k != "pcg":  # PCG's inner products sum per-rank partials: equal to rounding, not bitwise
            assert torch.equal(got, full), (k, rel(got, full))
    for c in ctxs:
        c.close()
    for c in comms:
        c.close()
    hub.close()


def test_widened_ghosts_carry_large_displacement(dr):
    """~6 cells/step (BASELINE config 5's displacement) with ghost planes (7, 8): bit-identical to one rank."""
    P, n = 2, (32, 16, 32)
    cfg = dr.Config(n=n, nt=2, ghost_lo=7, ghost_hi=8)
    rT = synth.round32(synth.blobs(21, n, kcut=5)).cuda()
    v = synth.round32(synth.smooth_vec(22, n, kmax=2, cells_per_step=6.0, nt=2)).cuda()
    vt = synth.round32(synth.smooth_vec(23, n, kmax=3)).cuda()
    ref = pipeline(dr.Context(cfg), rT, rT, v, vt)
    hub = dr.diffreg.Hub(P)
    comms = [hub.comm(r) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [dr.Context(cfg, stream=streams[r], comm=comms[r]) for r in range(P)]
    sl = lambda x, r: dr.dist.slab_of(x, cfg, P, r)  # noqa: E731
    ins = [(sl(rT, r), sl(rT, r), sl(v, r), sl(vt, r)) for r in range(P)]
    torch.cuda.synchronize()

    def rank(r):
        with torch.cuda.stream(streams[r]):
            out = pipeline(ctxs[r], *ins[r])
        streams[r].synchronize()
        return out

    outs = run_ranks(P, rank)
    for k, full in ref.items():
        if k == "_J":
            continue
        assert torch.equal(dr.dist.assemble([o[k] for o in outs]), full), k


@pytest.mark.parametrize("P,cells", [(2, 6.0), (4, 9.0)])
def test_scatter_of_far_departure_points(dr, P, cells):
    """Displacements beyond the default (4, 5) ghost planes -- up to 9 cells with 8-plane slabs, i.e.
    owners two slabs away -- go through the off-rank scatter (Alg. 1): owners interpolate
    the requested cells and return the values; the whole pipeline stays bit-identical to one rank."""
    n = (16, 16, 32)
    cfg = dr.Config(n=n, nt=2)
    rT = synth.round32(synth.blobs(24, n, kcut=5)).cuda()
    rR = synth.round32(synth.blobs(25, n, kcut=5)).cuda()
    v = synth.round32(synth.smooth_vec(4, n, kmax=2, cells_per_step=cells, nt=2)).cuda()
    vt = synth.round32(synth.smooth_vec(26, n, kmax=3)).cuda()
    ref = pipeline(dr.Context(cfg), rT, rR, v, vt)
    hub = dr.diffreg.Hub(P)
    comms = [hub.comm(r) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [dr.Context(cfg, stream=streams[r], comm=comms[r]) for r in range(P)]
    sl = lambda x, r: dr.dist.slab_of(x, cfg, P, r)  # noqa: E731
    ins = [(sl(rT, r), sl(rR, r), sl(v, r), sl(vt, r)) for r in range(P)]
    torch.cuda.synchronize()

    def rank(r):
        with torch.cuda.stream(streams[r]):
            out = pipeline(ctxs[r], *ins[r])
        streams[r].synchronize()
        return out

    outs = run_ranks(P, rank)
    for k, full in ref.items():
        if k == "_J":
            continue
        got = dr.dist.assemble([o[k] for o in outs])
        assert rel(got, full) < 1e-6, (k, rel(got, full))
        if k != "pcg":
            assert torch.equal(got, full), (k, rel(got, full))


def test_nccl_communicator_single_rank(dr):
    """The real NCCL backend (dlopen'ed libnccl.so.2, grouped ncclSend/ncclRecv) on the one GPU this box
    has: a 1-rank communicator passes the exchange self-test and carries a slab context's matvec."""
    uid = dr.diffreg.nccl_unique_id()
    comm = dr.diffreg.Comm.nccl(uid, 0, 1)
    assert comm.selftest()
    n = (16, 16, 16)
    cfg = dr.Config(n=n, nt=2)
    rT = synth.round32(synth.blobs(31, n, kcut=4)).cuda()
    v = synth.round32(synth.smooth_vec(32, n, kmax=2, cells_per_step=1.0, nt=2)).cuda()
    vt = synth.round32(synth.smooth_vec(33, n, kmax=3)).cuda()
    a = pipeline(dr.Context(cfg, comm=comm), rT, rT, v, vt)
    b = pipeline(dr.Context(cfg), rT, rT, v, vt)
    for k in b:
        if k != "_J":
            assert torch.equal(a[k], b[k]), k
    comm.close()


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_communicator_selftest(dr, P):
    hub = dr.diffreg.Hub(P)
    comms = [hub.comm(r) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    assert run_ranks(P, lambda r: comms[r].selftest(streams[r])) == [True] * P


def run_slabs(dr, cfg, P, ins_full, profile=False):
    """The pipeline on P loopback ranks (contexts created in this thread, so they see the current
    environment); returns per-rank outputs and, with profile, each rank's profiler tags."""
    hub = dr.diffreg.Hub(P)
    comms = [hub.comm(r) for r in range(P)]
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [dr.Context(cfg, stream=streams[r], comm=comms[r]) for r in range(P)]
    sl = lambda x, r: dr.dist.slab_of(x, cfg, P, r)  # noqa: E731
    ins = [tuple(sl(x, r) for x in ins_full) for r in range(P)]
    torch.cuda.synchronize()

    def rank(r):
        with torch.cuda.stream(streams[r]):
            if profile:
                ctxs[r].profile_reset()
                ctxs[r].profile_enable(True)
            out = pipeline(ctxs[r], *ins[r])
            if profile:
                out["_prof"] = ctxs[r].profile()[0]
        streams[r].synchronize()
        return out

    outs = run_ranks(P, rank)
    for c in ctxs:
        c.close()
    for c in comms:
        c.close()
    hub.close()
    return outs


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("case", [0, 1, 3])
def test_peer_ghosts_match_single_rank(dr, monkeypatch, P, case):
    """Fused ghost exchange (DR_PEER_GHOSTS=1, include/diffreg.h dr_peer_export): the producing gathers
    store their boundary planes into the neighbours' ghosts through peer pointers (the other loopback
    contexts' workspaces) and the consumers only wait for their neighbours; the x2 forward pass and the
    x3 middle pass store their transpose chunks into the owning ranks' buffers -- every observable of the
    pipeline (state, adjoint, GN / full-Newton matvec, gradient, deformation map) stays bit-identical to
    one rank, and the profiler shows the neighbour barriers that replaced the ghost exchanges."""
    n, nt, iso, vgen = CASES[case][:4]
    newton = len(CASES[case]) > 4 and CASES[case][4]
    cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2, isochoric=iso, newton=newton)
    if dr.diffreg.dr_workspace_bytes_dist(cfg, P) == 0:
        pytest.skip("grid not divisible into P slabs")
    rT = synth.round32(synth.blobs(11, n, kcut=6)).cuda()
    rR = synth.round32(synth.blobs(12, n, kcut=6)).cuda()
    v = synth.round32(vgen(n)).cuda()
    vt = synth.round32(synth.smooth_vec(13, n, kmax=4)).cuda()
    ref = pipeline(dr.Context(cfg), rT, rR, v, vt)
    monkeypatch.setenv("DR_PEER_GHOSTS", "1")
    outs = run_slabs(dr, cfg, P, (rT, rR, v, vt), profile=True)
    for o in outs:  # neighbour barriers replaced ghost exchanges, all-rank barriers the transposes
        assert "peer_sync" in o["_prof"] and "peer_barrier" in o["_prof"], sorted(o["_prof"])
    for k, full in ref.items():
        if k in ("_J", "_prof"):
            continue
        got = dr.dist.assemble([o[k] for o in outs])
        if k != "pcg":
            assert torch.equal(got, full), (k, rel(got, full))
        else:
            assert rel(got, full) < 1e-6


@pytest.mark.parametrize("P,cells", [(2, 6.0), (4, 9.0)])
def test_peer_ghosts_with_far_departure_points(dr, monkeypatch, P, cells):
    """Peer-stored ghosts together with the off-rank scatter (points beyond the ghosts: owners interpolate
    through their peer-filled ghosts, requesters' fixups peer-store boundary values): bit-identical."""
    n = (16, 16, 32)
    cfg = dr.Config(n=n, nt=2)
    rT = synth.round32(synth.blobs(24, n, kcut=5)).cuda()
    rR = synth.round32(synth.blobs(25, n, kcut=5)).cuda()
    v = synth.round32(synth.smooth_vec(4, n, kmax=2, cells_per_step=cells, nt=2)).cuda()
    vt = synth.round32(synth.smooth_vec(26, n, kmax=3)).cuda()
    ref = pipeline(dr.Context(cfg), rT, rR, v, vt)
    monkeypatch.setenv("DR_PEER_GHOSTS", "1")
    outs = run_slabs(dr, cfg, P, (rT, rR, v, vt))
    for k, full in ref.items():
        if k == "_J":
            continue
        got = dr.dist.assemble([o[k] for o in outs])
        if k != "pcg":
            assert torch.equal(got, full), (k, rel(got, full))
