"""Small end-to-end driver for compute-sanitizer (one tool per call): the full single-rank pipeline
(set_velocity, forward/adjoint solves, GN and full-Newton matvecs, preconditioner, gradient, objective,
PCG, deformation) on a 16^3 grid, plus a 2-rank loopback slab run with far departure points (scatter)."""
import os
import sys
import threading

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1608_03630_b200 as dr  # noqa: E402


def pipeline(ctx, n, cells, seed):
    rT = synth.round32(synth.blobs(seed, n, kcut=4)).cuda()
    rR = synth.round32(synth.blobs(seed + 1, n, kcut=4)).cuda()
    v = synth.round32(synth.smooth_vec(seed + 2, n, kmax=2, cells_per_step=cells, nt=ctx.cfg.nt,
                                       divfree=ctx.cfg.isochoric)).cuda()
    vt = synth.round32(synth.smooth_vec(seed + 3, n, kmax=3, divfree=ctx.cfg.isochoric)).cuda()
    return rT, rR, v, vt


def run(ctx, rT, rR, v, vt):
    ctx.set_images(rT, rR)
    ctx.set_velocity(v)
    ctx.forward_solve()
    ctx.adjoint_solve()
    Hv = ctx.hessian_matvec(vt)
    ctx.precond_apply(Hv)
    ctx.gradient()
    ctx.objective()
    ctx.pcg(vt, 0.1, 3)
    ctx.deformation()
    ctx.sync()


n = (16, 16, 16)
for iso in (False, True):
    for newton in (False, True):
        ctx = dr.Context(dr.Config(n=n, nt=2, isochoric=iso, newton=newton))
        run(ctx, *pipeline(ctx, n, 1.5, 10))
        ctx.close()
# x2 extents that are not powers of two (Bluestein x2 passes, ragged x2 tiles)
for nb in ((16, 12, 16), (8, 20, 8)):
    for iso in (False, True):
        ctx = dr.Context(dr.Config(n=nb, nt=2, isochoric=iso))
        run(ctx, *pipeline(ctx, nb, 1.5, 30))
        ctx.close()
# slabs with scatter (isochoric with DR_SANITIZE_ISO=1: the split-layout ColDivPass and kind 9)
P, n2 = 2, (16, 16, 32)
cfg = dr.Config(n=n2, nt=2, isochoric=os.environ.get("DR_SANITIZE_ISO") == "1")
hub = dr.diffreg.Hub(P)
comms = [hub.comm(r) for r in range(P)]
streams = [torch.cuda.Stream() for _ in range(P)]
ctxs = [dr.Context(cfg, stream=streams[r], comm=comms[r]) for r in range(P)]
full = pipeline(ctxs[0], n2, 6.0, 20)
ins = [[dr.dist.slab_of(x, cfg, P, r) for x in full] for r in range(P)]
torch.cuda.synchronize()
errs = []


def body(r):
    try:
        with torch.cuda.stream(streams[r]):
            run(ctxs[r], *ins[r])
    except BaseException as e:  # noqa: BLE001
        errs.append(e)


ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
for t in ts:
    t.start()
for t in ts:
    t.join()
assert not errs, errs
print("sanitize_run: ok")
