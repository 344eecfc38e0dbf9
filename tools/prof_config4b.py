"""Per-kernel times of one 512^3 matvec (BJ config 4 shape), isochoric and not: python tools/prof_config4b.py"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth, paper_1608_03630_b200 as dr
n, nt = 512, 4
for iso in (True, False):
    cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2, isochoric=iso)
    ctx = dr.Context(cfg)
    rT = synth.round32(synth.blobs(100, n, device="cuda")).contiguous()
    v = synth.round32(synth.smooth_vec(4, n, kmax=8, cells_per_step=3.0, nt=nt, divfree=iso, device="cuda")).contiguous()
    vt = synth.round32(synth.smooth_vec(5, n, kmax=8, divfree=iso, device="cuda")).contiguous()
    ctx.set_images(rT, rT); ctx.set_velocity(v); ctx.forward_solve()
    Hv = ctx.hessian_matvec(vt); z = ctx.precond_apply(Hv); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        ctx.hessian_matvec(vt, Hv)
    b.record(); torch.cuda.synchronize()
    print(f"iso={iso} matvec {a.elapsed_time(b)/3:.2f} ms")
    ctx.profile_reset(); ctx.profile_enable(True)
    for _ in range(3):
        ctx.hessian_matvec(vt, Hv)
    torch.cuda.synchronize()
    p, l = ctx.profile()
    ctx.profile_enable(False)
    for k, (cnt, ms) in sorted(p.items(), key=lambda x: -x[1][1]):
        print(f"   {k:22s} {cnt//3:3d}/mv {ms / cnt * 1000:9.1f} us  {ms/3:7.3f} ms/mv")
    del ctx; torch.cuda.empty_cache()
