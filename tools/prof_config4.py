import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import synth, paper_1608_03630_b200 as dr
n, nt = 512, 4
cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2, isochoric=True)
ctx = dr.Context(cfg)
rT = synth.round32(synth.blobs(100, n, device="cuda")).contiguous()
v = synth.round32(synth.smooth_vec(4, n, kmax=8, cells_per_step=3.0, nt=nt, divfree=True, device="cuda")).contiguous()
vt = synth.round32(synth.smooth_vec(5, n, kmax=8, divfree=True, device="cuda")).contiguous()
ctx.set_images(rT, rT); ctx.set_velocity(v); ctx.forward_solve()
Hv = ctx.hessian_matvec(vt); z = ctx.precond_apply(Hv); torch.cuda.synchronize()
ctx.profile_reset(); ctx.profile_enable(True)
for _ in range(3):
    ctx.hessian_matvec(vt, Hv)
p, l = ctx.profile()
for k, (cnt, ms) in sorted(p.items(), key=lambda x: -x[1][1]):
    print(k, cnt, round(ms / cnt * 1000, 1), 'us')
