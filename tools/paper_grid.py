"""One GN matvec on the paper's 256 x 300 x 256 grid (x2 by Bluestein): time per matvec and the
per-kernel table.  python tools/paper_grid.py"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth, paper_1608_03630_b200 as dr
n, nt = (256, 300, 256), 4
cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2)
ctx = dr.Context(cfg)
rT = synth.round32(synth.blobs(100, n, device="cuda")).contiguous()
rR = synth.round32(synth.blobs(101, n, device="cuda")).contiguous()
v = synth.round32(synth.smooth_vec(3, n, kmax=8, cells_per_step=2.0, nt=nt, device="cuda")).contiguous()
vt = synth.round32(synth.smooth_vec(1000, n, kmax=8, device="cuda")).contiguous()
ctx.set_images(rT, rR); ctx.set_velocity(v); ctx.forward_solve()
Hv = ctx.hessian_matvec(vt); z = ctx.precond_apply(Hv); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    ctx.hessian_matvec(vt, Hv)
b.record(); torch.cuda.synchronize()
print(f"256x300x256 GN matvec {a.elapsed_time(b)/5:.3f} ms")
ctx.profile_reset(); ctx.profile_enable(True)
ctx.hessian_matvec(vt, Hv); ctx.precond_apply(Hv, z)
torch.cuda.synchronize()
p, l = ctx.profile()
ctx.profile_enable(False)
for k, (cnt, ms) in sorted(p.items(), key=lambda x: -x[1][1]):
    print(f"   {k:22s} {cnt:3d} x {ms / cnt * 1000:9.1f} us")
