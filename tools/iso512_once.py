"""One 512^3 isochoric matvec after setup (for ncu launch lists): python tools/iso512_once.py [n]"""
import sys, os, torch
sys.path.insert(0, os.getcwd())
import synth, paper_1608_03630_b200 as dr
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nt = 4
cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2, isochoric=True)
ctx = dr.Context(cfg)
rT = synth.round32(synth.blobs(100, n, device="cuda")).contiguous()
v = synth.round32(synth.smooth_vec(4, n, kmax=8, cells_per_step=3.0, nt=nt, divfree=True, device="cuda")).contiguous()
vt = synth.round32(synth.smooth_vec(5, n, kmax=8, divfree=True, device="cuda")).contiguous()
ctx.set_images(rT, rT); ctx.set_velocity(v); ctx.forward_solve()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
Hv = ctx.hessian_matvec(vt)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", float(Hv.norm()))
