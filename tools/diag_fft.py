"""Diagnostic: accuracy of the GPU spectral passes vs fp64 and vs a float32 CPU FFT (scipy)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.fft as sf, torch
import synth
import paper_1608_03630_b200 as dr
from oracle import oracle as O

def rel(a, b): return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))
for n in [(32, 16, 64), (64, 64, 64), (16, 16, 16)]:
    u = synth.round32(synth.smooth_vec(6, n, kmax=5))
    u64 = synth.promote64(u)
    for reg in (1, 2):
        ctx = dr.Context(dr.Config(n=n, nt=2, reg=reg, beta=1.0))
        g = ctx.op_spectral(dr.DR_OP_REG, u.cuda()).cpu().double().numpy()
        ref = O.reg_apply(u64, reg, 1.0)
        N1, N2, N3 = n
        k1 = np.fft.fftfreq(N1, 1 / N1); k2 = np.fft.fftfreq(N2, 1 / N2); k3 = np.fft.fftfreq(N3, 1 / N3)
        kk = k3[:, None, None] ** 2 + k2[None, :, None] ** 2 + k1[None, None, :] ** 2
        a = (kk ** reg).astype(np.float32)
        sc = np.stack([sf.ifftn(sf.fftn(u.numpy()[c]) * a).real for c in range(3)])
        print(n, "reg", reg, "gpu", rel(g, ref), "scipy32", rel(sc, ref))
    ctx = dr.Context(dr.Config(n=n, nt=2))
    f = synth.round32(synth.blobs(5, n, kcut=5))
    gg = ctx.op_spectral(dr.DR_OP_GRAD, f.cuda()).cpu().double().numpy()
    print(n, "grad", rel(gg, O.grad(synth.promote64(f))), [rel(gg[a], O.grad(synth.promote64(f))[a]) for a in range(3)])
    # precond and leray
    print(n, "precond", rel(ctx.op_spectral(dr.DR_OP_PRECOND, u.cuda()).cpu().double().numpy(), O.precond(u64, 2, 1e-2, False)))
    print(n, "leray", rel(ctx.op_spectral(dr.DR_OP_LERAY, u.cuda()).cpu().double().numpy(), O.leray(u64)))
    # single modes through REG (H1): sin(k.x) for a few k
    x1, x2, x3 = [t.numpy() for t in synth.grid_coords(n)]
    for kv in [(1, 0, 0), (0, 1, 0), (0, 0, 1), (3, 2, 5), (N1 // 2 - 1, 0, 0), (0, N2 // 2 - 1, 0), (0, 0, N3 // 2 - 1)]:
        s = np.broadcast_to(np.sin(kv[0] * x1 + kv[1] * x2 + kv[2] * x3), (N3, N2, N1))
        uu = torch.tensor(np.stack([s, s, s]), dtype=torch.float32)
        ctx1 = dr.Context(dr.Config(n=n, nt=2, reg=1, beta=1.0))
        out = ctx1.op_spectral(dr.DR_OP_REG, uu.cuda()).cpu().double().numpy()
        exp = sum(k * k for k in kv) * synth.promote64(uu)
        print("   mode", kv, rel(out, exp))
