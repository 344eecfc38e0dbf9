"""Cost of the library's per-kernel CUDA-event profiler on the bench step: the same 256^3 step timed
with dr_profile_enable on and off (alternating, 3 rounds each)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1608_03630_b200 as dr  # noqa: E402

n, dev = 256, torch.device("cuda", 0)
ctx = dr.Context(dr.Config(n=n, nt=bench.NT, reg=dr.DR_REG_H2, beta=1e-2), device=dev)
rT, rR, v, vts = bench.make_inputs(n, dev)
ctx.set_images(rT, rR)
Hv = [torch.empty_like(vts[0]) for _ in vts]
Z = [torch.empty_like(vts[0]) for _ in vts]


def step():
    ctx.set_velocity(v)
    ctx.forward_solve()
    ctx.adjoint_solve()
    for i in range(len(vts)):
        ctx.hessian_matvec(vts[i], Hv[i])
        ctx.precond_apply(Hv[i], Z[i])


def timed(prof, steps=5):
    ctx.profile_reset()
    ctx.profile_enable(prof)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ctx.stream)
    for _ in range(steps):
        step()
    b.record(ctx.stream)
    torch.cuda.synchronize()
    ctx.profile_enable(False)
    return a.elapsed_time(b) / steps


for _ in range(3):
    step()
res = {True: [], False: []}
for _ in range(3):
    for p in (True, False):
        res[p].append(timed(p))
print({("profiler on" if k else "profiler off"): [round(x, 3) for x in v] for k, v in res.items()})
