"""PCG iteration time with and without the CUDA-graph iteration (small grids are launch-bound)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_1608_03630_b200 as dr  # noqa: E402

for n in (32, 64, 128, 256):
    res = {}
    for mode in ("0", "1"):
        os.environ["DR_GRAPHS"] = mode
        ctx = dr.Context(dr.Config(n=n, nt=4))
        rT = synth.round32(synth.blobs(1, n, kcut=min(n // 3, 20), device="cuda")).contiguous()
        v = synth.round32(synth.smooth_vec(2, n, kmax=4, cells_per_step=1.5, nt=4, device="cuda")).contiguous()
        g = synth.round32(synth.smooth_vec(3, n, kmax=4, device="cuda")).contiguous()
        ctx.set_images(rT, rT)
        ctx.set_velocity(v)
        ctx.forward_solve()
        ctx.pcg(g, 0.0, 2)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, it, _ = ctx.pcg(g, 0.0, 20)
        torch.cuda.synchronize()
        res[mode] = (time.perf_counter() - t0) / it * 1e3
    print(f"{n}^3: PCG iteration {res['0']:.3f} ms host loop, {res['1']:.3f} ms graph")
