"""Secondary measurements (not the bench.py contract line): per-call device times of the hot path on
BASELINE.json configs 3 (256^3, n_t = 4, H2, non-isochoric) and 4 (512^3, n_t = 4, H2, isochoric, one
GPU), with the SURVEY §8(d) algorithmic bytes per matvec (21 n_t + 47 / 20 n_t + 59 fp32 values per
voxel).  Prints one JSON object per config."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_1608_03630_b200 as dr  # noqa: E402

PEAK = 6443.2


def timeit(fn, reps):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run(n, nt, iso, cells, reps=5):
    cfg = dr.Config(n=n, nt=nt, reg=dr.DR_REG_H2, beta=1e-2, isochoric=iso)
    ctx = dr.Context(cfg)
    rT = synth.round32(synth.blobs(100, n, device="cuda")).contiguous()
    rR = synth.round32(synth.blobs(101, n, device="cuda")).contiguous()
    v = synth.round32(synth.smooth_vec(4 if iso else 3, n, kmax=8, cells_per_step=cells, nt=nt, divfree=iso,
                                       device="cuda")).contiguous()
    vt = synth.round32(synth.smooth_vec(5, n, kmax=8, divfree=iso, device="cuda")).contiguous()
    Hv = torch.empty_like(vt)
    z = torch.empty_like(vt)
    ctx.set_images(rT, rR)

    def setup():
        ctx.set_velocity(v)
        ctx.forward_solve()

    setup()
    ctx.hessian_matvec(vt, Hv)
    t_setup = timeit(setup, 2)
    t_mv = timeit(lambda: ctx.hessian_matvec(vt, Hv), reps)
    t_pc = timeit(lambda: ctx.precond_apply(Hv, z), reps)
    M = n ** 3
    vals = (20 * nt + 59) if iso else (21 * nt + 47)
    gbs = vals * 4 * M / (t_mv * 1e-3) / 1e9
    return {"config": f"{n}^3 nt={nt} H2 {'isochoric' if iso else 'non-isochoric'} {cells} cells/step",
            "matvec_ms": t_mv, "matvecs_per_s": 1e3 / t_mv, "precond_ms": t_pc, "setup_ms": t_setup,
            "voxel_steps_per_s": 2 * nt * M / (t_mv * 1e-3), "algorithmic_values_per_voxel": vals,
            "algorithmic_GBs": gbs, "frac_of_measured_hbm": gbs / PEAK,
            "workspace_GB": dr.dr_workspace_bytes(cfg) / 1e9}


if __name__ == "__main__":
    out = [run(256, 4, False, 2.0), run(512, 4, True, 3.0)]
    for o in out:
        print(json.dumps(o))
