"""bench.py's multi-GPU entry point on CPU: `bench.py --gpus N` without a torchrun environment
re-launches itself as N ranks (one process per GPU), and fails loudly when fewer than N GPUs are
visible.  The launch itself is stubbed (DR_BENCH_DRYRUN prints the command)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def run(args, **env):
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    e.update(env)
    return subprocess.run([sys.executable, BENCH, *args], capture_output=True, text=True, env=e, timeout=300)


def test_too_few_gpus_fails_loudly():
    r = run(["--gpus", "2", "--steps", "1", "--warmup", "3"], DR_BENCH_VISIBLE_GPUS="1")
    assert r.returncode != 0
    assert "needs 2 visible GPUs" in r.stderr and "found 1" in r.stderr


def test_relaunches_as_n_ranks_over_loopback():
    r = run(["--gpus", "8", "--steps", "4", "--warmup", "3"], DR_BENCH_VISIBLE_GPUS="8", DR_BENCH_DRYRUN="1")
    assert r.returncode == 0, r.stderr
    cmd = json.loads(r.stdout.strip().splitlines()[-1])["launch"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "--nnodes=1" in cmd and "--master-addr=127.0.0.1" in cmd
    i = cmd.index(BENCH)
    assert cmd[i + 1:] == ["--gpus", "8", "--steps", "4", "--warmup", "3"]


def test_algorithmic_bytes_follow_survey_8d():
    """The roofline numerators: per-launch §8(d) values summed over one matvec give 21 n_t + 47 values
    per voxel (131 at n_t = 4), the preconditioner 30."""
    sys.path.insert(0, ROOT)
    import bench
    n, nt = 64, 4
    M4 = 4 * n ** 3
    mv = (bench.algo_bytes("inc_init", n, nt) + (nt - 1) * bench.algo_bytes("sl_inc_state", n, nt)
          + bench.algo_bytes("sl_inc_state_b", n, nt) + nt * bench.algo_bytes("sl_inc_adjoint_q2", n, nt)
          + sum(bench.algo_bytes(t, n, nt) for t in ("row_r2c_f64_x3", "col_fft_fwd_f64_x3", "col_middle_f64_x3",
                                                      "col_fft_inv_x3", "row_c2r_add_x3")))
    assert abs(mv / M4 - bench.MATVEC_VALUES(nt)) < 1e-6 and bench.MATVEC_VALUES(4) == 131
    pc = sum(bench.algo_bytes(t, n, nt) for t in ("row_r2c_f32_x3", "col_fft_fwd_f32_x3", "col_middle_f32_x3",
                                                  "col_fft_inv_x3", "row_c2r_x3"))
    assert pc == 30 * M4
