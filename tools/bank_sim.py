"""Shared-memory bank-conflict model of the gather's stencil loads (CPU, numpy).

For the bench workload's displacement (v = smooth_vec(3) at 2 cells/step, d ~ v dt / h) this counts,
for every warp-wide LDS of k_sl_gather (lanes = 32 consecutive x at one (y, z); the 64 loads
(a, b, c) of the tricubic stencil), the conflict degree = max over the 32 banks of the number of
distinct 4-byte words the lanes read in that bank.  Used to explain ncu's "LDS wavefronts / ideal"
and to try box layouts / lane mappings before writing them."""
import sys
import os
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402


def degree(addr):
    """addr: (W, 32) int word addresses -> (W,) conflict degree."""
    bank = addr % 32
    out = np.ones(addr.shape[0], dtype=np.int64)
    for b in range(32):
        m = bank == b
        # distinct addresses per bank per warp
        a = np.where(m, addr, -1)
        a.sort(axis=1)
        distinct = ((a[:, 1:] != a[:, :-1]) & (a[:, 1:] >= 0)).sum(axis=1) + (a[:, 0] >= 0)
        out = np.maximum(out, distinct)
    return out


def main(n=256, nwarps=20000, seed=0):
    v = synth.smooth_vec(3, n, kmax=8, cells_per_step=2.0, nt=4).double().numpy()  # (3, z, y, x)
    h = 2 * np.pi / n
    d = v * (1.0 / 4) / h  # cells per step
    rng = np.random.default_rng(seed)
    ys = rng.integers(0, n, nwarps)
    zs = rng.integers(0, n, nwarps)
    x0 = rng.integers(0, n // 32, nwarps) * 32
    lane = np.arange(32)
    X = (x0[:, None] + lane[None, :]) % n
    Y = np.broadcast_to(ys[:, None], X.shape)
    Z = np.broadcast_to(zs[:, None], X.shape)
    q1 = X + np.floor(-d[0][Z, Y, X]).astype(np.int64)
    q2 = Y + np.floor(-d[1][Z, Y, X]).astype(np.int64)
    q3 = Z + np.floor(-d[2][Z, Y, X]).astype(np.int64)
    span = q1.max(1) - q1.min(1)
    print(f"x-span of the warp's q1: mean {span.mean():.2f}, P(span >= 32) = {(span >= 32).mean():.3f}")
    for name, BX, PS in [("BX=64 (current)", 64, 64 * 15), ("BX=64, plane +16", 64, 64 * 15 + 16),
                         ("BX=72", 72, 72 * 15), ("BX=65", 65, 65 * 15)]:
        degs = []
        for c in range(4):
            for b in range(4):
                for a in range(4):
                    addr = (q3 + c) * PS + (q2 + b) * BX + (q1 + a) + 10 ** 6
                    degs.append(degree(addr))
        degs = np.stack(degs)
        print(f"{name:20s} mean wavefronts/LDS {degs.mean():.3f}  (P(deg>1) = {(degs > 1).mean():.3f})")




def rotated(n=256, nwarps=20000, seed=0):
    """Per-lane tap rotation: at the a-th x1 load of each stencil row, a lane reads tap (a - s) mod 4,
    s = floor(-d1) mod 4 (a per-point rule, so every path could sum in the same order).  Lanes whose x1
    floors differ by one then read the same column offset from their own x in 3 of the 4 loads instead
    of none, so the end-lane collision of a 33-column warp span hits one load in four."""
    v = synth.smooth_vec(3, n, kmax=8, cells_per_step=2.0, nt=4).double().numpy()
    d = v * (1.0 / 4) / (2 * np.pi / n)
    rng = np.random.default_rng(seed)
    ys, zs = rng.integers(0, n, nwarps), rng.integers(0, n, nwarps)
    x0 = rng.integers(0, n // 32, nwarps) * 32
    X = (x0[:, None] + np.arange(32)[None, :]) % n
    Y, Z = np.broadcast_to(ys[:, None], X.shape), np.broadcast_to(zs[:, None], X.shape)
    f = [np.floor(-d[a][Z, Y, X]).astype(np.int64) for a in range(3)]
    q1, q2, q3 = X + f[0], Y + f[1], Z + f[2]
    s = np.mod(f[0], 4)
    # "by node column mod 4": at load a read the tap whose box column is congruent to a (mod 4) — a rule
    # of the stencil's lowest node q1 alone, so the box, global-memory and owner-side paths can all use it.
    for name, rot in (("natural order", np.zeros_like(s)), ("rotated by floor mod 4", s),
                      ("by node column mod 4", np.mod(q1, 4))):
        degs = []
        for c in range(4):
            for b in range(4):
                for a in range(4):
                    tap = np.mod(a - rot, 4)
                    degs.append(degree((q3 + c) * 64 * 15 + (q2 + b) * 64 + (q1 + tap) + 10 ** 6))
        degs = np.stack(degs)
        print(f"{name:24s} mean wavefronts/LDS {degs.mean():.3f}  (P(deg>1) = {(degs > 1).mean():.3f})")


if __name__ == "__main__":
    rotated() if "--rotated" in sys.argv else main()
