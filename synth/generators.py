"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the registration method (no transport, no
interpolation, no spectral operator of the paper).  It only draws seeded random
numbers and synthesises band-limited periodic fields from closed-form Fourier
coefficients (SURVEY.md §8(d) G1–G5).  Both sides of every parity test receive the
same arrays from here; neither side imports the other.

Conventions:
  * grid n = (N1, N2, N3); x_a = 2*pi*i_a/N_a on [0, 2*pi)^3 (§III-B1);
  * scalar arrays have shape (N3, N2, N1) -- x1 fastest, C order (index i1 + N1*(i2 + N2*i3));
  * vector arrays have shape (3, N3, N2, N1) (SoA);
  * everything is produced in float64; `round32` rounds once to float32 and the oracle
    consumes the rounded values promoted back to float64.

The paper measures on its synthetic problem (§IV-A1) and on NIREP
brain MRI (not in this container).  G1/G3 are the paper's synthetic problem; G5
("blobs") stands in for image statistics of BASELINE.json configs 3-5.
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np
import torch

TWO_PI = 2.0 * math.pi


def _dims(n) -> tuple[int, int, int]:
    if isinstance(n, int):
        return (n, n, n)
    n = tuple(int(x) for x in n)
    assert len(n) == 3
    return n


def grid_coords(n, device="cpu"):
    """Return broadcastable coordinate arrays x1 (1,1,N1), x2 (1,N2,1), x3 (N3,1,1) in float64."""
    N1, N2, N3 = _dims(n)
    x1 = torch.arange(N1, dtype=torch.float64, device=device) * (TWO_PI / N1)
    x2 = torch.arange(N2, dtype=torch.float64, device=device) * (TWO_PI / N2)
    x3 = torch.arange(N3, dtype=torch.float64, device=device) * (TWO_PI / N3)
    return x1.view(1, 1, N1), x2.view(1, N2, 1), x3.view(N3, 1, 1)


# --------------------------------------------------------------------------- G1-G3

def rho_t_paper(n, device="cpu") -> torch.Tensor:
    """G1: rho_T = (sin^2 x1 + sin^2 x2 + sin^2 x3)/3  (§IV-A1)."""
    x1, x2, x3 = grid_coords(n, device)
    return (torch.sin(x1) ** 2 + torch.sin(x2) ** 2 + torch.sin(x3) ** 2) / 3.0


def v_cfg1(n, device="cpu") -> torch.Tensor:
    """G2: 0.5*(sin x3 cos x2 sin x2, sin x1 cos x3 sin x3, sin x2 cos x1 sin x1) (BASELINE.json config 1).

    Divergence-free: component a does not depend on x_a.
    """
    x1, x2, x3 = grid_coords(n, device)
    N1, N2, N3 = _dims(n)
    shape = (N3, N2, N1)
    v = torch.empty((3,) + shape, dtype=torch.float64, device=device)
    v[0] = (0.5 * torch.sin(x3) * torch.cos(x2) * torch.sin(x2)).expand(shape)
    v[1] = (0.5 * torch.sin(x1) * torch.cos(x3) * torch.sin(x3)).expand(shape)
    v[2] = (0.5 * torch.sin(x2) * torch.cos(x1) * torch.sin(x1)).expand(shape)
    return v


def v_star(n, device="cpu") -> torch.Tensor:
    """G3: v* = (cos x1 sin x2, cos x2 sin x1, cos x1 sin x3)  (§IV-A1). Not div-free."""
    x1, x2, x3 = grid_coords(n, device)
    N1, N2, N3 = _dims(n)
    shape = (N3, N2, N1)
    v = torch.empty((3,) + shape, dtype=torch.float64, device=device)
    v[0] = (torch.cos(x1) * torch.sin(x2)).expand(shape)
    v[1] = (torch.cos(x2) * torch.sin(x1)).expand(shape)
    v[2] = (torch.cos(x1) * torch.sin(x3)).expand(shape)
    return v


# --------------------------------------------------------------------------- spectral synthesis helpers

def _fft_index(k: np.ndarray, N: int) -> np.ndarray:
    return np.mod(k, N)


def _synth_real(coeffs: Sequence[tuple[np.ndarray, np.ndarray]], n, device) -> torch.Tensor:
    """Evaluate u(x) = Re sum_k c_k exp(i k.x) on the grid, given (K[count,3] int, c[count] complex).

    Uses numpy's DFT convention: F[k] accumulates M*c/2 at k and M*conj(c)/2 at -k; u = ifftn(F).real.
    Exact grid evaluation (aliased modes accumulate into the same bin).
    """
    N1, N2, N3 = _dims(n)
    M = N1 * N2 * N3
    out = []
    for K, c in coeffs:
        F = torch.zeros((N3, N2, N1), dtype=torch.complex128, device=device)
        ct = torch.as_tensor(c, dtype=torch.complex128, device=device) * (M / 2.0)
        for sgn, val in ((1, ct), (-1, torch.conj(ct))):
            i1 = torch.as_tensor(_fft_index(sgn * K[:, 0], N1), device=device)
            i2 = torch.as_tensor(_fft_index(sgn * K[:, 1], N2), device=device)
            i3 = torch.as_tensor(_fft_index(sgn * K[:, 2], N3), device=device)
            F.index_put_((i3, i2, i1), val, accumulate=True)
        out.append(torch.fft.ifftn(F).real)
        del F
    return torch.stack(out)


def _modes(kmax: int) -> np.ndarray:
    """All integer k in [-kmax, kmax]^3 with 0 < |k|_2 <= kmax, lexicographic in (k1, k2, k3)."""
    r = np.arange(-kmax, kmax + 1)
    K = np.stack(np.meshgrid(r, r, r, indexing="ij"), axis=-1).reshape(-1, 3)
    k2 = (K * K).sum(axis=1)
    return K[(k2 > 0) & (k2 <= kmax * kmax)]


def smooth_vec(seed: int, n, kmax: int = 8, divfree: bool = False, rms: float | None = 1.0,
               cells_per_step: float | None = None, nt: int | None = None, device="cpu") -> torch.Tensor:
    """G4: random smooth vector field with Gaussian Fourier coefficients, |k| <= kmax (BASELINE.json config 2).

    For each component a and each mode k (lexicographic, 0 < |k| <= kmax) draw c_a(k) = (xi + i eta)/sqrt(2),
    xi, eta ~ N(0,1) from numpy.random.default_rng(seed), in the order (a, k, [xi, eta]).
    u_a = Re sum_k c_a(k) e^{ik.x}.

    divfree=True returns the curl of that field instead: u_hat(k) = i k x c(k) (exactly divergence-free
    at every mode; this is NOT the paper's Leray operator, which stays out of this module).

    Scaling: if cells_per_step is given, scale so that max_{a,i} |u_a| * (1/nt) / h_a == cells_per_step;
    else if rms is given, scale to unit-RMS * rms over all components.
    """
    N1, N2, N3 = _dims(n)
    K = _modes(kmax)
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((3, K.shape[0], 2))
    c = (z[..., 0] + 1j * z[..., 1]) / math.sqrt(2.0)  # (3, count)
    if divfree:
        kc = K.astype(np.float64)
        # (i k x c)_a
        cu = np.empty_like(c)
        cu[0] = 1j * (kc[:, 1] * c[2] - kc[:, 2] * c[1])
        cu[1] = 1j * (kc[:, 2] * c[0] - kc[:, 0] * c[2])
        cu[2] = 1j * (kc[:, 0] * c[1] - kc[:, 1] * c[0])
        c = cu
    u = _synth_real([(K, c[a]) for a in range(3)], (N1, N2, N3), device)
    if cells_per_step is not None:
        assert nt is not None and nt >= 1
        h = torch.tensor([TWO_PI / N1, TWO_PI / N2, TWO_PI / N3], dtype=torch.float64, device=device)
        cells = (u.abs().amax(dim=(1, 2, 3)) / nt / h).max()
        u = u * (cells_per_step / cells)
    elif rms is not None:
        u = u * (rms / torch.sqrt((u * u).mean()).clamp_min(1e-300))
    return u


def blobs(seed: int, n, nblobs: int = 16, kcut: float = 64.0, device="cpu") -> torch.Tensor:
    """G5: sum of `nblobs` periodised anisotropic Gaussians, band-limited to |k|_2 <= kcut (BASELINE.json cfg 3-5).

    Per blob, in draw order: centre c ~ U[0,2pi)^3, sigma ~ U[0.1,0.4]^3, amplitude alpha ~ U[0.5,1].
    rho_hat(k) = sum_b alpha_b prod_a (sigma_ba/sqrt(2pi)) exp(-sigma_ba^2 k_a^2/2 - i k_a c_ba) for |k| <= kcut.
    Synthesis: F = M * rho_hat on the FFT index range k_a in [-N_a/2+1, N_a/2]; rho = Re ifftn(F).
    """
    N1, N2, N3 = _dims(n)
    M = N1 * N2 * N3
    rng = np.random.default_rng(seed)
    params = []
    for _ in range(nblobs):
        cen = rng.uniform(0.0, TWO_PI, 3)
        sig = rng.uniform(0.1, 0.4, 3)
        amp = rng.uniform(0.5, 1.0)
        params.append((cen, sig, amp))

    def kvec(N):
        i = torch.arange(N, dtype=torch.float64, device=device)
        return torch.where(i <= N // 2, i, i - N)

    k1, k2, k3 = kvec(N1), kvec(N2), kvec(N3)
    F = torch.zeros((N3, N2, N1), dtype=torch.complex128, device=device)
    for cen, sig, amp in params:
        f1 = (sig[0] / math.sqrt(TWO_PI)) * torch.exp(-0.5 * sig[0] ** 2 * k1 ** 2 - 1j * k1 * cen[0])
        f2 = (sig[1] / math.sqrt(TWO_PI)) * torch.exp(-0.5 * sig[1] ** 2 * k2 ** 2 - 1j * k2 * cen[1])
        f3 = (sig[2] / math.sqrt(TWO_PI)) * torch.exp(-0.5 * sig[2] ** 2 * k3 ** 2 - 1j * k3 * cen[2])
        F += amp * (f3.view(N3, 1, 1) * f2.view(1, N2, 1) * f1.view(1, 1, N1))
    kk = k3.view(N3, 1, 1) ** 2 + k2.view(1, N2, 1) ** 2 + k1.view(1, 1, N1) ** 2
    F = torch.where(kk <= kcut * kcut, F, torch.zeros((), dtype=F.dtype, device=device))
    F *= M
    return torch.fft.ifftn(F).real


def blobs_direct(seed: int, n, nblobs: int = 16, nimg: int = 3) -> np.ndarray:
    """Direct periodised Gaussian sum (no band limit), for pinning `blobs` at kcut large (tests only)."""
    N1, N2, N3 = _dims(n)
    rng = np.random.default_rng(seed)
    out = np.zeros((N3, N2, N1))
    xs = [np.arange(N) * TWO_PI / N for N in (N1, N2, N3)]
    for _ in range(nblobs):
        cen = rng.uniform(0.0, TWO_PI, 3)
        sig = rng.uniform(0.1, 0.4, 3)
        amp = rng.uniform(0.5, 1.0)
        g = []
        for a in range(3):
            x = xs[a]
            s = sum(np.exp(-((x - cen[a] + TWO_PI * m) ** 2) / (2 * sig[a] ** 2)) for m in range(-nimg, nimg + 1))
            g.append(s)
        out += amp * g[2][:, None, None] * g[1][None, :, None] * g[0][None, None, :]
    return out


def round32(x: torch.Tensor) -> torch.Tensor:
    """Round once to float32 (the GPU input) ..."""
    return x.to(torch.float32)


def promote64(x: torch.Tensor) -> np.ndarray:
    """... and promote the rounded values back to float64 for the oracle."""
    return x.detach().to("cpu", torch.float64).numpy().copy()
