"""Random quartic families for the quartic-minimiser microbench
(BASELINE.json configs[4]; paper §III-C "Generate N random sets of quartic
coefficients").

  family 'C' (config-literal "convex" quartics): A ~ U[0.1, 10], B ~ U[-10, 10],
      C = 3 B^2 / (8 A) + U[0, 10], D ~ U[-10, 10]  -> J'' >= 0 everywhere.
  family 'R' (paper-style random): A ~ U[0.1, 10]; B, C, D ~ U[-10, 10].
  box: lo, hi = sorted(U[-5, 5]^2).

Generated with torch so the same call can fill host or device memory; the CPU
and CUDA generators give different streams for one seed, so parity tests copy
the device-resident inputs back rather than regenerating them.  Pure data
generation -- no arithmetic of the method.
"""

from __future__ import annotations


def quartic_family(family: str, N: int, seed: int = 190310041, device="cpu"):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed * 7 + (0 if family == "C" else 1))
    f64 = torch.float64

    def U(lo, hi):
        return torch.rand(N, generator=g, dtype=f64, device=device) * (hi - lo) + lo

    A = U(0.1, 10.0)
    B = U(-10.0, 10.0)
    if family == "C":
        C = 3.0 * B * B / (8.0 * A) + U(0.0, 10.0)
    elif family == "R":
        C = U(-10.0, 10.0)
    else:
        raise ValueError(f"unknown quartic family {family!r}")
    D = U(-10.0, 10.0)
    u = U(-5.0, 5.0)
    v = U(-5.0, 5.0)
    lo = torch.minimum(u, v)
    hi = torch.maximum(u, v)
    return A, B, C, D, lo, hi
