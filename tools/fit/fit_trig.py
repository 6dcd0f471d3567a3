"""Fit the polynomial kernels of the device angle functions in quartic.cuh
(build-time derivation, not run by the product or the tests).

  atan(r)   = r + r*s*PA(s),  s = r^2,  r in [0, 1]
  cos(phi)  = 1 + w*PC(w),    w = phi^2, phi in [0, pi/3]
  sin(phi)  = phi + phi*w*PS(w)

Chebyshev fits in 60-digit arithmetic (mpmath.chebyfit), coefficients rounded
to double; prints the C initialisers and the max error of the rounded
polynomials evaluated in float64 against mpmath on dense grids.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 60


def fit(f, a, b, deg):
    poly, err = mp.chebyfit(f, [a, b], deg + 1, error=True)
    return [float(c) for c in poly], float(err)  # highest degree first


def horner(c, x):
    y = np.zeros_like(x) + c[0]
    for k in c[1:]:
        y = y * x + k
    return y


def PA(s):
    if s == 0:
        return mp.mpf(-1) / 3
    r = mp.sqrt(s)
    return (mp.atan(r) / r - 1) / s


def PC(w):
    if w == 0:
        return mp.mpf(-1) / 2
    return (mp.cos(mp.sqrt(w)) - 1) / w


def PS(w):
    if w == 0:
        return mp.mpf(-1) / 6
    r = mp.sqrt(w)
    return (mp.sin(r) / r - 1) / w


W = float((mp.pi / 3) ** 2)
for name, f, a, b, degs in [("ATAN", PA, 0, 1, range(16, 24)), ("COS", PC, 0, W, range(6, 11)),
                            ("SIN", PS, 0, W, range(6, 11))]:
    for deg in degs:
        c, err = fit(f, a, b, deg)
        x = np.linspace(a, b, 20001)
        ref = np.array([float(f(mp.mpf(float(v)))) for v in x[::50]])
        got = horner(c, x[::50])
        print(f"{name} deg {deg}: fit err {err:.2e}, rounded max abs err {np.abs(got - ref).max():.2e}")
        if (name == "ATAN" and deg == 22) or (name != "ATAN" and deg == 8):
            print(f"  // {name}: degree {deg}, highest first")
            print("  {" + ", ".join(repr(v) for v in c) + "}")
