"""Coefficients of the fast-mode erf (dmath.cuh kErfSmall): erf(x) = x P(x^2) on
|x| <= 1.5, P of degree 13 from a Chebyshev fit of erf(sqrt(u))/sqrt(u) on
u in [0, 2.25] with mpmath at 40 digits.  Prints the coefficients (highest
degree first) and the max error of a double-precision Horner evaluation."""
import math
import struct

import mpmath as mp
import numpy as np

mp.mp.dps = 40
T, DEG = 1.5, 13


def f(u):
    if u == 0:
        return 2 / mp.sqrt(mp.pi)
    s = mp.sqrt(u)
    return mp.erf(s) / s


poly, err = mp.chebyfit(f, [0, T * T], DEG + 1, error=True)
print("fit error", mp.nstr(err, 3))
cs = [float(c) for c in poly]
for c in cs:
    print("%.17e  %s" % (c, hex(struct.unpack("<Q", struct.pack("<d", c))[0])))
worst = 0.0
for t in np.linspace(1e-6, T, 20001):
    u = t * t
    p = cs[0]
    for c in cs[1:]:
        p = p * u + c
    ref = float(mp.erf(mp.mpf(t)))
    worst = max(worst, abs(t * p - ref) / ref / 2.220446049250313e-16)
print("max error (ulp of erf, double Horner without FMA)", round(worst, 2))
