"""Derive polynomial coefficients for the device math library (musr_math.cuh).

Near-minimax fits by Chebyshev interpolation in 60-digit arithmetic
(mpmath.chebyfit), rounded to binary64.  Prints C literals and the fit error.
"""
import mpmath as mp

mp.mp.dps = 60


def fit(f, a, b, n, label):
    poly, err = mp.chebyfit(f, [a, b], n, error=True)
    coeffs = [float(c) for c in poly]          # highest degree first
    print(f"// {label}: degree {n - 1}, fit error {mp.nstr(err, 3)}")
    for c in coeffs:
        print(f"  {c.hex()},  // {c!r}")
    return coeffs, err


if __name__ == "__main__":
    ln2 = mp.log(2)
    # exp(r) on [-ln2/2, ln2/2]
    for n in (11, 12):
        fit(mp.exp, -ln2 / 2, ln2 / 2, n, "exp(r)")
    # cos(r) = C(s), s = r^2 in [0, (pi/2)^2]
    hs = (mp.pi / 2) ** 2
    for n in (10, 11, 12):
        fit(lambda s: mp.cos(mp.sqrt(s)), 0, hs, n, "cos(sqrt(s))")
    # sin(r) = r * S(s)
    for n in (10, 11, 12):
        fit(lambda s: mp.sin(mp.sqrt(s)) / mp.sqrt(s) if s != 0 else mp.mpf(1), 0, hs, n, "sin(sqrt(s))/sqrt(s)")
