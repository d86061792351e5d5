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


def log_table():
    """Reduction table of musr_log_fast (musr_math.cuh), 128 entries.

    x = 2^k z with z in [OFF, 2 OFF), OFF = 0x3fe6000000000000 (0.6875); entry i
    covers the z whose bit pattern lies in OFF + [i, i+1) * 2^45.  invc =
    RN(1/c) for the interval midpoint c; the two entries around 1.0 (79, 80)
    use c = 1 exactly, so r = z - 1 is exact there and log(x) near 1 keeps full
    relative accuracy.  logc = -log(invc) as a double-double (hi, lo)."""
    import struct
    off = 0x3fe6000000000000
    asd = lambda u: struct.unpack("<d", struct.pack("<Q", u))[0]
    out = []
    for i in range(128):
        lo, hi = asd(off + (i << 45)), asd(off + ((i + 1) << 45))
        invc = 1.0 if i in (79, 80) else float(1 / ((mp.mpf(lo) + mp.mpf(hi)) / 2))
        L = -mp.log(mp.mpf(invc))
        h = float(L)
        out.append((invc, h, float(L - mp.mpf(h))))
    print("... musr_log_t[128 * 4] = {  // invc, logc_hi, logc_lo, 0  (see musr_math.cuh)")
    for invc, h, l in out:
        print(f"    {invc.hex()}, {h.hex()}, {l.hex()}, 0.0,")
    print("};")
    return out


def log1p_tail():
    """(log1p(r) - r) / r^2 on |r| <= 2^-7, degree 5 (error 7e-18 of log1p(r))."""
    a, b = -mp.mpf(2) ** -7, mp.mpf(2) ** -7 * (1 + mp.mpf(10) ** -30)
    f = lambda r: (mp.mpf(-0.5) + r / 3) if abs(r) < mp.mpf(10) ** -25 else (mp.log1p(r) - r) / r ** 2
    return fit(f, a, b, 6, "(log1p(r) - r) / r^2")
