"""Generate the near-minimax polynomial coefficients used by masw_det.cuh (mpmath).

Chebyshev fits (mpmath.chebyfit, 50 digits) in u = r^2, coefficients rounded to fp64 and
re-checked at 2001 points for the maximum relative error:
    E(u) = (cosh r - 1)/r^2, O(u) = sinh r / r     on |r| <= ln2/2   (degree 5)
    S(u) = sin r / r                               on |r| <= pi/4    (degree 6)
    C(u) = cos r                                   on |r| <= pi/4    (degree 7)
"""
import mpmath as mp

mp.mp.dps = 50


def fit(f, hi, deg):
    poly = mp.chebyfit(f, [0, hi], deg + 1)
    cs = [float(c) for c in poly]
    xs = [hi * i / 2000 for i in range(2001)]
    rel = max(abs(mp.polyval([mp.mpf(c) for c in cs], x) - f(x)) / abs(f(x)) for x in xs)
    return cs, rel


def main():
    ue = (mp.log(2) / 2) ** 2
    ut = (mp.pi / 4) ** 2
    sq = mp.sqrt
    specs = [
        ("c_expE", lambda u: (mp.cosh(sq(u)) - 1) / u if u else mp.mpf(1) / 2, ue, 5),
        ("c_expO", lambda u: mp.sinh(sq(u)) / sq(u) if u else mp.mpf(1), ue, 5),
        ("c_sin", lambda u: mp.sin(sq(u)) / sq(u) if u else mp.mpf(1), ut, 6),
        ("c_cos", lambda u: mp.cos(sq(u)), ut, 7),
    ]
    for name, f, hi, deg in specs:
        cs, rel = fit(f, hi, deg)
        print(f"{name}: max rel err {mp.nstr(rel, 3)}")
        print("   {" + ", ".join(repr(c) for c in cs) + "}")


if __name__ == "__main__":
    main()
