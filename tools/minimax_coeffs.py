"""Near-minimax polynomial coefficients for dmath.cuh's exp_d / log_d
(developer tool): Chebyshev interpolation in 50-digit arithmetic, converted to
the power basis, with the max relative error measured on a dense grid.

    python tools/minimax_coeffs.py
"""
import mpmath as mp

mp.mp.dps = 50


def cheb_fit(f, a, b, deg):
    n = deg + 1
    nodes = [mp.mpf(a + b) / 2 + mp.mpf(b - a) / 2 * mp.cos(mp.pi * (k + mp.mpf(1) / 2) / n) for k in range(n)]
    # solve the Vandermonde system in high precision (interpolation at Chebyshev nodes)
    A = mp.matrix([[x ** j for j in range(n)] for x in nodes])
    y = mp.matrix([f(x) for x in nodes])
    return list(mp.lu_solve(A, y))


def max_rel_err(c, f, a, b, grid=4000):
    worst = mp.mpf(0)
    for i in range(grid + 1):
        x = a + (b - a) * mp.mpf(i) / grid
        # evaluate with float64-rounded coefficients (what the device uses)
        p = mp.mpf(0)
        for cj in reversed(c):
            p = p * x + mp.mpf(float(cj))
        worst = max(worst, abs(p / f(x) - 1))
    return worst


ln2h = mp.log(2) / 2
for deg in (7, 8, 9, 10):
    c = cheb_fit(mp.exp, -ln2h, ln2h, deg)
    print(f"exp deg {deg}: max rel err {mp.nstr(max_rel_err(c, mp.exp, -ln2h, ln2h), 3)}")
    print("  coeffs (high->low):", ", ".join(repr(float(x)) for x in reversed(c)))

zmax = ((mp.sqrt(2) - 1) / (mp.sqrt(2) + 1)) ** 2
Q = lambda z: mp.mpf(1) if z == 0 else mp.atanh(mp.sqrt(z)) / mp.sqrt(z)
for deg in (4, 5, 6, 7):
    c = cheb_fit(Q, mp.mpf(0), zmax, deg)
    print(f"log Q deg {deg}: max rel err {mp.nstr(max_rel_err(c, Q, mp.mpf(0), zmax), 3)}")
    print("  coeffs (high->low):", ", ".join(repr(float(x)) for x in reversed(c)))
