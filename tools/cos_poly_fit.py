"""Fit and check the single cos polynomial of csrc/cupso_device.cuh:cos_pso.

cos(p) = (-1)^k P(r^2), k = rint(p / pi), r = p - k*pi (3-part Cody-Waite),
P = the degree-8 interpolant of cos(sqrt z) at Chebyshev nodes of
[0, (pi/2)^2 * 1.0001], solved in 80-bit long double. The check emulates the
device arithmetic (FMA = one rounding of the long-double a*b+c) against glibc
cos over the griewank (|p| <= 600) and rastrigin (p = fl(2pi * v), |v| <= 5.12)
argument ranges.

    python tools/cos_poly_fit.py
"""
import math

import numpy as np

L = np.longdouble
PI = L("3.14159265358979323846264338327950288")
P1, P2, P3 = 3.14159265358979311600e+00, 1.22464679914735317723e-16, -2.99476980971833966425e-33
INVPI = 0.31830988618379067154


def fit(deg=8, zmax=float((PI / 2) ** 2 * L(1.0001))):
    n = deg + 1
    x = np.cos(PI * (np.arange(n).astype(L) + L(0.5)) / L(n))
    z = (x + 1) * L(zmax) / 2
    A = np.array([[zz ** k for k in range(n)] for zz in z], dtype=L)
    b = np.cos(np.sqrt(z))
    for i in range(n):  # Gaussian elimination, partial pivoting, long double
        p = i + int(np.argmax(abs(A[i:, i])))
        A[[i, p]], b[[i, p]] = A[[p, i]], b[[p, i]]
        for r in range(i + 1, n):
            f = A[r, i] / A[i, i]
            A[r, i:] -= f * A[i, i:]
            b[r] -= f * b[i]
    c = np.zeros(n, dtype=L)
    for i in range(n - 1, -1, -1):
        c[i] = (b[i] - np.dot(A[i, i + 1:], c[i + 1:])) / A[i, i]
    return [float(v) for v in c]


def fma(a, b, c):
    return float(np.float64(L(a) * L(b) + L(c)))


def cos_dev(p, coef):
    big = 6755399441055744.0
    t = fma(p, INVPI, big)
    k = t - big
    r = fma(-k, P3, fma(-k, P2, fma(-k, P1, p)))
    z = r * r
    q = coef[-1]
    for c in coef[-2::-1]:
        q = fma(q, z, c)
    return -q if int(k) & 1 else q


def main():
    coef = fit()
    print("P0..P8 =", coef)
    rng = np.random.default_rng(1)
    ps = np.concatenate([rng.uniform(-600, 600, 100000), np.arange(-400, 401) * math.pi / 2])
    e = np.array([abs(cos_dev(float(p), coef) - math.cos(p)) for p in ps])
    print(f"griewank range: max abs err {e.max():.3g}, bit-identical {100 * (e == 0).mean():.1f}%")
    vs = rng.uniform(-5.12, 5.12, 100000)
    te = np.array([abs(((v * v - 10 * math.cos(6.283185307179586 * v)) + 10)
                       - ((v * v - 10 * cos_dev(6.283185307179586 * v, coef)) + 10)) for v in vs])
    print(f"rastrigin terms: max abs err {te.max():.3g}, bit-identical {100 * (te == 0).mean():.1f}%")


if __name__ == "__main__":
    main()
