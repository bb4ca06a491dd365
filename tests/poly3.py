"""Exact polynomial oracle (test infrastructure), restating tests/oracles.cpp:9-113.

Polynomials in (xi1, xi2, xi3) with rational coefficients; closed-form
integrals over the reference prism (triangle x [-1, 1]):
  int_T xi1^a xi2^b = a! b! / (a+b+2)!      (oracles.cpp:9-18)
  int_{-1}^{1} xi3^c = 2/(c+1), c even      (oracles.cpp:20-23)
"""
from fractions import Fraction
from math import factorial

# Legendre monomial coefficients, constant term first (oracles.cpp:86-98).
LEGENDRE = {
    0: [1], 1: [0, 1], 2: [Fraction(-1, 2), 0, Fraction(3, 2)],
    3: [0, Fraction(-3, 2), 0, Fraction(5, 2)],
    4: [Fraction(3, 8), 0, Fraction(-30, 8), 0, Fraction(35, 8)],
    5: [0, Fraction(15, 8), 0, Fraction(-70, 8), 0, Fraction(63, 8)],
    6: [Fraction(-5, 16), 0, Fraction(105, 16), 0, Fraction(-315, 16), 0, Fraction(231, 16)],
    7: [0, Fraction(-35, 16), 0, Fraction(315, 16), 0, Fraction(-693, 16), 0, Fraction(429, 16)],
}


class Poly3:
    def __init__(self, terms=None):
        self.t = {k: v for k, v in (terms or {}).items() if v != 0}

    @staticmethod
    def monomial(a, b, c, coeff=1):
        return Poly3({(a, b, c): Fraction(coeff)})

    def __add__(self, o):
        t = dict(self.t)
        for k, v in o.t.items():
            t[k] = t.get(k, 0) + v
        return Poly3(t)

    def __mul__(self, o):
        t = {}
        for ka, va in self.t.items():
            for kb, vb in o.t.items():
                k = (ka[0] + kb[0], ka[1] + kb[1], ka[2] + kb[2])
                t[k] = t.get(k, 0) + va * vb
        return Poly3(t)

    def derivative(self, axis):
        t = {}
        for k, v in self.t.items():
            if k[axis] == 0:
                continue
            kk = list(k)
            kk[axis] -= 1
            t[tuple(kk)] = t.get(tuple(kk), 0) + v * k[axis]
        return Poly3(t)

    def integral_over_reference_prism(self):
        s = Fraction(0)
        for (a, b, c), v in self.t.items():
            if c % 2:
                continue
            s += v * Fraction(factorial(a) * factorial(b), factorial(a + b + 2)) * Fraction(2, c + 1)
        return s


def triangle_monomials(p):
    """(a, b) ordered by total degree, then a (reference_element.cpp:195-205)."""
    return [(a, d - a) for d in range(p + 1) for a in range(d + 1)]


def basis_polynomial(p, dof):
    """Basis function dof = tri*(p+1) + k (oracles.cpp:100-113)."""
    tri = triangle_monomials(p)
    t, k = divmod(dof, p + 1)
    a, b = tri[t]
    out = Poly3()
    for c, coeff in enumerate(LEGENDRE[k]):
        if coeff:
            out = out + Poly3.monomial(a, b, c, coeff)
    return out
