"""ctypes wrappers over the CHECKERS (test infrastructure only).

* ``Oracle``    -- oracle/liboracle.so, the plain-C restatement of the reference
                   arithmetic (oracle/prism_oracle.c).
* ``Reference`` -- oracle/_ref/libprismint_ref.so, the unmodified reference
                   sources compiled by oracle/Makefile (absent when the
                   reference tree was not available at build time).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libprismint_ref.so"

_dp = C.POINTER(C.c_double)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def shape_count(p: int) -> int:
    return (p + 1) * (p + 1) * (p + 2) // 2


QUAD_COUNTS = {1: 6, 2: 18, 3: 48, 4: 80, 5: 150, 6: 231, 7: 336}


class Oracle:
    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.po_integrate_generic.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, C.POINTER(C.c_int)]
        L.po_load_vector.argtypes = [C.c_int, _dp, C.c_double, _dp]
        L.po_generate_box_mesh.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _dp]
        L.po_prism_quadrature.argtypes = [C.c_int, _dp, _dp]
        L.po_tabulate_shapes.argtypes = [C.c_int, _dp]
        L.po_jacobian_terms.argtypes = [_dp, _dp, _dp, _dp]
        L.po_elasticity_tensor.argtypes = [C.c_double, C.c_double, _dp]
        L.po_gauss_legendre.argtypes = [C.c_int, _dp, _dp]
        L.po_triangle_rule.argtypes = [C.c_int, _dp, _dp]

    def quadrature(self, p):
        nq = QUAD_COUNTS[p]
        pts = np.zeros((nq, 3))
        w = np.zeros(nq)
        assert self.lib.po_prism_quadrature(p, _ptr(pts), _ptr(w)) == nq
        return pts, w

    def shape_table(self, p):
        t = np.zeros((QUAD_COUNTS[p], 4, shape_count(p)))
        assert self.lib.po_tabulate_shapes(p, _ptr(t)) == 0
        return t

    def triangle_rule(self, degree):
        pts = np.zeros((64, 2))
        w = np.zeros(64)
        n = self.lib.po_triangle_rule(degree, _ptr(pts), _ptr(w))
        if n < 0:
            raise ValueError(f"unsupported degree {degree}")
        return pts[:n].copy(), w[:n].copy()

    def gauss_legendre(self, n):
        x = np.zeros(n)
        w = np.zeros(n)
        self.lib.po_gauss_legendre(n, _ptr(x), _ptr(w))
        return x, w

    def jacobian_terms(self, geom, xi):
        geom = np.ascontiguousarray(geom, dtype=np.float64).reshape(18)
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        det = np.zeros(1)
        inv = np.zeros(9)
        rc = self.lib.po_jacobian_terms(_ptr(geom), _ptr(xi), _ptr(det), _ptr(inv))
        return rc, det[0], inv.reshape(3, 3)

    def integrate_generic(self, p, geom, coeff, n_eq=1):
        """One element; geom [6][3], coeff [n_eq][n_eq][4][4]. Raises on inversion."""
        geom = np.ascontiguousarray(geom, dtype=np.float64).reshape(18)
        coeff = np.ascontiguousarray(coeff, dtype=np.float64).reshape(n_eq * n_eq * 16)
        dim = n_eq * shape_count(p)
        out = np.zeros((dim, dim))
        bad = C.c_int(-1)
        rc = self.lib.po_integrate_generic(p, n_eq, _ptr(geom), _ptr(coeff), _ptr(out), C.byref(bad))
        if rc == 1:
            raise InvertedElement(bad.value)
        assert rc == 0
        return out

    def integrate_batch(self, p, geoms, coeffs, n_eq=1):
        """geoms [E][6][3]; coeffs [E][...] or a single tensor."""
        geoms = np.asarray(geoms, dtype=np.float64).reshape(-1, 18)
        coeffs = np.asarray(coeffs, dtype=np.float64).reshape(-1, n_eq * n_eq * 16)
        out = [
            self.integrate_generic(p, geoms[e], coeffs[e if len(coeffs) > 1 else 0], n_eq)
            for e in range(len(geoms))
        ]
        return np.stack(out)

    def load_vector(self, p, geom, f):
        geom = np.ascontiguousarray(geom, dtype=np.float64).reshape(18)
        out = np.zeros(shape_count(p))
        assert self.lib.po_load_vector(p, _ptr(geom), float(f), _ptr(out)) == 0
        return out

    def box_mesh(self, nx, ny, nz, distortion, seed):
        out = np.zeros((2 * nx * ny * nz, 6, 3))
        assert self.lib.po_generate_box_mesh(nx, ny, nz, distortion, seed, _ptr(out)) == 0
        return out

    def elasticity_tensor(self, young, nu):
        out = np.zeros((3, 3, 4, 4))
        assert self.lib.po_elasticity_tensor(young, nu, _ptr(out)) == 0
        return out


class InvertedElement(Exception):
    def __init__(self, where):
        super().__init__(f"inverted element at {where}")
        self.where = where


class RefError(C.Structure):
    _fields_ = [("code", C.c_int), ("element", C.c_int64), ("det", C.c_double),
                ("message", C.c_char * 256)]


class Reference:
    """The reference's own arithmetic (oracle/_ref)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing (reference not built here)")
        self.lib = C.CDLL(str(path))
        L = self.lib
        L.ref_prism_quadrature.argtypes = [C.c_int, _dp, _dp, C.POINTER(RefError)]
        L.ref_tabulate_shapes.argtypes = [C.c_int, _dp, C.POINTER(RefError)]
        L.ref_generate_box_mesh.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, _dp,
                                            C.POINTER(RefError)]
        L.ref_integrate_generic_batch.argtypes = [C.c_int, C.c_int, C.c_int64, _dp, _dp, C.c_int, _dp,
                                                  C.c_int64, C.c_int, C.POINTER(RefError)]
        L.ref_integrate_optimized.argtypes = [C.c_int, _dp, C.c_double, C.c_double, _dp,
                                              C.POINTER(RefError)]
        L.ref_jacobian_terms.argtypes = [_dp, _dp, _dp, _dp, C.c_int64, C.POINTER(RefError)]
        L.ref_gauss_legendre.argtypes = [C.c_int, _dp, _dp, C.POINTER(RefError)]
        L.ref_triangle_rule.argtypes = [C.c_int, _dp, _dp, C.POINTER(RefError)]
        L.ref_elasticity_tensor.argtypes = [C.c_double, C.c_double, _dp, C.POINTER(RefError)]
        L.ref_integrate_optimized_batch.argtypes = [C.c_int, C.c_int64, _dp, _dp, _dp, C.c_int,
                                                    C.POINTER(RefError)]
        self.has_io = hasattr(L, "ref_save_stiffness")
        if self.has_io:
            L.ref_save_stiffness.argtypes = [C.c_char_p, C.c_int, C.c_int, _dp, C.c_int64, C.POINTER(RefError)]
            L.ref_load_stiffness.argtypes = [C.c_char_p, _dp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int),
                                             C.POINTER(C.c_int), C.POINTER(RefError)]

    def _check(self, rc, err):
        if rc != 0:
            raise RuntimeError(f"reference error code {rc}: {err.message.decode()} (element {err.element})")

    def quadrature(self, p):
        nq = QUAD_COUNTS[p]
        pts = np.zeros((nq, 3))
        w = np.zeros(nq)
        err = RefError()
        self._check(self.lib.ref_prism_quadrature(p, _ptr(pts), _ptr(w), C.byref(err)), err)
        return pts, w

    def shape_table(self, p):
        t = np.zeros((QUAD_COUNTS[p], 4, shape_count(p)))
        err = RefError()
        self._check(self.lib.ref_tabulate_shapes(p, _ptr(t), C.byref(err)), err)
        return t

    def box_mesh(self, nx, ny, nz, distortion, seed):
        out = np.zeros((2 * nx * ny * nz, 6, 3))
        err = RefError()
        self._check(self.lib.ref_generate_box_mesh(nx, ny, nz, distortion, seed, _ptr(out), C.byref(err)), err)
        return out

    def integrate_batch(self, p, geoms, coeffs, n_eq=1, threads=0, element_id_base=0):
        """Returns (out [E][dim][dim], err) ; err is None or a RefError."""
        geoms = np.ascontiguousarray(geoms, dtype=np.float64).reshape(-1, 18)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.float64).reshape(-1, n_eq * n_eq * 16)
        per_el = 1 if len(coeffs) > 1 else 0
        dim = n_eq * shape_count(p)
        out = np.zeros((len(geoms), dim, dim))
        err = RefError()
        rc = self.lib.ref_integrate_generic_batch(p, n_eq, len(geoms), _ptr(geoms), _ptr(coeffs), per_el,
                                                  _ptr(out), element_id_base, threads, C.byref(err))
        return out, (err if rc else None)

    def integrate_optimized(self, p, geom, young, nu):
        geom = np.ascontiguousarray(geom, dtype=np.float64).reshape(18)
        dim = 3 * shape_count(p)
        out = np.zeros((dim, dim))
        err = RefError()
        self._check(self.lib.ref_integrate_optimized(p, _ptr(geom), young, nu, _ptr(out), C.byref(err)), err)
        return out

    def save_stiffness(self, path, p, n_eq, k, element_id):
        """The reference's save_stiffness (io.cpp:112-127), PRISTIF1."""
        k = np.ascontiguousarray(k, dtype=np.float64)
        err = RefError()
        self._check(self.lib.ref_save_stiffness(str(path).encode(), p, n_eq, _ptr(k), element_id, C.byref(err)), err)

    def load_stiffness(self, path, capacity=2 ** 22):
        """The reference's load_stiffness (io.cpp:129-168): (matrix, element_id, p, n_eq)."""
        out = np.zeros(capacity)
        eid, p, n_eq = C.c_int64(), C.c_int(), C.c_int()
        err = RefError()
        self._check(self.lib.ref_load_stiffness(str(path).encode(), _ptr(out), capacity, C.byref(eid), C.byref(p),
                                                C.byref(n_eq), C.byref(err)), err)
        dim = n_eq.value * shape_count(p.value)
        return out[:dim * dim].reshape(dim, dim), eid.value, p.value, n_eq.value

    def integrate_optimized_batch(self, p, geoms, mats, threads=0):
        """integrate_optimized per element, mats [n][2] = (E, nu); element-parallel."""
        geoms = np.ascontiguousarray(geoms, dtype=np.float64).reshape(-1, 18)
        mats = np.ascontiguousarray(mats, dtype=np.float64).reshape(-1, 2)
        dim = 3 * shape_count(p)
        out = np.zeros((len(geoms), dim, dim))
        err = RefError()
        self._check(self.lib.ref_integrate_optimized_batch(p, len(geoms), _ptr(geoms), _ptr(mats), _ptr(out),
                                                           threads, C.byref(err)), err)
        return out


def rel_frobenius(ref: np.ndarray, other: np.ndarray, axis=None) -> np.ndarray:
    """verify.cpp:461-469 / oracles.cpp:163-172: sqrt(sum (a-b)^2 / sum a^2)."""
    ref = np.asarray(ref)
    other = np.asarray(other)
    if axis is None:
        num = np.sum((ref - other) ** 2)
        den = np.sum(ref * ref)
        return np.sqrt(num / den) if den > 0 else np.sqrt(num)
    num = np.sum((ref - other) ** 2, axis=axis)
    den = np.sum(ref * ref, axis=axis)
    return np.where(den > 0, np.sqrt(num / np.where(den > 0, den, 1)), np.sqrt(num))


def sample_indices(n: int, want: int):
    """verify.cpp:50-59: evenly spaced sample."""
    if n == 0:
        return []
    want = min(want, n)
    return [0 if want == 1 else i * (n - 1) // (want - 1) for i in range(want)]


def laplace_tensor():
    c = np.zeros((1, 1, 4, 4))
    for d in range(1, 4):
        c[0, 0, d, d] = 1.0
    return c


def _mix64(z):
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def cdr_coefficients(seed: int, first: int, count: int) -> np.ndarray:
    """numpy restatement of the synthetic per-element CDR tensors of SURVEY.md
    8(d) config 3 (the generator behind pi_generate_cdr_coefficients): element
    g draws 10 counter-based uniforms (splitmix64 of key + 16 g + i), D = R
    diag(lambda) R^T with lambda in U[0.5, 2] and R a uniform rotation (unit
    quaternion), convection b in U[-1, 1]^3 at [0][1..3], reaction r in U[0, 1]
    at [0][0].  AoS [count][16].  Used by bench.py's reference arm so that arm
    never loads the product library; equal to the product's generator to
    rounding (tests/test_host.py)."""
    key = _mix64(np.array([seed ^ 0x43445231], dtype=np.uint64))[0]
    g = np.arange(first, first + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = _mix64(key + g[:, None] * np.uint64(16) + np.arange(10, dtype=np.uint64)[None, :])
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    lam = 0.5 + 1.5 * u[:, 0:3]
    r1, r2 = np.sqrt(1.0 - u[:, 3]), np.sqrt(u[:, 3])
    t1, t2 = 2.0 * np.pi * u[:, 4], 2.0 * np.pi * u[:, 5]
    qx, qy, qz, qw = r1 * np.sin(t1), r1 * np.cos(t1), r2 * np.sin(t2), r2 * np.cos(t2)
    R = np.empty((count, 3, 3))
    R[:, 0, 0] = 1 - 2 * (qy * qy + qz * qz)
    R[:, 0, 1] = 2 * (qx * qy - qz * qw)
    R[:, 0, 2] = 2 * (qx * qz + qy * qw)
    R[:, 1, 0] = 2 * (qx * qy + qz * qw)
    R[:, 1, 1] = 1 - 2 * (qx * qx + qz * qz)
    R[:, 1, 2] = 2 * (qy * qz - qx * qw)
    R[:, 2, 0] = 2 * (qx * qz - qy * qw)
    R[:, 2, 1] = 2 * (qy * qz + qx * qw)
    R[:, 2, 2] = 1 - 2 * (qx * qx + qy * qy)
    c = np.zeros((count, 4, 4))
    c[:, 1:, 1:] = np.einsum("eik,ek,ejk->eij", R, lam, R)
    c[:, 0, 1:] = 2.0 * u[:, 6:9] - 1.0
    c[:, 0, 0] = u[:, 9]
    return c.reshape(count, 16)


def materials(first: int, count: int) -> np.ndarray:
    """Synthetic per-element (young_E, poisson_nu), AoS [count][2]: the same
    pure function of the global id as paper_1310_1191_b200.generate_materials."""
    g = np.arange(first, first + count, dtype=np.uint64)
    u = ((g * np.uint64(2654435761)) % np.uint64(1000003)).astype(np.float64) / 1000003.0
    v = ((g * np.uint64(40503) + np.uint64(17)) % np.uint64(999983)).astype(np.float64) / 999983.0
    return np.ascontiguousarray(np.stack([1.0 + u, 0.2 + 0.15 * v]).T)
