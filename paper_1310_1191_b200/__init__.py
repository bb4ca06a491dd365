"""B200-native prismatic element integration (arXiv 1310.1191 hot path).

Python mirror of the reference's integration interface (prismint,
/root/reference/proj), driving the sm_100a kernels through the C ABI in
``include/prism_b200.h`` (library ``libprism_b200.so``, built in-tree).

Reference name            -> here
  prism_quadrature(p)        prism_quadrature(p)            (reference_element.cpp:175)
  tabulate_shapes(p, rule)   tabulate_shapes(p, points)     (reference_element.cpp:272)
  generate_box_mesh(...)     generate_box_mesh(...)         (geometry.cpp:134)
  integrate_generic(...)     Integrator.integrate_device / integrate_host (batched)
  run_batch(...)             run_batch(...)                 (kernels.cpp:485)
  prismint::Error & co.      Error, ConfigError, ... InvertedElementError

There is no CPU fallback: importing works without a GPU (for the host-side
helpers), but every integration call requires the CUDA library and a device
and raises otherwise.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

__all__ = [
    "Error", "ConfigError", "DomainError", "UnsupportedDegreeError", "InvertedElementError",
    "CapacityError", "SharedMemoryError", "ContractViolation", "IoError", "CudaError",
    "LAPLACE", "UNIFORM", "PER_ELEMENT", "ELASTICITY", "ELASTICITY_UNIFORM", "OUT_CANONICAL", "OUT_SOA",
    "VARIANT_AUTO", "VARIANT_DENSE", "VARIANT_SUMFACT", "VARIANT_TC32", "LOAD_AUTO", "LOAD_FUSED", "LOAD_SEPARATE",
    "shape_count", "quadrature_point_count", "prism_quadrature", "tabulate_shapes",
    "generate_box_mesh", "generate_cdr_coefficients", "generate_materials", "laplace_tensor",
    "Integrator", "run_batch", "integrate_host_multi", "measure_fp64_peak", "PRISTIF1", "PRISTIF2", "save_stiffness", "load_stiffness",
    "stiffness_info", "flops_dense_per_element", "bytes_per_element", "library",
]

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libprism_b200.so"

LAPLACE, UNIFORM, PER_ELEMENT = 0, 1, 2
# n_eq = 3 isotropic elasticity from MaterialData (young_E, poisson_nu): per element
# (device SoA [2][ld] / host AoS [n][2]) or one material for all elements (host [2]).
ELASTICITY, ELASTICITY_UNIFORM = 3, 4
OUT_CANONICAL, OUT_SOA = 0, 1
VARIANT_AUTO, VARIANT_DENSE, VARIANT_SUMFACT, VARIANT_TC32 = 0, 1, 2, 3
LOAD_AUTO, LOAD_FUSED, LOAD_SEPARATE = 0, 1, 2


# ---- errors: prismint::errc (errors.hpp:10-19) plus CUDA ----
class Error(RuntimeError):
    code = "unknown"


class ConfigError(Error):
    code = "config"


class DomainError(Error):
    code = "domain"


class UnsupportedDegreeError(Error):
    code = "unsupported_degree"


class InvertedElementError(Error):
    """Carries the global element id, det and reference point (errors.hpp:43-54)."""
    code = "inverted_element"

    def __init__(self, message, element=-1, det=0.0, xi=(0.0, 0.0, 0.0)):
        super().__init__(message)
        self.element = element
        self.det = det
        self.xi = tuple(xi)


class CapacityError(Error):
    code = "capacity"


class SharedMemoryError(Error):
    code = "shared_memory_exhausted"


class ContractViolation(Error):
    code = "contract_violation"


class IoError(Error):
    code = "io"


class CudaError(Error):
    code = "cuda"


_ERRORS = {1: ConfigError, 2: DomainError, 3: UnsupportedDegreeError, 4: InvertedElementError,
           5: CapacityError, 6: SharedMemoryError, 7: ContractViolation, 8: IoError, 9: CudaError}


class _ErrInfo(C.Structure):
    _fields_ = [("element", C.c_int64), ("det", C.c_double), ("xi", C.c_double * 3),
                ("cuda_error", C.c_int), ("message", C.c_char * 256)]


_dp = C.POINTER(C.c_double)
_lib = None


def library():
    """Loads libprism_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = LIB_PATH
    alt = os.environ.get("PRISM_B200_LIB")  # developer A/B builds (make ... LIB=...)
    if alt:
        path = Path(alt) if Path(alt).is_absolute() else LIB_PATH.parent / alt
    if not path.exists():
        raise ImportError(f"{path} not built: run `python __graft_entry__.py` build() or "
                          f"`make -C paper_1310_1191_b200`")
    L = C.CDLL(str(path))
    E = C.POINTER(_ErrInfo)
    vp = C.c_void_p
    L.pi_shape_count.argtypes = [C.c_int]
    L.pi_quadrature_point_count.argtypes = [C.c_int]
    L.pi_prism_quadrature.argtypes = [C.c_int, _dp, _dp, E]
    L.pi_tabulate_shapes.argtypes = [C.c_int, _dp, C.c_int, _dp, E]
    L.pi_generate_box_mesh.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int64,
                                       C.c_int64, C.c_int, C.c_int64, C.c_int, _dp, E]
    L.pi_generate_cdr_coefficients.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int, C.c_int64, _dp, E]
    L.pi_context_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp,
                                    C.POINTER(vp), E]
    L.pi_context_destroy.argtypes = [vp]
    L.pi_context_set_variant.argtypes = [vp, C.c_int, E]
    L.pi_context_set_load_fusion.argtypes = [vp, C.c_int, E]
    L.pi_context_variant.argtypes = [vp, C.c_int]
    L.pi_context_stream.argtypes = [vp]
    L.pi_context_stream.restype = vp
    L.pi_integrate.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int64, C.c_int, vp, C.c_int64, vp, C.c_int,
                               C.c_int64, vp, E]
    L.pi_integrate_f32.argtypes = L.pi_integrate.argtypes
    L.pi_integrate_load.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int64, C.c_int, vp, C.c_int64, vp, C.c_int,
                                    C.c_int64, vp, C.c_double, vp, vp, E]
    L.pi_integrate_host_multi.argtypes = [C.POINTER(vp), C.c_int, C.c_int64, C.c_int64, vp, C.c_int, vp, vp,
                                          C.c_int64, E]
    L.pi_load_vectors.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int64, vp, C.c_double, vp, vp, E]
    L.pi_check.argtypes = [vp, E]
    L.pi_integrate_host.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int, vp, vp, C.c_int64, E]
    L.pi_integrate_host_load.argtypes = [vp, C.c_int64, C.c_int64, vp, C.c_int, vp, vp, C.c_double, vp, vp,
                                         C.c_int64, E]
    L.pi_flops_dense_per_element.argtypes = [C.c_int, C.c_int, C.c_int]
    L.pi_flops_dense_per_element.restype = C.c_double
    L.pi_flops_executed_per_element.argtypes = [vp, C.c_int]
    L.pi_flops_executed_per_element.restype = C.c_double
    L.pi_bytes_per_element.argtypes = [C.c_int, C.c_int, C.c_int]
    L.pi_bytes_per_element.restype = C.c_double
    L.pi_measure_fp64_peak.argtypes = [C.c_int, _dp, _dp]
    L.pi_save_stiffness.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, vp, E]
    L.pi_stiffness_info.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int64), C.POINTER(C.c_int64), E]
    L.pi_load_stiffness.argtypes = [C.c_char_p, vp, C.c_int64, E]
    L.pi_status_name.restype = C.c_char_p
    L.pi_version.restype = C.c_char_p
    _lib = L
    return L


def _raise(status, err: _ErrInfo):
    if status == 0:
        return
    cls = _ERRORS.get(status, Error)
    msg = err.message.decode(errors="replace")
    if cls is InvertedElementError:
        raise InvertedElementError(msg, err.element, err.det, tuple(err.xi))
    raise cls(msg)


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _addr(x):
    """Raw address of a numpy array or torch tensor (device or host)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags.c_contiguous
        return x.ctypes.data
    return x.data_ptr()


# ---- per-p constants ----
def shape_count(p: int) -> int:
    n = library().pi_shape_count(p)
    if n < 0:
        raise DomainError(f"approximation order p={p} outside supported range [1, 7]")
    return n


def quadrature_point_count(p: int) -> int:
    n = library().pi_quadrature_point_count(p)
    if n < 0:
        raise DomainError(f"approximation order p={p} outside supported range [1, 7]")
    return n


def prism_quadrature(p: int):
    """(points [n_q][3], weights [n_q]) -- reference_element.cpp:175-193."""
    nq = quadrature_point_count(p)
    pts = np.zeros((nq, 3))
    w = np.zeros(nq)
    err = _ErrInfo()
    _raise(library().pi_prism_quadrature(p, _ptr(pts), _ptr(w), C.byref(err)), err)
    return pts, w


def tabulate_shapes(p: int, points=None):
    """[n_q][4][n_shape] -- reference_element.cpp:272-286."""
    if points is None:
        points, _ = prism_quadrature(p)
    points = np.ascontiguousarray(points, dtype=np.float64)
    out = np.zeros((len(points), 4, shape_count(p)))
    err = _ErrInfo()
    _raise(library().pi_tabulate_shapes(p, _ptr(points), len(points), _ptr(out), C.byref(err)), err)
    return out


def generate_box_mesh(nx, ny, nz, distortion, seed=0x5072697342657631, first=0, count=None, soa=False,
                      ld=None, validate=False, out=None):
    """Seeded box mesh (geometry.cpp:134-201).  AoS [count][6][3] or SoA [18][ld]."""
    total = 2 * nx * ny * nz
    count = total - first if count is None else count
    if soa:
        ld = count if ld is None else ld
        out = np.zeros((18, ld)) if out is None else out
    else:
        out = np.zeros((count, 6, 3)) if out is None else out
    err = _ErrInfo()
    _raise(library().pi_generate_box_mesh(nx, ny, nz, distortion, seed, first, count, int(soa), ld or 0,
                                          int(validate), _ptr(out), C.byref(err)), err)
    return out


def generate_cdr_coefficients(seed, first, count, soa=False, ld=None):
    """Seeded convection-diffusion-reaction tensors, AoS [count][16] or SoA [16][ld]."""
    if soa:
        ld = count if ld is None else ld
        out = np.zeros((16, ld))
    else:
        out = np.zeros((count, 16))
    err = _ErrInfo()
    _raise(library().pi_generate_cdr_coefficients(seed, first, count, int(soa), ld or 0, _ptr(out),
                                                  C.byref(err)), err)
    return out


def generate_materials(first, count, soa=False):
    """Synthetic per-element isotropic materials (young_E, poisson_nu), a pure
    function of the global element id (any sub-range reproduces the full run):
    E in [1, 2), nu in [0.2, 0.35).  AoS [count][2] or SoA [2][count]."""
    g = np.arange(first, first + count, dtype=np.uint64)
    u = ((g * np.uint64(2654435761)) % np.uint64(1000003)).astype(np.float64) / 1000003.0
    v = ((g * np.uint64(40503) + np.uint64(17)) % np.uint64(999983)).astype(np.float64) / 999983.0
    m = np.stack([1.0 + u, 0.2 + 0.15 * v])
    return np.ascontiguousarray(m) if soa else np.ascontiguousarray(m.T)


def laplace_tensor():
    c = np.zeros((1, 1, 4, 4))
    for d in range(1, 4):
        c[0, 0, d, d] = 1.0
    return c


def flops_dense_per_element(p, coeff_mode=LAPLACE, n_eq=1):
    return library().pi_flops_dense_per_element(p, n_eq, coeff_mode)


def bytes_per_element(p, coeff_mode=LAPLACE, n_eq=1):
    return library().pi_bytes_per_element(p, n_eq, coeff_mode)


PRISTIF1, PRISTIF2 = 1, 2


def save_stiffness(path, k, p, n_eq=1, element_id_base=0, fmt=PRISTIF2):
    """Stiffness container.  PRISTIF2: FP64 batch [count][dim][dim];
    PRISTIF1: the reference's single-element f32 container (io.cpp:112-127)."""
    k = np.ascontiguousarray(k, dtype=np.float64)
    dim = n_eq * shape_count(p)
    count = k.size // (dim * dim)
    if count * dim * dim != k.size:
        raise ContractViolation(f"matrix size {k.size} is not a multiple of dim^2 = {dim * dim}")
    err = _ErrInfo()
    _raise(library().pi_save_stiffness(str(path).encode(), fmt, p, n_eq, count, element_id_base, _addr(k),
                                       C.byref(err)), err)


def stiffness_info(path):
    fmt, p, n_eq = C.c_int(), C.c_int(), C.c_int()
    count, base = C.c_int64(), C.c_int64()
    err = _ErrInfo()
    _raise(library().pi_stiffness_info(str(path).encode(), C.byref(fmt), C.byref(p), C.byref(n_eq), C.byref(count),
                                       C.byref(base), C.byref(err)), err)
    return {"format": fmt.value, "p": p.value, "n_eq": n_eq.value, "count": count.value,
            "element_id_base": base.value}


def load_stiffness(path):
    """(matrices [count][dim][dim] float64, info dict) -- io.cpp:129-168 for PRISTIF1."""
    info = stiffness_info(path)
    dim = info["n_eq"] * shape_count(info["p"])
    out = np.empty((info["count"], dim, dim))
    err = _ErrInfo()
    _raise(library().pi_load_stiffness(str(path).encode(), _addr(out), out.size, C.byref(err)), err)
    return out, info


def measure_fp64_peak(device=0):
    """(DMMA TFLOP/s, DFMA TFLOP/s) measured on the device."""
    a = C.c_double()
    b = C.c_double()
    if library().pi_measure_fp64_peak(device, C.byref(a), C.byref(b)) != 0:
        raise CudaError("FP64 peak probe failed")
    return a.value, b.value


class Integrator:
    """One context: device + p (+ the rule / shape table, the reference's own if given)."""

    def __init__(self, p, device=0, n_eq=1, points=None, weights=None, shape_table=None, variant=VARIANT_AUTO):
        L = library()
        self.p = p
        self.device = device
        self.n_eq = n_eq
        self.n_shape = shape_count(p)
        self.n_q = quadrature_point_count(p)
        self.dim = n_eq * self.n_shape
        self._keep = []
        args = [None, None, None]
        n_q, n_shape = self.n_q, self.n_shape
        if points is not None:
            arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (points, weights, shape_table)]
            self._keep = arrs
            args = [_ptr(a) for a in arrs]
            n_q, n_shape = len(arrs[0]), arrs[2].shape[-1]
            if arrs[2].size != n_q * 4 * n_shape or arrs[1].size != n_q:
                raise ContractViolation("rule / shape table sizes are inconsistent")
        h = C.c_void_p()
        err = _ErrInfo()
        _raise(L.pi_context_create(device, p, n_eq, n_q, n_shape, *args, C.byref(h), C.byref(err)), err)
        self._h = h
        if variant != VARIANT_AUTO:
            self.set_variant(variant)

    def close(self):
        if getattr(self, "_h", None):
            library().pi_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_variant(self, variant):
        err = _ErrInfo()
        _raise(library().pi_context_set_variant(self._h, variant, C.byref(err)), err)

    def set_load_fusion(self, mode):
        """LOAD_AUTO / LOAD_FUSED / LOAD_SEPARATE: strategy of integrate_device(load_out=...)."""
        err = _ErrInfo()
        _raise(library().pi_context_set_load_fusion(self._h, mode, C.byref(err)), err)

    def variant(self, coeff_mode=LAPLACE):
        return library().pi_context_variant(self._h, coeff_mode)

    @property
    def stream(self):
        return library().pi_context_stream(self._h)

    def flops_executed_per_element(self, coeff_mode=LAPLACE):
        return library().pi_flops_executed_per_element(self._h, coeff_mode)

    def _check_tensor(self, name, t, min_numel, dtypes=("torch.float64",), rows=None, min_cols=None):
        """Contract checks for a torch tensor handed to the C ABI (kernels.cpp:423-462
        style ContractViolation); raw integer addresses are the caller's responsibility."""
        if t is None or isinstance(t, int) or not hasattr(t, "is_cuda"):
            return
        if str(t.dtype) not in dtypes:
            raise ContractViolation(f"{name}: dtype {t.dtype}, expected {' or '.join(dtypes)}")
        if not t.is_cuda or (t.device.index is not None and t.device.index != self.device):
            raise ContractViolation(f"{name}: must live on cuda:{self.device} (got {t.device})")
        if not t.is_contiguous():
            raise ContractViolation(f"{name}: must be contiguous (a SoA [rows][ld] buffer)")
        if t.numel() < min_numel:
            raise ContractViolation(f"{name}: {t.numel()} entries, needs at least {min_numel}")
        if rows is not None and t.dim() == 2 and t.shape[0] != rows:
            raise ContractViolation(f"{name}: {t.shape[0]} rows, the weak form needs {rows}")
        if min_cols is not None and t.dim() == 2 and t.shape[1] < min_cols:
            raise ContractViolation(f"{name}: leading dimension {t.shape[1]} < n_elem {min_cols}")

    def _coeff_width(self, coeff_mode):
        return {PER_ELEMENT: 16 * self.n_eq * self.n_eq, ELASTICITY: 2}.get(coeff_mode)

    # -- device buffers (torch tensors or raw addresses); asynchronous --
    def integrate_device(self, n_elem, geom, out, coeff_mode=LAPLACE, coeff=None, element_id_base=0,
                         geom_ld=None, coeff_ld=None, out_layout=OUT_CANONICAL, ld_out=0, stream=None,
                         precision=None, load_out=None, f=None, f_const=1.0):
        """pi_integrate on device memory.  geom: SoA [18][geom_ld]; out: device buffer
        (float64; float32 selects the FP32 output variant, or precision="f32" for raw addresses).
        load_out (device [n_elem][n_shape] float64): also the load vectors in the same pass
        (pi_integrate_load; f: device [n_elem] per-element values, else f_const)."""
        err = _ErrInfo()
        cbuf = None
        if coeff_mode in (UNIFORM, ELASTICITY_UNIFORM):
            cbuf = np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1)
            caddr = cbuf.ctypes.data
        else:
            caddr = _addr(coeff) if coeff_mode in (PER_ELEMENT, ELASTICITY) else None
        if geom_ld is None:
            geom_ld = geom.shape[1] if hasattr(geom, "shape") else n_elem
        if coeff_ld is None and coeff_mode in (PER_ELEMENT, ELASTICITY):
            coeff_ld = coeff.shape[1] if hasattr(coeff, "shape") else n_elem
        # float32 output buffer -> the FP32 output variant (pi_integrate_f32)
        f32 = precision == "f32" or (precision is None and str(getattr(out, "dtype", "")) in ("torch.float32", "float32"))
        if n_elem > 0:
            self._check_tensor("geometry", geom, 18 * geom_ld, rows=18 if getattr(geom, "dim", lambda: 0)() == 2 else None,
                               min_cols=n_elem)
            kk = self.dim * self.dim
            need = n_elem * kk if out_layout == OUT_CANONICAL else kk * max(ld_out, n_elem)
            self._check_tensor("out", out, need, dtypes=("torch.float32",) if f32 else ("torch.float64",))
            if coeff_mode in (PER_ELEMENT, ELASTICITY):
                self._check_tensor("coefficients", coeff, self._coeff_width(coeff_mode) * (coeff_ld or n_elem),
                                   rows=self._coeff_width(coeff_mode), min_cols=n_elem)
        if load_out is not None:
            if f32:
                raise ContractViolation("fused load vectors need an FP64 stiffness output")
            if n_elem > 0:
                self._check_tensor("load_out", load_out, n_elem * self.n_shape)
                self._check_tensor("f", f, n_elem)
            st = library().pi_integrate_load(self._h, n_elem, element_id_base, _addr(geom), geom_ld, coeff_mode,
                                             caddr, coeff_ld or 0, _addr(out), out_layout, ld_out, _addr(f),
                                             float(f_const), _addr(load_out), stream, C.byref(err))
            _raise(st, err)
            return
        fn = library().pi_integrate_f32 if f32 else library().pi_integrate
        st = fn(self._h, n_elem, element_id_base, _addr(geom), geom_ld, coeff_mode, caddr, coeff_ld or 0,
                _addr(out), out_layout, ld_out, stream, C.byref(err))
        _raise(st, err)

    def load_vectors_device(self, n_elem, geom, out, f=None, f_const=1.0, element_id_base=0, geom_ld=None,
                            stream=None):
        err = _ErrInfo()
        if geom_ld is None:
            geom_ld = geom.shape[1] if hasattr(geom, "shape") else n_elem
        st = library().pi_load_vectors(self._h, n_elem, element_id_base, _addr(geom), geom_ld, _addr(f),
                                       float(f_const), _addr(out), stream, C.byref(err))
        _raise(st, err)

    def check(self):
        """Synchronises and raises InvertedElementError / CudaError (pi_check)."""
        err = _ErrInfo()
        _raise(library().pi_check(self._h, C.byref(err)), err)

    # -- host buffers: the run_batch-style drop-in --
    def integrate_host_load(self, geoms, coeff_mode=LAPLACE, coeff=None, f=None, f_const=1.0, element_id_base=0,
                            chunk_elems=0):
        """pi_integrate_host_load: host [n][6][3] in, (K [n][dim][dim], F [n][n_shape]) out."""
        geoms = np.ascontiguousarray(geoms, dtype=np.float64).reshape(-1, 18)
        n = len(geoms)
        out = np.empty((n, self.dim, self.dim))
        load = np.empty((n, self.n_shape))
        cbuf = _host_coeff(self, coeff_mode, coeff, n)
        fbuf = None if f is None else np.ascontiguousarray(f, dtype=np.float64).reshape(n)
        err = _ErrInfo()
        st = library().pi_integrate_host_load(self._h, n, element_id_base, _addr(geoms), coeff_mode, _addr(cbuf),
                                              _addr(fbuf), float(f_const), _addr(out), _addr(load), chunk_elems,
                                              C.byref(err))
        _raise(st, err)
        return out, load

    def integrate_host(self, geoms, coeff_mode=LAPLACE, coeff=None, element_id_base=0, out=None, chunk_elems=0):
        """geoms: host [n][6][3]; returns host [n][dim][dim] (canonical)."""
        geoms = np.ascontiguousarray(geoms, dtype=np.float64).reshape(-1, 18)
        n = len(geoms)
        if out is None:
            out = np.empty((n, self.dim, self.dim))
        elif out.size < n * self.dim * self.dim or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise ContractViolation(f"out: needs a C-contiguous float64 [{n}][{self.dim}][{self.dim}] buffer")
        cbuf = None
        if coeff_mode in (UNIFORM, ELASTICITY_UNIFORM):
            cbuf = np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1)
            want = 16 * self.n_eq * self.n_eq if coeff_mode == UNIFORM else 2
            if cbuf.size != want:
                raise ContractViolation(f"uniform coefficients: {cbuf.size} values, needs {want}")
        elif coeff_mode in (PER_ELEMENT, ELASTICITY):
            cbuf = np.ascontiguousarray(coeff, dtype=np.float64).reshape(n, -1)
            if cbuf.shape[1] != self._coeff_width(coeff_mode):
                raise ContractViolation(f"per-element coefficients: width {cbuf.shape[1]}, the weak form needs "
                                        f"{self._coeff_width(coeff_mode)}")
        err = _ErrInfo()
        st = library().pi_integrate_host(self._h, n, element_id_base, _addr(geoms), coeff_mode, _addr(cbuf),
                                         _addr(out), chunk_elems, C.byref(err))
        _raise(st, err)
        return out


def _host_coeff(it, coeff_mode, coeff, n):
    if coeff_mode in (UNIFORM, ELASTICITY_UNIFORM):
        return np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1)
    if coeff_mode in (PER_ELEMENT, ELASTICITY):
        return np.ascontiguousarray(coeff, dtype=np.float64).reshape(n, -1)
    return None


def integrate_host_multi(integrators, geoms, coeff_mode=LAPLACE, coeff=None, element_id_base=0, out=None,
                         chunk_elems=0):
    """pi_integrate_host_multi: contiguous element ranges over several contexts
    (one per GPU), one host thread each; bitwise equal to a single context."""
    its = list(integrators)
    geoms = np.ascontiguousarray(geoms, dtype=np.float64).reshape(-1, 18)
    n = len(geoms)
    dim = its[0].dim
    if out is None:
        out = np.empty((n, dim, dim))
    cbuf = None
    if coeff_mode in (UNIFORM, ELASTICITY_UNIFORM):
        cbuf = np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1)
    elif coeff_mode in (PER_ELEMENT, ELASTICITY):
        cbuf = np.ascontiguousarray(coeff, dtype=np.float64).reshape(n, -1)
    handles = (C.c_void_p * len(its))(*[it._h.value for it in its])
    err = _ErrInfo()
    st = library().pi_integrate_host_multi(handles, len(its), n, element_id_base, _addr(geoms), coeff_mode,
                                           _addr(cbuf), _addr(out), chunk_elems, C.byref(err))
    _raise(st, err)
    return out


def run_batch(p, mesh, coeff_mode=LAPLACE, coeff=None, device=0, **kw):
    """run_batch (kernels.cpp:485-514) semantics: matrices in mesh order."""
    if len(mesh) == 0:
        raise ConfigError("run_batch: empty mesh")
    with Integrator(p, device=device, **kw) as it:
        return it.integrate_host(mesh, coeff_mode, coeff)
