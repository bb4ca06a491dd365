"""Generates tests/golden/*.npz by running the REFERENCE itself.

Uses oracle/_ref/libprismint_ref.so (the unmodified reference sources under
/root/reference/proj/src compiled by oracle/Makefile).  Re-run with
    make -C oracle && python tests/golden/gen_golden.py
The fixtures pin the oracle restatement (tests/test_oracle.py), the product's
host constants (tests/test_host.py) and, on the GPU, the kernels
(tests/test_gpu_golden.py).
"""
import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import Reference, laplace_tensor  # noqa: E402

DEFAULT_SEED = 0x5072697342657631


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def cdr_tensor(seed):
    """A fixed nonsymmetric CDR tensor (independent of the product's generator)."""
    rng = np.random.default_rng(seed)
    c = np.zeros((4, 4))
    a = rng.uniform(-0.3, 0.3, (3, 3))
    c[1:, 1:] = np.eye(3) + 0.5 * (a + a.T)
    c[0, 1:] = rng.uniform(-1, 1, 3)
    c[0, 0] = rng.uniform(0, 1)
    return c


def main():
    r = Reference()
    out = {}
    # per-p constants (reference_element.cpp:175-286)
    for p in range(1, 8):
        pts, w = r.quadrature(p)
        out[f"quad_points_p{p}"] = pts
        out[f"quad_weights_p{p}"] = w
        tab = r.shape_table(p)
        out[f"shape_sha_p{p}"] = np.array(sha(tab))
        if p <= 3:
            out[f"shape_table_p{p}"] = tab
        else:
            out[f"shape_table_q0_p{p}"] = tab[0]
            out[f"shape_table_qlast_p{p}"] = tab[-1]
    # meshes (geometry.cpp:134-201)
    out["mesh_4_3_2_d02_s5"] = r.box_mesh(4, 3, 2, 0.2, 5)
    out["mesh_2_2_2_d02_s5"] = r.box_mesh(2, 2, 2, 0.2, 5)
    out["mesh_1_1_1_d0_default"] = r.box_mesh(1, 1, 1, 0.0, DEFAULT_SEED)
    out["mesh_sha_16_16_8_d01_s42"] = np.array(sha(r.box_mesh(16, 16, 8, 0.1, 42)))
    # element matrices: the reference's own "right" and "distorted" prisms
    # (test_integrate_ref.cpp:118-119) plus more elements at low p.
    right = out["mesh_1_1_1_d0_default"][0]
    distorted = out["mesh_2_2_2_d02_s5"][9]
    small = out["mesh_4_3_2_d02_s5"]
    cdr = cdr_tensor(1310)
    out["cdr_tensor"] = cdr
    for p in range(1, 8):
        geoms = np.stack([right, distorted] + ([small[i] for i in (0, 7, 23, 40)] if p <= 3 else []))
        out[f"K_laplace_geoms_p{p}"] = geoms
        k, err = r.integrate_batch(p, geoms, laplace_tensor(), threads=0)
        assert err is None
        out[f"K_laplace_p{p}"] = k
        k, err = r.integrate_batch(p, geoms, cdr.reshape(1, 1, 4, 4), threads=0)
        assert err is None
        out[f"K_cdr_p{p}"] = k
    # elasticity through the generic path (n_eq = 3) and integrate_optimized
    for p in (1, 2):
        el = np.zeros((3, 3, 4, 4))
        r.lib.ref_elasticity_tensor(3.0, 0.25, el.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_double)), None)
        out["elasticity_tensor_3_025"] = el
        k, err = r.integrate_batch(p, distorted[None], el, n_eq=3, threads=1)
        assert err is None
        out[f"K_elasticity_generic_p{p}"] = k[0]
        out[f"K_elasticity_optimized_p{p}"] = r.integrate_optimized(p, distorted, 3.0, 0.25)
    np.savez_compressed(HERE / "reference_golden.npz", **out)
    print("wrote", HERE / "reference_golden.npz", sum(v.nbytes for v in out.values()), "bytes raw")


if __name__ == "__main__":
    main()
