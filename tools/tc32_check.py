"""FP32 tcgen05 path vs the FP64 kernels: per-element relative Frobenius, and timing."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1310_1191_b200 as pb  # noqa: E402

mesh = pb.generate_box_mesh(6, 4, 3, 0.2, seed=5)
n = len(mesh)
geom = torch.from_numpy(np.ascontiguousarray(mesh.reshape(n, 18).T)).cuda()
cdr = torch.from_numpy(np.ascontiguousarray(pb.generate_cdr_coefficients(42, 0, n).T)).cuda()
for p in map(int, (sys.argv[1] if len(sys.argv) > 1 else "3,4,5,6,7").split(",")):
    for mode, c in ((pb.LAPLACE, None), (pb.PER_ELEMENT, cdr)):
        with pb.Integrator(p, variant=pb.VARIANT_TC32) as it:
            d = it.dim
            k64 = torch.empty((n, d, d), dtype=torch.float64, device="cuda")
            k32 = torch.full((n, d, d), float("nan"), dtype=torch.float32, device="cuda")
            it.integrate_device(n, geom, k64, mode, c)
            it.integrate_device(n, geom, k32, mode, c)
            it.check()
            a, b = k64.cpu().numpy(), k32.double().cpu().numpy()
            err = np.sqrt(((a - b) ** 2).sum(axis=(1, 2)) / (a ** 2).sum(axis=(1, 2)))
            nanc = int(np.isnan(b).sum())
            print(f"p={p} mode={mode}: max rel {np.nanmax(err):.3e}  nan={nanc}", flush=True)
    # timing
    E = 2 * 128 * 64 * 16
    g = torch.from_numpy(pb.generate_box_mesh(128, 64, 16, 0.1, 42, soa=True)).cuda()
    with pb.Integrator(p, variant=pb.VARIANT_TC32) as it:
        d = it.dim
        ch = min(E, int(20e9 / 4) // (d * d))
        out = torch.empty(ch * d * d, dtype=torch.float32, device="cuda")
        st = torch.cuda.Stream()
        for rep in range(3):
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(st)
            for lo in range(0, E, ch):
                m = min(ch, E - lo)
                it.integrate_device(m, g.data_ptr() + 8 * lo, out, pb.LAPLACE, geom_ld=E, precision="f32",
                                    stream=st.cuda_stream)
            t1.record(st)
            torch.cuda.synchronize()
        it.check()
        ms = t0.elapsed_time(t1)
        print(f"p={p} FP32 tc: {E / ms * 1e3:.3e} el/s ({ms:.2f} ms for {E}), HBM {E * (d * d * 4 + 144) / ms / 1e6:.0f} GB/s",
              flush=True)
