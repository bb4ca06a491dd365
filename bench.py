#!/usr/bin/env python
"""Benchmark: element stiffness integration for prisms (arXiv 1310.1191) on B200.

Metric (BASELINE.json): elements integrated per second per degree p, plus the
fraction of the FP64 / HBM roofline.  Workload (BASELINE.json configs[1]):
Laplace weak form, p = 2, 3, 4, 1,048,576 synthetic prisms per GPU
(generate_box_mesh(128, 64, 64*N, 0.1, 42), rank r owns the contiguous range
[r*E, (r+1)*E) -- weak scaling, no collective on the data path).

One step = one pass of the hot path over the rank's elements at every p in
--p (three launches of the sm_100a kernels, outputs device-resident).
value = elements processed by all ranks in the timed steps / max-over-ranks
device time.  e2e = the same step through the host-buffer C-ABI call
(pi_integrate_host): pinned host geometry in, pinned host K out, all copies
inside the timed region.

  python bench.py [--gpus N --steps K --warmup W --p 2,3,4 --coeff laplace|cdr]
  python bench.py --impl reference ...   # the reference CPU integrate_generic
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "elements integrated/sec per degree p (1 and 8 B200) and % of FP64/HBM roofline"
NX, NY, NZ_PER_RANK, DISTORTION, SEED = 128, 64, 64, 0.1, 42
COEFF_SEED = 42


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", default="2,3,4")
    ap.add_argument("--coeff", default="laplace", choices=["laplace", "cdr", "elasticity"],
                    help="weak form: Laplace, per-element CDR tensors, or n_eq=3 elasticity with per-element (E, nu)")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="K output precision (f32: the FP32 output variant, SURVEY 8f row f3)")
    ap.add_argument("--out-gb", type=float, default=120.0,
                    help="device output budget; larger steps stream through a ring of chunks")
    ap.add_argument("--nz", type=int, default=NZ_PER_RANK, help="mesh layers per rank (64 -> 1M elements)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=18.0, help="CPU baseline budget")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------- CPU legs
def cpu_reference_rates(ps, coeff_kind, budget_s, mesh_aos, coeffs_aos):
    """Reference integrate_generic (oracle/_ref, all host threads) el/s per p on a
    bounded sample of the same mesh -- integrate_optimized, the reference's
    fastest FP64 path, for elasticity.  Returns (rates, sample description, cores, kind)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REF_SO, Oracle, Reference, laplace_tensor  # test infrastructure (checker)

    cores = os.cpu_count() or 1
    kind = "reference" if REF_SO.exists() else "port"
    rates, samples = {}, {}
    per_p = budget_s / max(1, len(ps))
    for p in ps:
        n = 16
        while True:
            g = mesh_aos[:n]
            c = laplace_tensor() if coeff_kind == "laplace" else (coeffs_aos[:n] if coeffs_aos is not None else None)
            t0 = time.perf_counter()
            if coeff_kind == "elasticity":
                if kind == "reference":
                    Reference().integrate_optimized_batch(p, g, coeffs_aos[:n], threads=cores)
                else:
                    o = Oracle()
                    o.integrate_batch(p, g, np.stack([o.elasticity_tensor(*m) for m in coeffs_aos[:n]]), n_eq=3)
            elif kind == "reference":
                _, err = Reference().integrate_batch(p, g, c, threads=cores)
                assert err is None
            else:
                Oracle().integrate_batch(p, g, c)
            dt = time.perf_counter() - t0
            if dt >= per_p * 0.25 or n >= len(mesh_aos):
                break
            n = min(len(mesh_aos), int(n * max(2.0, per_p * 0.3 / max(dt, 1e-4))))
        rates[p] = n / dt
        samples[p] = n
    desc = ", ".join(f"p={p}: first {samples[p]} elements" for p in ps)
    return rates, desc, cores if kind == "reference" else 1, kind


def step_rate(rates, ps):
    """Elements/s of one step (E elements at every p) from per-p rates."""
    return len(ps) / sum(1.0 / rates[p] for p in ps)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
                power.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax), "power_w_max": max(power),
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------ reference arm
def run_reference_arm(args, ps, ws, rank):
    if rank != 0:
        return 0
    import paper_1310_1191_b200 as pb  # host-side mesh generator only (no GPU use)

    E = 2 * NX * NY * args.nz
    n_probe = min(E, 200_000)
    mesh = pb.generate_box_mesh(NX, NY, args.nz * ws, DISTORTION, SEED, first=0, count=n_probe)
    coeffs = (pb.generate_cdr_coefficients(COEFF_SEED, 0, n_probe) if args.coeff == "cdr"
              else pb.generate_materials(0, n_probe) if args.coeff == "elasticity" else None)
    budget = 6.0  # seconds of CPU work per step
    rates, desc, cores, kind = cpu_reference_rates(ps, args.coeff, budget, mesh, coeffs)
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import Reference, laplace_tensor

    ref = Reference()
    n_p = {p: min(len(mesh), max(1, int(rates[p] * budget / len(ps)))) for p in ps}

    def one_step(acc):
        for p in ps:
            c = laplace_tensor() if args.coeff == "laplace" else coeffs[: n_p[p]]
            t0 = time.perf_counter()
            if args.coeff == "elasticity":
                ref.integrate_optimized_batch(p, mesh[: n_p[p]], c, threads=cores)
            else:
                _, err = ref.integrate_batch(p, mesh[: n_p[p]], c, threads=cores)
                assert err is None
            acc[p] += time.perf_counter() - t0

    scratch = {p: 0.0 for p in ps}
    for _ in range(args.warmup):
        one_step(scratch)
    tsum = {p: 0.0 for p in ps}
    for _ in range(args.steps):
        one_step(tsum)
    # Per-element cost depends only on p: the bounded sample's
    # rate is the rate of the full E-element step.
    per_p_rate = {p: n_p[p] * args.steps / tsum[p] for p in ps}
    value = step_rate(per_p_rate, ps)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * len(ps) * E / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generate_box_mesh 128x64x64, distortion 0.1, seed 42)",
        "config": {"workload": f"{args.coeff} p={','.join(map(str, ps))}, {E} prisms per GPU",
                   "elements_per_gpu": E, "p": ps, "coeff": args.coeff},
        "per_p": {str(p): {"elements_per_s": per_p_rate[p], "sample_elements": n_p[p]} for p in ps},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": kind,
                         "sample": f"per step, p-wise first elements: {n_p}"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    ps = [int(x) for x in args.p.split(",")]
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, ps, ws, rank)

    import torch
    import paper_1310_1191_b200 as pb

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    E = 2 * NX * NY * args.nz
    first = rank * E
    n_eq = 3 if args.coeff == "elasticity" else 1
    mode = {"laplace": pb.LAPLACE, "cdr": pb.PER_ELEMENT, "elasticity": pb.ELASTICITY}[args.coeff]
    # Synthetic inputs for this rank's contiguous range (host-generated, not timed).
    geom_host = pb.generate_box_mesh(NX, NY, args.nz * ws, DISTORTION, SEED, first=first, count=E, soa=True)
    geom = torch.from_numpy(geom_host).to(dev)
    coeff = None
    coeff_host = None
    if mode == pb.PER_ELEMENT:
        coeff_host = pb.generate_cdr_coefficients(COEFF_SEED, first, E, soa=True)
    elif mode == pb.ELASTICITY:
        coeff_host = pb.generate_materials(first, E, soa=True)
    if coeff_host is not None:
        coeff = torch.from_numpy(coeff_host).to(dev)
    dim = {p: n_eq * pb.shape_count(p) for p in ps}
    kk = {p: dim[p] ** 2 for p in ps}
    # Output: device resident.  A step whose matrices exceed --out-gb streams
    # through one reused chunk buffer (the ring of SURVEY 8d: K is produced
    # and left in HBM chunk by chunk; every element is still integrated).
    esz = 4 if args.precision == "f32" else 8
    budget = int(args.out_gb * 1e9 / esz)
    chunk = {p: min(E, max(1, budget // kk[p])) for p in ps}
    out = torch.empty(max(chunk[p] * kk[p] for p in ps), dtype=torch.float32 if esz == 4 else torch.float64,
                      device=dev)
    ctxs = {p: pb.Integrator(p, device=local, n_eq=n_eq) for p in ps}
    # A dedicated stream: a NULL handle would mean "the context's own stream"
    # in the C ABI, so torch's legacy default stream (handle 0) is never used.
    stream = torch.cuda.Stream(dev)
    sptr = stream.cuda_stream
    g0 = geom.data_ptr()
    c0 = coeff.data_ptr() if coeff is not None else None

    def launch(p, lo, n):
        ctxs[p].integrate_device(n, g0 + 8 * lo, out.data_ptr(), mode, None if c0 is None else c0 + 8 * lo,
                                 element_id_base=first + lo, geom_ld=E, coeff_ld=E, stream=sptr,
                                 precision=args.precision)

    def step(events=None):
        for p in ps:
            if events is not None:
                events[p][0].record(stream)
            for lo in range(0, E, chunk[p]):
                launch(p, lo, min(chunk[p], E - lo))
            if events is not None:
                events[p][1].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    for p in ps:
        ctxs[p].check()
    torch.cuda.synchronize(dev)

    ev = [{p: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for p in ps}
          for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            step(ev[k])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    for p in ps:
        ctxs[p].check()
    elapsed_ms = t_start.elapsed_time(t_end)
    per_p_ms = {p: float(np.mean([ev[k][p][0].elapsed_time(ev[k][p][1]) for k in range(args.steps)])) for p in ps}
    if dist:
        t = torch.tensor([elapsed_ms] + [per_p_ms[p] for p in ps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t[0])
        per_p_ms = {p: float(t[1 + i]) for i, p in enumerate(ps)}
    clk = clocks.summary()
    ms_per_step = elapsed_ms / args.steps
    value = ws * E * len(ps) / (ms_per_step * 1e-3)
    launches = sum((E + chunk[p] - 1) // chunk[p] for p in ps)

    # -------- parity spot check of the timed outputs (not timed) --------
    parity = None
    if rank == 0:
        sys.path.insert(0, str(ROOT / "tests"))
        from oracle_lib import REF_SO, Oracle, Reference, laplace_tensor, rel_frobenius

        worst = 0.0
        n_checked = 0
        for p in ps:
            lo = (E - 1) - ((E - 1) % chunk[p])  # the last chunk is the one left in the buffer
            idx = sorted({lo, lo + (E - lo) // 2, E - 1})
            launch(p, lo, E - lo)
            torch.cuda.synchronize(dev)
            got = np.stack([out[(i - lo) * kk[p]:(i - lo + 1) * kk[p]].double().cpu().numpy().reshape(dim[p], dim[p])
                            for i in idx])
            mesh_aos = geom_host[:, idx].T.reshape(len(idx), 6, 3)
            if mode == pb.ELASTICITY:
                mats = coeff_host[:, idx].T
                if REF_SO.exists():
                    ref = Reference().integrate_optimized_batch(p, mesh_aos, mats)
                else:
                    o = Oracle()
                    ref = o.integrate_batch(p, mesh_aos, np.stack([o.elasticity_tensor(*m) for m in mats]), n_eq=3)
            else:
                c = laplace_tensor() if mode == pb.LAPLACE else coeff_host[:, idx].T.copy()
                if REF_SO.exists():
                    ref, err = Reference().integrate_batch(p, mesh_aos, c, threads=0)
                else:
                    ref = Oracle().integrate_batch(p, mesh_aos, c)
            worst = max(worst, float(rel_frobenius(ref, got, axis=(1, 2)).max()))
            n_checked += len(idx)
        parity = {"max_rel_frobenius": worst, "tolerance": 1e-12 if esz == 8 else 5e-5, "elements_checked": n_checked,
                  "checker": ("reference integrate_optimized" if mode == pb.ELASTICITY else
                              "reference integrate_generic") + " (oracle/_ref)" if REF_SO.exists() else "oracle port"}

    # -------- roofline (dominant kernel = largest share of the step) --------
    dmma_tf, dfma_tf = pb.measure_fp64_peak(local)
    peaks = json.load(open(ROOT / "MEASURED_PEAKS.json")) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    per_p = {}
    for p in ps:
        t = per_p_ms[p] * 1e-3
        f_dense = pb.flops_dense_per_element(p, mode, n_eq)
        f_exec = ctxs[p].flops_executed_per_element(mode)
        byts = pb.bytes_per_element(p, mode, n_eq) - (8 - esz) * kk[p]
        bound_s = max(f_dense * E / (dmma_tf * 1e12), byts * E / (hbm_peak * 1e9))
        per_p[str(p)] = {
            "elements_per_s": E / t, "ms": per_p_ms[p], "launches": (E + chunk[p] - 1) // chunk[p],
            "dense_flop_alg_per_element": f_dense, "executed_flop_per_element": f_exec,
            "bytes_per_element": byts,
            "dense_tflops": f_dense * E / t / 1e12, "executed_tflops": f_exec * E / t / 1e12,
            "hbm_gbs": byts * E / t / 1e9,
            "roofline_bound_elements_per_s": E / bound_s,
            "frac_of_dense_roofline": bound_s / t,
            "frac_executed_fp64": f_exec * E / t / 1e12 / dmma_tf,
            "frac_hbm": byts * E / t / 1e9 / hbm_peak,
        }
    dom = max(ps, key=lambda p: per_p_ms[p])
    d = per_p[str(dom)]
    # DRAM bytes per launch of the dominant kernel: per-element bytes from the
    # committed ncu capture (profiles/traffic.json, dram__bytes_read+write)
    # scaled to this launch's element count.
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            per_el = json.load(open(tf)).get(f"p{dom}_{args.coeff}")
            traffic = per_el * chunk[dom] if per_el is not None else None
        except Exception:
            traffic = None
    kname = ("p1_thread_kernel" if dom == 1 else "p2_lane_kernel") if (dom <= 2 and n_eq == 1) else \
        f"sumfact_kernel<{dom}, n_eq={n_eq}> (FP64 DMMA)"
    roofline = {
        "bound": "tensor" if not (dom <= 2 and n_eq == 1) else "fp64", "kernel": kname,
        "achieved": d["dense_tflops"], "peak": dmma_tf, "unit": "TFLOP/s", "frac": d["dense_tflops"] / dmma_tf,
        "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram read+write, profiles/traffic.json)",
        "algorithmic_bytes": d["bytes_per_element"] * chunk[dom],
        "achieved_note": "SURVEY 8(d) dense FLOP_alg per element x elements / kernel time; the kernels "
                         "execute fewer FLOPs (sum factorisation, structural zeros, symmetry), so frac can exceed 1",
        "executed_tflops": d["executed_tflops"], "executed_frac": d["executed_tflops"] / dmma_tf,
        "hbm_gbs": d["hbm_gbs"], "hbm_peak_gbs": hbm_peak, "hbm_frac": d["hbm_gbs"] / hbm_peak,
        "peak_source": f"FP64 DMMA m8n8k4 peak measured in-run (DFMA {dfma_tf:.1f} TF/s); "
                       f"HBM from MEASURED_PEAKS.json" + ("" if peaks else " (absent: B200_PROFILING fallback)"),
    }

    # -------- end to end through the host-buffer C-ABI call --------
    e2e = None
    if not args.no_e2e and esz == 8:
        geom_aos = torch.from_numpy(np.ascontiguousarray(geom_host.T)).pin_memory()
        coeff_aos = torch.from_numpy(np.ascontiguousarray(coeff_host.T)).pin_memory() if coeff_host is not None else None
        # pinned host output: <= 16 GB per rank (8 ranks on one box must not pin
        # hundreds of GB); every element's K still crosses PCIe into it
        host_n = {p: min(E, max(1, int(16e9 / 8) // kk[p])) for p in ps}
        host_out = torch.empty(max(host_n[p] * kk[p] for p in ps), dtype=torch.float64).pin_memory()
        ga = geom_aos.numpy()
        ca = coeff_aos.numpy() if coeff_aos is not None else None

        def e2e_step():
            for p in ps:
                it = ctxs[p]
                for lo in range(0, E, host_n[p]):
                    n = min(host_n[p], E - lo)
                    o = host_out[: n * kk[p]].numpy().reshape(n, dim[p], dim[p])
                    it.integrate_host(ga[lo:lo + n], mode, None if ca is None else ca[lo:lo + n],
                                      element_id_base=first + lo, out=o)

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t[0])
        cw = 0 if coeff_host is None else coeff_host.shape[0]
        h2d = E * 18 * 8 * len(ps) + E * cw * 8 * len(ps)
        d2h = sum(E * kk[p] * 8 for p in ps)
        e2e = {"value": ws * E * len(ps) * args.steps / dt, "unit": "elements/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "pi_integrate_host (pinned host AoS geometry in, pinned host canonical K out, "
                       "chunked H2D/kernel/D2H on two streams)"}

    # -------- CPU baseline (rank 0, N = 1) --------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        n_probe = min(E, 100_000)
        mesh_aos = np.ascontiguousarray(geom_host[:, :n_probe].T).reshape(n_probe, 6, 3)
        caos = np.ascontiguousarray(coeff_host[:, :n_probe].T) if coeff_host is not None else None
        rates, desc, cores, kind = cpu_reference_rates(ps, args.coeff, args.cpu_seconds, mesh_aos, caos)
        cpu = {"value": step_rate(rates, ps), "unit": "elements/s", "cores": cores, "kind": kind,
               "sample": desc, "per_p": {str(p): rates[p] for p in ps},
               "reference_path": "integrate_optimized" if mode == pb.ELASTICITY else "integrate_generic"}

    if rank == 0:
        form = {"laplace": "Laplace c=I", "cdr": "seeded per-element CDR tensors",
                "elasticity": "n_eq=3 isotropic elasticity, per-element (E, nu)"}[args.coeff]
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if esz == 8 else "f64 compute, f32 K",
            "data": f"synthetic (generate_box_mesh 128x64x(64*N), distortion 0.1, seed 42; {form})",
            "config": {"workload": f"{args.coeff} p={','.join(map(str, ps))}, {E} prisms per GPU"
                                   + (" (BASELINE configs[1])" if args.coeff == "laplace" and ps == [2, 3, 4] else ""),
                       "elements_per_gpu": E, "p": ps, "coeff": args.coeff, "n_eq": n_eq, "precision": args.precision,
                       "parallelism": f"element-range x{ws}",
                       "chunk_elements": {str(p): chunk[p] for p in ps},
                       "l2": "inputs (151 MB geometry) and outputs (GBs) exceed the 126 MB L2"},
            "per_p": per_p, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps * launches, "clocks": clk, "parity": parity,
        }
        print(json.dumps(line), flush=True)
    for c in ctxs.values():
        c.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
