#!/usr/bin/env python
"""Benchmark: element stiffness integration for prisms (arXiv 1310.1191) on B200.

Metric (BASELINE.json): elements integrated per second per degree p, plus the
fraction of the FP64 / HBM roofline.

Headline workload (BASELINE.json configs[1]): Laplace weak form, p = 2, 3, 4,
1,048,576 synthetic prisms per GPU.  One step = one pass of the hot path over
the rank's elements at every p (outputs device-resident).  `value` = elements
processed by all ranks in the timed steps / max-over-ranks device time.

  --scaling weak   (default) generate_box_mesh(128, 64, 64*N, 0.1, 42); rank r
                   owns the contiguous range [r*E, (r+1)*E), E = 1,048,576.
  --scaling strong generate_box_mesh(256, 256, 128, 0.1, 42) = 16,777,216
                   prisms (BASELINE configs[4]) split into N contiguous ranges
                   [floor(rT/N), floor((r+1)T/N)).  No collective on the data path.

Beside the headline the line carries
  * `sweep`: every p = 1..7 for Laplace and per-element CDR (configs[2], [3])
    over the same per-rank elements, median of --reps event-timed passes, with
    executed-FP64 / HBM / dense-count roofline fractions and parity samples;
  * `parity`: SURVEY.md 8(d) sample counts (256 at p <= 4, 64 at p = 5, 16 at
    p >= 6, evenly spaced `sample_indices`, verify.cpp:50-59) against the
    reference's integrate_generic, plus a placement check (each sampled element
    re-integrated alone is bitwise equal) and a digest of the sampled matrices
    (equal across N in strong scaling);
  * `load_vectors`: per p of the step, K alone vs K + load vectors fused into
    the stiffness kernel vs K + the separate sum-factorised load-vector launch
    (pi_integrate_load, LOAD_FUSED / LOAD_SEPARATE), the load kernel alone, and
    F against f x column 0 of the reference's mass matrix;
  * `e2e`: the same step through the host-buffer C-ABI call (pi_integrate_host:
    pinned host geometry in, pinned host K out, all copies timed);
  * `cpu_baseline`: the reference's integrate_generic (oracle/_ref) on the
    host cores (all threads, plus a 1-core figure) over a bounded sample.

  python bench.py [--gpus N --steps K --warmup W --p 2,3,4 --coeff laplace|cdr|elasticity]
  python bench.py --impl reference ...   # the reference CPU integrate_generic, same config
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "elements integrated/sec per degree p (1 and 8 B200) and % of FP64/HBM roofline"
WEAK_MESH = (128, 64, 64)      # per rank: 2*128*64*64 = 1,048,576 prisms
STRONG_MESH = (256, 256, 128)  # 16,777,216 prisms in total
DISTORTION, SEED, COEFF_SEED = 0.1, 42, 42
FORMS = {"laplace": 0, "cdr": 2, "elasticity": 3}  # PI_COEFF_* of the weak form


def sample_count(p: int) -> int:
    """Parity sample per p."""
    return 256 if p <= 4 else 64 if p == 5 else 16


def sample_indices(n: int, want: int):
    """verify.cpp:50-59: evenly spaced sample."""
    if n == 0:
        return []
    want = min(want, n)
    return [0 if want == 1 else i * (n - 1) // (want - 1) for i in range(want)]


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", default="2,3,4")
    ap.add_argument("--coeff", default="laplace", choices=list(FORMS),
                    help="weak form: Laplace, per-element CDR tensors, or n_eq=3 elasticity with per-element (E, nu)")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="f32: the FP32 variant (SURVEY 8f row f3), K in float32")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--mesh", default=None,
                    help="NX,NY,NZ: per-rank box (weak, NZ multiplied by N) or the whole box (strong)")
    ap.add_argument("--out-gb", type=float, default=120.0,
                    help="device output budget per GPU; larger passes stream through it chunk by chunk")
    ap.add_argument("--sweep", default="laplace,cdr", help="weak forms of the p-sweep ('' disables)")
    ap.add_argument("--sweep-p", default="1,2,3,4,5,6,7")
    ap.add_argument("--reps", type=int, default=3, help="timed passes per sweep entry (median reported)")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-load", action="store_true", help="skip the load-vector measurements")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=16.0, help="CPU baseline budget (all threads)")
    ap.add_argument("--cpu1-seconds", type=float, default=4.0, help="CPU baseline budget (1 thread)")
    ap.add_argument("--csv", default=None, help="also write the reference's bench CSV rows (bench.cpp:136-141)")
    # legacy spelling of the per-rank layer count
    ap.add_argument("--nz", type=int, default=None, help=argparse.SUPPRESS)
    a = ap.parse_args(argv)
    if a.nz is not None and a.mesh is None:
        a.mesh = f"{WEAK_MESH[0]},{WEAK_MESH[1]},{a.nz}"
    return a


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Workload:
    """Mesh, this rank's contiguous element range and the config dict both arms print."""

    def __init__(self, args, ws, rank):
        self.scaling = args.scaling
        self.ps = [int(x) for x in args.p.split(",")]
        self.coeff = args.coeff
        if args.scaling == "weak":
            nx, ny, nz = (int(v) for v in args.mesh.split(",")) if args.mesh else WEAK_MESH
            self.mesh = (nx, ny, nz * ws)
            self.total = 2 * nx * ny * nz * ws
            self.E = 2 * nx * ny * nz
            self.first = rank * self.E
        else:
            self.mesh = tuple(int(v) for v in args.mesh.split(",")) if args.mesh else STRONG_MESH
            self.total = 2 * self.mesh[0] * self.mesh[1] * self.mesh[2]
            self.first = rank * self.total // ws                       # partition.rank_range
            self.E = (rank + 1) * self.total // ws - self.first
        self.ws = ws
        self.precision = args.precision
        self.n_eq = 3 if args.coeff == "elasticity" else 1

    def config(self):
        nx, ny, nz = self.mesh
        form = {"laplace": "Laplace c=I", "cdr": "seeded per-element CDR tensors",
                "elasticity": "n_eq=3 isotropic elasticity, per-element (E, nu)"}[self.coeff]
        tag = ""
        if self.coeff == "laplace" and self.ps == [2, 3, 4] and self.scaling == "weak":
            tag = " (BASELINE configs[1])"
        per = "per GPU" if self.scaling == "weak" else f"in total over {self.ws} GPU(s)"
        n = self.E if self.scaling == "weak" else self.total
        return {"workload": f"{self.coeff} p={','.join(map(str, self.ps))}, {n} prisms {per}{tag}",
                "mesh": f"generate_box_mesh({nx}, {ny}, {nz}, {DISTORTION}, {SEED})", "weak_form": form,
                "elements_per_gpu": self.E if self.scaling == "weak" else None, "total_elements": self.total,
                "p": self.ps, "coeff": self.coeff, "n_eq": self.n_eq, "precision": self.precision,
                "parallelism": f"element-range x{self.ws}", "scaling": self.scaling,
                "l2": "no flush needed: inputs (151 MB geometry per 1M prisms) and outputs (GBs) exceed the 126 MB L2"}

    def data(self):
        return (f"synthetic: generate_box_mesh{self.mesh} distortion {DISTORTION} seed {SEED} (the reference's "
                f"generator, geometry.cpp:134-201); coefficients seeded per element ({self.coeff})")


# ----------------------------------------------------------------- CPU legs
def cpu_reference_rates(ps, coeff_kind, budget_s, mesh_aos, coeffs_aos, threads=0):
    """Reference integrate_generic (oracle/_ref) el/s per p on a bounded sample of
    the same mesh -- integrate_optimized, the reference's fastest FP64 path, for
    elasticity.  threads 0 = all host threads.  Returns (rates, samples, cores, kind)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REF_SO, Oracle, Reference, laplace_tensor  # test infrastructure (checker)

    cores = (os.cpu_count() or 1) if threads <= 0 else threads
    kind = "reference" if REF_SO.exists() else "port"
    rates, samples = {}, {}
    per_p = budget_s / max(1, len(ps))
    for p in ps:
        n = 4
        while True:
            g = mesh_aos[:n]
            c = laplace_tensor() if coeff_kind == "laplace" else coeffs_aos[:n]
            t0 = time.perf_counter()
            if coeff_kind == "elasticity":
                if kind == "reference":
                    Reference().integrate_optimized_batch(p, g, c, threads=cores)
                else:
                    o = Oracle()
                    o.integrate_batch(p, g, np.stack([o.elasticity_tensor(*m) for m in c]), n_eq=3)
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
    return rates, samples, cores if kind == "reference" else 1, kind


def step_rate(rates, ps):
    """Elements/s of one step (E elements at every p) from per-p rates."""
    return len(ps) / sum(1.0 / rates[p] for p in ps)


def checker(p, mode, geoms, coeffs, threads=0):
    """The reference's own arithmetic on sampled elements (oracle/_ref), else the C port."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REF_SO, Oracle, Reference, laplace_tensor

    if mode == FORMS["elasticity"]:
        if REF_SO.exists():
            return Reference().integrate_optimized_batch(p, geoms, coeffs, threads=threads)
        o = Oracle()
        return o.integrate_batch(p, geoms, np.stack([o.elasticity_tensor(*m) for m in coeffs]), n_eq=3)
    c = laplace_tensor() if mode == FORMS["laplace"] else coeffs
    if REF_SO.exists():
        out, err = Reference().integrate_batch(p, geoms, c, threads=threads)
        assert err is None, err.message
        return out
    return Oracle().integrate_batch(p, geoms, c)


def checker_name(mode):
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REF_SO

    fn = "integrate_optimized" if mode == FORMS["elasticity"] else "integrate_generic"
    return f"reference {fn} (oracle/_ref)" if REF_SO.exists() else f"oracle port of {fn}"


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


def peaks_hbm():
    """HBM denominator: the driver's MEASURED_PEAKS.json, else the committed copy
    of this pool's measurement (profiles/measured_peaks_pool.json), else the
    B200_PROFILING.md fallback."""
    for path, tag in ((ROOT / "MEASURED_PEAKS.json", "of measured (MEASURED_PEAKS.json)"),
                      (ROOT / "profiles" / "measured_peaks_pool.json",
                       "of measured (this pool's MEASURED_PEAKS.json, committed copy)")):
        try:
            return float(json.load(open(path))["hbm_gbs"]), tag
        except Exception:
            continue
    return 6650.0, "of fallback (B200_PROFILING.md)"


# ------------------------------------------------------------ reference arm
def run_reference_arm(args, ws, rank):
    """The reference's own CPU implementation of the path (oracle/_ref
    integrate_generic, all host threads) on a bounded sample of the same
    workload.  Loads only oracle/ -- never the product library."""
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REF_SO, Oracle, Reference, cdr_coefficients, materials

    W = Workload(args, ws, 0)
    ps = W.ps
    n_probe = min(W.E, 200_000)
    gen = Reference() if REF_SO.exists() else Oracle()
    mesh = gen.box_mesh(*W.mesh, DISTORTION, SEED)[:n_probe].copy()   # rank 0's range starts at 0
    coeffs = (cdr_coefficients(COEFF_SEED, 0, n_probe) if args.coeff == "cdr"
              else materials(0, n_probe) if args.coeff == "elasticity" else None)
    mode = FORMS[args.coeff]
    budget = 6.0  # seconds of CPU work per step
    rates, _, cores, kind = cpu_reference_rates(ps, args.coeff, budget, mesh, coeffs)
    n_p = {p: min(len(mesh), max(1, int(rates[p] * budget / len(ps)))) for p in ps}

    def one_step(acc):
        for p in ps:
            t0 = time.perf_counter()
            checker(p, mode, mesh[: n_p[p]], None if coeffs is None else coeffs[: n_p[p]], threads=cores)
            acc[p] += time.perf_counter() - t0

    scratch = {p: 0.0 for p in ps}
    for _ in range(args.warmup):
        one_step(scratch)
    tsum = {p: 0.0 for p in ps}
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step(tsum)
    wall = time.perf_counter() - t0
    # Per-element cost depends only on p: the bounded sample's
    # rate is the rate of the full step of E elements at every p.
    per_p_rate = {p: n_p[p] * args.steps / tsum[p] for p in ps}
    value = step_rate(per_p_rate, ps)
    sample = (f"each step integrates the first {n_p} elements (per p) of rank 0's range; ms_per_step is that "
              f"sampled step's measured wall time")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": W.data(), "config": W.config(),
        "per_p": {str(p): {"elements_per_s": per_p_rate[p], "sample_elements_per_step": n_p[p]} for p in ps},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": cores, "kind": kind, "sample": sample,
                         "reference_path": checker_name(mode)},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ our arm
class Runner:
    """One rank's device state: inputs resident in HBM, one reused output ring."""

    def __init__(self, args, W, torch, pb, dev, dev_idx, ranks_per_dev):
        self.args, self.W, self.torch, self.pb, self.dev = args, W, torch, pb, dev
        E = W.E
        self.geom_host = pb.generate_box_mesh(*W.mesh, DISTORTION, SEED, first=W.first, count=E, soa=True)
        self.geom = torch.from_numpy(self.geom_host).to(dev)
        self.coeff_host, self.coeff = {}, {}
        self.esz = 4 if args.precision == "f32" else 8
        self.budget = int(args.out_gb / ranks_per_dev * 1e9 / self.esz)
        self.out = None
        self.ctxs = {}
        self.dev_idx = dev_idx
        # a dedicated stream: a NULL handle would mean "the context's own stream"
        self.stream = torch.cuda.Stream(dev)
        self.sptr = self.stream.cuda_stream

    def coeffs(self, form):
        pb, torch = self.pb, self.torch
        if form == "laplace":
            return None, None
        if form not in self.coeff:
            if form == "cdr":
                h = pb.generate_cdr_coefficients(COEFF_SEED, self.W.first, self.W.E, soa=True)
            else:
                h = pb.generate_materials(self.W.first, self.W.E, soa=True)
            self.coeff_host[form] = h
            self.coeff[form] = torch.from_numpy(h).to(self.dev)
        return self.coeff_host[form], self.coeff[form]

    def ctx(self, p, form):
        n_eq = 3 if form == "elasticity" else 1
        if (p, n_eq) not in self.ctxs:
            self.ctxs[(p, n_eq)] = self.pb.Integrator(p, device=self.dev_idx, n_eq=n_eq)
        return self.ctxs[(p, n_eq)]

    def kk(self, p, form):
        n_eq = 3 if form == "elasticity" else 1
        return (n_eq * self.pb.shape_count(p)) ** 2

    def chunk(self, p, form):
        return min(self.W.E, max(1, self.budget // self.kk(p, form)))

    def ensure_out(self, need):
        torch = self.torch
        if self.out is None or self.out.numel() < need:
            self.out = None
            torch.cuda.empty_cache()
            self.out = torch.empty(need, dtype=torch.float32 if self.esz == 4 else torch.float64, device=self.dev)

    def launch(self, p, form, lo, n, out_ptr=None, load=None):
        """load: (device F buffer [E][n_shape], device f [E]) -> pi_integrate_load."""
        _, cdev = self.coeffs(form)
        c0 = None if cdev is None else cdev.data_ptr() + 8 * lo
        kw = {}
        if load is not None:
            nsh = self.pb.shape_count(p)
            kw = {"load_out": load[0].data_ptr() + 8 * nsh * lo, "f": load[1].data_ptr() + 8 * lo}
        self.ctx(p, form).integrate_device(
            n, self.geom.data_ptr() + 8 * lo, out_ptr if out_ptr is not None else self.out.data_ptr(),
            FORMS[form], c0, element_id_base=self.W.first + lo, geom_ld=self.W.E, coeff_ld=self.W.E,
            stream=self.sptr, precision=self.args.precision, **kw)

    def one_pass(self, p, form, on_chunk=None, load=None):
        """Every element of the rank at degree p, chunk by chunk through the output ring."""
        E, ch = self.W.E, self.chunk(p, form)
        n_launch = 0
        for lo in range(0, E, ch):
            n = min(ch, E - lo)
            self.launch(p, form, lo, n, load=load)
            n_launch += 1
            if on_chunk is not None:
                on_chunk(lo, n)
        return n_launch

    def samples(self, p, form, local_idx):
        """Integrate every element (chunked) and copy out the sampled elements' K."""
        torch, kk = self.torch, self.kk(p, form)
        got = {}

        def grab(lo, n):
            sel = [i for i in local_idx if lo <= i < lo + n]
            if not sel:
                return
            self.stream.synchronize()
            for i in sel:
                got[i] = self.out[(i - lo) * kk:(i - lo + 1) * kk].double().cpu().numpy()

        self.ensure_out(self.chunk(p, form) * kk)
        self.one_pass(p, form, grab)
        self.stream.synchronize()
        return np.stack([got[i] for i in local_idx]) if local_idx else np.zeros((0, kk))

    def alone(self, p, form, local_idx):
        """Each sampled element re-integrated as its own 1-element batch (another
        placement: other CTA, other chunk) -- must be bitwise equal."""
        torch, kk = self.torch, self.kk(p, form)
        buf = torch.empty(max(1, len(local_idx)) * kk, dtype=self.out.dtype, device=self.dev)
        for k, i in enumerate(local_idx):
            self.launch(p, form, i, 1, out_ptr=buf.data_ptr() + self.esz * k * kk)
        self.stream.synchronize()
        return buf[: len(local_idx) * kk].double().cpu().numpy().reshape(len(local_idx), kk)

    def close(self):
        for c in self.ctxs.values():
            c.close()


def main_ours(args, ws, rank, local):
    import torch
    import paper_1310_1191_b200 as pb

    ndev = max(1, torch.cuda.device_count())
    dev_idx = local % ndev
    shared = ws > ndev  # several ranks on one GPU (test runs on a 1-GPU box): gloo for the reductions
    torch.cuda.set_device(dev_idx)
    dev = torch.device("cuda", dev_idx)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    red_dev = torch.device("cpu") if shared else dev

    def reduce_max(vals):
        if not dist:
            return [float(v) for v in vals]
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.cpu().tolist()

    def gather(obj):
        if not dist:
            return [obj]
        out = [None] * ws
        dist.all_gather_object(out, obj)
        return out

    def barrier():
        if dist:
            dist.barrier()

    W = Workload(args, ws, rank)
    ps, E = W.ps, W.E
    form = args.coeff
    mode = FORMS[form]
    n_eq = W.n_eq
    ranks_per_dev = max(1, -(-ws // ndev)) if shared else 1
    R = Runner(args, W, torch, pb, dev, dev_idx, ranks_per_dev)
    kk = {p: R.kk(p, form) for p in ps}
    R.ensure_out(max(R.chunk(p, form) * kk[p] for p in ps))
    stream = R.stream

    # ---------------- headline: timed steps ----------------
    def step(events=None):
        n = 0
        for p in ps:
            if events is not None:
                events[p][0].record(stream)
            n += R.one_pass(p, form)
            if events is not None:
                events[p][1].record(stream)
        return n

    for _ in range(max(3, args.warmup)):
        step()
    for p in ps:
        R.ctx(p, form).check()
    torch.cuda.synchronize(dev)

    ev = [{p: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for p in ps}
          for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize(dev)
    launches = 0
    with ClockSampler(dev_idx) as clocks:
        t_start.record(stream)
        for k in range(args.steps):
            launches += step(ev[k])
        t_end.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    for p in ps:
        R.ctx(p, form).check()
    elapsed_ms = t_start.elapsed_time(t_end)
    per_p_ms = {p: float(np.mean([ev[k][p][0].elapsed_time(ev[k][p][1]) for k in range(args.steps)])) for p in ps}
    red = reduce_max([elapsed_ms] + [per_p_ms[p] for p in ps])
    elapsed_ms, per_p_ms = red[0], {p: red[1 + i] for i, p in enumerate(ps)}
    clk = clocks.summary()
    ms_per_step = elapsed_ms / args.steps
    value = W.total * len(ps) / (ms_per_step * 1e-3) if args.scaling == "strong" else ws * E * len(ps) / (ms_per_step * 1e-3)

    # ---------------- roofline inputs ----------------
    dmma_tf, dfma_tf = pb.measure_fp64_peak(dev_idx)
    sm_clock_ghz = (clk.get("sm_mhz") or 1965.0) / 1e3
    fp32_peak_tf = torch.cuda.get_device_properties(dev).multi_processor_count * 128 * 2 * sm_clock_ghz / 1e3
    hbm_peak, hbm_src = peaks_hbm()

    def fractions(p, frm, ms):
        n_eq_f = 3 if frm == "elasticity" else 1
        t = ms * 1e-3
        f_dense = pb.flops_dense_per_element(p, FORMS[frm], n_eq_f)
        f_exec = R.ctx(p, frm).flops_executed_per_element(FORMS[frm])
        byts = pb.bytes_per_element(p, FORMS[frm], n_eq_f) - (8 - R.esz) * R.kk(p, frm)
        ex = f_exec * E / t / 1e12
        hb = byts * E / t / 1e9
        dense_bound_s = max(f_dense * E / (dmma_tf * 1e12), byts * E / (hbm_peak * 1e9))
        # the FP32 variant's p <= 2 scalar kernels compute on the FP32 pipe: their
        # executed FLOPs against the nominal FP32 FMA peak (128 lanes x 2 x SM clock)
        fp32_arith = R.esz == 4 and p <= 2 and n_eq_f == 1
        pipe_peak = fp32_peak_tf if fp32_arith else dmma_tf
        fe, fh = ex / pipe_peak, hb / hbm_peak
        pipe = "fp32" if fp32_arith else "fp64"
        return {
            "elements_per_s": E / t, "ms": ms, "launches": -(-E // R.chunk(p, frm)),
            "dense_flop_alg_per_element": f_dense, "executed_flop_per_element": f_exec, "bytes_per_element": byts,
            "executed_tflops": ex, "hbm_gbs": hb, "dense_tflops": f_dense * E / t / 1e12,
            f"frac_executed_{pipe}": fe, "frac_hbm": hb / hbm_peak,
            "binding": pipe if fe >= fh else "hbm", "frac": max(fe, fh),
            "dense_roofline_elements_per_s": E / dense_bound_s, "frac_of_dense_roofline": dense_bound_s / t,
        }

    per_p = {str(p): fractions(p, form, per_p_ms[p]) for p in ps}

    # ---------------- parity: SURVEY 8(d) samples + placement + digest ----------------
    cores = os.cpu_count() or 1
    chk_threads = max(1, cores // min(ws, cores))

    def parity_for(p, frm):
        ch_host, _ = R.coeffs(frm)
        md = FORMS[frm]
        if args.scaling == "strong":
            gidx = sample_indices(W.total, sample_count(p))
        else:
            gidx = sample_indices(W.total, sample_count(p) * ws)
        lidx = [g - W.first for g in gidx if W.first <= g < W.first + E]
        got = R.samples(p, frm, lidx)
        R.ctx(p, frm).check()
        alone = R.alone(p, frm, lidx)
        same = bool(np.array_equal(got.view(np.uint64), alone.view(np.uint64)))
        digests = {W.first + i: hashlib.sha256(got[k].tobytes()).hexdigest() for k, i in enumerate(lidx)}
        worst = 0.0
        if lidx:
            sys.path.insert(0, str(ROOT / "tests"))
            from oracle_lib import rel_frobenius
            geoms = np.ascontiguousarray(R.geom_host[:, lidx].T).reshape(len(lidx), 6, 3)
            cc = None if ch_host is None else np.ascontiguousarray(ch_host[:, lidx].T)
            ref = checker(p, md, geoms, cc, threads=chk_threads)
            dim = int(round(np.sqrt(got.shape[1])))
            worst = float(rel_frobenius(ref, got.reshape(len(lidx), dim, dim), axis=(1, 2)).max())
        parts = gather((worst, len(lidx), same, digests))
        all_d = {}
        for _, _, _, d in parts:
            all_d.update(d)
        combined = hashlib.sha256("".join(all_d[g] for g in sorted(all_d)).encode()).hexdigest()
        return {"max_rel_frobenius": max(x[0] for x in parts), "elements_checked": sum(x[1] for x in parts),
                "tolerance": 1e-12 if R.esz == 8 else 5e-5, "placement_bitwise_equal": all(x[2] for x in parts),
                "sample_digest": combined[:32], "checker": checker_name(md)}

    parity = None
    if not args.no_parity:
        per_p_parity = {str(p): parity_for(p, form) for p in ps}
        parity = {"max_rel_frobenius": max(v["max_rel_frobenius"] for v in per_p_parity.values()),
                  "tolerance": 1e-12 if R.esz == 8 else 5e-5,
                  "elements_checked": sum(v["elements_checked"] for v in per_p_parity.values()),
                  "placement_bitwise_equal": all(v["placement_bitwise_equal"] for v in per_p_parity.values()),
                  "samples": "sample_indices per p: 256 (p<=4), 64 (p=5), 16 (p>=6), SURVEY 8(d)",
                  "checker": checker_name(mode), "per_p": per_p_parity}

    # ---------------- sweep: p = 1..7, Laplace and CDR ----------------
    sweep = {}
    sweep_forms = [f for f in args.sweep.split(",") if f]
    sweep_ps = [int(x) for x in args.sweep_p.split(",") if x]
    for frm in sweep_forms:
        for p in sweep_ps:
            R.ensure_out(R.chunk(p, frm) * R.kk(p, frm))
            R.one_pass(p, frm)  # warm-up
            R.ctx(p, frm).check()
            times = []
            for _ in range(max(1, args.reps)):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                barrier()
                torch.cuda.synchronize(dev)
                a.record(stream)
                R.one_pass(p, frm)
                b.record(stream)
                torch.cuda.synchronize(dev)
                times.append(a.elapsed_time(b))
            R.ctx(p, frm).check()
            ms = reduce_max([float(np.median(times))])[0]
            entry = fractions(p, frm, ms)
            entry["elements_per_s"] = (W.total if args.scaling == "strong" else ws * E) / (ms * 1e-3)
            entry["reps"] = len(times)
            if not args.no_parity:
                entry["parity"] = parity_for(p, frm)
            sweep[f"{frm}/p{p}"] = entry

    # ---------------- load vectors: fused into the stiffness pass vs standalone ----------------
    loadv = None
    if not args.no_load and n_eq == 1 and R.esz == 8:
        loadv = {}
        fvals = torch.linspace(0.5, 2.0, E, dtype=torch.float64, device=dev)

        def timed(fn):
            fn()
            times = []
            for _ in range(3):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize(dev)
                a.record(stream)
                fn()
                b.record(stream)
                torch.cuda.synchronize(dev)
                times.append(a.elapsed_time(b))
            return reduce_max([float(np.median(times))])[0]

        for p in ps:
            nsh = pb.shape_count(p)
            fbuf = torch.empty(E * nsh, dtype=torch.float64, device=dev)
            R.ensure_out(R.chunk(p, form) * R.kk(p, form))
            it = R.ctx(p, form)
            it.set_load_fusion(pb.LOAD_FUSED)
            ms_fused = timed(lambda: R.one_pass(p, form, load=(fbuf, fvals)))
            it.set_load_fusion(pb.LOAD_SEPARATE)
            ms_sep = timed(lambda: R.one_pass(p, form, load=(fbuf, fvals)))
            it.set_load_fusion(pb.LOAD_AUTO)
            ms_alone = timed(lambda: it.load_vectors_device(E, R.geom, fbuf, f=fvals, stream=R.sptr))
            it.check()
            entry = {"stiffness_only_ms": per_p_ms[p],
                     "fused_ms": ms_fused, "fused_elements_per_s": ws * E / (ms_fused * 1e-3),
                     "fusion_overhead": ms_fused / per_p_ms[p] - 1.0,
                     "separate_ms": ms_sep, "separate_elements_per_s": ws * E / (ms_sep * 1e-3),
                     "auto": "fused" if p == 1 else "separate",
                     "load_kernel_ms": ms_alone, "load_kernel_elements_per_s": ws * E / (ms_alone * 1e-3),
                     "load_kernel_hbm_gbs": (144 + 8 + 8 * nsh) * E / (ms_alone * 1e-3) / 1e9}
            if not args.no_parity:
                # F = f * column 0 of the c[0][0][0][0] = 1 mass matrix (the reference's integrate_generic)
                lidx = sample_indices(E, 64)
                R.one_pass(p, form, load=(fbuf, fvals))  # the AUTO strategy
                torch.cuda.synchronize(dev)
                got = fbuf.view(E, nsh)[lidx].cpu().numpy()
                sys.path.insert(0, str(ROOT / "tests"))
                from oracle_lib import rel_frobenius
                geoms = np.ascontiguousarray(R.geom_host[:, lidx].T).reshape(len(lidx), 6, 3)
                cm = np.zeros((len(lidx), 16))
                cm[:, 0] = 1.0
                mass = checker(p, FORMS["cdr"], geoms, cm, threads=chk_threads)
                ref = mass[:, :, 0] * fvals[lidx].cpu().numpy()[:, None]
                entry["parity"] = {"max_rel_frobenius": float(rel_frobenius(ref, got, axis=1).max()),
                                   "tolerance": 1e-12, "elements_checked": len(lidx),
                                   "checker": "f x column 0 of the reference integrate_generic mass matrix"}
            loadv[str(p)] = entry
            del fbuf

    dom = max(ps, key=lambda p: per_p_ms[p])
    d = per_p[str(dom)]
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and R.esz == 8:  # the committed DRAM measurements are of the FP64 kernels
        try:
            per_el = json.load(open(tf)).get(f"p{dom}_{form}")
            traffic = per_el * R.chunk(dom, form) if per_el is not None else None
        except Exception:
            traffic = None
    ctx_dom = R.ctx(dom, form)
    kname = {(1, 1): "p1_thread_kernel", (2, 1): "p2_lane_kernel", (1, 3): "p1_elastic_lane_kernel",
             (2, 3): "p2_elastic_warp_kernel", (3, 3): "p3_elastic_cta_kernel"}.get(
        (dom, n_eq), f"sumfact_kernel<{dom}, n_eq={n_eq}> (FP64 DMMA)")
    fp64_binds = d["binding"] in ("fp64", "fp32")
    fp32_dom = "frac_executed_fp32" in d
    roofline = {
        "bound": "tensor" if fp64_binds else "hbm", "kernel": kname,
        "achieved": d["executed_tflops"] if fp64_binds else d["hbm_gbs"],
        "peak": (fp32_peak_tf if fp32_dom else dmma_tf) if fp64_binds else hbm_peak,
        "unit": "TFLOP/s" if fp64_binds else "GB/s",
        "frac": d["frac"],
        "traffic": traffic, "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read+write, profiles/traffic.json)",
        "algorithmic_bytes": d["bytes_per_element"] * R.chunk(dom, form),
        "note": ("binding-resource fraction: FLOPs the kernel executes (the analytical count of "
                 "pi_flops_executed_per_element, checked against ncu pipe counters) per launch / launch time, "
                 "against the FP64 pipe peak measured in-run (DMMA m8n8k4; DMMA and DFMA share one FP64 pipe), "
                 "or HBM bytes against the measured copy bandwidth -- whichever is the larger fraction"),
        ("fp32" if fp32_dom else "fp64"): (
            {"executed_tflops": d["executed_tflops"], "peak_tflops": fp32_peak_tf, "frac": d["frac_executed_fp32"],
             "peak_source": "nominal FP32 FMA peak: SMs x 128 lanes x 2 x median SM clock"} if fp32_dom else
            {"executed_tflops": d["executed_tflops"], "peak_tflops": dmma_tf, "frac": d["frac_executed_fp64"],
             "peak_source": f"DMMA m8n8k4 measured in-run (DFMA {dfma_tf:.1f} TF/s)"}),
        "hbm": {"gbs": d["hbm_gbs"], "peak_gbs": hbm_peak, "frac": d["frac_hbm"], "peak_source": hbm_src},
        "dense_count": {"tflops": d["dense_tflops"], "frac_of_fp64_peak": d["dense_tflops"] / dmma_tf,
                        "note": "SURVEY 8(d) dense FLOP_alg (no symmetry / sum-factorisation credit); the kernels "
                                "execute fewer FLOPs, so this ratio exceeds 1 and is not a utilisation"},
        "executed_flop_per_element": ctx_dom.flops_executed_per_element(mode),
    }

    # ---------------- end to end through the host-buffer C-ABI call ----------------
    e2e = None
    if not args.no_e2e and R.esz == 8:
        ch_host, _ = R.coeffs(form)
        geom_aos = torch.from_numpy(np.ascontiguousarray(R.geom_host.T)).pin_memory()
        coeff_aos = torch.from_numpy(np.ascontiguousarray(ch_host.T)).pin_memory() if ch_host is not None else None
        # pinned host output: <= 16 GB per rank; every element's K still crosses PCIe into it
        host_n = {p: min(E, max(1, int(16e9 / 8) // kk[p])) for p in ps}
        host_out = torch.empty(max(host_n[p] * kk[p] for p in ps), dtype=torch.float64).pin_memory()
        ga = geom_aos.numpy()
        ca = coeff_aos.numpy() if coeff_aos is not None else None

        def e2e_step():
            for p in ps:
                it = R.ctx(p, form)
                for lo in range(0, E, host_n[p]):
                    n = min(host_n[p], E - lo)
                    o = host_out[: n * kk[p]].numpy().reshape(n, R.ctx(p, form).dim, R.ctx(p, form).dim)
                    it.integrate_host(ga[lo:lo + n], mode, None if ca is None else ca[lo:lo + n],
                                      element_id_base=W.first + lo, out=o)

        for _ in range(max(1, min(args.warmup, 2))):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        dt = reduce_max([time.perf_counter() - t0])[0]
        cw = 0 if ch_host is None else ch_host.shape[0]
        h2d = E * 18 * 8 * len(ps) + E * cw * 8 * len(ps)
        d2h = sum(E * kk[p] * 8 for p in ps)
        n_all = W.total if args.scaling == "strong" else ws * E
        e2e = {"value": n_all * len(ps) * args.steps / dt, "unit": "elements/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "pcie_gbs": (h2d + d2h) * args.steps / dt / 1e9,
               "path": "pi_integrate_host (pinned host AoS geometry in, pinned host canonical K out, "
                       "chunked H2D/kernel/D2H on two streams)"}

    # ---------------- CPU baseline (rank 0, N = 1) ----------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        ch_host, _ = R.coeffs(form)
        n_probe = min(E, 100_000)
        mesh_aos = np.ascontiguousarray(R.geom_host[:, :n_probe].T).reshape(n_probe, 6, 3)
        caos = np.ascontiguousarray(ch_host[:, :n_probe].T) if ch_host is not None else None
        rates, samples, cores_used, kind = cpu_reference_rates(ps, form, args.cpu_seconds, mesh_aos, caos)
        rates1, samples1, _, _ = cpu_reference_rates(ps, form, args.cpu1_seconds, mesh_aos, caos, threads=1)
        cpu = {"value": step_rate(rates, ps), "unit": "elements/s", "cores": cores_used, "kind": kind,
               "sample": ", ".join(f"p={p}: first {samples[p]} elements" for p in ps) + f" of the same mesh, "
                         f"{cores_used} threads",
               "per_p": {str(p): rates[p] for p in ps},
               "one_core": {"value": step_rate(rates1, ps), "per_p": {str(p): rates1[p] for p in ps},
                            "sample": ", ".join(f"p={p}: first {samples1[p]} elements" for p in ps)},
               "reference_path": checker_name(mode)}

    if args.csv and rank == 0:
        write_csv(args.csv, per_p, sweep, form, E)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64" if R.esz == 8 else "f64 compute, f32 K",
            "data": W.data(), "config": W.config(),
            "chunk_elements": {str(p): R.chunk(p, form) for p in ps},
            "per_p": per_p, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk, "parity": parity, "sweep": sweep, "load_vectors": loadv,
            "ranks_share_gpu": shared,
        }
        print(json.dumps(line), flush=True)
    R.close()
    if dist:
        dist.destroy_process_group()
    return 0


def write_csv(path, per_p, sweep, form, E):
    """Rows in the reference's bench CSV schema (bench.cpp:136-141); `kernel_s`
    is the event-timed device time of one pass over the rank's elements."""
    cols = ("variant,p,device,elements,input_prep_s,buffer_init_s,kernel_s,output_convert_s,total_s,flops,"
            "throughput_gflops,input_jac_bytes,input_nojac_bytes,output_bytes")
    rows = [cols]
    items = [(f"b200-{form}", int(p), v) for p, v in per_p.items()]
    items += [(f"b200-{k.split('/')[0]}", int(k.split('/p')[1]), v) for k, v in sweep.items()]
    for var, p, v in items:
        ks = v["ms"] * 1e-3
        flops = v["dense_flop_alg_per_element"] * E
        out_b = int(round((v["bytes_per_element"] - 144) * E))
        rows.append(f"{var},{p},\"NVIDIA B200\",{E},0,0,{ks},0,{ks},{int(flops)},{flops / ks / 1e9},"
                    f"{144 * E},0,{out_b}")
    Path(path).write_text("\n".join(rows) + "\n")


def main(argv=None):
    args = parse(argv)
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, ws, rank)
    return main_ours(args, ws, rank, local)


if __name__ == "__main__":
    sys.exit(main())
