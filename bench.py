#!/usr/bin/env python
"""Benchmark: MD atom-steps/s (Cu, FP64) of the B200-native Deep Potential step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c3|c5]

Workload (BASELINE.json configs[1], "C2"): copper-like DP-SE model gen_model(seed 7) with random
weights, compression tables h = 0.01, jittered FCC Cu 20x20x20 cells (32,000 atoms, seed 11),
velocities 330 K (seed 99), velocity-Verlet NVE, dt = 1 fs, list buffer 2 A rebuilt every 50
steps. A step = half kick + drift + (list rebuild on its cadence) + staleness check + full
energy/force/virial evaluation + half kick -- the reference's run_md step (md.cpp:204-225).

Arms:
  ours       value: K device-resident MD steps timed with CUDA events on the library's stream;
             e2e:   the same steps driven through the reference-facing C-ABI dp_compute with host
                    (pinned) buffers: positions up, forces/energy/virial/atom energies down every
                    step, host Verlet update (what a host MD code calling the operator does).
  reference  the unmodified reference library (oracle/_ref, built from /root/reference) timing
             compute_energy_forces_virial_tabulated on the same configuration with every host
             thread, plus its cell-list build amortized over the 50-step rebuild cadence.
Multi-GPU (torchrun): each rank owns its own C2-sized slab (weak scaling); see DESIGN.md §6.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    "c2": dict(cells=(20, 20, 20), label="C2: Cu FCC 20x20x20 (32,000 atoms) NVE MD step"),
    "c3": dict(cells=(64, 64, 64), label="C3: Cu FCC 64x64x64 (1,048,576 atoms) NVE MD step"),
    "c4": dict(cells=(150, 150, 150), strong=True,
               label="C4: Cu FCC 150x150x150 (13,500,000 atoms, the paper's case) NVE MD step"),
    "c5": dict(cells=(100, 100, 100), label="C5: Cu FCC 100x100x100 (4,000,000 atoms) NVE MD step"),
}
MACS_FIT = None  # filled from the model shape


def fitting_flops_per_atom(m) -> float:
    s = m.shape
    din = s.m_lt * 4 * s.d1
    w = s.fit_width
    fwd = din * w + (s.fit_hidden - 1) * w * w + w
    bwd = (s.fit_hidden - 1) * w * w + din * w
    return 2.0 * (fwd + bwd)


def algorithmic_flops_per_atom(m, n_real: float) -> float:
    """SURVEY.md §8d accounting: fitting fwd+bwd + 7,060 FLOP per real neighbour."""
    return fitting_flops_per_atom(m) + 16384 + 32768 + 7060.0 * n_real


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
bus, period = sys.argv[1], float(sys.argv[2])
try:
    h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
except Exception:
    h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[3]))
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
print("ready", flush=True)
import select
while True:
    r, _, _ = select.select([sys.stdin], [], [], period)
    print(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), mx, int(fn(h)), flush=True)
    if r:
        break
"""


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region by a separate NVML process
    (started with the sampler, not forked from a thread mid-run). In-process NVML or nvidia-smi
    queries from a thread of this CUDA process stalled the timed region at random; the sampling
    period is 100 ms."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}

    def __init__(self, gpu: int, period: float = float(os.environ.get("BENCH_CLK_PERIOD", "0.1")),
                 enabled: bool = True):
        self.gpu, self.period, self.enabled = gpu, period, enabled
        self.samples = []
        self._p = None
        try:
            import torch
            pr = torch.cuda.get_device_properties(gpu)
            self.bus = "%08X:%02X:%02X.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        except Exception:
            self.bus = ""

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS") or not self.enabled:
            return self
        try:
            self._p = subprocess.Popen([sys.executable, "-c", _SAMPLER, self.bus, str(self.period), str(self.gpu)],
                                       stdin=subprocess.PIPE, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                       text=True)
            line = self._p.stdout.readline()
            if not line.startswith("ready"):
                self._p = None
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        try:
            out, _ = self._p.communicate("stop\n", timeout=10)
            for line in out.splitlines():
                f = line.split()
                if len(f) == 3:
                    self.samples.append((float(f[0]), float(f[1]), int(f[2])))
        except Exception:
            self._p.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [s[0] for s in self.samples]
        reasons = sorted({name for s in self.samples for bit, name in self.REASONS.items() if s[2] & bit})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": reasons, "samples": len(self.samples), "source": "NVML (sampler process, 100 ms)"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    return world, rank, local, dist


def max_over_ranks(x: float, dist) -> float:
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


def _ref_lib():
    """ctypes handle on oracle/_ref/libdpref.so (the unmodified reference + its C shim), loaded
    WITHOUT importing the product package: nothing of paper_2201_01446_b200 is on this path."""
    import ctypes as C
    so = ROOT / "oracle" / "_ref" / "libdpref.so"
    if not so.exists():
        return None
    L = C.CDLL(str(so))
    D, I64P = C.POINTER(C.c_double), C.POINTER(C.c_int64)
    L.ref_last_error.restype = C.c_char_p
    L.ref_bench_steps.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_uint64,
                                  C.c_uint64, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                                  C.c_int, C.c_double, I64P, D, D, C.POINTER(C.c_int), D]
    return L


def reference_steps(cells, threads: int, warmup: int, max_steps: int, min_steps: int, budget_s: float):
    """The reference's own MD-step cost on its own inputs (ref_shim.cpp ref_bench_steps): gen_model
    (copper-like, seed 7), build_tables(h = 0.01), gen_config(cells, jitter 0.1, seed 11), the cell
    list at r_c + 2 A built once (timed, amortized over the 50-step rebuild cadence), then one
    compute_energy_forces_virial_tabulated (fused.cpp:245) per step with `threads` OpenMP workers."""
    import ctypes as C
    L = _ref_lib()
    if L is None:
        return None
    n_atoms, list_s, n_done, energy = C.c_int64(), C.c_double(), C.c_int(), C.c_double()
    ev = np.zeros(max(max_steps, 1))
    rc = L.ref_bench_steps(b"copper-like", cells[0], cells[1], cells[2], 0.1, 11, 7, 0.01, 2.0, threads,
                           warmup, max_steps, min_steps, budget_s, C.byref(n_atoms), C.byref(list_s),
                           ev.ctypes.data_as(C.POINTER(C.c_double)), C.byref(n_done), C.byref(energy))
    if rc:
        raise RuntimeError("reference bench failed: " + L.ref_last_error().decode())
    ev = ev[: n_done.value]
    step_s = float(np.mean(ev)) + list_s.value / 50.0
    return {"n_atoms": int(n_atoms.value), "list_s": list_s.value, "eval_s": ev.tolist(),
            "step_s": step_s, "value": n_atoms.value / step_s, "energy": energy.value, "cores": threads}


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU implementation of the path on this host, every
    host thread, on the configuration our arm reports (C2 per GPU: Cu 20x20x20 per rank, slabs
    along x, as run_ours builds it). Step = one evaluation + the cell-list build / 50. Rank 0 only.
    """
    if rank != 0:
        return
    spec = CONFIGS[args.config]
    cells = spec["cells"]
    cells = (cells[0] * (1 if spec.get("strong") else world), cells[1], cells[2])
    threads = os.cpu_count() or 1
    if _ref_lib() is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libdpref.so not built (build() needs /root/reference)"}))
        return
    n_cfg = 4 * cells[0] * cells[1] * cells[2]
    if n_cfg > 2_000_000:
        # C3-C5 take minutes per evaluation on the host: time a 32,000-atom block of the same crystal
        # (the reference's cost is O(N))
        cells = (20, 20, 20)
    r = reference_steps(cells, threads, warmup=1, max_steps=args.steps, min_steps=2,
                        budget_s=float(os.environ.get("BENCH_REF_BUDGET_S", "90")))
    st = r["step_s"]
    print(json.dumps({
        "metric": "MD atom-steps/s (Cu, FP64)", "value": r["value"], "unit": "atom-steps/s",
        "impl": "reference", "n_gpus": world, "steps": len(r["eval_s"]), "warmup": 1,
        "ms_per_step": st * 1e3, "higher_is_better": True,
        "scaling": "strong" if spec.get("strong") else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": spec["label"] + (" per GPU (weak scaling, slabs along x)"
                                                if world > 1 and not spec.get("strong") else ""),
                   "atoms_total": r["n_atoms"], "same_config": r["n_atoms"] == n_cfg,
                   "model": "copper-like DP-SE, random weights (reference gen_model seed 7), tables h=0.01",
                   "list": "reference cell list r_c+2 A built once, cost amortized /50"},
        "cpu_baseline": {"value": r["value"], "unit": "atom-steps/s", "cores": threads, "kind": "reference",
                         "sample": f"per step: compute_energy_forces_virial_tabulated on {r['n_atoms']} atoms "
                                   f"(reference gen_config {cells}), {threads} OpenMP threads; "
                                   f"list build {r['list_s']:.2f} s / 50"},
        "e2e": {"value": r["value"], "unit": "atom-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference": {"library": "oracle/_ref/libdpref.so (unmodified /root/reference/proj/src + C shim)",
                      "energy": r["energy"], "eval_s": r["eval_s"], "list_s": r["list_s"]},
        "ns_per_day": r["value"] / r["n_atoms"] * 0.0864,
    }))


def run_ours(args, world, rank, local, dist):
    import torch
    import paper_2201_01446_b200 as dp

    spec = CONFIGS[args.config]
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    cells = spec["cells"]
    strong = bool(spec.get("strong"))
    # weak scaling: the global box grows along x, one C2-sized slab per GPU (partition_domain
    # slices the roomiest axis); N = 1 is the plain single-GPU configuration. Strong scaling
    # (C4): the same 13.5 M-atom box split over the N GPUs.
    gcfg = dp.gen_config("copper-like", cells[0] * (1 if strong else world), cells[1], cells[2], 0.1, 11)
    gvel = dp.init_velocities(gcfg, m, 330.0, 99)
    n_total = gcfg.n_atoms
    n = n_total // world
    pot = dp.DeepPot(m, t, device=local, precision=args.precision)
    if world > 1:
        uid = [dp.DeepPot.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        pot.dist_init(rank, world, uid[0])
    mc = dp.MDConfig(n_steps=args.warmup + args.steps + 140, dt=1.0, buffer=2.0, rebuild_every=50,
                     thermo_every=10 ** 9)
    pot.md_begin(gcfg, gvel, mc)
    pot.md_step(args.warmup)
    stream = torch.cuda.ExternalStream(pot.stream, device=torch.device("cuda", local))
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # clocks sampled by rank 0 only (one NVML process per box; every rank's GPU runs the same
    # step). The sampler process is started BEFORE the barrier: started after it, its ~0.1 s
    # start-up delayed rank 0's first launches while the other ranks' windows were already
    # open, and they waited for rank 0 in the first halo exchange (C2 on 2 GPUs: rank windows
    # 467 vs 579 ms for 100 steps).
    with ClockSampler(local, enabled=rank == 0) as clk:
        torch.cuda.synchronize()
        barrier(dist)
        torch.cuda.synchronize()
        l0 = pot.launch_count
        ev0.record(stream)
        pot.md_step(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier(dist)
    launches = pot.launch_count - l0
    ms_window = ev0.elapsed_time(ev1)
    if world > 1:
        print(f"[bench rank {rank}] window {ms_window:.2f} ms for {args.steps} steps", file=sys.stderr, flush=True)
    # Rebuild amortization: the list is rebuilt every 50 steps, so a K-step window should carry
    # K/50 rebuilds; it carries as many as multiples of 50 fall inside it (often none). Time the
    # next rebuild step alone against single ordinary steps and add the difference for the
    # missing (or extra) share, so `value` is the steady-state rate including rebuilds.
    W, K = args.warmup, args.steps
    in_window = sum(1 for s_ in range(W + 1, W + K + 1) if s_ % 50 == 0)
    to_next = 50 - (W + K) % 50
    if to_next > 1:
        pot.md_step(to_next - 1)

    def one_step():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier(dist)
        a.record(stream)
        pot.md_step(1)
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b)

    rb_ms = [one_step()]
    plain = sorted(one_step() for _ in range(5))
    plain_ms = plain[len(plain) // 2]
    # a rebuild step occasionally carries a one-off buffer growth (seen once: +1.3 s at C3); when
    # 44 more steps are cheap, the following rebuild is timed too and the smaller sample is used
    if max_over_ranks(plain_ms, dist) * 44 < 15000.0:
        pot.md_step(44)
        rb_ms.append(one_step())
    rebuild_extra = max(min(rb_ms) - plain_ms, 0.0)
    ms = ms_window + (K / 50.0 - in_window) * rebuild_extra
    # breakdown pass (not part of the measurement): per-phase CUDA events need the evaluation
    # un-pipelined, so each kernel group's duration is its own (the roofline below uses it)
    nb = min(args.steps, 20)
    pot.set_pipeline(False)
    pot.set_timing(True)
    pot.phase_times()
    pot.md_step(nb)
    phases = pot.phase_times()
    pot.set_timing(False)
    pot.set_pipeline(True)
    res = pot.md_end()
    ms_max = max_over_ranks(ms, dist)
    step_ms = ms_max / args.steps
    value = n_total * args.steps / (ms_max / 1e3)
    cfg, vel = gcfg, gvel

    # roofline of the dominant kernel group: the fitting-net FP64 DMMA GEMMs
    fit_ms, fit_cnt = phases["fitting"]
    fit_flop_launch = fitting_flops_per_atom(m) * n
    # one phase window per evaluation chunk (large systems run in chunks): per step = / nb
    fit_launch_ms = fit_ms / max(nb, 1)
    mixed = args.precision == "mixed"
    if mixed:
        # 3xTF32: three tensor-core products per FP64-equivalent MAC, against the TF32 dense peak
        # (half the measured bf16 dense rate of MEASURED_PEAKS.json)
        achieved = 3 * fit_flop_launch / (fit_launch_ms / 1e3) / 1e12
        try:
            peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"] / 2
            peak_src = "MEASURED_PEAKS.json bf16_tflops / 2 (TF32 dense rate is half of BF16)"
        except Exception:
            peak = 1125.0
            peak_src = "nominal B200 dense TF32 (MEASURED_PEAKS.json unavailable)"
        kernel = ("fitting-net tcgen05 kind::tf32 3xTF32 GEMMs (k_tc_fwd64 forward with FP64-accumulated "
                  "chains, k_tc_gemm backward; 6 launches per chunk)")
    else:
        achieved = fit_flop_launch / (fit_launch_ms / 1e3) / 1e12
        peak = 37.15
        peak_src = ("measured DMMA.8x8x4 37.15 TFLOP/s (profiles/r01_fp64_peak_microbench.log); "
                    "MEASURED_PEAKS.json has no FP64 entry")
        kernel = "fitting-net FP64 DMMA GEMMs (k_gemm, 6 launches/step)"
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            per_atom = json.loads(tf.read_text()).get(args.precision, {}).get("fitting_bytes_per_atom")
            traffic = per_atom * n if per_atom else None
        except Exception:
            traffic = None
    # real pairs per atom of the whole job (md_end sums the counters over the ranks)
    n_real = res.counters.rows_forward / max(res.force_evals, 1) / n_total
    alg = algorithmic_flops_per_atom(m, n_real) * n_total  # FLOP per step, all ranks
    total_phase_ms = sum(v[0] for v in phases.values())

    # e2e through the reference-facing C-ABI with host buffers
    e2e = None
    if not args.no_e2e and world == 1:
        # dp_compute per step: positions up, forces/energy/virial/atom energies down (pinned)
        pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
        c2 = dp.AtomicConfig(cfg.pos, cfg.type, cfg.h)
        pos = pin((n, 3)); pos[:] = cfg.pos
        c2.pos = pos
        v = pin((n, 3)); v[:] = vel
        acc = (1.0 / (1.0e7 / (6.02214076e23 * 1.602176634e-19))) / m.masses[0]
        pot.set_skin(2.0)
        r = pot.compute(c2)
        f = pin((n, 3)); f[:] = r.forces
        ke = args.e2e_steps
        # host integrator (leapfrog kick-drift, in place on the pinned arrays through torch's
        # multithreaded CPU ops: numpy's three temporaries cost 0.2 ms per step at C2)
        tv, tf, tp = torch.from_numpy(v), torch.from_numpy(f), torch.from_numpy(pos)
        tv.add_(tf, alpha=0.5 * acc)
        for k in range(args.warmup + ke):
            if k == args.warmup:
                t0 = time.perf_counter()
            tp.add_(tv)
            r = pot.compute(c2, forces_out=f)
            tv.add_(tf, alpha=acc)
        el = time.perf_counter() - t0
        e2e = {"value": n * ke / el, "unit": "atom-steps/s", "h2d_bytes_per_step": int(n * 24),
               "d2h_bytes_per_step": int(n * 24 + n * 8 + 80), "steps": ke,
               "api": "dp_compute (C-ABI) with pinned host buffers + host leapfrog, list skin 2 A"}
    elif not args.no_e2e:
        # decomposed run through the C-ABI: global state up (dp_md_begin), K steps, global state
        # down (dp_md_end); host wall clock, max over ranks
        ke = args.e2e_steps
        mc2 = dp.MDConfig(n_steps=ke, dt=1.0, buffer=2.0, rebuild_every=50, thermo_every=10 ** 9)
        pos_out = np.empty_like(gcfg.pos)
        vel_out = np.empty_like(gvel)
        barrier(dist)
        t0 = time.perf_counter()
        pot.md_begin(gcfg, gvel, mc2)
        pot.md_step(ke)
        pot.md_end(pos_out, vel_out)
        el = max_over_ranks(time.perf_counter() - t0, dist)
        e2e = {"value": n_total * ke / el, "unit": "atom-steps/s",
               "h2d_bytes_per_step": int(n_total * 52 / ke), "d2h_bytes_per_step": int(n_total * 48 / ke),
               "steps": ke, "api": "dp_md_begin/step/end (C-ABI), global state host<->device each run"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # bounded sample of the same workload on the host: the reference library itself on its own
        # C2 inputs (C3-C5: the C2 block, the reference's cost is O(N))
        thr = os.cpu_count() or 1
        r = reference_steps((20, 20, 20), thr, warmup=0, max_steps=3, min_steps=1, budget_s=15.0)
        if r is not None:
            cpu = {"value": r["value"], "unit": "atom-steps/s", "cores": thr, "kind": "reference",
                   "sample": f"C2 Cu 20x20x20 ({r['n_atoms']} atoms, reference gen_config): "
                             f"{len(r['eval_s'])} x compute_energy_forces_virial_tabulated "
                             f"({np.mean(r['eval_s']):.2f} s each) + cell list {r['list_s']:.2f} s / 50"}
    if rank == 0:
        out = {
            "metric": "MD atom-steps/s (Cu, FP64)" if args.precision == "fp64" else
                      "MD atom-steps/s (Cu, mixed: tcgen05 3xTF32 fitting + tanh table, 1e-5)",
            "value": value, "unit": "atom-steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f64 env/tabulate, tf32x3 fitting",
            "data": "synthetic",
            "config": {"workload": spec["label"] + (" per GPU (weak scaling, slabs along x)"
                                                    if world > 1 and not strong else ""),
                       "atoms_per_gpu": n, "atoms_total": n_total,
                       "model": "copper-like DP-SE, random weights (gen_model seed 7), tables h=0.01",
                       "dt_fs": 1.0, "list": "r_c + 2 A, rebuilt every 50 steps",
                       "parallelism": ("spatial domain decomposition over %d GPUs, NCCL halo send/recv" % world)
                       if world > 1 else "single GPU",
                       "l2": "working set per step > 1 GB (neighbour rows, descriptors), larger than the 126 MB L2"},
            "ns_per_day": value / n_total * 0.0864,
            "roofline": {"bound": "tensor", "kernel": kernel,
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "peak_source": peak_src,
                         "traffic": traffic, "flop_per_launch_group": fit_flop_launch,
                         "group_ms_per_step": fit_launch_ms},
            "step_roofline": {"algorithmic_flop_per_atom_step": alg / n_total,
                              "achieved_tflops": alg * args.steps / (ms_max / 1e3) / 1e12,
                              "frac_of_fp64_peak": alg * args.steps / (ms_max / 1e3) / 1e12 / (37.15 * world),
                              "note": ("FP64-equivalent FLOP of the whole step against the FP64 peak of all GPUs"
                                       + ("; mixed mode runs the fitting on the tf32 tensor cores, so values "
                                          "above 1 are possible" if args.precision == "mixed" else ""))},
            "phases_ms_per_step": {k: v[0] / nb for k, v in phases.items()},
            "phase_sum_ms_per_step": total_phase_ms / nb,
            "phases_note": "breakdown pass of %d further steps with the two-stream pipelining off" % nb,
            "rebuild": {"steps_in_window": in_window, "expected_in_window": K / 50.0,
                        "rebuild_step_extra_ms": rebuild_extra, "rebuild_step_samples_ms": rb_ms,
                        "plain_step_ms": plain_ms,
                        "window_ms": ms_window, "amortized_ms": ms,
                        "note": "value includes the list rebuild every 50 steps at its amortized share"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        if e2e:
            out["e2e"] = e2e
        if cpu:
            out["cpu_baseline"] = cpu
        print(json.dumps(out))
    pot.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=30)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "mixed"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        # CPU only: no process group, no device; under torchrun rank 0 alone runs
        run_reference_arm(args, int(os.environ.get("WORLD_SIZE", str(args.gpus))),
                          int(os.environ.get("RANK", "0")))
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # `python bench.py --gpus N`: start the N ranks ourselves (one process per GPU)
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) visible", file=sys.stderr)
            sys.exit(1)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world, rank, local, dist = dist_setup()
    if world != args.gpus and "WORLD_SIZE" in os.environ and "--gpus" in " ".join(sys.argv):
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(1)
    run_ours(args, world, rank, local, dist)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
