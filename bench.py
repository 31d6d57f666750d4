#!/usr/bin/env python
"""Benchmark: particles moved + interpolated per second on 3D GEM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[2], the metric's "GEM 3D"): 128x64x64 cells,
4 species x 125 particles per cell = 262,144,000 particles, f32 storage
("single" precision), dt 0.25, 3 mover iterations, decks/gem_full.deck
physics; synthetic GEM-shaped particles drawn in HBM (gem.init_gem_device),
the Harris + perturbation B of gem.py and a smooth non-zero E of amplitude
1e-4 (gem.smooth_e_field: ten times the reconnection field 0.1 B0 vA ~ 1e-5
of this deck; the GEM start has E = 0, which would flatter the mover's
boundary-skip test).  The total population is
fixed and split over the ranks by contiguous cell ranges (strong scaling).

A step is one cycle of the device path: E/B broadcast (N>1), zeroing of the
int64 accumulators, the fused mover + deposition kernel for every species,
the per-species exact NCCL all-reduce (N>1), the on-device periodic fold, and
every `sort_period` (10) steps the on-device cell sort.  `value` is
particles x steps / (max over ranks of the CUDA-event time of the K steps).
Inputs (13.6 GB of particle traffic per step) exceed L2 (126 MB), so no L2
flush is needed between steps.

The headline arithmetic is "fast" (native f32 with FMA; within 1e-4 of the
reference, tests/test_gpu_kernels.py); the bitwise "parity" arithmetic is
measured beside it.  `e2e` runs the same workload through the C ABI's
host-buffer entry point bp_fused_span_host (particles in pinned host memory,
streamed H2D -> kernel -> D2H every step).  `cpu_baseline` and the
reference arm time the reference arithmetic (oracle/oracle.cpp, the C++
restatement pinned bitwise to the reference's numba kernels) on the host
cores over a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("particles moved+interpolated/sec (GEM 3D) at 1/2/4/8 B200; HBM GB/s fraction")
UNIT = "particles/s"
BYTES_PER_PARTICLE = {"single": 52, "mixed": 52, "double": 104}  # 13 words, SURVEY §8d
# algorithmic words per particle of each kernel of the f32 fast path
# (bp_split.cu): the mover reads and writes x y z u v w, the deposit reads
# x y z u v w q
KERNEL_WORDS = {"mover": 12, "deposit": 7, "span": 13}
E_AMP = 1e-4  # smooth E in the timed steps (gem.smooth_e_field)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cells", default="128,64,64")
    ap.add_argument("--ppc", type=int, default=125)
    ap.add_argument("--precision", default="single", choices=("single", "mixed", "double"))
    ap.add_argument("--arith", default="fast", choices=("fast", "parity"))
    ap.add_argument("--sort-period", type=int, default=10)
    ap.add_argument("--layout", default="auto", choices=("auto", "flat", "bins"),
                    help="particle layout of the device path (pipeline.DeviceSimulation)")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-shuffled", action="store_true")
    ap.add_argument("--no-c2-double", action="store_true",
                    help="skip the C2 f64 leg (extra.c2_double)")
    ap.add_argument("--no-streams-leg", action="store_true",
                    help="skip the two-stream leg (extra.bin_streams_2)")
    ap.add_argument("--bin-slack", default=None,
                    help="binned layout headroom 'frac,min' (DeviceSimulation.bin_slack)")
    return ap.parse_args()


def slack_kw(args):
    if not args.bin_slack:
        return {}
    f, m = args.bin_slack.split(",")
    return {"bin_slack": (float(f), int(m))}


def workload_config(args, world):
    cells = tuple(int(c) for c in args.cells.split(","))
    n = int(np.prod(cells)) * args.ppc * 4
    dim = "2d" if cells[2] == 1 else "3d"
    traffic = n * 13 * (8 if args.precision == "double" else 4) / 1e9
    return cells, n, {
        "workload": f"gem{dim}_{cells[0]}x{cells[1]}x{cells[2]}_ppc{args.ppc}x4",
        "cells": list(cells), "particles": n, "species": 4, "ppc": args.ppc,
        "precision": args.precision, "arith": args.arith, "mover_iters": 3, "dt": 0.25,
        "sort_period": args.sort_period, "layout": args.layout,
        "decomposition": f"particles/{world} ranks",
        "l2_flush": f"none: {traffic:.1f} GB of particle traffic per step >> 126 MB L2",
    }


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the newest committed ncu capture
    summary that has it (profiles/ncu_summary_r02p.json, then r02o, r02n, r02m, r02h, r02f, r02e, r02b), or None."""
    for tag in ("r02p", "r02o", "r02n", "r02m", "r02h", "r02f", "r02e", "r02b"):
        try:
            with open(os.path.join(ROOT, "profiles", f"ncu_summary_{tag}.json")) as f:
                return float(json.load(f)[kernel]["dram_bytes_per_launch"])
        except Exception:
            continue
    return None


class ClockMonitor:
    """SM clock, power and throttle reasons sampled during the timed region
    (the profiling recipe's clocks line): NVML polled every 2 ms from a
    thread (short timed regions, e.g. 20 steps at 8 GPUs, still get
    samples; one sample is taken at entry and one at exit), else
    nvidia-smi -lms 50."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.thread = None
        self.rows = []

    def _nvml_handle(self, nv):
        try:  # the CUDA device's own PCI address (CUDA and NVML orders can differ)
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _sample(self, nv, h):
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        self.rows.append((float(sm), float(mx), pw,
                          ["Active" if rs & b else "Not Active" for b in bits]))

    def __enter__(self):
        import threading
        self.rows = []
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._nvml_handle(nv)
            self._nv, self._h = nv, h
            self._stop = threading.Event()
            self._sample(nv, h)

            def poll():
                while not self._stop.wait(0.002):
                    try:
                        self._sample(nv, h)
                    except Exception:
                        return
            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=5)
            try:
                self._sample(self._nv, self._h)
            except Exception:
                pass
            return
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for ln in out.splitlines():
                p = [x.strip() for x in ln.split(",")]
                try:
                    self.rows.append((float(p[0]), float(p[1]), float(p[2]), p[3:7]))
                except Exception:
                    continue

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({n for r in rows for n, v in zip(self.NAMES, r[3])
                          if v.lower() == "active"})
        return {"sm_mhz": float(np.median([r[0] for r in rows])), "sm_max_mhz": rows[0][1],
                "power_w_max": max(r[2] for r in rows), "samples": len(rows),
                "source": "nvml" if self.thread is not None else "nvidia-smi",
                "reasons": reasons}


# ------------------------------------------------------------------ CPU legs

def cpu_fused_rate(geom, species, prec, seconds, nthreads, cells_hint=2048):
    """Reference arithmetic (oracle C++ port, all threads) on a bounded GEM
    sample: returns (particles/s, sample description)."""
    from oracle import oracle as O
    from paper_2008_04397_b200.gem import gem_fields, sample_host, GemInit
    from paper_2008_04397_b200.kernels import kernel_scalars, make_geo_arrays
    from paper_2008_04397_b200.fields import MOMENT_SCALE
    O.build()
    fields = gem_fields(geom, GemInit(), prec)
    pd, fd = prec.particle_dtype, prec.field_dtype
    inv = geom.inv_node_volume(fd)
    geo_f, geo_i = make_geo_arrays(geom, pd)
    geo_g, _ = make_geo_arrays(geom, fd)
    acc = np.zeros((10,) + geom.node_shape, np.int64)

    def run(cells):
        bufs = sample_host(geom, species, (geom.n_cells // 3, cells), precision=prec)
        n = sum(b.n for b in bufs)
        t0 = time.perf_counter()
        for s, b in zip(species, bufs):
            sc = kernel_scalars(s, 0.25, 1.0, pd)
            st = O.fused_parallel(b.x, b.y, b.z, b.u, b.v, b.w, b.q_p, 0, b.n, fields.E, fields.B,
                                  acc, inv, geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"],
                                  sc["beta"], sc["one"], s.mover_iters, fd(MOMENT_SCALE),
                                  1 if pd != fd else 0, nthreads)
            assert st == 0, st
        return n, time.perf_counter() - t0

    cells = cells_hint
    n, t = run(cells)  # grow the sample until it is ~`seconds` of CPU work
    while t < 0.5 * seconds and cells < geom.n_cells // 2:
        cells = min(geom.n_cells // 2, int(cells * min(8.0, max(2.0, seconds / max(t, 1e-3)))))
        n, t = run(cells)
    return n / t, (f"{n} particles ({cells} cells x {species[0].ppc} ppc x 4 species, "
                   f"GEM-shaped, cell-sorted) through oracle.fused_parallel, {t:.1f} s")


def reference_arm(args):
    """--impl reference: the reference CPU arithmetic on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import gem_geometry, gem_species
    cells, n_total, config = workload_config(args, world)
    geom = gem_geometry(cells)
    species = gem_species(args.ppc)
    prec = PrecisionMode.from_label(args.precision)
    cores = os.cpu_count() or 1
    per_step = max(1.0, min(args.cpu_seconds, 150.0 / max(args.steps + args.warmup, 1)))
    rates = []
    desc = ""
    for i in range(args.warmup + args.steps):
        r, desc = cpu_fused_rate(geom, species, prec, per_step, cores)
        if i >= args.warmup:
            rates.append(r)
    v = float(np.median(rates))
    config = dict(config, arith="parity (reference numba arithmetic, C++ port)")
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": n_total / v * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f32" if args.precision != "double"
           else "f64", "data": "synthetic", "config": config,
           "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                            "sample": desc + " per step (median of steps)"},
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------ GPU arm

def main_ours(args):
    import torch
    from paper_2008_04397_b200 import _lib
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                           init_gem_device, smooth_e_field)
    from paper_2008_04397_b200.pipeline import DeviceSimulation, shard_span

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; BP_DIST_BACKEND=gloo lets several ranks share one
    # GPU to exercise the multi-rank path where only one GPU exists (testing)
    backend = os.environ.get("BP_DIST_BACKEND", "nccl")
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    L = _lib.load()

    cells, n_total, config = workload_config(args, world)
    geom = gem_geometry(cells)
    species = gem_species(args.ppc)
    prec = PrecisionMode.from_label(args.precision)
    sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith=args.arith,
                           sort_period=args.sort_period, device=dev, distributed=world > 1,
                           layout=args.layout, **slack_kw(args))
    config["layout"] = "bins" if sim.binned else "flat"
    if sim.binned:
        config["bin_slack"] = list(sim.bin_slack)
    c0, nc = shard_span(geom.n_cells, rank, world)
    for sid, p in enumerate(init_gem_device(geom, species, dev, precision=prec, cells=(c0, nc))):
        sim.load_species(sid, p)
    f = gem_fields(geom, GemInit(), prec)
    f.E[...] = smooth_e_field(geom, E_AMP, f.E.dtype)
    sim.set_fields(f.E, f.B)
    n_local = sum(p.n for p in sim.particles)
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()

    def step(timing):
        t = sim.run_cycle()  # phase 1 (N>1): E/B broadcast from rank 0 inside
        timing.append(t)

    # the loaded particles are already cell-sorted: this sort only sizes the
    # sort workspace, before the warm-up, so the timed window starts at a
    # steady-state point of the sort period (warm-up steps move particles)
    sim.sort()
    warm = []
    for _ in range(args.warmup):
        step(warm)
    barrier()
    torch.cuda.synchronize()
    launches0 = L.bp_kernel_launches()
    L.bp_timing_enable(1)
    _lib.timing_read()  # discard anything recorded before the timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timed = []
    with ClockMonitor(local_dev) as mon:
        e0.record()
        for _ in range(args.steps):
            step(timed)
        e1.record()
        torch.cuda.synchronize()
    barrier()
    ktimes = _lib.timing_read()
    L.bp_timing_enable(0)
    launches = L.bp_kernel_launches() - launches0
    elapsed = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    kern = torch.tensor([sum(t.kernel_ms for t in timed)], dtype=torch.float64, device=dev)
    sortms = torch.tensor([sum(t.sort_ms for t in timed)], dtype=torch.float64, device=dev)
    if dist is not None:
        for t in (elapsed, kern, sortms):
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms, kern_ms, sort_ms = float(elapsed), float(kern), float(sortms)
    value = n_total * args.steps / (elapsed_ms * 1e-3)

    # roofline of the dominant kernel (largest device time in the timed
    # region, CUDA events on its launch stream): algorithmic bytes per launch
    # (KERNEL_WORDS x word size x the launch's particles) / mean launch time
    hbm, peak_kind = peaks()
    word = BYTES_PER_PARTICLE[args.precision] // 13
    per_launch_particles = n_local / len(species)
    kinfo = {}
    for k, (ms, cnt) in ktimes.items():
        if cnt and k in KERNEL_WORDS:
            lm = ms / cnt
            ab = per_launch_particles * KERNEL_WORDS[k] * word
            kinfo[k] = {"launches": cnt, "ms_per_launch": lm,
                        "algorithmic_bytes_per_launch": ab,
                        "achieved_gbs": ab / (lm * 1e-3) / 1e9,
                        "frac": ab / (lm * 1e-3) / 1e9 / hbm,
                        "share_of_step": ms / elapsed_ms}
    dom = max(kinfo, key=lambda k: kinfo[k]["ms_per_launch"] * kinfo[k]["launches"])
    dk = kinfo[dom]
    names = {"mover": "bp::sk::mover_kernel (implicit mover, 3 iterations)",
             "deposit": "bp::sk::deposit_kernel (10-moment interpolation)",
             "span": "bp::span_kernel (generic fused mover + deposit)"}
    if sim.binned:
        names.update(mover="bp::bins::mover_bins (implicit mover on cell bins, 3 iterations)",
                     deposit="bp::bins::deposit_bins (10-moment interpolation on cell bins)")
    traffic = ncu_traffic(dom + ("_bins" if sim.binned else "")) if (world == 1 and cells == (128, 64, 64) and args.ppc == 125
                                   and args.precision == "single"
                                   and args.arith == "fast") else None
    roofline = {"bound": "hbm", "achieved": dk["achieved_gbs"], "peak": hbm, "unit": "GB/s",
                "frac": dk["frac"], "traffic": traffic,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs copy)",
                "kernel": names[dom],
                "algorithmic_bytes_per_launch": dk["algorithmic_bytes_per_launch"],
                "launch_ms": dk["ms_per_launch"], "kernels": kinfo}
    # the whole fused phase against the north star's 13 words per particle
    bpp = BYTES_PER_PARTICLE[args.precision]
    launch_ms = kern_ms / (args.steps * len(species))
    roofline["fused_phase"] = {
        "ms_per_species": launch_ms,
        "achieved_gbs": per_launch_particles * bpp / (launch_ms * 1e-3) / 1e9,
        "frac": per_launch_particles * bpp / (launch_ms * 1e-3) / 1e9 / hbm}

    # per-cycle phase-3 device time (the reference's metric: N / phase-3
    # seconds, median and mean +- stddev over the cycles)
    p3 = np.array([t.phase3_ms for t in timed], np.float64)
    extra_p3 = {"median_ms": float(np.median(p3)), "mean_ms": float(p3.mean()),
                "std_ms": float(p3.std()),
                "rank0_particles_per_s_median": n_local / (float(np.median(p3)) * 1e-3)}
    extra = {"phase3_per_cycle": extra_p3,
             "phase3_kernel_ms_per_step": kern_ms / args.steps,
             "sort_ms_per_sort": sort_ms / max(1, sum(t.sorted_this_cycle for t in timed)),
             "phase3_particles_per_s": n_total / (kern_ms / args.steps * 1e-3)}
    if sim.binned:
        # per species, last timed cycle: leavers, overflowed, misplaced, lost,
        # rebuilds so far
        extra["bin_stats"] = sim.bin_stats()

    # bitwise reference arithmetic beside it
    if not args.no_parity and args.arith != "parity":
        # the bitwise arithmetic runs on the flat layout: a second simulation
        # over this one's particles (exported in cell order)
        psim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="parity",
                                sort_period=args.sort_period, device=dev,
                                distributed=world > 1, layout="flat")
        for sid, p in enumerate(sim.particles):
            psim.load_species(sid, p)
        psim.set_fields(f.E, f.B)

        def pstep(timing):
            timing.append(psim.run_cycle())
        pt = []
        for _ in range(2):
            pstep(pt)
        pt = []
        barrier()
        torch.cuda.synchronize()
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ks = max(2, min(args.steps, 5))
        p0.record()
        for _ in range(ks):
            pstep(pt)
        p1.record()
        torch.cuda.synchronize()
        pe = torch.tensor([p0.elapsed_time(p1)], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(pe, op=dist.ReduceOp.MAX)
        extra["parity_arith"] = {"value": n_total * ks / (float(pe) * 1e-3), "unit": UNIT,
                                 "steps": ks, "note": "bitwise-reference arithmetic"}
        del psim, pt
        torch.cuda.empty_cache()

    # the same workload with the species on two streams (BP_BIN_STREAMS=2:
    # one species' deposit shares the SMs with the next one's mover); kept
    # out of the headline so that its per-kernel event times (the roofline)
    # are not inflated by the overlap
    if sim.binned and world == 1 and not args.no_streams_leg:
        os.environ["BP_BIN_STREAMS"] = "2"
        try:
            for _ in range(2):
                sim.run_cycle()
            torch.cuda.synchronize()
            b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with ClockMonitor(local_dev) as mon2:
                b0.record()
                for _ in range(args.steps):
                    sim.run_cycle()
                b1.record()
                torch.cuda.synchronize()
            extra["bin_streams_2"] = {"value": n_total * args.steps / (b0.elapsed_time(b1) * 1e-3),
                                      "unit": UNIT, "steps": args.steps,
                                      "ms_per_step": b0.elapsed_time(b1) / args.steps,
                                      "clocks": mon2.summary()}
        finally:
            os.environ.pop("BP_BIN_STREAMS", None)

    # BASELINE configs[1] (C2, 2D GEM 256 x 128 x 1, f64): the binned f64 fast
    # path, the flat generic f64 fast path and the bitwise arithmetic, with
    # their own clocks (one GPU; skipped when the headline already is f64)
    if world == 1 and not args.no_c2_double and args.precision != "double":
        extra["c2_double"] = c2_double_leg(dev)

    # unsorted worst case: the flat layout with every species randomly
    # permuted and no sort (each particle's cell record and deposit target is
    # a random cell: L2 instead of L1 reuse)
    if not args.no_shuffled and args.precision != "double":
        extra["shuffled"] = shuffled_leg(args, sim, geom, species, prec, f, dist, dev, n_total)

    # end to end through the host-buffer C ABI (pinned host particles)
    e2e = None
    if not args.no_e2e:
        extra["e2e_cycle"] = e2e_cycle_leg(args, sim, f, dist, dev, n_total)
        e2e = e2e_leg(args, sim, species, prec, geom, dist, dev, n_total)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = os.cpu_count() or 1
        rate, desc = cpu_fused_rate(geom, species, prec, args.cpu_seconds, cores)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "port", "sample": desc}
        r1, d1 = cpu_fused_rate(geom, species, prec, max(2.0, args.cpu_seconds / 3), 1,
                                cells_hint=256)
        extra["cpu_1thread"] = {"value": r1, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": d1}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup,
               "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None,
               "dtype": "f32" if args.precision != "double" else "f64",
               "data": "synthetic: the reference GEM loader's particles (Philox seed 20250809, "
                       "generated bit-exactly in HBM by gem.init_gem_device), Harris + "
                       "perturbation B, smooth E",
               "config": config, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": launches, "clocks": mon.summary(), "extra": extra}
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def c2_double_leg(dev, steps=10, warmup=3):
    """C2 in double precision (BASELINE configs[1]): particles/s per step of
    the f64 binned fast path (csrc/bp_bins64.cu), of the flat generic f64
    fast path and of the bitwise reference arithmetic, each over `steps`
    device-timed cycles after `warmup`, one NVML clock record for all."""
    import torch
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                           init_gem_device, smooth_e_field)
    from paper_2008_04397_b200.pipeline import DeviceSimulation
    geom = gem_geometry((256, 128, 1))
    species = gem_species(125)
    prec = PrecisionMode.from_label("double")
    f = gem_fields(geom, GemInit(), prec)
    f.E[...] = smooth_e_field(geom, E_AMP, f.E.dtype)
    n_total = geom.n_cells * 125 * len(species)
    out = {"workload": "gem2d_256x128x1_ppc125x4", "particles": n_total, "steps": steps,
           "warmup": warmup, "unit": UNIT}
    with ClockMonitor(dev.index) as mon:
        for name, arith, layout in (("bins_fast", "fast", "bins"), ("flat_fast", "fast", "flat"),
                                    ("parity", "parity", "flat")):
            sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith=arith,
                                   sort_period=10, device=dev, layout=layout)
            for sid, p in enumerate(init_gem_device(geom, species, dev, precision=prec)):
                sim.load_species(sid, p)
            sim.set_fields(f.E, f.B)
            sim.sort()
            for _ in range(warmup):
                sim.run_cycle()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                sim.run_cycle()
            e1.record()
            torch.cuda.synchronize()
            out[name] = n_total * steps / (e0.elapsed_time(e1) * 1e-3)
            del sim
            torch.cuda.empty_cache()
    out["bins_over_parity"] = out["bins_fast"] / out["parity"]
    out["clocks"] = mon.summary()
    return out


def shuffled_leg(args, sim, geom, species, prec, fields, dist, dev, n_total):
    """Fused phase on randomly permuted particles (flat layout, no sort):
    device time of a few cycles, max over ranks."""
    import torch
    from paper_2008_04397_b200.pipeline import DeviceSimulation
    from paper_2008_04397_b200.particles import DeviceParticles
    ssim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith=args.arith,
                            sort_period=0, device=dev, distributed=dist is not None,
                            layout="flat")
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    for sid, p in enumerate(sim.particles):
        perm = torch.randperm(p.n, device=dev, generator=g)
        ssim.load_species(sid, DeviceParticles(*[a[perm] for a in p.arrays()], p.ids[perm],
                                               species_id=p.species_id))
        del perm
    ssim.set_fields(fields.E, fields.B)
    ssim.run_cycle()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ks = 3
    e0.record()
    for _ in range(ks):
        ssim.run_cycle()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del ssim
    torch.cuda.empty_cache()
    return {"value": n_total * ks / (float(t) * 1e-3), "unit": UNIT, "steps": ks,
            "note": "flat layout, every species randomly permuted, no sort"}


def e2e_cycle_leg(args, sim, fields, dist, dev, n_total):
    """The cycle-level public API with device-resident particles: every step
    the host field solve's E/B go up (pinned host -> HBM), the cycle runs
    (phases 1-4, sort when due), and the moments come back for the solver
    (wall clock, max over ranks)."""
    import torch
    E = torch.from_numpy(np.ascontiguousarray(fields.E)).pin_memory()
    B = torch.from_numpy(np.ascontiguousarray(fields.B)).pin_memory()

    def one():
        # (single rank: each species' folded grid goes D2H while the next
        # species runs; N > 1 reduces on device first, then one copy each)
        sim.run_cycle(E.numpy() if sim.rank == 0 else None, B.numpy() if sim.rank == 0 else None,
                      stream_moments=True)
        return sim.moments_host(reuse=True)

    one()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    steps = max(2, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    nn = sim.geom.n_nodes
    return {"value": n_total * steps / float(dt), "unit": UNIT,
            "h2d_bytes_per_step": int(2 * E.numel() * E.element_size()),
            "d2h_bytes_per_step": int(len(sim.species) * 10 * nn * 8), "steps": steps,
            "path": "DeviceSimulation.run_cycle(E, B, stream_moments=True) + moments_host(): "
                    "particles resident in HBM, E/B H2D and the int64 moments D2H every step "
                    "(each species' copy overlapping the next species' kernels), wall clock"}


def e2e_leg(args, sim, species, prec, geom, dist, dev, n_total):
    """Same workload through bp_fused_span_host: every step streams each
    species from pinned host memory through the device and back."""
    import torch
    from paper_2008_04397_b200 import _lib
    from paper_2008_04397_b200.fields import MOMENT_SCALE
    L = _lib.load()
    host = []
    for p in sim.particles:
        arrs = []
        for a in p.arrays():
            h = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
            h.copy_(a)
            arrs.append(h)
        host.append(arrs)
    E = sim.E.cpu().numpy()
    B = sim.B.cpu().numpy()
    inv = sim.invvol.cpu().numpy()
    accs = [np.zeros((10,) + geom.node_shape, np.int64) for _ in species]
    hp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    tp = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    arith = _lib.ARITH_FAST if args.arith == "fast" else _lib.ARITH_PARITY
    pb = host[0][0].element_size()
    fb = E.dtype.itemsize

    # the species' calls run concurrently from a thread pool, as the
    # reference's phase 3 issues its batch tasks (pipeline.py:164-165,
    # 255-257): each calling thread has its own host pipeline in the library
    from concurrent.futures import ThreadPoolExecutor
    pool = ThreadPoolExecutor(max_workers=len(species))

    def one_species(sid):
        torch.cuda.set_device(dev)  # a worker thread's CUDA device
        s, arrs = species[sid], host[sid]
        sc = sim.scalars[sid]
        rc = L.bp_fused_span_host(arith, pb, fb, *[tp(a) for a in arrs], 0, arrs[0].numel(),
                                  hp(E), hp(B), hp(accs[sid]), hp(inv), hp(sim.geo_f),
                                  hp(sim.geo_g), hp(sim.geo_i), float(sc["dt"]),
                                  float(sc["dth"]), float(sc["qdt2m"]), float(sc["beta"]),
                                  float(sc["one"]), s.mover_iters, sim.scale, sim.mixed,
                                  int(os.environ.get("BP_HOST_BATCH", "0")))
        _lib.check(rc, "bp_fused_span_host")  # (the error text is per thread)

    def one_step():
        list(pool.map(one_species, range(len(species))))

    one_step()  # warm-up (allocations)
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        one_step()
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    pool.shutdown()
    n_local = sum(a[0].numel() for a in host)
    nn = geom.n_nodes
    h2d = n_local * 7 * pb + len(species) * (2 * 3 * nn * fb + nn * fb + 10 * nn * 8)
    d2h = n_local * 6 * pb + len(species) * 10 * nn * 8
    return {"value": n_total * args.e2e_steps / float(dt), "unit": UNIT,
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": args.e2e_steps,
            "path": "bp_fused_span_host (pinned host SoA -> H2D -> fused kernel -> D2H), "
                    "the species' calls from a thread pool (the reference's phase-3 "
                    "concurrency), wall clock, max over ranks"}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
