"""C5 (BASELINE.json configs[4]): uniform Maxwellian plasma, particle-count
sweep 1e7..1e9 per GPU, double / single / mixed precision, fast and parity
arithmetic: throughput and fraction of the HBM roofline of the fused phase.

  python scripts/sweep_c5.py [--sizes 1e7,1e8,1e9] [--steps 10] > out.jsonl
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_04397_b200.config import PrecisionMode, SpeciesParams
from paper_2008_04397_b200.gem import VTH_E, gem_geometry, init_uniform_device
from paper_2008_04397_b200.pipeline import DeviceSimulation
from bench import ClockMonitor

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="1e7,1e8,1e9")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--modes", default="single,mixed,double")
ap.add_argument("--ariths", default="fast,parity")
ap.add_argument("--bin-slack", default="0.25,16",
                help="binned-layout headroom (1e9 particles: two buffer sets must fit)")
args = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
dev = torch.device("cuda")
geom = gem_geometry((128, 64, 64))
for n_target in (float(x) for x in args.sizes.split(",")):
    ppc = max(1, round(n_target / geom.n_cells))
    for mode in args.modes.split(","):
        prec = PrecisionMode.from_label(mode)
        sp = (SpeciesParams(0, -1.0, 1.0 / 64.0, ppc, vth=(VTH_E,) * 3),)
        for arith in args.ariths.split(","):
            fr, mn = args.bin_slack.split(",")
            sim = DeviceSimulation(geom, sp, dt=0.25, precision=prec, arith=arith,
                                   sort_period=10, device=dev, bin_slack=(float(fr), int(mn)))
            sim.load_species(0, init_uniform_device(geom, sp, dev, n0=0.0795774715,
                                                    precision=prec)[0])
            n = sim.particles[0].n
            for _ in range(2):
                sim.run_cycle()
            sim.sort()  # spare buffers and sort workspace sized outside the timed steps
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            kern = 0.0
            with ClockMonitor(torch.cuda.current_device()) as mon:
                e0.record()
                for _ in range(args.steps):
                    kern += sim.run_cycle().kernel_ms
                e1.record()
                torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            bpp = 104 if mode == "double" else 52
            rate_k = n / (kern / args.steps * 1e-3)
            print(json.dumps({"config": "C5 uniform maxwellian", "particles": n, "ppc": ppc,
                              "precision": mode, "arith": arith,
                              "particles_per_s_step": n / (ms * 1e-3),
                              "particles_per_s_kernel": rate_k,
                              "hbm_frac_kernel": rate_k * bpp / 1e9 / peak,
                              "ms_per_step": ms,
                              "layout": "bins" if sim.binned else "flat",
                              "clocks": mon.summary()}), flush=True)
            del sim
            torch.cuda.empty_cache()
