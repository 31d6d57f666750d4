"""Probe the binned layout at a given size: stats per cycle, count invariant."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import GemInit, gem_fields, gem_geometry, gem_species, init_gem_device, smooth_e_field
from paper_2008_04397_b200.pipeline import DeviceSimulation
cells = tuple(int(c) for c in sys.argv[1].split(",")) if len(sys.argv) > 1 else (128, 64, 64)
ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 125
geom = gem_geometry(cells); species = gem_species(ppc); prec = PrecisionMode.from_label("single")
dev = torch.device("cuda", 0)
sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="fast", device=dev, bin_slack=(float(os.environ.get("SLACK", "0.25")), 16))
parts = init_gem_device(geom, species, dev, precision=prec)
for sid, p in enumerate(parts):
    sim.load_species(sid, p)
    b = sim._bins[sid]
    cnt = b.count.cpu().numpy(); st = b.start.cpu().numpy()
    print("species", sid, "n", p.n, "count sum", cnt.sum(), "min/max", cnt.min(), cnt.max(), "cap", st[-1], "caps min", np.diff(st).min())
f = gem_fields(geom, GemInit(), prec); f.E[...] = smooth_e_field(geom, 1e-4, f.E.dtype)
sim.set_fields(f.E, f.B)
for cyc in range(int(os.environ.get("CYC", "3"))):
    try:
        sim.run_cycle()
    except Exception as e:
        print("cycle", cyc, "raised", e)
    print("cycle", cyc, "stats", sim.bin_stats())
    print("  max counts", [int(b.count.max()) for b in sim._bins])
