"""Steady-state behaviour of the binned layout at C3: per cycle the stats of
every species, re-slacks / rebuilds and the cycle time (CUDA events around
run_cycle, host work included), plus the slot occupancy."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                       init_gem_device, smooth_e_field)
from paper_2008_04397_b200.pipeline import DeviceSimulation
geom = gem_geometry((128, 64, 64)); species = gem_species(125)
prec = PrecisionMode.from_label("single")
dev = torch.device("cuda", 0)
sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="fast", device=dev)
for sid, p in enumerate(init_gem_device(geom, species, dev, precision=prec)):
    sim.load_species(sid, p)
f = gem_fields(geom, GemInit(), prec); f.E[...] = smooth_e_field(geom, 1e-4, f.E.dtype)
sim.set_fields(f.E, f.B)
torch.cuda.synchronize()
for cyc in range(int(os.environ.get("CYC", "40"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0 = [b.rebuilds for b in sim._bins]
    e0.record(); t0 = time.perf_counter()
    sim.run_cycle()
    e1.record(); torch.cuda.synchronize()
    r1 = [b.rebuilds for b in sim._bins]
    st = [b.last_stats for b in sim._bins]
    occ = [round(float(b.count.sum()) / b.cap, 3) for b in sim._bins]
    mx = [int((b.count.to(torch.int64) - (b.start[1:] - b.start[:-1])).max()) for b in sim._bins]
    print(f"cycle {cyc:3d} {e0.elapsed_time(e1):7.2f} ms wall {1e3*(time.perf_counter()-t0):7.2f}"
          f" rebuilt {[a - b for a, b in zip(r1, r0)]} overflow {[s[1] for s in st]}"
          f" misplaced {[s[2] for s in st]} occupancy {occ} max(count-cap) {mx}", flush=True)
