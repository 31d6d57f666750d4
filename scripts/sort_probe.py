"""Dev probe: warm device time of the cell sort of one C3 species (65.5M
particles) after 10 GEM steps of disorder."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import GemInit, gem_fields, gem_geometry, gem_species, init_gem_device
from paper_2008_04397_b200.pipeline import DeviceSimulation
geom = gem_geometry((128, 64, 64)); sp = gem_species(125); prec = PrecisionMode.from_label("single")
dev = torch.device("cuda")
sim = DeviceSimulation(geom, sp, dt=0.25, precision=prec, arith="fast", sort_period=0, device=dev)
for sid, p in enumerate(init_gem_device(geom, sp, dev, precision=prec)):
    sim.load_species(sid, p)
f = gem_fields(geom, GemInit(), prec); sim.set_fields(f.E, f.B)
for _ in range(10):
    sim.run_cycle()
p = sim.particles[0]
snap = [a.clone() for a in p.arrays()] + [p.ids.clone()]
def restore():
    for a, b in zip(list(p.arrays()) + [p.ids], snap): a.copy_(b)
ts = []
for it in range(4):
    restore(); p.sort_by_cell(geom); torch.cuda.synchronize()
    restore(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); p.sort_by_cell(geom); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("sort ms per species (65.5M):", " ".join(f"{t:.3f}" for t in ts))
