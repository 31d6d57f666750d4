"""Dev probe: time fused vs push-only vs deposit-only on the GEM bench state
(species 0 and 1), after `steps` cycles of disorder."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
from paper_2008_04397_b200 import kernels as K
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import GemInit, gem_fields, gem_geometry, gem_species, init_gem_device
from paper_2008_04397_b200.pipeline import DeviceSimulation
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
arith = sys.argv[2] if len(sys.argv) > 2 else "fast"
geom = gem_geometry((128, 64, 64)); sp = gem_species(125); prec = PrecisionMode.from_label("single")
dev = torch.device("cuda")
sim = DeviceSimulation(geom, sp, dt=0.25, precision=prec, arith=arith, sort_period=0, device=dev)
for sid, p in enumerate(init_gem_device(geom, sp, dev, precision=prec)):
    sim.load_species(sid, p)
f = gem_fields(geom, GemInit(), prec); sim.set_fields(f.E, f.B)
for _ in range(steps):
    sim.run_cycle()
st = torch.zeros(1, dtype=torch.int32, device=dev)
def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for sid in (0, 1):
    p = sim.particles[sid]; sc = sim.scalars[sid]
    snap = [a.clone() for a in p.arrays()]
    def restore():
        for a, b in zip(p.arrays(), snap): a.copy_(b)
    def fused():
        restore()
        K.fused_span(*p.arrays(), 0, p.n, sim.E, sim.B, sim.acc[sid], sim.invvol, sim.geo_f, sim.geo_g, sim.geo_i,
                     sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3, sim.scale, 0, arith=arith, d_status=st)
    def push():
        restore()
        K.push_span(*p.arrays()[:6], 0, p.n, sim.E, sim.B, sim.geo_f, sim.geo_g, sim.geo_i,
                    sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3, 1, 0, d_status=st)
    def dep():
        restore()
        K.deposit_span(*p.arrays(), 0, p.n, sim.acc[sid], sim.invvol, sim.geo_g, sim.geo_i, 1.0, sim.scale, d_status=st)
    tr = timeit(restore)
    tf, tp, td = timeit(fused) - tr, timeit(push) - tr, timeit(dep) - tr
    print(f"steps {steps} species {sid}: fused {tf:.2f} ms  push(parity) {tp:.2f}  deposit(parity) {td:.2f}  restore {tr:.2f}", flush=True)
