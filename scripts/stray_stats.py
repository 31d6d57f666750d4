"""Dev probe: per 32-particle tile, how many particles deposit outside the
tile's majority cell, after k steps of the GEM bench workload."""
import sys, os
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
def stats(step):
    for sid in (0, 1, 2, 3):
        p = sim.particles[sid]
        i = ((p.x.double() / geom.dx).long().clamp(max=geom.nx - 1))
        j = ((p.y.double() / geom.dy).long().clamp(max=geom.ny - 1))
        k = ((p.z.double() / geom.dz).long().clamp(max=geom.nz - 1))
        key = (i * 65 + j) * 65 + k
        n = key.numel() // 32 * 32
        t = key[:n].view(-1, 32)
        mode = torch.mode(t, dim=1).values
        nonmaj = (t != mode[:, None]).sum(1).double()
        srt = torch.sort(t, dim=1).values
        distinct = 1 + (srt[:, 1:] != srt[:, :-1]).sum(1).double()
        # distinct stray cells across a window of 4 consecutive tiles of a warp
        w4 = t[: t.shape[0] // 4 * 4].view(-1, 128)
        s4 = torch.sort(w4, dim=1).values
        d4 = 1 + (s4[:, 1:] != s4[:, :-1]).sum(1).double()
        print(f"step {step} species {sid}: non-majority/tile {nonmaj.mean():.2f}, "
              f"distinct cells/tile {distinct.mean():.2f}, distinct cells/4 tiles {d4.mean():.2f}, "
              f"uniform tiles {(nonmaj == 0).double().mean():.3f}", flush=True)
sim.sort(); stats(0)
for s in range(1, 11):
    sim.run_cycle()
    if s in (1, 2, 5, 10):
        stats(s)
