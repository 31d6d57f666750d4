"""Small end-to-end workload for compute-sanitizer (scripts/sanitize.sh):
every kernel family of the library on a small GEM box — the flat split f32
kernels (mover, deposit with its shared-memory node patches and __syncwarp
protocol) with the on-device sort, the binned path (TMA bulk-copied cell
records + mbarriers, leaver migration, quarter-warp deposit, re-slack), the
generic parity/f64 kernels, and the generic kernel's TMA particle streaming
(BP_TMA_STREAM=1, set by the caller)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                       init_gem_device, smooth_e_field)
from paper_2008_04397_b200.pipeline import DeviceSimulation

geom = gem_geometry((16, 8, 8), (3.2, 1.6, 1.6))
species = gem_species(48)
dev = torch.device("cuda", 0)
runs = [("single", "fast", "flat"), ("single", "fast", "bins"), ("single", "parity", "flat"),
        ("double", "fast", "flat"), ("double", "fast", "bins"), ("mixed", "parity", "flat")]
for label, arith, layout in runs:
    prec = PrecisionMode.from_label(label)
    sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith=arith, sort_period=2,
                           device=dev, layout=layout,
                           bin_slack=(0.05, 0) if layout == "bins" else (0.5, 64))
    for sid, p in enumerate(init_gem_device(geom, species, dev, precision=prec)):
        sim.load_species(sid, p)
    f = gem_fields(geom, GemInit(), prec)
    f.E[...] = smooth_e_field(geom, 1e-3, f.E.dtype)
    sim.set_fields(f.E, f.B)
    for _ in range(3):
        sim.run_cycle()
    sim.fold_moments()
    torch.cuda.synchronize()
    print(label, arith, layout, "ok", sim.bin_stats() if sim.binned else "")
