"""Small end-to-end workload for compute-sanitizer (scripts/sanitize.sh):
every kernel family of the library on a small GEM box — the flat split f32
kernels (mover, deposit with its shared-memory node patches and __syncwarp
protocol) with the on-device sort, the binned path (TMA bulk-copied cell
records + mbarriers, leaver migration, quarter-warp deposit, re-slack), the
generic parity/f64 kernels, the generic kernel's TMA particle streaming
(BP_TMA_STREAM=1, set by the caller), and the host-array pipeline with two
concurrent calls."""
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

# the host-array pipeline (bp_fused_span_host), two calls at once from two
# threads (each borrows its own pipeline), f32 fast and f64 fast
from concurrent.futures import ThreadPoolExecutor
import numpy as np
from paper_2008_04397_b200 import kernels as K
from paper_2008_04397_b200.fields import MOMENT_SCALE
for label in ("single", "double"):
    prec = PrecisionMode.from_label(label)
    pd, fd = prec.particle_dtype, prec.field_dtype
    p = init_gem_device(geom, species, dev, precision=prec)[0]
    base = [a.cpu().numpy() for a in p.arrays()]
    f = gem_fields(geom, GemInit(), prec)
    inv = geom.inv_node_volume(fd)
    geo_f, geo_i = K.make_geo_arrays(geom, pd)
    geo_g, _ = K.make_geo_arrays(geom, fd)
    sc = K.kernel_scalars(species[0], 0.25, 1.0, pd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
            fd(MOMENT_SCALE), 0)

    def call(_):
        torch.cuda.set_device(dev)
        arrs = [a.copy() for a in base]
        acc = np.zeros((10,) + geom.node_shape, np.int64)
        return K.fused_span(*arrs, 0, p.n, f.E, f.B, acc, inv, *tail, arith="fast",
                            batch_particles=4099)

    with ThreadPoolExecutor(max_workers=2) as pool:
        print(label, "host pipeline ok", list(pool.map(call, range(2))))
