"""Out-of-core path (BASELINE.json configs[3]): a population held in pinned
host memory is streamed through the device every step by the C ABI's
bp_fused_span_host (three batches in flight on three CUDA streams), with the
device working set capped by a byte budget (the reference's ByteBudget,
pipeline.py:47-77).  Reported against the measured host<->device link.

The full C4 deck (256x128x128, 7.25e9 f32 particles, 203 GB) exceeds this
box's host RAM (196 GB), so the run streams a population --particles large
through a --budget-gb device budget.

  python scripts/bench_out_of_core.py [--particles 2e9] [--budget-gb 2] [--steps 2] [--precision double]
"""
import argparse, ctypes, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_04397_b200 import _lib
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.fields import MOMENT_SCALE
from paper_2008_04397_b200.gem import GemInit, gem_fields, gem_geometry, gem_species, init_gem_device
from paper_2008_04397_b200.kernels import kernel_scalars, make_geo_arrays
from bench import ClockMonitor

ap = argparse.ArgumentParser()
ap.add_argument("--particles", type=float, default=2e9)
ap.add_argument("--budget-gb", type=float, default=2.0)  # 6-12M-particle batches: less pipeline fill / drain per species (8 GB: -11%)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--arith", default="fast")
ap.add_argument("--precision", default="single", choices=("single", "double"),
                help="BASELINE configs[3] is f64; single is the f32 variant")
args = ap.parse_args()
dev = torch.device("cuda")
L = _lib.load()
prec = PrecisionMode.from_label(args.precision)
pd = prec.particle_dtype
tdt = torch.float32 if pd == np.float32 else torch.float64
pb = np.dtype(pd).itemsize
geom = gem_geometry((256, 128, 128))
ppc = max(1, int(round(args.particles / (4 * geom.n_cells))))
species = gem_species(ppc)

# link bandwidth: pinned 1 GiB copies
def link_bw():
    h = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
    d = torch.empty(1 << 28, dtype=torch.float32, device=dev)
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5): fn()
        torch.cuda.synchronize()
        out[name] = 5 * (1 << 30) / (time.perf_counter() - t) / 1e9
    return out
bw = link_bw()

# build the host population species by species in slabs of cells (the
# bit-exact device loader, then D2H into pinned host memory)
from paper_2008_04397_b200.gem import sheet_drifts
from paper_2008_04397_b200.particles import init_maxwellian_device
init = GemInit()
yc, lam = geom.origin[1] + 0.5 * geom.Ly, init.sheet_thickness
u_e, u_i = sheet_drifts(species, init, 1.0)
dens = [lambda x, y, z: init.n0 / np.cosh((y - yc) / lam) ** 2,
        lambda x, y, z: np.full_like(np.asarray(y, dtype=np.float64),
                                     init.background_fraction * init.n0)]
drifts = [(0.0, 0.0, u_e), (0.0, 0.0, u_i), (0.0, 0.0, 0.0), (0.0, 0.0, 0.0)]
host = []
slab = 1 << 20
for s in species:
    n = geom.n_cells * s.ppc
    arrs = [torch.empty(n, dtype=tdt, pin_memory=True) for _ in range(7)]
    for c0 in range(0, geom.n_cells, slab):
        nc = min(slab, geom.n_cells - c0)
        part = init_maxwellian_device(s, geom, dev, density_fn=dens[0 if s.species_id < 2 else 1],
                                      seed=init.seed, precision=prec,
                                      drift=drifts[s.species_id], cells=(c0, nc))
        for h, d in zip(arrs, part.arrays()):
            h[c0 * s.ppc:(c0 + nc) * s.ppc].copy_(d)
        del part
    host.append(arrs)
torch.cuda.empty_cache()
f = gem_fields(geom, GemInit(), prec)
E, B = f.E, f.B
inv = geom.inv_node_volume(prec.field_dtype)
accs = [np.zeros((10,) + geom.node_shape, np.int64) for _ in species]
geo_f, geo_i = make_geo_arrays(geom, pd)
gf = np.ascontiguousarray(geo_f, np.float64)
gi = np.ascontiguousarray(geo_i, np.int64)
# three slots x 7 arrays x batch x 4 B within the budget (fields / acc aside)
batch = min(int(args.budget_gb * 1e9 / (3 * 7 * pb)), 1 << 25)  # >= ~16 batches/species keep the pipeline full
hp = lambda a: ctypes.c_void_p(a.ctypes.data)
tp = lambda t: ctypes.c_void_p(t.data_ptr())
arith = _lib.ARITH_FAST if args.arith == "fast" else _lib.ARITH_PARITY

def step():
    for sid, (s, arrs) in enumerate(zip(species, host)):
        sc = kernel_scalars(s, 0.25, 1.0, pd)
        rc = L.bp_fused_span_host(arith, pb, E.dtype.itemsize, *[tp(a) for a in arrs], 0,
                                  arrs[0].numel(), hp(E),
                                  hp(B), hp(accs[sid]), hp(inv), hp(gf), hp(gf), hp(gi),
                                  float(sc["dt"]), float(sc["dth"]), float(sc["qdt2m"]),
                                  float(sc["beta"]), float(sc["one"]), s.mover_iters,
                                  float(MOMENT_SCALE), 0, batch)
        _lib.check(rc, "bp_fused_span_host")
step()
with ClockMonitor(torch.cuda.current_device()) as mon:
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t) / args.steps
n = sum(a[0].numel() for a in host)
h2d, d2h = n * 7 * pb, n * 6 * pb
print(json.dumps({"config": "C4-style out-of-core GEM 3D 256x128x128", "particles": n, "ppc": ppc,
                  "precision": args.precision,
                  "host_bytes": n * 7 * pb, "device_budget_gb": args.budget_gb,
                  "batch_particles": batch, "arith": args.arith,
                  "particles_per_s": n / dt, "s_per_step": dt,
                  "link_gbs_measured": bw, "h2d_gbs": h2d / dt / 1e9, "d2h_gbs": d2h / dt / 1e9,
                  "link_frac_h2d": h2d / dt / 1e9 / bw["h2d"],
                  "clocks": mon.summary(),
                  "note": "full C4 (7.25e9 particles, 203 GB) exceeds the 196 GB host RAM"}),
      flush=True)
