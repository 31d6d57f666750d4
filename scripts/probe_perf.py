"""Dev probe: time the fused parity kernel on one C3-sized species
(128x64x64 cells, ppc 125 -> 65.5M particles), cell-sorted and shuffled."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, threading
try:
    import pynvml; pynvml.nvmlInit(); _h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:
    _h = None
def clocks():
    if _h is None: return -1, -1
    return pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(_h) // 1000
from paper_2008_04397_b200 import kernels as K
from paper_2008_04397_b200.geometry import GridGeometry
from paper_2008_04397_b200.config import SpeciesParams

mode = sys.argv[1] if len(sys.argv) > 1 else "single"
ppc = int(sys.argv[2]) if len(sys.argv) > 2 else 125
arith = sys.argv[3] if len(sys.argv) > 3 else "parity"
pd, fd = {"double": (torch.float64, torch.float64), "single": (torch.float32, torch.float32),
          "mixed": (torch.float32, torch.float64)}[mode]
npd = np.float64 if pd == torch.float64 else np.float32
nfd = np.float64 if fd == torch.float64 else np.float32
cells = tuple(int(c) for c in os.environ.get("PROBE_CELLS", "128,64,64").split(","))
geom = GridGeometry.from_box(cells, tuple(0.2 * c for c in cells), bc=("periodic", "reflecting", "periodic"))
vth = float(os.environ.get("PROBE_VTH", "0.0224"))
dev = torch.device("cuda")
nc = geom.n_cells
n = nc * ppc
g = torch.Generator(device=dev); g.manual_seed(1)
cell = torch.arange(nc, device=dev).repeat_interleave(ppc)
ci = cell % cells[0]; cj = (cell // cells[0]) % cells[1]; ck = cell // (cells[0] * cells[1])
x = ((ci + torch.rand(n, device=dev, generator=g, dtype=torch.float64)) * geom.dx).to(pd)
y = ((cj + torch.rand(n, device=dev, generator=g, dtype=torch.float64)) * geom.dy).to(pd)
z = ((ck + torch.rand(n, device=dev, generator=g, dtype=torch.float64)) * geom.dz).to(pd)
u = (torch.randn(n, device=dev, generator=g, dtype=torch.float64) * vth).to(pd)
v = (torch.randn(n, device=dev, generator=g, dtype=torch.float64) * vth).to(pd)
w = (torch.randn(n, device=dev, generator=g, dtype=torch.float64) * vth).to(pd)
q = torch.full((n,), -1e-4, device=dev, dtype=pd)
shp = (3,) + geom.node_shape
ebs = float(os.environ.get("PROBE_EB", "1"))
E = (torch.randn(shp, device=dev, generator=g, dtype=torch.float64) * 1e-3 * ebs).to(fd)
B = (torch.randn(shp, device=dev, generator=g, dtype=torch.float64) * 1e-2 * ebs).to(fd)
inv = torch.from_numpy(geom.inv_node_volume(nfd)).to(dev)
acc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device=dev)
sp = SpeciesParams(0, -1.0, 1 / 64.0, ppc)
geo_f, geo_i = K.make_geo_arrays(geom, npd)
geo_g, _ = K.make_geo_arrays(geom, nfd)
sc = K.kernel_scalars(sp, 0.25, 1.0, npd)
mixed = 1 if pd != fd else 0
st = torch.zeros(1, dtype=torch.int32, device=dev)
def run():
    K.fused_span(x, y, z, u, v, w, q, 0, n, E, B, acc, inv, geo_f, geo_g, geo_i, sc["dt"], sc["dth"],
                 sc["qdt2m"], sc["beta"], sc["one"], 3, nfd(2.0**43), mixed, arith=arith, d_status=st)
labels = ("sorted",) if os.environ.get("PROBE_SORTED_ONLY") else ("sorted", "shuffled")
for label in labels:
    if label == "shuffled":
        perm = torch.randperm(n, device=dev, generator=g)
        for t in (x, y, z, u, v, w):
            t.copy_(t[perm])
    for _ in range(2): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    it = int(os.environ.get("PROBE_IT", "5"))
    e0.record()
    for _ in range(it): run()
    samples = []
    stop = threading.Event()
    def mon():
        while not stop.is_set():
            samples.append(clocks()); time.sleep(0.002)
    th = threading.Thread(target=mon); th.start()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / it
    bytes_ = n * 13 * (4 if pd == torch.float32 else 8)
    print(f"{mode} {arith} {label}: n={n} {ms:.3f} ms/pass  {n/ms/1e6:.2f} G particles/s  "
          f"{bytes_/ms/1e6:.0f} GB/s algorithmic  status={int(st.item())} clk/W={samples[len(samples)//2] if samples else None}", flush=True)
