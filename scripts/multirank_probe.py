"""Dev probe: the 2-rank device path under torchrun (gloo on one GPU)."""
import faulthandler, os, sys, sys
faulthandler.dump_traceback_later(60, exit=True)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2008_04397_b200.config import PrecisionMode
from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
from paper_2008_04397_b200.pipeline import DeviceSimulation
dist.init_process_group("gloo")
rank = dist.get_rank()
torch.cuda.set_device(0)
print("rank", rank, "init ok", flush=True)
geom = gem_geometry((16, 8, 8), (6.4, 3.2, 3.2))
species = gem_species(8)
prec = PrecisionMode.from_label("single")
bufs, fields = init_gem_host(geom, species, GemInit(seed=3), prec)
sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="fast", sort_period=2, distributed=True)
sim.load_host_buffers(bufs)
print("rank", rank, "loaded", flush=True)
for c in range(3):
    t = sim.run_cycle(fields.E if rank == 0 else None, fields.B if rank == 0 else None)
    print("rank", rank, "cycle", c, t.particles, flush=True)
dist.destroy_process_group()
print("rank", rank, "done", flush=True)
