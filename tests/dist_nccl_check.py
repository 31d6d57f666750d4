"""Run under torchrun (tests/test_gpu_nccl.py): the NCCL backend on the GPU
path of pipeline.DeviceSimulation — E/B broadcast, per-species exact int64
moment reduction (all-reduce and reduce-to-root) — must give the same moments
and particles as a non-distributed simulation of the same shard."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    from paper_2008_04397_b200.pipeline import DeviceSimulation

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    geom = gem_geometry((16, 8, 8), (6.4, 3.2, 3.2))
    species = gem_species(8)
    out = {}
    for reduce in ("all", "root"):
        for label in ("single", "double"):
            prec = PrecisionMode.from_label(label)
            bufs, fields = init_gem_host(geom, species, GemInit(seed=5), prec)
            sims = {}
            for distributed in (True, False):
                sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="parity",
                                       sort_period=2, device=dev, distributed=distributed,
                                       reduce=reduce)
                sim.load_host_buffers([b.copy() for b in bufs])
                for _ in range(3):
                    sim.run_cycle(fields.E if rank == 0 else None,
                                  fields.B if rank == 0 else None)
                sims[distributed] = sim
            a, b = sims[True], sims[False]
            if world == 1 or rank == 0 or reduce == "all":
                for x, y in zip(a.acc, b.acc):
                    assert torch.equal(x, y), (reduce, label)
            for pa, pb in zip(a.particles, b.particles):
                for x, y in zip(pa.arrays(), pb.arrays()):
                    assert torch.equal(x, y), (reduce, label)
            out[(reduce, label)] = int(sum(int(t.abs().sum()) for t in a.acc))
    backend = dist.get_backend()
    dist.destroy_process_group()
    if rank == 0:
        print(f"NCCL_OK backend={backend} world={world} cases={len(out)}")


if __name__ == "__main__":
    main()
