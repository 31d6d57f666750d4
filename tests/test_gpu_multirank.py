"""Particle decomposition on the device path: two ranks (gloo, sharing one
GPU) each push their shard of every species and all-reduce the int64
moments; the result must be bit-identical to one rank pushing everything
(the exact lattice makes the moment merge order-free).

Fast arithmetic rounds per-tile partial sums onto the lattice
(bp_split.cu), so its moments depend on how particles fall into tiles: the
particles stay bitwise, the moments agree within the f32 / f64 tolerance."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, port, arith, label, out):
    import torch
    import torch.distributed as dist
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    from paper_2008_04397_b200.pipeline import DeviceSimulation
    distributed = world > 1
    if distributed:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    geom = gem_geometry((16, 8, 8), (6.4, 3.2, 3.2))
    species = gem_species(8)
    prec = PrecisionMode.from_label(label)
    bufs, fields = init_gem_host(geom, species, GemInit(seed=3), prec)
    sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith=arith, sort_period=2,
                           distributed=distributed)
    sim.load_host_buffers(bufs)
    for _ in range(3):
        sim.run_cycle(fields.E if rank == 0 else None, fields.B if rank == 0 else None)
    accs = sim.moments_host()
    parts = [p.to_host() for p in sim.particles]
    if rank == 0:
        out["accs"] = accs
    out[f"parts{rank}"] = [(b.ids, b.x, b.u) for b in parts]
    if distributed:
        dist.destroy_process_group()


@pytest.mark.parametrize("arith,label", [("parity", "single"), ("fast", "double"),
                                         ("fast", "single")])
def test_two_ranks_bitwise_equal_one_rank(gpu, arith, label):
    import torch.multiprocessing as mp
    exact = arith == "parity" or label == "double"  # f64 fast: exact lattice
    tol = 1e-5
    with mp.Manager() as m:
        one = m.dict()
        mp.spawn(_run, args=(1, 0, arith, label, one), nprocs=1, join=True)
        two = m.dict()
        mp.spawn(_run, args=(2, _port(), arith, label, two), nprocs=2, join=True)
        a1, a2 = one["accs"], two["accs"]
        for x, y in zip(a1, a2):
            if exact:
                assert np.array_equal(x, y)
            else:
                for r in range(x.shape[0]):
                    ref = x[r].astype(np.float64)
                    err = np.abs(y[r] - ref).max() / max(np.abs(ref).max(), 1.0)
                    assert err <= tol, (r, err)
        for s in range(4):
            ids1, x1, u1 = one["parts0"][s]
            ids = np.concatenate([two["parts0"][s][0], two["parts1"][s][0]])
            x = np.concatenate([two["parts0"][s][1], two["parts1"][s][1]])
            u = np.concatenate([two["parts0"][s][2], two["parts1"][s][2]])
            o1, o2 = np.argsort(ids1), np.argsort(ids)
            assert np.array_equal(ids1[o1], ids[o2])
            assert np.array_equal(x1[o1], x[o2]) and np.array_equal(u1[o1], u[o2])
