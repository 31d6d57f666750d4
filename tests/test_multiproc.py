"""Multi-rank host logic on CPU (gloo, world size 2): particle shards, field
broadcast and the exact int64 moment all-reduce of pipeline.py reproduce the
single-process result bit for bit.  The per-shard compute is the CPU oracle
(test-side stand-in for the CUDA kernel; the product path never calls it)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    geom = gem_geometry((8, 8, 4), (6.4, 6.4, 3.2))
    species = gem_species(6)
    bufs, fields = init_gem_host(geom, species, GemInit(seed=7), PrecisionMode())
    return geom, species, bufs, fields


def _oracle_moments(O, geom, species, bufs, fields, spans):
    from paper_2008_04397_b200 import kernels as K
    geo_f, geo_i = K.make_geo_arrays(geom, np.float64)
    inv = geom.inv_node_volume(np.float64)
    out = []
    for s, b, (st, cnt) in zip(species, bufs, spans):
        sc = K.kernel_scalars(s, 0.25, 1.0, np.float64)
        acc = np.zeros((10,) + geom.node_shape, np.int64)
        rc = O.fused_span(b.x, b.y, b.z, b.u, b.v, b.w, b.q_p, st, cnt, fields.E, fields.B, acc,
                          inv, geo_f, geo_f, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"],
                          sc["one"], s.mover_iters, 2.0 ** 43, 0)
        assert rc == 0
        out.append(acc)
    return out


def _worker(rank, world, port, result, root=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2008_04397_b200.pipeline import broadcast_fields, reduce_moments, shard_span
        geom, species, bufs, fields = _setup()
        E = torch.from_numpy(fields.E.copy()) if rank == 0 else torch.zeros(fields.E.shape,
                                                                             dtype=torch.float64)
        B = torch.from_numpy(fields.B.copy()) if rank == 0 else torch.zeros(fields.B.shape,
                                                                             dtype=torch.float64)
        broadcast_fields(E, B, src=0)
        assert np.array_equal(E.numpy(), fields.E) and np.array_equal(B.numpy(), fields.B)
        spans = [shard_span(b.n, rank, world) for b in bufs]
        accs = _oracle_moments(O, geom, species, bufs, fields, spans)
        t = [torch.from_numpy(a) for a in accs]
        works = reduce_moments(t, async_op=True, root=root)
        for w in works:
            w.wait()
        if rank == 0:
            result["accs"] = [x.numpy().copy() for x in t]
            result["parts"] = [(b.x[st:st + c].copy(), b.u[st:st + c].copy())
                               for b, (st, c) in zip(bufs, spans)]
    finally:
        dist.destroy_process_group()


def test_shards_cover_every_particle_once():
    from paper_2008_04397_b200.pipeline import shard_span
    for n in (0, 1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            spans = [shard_span(n, r, world) for r in range(world)]
            assert spans[0][0] == 0
            assert all(a[0] + a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert sum(c for _, c in spans) == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


@pytest.mark.parametrize("root", [None, 0], ids=["allreduce", "reduce_to_root"])
def test_two_rank_reduce_equals_single_process(root):
    from oracle import oracle as O
    O.build()
    geom, species, bufs, fields = _setup()
    ref = _oracle_moments(O, geom, species, [b.copy() for b in bufs], fields,
                          [(0, b.n) for b in bufs])
    port = _free_port()
    with mp.Manager() as m:
        result = m.dict()
        mp.spawn(_worker, args=(2, port, result, root), nprocs=2, join=True)
        accs = result["accs"]
    for a, r in zip(accs, ref):
        assert np.array_equal(a, r)
