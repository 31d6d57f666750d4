"""Full-size checks of the BASELINE.json configurations the headline tests do
not cover ("untested configs"):

* C3 in "mixed" precision (f32 particles, f64 fields, kernels.py's mixed
  promotions): one 65.5M-particle species bitwise against the oracle in parity
  arithmetic and within the north star's 1e-4 in fast arithmetic;
* C4's out-of-core path, bp_fused_span_host (pinned-host batches streamed
  through the device, csrc/bp_capi.cu): several batches whose size is not a
  multiple of 32, bitwise against the oracle on the whole span;
* C5's uniform Maxwellian loader (gem.init_uniform_device) in all three
  precisions: the loaded population (counts per cell, cell-major order,
  charge weight, velocity moments) and one fused step of it bitwise against
  the oracle.
"""

import os

import numpy as np
import pytest

from test_gpu_fullsize import SCALE, _species0
from test_gpu_kernels import _assert_close

pytestmark = pytest.mark.gpu


def _oracle_run(oracle, arrs, n, E, B, inv, tail):
    ref = [a.copy() for a in arrs]
    acc = np.zeros((10,) + inv.shape, np.int64)
    st = oracle.fused_parallel(*ref, 0, n, E, B, acc, inv, *tail, os.cpu_count() or 1)
    return st, ref, acc


@pytest.mark.parametrize("arith", ["parity", "fast"])
def test_c3_species_mixed(gpu, oracle, arith):
    import torch
    from paper_2008_04397_b200 import kernels as K
    geom, p, E, B, inv, tail = _species0((128, 64, 64), "mixed", 1e-3)
    n = p.n
    assert n == 128 * 64 * 64 * 125 and E.dtype == np.float64 and tail[-1] == 1
    st_ref, ref, acc_ref = _oracle_run(oracle, [a.cpu().numpy() for a in p.arrays()], n, E, B,
                                       inv, tail)
    d = list(p.arrays())
    dE, dB, dinv = (torch.from_numpy(a).cuda() for a in (E, B, inv))
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith=arith)
    assert st == st_ref == 0
    got = [t.cpu().numpy() for t in d[:6]]
    acc = dacc.cpu().numpy()
    if arith == "parity":
        for name, r, t in zip("xyzuvw", ref, got):
            assert np.array_equal(r, t), name
        assert np.array_equal(acc_ref, acc)
        return
    # fast: within 1e-4 of each array's max; particles committed within
    # rounding of the reflecting wall may be mirrored by one arithmetic and
    # not the other (tests/test_gpu_fullsize.py), at most 1e-6 of them
    lo, hi = np.float32(geom.origin[1]), np.float32(geom.origin[1] + geom.Ly)
    ulp = np.spacing(hi)
    at_wall = (np.abs(got[1] - hi) <= 4 * ulp) | (np.abs(got[1] - lo) <= 4 * ulp)
    flip = at_wall & (np.sign(got[4]) == -np.sign(ref[4])) & (ref[4] != 0)
    assert flip.sum() <= 1e-6 * n, int(flip.sum())
    got[4] = np.where(flip, -got[4], got[4])
    for name, r, t, per in zip("xyzuvw", ref, got, (geom.Lx, None, geom.Lz, None, None, None)):
        _assert_close(name, r, t, 1e-4, per)
    for m in range(10):
        _assert_close(f"moment {m}", acc_ref[m] * 2.0 ** -43, acc[m] * 2.0 ** -43, 1e-4)


@pytest.mark.parametrize("label", ["single", "double"])
def test_c4_host_streaming_batches(gpu, oracle, label):
    """The pinned-host batch pipeline (kernels.fused_span on numpy arrays ->
    bp_fused_span_host): 4.1M particles in batches of 999,983 (prime, not a
    multiple of 32: five batches, the last one short), bitwise equal to the
    oracle over the whole span, moments included."""
    from paper_2008_04397_b200 import kernels as K
    geom, p, E, B, inv, tail = _species0((64, 32, 16), label, 1e-3)
    n = p.n
    assert n == 64 * 32 * 16 * 125
    host = [a.cpu().numpy().copy() for a in p.arrays()]
    st_ref, ref, acc_ref = _oracle_run(oracle, host, n, E, B, inv, tail)
    acc = np.zeros((10,) + geom.node_shape, np.int64)
    st = K.fused_span(*host, 0, n, E, B, acc, inv, *tail, arith="parity",
                      batch_particles=999_983)
    assert st == st_ref == 0
    for name, r, t in zip("xyzuvw", ref, host[:6]):
        assert np.array_equal(r, t), name
    assert np.array_equal(acc_ref, acc)


@pytest.mark.parametrize("label", ["single", "mixed", "double"])
def test_c5_uniform_loader(gpu, oracle, label):
    """init_uniform_device (the reference's init.kind = uniform,
    pipeline.py:140-151): ppc particles per cell in cell-major order inside
    their cell, charge weight q n0 V / ppc, Maxwellian velocities; then one
    fused step of the loaded species bitwise against the oracle."""
    import torch
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.config import PrecisionMode, SpeciesParams
    from paper_2008_04397_b200.gem import gem_geometry, init_uniform_device
    geom = gem_geometry((32, 16, 16), (6.4, 3.2, 3.2))
    ppc, vth, drift = 64, 0.02, (0.0, 0.0, 0.01)
    species = (SpeciesParams(0, -1.0, 1.0 / 64.0, ppc, vth=(vth,) * 3, drift=drift),)
    prec = PrecisionMode.from_label(label)
    pd, fd = prec.particle_dtype, prec.field_dtype
    p = init_uniform_device(geom, species, torch.device("cuda"), n0=1.0, precision=prec)[0]
    n = geom.n_cells * ppc
    assert p.n == n and p.x.dtype == (torch.float32 if pd == np.float32 else torch.float64)
    h = [a.cpu().numpy() for a in p.arrays()]
    # cell-major, x fastest: particle i lies in cell i // ppc
    cell = np.repeat(np.arange(geom.n_cells), ppc)
    idx = (cell % geom.nx, (cell // geom.nx) % geom.ny, cell // (geom.nx * geom.ny))
    for a in range(3):
        g = (h[a].astype(np.float64) - geom.origin[a]) / geom.spacings[a]
        assert np.all(g >= idx[a] - 1e-6) and np.all(g <= idx[a] + 1 + 1e-6), a
    assert np.all(h[6] == pd(species[0].charge * geom.cell_volume / ppc))
    for a in range(3):
        v = h[3 + a].astype(np.float64)
        assert abs(v.mean() - drift[a]) < 6 * vth / np.sqrt(n), a
        assert abs(v.std() / vth - 1) < 0.01, a
    # one fused step of the loaded species, bitwise against the oracle
    rng = np.random.default_rng(5)
    E = (rng.standard_normal((3,) + geom.node_shape) * 1e-3).astype(fd)
    B = (rng.standard_normal((3,) + geom.node_shape) * 1e-2).astype(fd)
    inv = geom.inv_node_volume(fd)
    geo_f, geo_i = K.make_geo_arrays(geom, pd)
    geo_g, _ = K.make_geo_arrays(geom, fd)
    sc = K.kernel_scalars(species[0], 0.25, 1.0, pd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"],
            3, fd(SCALE), 1 if pd != fd else 0)
    st_ref, ref, acc_ref = _oracle_run(oracle, h, n, E, B, inv, tail)
    d = list(p.arrays())
    dE, dB, dinv = (torch.from_numpy(a).cuda() for a in (E, B, inv))
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith="parity")
    assert st == st_ref == 0
    for name, r, t in zip("xyzuvw", ref, d[:6]):
        assert np.array_equal(r, t.cpu().numpy()), name
    assert np.array_equal(acc_ref, dacc.cpu().numpy())


@pytest.mark.parametrize("arith", ["parity", "fast"])
def test_host_pipeline_concurrent_calls(gpu, arith):
    """Four threads call fused_span on host (numpy) arrays at once — the
    reference's phase-3 thread pool — each with its own particles and
    accumulator: every result bitwise the one of the same call made alone
    (each call borrows its own pipeline, csrc/bp_capi.cu)."""
    from concurrent.futures import ThreadPoolExecutor
    import torch
    from paper_2008_04397_b200 import kernels as K
    geom, p, E, B, inv, tail = _species0((32, 16, 16), "single", 1e-3)
    base = [a.cpu().numpy() for a in p.arrays()]
    n = p.n
    dev = torch.cuda.current_device()

    def run(seed):
        rng = np.random.default_rng(seed)
        perm = rng.permutation(n)  # each task its own particle order
        arrs = [a[perm].copy() for a in base]
        acc = np.zeros((10,) + geom.node_shape, np.int64)
        torch.cuda.set_device(dev)
        st = K.fused_span(*arrs, 0, n, E, B, acc, inv, *tail, arith=arith,
                          batch_particles=100_003)
        return st, arrs, acc

    alone = [run(s) for s in range(4)]
    with ThreadPoolExecutor(max_workers=4) as pool:
        together = list(pool.map(run, range(4)))
    for (s1, a1, c1), (s2, a2, c2) in zip(alone, together):
        assert s1 == s2 == 0
        for x, y in zip(a1, a2):
            assert np.array_equal(x, y)
        assert np.array_equal(c1, c2)
