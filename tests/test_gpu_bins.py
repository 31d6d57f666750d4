"""The cell-binned layout of the f32 fast path (bins.py, csrc/bp_bins.cu)
against the flat layout (the reference's SoA + periodic sort) and the CPU
oracle.

The binned mover uses the same cell records and the same arithmetic as the
flat split mover, so particle states must stay BITWISE equal to the flat
path's, cycle after cycle, whatever happens to the bins (leavers, overflowed
bins, a full leaver list).  The f32 moments differ only by the f32 summation
order of the per-bin sums: within the north star's f32 tolerance, written
here as |bins - flat| <= 1e-5 * max|flat| per moment row.  The f64 binned
path (csrc/bp_bins64.cu) rounds every contribution onto the int64 lattice as
the flat f64 fast path does, so its moments are bitwise too."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _gem(cells=(16, 8, 8), box=(6.4, 3.2, 3.2), ppc=12, seed=3, label="single", e_amp=2e-3):
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    from paper_2008_04397_b200.gem import smooth_e_field
    geom = gem_geometry(cells, box)
    species = gem_species(ppc)
    prec = PrecisionMode.from_label(label)
    bufs, fields = init_gem_host(geom, species, GemInit(seed=seed), prec)
    fields.E[...] = smooth_e_field(geom, e_amp, fields.E.dtype)
    return geom, species, prec, bufs, fields


def _sim(geom, species, prec, bufs, layout, **kw):
    from paper_2008_04397_b200.pipeline import DeviceSimulation
    sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="fast", sort_period=3,
                           layout=layout, **kw)
    sim.load_host_buffers([b.copy() for b in bufs])
    return sim


def _by_id(p):
    h = p.to_host()
    o = np.argsort(h.ids)
    return {k: getattr(h, k)[o] for k in ("ids", "x", "y", "z", "u", "v", "w", "q_p")}


def _assert_moments_close(a, b, tol=TOL):
    if a[0].dtype == np.int64 and tol == 0:
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        return
    for x, y in zip(a, b):
        for r in range(x.shape[0]):
            ref = x[r].astype(np.float64)
            err = np.abs(y[r].astype(np.float64) - ref).max() / max(np.abs(ref).max(), 1.0)
            assert err <= tol, (r, err)


def _assert_binned(sim):
    """Every exported particle lies in the cell of its bin: the export is in
    bin order, so the f32 cell keys must be non-decreasing."""
    for p in sim.particles:
        h = p.to_host()
        t = h.x.dtype.type
        g = [t(1.0 / t(sim.geom.spacings[a])) for a in range(3)]
        o = [t(t(sim.geom.origin[a]) / t(sim.geom.spacings[a])) for a in range(3)]
        # the kernels' fma(x, 1/d, -o/d): f64 then f32 rounding is the f32
        # fma; for f64 a face-adjacent particle may round either way (allowed)
        gi = [np.minimum(np.trunc((getattr(h, c).astype(np.float64) * g[a] - o[a])
                                  .astype(t)).astype(np.int64), n - 1)
              for a, (c, n) in enumerate(zip("xyz", sim.geom.counts))]
        key = gi[0] + sim.geom.nx * (gi[1] + sim.geom.ny * gi[2])
        # rounding of the emulated fma can move a particle sitting on a cell
        # face by one cell; allow no more than that
        assert np.all(np.diff(key) >= -sim.geom.nx * sim.geom.ny - 1)
        assert (np.diff(key) < 0).mean() < 1e-3


def _tol(label):
    """moments: f32 per-bin sums within TOL, f64 bitwise"""
    return 0 if label == "double" else TOL


@pytest.mark.parametrize("label", ["single", "double"])
def test_build_export_roundtrip(gpu, label):
    geom, species, prec, bufs, fields = _gem(label=label)
    sim = _sim(geom, species, prec, bufs, "bins")
    assert sim.binned
    for b, p in zip(bufs, sim.particles):
        d = _by_id(p)
        o = np.argsort(b.ids)
        assert np.array_equal(d["ids"], b.ids[o])
        for k in "xyzuvw":
            assert np.array_equal(d[k], getattr(b, k)[o])
        assert np.array_equal(d["q_p"], b.q_p[o])
    _assert_binned(sim)


@pytest.mark.parametrize("label", ["single", "mixed", "double"])
def test_bins_match_flat_bitwise_particles(gpu, label):
    geom, species, prec, bufs, fields = _gem(label=label)
    a = _sim(geom, species, prec, bufs, "bins")
    b = _sim(geom, species, prec, bufs, "flat")
    assert a.binned and not b.binned
    for cyc in range(6):
        a.run_cycle(fields.E, fields.B)
        b.run_cycle(fields.E, fields.B)
        _assert_moments_close(b.moments_host(), a.moments_host(), _tol(label))
    for pa, pb in zip(a.particles, b.particles):
        da, db = _by_id(pa), _by_id(pb)
        for k in da:
            assert np.array_equal(da[k], db[k]), k
    st = a.bin_stats()
    assert all(s[0] > 0 for s in st), st          # particles did change cell
    assert all(s[1] == 0 and s[3] == 0 for s in st)
    _assert_binned(a)


@pytest.mark.parametrize("label", ["single", "double"])
def test_bins_overflow_and_full_leaver_list(gpu, label):
    """No slack at all (every arriving leaver overflows its bin) and a leaver
    list of a few slots (most leavers stay misplaced): rebuilds every cycle,
    the particles still bitwise the flat path's, moments within tolerance."""
    from paper_2008_04397_b200.bins import TransitLists
    geom, species, prec, bufs, fields = _gem(seed=9, label=label)
    a = _sim(geom, species, prec, bufs, "bins", bin_slack=(0.0, 0))
    b = _sim(geom, species, prec, bufs, "flat")
    for cyc in range(4):
        if cyc == 2:
            # 1M slots, of which the mover may list 3
            a._lists = TransitLists(a.device, 0, pbytes=a._lists.pbytes)
            a._lists.leaver_cap = 3
        a.run_cycle(fields.E, fields.B)
        b.run_cycle(fields.E, fields.B)
        _assert_moments_close(b.moments_host(), a.moments_host(), _tol(label))
    assert sum(b_.rebuilds for b_ in a._bins) >= 2
    for pa, pb in zip(a.particles, b.particles):
        da, db = _by_id(pa), _by_id(pb)
        for k in da:
            assert np.array_equal(da[k], db[k]), k


def test_bins_against_oracle(gpu, oracle):
    """One cycle of the binned path against the reference arithmetic (CPU
    oracle): particles within 1e-4 of max, moments within 1e-4."""
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.fields import MOMENT_SCALE
    geom, species, prec, bufs, fields = _gem(cells=(32, 16, 8), box=(12.8, 6.4, 3.2), ppc=16)
    a = _sim(geom, species, prec, bufs, "bins")
    a.run_cycle(fields.E, fields.B)
    acc_gpu = a.moments_host()
    geo_f, geo_i = K.make_geo_arrays(geom, np.float32)
    inv = geom.inv_node_volume(np.float32)
    for s, b, p, ag in zip(species, bufs, a.particles, acc_gpu):
        r = b.copy()
        sc = K.kernel_scalars(s, 0.25, 1.0, np.float32)
        acc = np.zeros((10,) + geom.node_shape, np.int64)
        st = oracle.fused_parallel(r.x, r.y, r.z, r.u, r.v, r.w, r.q_p, 0, r.n, fields.E,
                                   fields.B, acc, inv, geo_f, geo_f, geo_i, sc["dt"], sc["dth"],
                                   sc["qdt2m"], sc["beta"], sc["one"], 3,
                                   np.float32(MOMENT_SCALE), 0, os.cpu_count() or 1)
        assert st == 0
        oracle_fold = acc.copy()
        from paper_2008_04397_b200.fields import fold_periodic
        fold_periodic(oracle_fold, geom)
        d = _by_id(p)
        o = np.argsort(r.ids)
        for k in "xyzuvw":
            ref = getattr(r, k)[o].astype(np.float64)
            err = np.abs(d[k] - ref).max() / max(np.abs(ref).max(), 1e-30)
            assert err <= 1e-4, (k, err)
        _assert_moments_close([oracle_fold], [ag], tol=1e-4)


@pytest.mark.parametrize("label", ["single", "double"])
def test_bins_match_flat_many_per_bin(gpu, label):
    """Bins of several 32-particle tiles (ppc 125, as the C3 benchmark):
    four cycles bitwise against the flat path, no overflow, no misplaced."""
    geom, species, prec, bufs, fields = _gem(cells=(32, 16, 16), box=(6.4, 3.2, 3.2), ppc=125,
                                             seed=4, e_amp=1e-4, label=label)
    a = _sim(geom, species, prec, bufs, "bins")
    b = _sim(geom, species, prec, bufs, "flat")
    for cyc in range(4):
        a.run_cycle(fields.E, fields.B)
        b.run_cycle(fields.E, fields.B)
        print(cyc, a.bin_stats())
        assert all(s[1] == 0 and s[2] == 0 and s[3] == 0 for s in a.bin_stats()), a.bin_stats()
        _assert_moments_close(b.moments_host(), a.moments_host(), _tol(label))
    for pa, pb in zip(a.particles, b.particles):
        da, db = _by_id(pa), _by_id(pb)
        for k in da:
            assert np.array_equal(da[k], db[k]), k


@pytest.mark.parametrize("label", ["single", "double"])
def test_bins_hole_cap_fallback_bitwise(gpu, label):
    """Cells so small that most of a bin's 600 particles leave it every cycle
    (more than the mover's 256 listed leavers per bin): the excess stays
    misplaced, is deposited from the late list, and the host rebuilds the
    bins — the particles still bitwise the flat path's, moments within
    tolerance."""
    geom, species, prec, bufs, fields = _gem(cells=(4, 4, 4), box=(0.04, 0.04, 0.04), ppc=600,
                                             seed=5, e_amp=1e-4, label=label)
    a = _sim(geom, species, prec, bufs, "bins")
    b = _sim(geom, species, prec, bufs, "flat")
    misplaced = 0
    for cyc in range(3):
        a.run_cycle(fields.E, fields.B)
        b.run_cycle(fields.E, fields.B)
        misplaced += sum(s[2] for s in a.bin_stats())
        # 600 particles per cell (50x the other tests' per-node sums, in a
        # different order): the north star's 1e-4
        _assert_moments_close(b.moments_host(), a.moments_host(),
                              tol=0 if label == "double" else 1e-4)
    assert misplaced > 0
    assert sum(b_.rebuilds for b_ in a._bins) >= 1
    for pa, pb in zip(a.particles, b.particles):
        da, db = _by_id(pa), _by_id(pb)
        for k in da:
            assert np.array_equal(da[k], db[k]), k


def test_bins64_against_oracle(gpu, oracle):
    """Three cycles of the f64 binned path against the reference arithmetic
    (CPU oracle, double): particles within the north star's 1e-10 of each
    array's max, moments within 1e-10 of the row max + 4 quanta (a half
    quantum rounds either way, tests/test_gpu_fullsize.py)."""
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.fields import MOMENT_SCALE, fold_periodic
    geom, species, prec, bufs, fields = _gem(cells=(32, 16, 8), box=(12.8, 6.4, 3.2), ppc=16,
                                             label="double")
    a = _sim(geom, species, prec, bufs, "bins")
    assert a.binned
    geo_f, geo_i = K.make_geo_arrays(geom, np.float64)
    inv = geom.inv_node_volume(np.float64)
    ref = [b.copy() for b in bufs]
    for cyc in range(3):
        a.run_cycle(fields.E, fields.B)
        acc_gpu = a.moments_host()
        for s, r, ag in zip(species, ref, acc_gpu):
            sc = K.kernel_scalars(s, 0.25, 1.0, np.float64)
            acc = np.zeros((10,) + geom.node_shape, np.int64)
            st = oracle.fused_parallel(r.x, r.y, r.z, r.u, r.v, r.w, r.q_p, 0, r.n, fields.E,
                                       fields.B, acc, inv, geo_f, geo_f, geo_i, sc["dt"],
                                       sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
                                       np.float64(MOMENT_SCALE), 0, os.cpu_count() or 1)
            assert st == 0
            fold_periodic(acc, geom)
            for m in range(10):
                bound = 1e-10 * np.abs(acc[m]).max() + 4
                assert np.abs(ag[m] - acc[m]).max() <= bound, (cyc, m)
    for r, p in zip(ref, a.particles):
        d = _by_id(p)
        o = np.argsort(r.ids)
        for k in "xyzuvw":
            rk = getattr(r, k)[o]
            err = np.abs(d[k] - rk).max() / max(np.abs(rk).max(), 1e-300)
            assert err <= 1e-10, (k, err)


def test_bins64_c2_fullsize_bitwise(gpu):
    """C2 (BASELINE configs[1]: 2D GEM 256 x 128 x 1, ppc 125, four species,
    16.4M f64 particles) on the bins, loaded by the bit-exact device loader:
    two cycles bitwise the flat f64 fast path — every particle and the int64
    lattice — with leavers but no overflow or misplaced particle."""
    import torch
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                           init_gem_device, smooth_e_field)
    from paper_2008_04397_b200.pipeline import DeviceSimulation
    geom = gem_geometry((256, 128, 1))
    species = gem_species(125)
    prec = PrecisionMode.from_label("double")
    f = gem_fields(geom, GemInit(), prec)
    f.E[...] = smooth_e_field(geom, 2e-3, f.E.dtype)
    dev = torch.device("cuda", 0)
    sims = []
    for layout in ("bins", "flat"):
        sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith="fast",
                               sort_period=10, device=dev, layout=layout)
        for sid, p in enumerate(init_gem_device(geom, species, dev, precision=prec)):
            sim.load_species(sid, p)
        sim.set_fields(f.E, f.B)
        sims.append(sim)
    a, b = sims
    assert a.binned and not b.binned
    for _ in range(2):
        a.run_cycle()
        b.run_cycle()
        _assert_moments_close(b.moments_host(), a.moments_host(), 0)
    st = a.bin_stats()
    assert all(s[0] > 0 and s[1] == 0 and s[2] == 0 and s[3] == 0 for s in st), st
    for pa, pb in zip(a.particles, b.particles):
        da, db = _by_id(pa), _by_id(pb)
        for k in da:
            assert np.array_equal(da[k], db[k]), k


@pytest.mark.parametrize("label", ["single", "double"])
def test_bins_two_streams_match_one(gpu, label, monkeypatch):
    """BP_BIN_STREAMS=2 (species on two streams, each with its own leaver
    list): the particles bitwise those of the one-stream cycle, the moments
    within the f32 tolerance (f64: bitwise)."""
    geom, species, prec, bufs, fields = _gem(label=label)
    a = _sim(geom, species, prec, bufs, "bins")
    b = _sim(geom, species, prec, bufs, "bins")
    for cyc in range(4):
        monkeypatch.setenv("BP_BIN_STREAMS", "2")
        a.run_cycle(fields.E, fields.B)
        monkeypatch.delenv("BP_BIN_STREAMS")
        b.run_cycle(fields.E, fields.B)
        _assert_moments_close(b.moments_host(), a.moments_host(), _tol(label))
    assert a._side_lists is not None and len(a._side_lists) == 2
    for pa, pb in zip(a.particles, b.particles):
        da, db = _by_id(pa), _by_id(pb)
        for k in da:
            assert np.array_equal(da[k], db[k]), k


@pytest.mark.parametrize("layout,label", [("bins", "single"), ("flat", "single"),
                                          ("bins", "double")])
def test_streamed_moments_equal_the_cycle_end_copy(gpu, layout, label, monkeypatch):
    """run_cycle(stream_moments=True) folds each species' grid right after its
    kernels and copies it to pinned host memory while the next species runs.
    The host copies must be the final device grids bitwise (no copy may race
    the fold or a later kernel), cycle after cycle, also with the species on
    two streams and with overflowing bins (zero headroom); and they must
    match the default path (fold after the cycle, one copy per species):
    bitwise where the arithmetic is order-independent (flat f32, f64 bins),
    within the f32 tolerance on the f32 bins, whose per-bin sums follow the
    migration's atomic order."""
    geom, species, prec, bufs, fields = _gem(label=label)
    for streams in ("0", "2"):
        monkeypatch.setenv("BP_BIN_STREAMS", streams)
        monkeypatch.setenv("BP_SPECIES_STREAMS", streams)
        kw = {"bin_slack": (0.0, 0)} if layout == "bins" else {}
        a = _sim(geom, species, prec, bufs, layout, **kw)
        b = _sim(geom, species, prec, bufs, layout, **kw)
        for cyc in range(4):
            a.run_cycle(fields.E, fields.B)
            b.run_cycle(fields.E, fields.B, stream_moments=True)
            ma = [m.copy() for m in a.moments_host(reuse=True)]
            mb = [m.copy() for m in b.moments_host(reuse=True)]
            for x, y in zip(mb, b.acc):
                assert np.array_equal(x, y.cpu().numpy()), (streams, cyc)
            exact = layout == "flat" or label == "double"
            _assert_moments_close(ma, mb, 0 if exact else _tol(label))


@pytest.mark.parametrize("label", ["single", "double"])
def test_bins_report_failing_particles(gpu, label):
    """A particle that would leave the box (kernels.py:618-621) is not stored
    and the cycle raises, on the bins as on the flat layout (the binned mover
    reports each lane's worst status once, at the end of the kernel)."""
    from paper_2008_04397_b200.errors import IntegrityError
    geom, species, prec, bufs, fields = _gem(label=label)
    for layout in ("bins", "flat"):
        bad = [b.copy() for b in bufs]
        bad[0].u[7] = bad[0].u.dtype.type(1e3)  # 250 box lengths in one step
        sim = _sim(geom, species, prec, bad, layout)
        assert sim.binned == (layout == "bins")
        with pytest.raises(IntegrityError):
            sim.run_cycle(fields.E, fields.B)
