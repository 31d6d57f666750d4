"""N-cycle parity on config C1 (2D GEM 64x32x1, ppc 16 x 4 species): the
reference pipeline's own field history (tests/golden/c1_<mode>.npz) is
replayed through the device-resident driver for 10 cycles, with the on-device
cell sort after cycles 5 and 10.  Parity arithmetic must reproduce the final
particles (SHA-256 of every array, sorted order included), the last cycle's
folded moments and the energy ledger bit for bit; fast arithmetic must stay
within the north-star tolerances (1e-10 f64, 1e-4 f32, relative to the array
max) and match the energy drift."""

import hashlib

import numpy as np
import pytest

from conftest import MODES, golden

pytestmark = pytest.mark.gpu


def _run(mode, arith, layout="auto"):
    import torch
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    from paper_2008_04397_b200.pipeline import DeviceSimulation, field_energy
    g = golden(f"c1_{mode}.npz")
    geom = gem_geometry((64, 32, 1), (25.6, 12.8, 0.4))
    prec = PrecisionMode.from_label(mode)
    species = gem_species(16)
    bufs, _ = init_gem_host(geom, species, GemInit(), prec)
    sim = DeviceSimulation(geom, species, dt=0.25, precision=prec, arith=arith,
                           sort_period=5, batches=4, layout=layout)
    sim.load_host_buffers(bufs)
    ledger = []
    for c in range(int(g["cycles"])):
        t = sim.run_cycle(g["E"][c], g["B"][c])
        # the binned layout is cell-sorted every cycle and never sorts
        assert t.sorted_this_cycle == ((c + 1) % 5 == 0 and not sim.binned)
        Ef = g["E"][c + 1] if c + 1 < int(g["cycles"]) else g["E_final"]
        Bf = g["B"][c + 1] if c + 1 < int(g["cycles"]) else g["B_final"]
        ledger.append([field_energy(Ef, Bf, geom)] + sim.kinetic_energy())
    parts = [p.to_host() for p in sim.particles]
    sim.chi = sim.susceptibility(float(g["theta"])).cpu().numpy()
    sim.total = sim.total_moments().cpu().numpy()
    return g, parts, sim.moments_host(), np.array(ledger), sim


@pytest.mark.parametrize("mode", list(MODES))
def test_c1_replay_parity_bitwise(gpu, mode):
    g, parts, accs, ledger, sim = _run(mode, "parity")
    for s, buf in enumerate(parts):
        for nm in ("x", "y", "z", "u", "v", "w", "q_p", "ids"):
            sha = hashlib.sha256(np.ascontiguousarray(getattr(buf, nm)).tobytes()).hexdigest()
            assert sha == str(g[f"final_sha_{s}_{nm}"]), f"species {s} {nm}"
        assert np.array_equal(accs[s], g[f"acc_{s}"]), f"moments of species {s}"
    # kinetic terms are f64 sums in a different order than numpy's: compare to
    # a few ulps; the field term is the same formula on the same arrays
    assert np.allclose(ledger, g["ledger"], rtol=1e-13, atol=0)
    # device phase 4: exact species total and the host solve's susceptibility
    assert np.array_equal(sim.total, sum(g[f"acc_{s}"] for s in range(4)))
    assert np.array_equal(sim.chi, g["chi_last"])


@pytest.mark.parametrize("layout", ["flat", "bins"])
@pytest.mark.parametrize("mode", list(MODES))
def test_c1_replay_fast_within_tolerance(gpu, mode, layout):
    if layout == "bins" and mode == "double":
        pytest.skip("the binned layout holds f32 particles")
    g, parts, accs, ledger, sim = _run(mode, "fast", layout)
    assert sim.binned == (layout == "bins")
    rtol = 1e-10 if mode == "double" else 1e-4
    # chaotic orbits amplify round-off over 10 cycles; SURVEY.md §8c measured a
    # 1-ulp perturbation growing to 1.6e-14 (f64) / 2.7e-6 (f32) of the max
    for s, buf in enumerate(parts):
        order = np.argsort(buf.ids)
        assert np.array_equal(buf.ids[order], np.arange(buf.n))
        for nm, per in zip("xyzuvw", (25.6, None, 0.4, None, None, None)):
            ref = g[f"final_{s}_{nm}"]
            ref_ids = g[f"final_{s}_ids"]
            got = getattr(buf, nm)[order][ref_ids]
            d = np.abs(got.astype(np.float64) - ref)
            if per is not None:
                d = np.minimum(d, np.abs(per - d))
            assert d.max() <= rtol * np.abs(ref).max(), (s, nm, d.max() / np.abs(ref).max())
        ref_acc = g[f"acc_{s}"] * 2.0 ** -43
        got_acc = accs[s] * 2.0 ** -43
        for m in range(10):
            err = np.abs(got_acc[m] - ref_acc[m]).max() / max(np.abs(ref_acc[m]).max(), 1e-300)
            assert err <= rtol, (s, m, err)
    # total energy drift series matches the reference
    tot, tot_ref = ledger.sum(axis=1), g["ledger"].sum(axis=1)
    drift, drift_ref = tot / tot[0] - 1.0, tot_ref / tot_ref[0] - 1.0
    assert np.abs(drift - drift_ref).max() <= max(rtol, 1e-12) * 10


@pytest.mark.parametrize("arith", ["parity", "fast"])
def test_sorting_toggle_changes_nothing_bitwise(gpu, arith):
    """The reference's C9 / test_pipeline.py:146-152 on the device path: with
    and without the periodic on-device sort, particles (matched by id) and
    moments are bit-identical after 10 cycles (fast f32 arithmetic: the
    particles bitwise, the moments — per-tile f32 partial sums, bp_f32.cu —
    within the f32 tolerance)."""
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    from paper_2008_04397_b200.pipeline import DeviceSimulation
    g = golden("c1_single.npz")
    geom = gem_geometry((64, 32, 1), (25.6, 12.8, 0.4))
    prec = PrecisionMode.from_label("single")
    out = []
    for sp in (0, 3):
        bufs, _ = init_gem_host(geom, gem_species(16), GemInit(), prec)
        sim = DeviceSimulation(geom, gem_species(16), dt=0.25, precision=prec, arith=arith,
                               sort_period=sp)
        sim.load_host_buffers(bufs)
        for c in range(int(g["cycles"])):
            sim.run_cycle(g["E"][c], g["B"][c])
        out.append(([p.to_host() for p in sim.particles], sim.moments_host()))
    (pa, ma), (pb, mb) = out
    for x, y in zip(ma, mb):
        if arith == "parity":
            assert np.array_equal(x, y)
        else:
            for r in range(x.shape[0]):
                ref = x[r].astype(np.float64)
                err = np.abs(y[r] - ref).max() / max(np.abs(ref).max(), 1.0)
                assert err <= 1e-5, (r, err)
    for a, b in zip(pa, pb):
        oa, ob = np.argsort(a.ids), np.argsort(b.ids)
        for nm in ("x", "y", "z", "u", "v", "w", "q_p", "ids"):
            assert np.array_equal(getattr(a, nm)[oa], getattr(b, nm)[ob]), nm
