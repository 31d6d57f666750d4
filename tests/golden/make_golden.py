"""Generate golden fixtures from the REFERENCE package (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (committed, small):
  kernels_<mode>.npz  inputs + outputs of the reference numba kernels
                      fused_span / push_span / deposit_span / gather_span
                      (kernels.py:82,310,385,458) on an 8^3 periodic/
                      reflecting/periodic box, for mode in double/single/mixed,
                      at three velocity scales (the largest triggers
                      ERR_MIDPOINT / ERR_RUNAWAY paths) plus face-pinned
                      particles.
  sort.npz            cell keys + stable order of particles.sort_by_cell
                      (particles.py:157-167, geometry.py:152-159).
  c1_<mode>.npz       N-cycle replay of the reference pipeline on config C1
                      (2D GEM 64x32x1, ppc 16 x 4 species):
                      E/B at the start of every cycle (the host solver's
                      output, replayed as input), the energy ledger after
                      every cycle, per-species folded int64 moments of the
                      last cycle, SHA-256 of every final particle array and a
                      strided sample of final particle values.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

import batchpic
from batchpic import kernels as K
from batchpic.config import InitConfig, PrecisionMode, SimulationDeck, SpeciesParams
from batchpic.diagnostics import energy_ledger
from batchpic.fields import MOMENT_SCALE
from batchpic.geometry import GridGeometry
from batchpic.maxwell import plasma_susceptibility
from batchpic.particles import sort_by_cell, ParticleBuffer, write_particles
from batchpic.pipeline import make_state, run_cycle

OUT = os.path.dirname(os.path.abspath(__file__))
MODES = {"double": (np.float64, np.float64), "single": (np.float32, np.float32),
         "mixed": (np.float32, np.float64)}

B0 = 0.0097
VTH_E = 0.02240119044455748
VTH_I = 0.006261323076368657
N0 = 0.07957747154594767


def kernel_cases(mode):
    pd, fd = MODES[mode]
    geom = GridGeometry.from_box((8, 8, 8), (6.4, 6.4, 6.4),
                                 bc=("periodic", "reflecting", "periodic"))
    sp = SpeciesParams(0, -1.0, 0.1, 1, mover_iters=3)
    dt = 0.2
    rec = {"nx": 8, "L": 6.4, "qom": sp.qom, "dt": dt, "n_iters": 3}
    n = 3000
    for ci, vscale in enumerate((0.3, 4.0, 40.0)):
        rng = np.random.default_rng(100 + ci)
        x = (rng.random(n) * geom.Lx).astype(pd)
        y = (rng.random(n) * geom.Ly).astype(pd)
        z = (rng.random(n) * geom.Lz).astype(pd)
        # face-pinned particles (upper faces are legal positions)
        x[:20] = pd(geom.Lx); y[20:40] = pd(geom.Ly); y[40:60] = 0.0
        z[60:80] = pd(geom.Lz); x[80:100] = 0.0
        u = (rng.standard_normal(n) * vscale).astype(pd)
        v = (rng.standard_normal(n) * vscale).astype(pd)
        w = (rng.standard_normal(n) * vscale).astype(pd)
        q = (rng.random(n) * 1e-2).astype(pd)
        E = (rng.standard_normal((3, 9, 9, 9)) * 0.05).astype(fd)
        B = (rng.standard_normal((3, 9, 9, 9)) * 0.8).astype(fd)
        geo_f, geo_i = K.make_geo_arrays(geom, pd)
        geo_g, _ = K.make_geo_arrays(geom, fd)
        sc = K.kernel_scalars(sp, dt, 1.0, pd)
        inv = geom.inv_node_volume(fd)
        mixed = 1 if pd != fd else 0
        start, count = 7, n - 13  # non-trivial span
        pre = f"c{ci}_"
        for nm, a in zip("xyzuvwq", (x, y, z, u, v, w, q)):
            rec[pre + "in_" + nm] = a
        rec[pre + "E"] = E
        rec[pre + "B"] = B
        rec[pre + "span"] = np.array([start, count])
        # fused
        a = [t.copy() for t in (x, y, z, u, v, w, q)]
        acc = np.zeros((10, 9, 9, 9), np.int64)
        st = K.fused_span(*a, start, count, E, B, acc, inv, geo_f, geo_g, geo_i,
                          sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"],
                          3, fd(MOMENT_SCALE), mixed, np.empty(6, pd))
        rec[pre + "fused_status"] = np.array(st)
        rec[pre + "fused_acc"] = acc
        for nm, t in zip("xyzuvw", a):
            rec[pre + "fused_" + nm] = t
        # push, with and without boundaries
        for bc in (0, 1):
            a = [t.copy() for t in (x, y, z, u, v, w)]
            st = K.push_span(*a, start, count, E, B, geo_f, geo_g, geo_i,
                             sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"],
                             sc["one"], 3, bc, mixed, np.empty(6, pd))
            rec[pre + f"push{bc}_status"] = np.array(st)
            for nm, t in zip("xyzuvw", a):
                rec[pre + f"push{bc}_" + nm] = t
        # deposit at the input state (all inputs are in-domain)
        acc = np.zeros((10, 9, 9, 9), np.int64)
        K.deposit_span(x, y, z, u, v, w, q, start, count, acc,
                       geom.inv_node_volume(fd), geo_g, geo_i, fd(1.0),
                       fd(MOMENT_SCALE))
        rec[pre + "deposit_acc"] = acc
        # gather
        out = np.zeros((count, 6), pd)
        K.gather_span(x, y, z, start, count, E, B, geo_g, geo_i, pd(1.0), out)
        rec[pre + "gather_out"] = out
    np.savez_compressed(os.path.join(OUT, f"kernels_{mode}.npz"), **rec)


def sort_case():
    geom = GridGeometry.from_box((4, 4, 4), (4.0, 4.0, 4.0))
    rng = np.random.default_rng(7)
    n = 5000
    buf = ParticleBuffer.empty(n)
    buf.x[:] = rng.random(n) * geom.Lx
    buf.y[:] = rng.random(n) * geom.Ly
    buf.z[:] = rng.random(n) * geom.Lz
    buf.x[:10] = geom.Lx  # upper faces clamp into the last cell
    buf.u[:] = rng.standard_normal(n)
    rec = {"x": buf.x.copy(), "y": buf.y.copy(), "z": buf.z.copy()}
    rec["keys"] = geom.cell_index_of(buf.x, buf.y, buf.z)
    sort_by_cell(buf, geom)
    rec["ids_after"] = buf.ids.copy()
    np.savez_compressed(os.path.join(OUT, "sort.npz"), **rec)


def checkpoint_case():
    """Bytes of the reference's BPIC v1 checkpoint (particles.py:244-274)."""
    import tempfile
    rec = {}
    rng = np.random.default_rng(12)
    for dt in (np.float64, np.float32):
        buf = ParticleBuffer.empty(37, dtype=dt)
        for nm in ("x", "y", "z", "u", "v", "w", "q_p"):
            getattr(buf, nm)[:] = rng.random(37).astype(dt)
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, "p.bin")
            write_particles(buf, path)
            raw = open(path, "rb").read()
        tag = np.dtype(dt).name
        rec[f"bytes_{tag}"] = np.frombuffer(raw, np.uint8)
        for nm in ("x", "y", "z", "u", "v", "w", "q_p"):
            rec[f"{tag}_{nm}"] = getattr(buf, nm)
    np.savez_compressed(os.path.join(OUT, "checkpoint.npz"), **rec)


def c1_deck(mode, cycles):
    pd = {"double": ("double", "double"), "single": ("single", "single"),
          "mixed": ("single", "double")}[mode]
    geom = GridGeometry.from_box((64, 32, 1), (25.6, 12.8, 0.4),
                                 bc=("periodic", "reflecting", "periodic"))
    me = 1.0 / 64.0
    species = (
        SpeciesParams(0, -1.0, me, 16, vth=(VTH_E,) * 3, name="sheet_electrons"),
        SpeciesParams(1, 1.0, 1.0, 16, vth=(VTH_I,) * 3, name="sheet_ions"),
        SpeciesParams(2, -1.0, me, 16, vth=(VTH_E,) * 3, name="background_electrons"),
        SpeciesParams(3, 1.0, 1.0, 16, vth=(VTH_I,) * 3, name="background_ions"),
    )
    return SimulationDeck(
        geom=geom, species=species, dt=0.25, n_cycles=cycles, c=1.0, theta=0.5,
        susceptibility=True, clean_period=0, batches=4, groups=1, workers=1,
        sort_period=5, precision=PrecisionMode(*pd),
        init=InitConfig(kind="gem", seed=20250809, n0=N0, b0=B0,
                        sheet_thickness=0.5, perturbation=0.1,
                        background_fraction=0.2))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def c1_case(mode, cycles=10, stride=64):
    deck = c1_deck(mode, cycles)
    rec = {"cycles": cycles, "mode": mode}
    with make_state(deck) as state:
        for s, buf in enumerate(state.buffers):
            for nm in ("x", "y", "z", "u", "v", "w", "q_p"):
                rec[f"init_sha_{s}_{nm}"] = _sha(getattr(buf, nm))
        Es, Bs, led = [], [], []
        for c in range(cycles):
            Es.append(state.fields.E.copy())
            Bs.append(state.fields.B.copy())
            rep = run_cycle(state, c)
            assert rep.sorted_this_cycle == ((c + 1) % deck.sort_period == 0)
            L = energy_ledger(c + 1, state.fields, state.buffers, deck.species,
                              state.geom)
            led.append([L.field_energy, *L.kinetic_energy])
        rec["E"] = np.stack(Es)
        rec["B"] = np.stack(Bs)
        rec["E_final"] = state.fields.E.copy()
        rec["B_final"] = state.fields.B.copy()
        rec["ledger"] = np.array(led)
        # phase-4/5 consumer of the moments: the susceptibility the host solve
        # used for the last cycle (maxwell.py:163-179)
        rec["chi_last"] = plasma_susceptibility(
            [state.moments[s] for s in sorted(state.moments)], deck.species, deck.dt,
            deck.theta, state.geom)
        rec["theta"] = deck.theta
        for s, buf in enumerate(state.buffers):
            rec[f"acc_{s}"] = state.moments[s].acc.copy()  # folded (phase 4)
            for nm in ("x", "y", "z", "u", "v", "w", "q_p", "ids"):
                a = getattr(buf, nm)
                rec[f"final_sha_{s}_{nm}"] = _sha(a)
                rec[f"final_{s}_{nm}"] = a[::stride].copy()
    np.savez_compressed(os.path.join(OUT, f"c1_{mode}.npz"), **rec)


def main():
    assert os.path.isdir("/root/reference"), "needs the reference package"
    print("batchpic from", batchpic.__file__, file=sys.stderr)
    for mode in MODES:
        kernel_cases(mode)
    sort_case()
    checkpoint_case()
    for mode in MODES:
        c1_case(mode)
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
