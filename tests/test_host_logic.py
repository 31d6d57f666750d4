"""Host-side pieces of the path that need no GPU: the bitwise GEM loader,
batching, boundary map, geometry helpers, the energy ledger formula, and
that the product package refuses to run without its CUDA library."""

import hashlib

import numpy as np
import pytest

from conftest import MODES, golden


@pytest.mark.parametrize("mode", list(MODES))
def test_gem_host_init_is_bitwise_the_reference(mode):
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_host
    g = golden(f"c1_{mode}.npz")
    geom = gem_geometry((64, 32, 1), (25.6, 12.8, 0.4))
    bufs, f = init_gem_host(geom, gem_species(16), GemInit(), PrecisionMode.from_label(mode))
    for s, b in enumerate(bufs):
        for nm in ("x", "y", "z", "u", "v", "w", "q_p"):
            sha = hashlib.sha256(np.ascontiguousarray(getattr(b, nm)).tobytes()).hexdigest()
            assert sha == str(g[f"init_sha_{s}_{nm}"]), (s, nm)
    assert np.array_equal(f.E, g["E"][0]) and np.array_equal(f.B, g["B"][0])


def test_partition_batches_reference_rule():
    from paper_2008_04397_b200.particles import partition_batches
    plan = partition_batches(10, 4)
    assert plan.spans == ((0, 3), (3, 3), (6, 2), (8, 2))
    assert partition_batches(2, 4).spans[-1] == (2, 0)


def test_apply_boundaries_wrap_mirror_and_runaway():
    from paper_2008_04397_b200.errors import IntegrityError
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200.particles import ParticleBuffer, apply_boundaries
    geom = GridGeometry.from_box((4, 4, 4), (4.0, 4.0, 4.0),
                                 bc=("periodic", "reflecting", "periodic"))
    buf = ParticleBuffer.empty(3)
    buf.x[:] = [-0.5, 4.0, 4.5]
    buf.y[:] = [-0.25, 4.5, 2.0]
    buf.z[:] = 1.0
    buf.v[:] = [1.0, 2.0, 3.0]
    apply_boundaries(buf, geom)
    assert list(buf.x) == [3.5, 0.0, 0.5]
    assert list(buf.y) == [0.25, 3.5, 2.0] and list(buf.v) == [-1.0, -2.0, 3.0]
    snap = buf.copy()
    apply_boundaries(buf, geom)  # idempotent
    assert np.array_equal(buf.x, snap.x) and np.array_equal(buf.y, snap.y)
    buf.x[0] = 9.0
    with pytest.raises(IntegrityError):
        apply_boundaries(buf, geom)


def test_inv_node_volume_walls_and_weights():
    from paper_2008_04397_b200.geometry import GridGeometry
    geom = GridGeometry.from_box((4, 4, 4), (2.0, 2.0, 2.0),
                                 bc=("periodic", "reflecting", "periodic"))
    inv = geom.inv_node_volume()
    assert inv[1, 1, 1] == 8.0 and inv[1, 0, 1] == 16.0 and inv[0, 4, 0] == 16.0
    assert (geom.node_weights().sum() * geom.cell_volume) == pytest.approx(8.0)


def test_field_energy_matches_reference_formula():
    from paper_2008_04397_b200.gem import GemInit, gem_fields, gem_geometry
    from paper_2008_04397_b200.pipeline import field_energy
    g = golden("c1_double.npz")
    geom = gem_geometry((64, 32, 1), (25.6, 12.8, 0.4))
    # ledger[c][0] is the field energy after cycle c+1 (the fields of cycle c+2)
    assert field_energy(g["E"][1], g["B"][1], geom) == g["ledger"][0][0]


def test_product_path_refuses_without_library(tmp_path, monkeypatch):
    from paper_2008_04397_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(_lib.BackendError):
        _lib.load()


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_checkpoint_v1_is_the_reference_format(tmp_path, dtype):
    """write_particles(version=1) reproduces the reference's file byte for
    byte; read_particles reads the reference's file (q_p zero, fresh ids)."""
    from paper_2008_04397_b200.particles import ParticleBuffer, read_particles, write_particles
    g = golden("checkpoint.npz")
    n = g[f"{dtype}_x"].shape[0]
    buf = ParticleBuffer.empty(n, dtype=np.dtype(dtype).type)
    for nm in ("x", "y", "z", "u", "v", "w", "q_p"):
        getattr(buf, nm)[:] = g[f"{dtype}_{nm}"]
    path = tmp_path / "p.bin"
    write_particles(buf, path)
    assert path.read_bytes() == g[f"bytes_{dtype}"].tobytes()
    ref = tmp_path / "ref.bin"
    ref.write_bytes(g[f"bytes_{dtype}"].tobytes())
    back = read_particles(ref)
    assert back.dtype == np.dtype(dtype)
    for nm in ("x", "y", "z", "u", "v", "w"):
        assert np.array_equal(getattr(back, nm), getattr(buf, nm))
    assert (back.q_p == 0).all() and np.array_equal(back.ids, np.arange(n))


def test_checkpoint_v2_keeps_charge_and_ids(tmp_path):
    from paper_2008_04397_b200.particles import ParticleBuffer, read_particles, write_particles
    rng = np.random.default_rng(3)
    buf = ParticleBuffer.empty(100, species_id=2, dtype=np.float32)
    for nm in ("x", "y", "z", "u", "v", "w", "q_p"):
        getattr(buf, nm)[:] = rng.random(100).astype(np.float32)
    buf.ids[:] = rng.permutation(100)
    write_particles(buf, tmp_path / "p2.bin", version=2)
    back = read_particles(tmp_path / "p2.bin")
    assert back.species_id == 2
    for nm in ("x", "y", "z", "u", "v", "w", "q_p", "ids"):
        assert np.array_equal(getattr(back, nm), getattr(buf, nm)), nm


def test_binned_layout_estimate_and_auto_rule():
    """bins.layout_bytes, the memory rule behind DeviceSimulation's
    layout="auto": C3 f32 (the headline, ~43 GB) and the C5 sweep's f32 deck
    at 1e9 particles (~103 GB) fit a 180 GB B200 with its two buffer sets,
    C5 f64 at 1e9 (~185 GB) does not (it stays flat), and the estimate
    splits over ranks."""
    from paper_2008_04397_b200.bins import layout_bytes
    dev = 0.92 * 179.5e9
    c3 = layout_bytes(128 * 64 * 64, [125] * 4, (1.0, 64), 4)
    assert 40e9 < c3 < 46e9 and c3 < dev
    ppc = round(1e9 / (128 * 64 * 64))
    c5_f32 = layout_bytes(128 * 64 * 64, [ppc], (0.25, 16), 4)
    c5_f64 = layout_bytes(128 * 64 * 64, [ppc], (0.25, 16), 8)
    assert c5_f32 < dev < c5_f64
    assert abs(layout_bytes(128 * 64 * 64, [ppc], (0.25, 16), 8, world=8) - c5_f64 / 8) < 1.0
    # a slack minimum dominates sparse cells: ppc 12 with min 64 -> 76 slots
    assert layout_bytes(10, [12], (1.0, 64), 4) == 2 * 1.03 * 10 * 76 * 40
