"""The bit-exact device loader (csrc/bp_init.cu, particles.init_maxwellian_device)
against the reference loader (pkg/src/batchpic/particles.py:177-241, gem.py:64-115).

* C1 (2D GEM 64x32x1, ppc 16, 4 species, all three precisions): the
  device-loaded buffers hash to the SHA-256 the reference itself wrote into
  tests/golden/c1_<mode>.npz (init_sha_*), array by array;
* C2 size (256x128x1, ppc 125: 4.1M particles per species, ~1200 ziggurat
  tail-strip normals each): equal to the host restatement init_gem_host
  (numpy, itself pinned to the reference above), whole species and a rank's
  cell shard;
* the uniform loader (init_uniform_device) against particles.init_maxwellian
  with the uniform density of make_state (pipeline.py:140-151).
"""

import hashlib

import numpy as np
import pytest

from conftest import MODES, golden

pytestmark = pytest.mark.gpu

NAMES = ("x", "y", "z", "u", "v", "w", "q_p")


def _host(p):
    h = p.to_host()
    return {nm: getattr(h, nm) for nm in NAMES + ("ids",)}


@pytest.mark.parametrize("mode", list(MODES))
def test_c1_device_init_is_bitwise_the_reference(gpu, mode):
    import torch
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_device
    g = golden(f"c1_{mode}.npz")
    geom = gem_geometry((64, 32, 1), (25.6, 12.8, 0.4))
    parts = init_gem_device(geom, gem_species(16), torch.device("cuda"), GemInit(),
                            PrecisionMode.from_label(mode))
    for s, p in enumerate(parts):
        h = _host(p)
        for nm in NAMES:
            sha = hashlib.sha256(np.ascontiguousarray(h[nm]).tobytes()).hexdigest()
            assert sha == str(g[f"init_sha_{s}_{nm}"]), (s, nm)
        assert np.array_equal(h["ids"], np.arange(p.n))


@pytest.mark.parametrize("label", ["single", "double"])
def test_c2_device_init_equals_host_loader(gpu, label):
    import torch
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import GemInit, gem_geometry, gem_species, init_gem_device
    from paper_2008_04397_b200.gem import init_gem_host
    geom = gem_geometry((256, 128, 1))
    species = gem_species(125)
    prec = PrecisionMode.from_label(label)
    bufs, _ = init_gem_host(geom, species, GemInit(), prec)
    dev = init_gem_device(geom, species, torch.device("cuda"), GemInit(), prec)
    for b, p in zip(bufs, dev):
        h = _host(p)
        for nm in NAMES + ("ids",):
            assert np.array_equal(h[nm], getattr(b, nm)), (b.species_id, nm)
    # a rank's shard: cells [c0, c0 + nc) are the same slice of the species
    c0, nc = 5000, 9001
    shard = init_gem_device(geom, species, torch.device("cuda"), GemInit(), prec,
                            cells=(c0, nc))
    sl = slice(c0 * 125, (c0 + nc) * 125)
    for b, p in zip(bufs, shard):
        h = _host(p)
        for nm in NAMES + ("ids",):
            assert np.array_equal(h[nm], getattr(b, nm)[sl]), (b.species_id, nm)


@pytest.mark.parametrize("label", ["single", "mixed", "double"])
def test_uniform_device_init_equals_host_loader(gpu, label):
    import torch
    from paper_2008_04397_b200.config import PrecisionMode, SpeciesParams
    from paper_2008_04397_b200.gem import gem_geometry, init_uniform_device
    from paper_2008_04397_b200.particles import init_maxwellian
    geom = gem_geometry((32, 16, 16), (6.4, 3.2, 3.2))
    sp = SpeciesParams(2, -1.0, 1.0 / 64.0, 40, vth=(0.02, 0.03, 0.04), drift=(0.0, 0.01, 0.0))
    prec = PrecisionMode.from_label(label)
    n0 = 0.7

    def uniform(x, y, z):
        return np.full_like(np.asarray(y, dtype=np.float64), n0)

    ref = init_maxwellian(sp, geom, density_fn=uniform, seed=11, precision=prec)
    got = _host(init_uniform_device(geom, (sp,), torch.device("cuda"), n0=n0, precision=prec,
                                    seed=11)[0])
    for nm in NAMES + ("ids",):
        assert np.array_equal(got[nm], getattr(ref, nm)), nm
