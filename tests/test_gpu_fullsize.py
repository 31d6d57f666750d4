"""Full-size (C3) checks of the headline path: one species of the 3D GEM
workload (128x64x64 cells, ppc 125: 65.5M electrons, f32) against the oracle
on every host core — bitwise in parity arithmetic; in fast arithmetic within
the north star's 1e-4 relative to each array's max, plus the conservation
identities the deposit satisfies at any size (sum over nodes of moment /
invvol equals the particle sum of q, q v and q v v after the push)."""

import os

import numpy as np
import pytest

from test_gpu_kernels import _assert_close

pytestmark = pytest.mark.gpu

SCALE = 2.0 ** 43


def _smooth_e(geom, amp):
    """A smooth non-zero E (the GEM start has E = 0) so the E gather counts."""
    X, Y, Z = np.meshgrid(geom.node_coords(0), geom.node_coords(1), geom.node_coords(2),
                          indexing="ij")
    kx, ky, kz = (2 * np.pi / L for L in geom.lengths)
    return amp * np.stack([np.sin(kx * X + 0.3) * np.cos(ky * Y),
                           np.cos(kz * Z) * np.sin(kx * X),
                           np.sin(ky * Y + 0.7) * np.cos(kz * Z - 0.2)])


def test_c3_species_fast_within_tolerance_and_conserving(gpu, oracle):
    import torch
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                           init_gem_device)
    geom = gem_geometry((128, 64, 64))
    species = gem_species(125)
    sp = species[0]
    prec = PrecisionMode.from_label("single")
    dev = torch.device("cuda")
    p = init_gem_device(geom, species, dev, precision=prec)[0]  # sheet electrons
    n = p.n
    assert n == 128 * 64 * 64 * 125
    f = gem_fields(geom, GemInit(), prec)
    E = _smooth_e(geom, 1e-3).astype(np.float32)
    B = np.ascontiguousarray(f.B, np.float32)
    inv = geom.inv_node_volume(np.float32)
    geo_f, geo_i = K.make_geo_arrays(geom, np.float32)
    geo_g, _ = K.make_geo_arrays(geom, np.float32)
    sc = K.kernel_scalars(sp, 0.25, 1.0, np.float32)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"],
            3, np.float32(SCALE), 0)
    ref = [a.cpu().numpy() for a in p.arrays()]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    st_ref = oracle.fused_parallel(*ref, 0, n, E, B, acc_ref, inv, *tail, os.cpu_count() or 1)

    d = list(p.arrays())
    dE, dB, dinv = (torch.from_numpy(a).to(dev) for a in (E, B, inv))
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device=dev)
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith="fast")
    assert st == st_ref == 0

    got = [t.cpu().numpy() for t in d[:6]]
    # y is the reflecting axis.  A particle whose commit lands within rounding
    # of the wall is mirrored by one arithmetic and not by the other (the
    # reference decides on f64 intermediates, the fast kernel on f32): the
    # positions agree (both at the wall) and the velocities agree up to the
    # mirror.  Count those (a handful in 65.5M) and compare the rest exactly.
    lo, hi = np.float32(geom.origin[1]), np.float32(geom.origin[1] + geom.Ly)
    ulp = np.spacing(hi)
    at_wall = (np.abs(got[1] - hi) <= 4 * ulp) | (np.abs(got[1] - lo) <= 4 * ulp)
    flip = at_wall & (np.sign(got[4]) == -np.sign(ref[4])) & (ref[4] != 0)
    assert flip.sum() <= 1e-6 * n, int(flip.sum())
    got[4] = np.where(flip, -got[4], got[4])
    periods = (geom.Lx, None, geom.Lz, None, None, None)
    for name, r, t, per in zip("xyzuvw", ref, got, periods):
        _assert_close(name, r, t, 1e-4, per)
    got = dacc.cpu().numpy()
    for m in range(10):
        _assert_close(f"moment {m}", acc_ref[m] * 2.0 ** -43, got[m] * 2.0 ** -43, 1e-4)

    # conservation on the device result: node sums of moment / invvol
    w = 1.0 / dinv.double()
    node = [(dacc[m].double() * w).sum().item() * 2.0 ** -43 for m in range(10)]
    q = d[6].double()
    u, v, ww = (t.double() for t in d[3:6])
    one = torch.ones_like(u)
    mom = [one, u, v, ww, u * u, u * v, u * ww, v * v, v * ww, ww * ww]
    for m in range(10):
        part = (q * mom[m]).sum().item()
        # f32 contributions summed per tile, rounded once onto the lattice:
        # well inside 1e-5 of the sum of |contributions|
        scale = (q.abs() * mom[m].abs()).sum().item()
        assert abs(node[m] - part) <= 1e-5 * scale, (m, node[m], part, scale)


def test_c3_species_parity_bitwise(gpu, oracle):
    """The bitwise path at full size: 65.5M electrons through the parity
    kernels equal the oracle (the reference arithmetic) bit for bit."""
    import torch
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                           init_gem_device)
    geom = gem_geometry((128, 64, 64))
    species = gem_species(125)
    prec = PrecisionMode.from_label("single")
    dev = torch.device("cuda")
    p = init_gem_device(geom, species, dev, precision=prec)[0]
    n = p.n
    f = gem_fields(geom, GemInit(), prec)
    E = _smooth_e(geom, 1e-3).astype(np.float32)
    B = np.ascontiguousarray(f.B, np.float32)
    inv = geom.inv_node_volume(np.float32)
    geo_f, geo_i = K.make_geo_arrays(geom, np.float32)
    geo_g, _ = K.make_geo_arrays(geom, np.float32)
    sc = K.kernel_scalars(species[0], 0.25, 1.0, np.float32)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"],
            3, np.float32(SCALE), 0)
    ref = [a.cpu().numpy() for a in p.arrays()]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    st_ref = oracle.fused_parallel(*ref, 0, n, E, B, acc_ref, inv, *tail, os.cpu_count() or 1)
    d = list(p.arrays())
    dE, dB, dinv = (torch.from_numpy(a).to(dev) for a in (E, B, inv))
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device=dev)
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith="parity")
    assert st == st_ref
    for name, r, t in zip("xyzuvw", ref, d[:6]):
        assert np.array_equal(r, t.cpu().numpy()), name
    assert np.array_equal(acc_ref, dacc.cpu().numpy())


def _species0(cells, label, amp):
    """Sheet electrons of the GEM workload on `cells` in precision `label`,
    a smooth E of amplitude `amp`, the kernel argument tail and host copies."""
    import torch
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.gem import (GemInit, gem_fields, gem_geometry, gem_species,
                                           init_gem_device)
    geom = gem_geometry(cells)
    species = gem_species(125)
    prec = PrecisionMode.from_label(label)
    pd, fd = prec.particle_dtype, prec.field_dtype
    p = init_gem_device(geom, species, torch.device("cuda"), precision=prec)[0]
    f = gem_fields(geom, GemInit(), prec)
    E = _smooth_e(geom, amp).astype(fd)
    B = np.ascontiguousarray(f.B, fd)
    inv = geom.inv_node_volume(fd)
    geo_f, geo_i = K.make_geo_arrays(geom, pd)
    geo_g, _ = K.make_geo_arrays(geom, fd)
    sc = K.kernel_scalars(species[0], 0.25, 1.0, pd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"],
            3, fd(SCALE), 1 if pd != fd else 0)
    return geom, p, E, B, inv, tail


@pytest.mark.parametrize("arith", ["parity", "fast"])
def test_c2_species_double(gpu, oracle, arith):
    """C2 (2D GEM at paper scale, 256x128x1, ppc 125) in f64: 4.1M sheet
    electrons bitwise (parity) or within 1e-10 (fast) of the oracle."""
    import torch
    from paper_2008_04397_b200 import kernels as K
    geom, p, E, B, inv, tail = _species0((256, 128, 1), "double", 1e-3)
    n = p.n
    assert n == 256 * 128 * 125
    ref = [a.cpu().numpy() for a in p.arrays()]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    st_ref = oracle.fused_parallel(*ref, 0, n, E, B, acc_ref, inv, *tail, os.cpu_count() or 1)
    d = list(p.arrays())
    dE, dB, dinv = (torch.from_numpy(a).cuda() for a in (E, B, inv))
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith=arith)
    assert st == st_ref == 0
    got = [t.cpu().numpy() for t in d[:6]]
    if arith == "parity":
        for name, r, t in zip("xyzuvw", ref, got):
            assert np.array_equal(r, t), name
        assert np.array_equal(acc_ref, dacc.cpu().numpy())
        return
    periods = (geom.Lx, None, geom.Lz, None, None, None)
    for name, r, t, per in zip("xyzuvw", ref, got, periods):
        _assert_close(name, r, t, 1e-10, per)
    # the moments live on the 2^-43 lattice: a contribution within an ulp of a
    # half quantum rounds either way, so next to 1e-10 of the array max a few
    # quanta per node are the reference's own quantisation (on the small
    # current rows one quantum is more than 1e-10 of the row's max)
    acc = dacc.cpu().numpy()
    for m in range(10):
        diff = np.abs(acc[m] - acc_ref[m])
        bound = 1e-10 * np.abs(acc_ref[m]).max() + 4
        assert diff.max() <= bound, (m, int(diff.max()), bound)
        assert (diff > 0).mean() < 1e-3, (m, float((diff > 0).mean()))
