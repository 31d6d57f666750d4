"""The reference's mover / interpolation test strategy
(pkg/tests/test_mover.py) run against the B200 API: analytic oracles for
weights, gathers, rotation and drift, exact deposit dyadics, charge
conservation, and the fused == two-pass bitwise identity."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ULP = np.finfo(np.float64).eps


@pytest.fixture
def unit_geom():
    from paper_2008_04397_b200.geometry import GridGeometry
    return GridGeometry.from_box((4, 4, 4), (4.0, 4.0, 4.0))


@pytest.fixture
def mixed_bc_geom():
    from paper_2008_04397_b200.geometry import GridGeometry
    return GridGeometry.from_box((8, 8, 8), (6.4, 6.4, 6.4),
                                 bc=("periodic", "reflecting", "periodic"))


def uniform_fields(geom, E=(0.0, 0.0, 0.0), B=(0.0, 0.0, 0.0)):
    from paper_2008_04397_b200.fields import FieldGrid
    f = FieldGrid.zeros(geom)
    for c in range(3):
        f.E[c] = E[c]
        f.B[c] = B[c]
    return f


def _species(qom=1.0, iters=3):
    from paper_2008_04397_b200.config import SpeciesParams
    return SpeciesParams(0, qom, 1.0, 1, mover_iters=iters)


def test_gather_uniform_and_at_node(gpu, unit_geom):
    from paper_2008_04397_b200.fields import FieldGrid
    from paper_2008_04397_b200.mover import gather_fields
    f = uniform_fields(unit_geom, E=(1.0, 0.0, 0.0))
    s = gather_fields(np.array([1.37, 2.64, 0.11]), f, unit_geom)
    assert abs(s.E[0] - 1.0) <= 2 * ULP and s.E[1] == 0.0 and (s.B == 0.0).all()
    f = FieldGrid.zeros(unit_geom)
    f.E[0, 2, 1, 3] = 7.5
    assert gather_fields(np.array([2.0, 1.0, 3.0]), f, unit_geom).E[0] == 7.5


def test_gather_reproduces_linear_field(gpu, unit_geom):
    from paper_2008_04397_b200.fields import FieldGrid
    from paper_2008_04397_b200 import kernels as K
    a, b = 0.35, -1.2
    f = FieldGrid.zeros(unit_geom)
    f.E[0] = (a + b * unit_geom.node_coords(0))[:, None, None]
    rng = np.random.default_rng(1)
    pos = rng.random((3000, 3)) * 4.0
    geo_g, geo_i = K.make_geo_arrays(unit_geom, np.float64)
    out = np.empty((3000, 6))
    K.gather_span(*[np.ascontiguousarray(pos[:, k]) for k in range(3)], 0, 3000, f.E, f.B,
                  geo_g, geo_i, 1.0, out)
    expect = a + b * pos[:, 0]
    assert (np.abs(out[:, 0] - expect) <= 8 * ULP * np.maximum(1.0, np.abs(expect))).all()


def test_mover_free_streaming_bitwise(gpu, unit_geom):
    from paper_2008_04397_b200.fields import FieldGrid
    from paper_2008_04397_b200.mover import mover_iterate
    f = FieldGrid.zeros(unit_geom)
    x0, v0 = np.array([1.0, 2.0, 3.0]), np.array([0.3, -0.1, 0.07])
    x1, v1 = mover_iterate(x0, v0, f, _species(), 0.5, unit_geom)
    assert np.array_equal(v1, v0) and np.array_equal(x1, x0 + v0 * 0.5)


def test_mover_uniform_b_rotation_angle(gpu, unit_geom):
    from paper_2008_04397_b200.mover import mover_iterate
    from paper_2008_04397_b200.particles import ParticleBuffer, apply_boundaries
    B0, dt = 1.3, 0.2
    f = uniform_fields(unit_geom, B=(0.0, 0.0, B0))
    expected = 2.0 * np.arctan(dt / 2.0 * B0)
    x, v = np.array([2.0, 2.0, 2.0]), np.array([0.01, 0.0, 0.0])
    speed0 = np.linalg.norm(v)
    for _ in range(50):
        xn, vn = mover_iterate(x, v, f, _species(), dt, unit_geom)
        ang = np.arctan2(v[0] * vn[1] - v[1] * vn[0], v[0] * vn[0] + v[1] * vn[1])
        assert abs(abs(ang) - expected) <= 1e-12 * expected
        assert np.linalg.norm(vn) == pytest.approx(speed0, rel=8 * ULP)
        buf = ParticleBuffer.empty(1)
        buf.x[0], buf.y[0], buf.z[0] = xn
        buf.u[0], buf.v[0], buf.w[0] = vn
        apply_boundaries(buf, unit_geom)
        x, v = np.array([buf.x[0], buf.y[0], buf.z[0]]), vn


def test_exb_drift(gpu, unit_geom):
    from paper_2008_04397_b200.mover import push_buffer
    from paper_2008_04397_b200.particles import ParticleBuffer
    E0, B0, dt = 0.02, 1.0, 1.0
    f = uniform_fields(unit_geom, E=(0.0, E0, 0.0), B=(0.0, 0.0, B0))
    angle = 2.0 * np.arctan(dt / 2.0 * B0)
    n_steps = int(round(100 * 2.0 * np.pi / angle))
    buf = ParticleBuffer.empty(1)
    buf.x[0] = buf.y[0] = buf.z[0] = 2.0
    vsum = np.zeros(3)
    for _ in range(n_steps):
        push_buffer(buf, f, _species(), dt, unit_geom, apply_bc=True)
        vsum += [buf.u[0], buf.v[0], buf.w[0]]
    assert (vsum / n_steps)[0] == pytest.approx(E0 / B0, rel=0.02)


def test_midpoint_error_raises(gpu, unit_geom):
    from paper_2008_04397_b200.errors import IntegrityError
    from paper_2008_04397_b200.fields import FieldGrid
    from paper_2008_04397_b200.mover import mover_iterate
    with pytest.raises(IntegrityError):
        mover_iterate(np.array([2.0, 2.0, 2.0]), np.array([40.0, 0.0, 0.0]),
                      FieldGrid.zeros(unit_geom), _species(), 0.5, unit_geom)


def test_deposit_exact_values(gpu, unit_geom):
    from paper_2008_04397_b200.fields import MomentGrid
    from paper_2008_04397_b200.mover import deposit_moments
    m = MomentGrid.zeros(unit_geom)
    deposit_moments(np.array([2.0, 1.0, 3.0]), np.zeros(3), 1.0, m, unit_geom)
    assert m.rho[2, 1, 3] == 1.0 and m.rho.sum() == 1.0
    m = MomentGrid.zeros(unit_geom)
    deposit_moments(np.array([0.5, 0.5, 0.5]), np.array([2.0, 0.0, 0.0]), 1.0, m, unit_geom)
    sub = (slice(0, 2),) * 3
    assert np.array_equal(m.rho[sub], np.full((2, 2, 2), 0.125))
    assert np.array_equal(m.J[0][sub], np.full((2, 2, 2), 0.25))
    assert np.array_equal(m.P[0][sub], np.full((2, 2, 2), 0.5))
    assert m.P[1].sum() == 0.0


def test_deposit_charge_conservation(gpu, unit_geom):
    from paper_2008_04397_b200.fields import MomentGrid
    from paper_2008_04397_b200.mover import deposit_buffer
    from paper_2008_04397_b200.particles import ParticleBuffer
    rng = np.random.default_rng(8)
    n = 1_000_000
    buf = ParticleBuffer.empty(n)
    for a in ("x", "y", "z"):
        getattr(buf, a)[:] = rng.random(n) * 4.0
    for a in ("u", "v", "w"):
        getattr(buf, a)[:] = rng.standard_normal(n)
    buf.q_p[:] = rng.random(n) - 0.3
    m = MomentGrid.zeros(unit_geom)
    deposit_buffer(buf, m, unit_geom)
    m.fold(unit_geom)
    total = float((m.rho * unit_geom.node_weights()).sum()) * unit_geom.cell_volume
    assert total == pytest.approx(float(buf.q_p.sum()), rel=1e-12, abs=1e-9)


def _random_state(geom, n, seed, dtype=np.float64):
    from paper_2008_04397_b200.config import PrecisionMode
    from paper_2008_04397_b200.fields import FieldGrid
    from paper_2008_04397_b200.particles import ParticleBuffer
    rng = np.random.default_rng(seed)
    buf = ParticleBuffer.empty(n, dtype=dtype)
    buf.x[:] = rng.random(n) * geom.Lx
    buf.y[:] = rng.random(n) * geom.Ly
    buf.z[:] = rng.random(n) * geom.Lz
    for a in ("u", "v", "w"):
        getattr(buf, a)[:] = rng.standard_normal(n) * 0.1
    buf.q_p[:] = rng.random(n) * 1e-2
    mode = PrecisionMode() if dtype == np.float64 else PrecisionMode("single", "single")
    f = FieldGrid.zeros(geom, mode)
    f.E[:] = (rng.standard_normal(f.E.shape) * 0.01).astype(f.dtype)
    f.B[:] = (rng.standard_normal(f.B.shape) * 0.5).astype(f.dtype)
    return buf, f, mode


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_fused_equals_two_pass(gpu, mixed_bc_geom, dtype):
    from paper_2008_04397_b200.config import SpeciesParams
    from paper_2008_04397_b200.fields import MomentGrid
    from paper_2008_04397_b200.mover import deposit_buffer, move_and_deposit_batch, push_buffer
    geom = mixed_bc_geom
    sp = SpeciesParams(0, -1.0, 0.1, 1, mover_iters=3)
    buf, f, mode = _random_state(geom, 10_000, 21, dtype)
    fb, fm = buf.copy(), MomentGrid.zeros(geom, precision_mode=mode)
    move_and_deposit_batch((0, fb.n), fb, f, fm, sp, 0.2, geom)
    rb, rm = buf.copy(), MomentGrid.zeros(geom, precision_mode=mode)
    push_buffer(rb, f, sp, 0.2, geom, apply_bc=True)
    deposit_buffer(rb, rm, geom)
    for a in ("x", "y", "z", "u", "v", "w"):
        assert np.array_equal(getattr(fb, a), getattr(rb, a)), a
    assert np.array_equal(fm.acc, rm.acc)


def test_two_spans_equal_one_and_empty_span(gpu, mixed_bc_geom):
    from paper_2008_04397_b200.config import SpeciesParams
    from paper_2008_04397_b200.fields import MomentGrid
    from paper_2008_04397_b200.mover import move_and_deposit_batch
    geom = mixed_bc_geom
    sp = SpeciesParams(0, -1.0, 0.1, 1)
    buf, f, _ = _random_state(geom, 5000, 24)
    sb, ma, mb = buf.copy(), MomentGrid.zeros(geom), MomentGrid.zeros(geom)
    move_and_deposit_batch((0, 2500), sb, f, ma, sp, 0.2, geom)
    move_and_deposit_batch((2500, 2500), sb, f, mb, sp, 0.2, geom)
    ma.add(mb)
    wb, mw = buf.copy(), MomentGrid.zeros(geom)
    move_and_deposit_batch((0, 5000), wb, f, mw, sp, 0.2, geom)
    assert np.array_equal(ma.acc, mw.acc)
    for a in ("x", "y", "z", "u", "v", "w"):
        assert np.array_equal(getattr(sb, a), getattr(wb, a))
    m0 = MomentGrid.zeros(geom)
    before = buf.copy()
    move_and_deposit_batch((50, 0), buf, f, m0, sp, 0.1, geom)
    assert (m0.acc == 0).all() and np.array_equal(buf.x, before.x)


def test_device_sort_matches_reference_order(gpu):
    """bp_sort_by_cell == np.argsort(kind='stable') of the reference keys,
    on the golden sort fixture and on a large shuffled GEM shard."""
    import torch
    from conftest import golden
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200.particles import DeviceParticles, ParticleBuffer
    g = golden("sort.npz")
    geom = GridGeometry.from_box((4, 4, 4), (4.0, 4.0, 4.0))
    n = g["x"].shape[0]
    buf = ParticleBuffer.empty(n)
    buf.x[:], buf.y[:], buf.z[:] = g["x"], g["y"], g["z"]
    dp = DeviceParticles.from_host(buf, torch.device("cuda"))
    dp.sort_by_cell(geom)
    assert np.array_equal(dp.ids.cpu().numpy(), g["ids_after"])
    geom2 = GridGeometry.from_box((64, 32, 16), (25.6, 12.8, 6.4))
    rng = np.random.default_rng(3)
    n = 2_000_000
    b2 = ParticleBuffer.empty(n, dtype=np.float32)
    for a, L in zip("xyz", geom2.lengths):
        getattr(b2, a)[:] = (rng.random(n) * L).astype(np.float32)
    b2.u[:] = rng.standard_normal(n).astype(np.float32)
    keys = geom2.cell_index_of(b2.x, b2.y, b2.z)
    order = np.argsort(keys, kind="stable")
    d2 = DeviceParticles.from_host(b2, torch.device("cuda"))
    d2.sort_by_cell(geom2)
    assert np.array_equal(d2.ids.cpu().numpy(), order)
    assert np.array_equal(d2.u.cpu().numpy(), b2.u[order])


def test_inplace_and_swap_sorts_agree(gpu):
    """bp_sort_by_cell (in place) and bp_sort_by_cell_into (spare + swap)
    produce the same order and bytes; a position below the origin raises
    DomainError and leaves the buffer untouched."""
    import torch
    from paper_2008_04397_b200.errors import DomainError
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200.particles import DeviceParticles, ParticleBuffer
    geom = GridGeometry.from_box((32, 16, 8), (6.4, 3.2, 1.6))
    rng = np.random.default_rng(5)
    n = 300_000
    b = ParticleBuffer.empty(n, dtype=np.float32)
    for a, L in zip("xyzuvw", geom.lengths + (1.0, 1.0, 1.0)):
        getattr(b, a)[:] = (rng.random(n) * L).astype(np.float32)
    b.q_p[:] = rng.random(n).astype(np.float32)
    d1 = DeviceParticles.from_host(b, torch.device("cuda")).sort_by_cell(geom)
    d2 = DeviceParticles.from_host(b, torch.device("cuda")).sort_by_cell_inplace(geom)
    for a in ("x", "y", "z", "u", "v", "w", "q_p", "ids"):
        assert torch.equal(getattr(d1, a), getattr(d2, a)), a
    d1.sort_by_cell(geom)  # second sort reuses the spare set: already sorted -> same
    assert torch.equal(d1.ids, d2.ids)
    b.x[7] = -1.0
    d3 = DeviceParticles.from_host(b, torch.device("cuda"))
    before = d3.ids.clone()
    with pytest.raises(DomainError):
        d3.sort_by_cell(geom)
    assert torch.equal(d3.ids, before)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("n", [1, 3, 5, 1027, 100_003])
def test_device_sort_every_array_ragged(gpu, dtype, n):
    """The grouped gather of the sort (three in-order passes, four
    destinations per thread, a ragged tail) moves all eight arrays exactly as
    the stable numpy permutation, for sizes that are not multiples of 4."""
    import torch
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200.particles import DeviceParticles, ParticleBuffer
    geom = GridGeometry.from_box((16, 8, 4), (3.2, 1.6, 0.8))
    rng = np.random.default_rng(n)
    b = ParticleBuffer.empty(n, dtype=dtype)
    for a, L in zip("xyz", geom.lengths):
        getattr(b, a)[:] = (rng.random(n) * L).astype(dtype)
    for a in ("u", "v", "w", "q_p"):
        getattr(b, a)[:] = rng.standard_normal(n).astype(dtype)
    b.ids[:] = rng.permutation(n).astype(np.int64) * 7 + 3
    order = np.argsort(geom.cell_index_of(b.x, b.y, b.z), kind="stable")
    d = DeviceParticles.from_host(b, torch.device("cuda")).sort_by_cell(geom)
    for a in ("x", "y", "z", "u", "v", "w", "q_p", "ids"):
        assert np.array_equal(getattr(d, a).cpu().numpy(), getattr(b, a)[order]), a


def test_concurrent_sorts_on_side_streams(gpu):
    """Sorts of different buffers from host threads on their own streams
    (each leases its own workspace) give the sequential result."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200.particles import DeviceParticles, ParticleBuffer
    geom = GridGeometry.from_box((32, 16, 8), (6.4, 3.2, 1.6))
    bufs = []
    for k in range(4):
        rng = np.random.default_rng(100 + k)
        n = 400_000 + 13 * k
        b = ParticleBuffer.empty(n, dtype=np.float32)
        for a, L in zip("xyzuvw", geom.lengths + (1.0, 1.0, 1.0)):
            getattr(b, a)[:] = (rng.random(n) * L).astype(np.float32)
        bufs.append(b)
    dev = torch.device("cuda")
    seq = [DeviceParticles.from_host(b, dev).sort_by_cell(geom) for b in bufs]
    par = [DeviceParticles.from_host(b, dev) for b in bufs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in par]

    def one(i):
        with torch.cuda.device(dev):
            return par[i].sort_by_cell(geom, stream=streams[i])

    with ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(one, range(4)))
    torch.cuda.synchronize()
    for a, b in zip(seq, par):
        for name in ("x", "y", "z", "u", "v", "w", "ids"):
            assert torch.equal(getattr(a, name), getattr(b, name)), name
