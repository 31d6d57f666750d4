"""CUDA kernels through the C ABI against the reference golden vectors and the
CPU oracle: bitwise in parity arithmetic for double / single / mixed."""

import numpy as np
import pytest

from conftest import MODES, golden
from test_oracle_golden import case_args

pytestmark = pytest.mark.gpu

SCALE = 2.0 ** 43


def _dev(torch, arrs):
    return [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in arrs]


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("where", ["device", "host"])
def test_fused_matches_reference_golden(gpu, mode, ci, where):
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    g = golden(f"kernels_{mode}.npz")
    a = case_args(g, mode, ci)
    acc = np.zeros((10, 9, 9, 9), np.int64)
    args = (a["start"], a["count"])
    tail = (a["geo_f"], a["geo_g"], a["geo_i"], a["sc"]["dt"], a["sc"]["dth"],
            a["sc"]["qdt2m"], a["sc"]["beta"], a["sc"]["one"], 3, a["fd"](SCALE),
            a["mixed"])
    if where == "device":
        d = _dev(torch, a["arrs"])
        dE, dB, dacc, dinv = _dev(torch, [a["E"], a["B"], acc, a["inv"]])
        st = K.fused_span(*d, *args, dE, dB, dacc, dinv, *tail)
        out = [t.cpu().numpy() for t in d]
        acc = dacc.cpu().numpy()
    else:
        out = a["arrs"]
        st = K.fused_span(*out, *args, a["E"], a["B"], acc, a["inv"], *tail,
                          batch_particles=1000)
    assert st == int(g[a["pre"] + "fused_status"])
    for n, arr in zip("xyzuvw", out):
        assert np.array_equal(arr, g[a["pre"] + "fused_" + n]), n
    assert np.array_equal(acc, g[a["pre"] + "fused_acc"])


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("ci", [0, 2])
@pytest.mark.parametrize("bc", [0, 1])
def test_push_matches_reference_golden(gpu, mode, ci, bc):
    from paper_2008_04397_b200 import kernels as K
    g = golden(f"kernels_{mode}.npz")
    a = case_args(g, mode, ci)
    arrs = a["arrs"][:6]
    st = K.push_span(*arrs, a["start"], a["count"], a["E"], a["B"], a["geo_f"],
                     a["geo_g"], a["geo_i"], a["sc"]["dt"], a["sc"]["dth"],
                     a["sc"]["qdt2m"], a["sc"]["beta"], a["sc"]["one"], 3, bc,
                     a["mixed"])
    assert st == int(g[a["pre"] + f"push{bc}_status"])
    for n, arr in zip("xyzuvw", arrs):
        assert np.array_equal(arr, g[a["pre"] + f"push{bc}_" + n]), n


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("ci", [0, 1])
def test_deposit_and_gather_match_reference_golden(gpu, mode, ci):
    from paper_2008_04397_b200 import kernels as K
    g = golden(f"kernels_{mode}.npz")
    a = case_args(g, mode, ci)
    acc = np.zeros((10, 9, 9, 9), np.int64)
    st = K.deposit_span(*a["arrs"], a["start"], a["count"], acc, a["inv"], a["geo_g"],
                        a["geo_i"], a["fd"](1.0), a["fd"](SCALE))
    assert st == 0
    assert np.array_equal(acc, g[a["pre"] + "deposit_acc"])
    out = np.zeros((a["count"], 6), a["pd"])
    K.gather_span(a["arrs"][0], a["arrs"][1], a["arrs"][2], a["start"], a["count"],
                  a["E"], a["B"], a["geo_g"], a["geo_i"], a["pd"](1.0), out)
    assert np.array_equal(out, g[a["pre"] + "gather_out"])


def _random_state(mode, n, seed, cells=(16, 8, 8), box=(6.4, 3.2, 3.2), vscale=0.3,
                  order="random", bc=("periodic", "reflecting", "periodic")):
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.config import SpeciesParams
    pd, fd = MODES[mode]
    geom = GridGeometry.from_box(cells, box, bc=bc)
    rng = np.random.default_rng(seed)
    x = rng.random(n) * geom.Lx
    y = rng.random(n) * geom.Ly
    z = rng.random(n) * geom.Lz
    if order == "sorted":
        keys = geom.cell_index_of(x, y, z)
        o = np.argsort(keys, kind="stable")
        x, y, z = x[o], y[o], z[o]
    arrs = [x.astype(pd), y.astype(pd), z.astype(pd)] + [
        (rng.standard_normal(n) * vscale).astype(pd) for _ in range(3)] + [
        (rng.random(n) * 1e-3 + 1e-4).astype(pd)]
    shp = (3,) + geom.node_shape
    E = (rng.standard_normal(shp) * 0.05).astype(fd)
    B = (rng.standard_normal(shp) * 0.8).astype(fd)
    sp = SpeciesParams(0, -1.0, 0.1, 1, mover_iters=3)
    geo_f, geo_i = K.make_geo_arrays(geom, pd)
    geo_g, _ = K.make_geo_arrays(geom, fd)
    sc = K.kernel_scalars(sp, 0.2, 1.0, pd)
    return geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("order", ["random", "sorted"])
def test_fused_matches_oracle_large(gpu, oracle, mode, order):
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 400_000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state(
        mode, n, seed=11, order=order)
    inv = geom.inv_node_volume(fd)
    mixed = 1 if pd != fd else 0
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    ref = [a.copy() for a in arrs]
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"],
            sc["one"], 3, fd(SCALE), mixed)
    st_ref = oracle.fused_span(*ref, 0, n, E, B, acc_ref, inv, *tail)
    d = _dev(torch, arrs)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail)
    assert st == st_ref
    for name, r, t in zip("xyzuvw", ref, d):
        assert np.array_equal(r, t.cpu().numpy()), name
    assert np.array_equal(acc_ref, dacc.cpu().numpy())


def test_fused_empty_span_and_offsets(gpu, oracle):
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 5000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state("double", n, 3)
    inv = geom.inv_node_volume(fd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"],
            sc["one"], 3, SCALE, 0)
    d = _dev(torch, arrs)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    before = [t.clone() for t in d]
    assert K.fused_span(*d, 2500, 0, dE, dB, dacc, dinv, *tail) == 0
    assert int(dacc.abs().sum()) == 0
    assert all(torch.equal(a, b) for a, b in zip(before, d))
    # two disjoint spans into one accumulator == one span
    K.fused_span(*d, 0, 1234, dE, dB, dacc, dinv, *tail)
    K.fused_span(*d, 1234, n - 1234, dE, dB, dacc, dinv, *tail)
    ref = [a.copy() for a in arrs]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    oracle.fused_span(*ref, 0, n, E, B, acc_ref, inv, *tail)
    assert np.array_equal(acc_ref, dacc.cpu().numpy())
    for r, t in zip(ref, d):
        assert np.array_equal(r, t.cpu().numpy())
    with pytest.raises(IndexError):
        K.fused_span(*d, n - 10, 11, dE, dB, dacc, dinv, *tail)


def _assert_close(name, ref, got, rtol, period=None):
    ref = np.asarray(ref, np.float64)
    got = np.asarray(got, np.float64)
    d = np.abs(got - ref)
    if period is not None:  # periodic axes: a wrap decided on the other side of the face
        d = np.minimum(d, np.abs(period - d))
    scale = max(np.abs(ref).max(), 1e-300)
    worst = d.max() / scale if d.size else 0.0
    assert worst <= rtol, f"{name}: max |diff| / max |ref| = {worst:.3e} > {rtol:.1e}"


# north-star tolerances: 1e-10 (f64), 1e-4 (f32), relative to the array max
FAST_RTOL = {"double": 1e-10, "single": 1e-4, "mixed": 1e-4}


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("order", ["random", "sorted"])
def test_fast_arith_within_tolerance_of_oracle(gpu, oracle, mode, order):
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 300_000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state(
        mode, n, seed=17, order=order)
    inv = geom.inv_node_volume(fd)
    mixed = 1 if pd != fd else 0
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"],
            sc["one"], 3, fd(SCALE), mixed)
    ref = [a.copy() for a in arrs]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    st_ref = oracle.fused_span(*ref, 0, n, E, B, acc_ref, inv, *tail)
    d = _dev(torch, arrs)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith="fast")
    assert st == st_ref
    rtol = FAST_RTOL[mode]
    periods = (geom.Lx, None, geom.Lz, None, None, None)
    for name, r, t, per in zip("xyzuvw", ref, d, periods):
        _assert_close(name, r, t.cpu().numpy(), rtol, per)
    got = dacc.cpu().numpy()
    for m in range(10):
        _assert_close(f"moment {m}", acc_ref[m] * 2.0 ** -43, got[m] * 2.0 ** -43, rtol)


def test_fast_arith_deposit_is_order_independent(gpu):
    """Fast arithmetic keeps the exact int64 lattice: a shuffled span deposits
    bit-identical moments."""
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 200_000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state("single", n, seed=5)
    inv = geom.inv_node_volume(fd)
    out = []
    for perm in (np.arange(n), np.random.default_rng(1).permutation(n)):
        d = _dev(torch, [a[perm] for a in arrs])
        dinv = _dev(torch, [inv])[0]
        dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
        K.deposit_span(*d, 0, n, dacc, dinv, geo_g, geo_i, fd(1.0), fd(SCALE))
        out.append(dacc.cpu().numpy())
    assert np.array_equal(out[0], out[1])


@pytest.fixture
def tma_stream(monkeypatch):
    """Route full particle tiles through the TMA bulk-copy path."""
    monkeypatch.setenv("BP_TMA_STREAM", "1")
    yield


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("arith", ["parity", "fast"])
def test_tma_stream_path_matches(gpu, oracle, tma_stream, monkeypatch, mode, arith):
    """The bulk-copy (UBLKCP) streaming path gives the same bits as the plain
    path: bitwise vs the oracle in parity arithmetic, and identical to the
    plain fast path in fast arithmetic (a span with an unaligned start and a
    ragged tail exercises the fallback tiles)."""
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 100_003
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state(mode, n, seed=29,
                                                                       order="sorted")
    inv = geom.inv_node_volume(fd)
    mixed = 1 if pd != fd else 0
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
            fd(SCALE), mixed)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    for start in (0, 3):
        count = n - start
        out = []
        for env in ("1", "0"):
            monkeypatch.setenv("BP_TMA_STREAM", env)
            d = _dev(torch, arrs)
            dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
            st = K.fused_span(*d, start, count, dE, dB, dacc, dinv, *tail, arith=arith)
            out.append((st, dacc, d))
        (st, dacc, d), (st2, dacc2, d2) = out
        assert st == st2 and torch.equal(dacc, dacc2)
        assert all(torch.equal(a, b) for a, b in zip(d, d2))
        if arith == "parity":
            ref = [a.copy() for a in arrs]
            acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
            oracle.fused_span(*ref, start, count, E, B, acc_ref, inv, *tail)
            assert np.array_equal(acc_ref, dacc.cpu().numpy())
            assert all(np.array_equal(r, t.cpu().numpy()) for r, t in zip(ref, d))


@pytest.mark.parametrize("mode", ["single", "mixed"])
def test_fast_f32_fused_is_deterministic(gpu, mode):
    """The fast fused kernels (bp_split.cu) claim work dynamically but flush
    every chunk's sums on its own, so repeated launches give identical bits."""
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 250_000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state(mode, n, seed=41,
                                                                       order="sorted")
    inv = geom.inv_node_volume(fd)
    mixed = 1 if pd != fd else 0
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
            fd(SCALE), mixed)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    outs = []
    for _ in range(3):
        d = _dev(torch, arrs)
        dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
        K.fused_span(*d, 0, n, dE, dB, dacc, dinv, *tail, arith="fast")
        outs.append((dacc, d))
    for dacc, d in outs[1:]:
        assert torch.equal(dacc, outs[0][0])
        assert all(torch.equal(a, b) for a, b in zip(d, outs[0][1]))


_BCS = [(a, b, c) for a in ("periodic", "reflecting") for b in ("periodic", "reflecting")
        for c in ("periodic", "reflecting")]


@pytest.mark.parametrize("bc", _BCS, ids=["".join(k[0] for k in b) for b in _BCS])
@pytest.mark.parametrize("failing", [False, True])
@pytest.mark.parametrize("mode", ["single", "mixed", "double"])
def test_fast_split_every_boundary_kind(gpu, oracle, bc, failing, mode):
    """The fast kernels are instantiated per boundary kind (bp_split.cu): every
    combination against the oracle within 1e-4 (f32) / 1e-10 (f64), on a span
    with an unaligned start and a ragged tail.  `failing` gives one particle in 97 a velocity
    of 1e4 (a certain runaway / midpoint failure): those must be neither
    stored nor deposited, exactly as in the reference."""
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 60_013
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state(
        mode, n, seed=101, order="sorted", bc=bc)
    rtol = FAST_RTOL[mode]
    mixed = 1 if pd != fd else 0
    if failing:
        bad = np.arange(5, n, 97)
        arrs[3][bad] = pd(1e4)
        arrs[4][bad[::2]] = pd(-1e4)
    inv = geom.inv_node_volume(fd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
            fd(SCALE), mixed)
    start, count = 77, n - 77 - 5
    ref = [a.copy() for a in arrs]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    st_ref = oracle.fused_span(*ref, start, count, E, B, acc_ref, inv, *tail)
    d = _dev(torch, arrs)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, start, count, dE, dB, dacc, dinv, *tail, arith="fast")
    assert st == st_ref
    assert (st != 0) == failing
    periods = [geom.lengths[k] if bc[k] == "periodic" else None for k in range(3)]
    periods += [None, None, None]
    for name, r, t, per in zip("xyzuvw", ref, d, periods):
        got = t.cpu().numpy()
        # outside the span nothing moves
        assert np.array_equal(got[:start], r[:start]) and np.array_equal(got[start + count:],
                                                                            r[start + count:])
        _assert_close(name, r, got, rtol, per)
    got = dacc.cpu().numpy()
    for m in range(10):
        _assert_close(f"moment {m}", acc_ref[m] * 2.0 ** -43, got[m] * 2.0 ** -43, rtol)


def test_prepared_records_and_timing_api(gpu):
    """bp_field_records_build + bp_fused_span_rec give the same bits as the
    per-call record build, and bp_timing_read reports the f32 kernels."""
    import ctypes
    from paper_2008_04397_b200 import _lib
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    L = _lib.load()
    n = 100_000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state("single", n, seed=7,
                                                                       order="sorted")
    inv = geom.inv_node_volume(fd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
            fd(SCALE), 0)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    d1 = _dev(torch, arrs)
    acc1 = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    L.bp_timing_enable(1)
    _lib.timing_read()
    st1 = K.fused_span(*d1, 0, n, dE, dB, acc1, dinv, *tail, arith="fast")
    t = _lib.timing_read()
    L.bp_timing_enable(0)
    assert t["mover"][1] == 1 and t["deposit"][1] == 1 and t["records"][1] == 1
    assert t["mover"][0] > 0.0 and t["deposit"][0] > 0.0
    gi = np.ascontiguousarray(geo_i, np.int64)
    nbytes = L.bp_field_records_bytes(4, ctypes.c_void_p(gi.ctypes.data))
    assert nbytes > 0
    rec = torch.empty(nbytes // 4 + 64, dtype=torch.float32, device="cuda")
    ptr = (rec.data_ptr() + 255) & ~255
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert L.bp_field_records_build(4, 4, ctypes.c_void_p(dE.data_ptr()),
                                    ctypes.c_void_p(dB.data_ptr()),
                                    ctypes.c_void_p(gi.ctypes.data), ctypes.c_void_p(ptr),
                                    stream) == 0
    # misaligned records are refused
    assert L.bp_field_records_build(4, 4, ctypes.c_void_p(dE.data_ptr()),
                                    ctypes.c_void_p(dB.data_ptr()),
                                    ctypes.c_void_p(gi.ctypes.data), ctypes.c_void_p(ptr + 4),
                                    stream) == _lib.EINVAL
    d2 = _dev(torch, arrs)
    acc2 = torch.zeros_like(acc1)
    hp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    gf, gg = (np.ascontiguousarray(g, np.float64) for g in (geo_f, geo_g))
    st2 = L.bp_fused_span_rec(_lib.ARITH_FAST, 4, 4, *[ctypes.c_void_p(a.data_ptr()) for a in d2],
                              0, n, ctypes.c_void_p(dE.data_ptr()), ctypes.c_void_p(dB.data_ptr()),
                              ctypes.c_void_p(acc2.data_ptr()), ctypes.c_void_p(dinv.data_ptr()),
                              hp(gf), hp(gg), hp(gi), float(sc["dt"]), float(sc["dth"]),
                              float(sc["qdt2m"]), float(sc["beta"]), float(sc["one"]), 3,
                              float(SCALE), 0, ctypes.c_void_p(ptr), None, stream)
    assert st2 == st1
    assert torch.equal(acc1, acc2)
    assert all(torch.equal(a, b) for a, b in zip(d1, d2))



@pytest.mark.parametrize("count", [0, 1, 5, 31, 33, 511, 513])
def test_fast_split_tiny_spans(gpu, oracle, count):
    """Spans shorter than a tile, a chunk or a warp round, at an odd start."""
    from paper_2008_04397_b200 import kernels as K
    torch = gpu
    n = 2_000
    geom, arrs, E, B, geo_f, geo_g, geo_i, sc, pd, fd = _random_state("single", n, seed=3,
                                                                       order="sorted")
    inv = geom.inv_node_volume(fd)
    tail = (geo_f, geo_g, geo_i, sc["dt"], sc["dth"], sc["qdt2m"], sc["beta"], sc["one"], 3,
            fd(SCALE), 0)
    start = 13
    ref = [a.copy() for a in arrs]
    acc_ref = np.zeros((10,) + geom.node_shape, np.int64)
    st_ref = oracle.fused_span(*ref, start, count, E, B, acc_ref, inv, *tail)
    d = _dev(torch, arrs)
    dE, dB, dinv = _dev(torch, [E, B, inv])
    dacc = torch.zeros((10,) + geom.node_shape, dtype=torch.int64, device="cuda")
    st = K.fused_span(*d, start, count, dE, dB, dacc, dinv, *tail, arith="fast")
    assert st == st_ref
    for name, r, t in zip("xyzuvw", ref, d):
        got = t.cpu().numpy()
        assert np.array_equal(got[:start], r[:start])
        assert np.array_equal(got[start + count:], r[start + count:])
        if count:
            _assert_close(name, r[start:start + count], got[start:start + count], 1e-4,
                          geom.Lx if name == "x" else (geom.Lz if name == "z" else None))
    got = dacc.cpu().numpy()
    if count == 0:
        assert not got.any()
    for m in range(10):
        if count:
            _assert_close(f"moment {m}", acc_ref[m] * 2.0 ** -43, got[m] * 2.0 ** -43, 1e-4)


def _host_records(E, B, nx, ny, nz, out_dtype):
    """The cell-record contract of bp_field_records_build on the host: per cell
    (x fastest) the trilinear coefficients of (Ex Ey | Bx By | Ez Bz) from the
    8 nodes in f64, rounded once; then max |E| over the nodes, rounded up."""
    F = [np.asarray(E[0], np.float64), np.asarray(E[1], np.float64), np.asarray(E[2], np.float64),
         np.asarray(B[0], np.float64), np.asarray(B[1], np.float64), np.asarray(B[2], np.float64)]
    comp = (0, 1, 3, 4, 2, 5)
    co = []
    for m in comp:
        f = F[m]
        f000, f100, f010, f110 = f[:-1, :-1, :-1], f[1:, :-1, :-1], f[:-1, 1:, :-1], f[1:, 1:, :-1]
        f001, f101, f011, f111 = f[:-1, :-1, 1:], f[1:, :-1, 1:], f[:-1, 1:, 1:], f[1:, 1:, 1:]
        co.append([f000, f100 - f000, f010 - f000, f001 - f000,
                   (f110 - f100) - (f010 - f000), (f101 - f001) - (f100 - f000),
                   (f011 - f001) - (f010 - f000),
                   ((f111 - f011) - (f101 - f001)) - ((f110 - f010) - (f100 - f000))])
    slot = ((0, 1), (2, 4), (3, 5), (6, 7))
    rec = np.empty((nz, ny, nx, 48), out_dtype)  # cell index i + nx (j + ny k)
    q = 0
    for pr in range(3):
        for a, b in slot:
            for v in (co[2 * pr][a], co[2 * pr + 1][a], co[2 * pr][b], co[2 * pr + 1][b]):
                rec[..., q] = v.transpose(2, 1, 0).astype(out_dtype)
                q += 1
    e2 = F[0] ** 2 + F[1] ** 2 + F[2] ** 2
    return rec.reshape(-1), np.sqrt(e2.max())


@pytest.mark.parametrize("cells", [(13, 7, 5), (64, 3, 17), (33, 2, 1)])
def test_cell_records_match_host_formula(gpu, cells):
    """bp_field_records_build (tiles of 32 x 8 cells, partial tiles at the
    grid edge included) writes exactly the host-computed records and an
    upper bound on max |E| that is its f32 round-up."""
    import ctypes
    from paper_2008_04397_b200 import _lib
    torch = gpu
    L = _lib.load()
    nx, ny, nz = cells
    rng = np.random.default_rng(sum(cells))
    E = rng.standard_normal((3, nx + 1, ny + 1, nz + 1)).astype(np.float32)
    B = rng.standard_normal((3, nx + 1, ny + 1, nz + 1)).astype(np.float32)
    gi = np.array([nx, ny, nz, 0, 1, 0], np.int64)
    nbytes = L.bp_field_records_bytes(4, ctypes.c_void_p(gi.ctypes.data))
    rec = torch.zeros(nbytes // 4 + 64, dtype=torch.float32, device="cuda")
    ptr = (rec.data_ptr() + 255) & ~255
    off = (ptr - rec.data_ptr()) // 4
    dE, dB = _dev(torch, [E, B])
    assert L.bp_field_records_build(4, 4, ctypes.c_void_p(dE.data_ptr()),
                                    ctypes.c_void_p(dB.data_ptr()),
                                    ctypes.c_void_p(gi.ctypes.data), ctypes.c_void_p(ptr),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    torch.cuda.synchronize()
    got = rec.cpu().numpy()[off:off + nbytes // 4]
    want, emax = _host_records(E, B, nx, ny, nz, np.float32)
    assert np.array_equal(got[:want.size], want)
    g_emax = got[want.size]
    assert g_emax >= emax and g_emax == np.float32(np.nextafter(np.float32(emax), np.inf)) or \
        g_emax == np.float32(emax)
