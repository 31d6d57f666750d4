"""The CPU oracle (oracle/oracle.cpp) against golden vectors produced by the
reference numba kernels (tests/golden/make_golden.py): bitwise in all three
precision modes, including the error paths and face-pinned particles."""

import numpy as np
import pytest

from conftest import MODES, golden


def _geo(mode):
    from paper_2008_04397_b200.geometry import GridGeometry
    from paper_2008_04397_b200 import kernels as K
    pd, fd = MODES[mode]
    geom = GridGeometry.from_box((8, 8, 8), (6.4, 6.4, 6.4),
                                 bc=("periodic", "reflecting", "periodic"))
    geo_f, geo_i = K.make_geo_arrays(geom, pd)
    geo_g, _ = K.make_geo_arrays(geom, fd)
    return geom, geo_f, geo_g, geo_i


def case_args(g, mode, ci):
    from paper_2008_04397_b200 import kernels as K
    from paper_2008_04397_b200.config import SpeciesParams
    pd, fd = MODES[mode]
    geom, geo_f, geo_g, geo_i = _geo(mode)
    sp = SpeciesParams(0, -1.0, 0.1, 1, mover_iters=3)
    sc = K.kernel_scalars(sp, float(g["dt"]), 1.0, pd)
    pre = f"c{ci}_"
    arrs = [g[pre + "in_" + n].copy() for n in "xyzuvwq"]
    start, count = (int(v) for v in g[pre + "span"])
    return dict(geom=geom, geo_f=geo_f, geo_g=geo_g, geo_i=geo_i, sc=sc, arrs=arrs,
                E=g[pre + "E"], B=g[pre + "B"], start=start, count=count,
                inv=geom.inv_node_volume(fd), mixed=1 if pd != fd else 0, pd=pd,
                fd=fd, pre=pre)


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("ci", [0, 1, 2])
def test_oracle_fused_matches_reference(oracle, mode, ci):
    g = golden(f"kernels_{mode}.npz")
    a = case_args(g, mode, ci)
    acc = np.zeros((10, 9, 9, 9), np.int64)
    st = oracle.fused_span(*a["arrs"], a["start"], a["count"], a["E"], a["B"], acc,
                           a["inv"], a["geo_f"], a["geo_g"], a["geo_i"],
                           a["sc"]["dt"], a["sc"]["dth"], a["sc"]["qdt2m"],
                           a["sc"]["beta"], a["sc"]["one"], 3,
                           a["fd"](2.0 ** 43), a["mixed"])
    assert st == int(g[a["pre"] + "fused_status"])
    for n, arr in zip("xyzuvw", a["arrs"]):
        assert np.array_equal(arr, g[a["pre"] + "fused_" + n]), n
    assert np.array_equal(acc, g[a["pre"] + "fused_acc"])


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("ci", [0, 1, 2])
@pytest.mark.parametrize("bc", [0, 1])
def test_oracle_push_matches_reference(oracle, mode, ci, bc):
    g = golden(f"kernels_{mode}.npz")
    a = case_args(g, mode, ci)
    arrs = a["arrs"][:6]
    st = oracle.push_span(*arrs, a["start"], a["count"], a["E"], a["B"], a["geo_f"],
                          a["geo_g"], a["geo_i"], a["sc"]["dt"], a["sc"]["dth"],
                          a["sc"]["qdt2m"], a["sc"]["beta"], a["sc"]["one"], 3, bc,
                          a["mixed"])
    assert st == int(g[a["pre"] + f"push{bc}_status"])
    for n, arr in zip("xyzuvw", arrs):
        assert np.array_equal(arr, g[a["pre"] + f"push{bc}_" + n]), n


@pytest.mark.parametrize("mode", list(MODES))
@pytest.mark.parametrize("ci", [0, 1, 2])
def test_oracle_deposit_and_gather_match_reference(oracle, mode, ci):
    g = golden(f"kernels_{mode}.npz")
    a = case_args(g, mode, ci)
    acc = np.zeros((10, 9, 9, 9), np.int64)
    oracle.deposit_span(*a["arrs"], a["start"], a["count"], acc, a["inv"], a["geo_g"],
                        a["geo_i"], a["fd"](1.0), a["fd"](2.0 ** 43))
    assert np.array_equal(acc, g[a["pre"] + "deposit_acc"])
    out = np.zeros((a["count"], 6), a["pd"])
    oracle.gather_span(a["arrs"][0], a["arrs"][1], a["arrs"][2], a["start"], a["count"],
                       a["E"], a["B"], a["geo_g"], a["geo_i"], a["pd"](1.0), out)
    assert np.array_equal(out, g[a["pre"] + "gather_out"])


def test_oracle_sort_matches_reference(oracle):
    g = golden("sort.npz")
    keys = oracle.cell_keys(g["x"], g["y"], g["z"], (0.0, 0.0, 0.0), (1.0, 1.0, 1.0),
                            (4, 4, 4))
    assert np.array_equal(keys, g["keys"])
    order = oracle.stable_order(keys, 64)
    assert np.array_equal(order, g["ids_after"])
