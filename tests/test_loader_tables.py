"""CPU pin of the bit-exact loader's constants (csrc/bp_ziggurat_tables.h,
csrc/bp_init.cu): the committed ziggurat tables and the Philox4x64-10 /
next_double restatement reproduce numpy's Generator(Philox(key=[seed,
species])) draws — random() and standard_normal(), the reference loader's
streams (pkg/src/batchpic/particles.py:173-241) — bit for bit."""

import os
import re

import numpy as np

from conftest import ROOT

HDR = os.path.join(ROOT, "paper_2008_04397_b200", "csrc", "bp_ziggurat_tables.h")


def _tables():
    text = open(HDR).read()

    def body(name):
        return text.split(name + "[256] = {")[1].split("};")[0]

    ki = [int(v, 16) for v in re.findall(r"0x([0-9a-f]+)ULL", body("kKi"))]
    wi = [float.fromhex(v) for v in re.findall(r"(-?0x[0-9a-f.p+-]+)", body("kWi"))]
    fi = [float.fromhex(v) for v in re.findall(r"(-?0x[0-9a-f.p+-]+)", body("kFi"))]
    assert len(ki) == len(wi) == len(fi) == 256
    return ki, wi, fi


def test_tables_reproduce_numpy_standard_normal():
    import sys
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import gen_ziggurat_tables as G
    ki, wi, fi = _tables()
    key = [12345, 2]
    g = np.random.Generator(np.random.Philox(key=np.array(key, dtype=np.uint64)))
    ref_u = g.random(1000)
    ref_n = g.standard_normal(30000)
    got_u = [(G.philox([m // 4 + 1, 0, 0, 0], key)[m % 4] >> 11) * (1.0 / 9007199254740992.0)
             for m in range(1000)]
    assert np.array_equal(ref_u, np.array(got_u))
    got_n, paths = G.normals(key, 1000, 30000, ki, wi, fi)
    assert np.array_equal(ref_n, got_n)
    assert paths[1] > 0  # the wedge path was exercised
