"""The generated-source cache (qsv_tile_jit.cuh jit_pass_source): a pass whose
op / phase arrays match an earlier pass and whose payload facts the generator
read still hold reuses that pass's text.  Checked on CPU by generating the
sources of many circuits that share structure but differ in values --
random angles, exact 0 / +-1 entries, controlled phases, Pauli products --
with the cache on (one process, so later circuits hit it) and off, and
requiring byte-identical sources."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import glob, os, shutil, sys
sys.path.insert(0, os.environ["QSV_TEST_ROOT"])
sys.path.insert(0, os.path.join(os.environ["QSV_TEST_ROOT"], "tests"))
import numpy as np
from paper_2011_13524_b200 import workloads
from test_gpu_tiles import random_circuit, layered_circuit, qft_circuit
dump = os.environ["QSV_JIT_DUMP"]
circs = []
for seed in range(3):
    circs += [workloads.generate_cz_ladder(14, 6, seed=seed), workloads.generate_cnot_ring(13, seed=seed),
              workloads.vqe_ansatz(12, seed=seed), random_circuit(12, 120, seed),
              layered_circuit(12, 5, seed), qft_circuit(13, inverse_bits=seed % 2)]
c = workloads.vqe_ansatz(12)
c.set_parameter(0, 0.0)  # an exact identity rotation
c.set_parameter(1, np.pi)
circs.append(c)
for i, circ in enumerate(circs):
    for L in (8, 11):
        core = circ._core if hasattr(circ, "_core") else circ
        core.plan_stats(jit=1, tile_qubits=L)
        for f in glob.glob(os.path.join(dump, "pass_*.cu")):
            shutil.move(f, f + ".%d_%d" % (i, L))
"""


def _dump(tmp, cache):
    env = dict(os.environ, QSV_JIT_DUMP=str(tmp), QSV_JIT_SRC_CACHE=cache,
               QSV_TILE_VARIANT="4", QSV_TEST_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    out = {}
    for name in os.listdir(tmp):
        with open(os.path.join(tmp, name)) as fh:
            out[name] = fh.read()
    return out


def test_cached_sources_equal_fresh_sources(tmp_path):
    on, off = tmp_path / "on", tmp_path / "off"
    on.mkdir()
    off.mkdir()
    a, b = _dump(on, "1"), _dump(off, "0")
    assert len(a) > 50 and a.keys() == b.keys()
    for k in a:
        assert a[k] == b[k], k
