"""Programmatic dependent launch changes scheduling only, never results: a 2-layer BERT-style
stack (dropout on, forward + backward) gives bit-identical outputs and gradients with PDL on
(default) and off (SMPK_PDL=0), and across processes.  Each run is a subprocess
(tests/pdl_probe.py) because the switch is read once per process."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _digest(**env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, os.path.join(HERE, "pdl_probe.py")], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip().splitlines()[-1]


def test_pdl_on_off_bit_identical():
    on = _digest(SMPK_PDL="1")
    off = _digest(SMPK_PDL="0")
    again = _digest(SMPK_PDL="1")
    assert on == again, "run-to-run nondeterminism"
    assert on == off, "programmatic dependent launch changed the results"
