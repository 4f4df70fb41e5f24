"""The randomised parity sweeps of tools/*_fuzz.py (random shapes, dtypes,
strides, cue sets, trajectory layouts, sampler settings; every case compared
with the oracle) as GPU tests, so that the round-end GPU run repeats them with
fresh seeds each round (small case counts here; the tools take any count)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(tool, n, seed, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", tool), str(n), str(seed)],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout


@pytest.mark.parametrize("seed", [101, 202])
def test_margin_fuzz(seed):
    """K1 + K4 (every work split) on random rows vs the oracle."""
    assert "FAILURES: 0" in _run("margin_fuzz.py", 12, seed)


@pytest.mark.parametrize("seed", [303, 404])
def test_segment_fuzz(seed):
    """K2 + K3 on random cue sets / trajectory layouts vs the oracle."""
    assert "FAILURES: 0" in _run("segment_fuzz.py", 15, seed)


@pytest.mark.parametrize("seed", [505])
def test_sample_fuzz(seed):
    """The sampler (K4 + K5 + K6) on random rows and settings vs the oracle
    (draws within 1e-5 of a CDF edge excepted)."""
    assert "TOTAL mismatches beyond CDF edges: 0" in _run("sample_fuzz.py", 20, seed)
