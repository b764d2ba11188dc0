"""Test configuration: the `gpu` marker and shared fixtures.

CPU tests (`-m "not gpu"`) cover the oracle against the reference's golden
vectors, the host-side drop-in logic (tile store, config, API checks), the
multi-rank driver over gloo and the C-ABI symbol table.  GPU tests (`-m gpu`)
are the parity tests proper: the sm_100a library against the oracle / golden
fixtures through the C ABI.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built libqrb200.so")


@pytest.fixture(scope="session")
def golden():
    def load(name):
        with np.load(GOLDEN / name, allow_pickle=False) as z:
            return {k: z[k] for k in z.files}
    return load


def sign_normalise(r):
    s = np.sign(np.diag(r)).astype(np.float64)
    s[s == 0] = 1.0
    return r * s[:, None]


def rel_err(got, ref):
    den = np.abs(ref).max()
    return float(np.abs(got - ref).max() / (den if den > 0 else 1.0))
