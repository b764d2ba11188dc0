"""Every tuning key documented in include/qrb200.h is readable, and the writable
ones accept their current value back (qrb_set_tuning / qrb_get_tuning)."""

import re
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HEADER = Path(__file__).resolve().parent.parent / "include" / "qrb200.h"


def _documented_keys():
    text = HEADER.read_text()
    block = text[text.index("Process-wide tuning knobs"):text.index("QRB_API int qrb_set_tuning")]
    keys, read_only = [], set()
    for line in block.splitlines():
        for m in re.finditer(r'"([a-z0-9_]+)"', line):
            if m.group(1) not in keys:
                keys.append(m.group(1))
            if "(read only)" in line:
                read_only.add(m.group(1))
    return keys, read_only


def test_documented_tuning_keys_round_trip():
    from paper_1907_01891_b200 import _native
    from paper_1907_01891_b200.errors import GpuError

    _native.load()
    keys, read_only = _documented_keys()
    assert {"panel_algo", "lookahead", "la_sms", "la_sms_max", "sf_diag", "few_tiles_bn32",
            "gram_min_rows", "sm_count"} <= set(keys)
    for k in keys:
        v = _native.get_tuning(k)
        if k in read_only:
            with pytest.raises(GpuError):
                _native.set_tuning(k, v)
        else:
            _native.set_tuning(k, v)
            assert _native.get_tuning(k) == v, k
    with pytest.raises(GpuError):
        _native.set_tuning("no_such_knob", 1)
