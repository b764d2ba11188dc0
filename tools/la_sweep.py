"""Sweep of the look-ahead tuning on one config: python tools/la_sweep.py CFG
'la_sms=16,la_lat_us=450' 'la_sms=8' ...  (each spec applied on top of the
defaults; 'off' = lookahead 0).  Best of 2 factorizations after a warm-up."""
import sys

sys.path.insert(0, ".")
from paper_1907_01891_b200 import _native, ct_system as cs  # noqa: E402
from paper_1907_01891_b200.device import QrDevice  # noqa: E402

cfg = int(sys.argv[1])
g = cs.config_geometry(cfg)
m, n = g.n_rays, g.n_pixels
a = cs.densify_device(g, (m + 31) // 32 * 32)
fl = 2.0 * m * n * n - 2.0 * n ** 3 / 3.0
q = QrDevice(m, n)
defaults = {k: _native.get_tuning(k) for k in ("lookahead", "la_sms", "la_lat_us", "la_margin_pct",
                                               "outer_panels", "outer4_min_cols", "tn_tail")}
for spec in sys.argv[2:]:
    for k, v in defaults.items():
        _native.set_tuning(k, v)
    if spec == "off":
        _native.set_tuning("lookahead", 0)
    else:
        for kv in spec.split(","):
            k, v = kv.split("=")
            _native.set_tuning(k, int(v))
    best = 0.0
    for it in range(3):
        q.set_matrix_device(a)
        s0 = _native.get_tuning("la_steps")
        rep = q.factorize()
        if it:
            best = max(best, fl / rep["total_ms"] / 1e9)
    print(f"config {cfg} {spec:32s} {best:.3f} TFLOP/s  la_steps {_native.get_tuning('la_steps') - s0}",
          flush=True)
