"""Reading R18: tests/golden/tau_cfg.json (the oracle's measured score noise per
full-size configuration) is what scripts/measure_tau.py measures (checked on C1,
the configuration the oracle finishes in seconds), and its values sit on the
scale SURVEY App B.3 reports for the explicit-inverse form."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def test_tau_cfg_reproducible_C1():
    import measure_tau

    data = json.load(open(measure_tau.OUT))
    assert data["configs"]["C1"] == json.loads(json.dumps(measure_tau.measure("C1")))


def test_tau_cfg_scale():
    data = json.load(open(os.path.join(ROOT, "tests", "golden", "tau_cfg.json")))["configs"]
    for name in ("C1", "C2", "C3", "C3j", "C4"):
        assert name in data
    # App B.3: ~2e-5 (C1), ~4e-5 (C3 grid), ~6e-8 (C4); 8-d at N = 1e5 is well conditioned
    assert 1e-6 < data["C1"]["tau_cfg"] < 1e-4
    assert 1e-6 < data["C3"]["tau_cfg"] < 1e-4
    assert 1e-9 < data["C4"]["tau_cfg"] < 1e-6
    assert data["C2"]["tau_cfg"] < 1e-6
