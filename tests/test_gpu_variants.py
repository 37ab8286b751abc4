"""Every run-time selectable K1 / schedule variant against the oracle (B200 only).

The switches are read once per process, so each variant runs
tests/variant_check.py in its own process: config 1 against the reference's
golden output (fp64 bit for bit), a mid-size SBM at d = 80 (fp64 bit-exact), a
59999-entry hub row (split rows, <= 1e-13 / fp32 gate) and a power-law graph.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

VARIANTS = {
    "default": {},
    # index / value batches in shared memory for fp64 too (the fp32 default)
    "staged_batches_both_dtypes": {"CSEMB_K1_TMA": "3"},
    # register batches + shuffles for fp32 too (the fp64 default)
    "register_batches_both_dtypes": {"CSEMB_K1_TMA": "0"},
    # heavy-row chunks cut at column windows (tiny, so the test matrices get several)
    "heavy_windows": {"CSEMB_HEAVY_WINDOW_MB": "0.5"},
    # hot heavy rows swept in tiny column windows
    "hot_rows": {"CSEMB_HOT_ROWS": "8", "CSEMB_HOT_WINDOW": "64"},
}


@pytest.mark.parametrize("name", list(VARIANTS))
def test_variant_matches_oracle(name, gpu_lib):
    env = dict(os.environ)
    for k in ("CSEMB_K1_TMA", "CSEMB_HEAVY_WINDOW_MB", "CSEMB_HOT_ROWS", "CSEMB_HOT_WINDOW"):
        env.pop(k, None)
    env.update(VARIANTS[name])
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "variant_check.py")], env=env,
                         capture_output=True, text=True, timeout=900)
    assert res.returncode == 0 and "VARIANT_OK" in res.stdout, (name, res.stdout[-2000:], res.stderr[-4000:])
