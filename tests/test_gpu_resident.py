"""The whole-run resident kernel (k_resident: one cooperative launch per
emrkc_run on small grids) against the per-step kernels: final states and run
records bitwise equal, through clean runs, out-of-range voltages (the
reference-order ionic path), a NumericalAbort (pre-step state kept), a norm
guard (that step's result kept), the progressive variant and EXEX-RL. The
per-step side runs in a subprocess with EMRKC_RESIDENT=0 (read once per
process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _resident_cases as rc  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def per_step(tmp_path_factory):
    out = tmp_path_factory.mktemp("res") / "per_step.npz"
    env = dict(os.environ, EMRKC_RESIDENT="0")
    subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "_resident_cases.py"),
                    str(out)], check=True, env=env, timeout=600)
    return np.load(out)


@pytest.mark.parametrize("name", list(rc.CASES))
def test_resident_matches_per_step(per_step, name):
    assert os.environ.get("EMRKC_RESIDENT", "1") != "0"
    y, rec = rc.run_case(name)
    ref_y = per_step[name + "/y"]
    assert np.array_equal(y, ref_y, equal_nan=True), np.nanmax(np.abs(y - ref_y))
    for k, v in rec.items():
        if k == "device_ms":
            continue
        r = per_step[name + "/" + k]
        assert np.array_equal(np.asarray(v), r, equal_nan=True), (k, v, r)
