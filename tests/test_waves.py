"""Jobs larger than one device wave (MCB_WAVE_TILES tiles of partials + tile
table, default 2^29) run as consecutive waves of whole integrands; every
(integrand, trial) depends only on its own tiles, so the results are byte-
identical to a single launch set.  Forced here with a tiny wave."""
import os
import subprocess
import sys

import pytest

_SCRIPT = r'''
import hashlib, sys
sys.path.insert(0, sys.argv[1])
import paper_2104_10073_b200 as mcb
from paper_2104_10073_b200 import workloads
fns = list(workloads.c5(samples=300_000, n_fns=24)[0])
prog = mcb.Program("exp(-20*((x1-c)^2+(x2-c)^2)) + x1*x2", 2, ["c"])
fns.append(prog.integrand({"c": 0.3}, n_samples=500_000, index=24))
fns.append(mcb.stratify(mcb.harmonic(9.0, 4, unit_coeffs=True, n_samples=1_000_000, index=25)))
fns.append(mcb.stratify(mcb.make_integrand(mcb.FAMILY_ABS3, 3, a=1.0, b=1.0, n_samples=200_000, index=26),
                        cells_per_dim=3))
out = mcb.run_direct(fns, 99, 3)
print(hashlib.sha256(out.tobytes()).hexdigest(), int((out["status"] == mcb.TRIAL_OK).sum()))
'''


@pytest.mark.gpu
def test_wave_split_byte_identical(tmp_path):
    script = tmp_path / "waves.py"
    script.write_text(_SCRIPT)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    got = []
    for wave in ("", "700"):
        env = dict(os.environ)
        env.pop("MCB_WAVE_TILES", None)
        if wave:
            env["MCB_WAVE_TILES"] = wave
        r = subprocess.run([sys.executable, str(script), root], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        got.append(r.stdout.split())
    assert got[0] == got[1]
    assert int(got[0][1]) == 27 * 3
