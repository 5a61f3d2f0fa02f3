#!/usr/bin/env python
"""Small end-to-end exercise of every kernel family (direct, stratified
grid + warp tiles, tree cell lists, interpreter incl. warp tiles) for
compute-sanitizer runs:  compute-sanitizer --tool memcheck python tools/sanitize_smoke.py"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_10073_b200 as mcb  # noqa: E402

prog = mcb.Program("exp(-a*((x1-0.5)^2+(x2-0.5)^2)) + sin(x1)*cos(x2)", 2, ["a"])
fns = [
    mcb.harmonic(53 / (2 * math.pi), 4, unit_coeffs=True, n_samples=200_000, index=0),
    mcb.stratify(mcb.harmonic(3.0, 3, a=0.5, b=2.0, n_samples=100_000, index=1)),
    mcb.stratify(mcb.make_integrand(mcb.FAMILY_ABS3, 3, n_samples=70_000, index=2), cells_per_dim=2),
    mcb.tree(mcb.make_integrand(mcb.FAMILY_HARMONIC_VEC, 2, k=[3.0, -2.0], a=1.0, b=0.5, n_samples=50_000,
                                index=3), samples_per_cell=300),
    prog.integrand({"a": 30.0}, n_samples=80_000, index=4),
    mcb.stratify(prog.integrand({"a": 30.0}, n_samples=80_000, index=5)),
    mcb.tree(prog.integrand({"a": 100.0}, n_samples=60_000, index=6), samples_per_cell=512),
    mcb.stratify(mcb.harmonic(1.0, 2, n_samples=300_000, index=7), cells_per_dim=2),  # big cells: CTA tiles
]
out = mcb.run_direct(fns, 11, 3)
assert (out["status"] == mcb.TRIAL_OK).all(), out["status"]
st, leaves = mcb.tree_refine(fns[6], 11, 0, 0, leaves=True)
print("ok", len(leaves), float(out["value"][0, 0]))
