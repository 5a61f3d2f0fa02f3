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
    mcb.harmonic(40.0, 4, unit_coeffs=True, n_samples=200_001, index=8),  # odd count: the tail sample
    mcb.stratify(mcb.harmonic(9.0, 4, unit_coeffs=True, n_samples=1_000_000, index=9)),  # 8^4 cells: lane per cell
]
prog4 = mcb.Program("cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4, ["k"])
fns.append(mcb.stratify(prog4.integrand({"k": 9.0}, n_samples=1_000_000, index=10)))  # program lane kernel
out = mcb.run_direct(fns, 11, 3)
assert (out["status"] == mcb.TRIAL_OK).all(), out["status"]
two = mcb.run_direct(fns, 11, 3, devices=[0, 0])  # (integrand, trial) sharding
assert two.tobytes() == out.tobytes()
st, leaves = mcb.tree_refine(fns[6], 11, 0, 0, leaves=True)
pts = mcb.debug_points(11, 4, 0, 0, 0, 1001, [0.0, 0.0], [1.0, 1.0])
vals = prog.evaluate(pts, {"a": 30.0})  # k_program_points, odd point count
assert vals.shape == (1001,)
print("ok", len(leaves), float(out["value"][0, 0]))
