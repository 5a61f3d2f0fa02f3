"""bench.py's roofline inputs and the reference arm's isolation (CPU only).

* The per-sample instruction counts bench.py divides by are those of the
  compiled bench kernel: the hot loop of k_direct<HARMONIC, 4, 11> in
  csrc/_obj/direct_harmonic.o, read with cuobjdump (no GPU needed).
* The reference arm (bench.py --impl reference) loads only oracle/_ref and
  never imports the product package."""
import json
import os
import re
import shutil
import subprocess
import sys
from collections import Counter

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2104_10073_b200", "csrc", "_obj", "direct_harmonic.o")
KERNEL = "_ZN3mcb6detail8k_directILi0ELi4ELi11EEEvPKNS_3dev6FnDescEPKjmPNS2_11TilePartialE"


def _hot_loop_mix(sass: str) -> Counter:
    body = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    back = []
    for a, ins in body:
        t = re.search(r"BRA\s+`?\(?.*?0x([0-9a-f]+)", ins)
        if "BRA" in ins and t and int(t.group(1), 16) < a:
            back.append((a, int(t.group(1), 16)))
    hi, lo = max(back, key=lambda x: x[0] - x[1])
    return Counter(re.sub(r"^@!?U?P\w+\s+", "", ins).split()[0] for a, ins in body if lo <= a <= hi)


@pytest.mark.skipif(not (os.path.exists(OBJ) and shutil.which("cuobjdump")), reason="kernel object not built")
def test_instruction_counts_match_the_compiled_kernel():
    import bench
    sass = subprocess.run(["cuobjdump", "-sass", "-fun", KERNEL, OBJ], capture_output=True, text=True,
                          check=True).stdout
    mix = _hot_loop_mix(sass)
    # one loop iteration = one pair of 4-D samples
    assert mix["IMAD.WIDE.U32"] == 2 * bench.K_DIRECT_WIDE_PER_SAMPLE
    fp64 = sum(v for k, v in mix.items() if k.split(".")[0] in ("DFMA", "DMUL", "DADD"))
    assert fp64 == 2 * bench.K_DIRECT_FP64_PER_SAMPLE
    # and the committed evidence file says the same
    with open(os.path.join(ROOT, "profiles", "r02_k_direct_sass_mix.txt")) as fh:
        txt = fh.read()
    assert re.search(rf"\b{mix['IMAD.WIDE.U32']} IMAD.WIDE.U32", txt)


def _max_wide_loop_mix(sass: str) -> Counter:
    """Mix of the backward-branch loop with the most IMAD.WIDE (the pair loop)."""
    body = []
    for line in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            body.append((int(m.group(1), 16), m.group(2).strip()))
    best = Counter()
    for a, ins in body:
        t = re.search(r"BRA\s+`?\(?.*?0x([0-9a-f]+)", ins)
        if "BRA" in ins and t and int(t.group(1), 16) < a:
            lo = int(t.group(1), 16)
            c = Counter(re.sub(r"^@!?U?P\w+\s+", "", i).split()[0] for x, i in body if lo <= x <= a)
            if c["IMAD.WIDE.U32"] > best["IMAD.WIDE.U32"]:
                best = c
    return best


@pytest.mark.skipif(not (os.path.exists(OBJ) and shutil.which("cuobjdump")), reason="kernel object not built")
def test_config_kernel_mixes_match_the_compiled_kernels():
    """bench.K_DIRECT_PAIR_MIX (the per-config ALU ceilings of C3/C4/C5) is the
    hot-loop mix of each k_direct<family, dim, variant> in the object files."""
    import bench
    objs = {0: "direct_harmonic.o", 2: "direct_abs.o", 3: "direct_abs.o"}
    for (fam, dim, var), (wide, fp64) in bench.K_DIRECT_PAIR_MIX.items():
        name = f"_ZN3mcb6detail8k_directILi{fam}ELi{dim}ELi{var}EEEvPKNS_3dev6FnDescEPKjmPNS2_11TilePartialE"
        obj = os.path.join(ROOT, "paper_2104_10073_b200", "csrc", "_obj", objs[fam])
        sass = subprocess.run(["cuobjdump", "-sass", "-fun", name, obj], capture_output=True, text=True,
                              check=True).stdout
        mix = _max_wide_loop_mix(sass)
        got_fp64 = sum(v for k, v in mix.items() if k.split(".")[0] in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
        assert (mix["IMAD.WIDE.U32"], got_fp64) == (wide, fp64), (fam, dim, var)


def test_config_mix_ceilings():
    import bench
    from paper_2104_10073_b200 import workloads as w
    fns, _, _ = w.c3()
    assert bench.mix_clk_per_warp_sample(fns, lambda f: 0) == pytest.approx((49 * 86 + 51 * 126) / 100)
    fns, _, _ = w.c5(samples=70_000, n_fns=80)
    clk = bench.mix_clk_per_warp_sample(fns, lambda f: 11 if int(f.family) == 0 else 1)
    assert clk == pytest.approx((78 + 114 + 100 + 136 + 172 + 208 + 244 + 280) / 8)


def test_alu_roofline_arithmetic():
    import bench
    r = bench.alu_roofline(1.8e11, 1965.0)
    clk = 34 * 4.0 + 18 * 2.0
    assert r["clk_per_warp_sample"] == clk
    assert r["peak"] == pytest.approx(148 * 4 * 32 * 1.965e9 / clk / 1e9)
    assert r["frac"] == pytest.approx(1.8e11 / (148 * 128 * 1.965e9 / clk))
    assert bench.alu_roofline(1.0, None) is None


def test_strided_sample_spans_the_set():
    import bench
    first, count, stride = bench.strided_sample(50, 0)
    assert (first, count, stride) == (0, 50, 20)
    idx = [first + i * stride for i in range(count)]
    assert idx[-1] >= 950  # reaches the high-k end, not a prefix
    firsts = {bench.strided_sample(50, s)[0] for s in range(20)}
    assert firsts == set(range(20))  # successive steps rotate through the offsets
    assert bench.strided_sample(5000, 0) == (0, 1000, 1)


def test_configs_identical_in_both_arms():
    import bench
    for scaling in ("weak", "strong"):
        args = bench.parse(["--scaling", scaling])
        a = bench.bench_config(args, 8)
        b = bench.bench_config(bench.parse(["--impl", "reference", "--scaling", scaling]), 8)
        assert a == b


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmcbatch_ref.so")),
                    reason="reference library not built")
def test_reference_arm_loads_only_the_reference():
    code = ("import bench, sys, json\n"
            "bench.main(['--impl', 'reference', '--steps', '1', '--warmup', '0', '--samples', '20000',"
            " '--cpu-seconds', '1'])\n"
            "maps = [l.split()[-1] for l in open('/proc/self/maps') if l.rstrip().endswith('.so')]\n"
            "print(json.dumps({'so': sorted(set(maps)), 'mods': sorted(sys.modules)}))\n")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    line, loaded = lines[0], lines[1]
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference"
    assert line["cpu_baseline"]["cpu"]["logical_cpus"] >= 1
    assert not any("libmcb.so" in p for p in loaded["so"]), loaded["so"]
    assert any(p.endswith("oracle/_ref/libmcbatch_ref.so") for p in loaded["so"])
    assert not any(m.startswith("paper_2104_10073_b200") or m.startswith("tests") for m in loaded["mods"])
