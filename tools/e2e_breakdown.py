#!/usr/bin/env python
"""Where the end-to-end C-ABI call's time goes beyond the kernels (C2):
mcb_run_direct wall time vs the device-resident plan's launch (CUDA events),
with MCB_TREE_TRACE=1 printing the host-plan build time of each call."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2104_10073_b200 as mcb
    from paper_2104_10073_b200 import workloads
    fns, seed, trials = workloads.c2()
    arr = mcb.as_array(fns)
    s = torch.cuda.current_stream()
    plan = mcb.Plan(arr, seed, trials)
    for _ in range(3):
        plan.launch(s.cuda_stream)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ks = []
    for _ in range(5):
        a.record(s)
        plan.launch(s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        ks.append(a.elapsed_time(b))
    plan.close()
    es = []
    for i in range(8):
        t0 = time.perf_counter()
        mcb.run_direct(arr, seed, trials, devices=[0])
        es.append(1e3 * (time.perf_counter() - t0))
    print(f"plan launch (kernels): min {min(ks):.3f} ms; mcb_run_direct wall: min {min(es[2:]):.3f} ms "
          f"median {sorted(es[2:])[len(es[2:]) // 2]:.3f} ms; overhead {min(es[2:]) - min(ks):.3f} ms")


if __name__ == "__main__":
    main()
