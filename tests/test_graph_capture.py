"""Device-resident plans under CUDA graph capture: `mcb_plan_launch` only
enqueues kernels (family kernels, the specialised / interpreted program
kernels and the ordered combine) on the caller's stream — no allocation, no
synchronisation — so a relaunch loop can be captured once and replayed.  The
replayed results are byte-identical to eager launches."""
import pytest


@pytest.mark.gpu
def test_plan_launch_captured_in_a_cuda_graph(gpu):
    import torch
    from paper_2104_10073_b200 import workloads
    fns, seed, trials = workloads.c5(samples=300_000, n_fns=24)
    prog = gpu.Program("exp(-20*((x1-c)^2+(x2-c)^2)) + cos(k*(x1+x2)) + sin(k*(x1+x2))", 2, ["c", "k"])
    fns = list(fns) + [prog.integrand({"c": 0.3, "k": 7.0}, n_samples=200_000, index=24),
                       gpu.stratify(gpu.harmonic(9.0, 4, unit_coeffs=True, n_samples=1_000_000, index=25))]
    plan = gpu.Plan(fns, seed, trials)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        plan.launch(stream.cuda_stream)  # eager (also loads every kernel before capture)
    stream.synchronize()
    eager = plan.download(stream.cuda_stream)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        plan.launch(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    replayed = plan.download(stream.cuda_stream)
    plan.close()
    assert replayed.tobytes() == eager.tobytes()
    assert (eager["status"] == gpu.TRIAL_OK).all()
