"""Timing of the cfg4 shape evaluation (model.cost) pieces: host vs device."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_05709_b200 import configs, FemField
c = configs.case("cfg4")
mesh, model, phi, _ = configs.build(c)
x = torch.randn(model.space.dof_count, dtype=torch.float64, device="cuda")
for rep in range(3):
    st = FemField(model.space, x.clone())
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    J = model.cost(phi, [st])
    e1.record(); torch.cuda.synchronize()
    print(rep, "host ms", (time.perf_counter() - t0) * 1e3, "device ms", e0.elapsed_time(e1), J, flush=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
    st = FemField(model.space, x.clone())
    model.cost(phi, [st]); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=12))
