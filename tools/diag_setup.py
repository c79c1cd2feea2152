"""Host-side setup cost of a config's run (mesh, model, level set) vs its first iterations."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cProfile, pstats
import torch
import paper_2601_05709_b200 as lsg
from paper_2601_05709_b200 import configs
from paper_2601_05709_b200.driver import Optimizer
name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
c = configs.case(name)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
mesh, model, phi, params = configs.build(c)
torch.cuda.synchronize()
pr.disable()
t1 = time.perf_counter()
print("build s", t1 - t0, flush=True)
pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
opt = Optimizer(model, phi, params, timing=False)
for i in range(3):
    t = time.perf_counter(); r = opt.step(); torch.cuda.synchronize()
    print("step", i, time.perf_counter() - t, sum(r.cg_iters), flush=True)
