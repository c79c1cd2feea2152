"""cProfile of the host side of the device-resident loop (where 'other' time goes)."""
import cProfile, pstats, sys, os, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_05709_b200 import configs
from paper_2601_05709_b200.driver import Optimizer
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
c = configs.case(name)
c = type(c)(**{**c.__dict__, "niter": 8})
mesh, model, phi, params = configs.build(c)
opt = Optimizer(model, phi, params, timing=False)
for _ in range(3):
    opt.step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(4):
    opt.step()
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(45)
print(s.getvalue())
