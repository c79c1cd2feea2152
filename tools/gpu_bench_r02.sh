# Round-2 bench line (driver window) + calibration of the reference arm's counts
cd $GRAFT_REPO_ROOT
O=gpurun_out
python tools/calibrate.py cfg1 cfg3 cfg2 cfg5 > $O/r02_calibration.json 2> $O/calibrate.err; echo "calibrate rc=$?"
python bench.py --warmup 5 --steps 20 > $O/bench_w5k20.json 2> $O/bench_w5k20.err; echo "bench rc=$?"
cp $O/r02_calibration.json profiles/r02_calibration.json 2>/dev/null
python bench.py --impl reference --warmup 1 --steps 2 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
LSG_GRAPH_DEBUG=1 python -c "
import sys, ctypes; sys.path.insert(0, '.')
import torch
from paper_2601_05709_b200 import configs, _lib
from paper_2601_05709_b200.driver import Optimizer
c = configs.case('cfg5'); c = type(c)(**{**c.__dict__, 'niter': 4})
mesh, model, phi, params = configs.build(c)
opt = Optimizer(model, phi, params, timing=False)
lib = _lib.load()
for i in range(4):
    opt.step(); torch.cuda.synchronize()
    out = (ctypes.c_double * 4)(); lib.lsg_graph_stats(out); print('after it', i, list(out), flush=True)
" > $O/graph_debug.log 2>&1; echo "graphdbg rc=$?"
