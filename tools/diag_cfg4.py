import sys, time, torch, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2601_05709_b200 as lsg
from paper_2601_05709_b200 import configs, _lib
from paper_2601_05709_b200.fem import solve_batched, _workspace
for scale in (8, 4, 2, 1):
    c = configs.case("cfg4", scale=scale)
    mesh, model, phi, params = configs.build(c)
    op = model.operator(phi)
    b = model.load_vectors
    t0 = time.time()
    x, it = solve_batched(op, b, rtol=1e-8)
    torch.cuda.synchronize()
    ws = _workspace(op, 1)
    sc = ws.host_scal[0].tolist()
    tr = float(torch.linalg.vector_norm(b[0] - op.apply(x[0])))
    print(scale, mesh.n, "iters", int(it[0]), "time %.2f" % (time.time()-t0), "bnorm %.3e" % float(torch.linalg.vector_norm(b[0])),
          "rec %.3e" % (sc[4] ** 0.5), "true %.3e" % tr, "atol %.3e" % sc[0], "xmax %.3e" % float(x.abs().max()), flush=True)
