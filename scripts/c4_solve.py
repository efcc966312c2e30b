"""C4 test batch (64 samples, 128^2 pin cell, CL(16,8)): one SI-DSA solve to
1e-8 with the DSA inner tolerance tied to the stop test (for launch lists).
python scripts/c4_solve.py [dsa_inner] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2402_10488_b200 import configs, rte
inner = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
_, test = configs.c4_params(40, 64)
b = rte.TransportBatch(configs.pin_cell(rte)(128), rte.Mesh.rect_uniform(0, 1, 128, 0, 1, 128),
                       rte.chebyshev_legendre(16, 8), test)
rte.DsaOperator(b)
cfg = rte.SolveConfig(eps_sisa=1e-8, norm="abs", max_iters=500, dsa_inner=inner)
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rho, r = rte.sisa_solve(b, "DSA", cfg)
    e1.record()
    torch.cuda.synchronize()
    print("C4 SI-DSA: %.1f ms (%.3f ms/sample), mean iterations %.2f" %
          (e0.elapsed_time(e1), e0.elapsed_time(e1) / len(test), np.mean([x.iterations for x in r])), flush=True)
