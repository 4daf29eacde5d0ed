"""One AMG-PCG solve at n^3 (after a setup) -- the command profiled by scripts/gpu_amg_ncu.sh."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
s = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
A = ldu.LduMatrix.from_system(s)
b = torch.from_numpy(s.b).cuda()
A.amg_setup()
x = torch.zeros_like(b)
st, it, res = A.amg_pcg_solve(b, x, tol=1e-8, maxIter=500, batch=4)
torch.cuda.synchronize()
print(st, it, res, A.stats()["solveMs"])
