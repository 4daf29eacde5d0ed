"""AMG setup phase trace at n^3 (LDU_AMG_TRACE=1 prints per-phase times on stderr).
    python scripts/amg_setup_trace.py [n=256]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
s = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
A = ldu.LduMatrix.from_system(s)
b = torch.from_numpy(s.b).cuda()
for rep in range(int(os.environ.get('REPS', '3'))):
    t = time.time()
    info = A.amg_setup()
    torch.cuda.synchronize()
    print(f"setup {rep}: {info['setupMs']:.1f} ms device, {1e3 * (time.time() - t):.1f} ms wall, "
          f"levels {info['n']}", file=sys.stderr, flush=True)
x = torch.zeros_like(b)
st, it, res = A.amg_pcg_solve(b, x, tol=1e-8, maxIter=500)
print(f"amg_pcg: {st} {it} {res:.3e} solve {A.stats()['solveMs']:.1f} ms", file=sys.stderr)
