import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, meshgen, oracle, paper_1505_07630_b200 as ldu
torch.cuda.set_device(0)
n = int(sys.argv[1])
sys_ = meshgen.hex_laplacian(n, n, n); b = torch.from_numpy(meshgen.rhs_hot_face(n, n, n)).cuda()
with ldu.LduMatrix.from_system(sys_) as A:
    A.dic_setup()
    z = torch.empty_like(b); z2 = torch.empty_like(b)
    t = []
    for _ in range(5):
        A.dic_apply(b, z); t.append(A.stats()["solveMs"])
    os.environ.pop("X", None)
    out = {"n": n, "sf": os.environ.get("LDU_DIC_SF"), "blocks": os.environ.get("LDU_DIC_SF_BLOCKS"), "apply_ms": sorted(t)[:3]}
    if n <= 64:
        _, _, w = oracle.dic(sys_, b.cpu().numpy())
        out["rel"] = float(np.linalg.norm(z.cpu().numpy() - w) / np.linalg.norm(w))
    x = torch.zeros_like(b)
    st, it, res = A.dic_pcg_solve(b, x, tol=1e-8, maxIter=5000)
    out.update(status=st, it=it, ms=A.stats()["solveMs"])
print(json.dumps(out), flush=True)
