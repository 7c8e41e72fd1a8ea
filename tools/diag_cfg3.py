"""Diagnose fast-vs-oracle point failures on a cfg3 class (GPU box)."""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle'); sys.path.insert(0, 'tests')
import numpy as np, torch, oracle as O, parity
from paper_2105_12415_b200 import device as D, workloads as W
N = 1 << 15
cls = int(sys.argv[1]) if len(sys.argv) > 1 else 1
dt = np.float32
A, B = W.adversarial_pairs(N, seed=3)
sl = slice(cls * N, (cls + 1) * N)
A = A[sl].astype(dt); B = B[sl].astype(dt)
pk = dict(n_iterative=16, epsilon=1e-6)
o = D.run("hybrid", torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), D.Params(**pk), strict=False, ids=True)
torch.cuda.synchronize()
got = {k: v.cpu().numpy() for k, v in o.items()}
p = O.make_params(**pk)
eps = np.full(N, 1e-6, dt)
ref, _, _ = O.hybrid(A, B, p, eps, dtype=dt, threads=16)
L = parity.longest_edge(A, B)
pe = np.maximum(parity.rel_err(got["point_a"], ref["point_a"], L), parity.rel_err(got["point_b"], ref["point_b"], L))
for i in np.argsort(-pe)[:4]:
    print(i, "p_err %.3e" % pe[i], "d_err %.3e" % parity.rel_err(got["distance"][i:i+1], ref["distance"][i:i+1], L[i:i+1])[0],
          "ids got", got["ids"][i], "ref", ref["ids"][i], "kind", got["kind"][i], ref["kind"][i], "L", L[i])
    print("   pa got", got["point_a"][i], "ref", ref["point_a"][i])
    print("   pb got", got["point_b"][i], "ref", ref["point_b"][i], "dist", got["distance"][i], ref["distance"][i])
    base = {k: ref[k][i:i+1] for k in ref}
    for reps in (2, 8):
        s = parity.point_sensitivity(O, lambda a, b: O.hybrid(a, b, p, eps[i:i+1], dtype=dt)[0], A[i:i+1], B[i:i+1], dt, base, reps=reps)
        print("   sensitivity reps", reps, s)
