"""C5 solve cut to two restart cycles (max_restarts=2): runs the fused
restart pass (correction + U_new, k_tsmm) twice. For ncu: -k regex:k_tsmm."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_14206_b200 as sk  # noqa: E402

ctx = sk.default_context()
A = sk.SparseMatrix.convdiff3d_device(512, 200.0, 100.0, 50.0, ctx=ctx)
N = A.rows
b = torch.from_numpy(sk.gaussian_vector(N, 3)).cuda()
S = sk.SketchOperator.sparse_sign(N, 120, 0x5EED, 8, ctx=ctx)
r = sk.solve(A, b, sk.SolverConfig(m=50, k=10, t=2, s=120, tol=1e-7, max_restarts=2), sketch=S)
print(r.report.status, r.report.iterations, r.report.cycles)
