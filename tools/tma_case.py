import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import oracle.ref as R, paper_1905_09539_b200 as T
for dims, nmin in [((8,3,8),1), ((8,3,8),2), ((8,4,8),1), ((8,8,8),1), ((16,6,16),2), ((16,16,16),2), ((16,16,16),4)]:
    rs = R.RandomStream(1001)
    t, b = rs.reduced_laplace(list(dims))
    try:
        x = T.laplace_recursive(t, b, nmin)
        print(dims, nmin, "ok", np.linalg.norm(x - R.laplace_recursive(t, b, 2)) / np.linalg.norm(x))
    except Exception as e:
        print(dims, nmin, "FAIL", str(e)[:100]); break
