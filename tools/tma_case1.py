import sys, numpy as np
sys.path.insert(0, "/root/repo")
import oracle.ref as R, paper_1905_09539_b200 as T
rs = R.RandomStream(1001)
t, b = rs.reduced_laplace([8, 3, 8])
x = T.laplace_recursive(t, b, 1)
print("ok")
