"""lap16 (16^3 TMA kernel) vs the 8^3 kernel on reduced problems."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_09539_b200 as T

def quasi(n, rng, blocks=True):
    t = np.triu(rng.standard_normal((n, n))) / np.sqrt(n)
    t[np.arange(n), np.arange(n)] = 3 + rng.standard_normal(n) * 0.5
    if blocks:
        i = 0
        while i + 1 < n:
            if rng.random() < 0.4:
                a = t[i, i]
                t[i + 1, i + 1] = a
                t[i, i + 1] = abs(t[i, i + 1]) + 0.3
                t[i + 1, i] = -(0.2 + rng.random() * 0.3)
                i += 2
            else:
                i += 1
    return np.asfortranarray(t)

rng = np.random.default_rng(0)
for dims, nm, blocks in [((64, 64, 64), 16, False), ((64, 64, 64), 16, True), ((64, 64, 64), 8, True),
                         ((48, 80, 96), 16, True), ((256, 256, 256), 16, True)]:
    t = [quasi(n, rng, blocks) for n in dims]
    b = np.asfortranarray(rng.standard_normal(dims))
    os.environ["TSG_LAP16"] = "0"
    want = T.laplace_recursive(t, b, nm)
    os.environ["TSG_LAP16"] = "1"
    t0 = time.time()
    got = T.laplace_recursive(t, b, nm)
    err = np.linalg.norm(got - want) / np.linalg.norm(want)
    d = np.abs(got - want).reshape(dims, order="F")
    idx = np.unravel_index(np.argmax(d), dims)
    print(dims, nm, blocks, "rel err %.3e  worst at %s  (%.2fs)" % (err, idx, time.time() - t0), flush=True)
