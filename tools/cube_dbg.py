"""One solve through a plan (host buffers: `host`, or the streaming entry
point: `stream`) for a given shape, printing the time: used under `timeout`
to probe the overlap machinery for hangs, e.g.
  TSG_LAP16=1 TSG_CUBE=2 TSG_CUBE_GRID=4 timeout 30 python tools/cube_dbg.py host 144,136,128
(development)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1905_09539_b200 as T
from paper_1905_09539_b200.plan import Context, Plan
step = sys.argv[1]
dims = tuple(int(v) for v in sys.argv[2].split(","))
p = T.make_problem(2, dims, seed=12)
fs = [T.schur(a) for a in p.coeffs]
pl = Plan(Context(0), 0, [f[1] for f in fs], [f[0] for f in fs])
b = np.asfortranarray(np.random.default_rng(5).standard_normal(dims))
x = np.zeros_like(b)
t = time.time()
if step == "host":
    pl.execute_host(b, x)
elif step == "stream":
    pl.execute_stream([b.ctypes.data], [x.ctypes.data])
print(step, dims, "ok", time.time() - t, flush=True)
