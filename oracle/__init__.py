"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import anything under oracle/.  Two oracles live here:
  * ref.py      — the reference's own C++ solver (unmodified headers under
                  /root/reference, compiled by oracle/Makefile into
                  oracle/_ref/libtsylv_ref.so), called through ctypes;
  * restate.py  — a numpy restatement of the reference algorithm (recursion,
                  base case, transforms, residual, dense oracle), each
                  function citing the reference file:line it follows.
"""
