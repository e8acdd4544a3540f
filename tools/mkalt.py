"""Build a development variant of the library into tools/alt/<name>.so
(separate object directory; the shipped libtsylv_gpu.so is untouched).

    python tools/mkalt.py wprof -DWIDE_PROF=1 -DSMALL_PROF=1 -DTSG_DEVTOOLS
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_09539_b200 import build as B  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
os.environ["TSG_NVCC_FLAGS"] = " ".join(flags)
alt = os.path.join(B.ROOT, "tools", "alt")
B.OBJ = os.path.join(alt, "_build_" + name)
B.LIB = os.path.join(alt, name + ".so")
print(B.build())
