"""CTA-0 timeline of the TMEM-P attention (variant .so built with -DKRR_PP_TRACE)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0], "--boost", os.environ.get("BOOST", "1"), "--backends", "tc", "--reps", "1"]
import attn_bench  # noqa
attn_bench.main()
from paper_2504_02921_b200 import _lib
buf = (C.c_ulonglong * (16 * 8 * 64))()
_lib.lib().krr_fa_trace_read(buf)
t = np.array(buf, dtype=np.int64).reshape(16, 8, 64)
t0 = t[t > 0].min()
names = {(2, 4): "M.it", (2, 5): "M.vf", (2, 6): "M.kf", (2, 0): "M.pA", (2, 1): "M.A", (2, 2): "M.pB", (2, 3): "M.B",
         (3, 0): "A.sf", (3, 1): "A.ld", (3, 2): "A.mx", (3, 3): "A.P",
         (4, 0): "B.sf", (4, 1): "B.ld", (4, 2): "B.mx", (4, 3): "B.P"}
for g in range(16):
    row = sorted((t[r, e, g] - t0, n) for (r, e), n in names.items() if t[r, e, g])
    print(f"g={g:2d} " + " ".join(f"{n}@{v}" for v, n in row))
