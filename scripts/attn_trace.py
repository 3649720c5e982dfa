"""Print the CTA-0 event timeline of the ping-pong attention (variant .so built
with -DKRR_PP_TRACE, selected via KRR_LIB)."""
import ctypes as C, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0], "--boost", os.environ.get("BOOST", "16"), "--backends", "tc", "--reps", "1"]
import attn_bench  # noqa
attn_bench.main()
from paper_2504_02921_b200 import _lib
buf = (C.c_ulonglong * (16 * 8 * 64))()
_lib.lib().krr_pp_trace_read(buf)
t = np.array(buf, dtype=np.int64).reshape(16, 8, 64)
t0 = t[t > 0].min()
names = {(0, 0): "Kp", (1, 0): "Vp", (2, 0): "M.kf", (2, 1): "M.S",
         (2, 4): "M.SA0", (2, 5): "M.SA1", (2, 6): "M.PA0", (2, 7): "M.PA1", (2, 2): "M.vf", (2, 3): "M.PV", (3, 0): "A.sf", (3, 1): "A.ld",
         (3, 2): "A.mx", (3, 3): "A.P", (3, 6): "A.resc", (3, 7): "A.exp", (3, 4): "A.pvL", (3, 5): "A.epi",
         (4, 0): "B.sf", (4, 1): "B.ld", (4, 2): "B.mx", (4, 3): "B.P",
         (4, 4): "B.pvL", (4, 5): "B.epi"}
for g in range(27):
    row = []
    for (r, e), n in names.items():
        v = t[r, e, g]
        if v:
            row.append((v - t0, n))
    row.sort()
    print(f"g={g:2d} " + " ".join(f"{n}@{v}" for v, n in row))
