"""Debug: run one launch on a -DBSFA_WATCHDOG_RECORD=1 build and print the waits that timed out.

    BSFA_LIB_PATH=.../libbsfa_b200_wdrec.so python tools/stuck_probe.py [one_launch args]
Each record: (cta, warp, parity, shared barrier offset).
"""
import ctypes
import os
import runpy
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_07011_b200 import _lib  # noqa: E402

sys.argv = ["one_launch.py"] + sys.argv[1:]
try:
    runpy.run_path(os.path.join(os.path.dirname(__file__), "one_launch.py"), run_name="__main__")
except Exception as e:  # noqa: BLE001
    print("launch error:", e)
torch.cuda.synchronize()
lib = _lib.load_library()
buf = (ctypes.c_ulonglong * 64)()
n = lib.bsfa_debug_stuck(buf, 64)
print("stuck waits:", n)
for i in range(min(n, 64)):
    r = buf[i]
    print(f"  cta {r >> 32} warp {(r >> 24) & 0xff} parity {(r >> 23) & 1} bar 0x{r & 0x3fffff:x}")
