"""Debug: per-level operator parity (3D time-constant) for the fast and generic kernels."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import test_gpu_parity as T
for fast in ("0", "1"):
    os.environ["ST_NO_FAST"] = fast
    for args in [(3, 8, 8, True), (3, 4, 8, False), (3, 8, 8, False)]:
        try:
            T.test_coarse_operators(*args)
            print("fast" if fast == "0" else "generic", args, "OK", flush=True)
        except AssertionError as e:
            print("fast" if fast == "0" else "generic", args, "FAIL", str(e)[:160], flush=True)
