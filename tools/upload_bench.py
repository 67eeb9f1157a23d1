"""Host <-> device matrix transfer rates through the public API (plain
pageable numpy arrays): DeviceMatrix.from_host / to_dense."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2104_10785_b200 as K  # noqa: E402
from paper_2104_10785_b200 import _lib  # noqa: E402

ctx = _lib.get_context()
for rows, cols, dt in ((2000, 1000, np.float64), (20000, 5000, np.float64),
                       (100000, 10000, np.float64), (200000, 20000, np.float32)):
    A = np.ones((rows, cols), dtype=dt)
    ups, downs = [], []
    for rep in range(4):
        t0 = time.perf_counter()
        dm = K.DeviceMatrix.from_host(A)
        ctx.sync()
        t1 = time.perf_counter()
        B = dm.to_dense()
        t2 = time.perf_counter()
        dm.free()
        if rep:
            ups.append(t1 - t0)
            downs.append(t2 - t1)
    gb = A.nbytes / 1e9
    print(f"{rows}x{cols} {np.dtype(dt).name} ({gb:.2f} GB): upload {gb / np.median(ups):6.1f} GB/s "
          f"({1e3 * np.median(ups):.2f} ms), download {gb / np.median(downs):6.1f} GB/s "
          f"({1e3 * np.median(downs):.2f} ms)", flush=True)
