"""KLRM ingestion throughput: streamed device reader vs host read_matrix +
DeviceMatrix.from_host (the reference-shaped path), both from the page
cache.  Prints one JSON line."""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np

import paper_2104_10785_b200 as K
from paper_2104_10785_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=200_000)
ap.add_argument("--n", type=int, default=2_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--path", default="/tmp/ksvd_io_bench.klrm")
a = ap.parse_args()

op = synth.generate(synth.GenSpec(m=a.m, n=a.n, rank=50, seed=1, spectrum="harmonic", s0=1.0))
K.write_matrix_device(a.path, op)  # also exercises the device writer
nbytes = os.path.getsize(a.path)
res = {"m": a.m, "n": a.n, "file_bytes": nbytes}


def best(fn):
    ts = []
    for _ in range(a.reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return min(ts)


t = best(lambda: K.read_matrix_device(a.path))
res["stream_f64_GBps"] = nbytes / t / 1e9
t = best(lambda: K.read_matrix_device(a.path, dtype=np.float32))
res["stream_f32_GBps"] = nbytes / t / 1e9
t = best(lambda: K.DeviceMatrix.from_host(K.read_matrix(a.path)))
res["host_read_then_upload_GBps"] = nbytes / t / 1e9
t = best(lambda: K.write_matrix_device(a.path + ".out", op))
res["device_write_GBps"] = nbytes / t / 1e9
same = K.read_matrix_device(a.path).to_dense()[:1000]
res["bit_exact_head"] = bool(np.array_equal(same, op.to_dense()[:1000]))
print(json.dumps(res))
os.remove(a.path)
os.remove(a.path + ".out")
