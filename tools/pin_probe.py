"""Host->device transfer probe: pinned DMA rate, cudaHostRegister cost per
chunk, and register+DMA+unregister of a pageable numpy array in chunks."""
import ctypes as C
import time

import numpy as np
import torch

cudart = C.CDLL("libcudart.so.12") if False else None
try:
    cudart = C.CDLL("libcudart.so")
except OSError:
    import glob
    cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    cudart = C.CDLL(cands[0])
cudart.cudaHostRegister.argtypes = [C.c_void_p, C.c_size_t, C.c_uint]
cudart.cudaHostUnregister.argtypes = [C.c_void_p]
cudart.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
cudart.cudaDeviceSynchronize.argtypes = []

GB = 16
A = np.ones(GB * (1 << 30) // 8)
dev = torch.empty(A.size, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
# pinned DMA rate
pin = torch.empty(1 << 27, dtype=torch.float64).pin_memory()  # 1 GB
for _ in range(2):
    t0 = time.perf_counter()
    for k in range(8):
        dev[k * (1 << 27):(k + 1) * (1 << 27)].copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
print(f"pinned 1 GB buffer -> device x8: {8 / t:.1f} GB/s", flush=True)
for chunk_mb in (64, 256, 1024):
    cb = chunk_mb << 20
    nchunk = A.nbytes // cb
    base = A.ctypes.data
    treg = tcp = tun = 0.0
    t0 = time.perf_counter()
    for k in range(nchunk):
        a = time.perf_counter()
        r = cudart.cudaHostRegister(base + k * cb, cb, 0)
        b = time.perf_counter()
        r2 = cudart.cudaMemcpyAsync(dev.data_ptr() + k * cb, base + k * cb, cb, 1, None)
        cudart.cudaDeviceSynchronize()
        c = time.perf_counter()
        cudart.cudaHostUnregister(base + k * cb)
        d = time.perf_counter()
        treg += b - a; tcp += c - b; tun += d - c
        assert r == 0 and r2 == 0, (r, r2)
    tt = time.perf_counter() - t0
    gb = nchunk * cb / 1e9
    print(f"chunk {chunk_mb} MB: register {gb / treg:.1f} GB/s, dma {gb / tcp:.1f} GB/s, "
          f"unregister {gb / tun:.1f} GB/s, serial total {gb / tt:.1f} GB/s", flush=True)
