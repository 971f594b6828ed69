"""Host-side limits of the drop-in API's copies on the GPU box: threaded
memmove bandwidth into a pinned buffer, pinned DMA both ways, and the cost of
registering (page-locking) a caller's array in place.

    python scripts/hostlink_probe.py
"""

import ctypes
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

N = 64 << 20      # bytes per transfer (one staging chunk)


def best(fn, reps=5):
    fn()
    b = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        b = min(b, time.perf_counter() - t0)
    return b


def main():
    src = np.random.default_rng(0).integers(0, 255, 4 * N, dtype=np.uint8)
    pinned = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(N, dtype=torch.uint8, device="cuda")
    pool = ThreadPoolExecutor(32)
    for threads in (1, 2, 4, 8, 16, 32):
        step = N // threads

        def mm():
            fs = [pool.submit(ctypes.memmove, pinned.data_ptr() + i * step, src.ctypes.data + i * step, step)
                  for i in range(threads)]
            for f in fs:
                f.result()
        print(f"memmove host->pinned {threads:2d} threads: {N / best(mm) / 1e9:6.1f} GB/s")
    fresh = lambda: np.empty(N, np.uint8)

    def mm_fresh(threads=16):
        out = fresh()
        step = N // threads
        fs = [pool.submit(ctypes.memmove, out.ctypes.data + i * step, pinned.data_ptr() + i * step, step)
              for i in range(threads)]
        for f in fs:
            f.result()
    print(f"memmove pinned->fresh 16 threads: {N / best(mm_fresh) / 1e9:6.1f} GB/s")

    def h2d():
        dev.copy_(pinned, non_blocking=True)
        torch.cuda.synchronize()

    def d2h():
        pinned.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
    print(f"pinned DMA H2D: {N / best(h2d) / 1e9:6.1f} GB/s   D2H: {N / best(d2h) / 1e9:6.1f} GB/s")
    rt = torch.cuda.cudart()
    arr = np.ones(2 * N, dtype=np.uint8)
    big = torch.empty(2 * N, dtype=torch.uint8, device="cuda")

    def reg():
        t0 = time.perf_counter()
        assert rt.cudaHostRegister(arr.ctypes.data, arr.nbytes, 0) == 0
        t1 = time.perf_counter()
        big.copy_(torch.from_numpy(arr), non_blocking=True)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        assert rt.cudaHostUnregister(arr.ctypes.data) == 0
        t3 = time.perf_counter()
        return t1 - t0, t2 - t1, t3 - t2
    reg()
    r = min((reg() for _ in range(3)), key=sum)
    print(f"cudaHostRegister {2 * N >> 20} MiB: register {r[0] * 1e3:.2f} ms, DMA {r[1] * 1e3:.2f} ms, "
          f"unregister {r[2] * 1e3:.2f} ms -> {2 * N / sum(r) / 1e9:.1f} GB/s overall")


if __name__ == "__main__":
    main()
