"""hostio.to_device / to_bytes throughput over staging chunk size and copy
threads (AlexNet fc6, 151 MB FP32 / 75 MB packed at r=2).

    python scripts/hostio_sweep.py
"""

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2004_02297_b200 import hostio


def best(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    b = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        b = min(b, time.perf_counter() - t0)
    return b


def main():
    host = np.random.default_rng(1).standard_normal(37748736, dtype=np.float32)
    dev_u8 = torch.empty(host.nbytes // 2, dtype=torch.uint8, device="cuda").fill_(7)
    for chunk_mb in (8, 16, 32, 64):
        for threads in (4, 8, 16):
            hostio.CHUNK, hostio.THREADS = chunk_mb << 20, threads
            hostio._staging.clear()
            h2d = host.nbytes / best(lambda: hostio.to_device(host)) / 1e9
            d2h = dev_u8.numel() / best(lambda: hostio.to_bytes(dev_u8)) / 1e9
            print(f"chunk {chunk_mb:3d} MiB threads {threads:2d}: to_device {h2d:6.1f} GB/s  to_bytes {d2h:6.1f} GB/s")


if __name__ == "__main__":
    main()
