import ctypes, time, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2004_02297_b200 import hostio
print(open('/sys/kernel/mm/transparent_hugepage/enabled').read().strip(), open('/sys/kernel/mm/transparent_hugepage/defrag').read().strip())
libc = ctypes.CDLL(None, use_errno=True)
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
dev = torch.empty(75 << 20, dtype=torch.uint8, device='cuda').fill_(3)
def plain():
    return hostio.to_bytes(dev)
orig = hostio._from_device
def with_thp():
    flat = dev.reshape(-1)
    out = hostio._PyBytes_FromStringAndSize(None, flat.numel())
    p = hostio._PyBytes_AsString(out)
    a = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(a, (p + flat.numel() - a) & ~((2 << 20) - 1), 14)
    orig(flat, p)
    return out
def best(f):
    f(); torch.cuda.synchronize(); b = 1e9
    for _ in range(7):
        t = time.perf_counter(); f(); torch.cuda.synchronize(); b = min(b, time.perf_counter() - t)
    return dev.numel() / b / 1e9
for _ in range(2):
    print("plain", round(best(plain), 2), "thp", round(best(with_thp), 2))
def np_plain():
    return np.empty(75 << 20, np.uint8).fill(1)
print("np.empty+fill", round((75 << 20) / (lambda: (lambda t: (np_plain(), time.perf_counter() - t)[1])(time.perf_counter()))() / 1e9, 2))
