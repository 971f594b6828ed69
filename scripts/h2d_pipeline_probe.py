"""A/B of the CPU-master pipeline's scheduling (HostWeightSync): packer threads
x copy batch size x whether the calling thread also packs
(ADT_H2D_CALLER_PACKS; read once per process, so each value runs in a child).
Wall clock per transfer (launch + 16-B read-back + sync), median of 30.

    python scripts/h2d_pipeline_probe.py
"""

import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import numpy as np
    import torch

    from paper_2004_02297_b200 import hostsync, workloads
    from paper_2004_02297_b200.codec import bits_to_round_to
    from paper_2004_02297_b200.precision import FixedPrecision

    rng = np.random.default_rng(0)
    s = torch.cuda.current_stream()
    cp = os.environ.get("ADT_H2D_CALLER_PACKS", "1")
    for name, bits in (("alexnet", None), ("vgg16", 8)):
        counts = workloads.counts_of(name)
        rs = [bits_to_round_to(b) for b in workloads.default_bits(name, bits)]
        pinned = []
        for n in counts:
            t = torch.empty(n, dtype=torch.float32, pin_memory=True)
            t.numpy()[:] = rng.standard_normal(n, dtype=np.float32) * np.float32(0.1)
            pinned.append(t.numpy())

        class Fixed(FixedPrecision):
            def round_tos(self):
                return list(rs)

        for batch in tuple(int(x) << 10 for x in os.environ.get("PROBE_BATCH_KB", "256,1024,4096").split(",")):
            sync = hostsync.HostWeightSync(pinned, Fixed(len(counts), 32), min_copy_bytes=batch)
            tail = torch.empty(4, dtype=torch.float32, pin_memory=True)
            for th in (6, 8, 12, 16):
                sync.threads = th

                def one():
                    sync.launch(fused_norm=True)
                    tail.copy_(sync.replicas[-1][-4:], non_blocking=True)
                    s.synchronize()

                for _ in range(4):
                    one()
                ts = []
                for _ in range(30):
                    t0 = time.perf_counter()
                    one()
                    ts.append(time.perf_counter() - t0)
                print(f"{name:8s} caller_packs={cp} batch {batch >> 10:5d} KiB threads {th:2d}: "
                      f"{np.median(ts) * 1e3:7.3f} ms (min {np.min(ts) * 1e3:7.3f})", flush=True)
            del sync


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
        return
    for cp in os.environ.get("PROBE_CALLER", "1,0").split(","):
        subprocess.run([sys.executable, os.path.abspath(__file__), "child"],
                       env=dict(os.environ, ADT_H2D_CALLER_PACKS=cp), check=False)


if __name__ == "__main__":
    main()
