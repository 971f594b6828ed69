#!/usr/bin/env python
"""Table-2-shaped per-phase profile measured on the B200
for the BASELINE weight sets: transfer.measured_profile over one WeightSync.

    python scripts/table2.py > profiles/r01_table2.md
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import transfer, workloads


def main():
    torch.cuda.set_device(0)
    print("# Table-2-shaped profile on one B200 (transfer.measured_profile)\n")
    print("Per step, device ms. Paper (VGG-A 129.6M weights, x86 + K80): CPU->GPU FP32 153.93 -> "
          "A2DTWP 52.27 ms, Bitpack 19.71 ms (CPU), Bitunpack 4.51 ms, l2-norm 3.88 ms.\n")
    print("| weight set | widths (bits) | raw / wire MB (ratio) | H2D FP32 | H2D packed | H2D packed + unpack | "
          "zero-copy unpack | pack | pack + fused norm | standalone norm | unpack |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for name, bits in (("alexnet", None), ("vgg16", 8), ("vgg16", 16), ("resnet50", 8), ("lenet", 8)):
        counts = workloads.counts_of(name)
        b = workloads.default_bits(name, bits)
        g = torch.Generator(device="cuda").manual_seed(0)
        masters = [torch.randn(n, generator=g, device="cuda") * 0.1 for n in counts]

        class Fixed(adt.FixedPrecision):
            def round_tos(self, _b=b):
                return [adt.bits_to_round_to(x) for x in _b]

        sync = adt.WeightSync(masters, Fixed(len(counts), 32))
        p = transfer.measured_profile(sync)
        ph, ws = p["phases"], p["weight_stream"]
        f = lambda s: f"{s * 1e3:.3f}"  # noqa: E731
        wb = "/".join(map(str, b)) if len(set(b)) > 1 else str(b[0])
        print(f"| {name} | {wb} | {ws['raw_bytes'] / 1e6:.1f} / {ws['wire_bytes'] / 1e6:.1f} ({ws['ratio']:.2f}) | "
              f"{f(ph['to_worker']['raw_fp32_h2d_s'])} | {f(ph['to_worker']['packed_h2d_s'])} | "
              f"{f(ph['to_worker']['packed_h2d_plus_unpack_s'])} | {f(ph['to_worker']['zero_copy_unpack_s'])} | "
              f"{f(ph['pack']['device_s'])} | {f(ph['pack']['with_fused_l2_norm_s'])} | "
              f"{f(ph['l2_norm']['standalone_s'])} | {f(ph['unpack']['device_s'])} |")
        del sync, masters
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
