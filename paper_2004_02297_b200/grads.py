"""Gradient return path: worker gradients -> master update.

The reference returns every worker's gradients UNcompressed to the host
(4 bytes per parameter, transfer.py:247-251) and
`net.gather_and_update` (net.py:203-257) combines them:

    g = pairwise_sum([g_c * f32(count_c) for c]) / f32(total)     (float32)
    g += wd * W;  v = mu * v + g;  W -= lr * v

On B200 a worker's gradients live in one flat FP32 *bucket* per rank (every
layer at a 16-byte aligned offset), so a rank's master shard — a contiguous
range of the concatenated layers (sharded.ShardPlan) — is ONE contiguous range
of every bucket. The fused kernel `adt_reduce_sgd_pack` reads the shard's
range out of all contributions (peer buckets over NVLink, or the
all-to-all'd copies), combines them in registers with the reference's
association tree and rounding, applies the momentum step to the master shard
and packs it for the weight stream — one pass, bit-exact with the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

import torch

FLOAT_ALIGN = 4   # floats per 16 bytes


def bucket_offsets(counts: Sequence[int]) -> tuple[tuple[int, ...], int]:
    """Float offsets of each layer in a gradient bucket (16-B aligned) and the
    bucket length in floats (a multiple of 4)."""
    offs, pos = [], 0
    for n in counts:
        if n < 0:
            raise ValueError(f"negative weight count {n}")
        offs.append(pos)
        pos += -(-int(n) // FLOAT_ALIGN) * FLOAT_ALIGN
    return tuple(offs), pos



class ShapeMismatch(ValueError):
    """net.py:16-17 — gradients that do not fit the network (wrong layer
    count or layer size, or no contributions at all)."""

class GradBucket:
    """One worker's weight gradients in a flat CUDA float32 buffer.

    `views[l]` is layer l's gradient (shape of the layer, written by the
    backward pass or copied in); `sample_count` weights the contribution
    (GradientSet.sample_count, net.py:65-70)."""

    def __init__(self, shapes_or_counts, device=None, sample_count: int = 1):
        shapes = [tuple(s) if isinstance(s, (tuple, list, torch.Size)) else (int(s),) for s in shapes_or_counts]
        self.shapes = shapes
        self.counts = [int(torch.Size(s).numel()) for s in shapes]
        self.offsets, self.numel = bucket_offsets(self.counts)
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.flat = torch.zeros(max(FLOAT_ALIGN, self.numel), dtype=torch.float32, device=dev)
        self.views = [self.flat[o:o + n].view(s) for o, n, s in zip(self.offsets, self.counts, shapes)]
        self.sample_count = int(sample_count)

    @property
    def device(self) -> torch.device:
        return self.flat.device

    def load(self, grads: Sequence[torch.Tensor]) -> "GradBucket":
        """Copy per-layer gradient tensors in (stream-ordered)."""
        if len(grads) != len(self.views):
            raise ShapeMismatch(f"{len(grads)} gradients for a {len(self.views)}-layer bucket")
        for v, g in zip(self.views, grads):
            if g.numel() != v.numel():
                raise ShapeMismatch(f"gradient has {g.numel()} entries, layer has {v.numel()}")
            v.copy_(g.reshape(v.shape))
        return self

    def byte_offset(self, layer: int, lo: int = 0) -> int:
        return 4 * (self.offsets[layer] + lo)


@dataclass
class GradientSet:
    """net.py:65-70 — mean-loss gradients for every layer from `sample_count`
    samples. Biases are not part of the weight stream (they travel raw,
    PAPER.md:243-245) and are ignored by the device path."""

    weight_grads: list
    bias_grads: list = field(default_factory=list)
    sample_count: int = 1


def shard_ranges(plan, counts: Sequence[int]) -> list[tuple[int, int]]:
    """Per rank, the [begin, end) float range of a gradient bucket its master
    shard covers. Ranks own consecutive pieces of the concatenated layers in
    rank order, so each range is contiguous (inter-layer pad included) and the
    ranges tile the bucket exactly: rank q's gradients for every other rank p
    are one slice, which is what the NCCL transport's all-to-all moves."""
    offs, total = bucket_offsets(counts)
    starts = []
    for q in range(plan.world):
        ps = plan.pieces[q]
        starts.append(offs[ps[0].layer] + ps[0].lo if ps else None)
    out, nxt = [None] * plan.world, total
    for q in range(plan.world - 1, -1, -1):
        b = starts[q] if starts[q] is not None else nxt
        out[q] = (b, nxt)
        nxt = b
    if out and out[0][0] != 0:
        out[0] = (0, out[0][1])
    return out


def return_gradients_bytes(parameter_count: int) -> int:
    """transfer.py:247-251 — one worker's uncompressed gradient payload."""
    return 4 * int(parameter_count)
