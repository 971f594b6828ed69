"""Packed-buffer layout: where each layer's payload lives in HBM.

The reference keeps one `bytes` payload per layer (PackedBlock, codec.py:76-107;
payload = count * round_to bytes, weight i at [i*r, (i+1)*r), MSB first).
On the device all layers of a step share one uint8 buffer: layer l's payload
starts at `offsets[l]`, a multiple of 16 bytes so every 4096-weight tile
begins on a 16-byte boundary and moves with 128-bit vectors. The pad between
payloads (< 16 bytes per layer) is never counted as payload or wire bytes
(SURVEY.md §8d).
"""

from __future__ import annotations

from dataclasses import dataclass

ALIGN = 16


def align_up(x: int, a: int = ALIGN) -> int:
    return (x + a - 1) // a * a


@dataclass(frozen=True)
class PackedLayout:
    counts: tuple[int, ...]
    round_tos: tuple[int, ...]
    offsets: tuple[int, ...]
    nbytes: int  # buffer size including inter-layer pad

    @staticmethod
    def plan(counts, round_tos, base: int = 0, align: int = ALIGN) -> "PackedLayout":
        """align: payload offsets are multiples of this (16, or 64 for the host
        packer's full-line non-temporal stores, hostsync.HostWeightSync)."""
        if align < ALIGN or align % ALIGN:
            raise ValueError(f"align must be a multiple of {ALIGN}")
        counts = tuple(int(c) for c in counts)
        round_tos = tuple(int(r) for r in round_tos)
        if len(counts) != len(round_tos):
            raise ValueError("counts and round_tos differ in length")
        offsets = []
        pos = align_up(base, align)
        for n, r in zip(counts, round_tos):
            if n < 0:
                raise ValueError(f"negative weight count {n}")
            if not 1 <= r <= 4:
                raise ValueError(f"round_to must be an integer in [1, 4], got {r}")
            offsets.append(pos)
            pos = align_up(pos + n * r, align)
        return PackedLayout(counts, round_tos, tuple(offsets), pos - align_up(base, align))

    @property
    def num_layers(self) -> int:
        return len(self.counts)

    def payload_bytes(self, layer: int) -> int:
        return self.counts[layer] * self.round_tos[layer]

    @property
    def total_payload_bytes(self) -> int:
        """Σ n·r — the bytes that actually carry weights."""
        return sum(n * r for n, r in zip(self.counts, self.round_tos))

    @property
    def raw_bytes(self) -> int:
        return 4 * sum(self.counts)

    def span(self, layer: int) -> tuple[int, int]:
        o = self.offsets[layer]
        return o, o + self.payload_bytes(layer)

    @property
    def payload_end(self) -> int:
        """One past the last payload byte (a buffer must be at least this long)."""
        return max((o + n * r for o, n, r in zip(self.offsets, self.counts, self.round_tos)), default=0)

    def roundtrip_bytes(self) -> int:
        """Algorithmic HBM bytes of one pack + one unpack: 2·Σ(4 + r)·n."""
        return 2 * sum((4 + r) * n for n, r in zip(self.counts, self.round_tos))
