"""Device-resident AWP controller state (WeightSync(awp_on_device=True)).

The reference runs Algorithm 1 on the host after every batch
(precision.py:125-141; training.py:246-254) and the next pack waits for its
widths. On the B200 the decision itself is a one-CTA kernel
(`adt_awp_observe`), so the per-step chain pack -> norm -> decide -> re-pack ->
unpack stays on the device and replays as one CUDA graph; the host reads the
trace rows back in batches (`drain`), not every step.

This module owns the device memory of that controller: per-group state
(LayerPrecisionState as `adt_awp_group`), the group membership lists, the
width arrays and a ring of trace rows. It is initialised from, and written
back into, a host `PrecisionController`, which stays the authoritative object
users inspect (`state(layer)`, `round_tos()`).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .precision import PrecisionController

_GROUP_DT = np.dtype([("prev_norm", "<f8"), ("last_delta", "<f8"), ("bits", "<i4"), ("counter", "<i4"),
                      ("has_prev", "<i4"), ("has_delta", "<i4")])
_ROW_DT = np.dtype([("norm", "<f8"), ("delta", "<f8"), ("batch", "<i4"), ("layer", "<i4"), ("counter", "<i4"),
                    ("bits", "<i4"), ("has_delta", "<i4"), ("pad", "<i4")])
assert _GROUP_DT.itemsize == 32 and _ROW_DT.itemsize == 40


class DeviceAwp:
    def __init__(self, controller: PrecisionController, device: torch.device, ring_steps: int = 256):
        if not isinstance(controller, PrecisionController):
            raise TypeError("awp_on_device needs a PrecisionController schedule")
        self.controller = controller
        self.device = device
        L = controller.num_layers
        groups = controller.layer_groups
        gids = sorted(set(groups))
        self.gindex = {g: i for i, g in enumerate(gids)}
        members = [l for g in gids for l in range(L) if groups[l] == g]
        starts = np.cumsum([0] + [sum(1 for x in groups if x == g) for g in gids]).astype(np.int32)
        self.nlayers, self.ngroups, self.ring_steps = L, len(gids), int(ring_steps)
        self.members = torch.tensor(members, dtype=torch.int32, device=device)
        self.member_start = torch.from_numpy(starts).to(device)
        self.groups = torch.zeros(self.ngroups * _GROUP_DT.itemsize, dtype=torch.uint8, device=device)
        self.widths = torch.empty(L, dtype=torch.uint8, device=device)       # A: in force for the next pack
        self.widths_new = torch.empty(L, dtype=torch.uint8, device=device)   # B: written by the observation
        self.escalated = torch.zeros(L + 1, dtype=torch.int32, device=device)   # count, then layer ids
        self.ring = torch.zeros(self.ring_steps * L * _ROW_DT.itemsize, dtype=torch.uint8, device=device)
        self.counter = torch.zeros(2, dtype=torch.int64, device=device)
        cfg = controller.config
        self.config = _lib.AwpConfig(float(cfg.threshold), int(cfg.interval), int(cfg.step_bits), int(cfg.max_bits),
                                     int(bool(cfg.consecutive)))
        self.struct = _lib.AwpDevice(self.groups.data_ptr(), self.members.data_ptr(), self.member_start.data_ptr(),
                                     self.widths.data_ptr(), self.widths_new.data_ptr(), self.escalated.data_ptr(),
                                     self.ring.data_ptr(), self.counter.data_ptr(), L, self.ngroups, self.ring_steps, 0)
        self.drained = 0          # observations already read back
        self.pending = 0          # observations issued since the last drain
        self.label_set = False
        self.push_state()

    # ------------------------------------------------------ host <-> device
    def push_state(self) -> None:
        """Copy the host controller's state (and widths) to the device."""
        g = np.zeros(self.ngroups, _GROUP_DT)
        for gid, i in self.gindex.items():
            st = self.controller.group_state(gid)
            g[i] = (st.prev_norm if st.prev_norm is not None else 0.0,
                    st.last_delta if st.last_delta is not None else 0.0,
                    st.bits, st.interval_counter, int(st.prev_norm is not None), int(st.last_delta is not None))
        self.groups.copy_(torch.from_numpy(g.view(np.uint8)))
        w = torch.tensor(self.controller.round_tos(), dtype=torch.uint8)
        self.widths.copy_(w)
        self.widths_new.copy_(w)

    def set_next_label(self, batch: int) -> None:
        """Trace label of the next observation (consecutive after that)."""
        self.counter[1].fill_(int(batch))
        self.label_set = True

    def drain(self) -> list[tuple]:
        """Synchronise, read back the trace rows of every observation issued
        since the last drain (TRACE_HEADER order), and write the device state
        back into the host controller."""
        torch.cuda.current_stream().synchronize()
        count = int(self.counter[0].item())
        n = count - self.drained
        if n > self.ring_steps:
            raise RuntimeError(f"device AWP trace ring overflowed: {n} observations since the last drain, "
                               f"ring holds {self.ring_steps}")
        rows = []
        if n:
            ring = self.ring.cpu().numpy().view(_ROW_DT).reshape(self.ring_steps, self.nlayers)
            block = ring[[k % self.ring_steps for k in range(self.drained, count)]].reshape(-1)
            deltas = block["delta"].tolist()
            for i in np.flatnonzero(block["has_delta"] == 0).tolist():   # first observations only
                deltas[i] = None
            rows = list(zip(block["batch"].tolist(), block["layer"].tolist(), block["norm"].tolist(), deltas,
                            block["counter"].tolist(), block["bits"].tolist()))
        self.drained = count
        self.pending = 0
        g = self.groups.cpu().numpy().view(_GROUP_DT)
        for gid, i in self.gindex.items():
            st = self.controller.group_state(gid)
            st.bits = int(g[i]["bits"])
            st.interval_counter = int(g[i]["counter"])
            st.prev_norm = float(g[i]["prev_norm"]) if g[i]["has_prev"] else None
            st.last_delta = float(g[i]["last_delta"]) if g[i]["has_delta"] else None
        return rows

    def round_tos(self) -> list[int]:
        """Widths in force (a device read)."""
        return [int(x) for x in self.widths.cpu().tolist()]

