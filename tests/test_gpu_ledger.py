"""The measured ledger on a B200: LedgerRecorder around WeightSync (device
masters) and HostWeightSync (host masters) — one to_worker record per worker
and layer per step with the reference's byte columns and MEASURED seconds
(CUDA events, host wall clock), a CSV in LEDGER_HEADER form and a
profile_report over PHASES."""

import csv
import io

import numpy as np
import pytest
import torch

from oracle import weightpack_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def adt():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2004_02297_b200 as adt
    return adt


@pytest.mark.parametrize("where", ["device", "host"])
def test_recorder_measures_every_record(adt, where):
    from paper_2004_02297_b200 import transfer as T
    steps, workers = 6, 2
    walk = list(O.lenet_walk(steps, seed=7))
    L = len(walk[0][1])
    cfg = adt.PrecisionConfig(threshold=-2e-3, interval=2, step_bits=8, initial_bits=8)
    if where == "device":
        masters = [torch.from_numpy(w.copy()).cuda() for w in walk[0][1]]
        sync = adt.WeightSync(masters, adt.PrecisionController(L, cfg))
    else:
        masters = [w.copy() for w in walk[0][1]]
        sync = adt.HostWeightSync(masters, adt.PrecisionController(L, cfg))
    bias = [20 * 4, 50 * 4, 500 * 4, 10 * 4]
    rec = T.LedgerRecorder(sync, workers=workers, bias_bytes=bias)
    widths = []
    for t in range(steps):
        for m, w in zip(masters, walk[t][1]):
            if where == "device":
                m.copy_(torch.from_numpy(w))
            else:
                m[...] = w
        res = rec.step(batch=t)
        widths.append(res.round_tos)
        rec.gradients(batch=t, parameter_count=sum(sync.counts) + sum(bias) // 4)
    led = rec.ledger
    assert len(led) == steps * (workers * L + workers)
    k = 0
    for t in range(steps):
        for _ in range(workers):
            for layer in range(L):
                r = led.records[k]
                n, w = sync.counts[layer], widths[t][layer]
                assert (r.batch, r.direction, r.layer) == (t, "to_worker", layer)
                assert r.raw_bytes == 4 * n + bias[layer] and r.wire_bytes == 14 + n * w + bias[layer]
                assert r.pack_seconds > 0 and r.unpack_seconds > 0
                assert (r.link_seconds > 0) == (where == "host")
                k += 1
        for _ in range(workers):
            assert led.records[k].direction == "to_host" and led.records[k].layer == "all"
            k += 1
    buf = io.StringIO()
    led.write_csv(buf)
    rows = list(csv.DictReader(io.StringIO(buf.getvalue())))
    assert tuple(rows[0].keys()) == T.LEDGER_HEADER and len(rows) == len(led)
    rep = rec.report()
    assert set(rep["phases"]) == set(T.PHASES)
    assert rep["phases"]["pack"]["wall_s"] > 0 and rep["phases"]["unpack"]["wall_s"] > 0
    assert rep["weight_stream"]["ratio"] > 1.0
