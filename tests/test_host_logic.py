"""Host-side logic of the product package, CPU only: helpers, PackedBlock,
container format, layout planning, the AWP controller vs the reference's
golden traces, and the workload shapes."""

import io
import math
import struct

import numpy as np
import pytest

import paper_2004_02297_b200 as adt
from paper_2004_02297_b200 import workloads
from paper_2004_02297_b200.layout import PackedLayout


def test_round_to_helpers():
    # test_codec.py:42-63
    assert adt.bits_to_round_to(14) == 2
    assert [adt.bits_to_round_to(b) for b in (1, 8, 9, 16, 17, 24, 25, 32)] == [1, 1, 2, 2, 3, 3, 4, 4]
    for bad in (0, 33, -1):
        with pytest.raises(ValueError):
            adt.bits_to_round_to(bad)
    assert [adt.truncation_mask(r) for r in (1, 2, 3, 4)] == [0xFF000000, 0xFFFF0000, 0xFFFFFF00, 0xFFFFFFFF]
    for bad in (0, 5, 2.5, "x"):
        with pytest.raises(ValueError):
            adt.truncation_mask(bad)


def test_packed_block_invariants():
    b = adt.PackedBlock(3, 2, bytes(6))
    assert b.raw_bytes == 8 and b.wire_bytes == 14 + 6
    with pytest.raises(adt.MalformedBlock):
        adt.PackedBlock(2, 3, bytes(5))
    with pytest.raises(adt.MalformedBlock):
        adt.PackedBlock(1, -1, b"")
    with pytest.raises(ValueError):
        adt.PackedBlock(5, 0, b"")
    with pytest.raises(AttributeError):
        b.round_to = 2
    assert b == adt.PackedBlock(3, 2, bytearray(6))
    assert b != adt.PackedBlock(3, 2, bytes([1]) + bytes(5))
    # size law (test_codec.py:174-179; test_transfer.py:43-51: 1000 w @ r=3 -> 3014 wire bytes)
    assert adt.PackedBlock(3, 1000, bytes(3000)).wire_bytes == 3014


def _container(r, n, payload):
    buf = io.BytesIO()
    adt.write_stream(buf, adt.PackedBlock(r, n, payload))
    return buf.getvalue()


def test_container_layout_and_errors():
    # test_codec.py:182-244
    data = _container(3, 1, bytes([1, 2, 3]))
    assert data[:4] == b"ADT1" and data[4] == 1 and data[5] == 3 and data[6:14] == struct.pack("<Q", 1)
    assert data[14:] == bytes([1, 2, 3])
    assert adt.read_stream(io.BytesIO(data)) == adt.PackedBlock(3, 1, bytes([1, 2, 3]))
    good = _container(2, 4, bytes(range(8)))
    with pytest.raises(adt.MalformedBlock, match="byte 6"):
        adt.read_stream(io.BytesIO(good[:6]))
    with pytest.raises(adt.MalformedBlock, match="byte 19"):
        adt.read_stream(io.BytesIO(good[:-3]))
    with pytest.raises(adt.MalformedBlock, match="trailing data"):
        adt.read_stream(io.BytesIO(good + b"x"))
    with pytest.raises(adt.MalformedBlock, match="magic"):
        adt.read_stream(io.BytesIO(b"NOPE" + good[4:]))
    with pytest.raises(adt.MalformedBlock, match="version"):
        adt.read_stream(io.BytesIO(good[:4] + b"\x07" + good[5:]))
    with pytest.raises(adt.MalformedBlock, match="round_to"):
        adt.read_stream(io.BytesIO(good[:5] + b"\x05" + good[6:]))
    empty = adt.read_stream(io.BytesIO(_container(2, 0, b"")))
    assert empty.weight_count == 0


def test_layout_planning():
    lay = PackedLayout.plan([0, 1, 4097, 3], [2, 3, 3, 1])
    assert lay.offsets == (0, 0, 16, 12320)
    assert all(o % 16 == 0 for o in lay.offsets)
    assert lay.total_payload_bytes == 0 + 3 + 12291 + 3
    assert lay.payload_end == 12323 and lay.nbytes == 12336
    assert lay.span(2) == (16, 16 + 12291)
    assert lay.roundtrip_bytes() == 2 * (6 * 0 + 7 * 1 + 7 * 4097 + 5 * 3)
    with pytest.raises(ValueError):
        PackedLayout.plan([1], [5])


def test_alexnet_mixed_width_sizes():
    counts = workloads.counts_of("alexnet")
    rs = [adt.bits_to_round_to(b) for b in workloads.default_bits("alexnet")]
    lay = PackedLayout.plan(counts, rs)
    assert sum(counts) == 61_090_496
    assert lay.total_payload_bytes == 148_970_176
    assert lay.roundtrip_bytes() == 2 * (244_361_984 + 148_970_176)


def test_workload_shapes():
    assert sum(workloads.counts_of("lenet")) == 430_500
    assert sum(workloads.counts_of("vgg16")) == 138_344_128
    assert len(workloads.shapes_of("resnet50")) == 161 and sum(workloads.counts_of("resnet50")) == 25_557_032
    assert sum(workloads.counts_of("1b")) == 1 << 30
    try:
        import torchvision
    except ImportError:
        return
    for name in ("alexnet", "vgg16", "resnet50"):
        m = getattr(torchvision.models, name)()
        ref = [tuple(p.shape) for k, p in m.named_parameters()
               if name == "resnet50" or (k.endswith("weight") and p.dim() > 1)]
        assert ref == workloads.shapes_of(name)


def test_change_rate_edges():
    # precision.py:31-39; test_precision.py:41-52
    assert adt.change_rate(0.99, 1.0) == pytest.approx(-0.01)
    assert adt.change_rate(1.0, 1.0) == 0.0
    assert adt.change_rate(5.0, 0.0) == math.inf
    assert adt.change_rate(0.0, 0.0) == 0.0
    assert math.isnan(adt.change_rate(float("nan"), 1.0))


def test_config_validation():
    for kw in (dict(initial_bits=12), dict(interval=0), dict(step_bits=0), dict(initial_bits=16, max_bits=8)):
        with pytest.raises(ValueError):
            adt.PrecisionConfig(**kw)


def test_controller_matches_reference_traces(golden_awp):
    for run in golden_awp:
        L = run["norms"].shape[1]
        c = adt.PrecisionController(L, adt.PrecisionConfig(**run["cfg"]), run["groups"])
        k = 0
        for b, row in enumerate(run["norms"]):
            for (batch, layer, norm, delta, counter, bits) in c.observe_all(list(row), batch=b):
                assert bits == run["bits"][k] and counter == run["counter"][k], (run["name"], k)
                gd = run["delta"][k]
                assert (delta is None and math.isnan(gd)) or delta == gd, (run["name"], k)
                k += 1


def test_controller_edge_cases():
    cfg = adt.PrecisionConfig(threshold=-1e-3, interval=3, step_bits=8, initial_bits=8)
    c = adt.PrecisionController(3, cfg)
    c.observe_batch(0, 100.0)
    assert c.state(0).interval_counter == 0 and c.state(0).last_delta is None
    with pytest.raises(adt.UnknownLayer):
        c.observe_batch(3, 1.0)
    with pytest.raises(adt.UnknownLayer):
        c.current_round_to(-1)
    # clamp keeps resetting the counter (test_precision.py:87-92)
    c2 = adt.PrecisionController(1, adt.PrecisionConfig(threshold=-1e-3, interval=2, step_bits=8, initial_bits=32))
    n = 1.0
    for _ in range(7):
        c2.observe_batch(0, n)
        n *= 0.99
    assert c2.current_bits(0) == 32 and c2.state(0).interval_counter in (0, 1)
    # 14 bits -> 2 bytes (test_precision.py:125-132)
    c3 = adt.PrecisionController(1, adt.PrecisionConfig(threshold=-1e-3, interval=1, step_bits=6, initial_bits=8))
    c3.observe_batch(0, 1.0)
    c3.observe_batch(0, 0.998)
    assert c3.current_bits(0) == 14 and c3.current_round_to(0) == 2
    f = adt.FixedPrecision(2, 32)
    assert f.current_round_to(1) == 4 and f.round_tos() == [4, 4]
    with pytest.raises(adt.UnknownLayer):
        f.current_bits(2)
    with pytest.raises(ValueError):
        adt.FixedPrecision(1, 33)


def test_product_path_refuses_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(RuntimeError, match="CUDA"):
        adt.pack(np.zeros(4, np.float32), 2)
    with pytest.raises(RuntimeError, match="CUDA"):
        adt.l2_norm(np.zeros(4, np.float32))


def test_wire_accounting_matches_reference_ledger_arithmetic():
    # test_transfer.py:43-51 (1000 w @ r=3 -> 3014 wire) and :137-144 (mean r = 4/3 -> ~3x)
    from paper_2004_02297_b200 import transfer
    rec = transfer.send_weights_bytes(adt.PackedBlock(3, 1000, bytes(3000)), layer=0, bias_bytes=40)
    assert (rec.wire_bytes, rec.raw_bytes, rec.weight_wire_bytes, rec.weight_raw_bytes) == (3054, 4040, 3014, 4000)
    lay = PackedLayout.plan([10_000] * 3, [1, 1, 2])
    recs = transfer.layout_records(lay)
    assert 2.8 <= transfer.weight_stream_ratio(recs) <= 3.2
    assert [r.weight_wire_bytes for r in recs] == [14 + 10_000, 14 + 10_000, 14 + 20_000]
    with pytest.raises(ValueError):
        transfer.weight_stream_ratio([])
    # gradients return uncompressed (transfer.py:247-251): 4 bytes per parameter
    g = transfer.return_gradients_bytes(1234)
    assert (g.raw_bytes, g.wire_bytes, g.weight_raw_bytes, g.weight_wire_bytes) == (4936, 4936, 0, 0)
    with pytest.raises(ValueError):
        transfer.return_gradients_bytes(-1)
