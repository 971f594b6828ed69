"""§8f item 3: the measured transfer ledger in the reference's schemas.

The same run description (layers, widths per batch, bias bytes, workers,
gradient returns) goes through the reference's own TransferLedger /
send_weights / send_to_host / profile_report (weightpack from baseline/_ref,
transfer.py:19-286) and through ours: every byte column, the CSV header and
text layout, and every profile key must match (the seconds differ by design:
modeled there, measured here)."""

import io
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def wp():
    if not os.path.isdir(os.path.join(REF, "weightpack")):
        pytest.skip("baseline/_ref (the reference package) is not installed")
    sys.path.insert(0, REF)
    import weightpack.codec
    import weightpack.transfer
    return weightpack


COUNTS = [500, 25000, 400000, 5000]
BIAS = [80, 200, 2000, 40]
WIDTHS = [[1, 1, 1, 1], [1, 2, 1, 1], [2, 2, 1, 3], [4, 3, 2, 1]]


def _ours(workers=2):
    from paper_2004_02297_b200 import transfer as T
    led = T.TransferLedger()
    for b, rs in enumerate(WIDTHS):
        for _ in range(workers):
            for layer, (n, r) in enumerate(zip(COUNTS, rs)):
                T.record_weights(led, batch=b, layer=layer, count=n, round_to=r, bias_bytes=BIAS[layer],
                                 pack_seconds=1e-6 * (layer + 1), unpack_seconds=2e-6, link_seconds=3e-6)
        for _ in range(workers):
            T.record_gradients(led, batch=b, parameter_count=sum(COUNTS) + sum(BIAS) // 4, link_seconds=4e-6)
    return led


def _reference(wp, workers=2):
    T = wp.transfer
    led = T.TransferLedger()
    link = T.LinkModel(bandwidth=12e9, latency=1e-6)
    for b, rs in enumerate(WIDTHS):
        for _ in range(workers):
            for layer, (n, r) in enumerate(zip(COUNTS, rs)):
                blk = wp.codec.PackedBlock(r, n, bytes(n * r))
                T.send_weights(blk, link, led, batch=b, layer=layer, bias_bytes=BIAS[layer])
        for _ in range(workers):
            T.send_to_host((sum(COUNTS) + sum(BIAS) // 4) * 4, link, led, batch=b)
    return led


def test_constants_match(wp):
    from paper_2004_02297_b200 import transfer as T
    assert T.LEDGER_HEADER == wp.transfer.LEDGER_HEADER
    assert T.PHASES == wp.transfer.PHASES
    assert (T.TO_WORKER, T.TO_HOST) == (wp.transfer.TO_WORKER, wp.transfer.TO_HOST)


def test_records_and_csv_byte_columns_match(wp):
    ours, ref = _ours(), _reference(wp)
    assert len(ours) == len(ref)
    for a, b in zip(ours.records, ref.records):
        assert (a.batch, a.direction, a.layer, a.raw_bytes, a.wire_bytes, a.weight_raw_bytes, a.weight_wire_bytes) == \
               (b.batch, b.direction, b.layer, b.raw_bytes, b.wire_bytes, b.weight_raw_bytes, b.weight_wire_bytes)
    fa, fb = io.StringIO(), io.StringIO()
    ours.write_csv(fa)
    ref.write_csv(fb)
    la, lb = fa.getvalue().splitlines(), fb.getvalue().splitlines()
    assert la[0] == lb[0] and len(la) == len(lb)
    for x, y in zip(la[1:], lb[1:]):
        assert x.split(",")[:5] == y.split(",")[:5]
        assert all(float(v) >= 0.0 for v in x.split(",")[5:])
    assert ours.total_wire_bytes() == ref.total_wire_bytes()
    assert ours.weight_stream_ratio() == ref.weight_stream_ratio()


def test_profile_report_schema_matches(wp):
    from paper_2004_02297_b200 import transfer as T
    wall = {"pack": 0.5, "unpack": 0.25, "to_worker": 0.1}
    a, b = T.profile_report(_ours(), wall), wp.transfer.profile_report(_reference(wp), wall)

    def keys(d, pre=""):
        out = set()
        for k, v in d.items():
            out.add(pre + k)
            if isinstance(v, dict):
                out |= keys(v, pre + k + ".")
        return out
    assert keys(a) == keys(b)
    assert a["wire_bytes"] == b["wire_bytes"] and a["raw_bytes"] == b["raw_bytes"]
    assert a["weight_stream"] == b["weight_stream"]
    assert {k: v["wall_s"] for k, v in a["phases"].items()} == {k: v["wall_s"] for k, v in b["phases"].items()}
    with pytest.raises(T.EmptyLedger):
        T.profile_report(T.TransferLedger(), {})
