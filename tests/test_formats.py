"""Text formats on either side of the path, byte-identical to the reference's
own rendering (fixtures made by the reference, tests/golden/make_golden.py):
the bench-codec table / CSV / warnings (bench.py:74-104) and the AWP trace CSV
(training.py:304-321). CPU only."""

import io
import json
import os

from conftest import GOLDEN

from paper_2004_02297_b200 import codecbench
from paper_2004_02297_b200.precision import TRACE_HEADER, write_trace_csv


def _golden():
    with open(os.path.join(GOLDEN, "golden_formats.json")) as f:
        return json.load(f)


def test_bench_codec_table_csv_and_warnings_match_reference():
    g = _golden()
    rows = [tuple(r) for r in g["bench_rows"]]
    assert codecbench.render_bench_table(rows) == g["bench_table"]
    buf = io.StringIO()
    codecbench.write_bench_csv(buf, rows)
    assert buf.getvalue() == g["bench_csv"]
    assert codecbench.slow_vector_warnings(rows) == g["bench_warnings"]
    assert codecbench.BENCH_HEADER == ("path", "size", "round_to", "workers", "seconds", "bytes_per_s")


def test_trace_csv_matches_reference():
    g = _golden()
    rows = [tuple(float("nan") if nan else v for v, nan in zip(r, flags))
            for r, flags in zip(g["trace_rows"], g["trace_nan_cells"])]
    buf = io.StringIO()
    write_trace_csv(buf, rows)
    assert buf.getvalue() == g["trace_csv"]
    assert buf.getvalue().splitlines()[0] == ",".join(TRACE_HEADER)


def test_bench_codec_usage_errors():
    from paper_2004_02297_b200 import cli
    assert cli.main(["bench-codec", "--round-tos", "0,5"]) == 2
