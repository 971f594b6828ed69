"""CLI pack/unpack (reference cli.py:48-87): exit codes and container bytes."""

import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT
from paper_2004_02297_b200 import cli


def test_usage_errors_exit_2(capsys):
    with pytest.raises(SystemExit) as e:
        cli.main(["pack", "--input", "x"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["pack", "--input", "x", "--output", "y", "--round-to", "5"])
    assert e.value.code == 2


def test_malformed_container_exit_3(tmp_path, capsys):
    bad = tmp_path / "bad.adt"
    bad.write_bytes(b"NOPE" + bytes(10))
    assert cli.main(["unpack", "--input", str(bad), "--output", str(tmp_path / "o.f32")]) == 3
    assert "magic" in capsys.readouterr().err
    trunc = tmp_path / "t.adt"
    trunc.write_bytes(b"ADT1\x01\x02" + (5).to_bytes(8, "little") + bytes(3))
    assert cli.main(["unpack", "--input", str(trunc), "--output", str(tmp_path / "o.f32")]) == 3


def test_missing_or_ragged_input_exit_1(tmp_path, capsys):
    assert cli.main(["pack", "--input", str(tmp_path / "nope.f32"), "--round-to", "2",
                     "--output", str(tmp_path / "o.adt")]) == 1
    rag = tmp_path / "rag.f32"
    rag.write_bytes(bytes(7))
    assert cli.main(["pack", "--input", str(rag), "--round-to", "2", "--output", str(tmp_path / "o.adt")]) == 1


@pytest.mark.gpu
def test_pack_unpack_roundtrip_matches_oracle_container(tmp_path, capsys):
    from oracle import weightpack_oracle as O
    src = tmp_path / "w.f32"
    w = np.linspace(-1, 1, 1024).astype("<f4")
    w.tofile(src)
    for r in (1, 2, 3, 4):
        out = tmp_path / f"w{r}.adt"
        assert cli.main(["pack", "--input", str(src), "--round-to", str(r), "--output", str(out)]) == 0
        assert f"ratio {r / 4:.4f}" in capsys.readouterr().out
        assert out.read_bytes() == O.write_container(r, 1024, O.pack_vectorized(w, r))
        back = tmp_path / f"w{r}.csv"
        assert cli.main(["unpack", "--input", str(out), "--output", str(back)]) == 0
        got = np.loadtxt(back, ndmin=1).astype(np.float32)
        assert np.array_equal(got.view(np.uint32), w.view(np.uint32) & np.uint32(O.keep_mask(r)))
    res = subprocess.run([sys.executable, "-m", "paper_2004_02297_b200", "pack", "--input", str(src),
                          "--round-to", "3", "--output", str(tmp_path / "m.adt")], cwd=ROOT,
                         capture_output=True, text=True)
    assert res.returncode == 0, res.stderr


@pytest.mark.gpu
def test_bench_codec_runs_with_precheck(tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert cli.main(["bench-codec", "--sizes", "1000,5000", "--round-tos", "1,3", "--workers", "1,2",
                     "--repeats", "2", "--check-size", "20000", "--csv", str(out)]) == 0
    text = capsys.readouterr().out
    assert "precheck passed" in text and "device_unpack" in text
    lines = out.read_text().splitlines()
    assert lines[0] == "path,size,round_to,workers,seconds,bytes_per_s"
    assert len(lines) == 1 + 2 * 2 * (2 + 2 + 1 + 2)   # sizes x r x (scalar, vectorized, 2 parallel, unpack, 2 device)
