"""The reference's own hot-path test suites, run unmodified against the drop-in.

/root/reference/pkg/tests/test_codec.py (byte semantics, KATs, path
equivalence, mask / idempotence / size laws with hypothesis, the ADT1
container and its MalformedBlock diagnostics) and test_precision.py (l2_norm,
change_rate, Algorithm 1 traces against the reference's oracle_precision)
import `weightpack.codec` / `weightpack.precision`; tests/refsuite/run.py maps
those names to this package, so every codec / norm call in them runs on the
GPU through libadt.so. The files travel in baseline/_ref/tests (copied from
/root/reference by __graft_entry__.install_reference(), git-ignored)."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "tests")


@pytest.mark.parametrize("module", ["test_codec.py", "test_precision.py"])
def test_reference_suite_passes_on_the_drop_in(module, tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.exists(os.path.join(SUITE, module)):
        pytest.skip("reference tests not shipped (run __graft_entry__.build() where /root/reference exists)")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "refsuite", "run.py"), SUITE, module, "-rf"],
                       capture_output=True, text=True, timeout=900, cwd=tmp_path)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-4000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 20 and not re.search(r"\d+ (failed|errors?)\b", out), out[-4000:]
    assert "libadt.so" in out, out[-2000:]         # the runner reports the native library it drove


ALL_MODULES = ["test_codec.py", "test_precision.py", "test_transfer.py", "test_training.py", "test_acceptance.py",
               "test_cli.py", "test_net.py", "test_dataset_config.py"]


def test_reference_harness_runs_on_the_plugged_hot_path(tmp_path):
    """The reference's WHOLE test suite (acceptance criteria 1-9, the training
    loop's determinism / worker-invariance / r = 4 transparency tests, the
    transfer ledger, the CLI pack / unpack / train / report) against the
    unmodified reference package with only `codec` and `precision` replaced by
    this package (tests/refsuite/plug): the reference's run_training
    (training.py:207-254) drives our GPU pack / unpack / l2_norm and our
    PrecisionController at every step."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not all(os.path.exists(os.path.join(SUITE, m)) for m in ALL_MODULES):
        pytest.skip("reference tests not shipped (run __graft_entry__.build() where /root/reference exists)")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "refsuite", "run.py"), "--plug", SUITE,
                        *ALL_MODULES, "-rf"], capture_output=True, text=True, timeout=1500, cwd=tmp_path)
    out = p.stdout + p.stderr
    assert p.returncode == 0, out[-6000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 150 and not re.search(r"\d+ (failed|errors?)\b", out), out[-6000:]
    for k in range(1, 10):
        assert f"criterion {k} PASS" in out, out[-3000:]
    assert "libadt.so" in out, out[-2000:]
