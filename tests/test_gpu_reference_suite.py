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
