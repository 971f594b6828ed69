"""Run the reference's OWN hot-path test modules, unmodified, against this
package: `weightpack.codec` and `weightpack.precision` resolve to
paper_2004_02297_b200.codec / .precision (the drop-in), so every
`codec.pack(...)`, `codec.unpack(...)`, `precision.l2_norm(...)` in
/root/reference/pkg/tests/test_codec.py and test_precision.py runs on the GPU
through libadt.so. The test files come from baseline/_ref/tests (copied there
by __graft_entry__.install_reference() from /root/reference/pkg/tests;
git-ignored like the reference install, shipped with the snapshot).

    python tests/refsuite/run.py <tests dir> test_codec.py test_precision.py [pytest args]
"""

import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def install_shim():
    from paper_2004_02297_b200 import codec, precision
    pkg = types.ModuleType("weightpack")
    pkg.__path__ = []                       # a package, so `from weightpack.precision import X` resolves
    pkg.codec, pkg.precision = codec, precision
    sys.modules["weightpack"] = pkg
    sys.modules["weightpack.codec"] = codec
    sys.modules["weightpack.precision"] = precision


def main(argv):
    tests_dir, rest = argv[0], argv[1:]
    files = [a for a in rest if a.endswith(".py")]
    extra = [a for a in rest if not a.endswith(".py")]
    install_shim()
    sys.path.insert(0, tests_dir)            # oracle_precision, conftest helpers
    import pytest
    rc = pytest.main([os.path.join(tests_dir, f) for f in files] +
                     ["-q", "-p", "no:cacheprovider", "--rootdir", tests_dir, "-o", "addopts="] + extra)
    with open("/proc/self/maps") as f:                 # which native library the suite drove
        libs = sorted({line.split()[-1] for line in f if line.rstrip().endswith("libadt.so")})
    print("native:", " ".join(libs) or "none")
    return rc


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
