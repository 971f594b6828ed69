"""Run the reference's OWN hot-path test modules, unmodified, against this
package: `weightpack.codec` and `weightpack.precision` resolve to
paper_2004_02297_b200.codec / .precision (the drop-in), so every
`codec.pack(...)`, `codec.unpack(...)`, `precision.l2_norm(...)` in
/root/reference/pkg/tests/test_codec.py and test_precision.py runs on the GPU
through libadt.so. The test files come from baseline/_ref/tests (copied there
by __graft_entry__.install_reference() from /root/reference/pkg/tests;
git-ignored like the reference install, shipped with the snapshot).

    python tests/refsuite/run.py <tests dir> test_codec.py test_precision.py [pytest args]
    python tests/refsuite/run.py --plug <tests dir> test_training.py test_acceptance.py ...
        (the whole reference package with only codec + precision replaced)
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


def install_plugged(ref_root):
    """The UNMODIFIED reference package (baseline/_ref/weightpack: training
    loop, net, transfer ledger, config, CLI, report) with only its hot path
    replaced by this package's codec and precision modules
    (tests/refsuite/plug/weightpack). Set up for this process and, through
    PYTHONPATH, for the suite's `python -m weightpack` children."""
    here = os.path.dirname(os.path.abspath(__file__))
    os.environ["ADT_REFSUITE_REF"] = os.path.join(ref_root, "weightpack")
    front = [os.path.join(here, "plug"), os.path.join(here, "stubs"), ROOT]     # stubs: matplotlib (absent)
    os.environ["PYTHONPATH"] = os.pathsep.join(front + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])
    sys.path[:0] = front
    from paper_2004_02297_b200 import codec, precision
    import weightpack
    from weightpack import training
    assert weightpack.codec is codec and weightpack.precision is precision
    assert training.pack_vectorized is codec.pack_vectorized and training.l2_norm is precision.l2_norm
    assert training.__file__.startswith(os.environ["ADT_REFSUITE_REF"])


def main(argv):
    plug = "--plug" in argv
    argv = [a for a in argv if a != "--plug"]
    tests_dir, rest = argv[0], argv[1:]
    files = [a for a in rest if a.endswith(".py")]
    extra = [a for a in rest if not a.endswith(".py")]
    if plug:
        install_plugged(os.path.dirname(os.path.abspath(tests_dir)))
    else:
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
