"""`weightpack` = the UNMODIFIED reference package (baseline/_ref/weightpack)
with its hot path plugged: before the reference's own __init__ runs, its
`codec` and `precision` submodules are registered as this repo's drop-in
modules, so every `from .codec import ...` / `from .precision import ...`
inside the reference (training.py:25, 40; transfer.py:17; cli.py:15) binds
to the GPU codec and controller. Every other submodule (net, transfer,
training, config, cli, report, __main__) is the reference's own file:
__path__ points at the installed reference package. Test infrastructure for
tests/refsuite only (set up by tests/refsuite/run.py --plug, which also puts
this directory on PYTHONPATH so `python -m weightpack` children are plugged).
"""

import os
import sys

_REAL = os.environ["ADT_REFSUITE_REF"]
__path__ = [_REAL]

from paper_2004_02297_b200 import codec, precision  # noqa: E402

sys.modules[__name__ + ".codec"] = codec
sys.modules[__name__ + ".precision"] = precision

with open(os.path.join(_REAL, "__init__.py")) as _f:
    exec(compile(_f.read(), os.path.join(_REAL, "__init__.py"), "exec"))
