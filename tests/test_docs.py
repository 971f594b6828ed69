"""Documentation stays in step with the code: every ABI entry point in
include/adt.h is described in INTEGRATION.md, and every evidence file the
profiles index names exists."""

import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _read(*parts):
    with open(os.path.join(ROOT, *parts)) as f:
        return f.read()


def test_integration_covers_every_abi_function():
    header = _read("include", "adt.h")
    doc = _read("INTEGRATION.md")
    names = sorted(set(re.findall(r"\b(adt_[a-z0-9_]+)\s*\(", header)))
    prefixes = [p[:-1] for p in re.findall(r"`(adt_[a-z_]*\*)`", doc)]
    missing = [n for n in names if n not in doc and not any(n.startswith(p) for p in prefixes)]
    assert not missing, missing


def test_profiles_index_names_existing_files():
    index = _read("profiles", "README.md")
    named = sorted(set(re.findall(r"`(r01_[A-Za-z0-9_]+\.(?:md|json|jsonl|txt))`", index)))
    assert named
    missing = [f for f in named if not os.path.exists(os.path.join(ROOT, "profiles", f))]
    assert not missing, missing
