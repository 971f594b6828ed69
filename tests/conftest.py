"""Shared pytest wiring: the `gpu` marker and golden-fixture loaders."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # a fresh checkout has no libadt.so: build it (nvcc cross-compiles sm_100a without a GPU)
    from paper_2004_02297_b200 import _build
    if _build.needs_build():
        _build.build()


def _load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def golden_codec():
    """List of dicts: name, words (u32), r, payload (u8), unpacked (u32)."""
    g = _load("golden_codec.npz")
    return [
        dict(name=str(g[f"c{i}_name"]), words=g[f"c{i}_words"], r=int(g[f"c{i}_r"]),
             payload=g[f"c{i}_payload"], unpacked=g[f"c{i}_unpacked"])
        for i in range(int(g["ncases"]))
    ]


@pytest.fixture(scope="session")
def golden_norms():
    g = _load("golden_codec.npz")
    return [(g[f"n{i}_x"], float(g[f"n{i}_norm"])) for i in range(int(g["nnorms"]))]


@pytest.fixture(scope="session")
def golden_awp():
    g = _load("golden_awp.npz")
    runs = []
    for i in range(int(g["nruns"])):
        cfg = g[f"a{i}_cfg"]
        runs.append(dict(
            name=str(g[f"a{i}_name"]), norms=g[f"a{i}_norms"], groups=[int(x) for x in g[f"a{i}_groups"]],
            cfg=dict(threshold=float(cfg[0]), interval=int(cfg[1]), step_bits=int(cfg[2]),
                     initial_bits=int(cfg[3]), max_bits=int(cfg[4]), consecutive=bool(cfg[5])),
            delta=g[f"a{i}_delta"], counter=g[f"a{i}_counter"], bits=g[f"a{i}_bits"]))
    return runs


@pytest.fixture(scope="session")
def golden_lenet():
    return dict(_load("golden_lenet.npz"))


@pytest.fixture(scope="session")
def golden_sgd():
    g = _load("golden_sgd.npz")
    return [dict(w=g[f"s{i}_w"], v=g[f"s{i}_v"], g=g[f"s{i}_g"], hp=tuple(float(x) for x in g[f"s{i}_hp"]),
                 w1=g[f"s{i}_w1"], v1=g[f"s{i}_v1"]) for i in range(int(g["ncases"]))]


@pytest.fixture(scope="session")
def golden_reduce_sgd():
    g = _load("golden_reduce_sgd.npz")
    return [dict(w=g[f"r{i}_w"], v=g[f"r{i}_v"], g=g[f"r{i}_g"], counts=[int(x) for x in g[f"r{i}_counts"]],
                 hp=tuple(float(x) for x in g[f"r{i}_hp"]), w1=g[f"r{i}_w1"], v1=g[f"r{i}_v1"])
            for i in range(int(g["ncases"]))]
