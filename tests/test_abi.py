"""C-ABI checks that need no GPU: the in-tree library loads, exports every
entry point include/adt.h declares, and validates arguments before touching
the device (no compute calls here)."""

import ctypes
import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "adt.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(adt_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2004_02297_b200 import _lib
    return _lib


def test_header_declares_the_expected_surface():
    assert declared_functions() == sorted(
        ["adt_abi_version", "adt_strerror", "adt_partials_count", "adt_pack", "adt_norm_finalize", "adt_unpack",
         "adt_unpack_multi", "adt_unpack_multi_ex", "adt_copy_multi", "adt_peer_barrier", "adt_ipc_handle_bytes", "adt_ipc_get_handle", "adt_ipc_open",
         "adt_ipc_close", "adt_sumsq", "adt_sgd_pack", "adt_reduce_sgd_pack", "adt_pack_dyn", "adt_unpack_dyn",
         "adt_sgd_pack_dyn", "adt_reduce_sgd_pack_dyn", "adt_awp_observe", "adt_awp_fixup",
         "adt_unpack_multi_dyn", "adt_awp_combine", "adt_awp_fixup_pieces", "adt_awp_fixup_gather",
         "adt_device_sm_count", "adt_pack_host", "adt_host_to_device", "adt_host_threads", "adt_host_simd",
         "adt_sumsq_f64_partials", "adt_sumsq_f64", "adt_roundtrip", "adt_roundtrip_max_tiles",
         "adt_host_to_device_ring", "adt_host_to_device_ex"])


def test_library_exports_every_declared_symbol(lib):
    handle = lib.load()
    for name in declared_functions():
        assert hasattr(handle, name), name
    assert set(lib.EXPORTS) == set(declared_functions())
    assert handle.adt_abi_version() == lib.ABI_VERSION


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2004_02297_b200", "libadt.so")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_strerror_and_partials_count(lib):
    assert lib.strerror(0) == "ok"
    assert "round_to" in lib.strerror(lib.ADT_ERR_ROUND_TO)
    segs = lib.segment_array([(0, 0, 0, 1), (16, 4097, 16, 3), (32, 4096, 12304, 4)])
    assert lib.partials_count(segs, 3) == (0 + 2 + 1) * lib.PARTIALS_PER_TILE


def test_validation_happens_before_any_device_work(lib):
    h = lib.load()
    bad_r = lib.segment_array([(16, 10, 0, 5)])
    assert h.adt_pack(bad_r, 1, 16, None, None, None) == lib.ADT_ERR_ROUND_TO
    with pytest.raises(ValueError):
        lib.check(lib.ADT_ERR_ROUND_TO)
    misaligned = lib.segment_array([(8, 10, 0, 2)])
    assert h.adt_pack(misaligned, 1, 16, None, None, None) == lib.ADT_ERR_ALIGN
    bad_off = lib.segment_array([(16, 10, 8, 2)])
    assert h.adt_unpack(bad_off, 1, 16, None) == lib.ADT_ERR_ALIGN
    assert h.adt_unpack(lib.segment_array([(16, 10, 0, 2)]), 1, 0, None) == lib.ADT_ERR_ARG
    assert h.adt_pack(None, -1, 0, None, None, None) == lib.ADT_ERR_ARG
    # unpack_multi: source index out of range / too many sources
    seg = lib.segment_array([(16, 10, 0, 2, 1)])
    assert h.adt_unpack_multi(seg, 1, lib.pointer_array([16]), 1, None) == lib.ADT_ERR_ARG
    assert h.adt_unpack_multi(seg, 1, lib.pointer_array([16] * 17), 17, None) == lib.ADT_ERR_ARG
    assert h.adt_unpack_multi(seg, 1, lib.pointer_array([16, 8]), 2, None) == lib.ADT_ERR_ALIGN
    assert h.adt_ipc_handle_bytes() == 64
    # fused SGD + pack: bad width / misaligned velocity / sums without partials
    def sgd(ptrs, r, off=0):
        arr = (lib.SgdSegment * 1)()
        arr[0].weights, arr[0].velocity, arr[0].grad = ptrs
        arr[0].count, arr[0].offset, arr[0].round_to, arr[0].reserved = 10, off, r, 0
        return arr
    assert h.adt_sgd_pack(sgd((16, 32, 48), 5), 1, 0.1, 0.9, 0.0, 16, None, None, None) == lib.ADT_ERR_ROUND_TO
    assert h.adt_sgd_pack(sgd((16, 40, 48), 2), 1, 0.1, 0.9, 0.0, 16, None, None, None) == lib.ADT_ERR_ALIGN
    assert h.adt_sgd_pack(sgd((16, 32, 48), 2), 1, 0.1, 0.9, 0.0, 16, 16, None, None) == lib.ADT_ERR_ARG
    # sums requested without partials scratch
    assert h.adt_pack(lib.segment_array([(16, 10, 0, 2)]), 1, 16, 16, None, None) == lib.ADT_ERR_ARG
    assert h.adt_norm_finalize(lib.segment_array([(16, 10, 0, 2)]), 1, None, 16, None) == lib.ADT_ERR_ARG
    # norm pass without scratch
    assert h.adt_sumsq(lib.segment_array([(16, 10, 0, 2)]), 1, None, None, None) == lib.ADT_ERR_ARG
    # fused gradient reduce + SGD + pack: contribution count, alignment, width
    def red(r, goff=0, wptr=16):
        arr = (lib.GradSegment * 1)()
        arr[0].weights, arr[0].velocity = wptr, 32
        arr[0].count, arr[0].offset, arr[0].grad_offset, arr[0].round_to, arr[0].reserved = 10, 0, goff, r, 0
        return arr
    C = ctypes.c_int64
    cnt = (C * 17)(*([1] * 17))
    assert h.adt_reduce_sgd_pack(red(2), 1, lib.pointer_array([48]), cnt, 0, 0.1, 0.9, 0.0, 16, None, None, None, None) \
        == lib.ADT_ERR_ARG
    assert h.adt_reduce_sgd_pack(red(2), 1, lib.pointer_array([48] * 17), cnt, 17, 0.1, 0.9, 0.0, 16, None, None, None, None) == lib.ADT_ERR_ARG
    assert h.adt_reduce_sgd_pack(red(5), 1, lib.pointer_array([48]), cnt, 1, 0.1, 0.9, 0.0, 16, None, None, None, None) \
        == lib.ADT_ERR_ROUND_TO
    assert h.adt_reduce_sgd_pack(red(2, goff=8), 1, lib.pointer_array([48]), cnt, 1, 0.1, 0.9, 0.0, 16, None, None, None, None) == lib.ADT_ERR_ALIGN
    assert h.adt_reduce_sgd_pack(red(2), 1, lib.pointer_array([40]), cnt, 1, 0.1, 0.9, 0.0, 16, None, None, None, None) \
        == lib.ADT_ERR_ALIGN
    assert h.adt_reduce_sgd_pack(red(2, wptr=8), 1, lib.pointer_array([48]), cnt, 1, 0.1, 0.9, 0.0, 16, None, None, None, None) == lib.ADT_ERR_ALIGN
    assert h.adt_reduce_sgd_pack(red(2), 1, lib.pointer_array([48]), cnt, 1, 0.1, 0.9, 0.0, 16, 16, None, None, None) \
        == lib.ADT_ERR_ARG
    # peer barrier: rank outside [0, nranks), too many ranks, misaligned flags, zero poll budget
    assert h.adt_peer_barrier(lib.pointer_array([16, 32]), 2, 2, 48, 10, None) == lib.ADT_ERR_ARG
    assert h.adt_peer_barrier(lib.pointer_array([16] * 17), 17, 0, 48, 10, None) == lib.ADT_ERR_ARG
    assert h.adt_peer_barrier(lib.pointer_array([16, 34]), 2, 0, 48, 10, None) == lib.ADT_ERR_ALIGN
    assert h.adt_peer_barrier(lib.pointer_array([16, 32]), 2, 0, 48, 0, None) == lib.ADT_ERR_ARG
    # device AWP: capacity layout required (round_to 4), widths pointer required, struct sizes
    assert ctypes.sizeof(lib.AwpGroup) == 32 and ctypes.sizeof(lib.AwpRow) == 40
    assert h.adt_pack_dyn(lib.segment_array([(16, 10, 0, 2)]), 1, 16, None, 32, None) == lib.ADT_ERR_ARG
    assert h.adt_pack_dyn(lib.segment_array([(16, 10, 0, 4)]), 1, 16, None, None, None) == lib.ADT_ERR_ARG
    assert h.adt_unpack_dyn(lib.segment_array([(16, 10, 0, 3)]), 1, 16, 32, None) == lib.ADT_ERR_ARG
    dev = lib.AwpDevice()
    cfg = lib.AwpConfig(-2e-3, 50, 8, 32, 0)
    assert h.adt_awp_observe(16, ctypes.byref(dev), ctypes.byref(cfg), None, None) == lib.ADT_ERR_ARG   # empty device struct
    m, r = lib.segment_array([(16, 10, 0, 4)]), lib.segment_array([(48, 10, 16, 4)])
    assert h.adt_awp_fixup(m, r, 1, 16, 64, 80, None) == lib.ADT_ERR_ARG                        # offsets differ


def test_host_entry_points_validate_arguments(lib):
    """adt_pack_host / adt_host_to_device / adt_sumsq_f64 refuse bad input
    before doing any work (host pointers, no device needed)."""
    h = lib.load()
    bad_r = lib.segment_array([(16, 10, 0, 5)])
    assert h.adt_pack_host(bad_r, 1, 16, None, 0) == lib.ADT_ERR_ROUND_TO
    assert h.adt_pack_host(lib.segment_array([(18, 10, 0, 2)]), 1, 16, None, 0) == lib.ADT_ERR_ALIGN
    assert h.adt_pack_host(lib.segment_array([(16, 10, 0, 2)]), 1, None, None, 0) == lib.ADT_ERR_ARG
    assert h.adt_pack_host(None, -1, None, None, 0) == lib.ADT_ERR_ARG
    segs = lib.segment_array([(16, 10, 0, 2), (32, 10, 0, 2)])          # overlapping payloads
    assert h.adt_host_to_device(segs, segs, 2, 64, 64, 1 << 20, None, 0, 0, None) == lib.ADT_ERR_ARG
    one = lib.segment_array([(16, 10, 0, 2)])
    other = lib.segment_array([(16, 10, 0, 3)])                          # device side disagrees
    assert h.adt_host_to_device(one, other, 1, 64, 64, 1 << 20, None, 0, 0, None) == lib.ADT_ERR_ARG
    assert h.adt_host_to_device(one, one, 1, 64, 64, 8, None, 0, 0, None) == lib.ADT_ERR_ARG   # stream too short
    # _ex: unknown flag bits, DIRECT_FULL or ZERO_COPY without device segments, and ZERO_COPY from
    # staging that is not page-locked, are refused before any work
    assert h.adt_host_to_device_ex(one, one, 1, 64, 64, 1 << 20, None, 0, 0, 8, None, None) == lib.ADT_ERR_ARG
    assert h.adt_host_to_device_ex(one, None, 1, 64, 64, 1 << 20, None, 0, 0, lib.H2D_DIRECT_FULL, None,
                                   None) == lib.ADT_ERR_ARG
    assert h.adt_host_to_device_ex(one, None, 1, 64, 64, 1 << 20, None, 0, 0, lib.H2D_ZERO_COPY, None,
                                   None) == lib.ADT_ERR_ARG
    assert h.adt_host_to_device_ex(one, one, 1, 64, 64, 1 << 20, None, 0, 0, lib.H2D_ZERO_COPY, None,
                                   None) == lib.ADT_ERR_ARG
    assert h.adt_sumsq_f64(None, 10, 16, 16, None) == lib.ADT_ERR_ARG
    assert h.adt_sumsq_f64(12, 10, 16, 16, None) == lib.ADT_ERR_ALIGN
    n = ctypes.c_uint64(0)
    assert h.adt_sumsq_f64_partials(10 ** 9, ctypes.byref(n)) == lib.ADT_OK and 1 <= n.value <= 1184
    t = ctypes.c_int(0)
    assert h.adt_host_threads(ctypes.byref(t)) == lib.ADT_OK and t.value == len(os.sched_getaffinity(0))


def test_reference_plug_binds_the_hot_path_modules(tmp_path):
    """tests/refsuite/plug: the UNMODIFIED reference package (baseline/_ref)
    imports with weightpack.codec / weightpack.precision bound to this
    package and every other module from the reference — checked without a
    GPU (nothing is called); the GPU run of the suite is
    tests/test_gpu_reference_suite.py."""
    import subprocess
    import sys
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "weightpack")):
        pytest.skip("baseline/_ref not installed (run __graft_entry__.build() where /root/reference exists)")
    code = (
        "import sys; sys.path.insert(0, %r); import run; run.install_plugged(%r)\n"
        "import weightpack, weightpack.training as t, weightpack.cli as c, weightpack.transfer as tr\n"
        "import paper_2004_02297_b200.codec as oc, paper_2004_02297_b200.precision as op\n"
        "assert weightpack.pack_vectorized is oc.pack_vectorized and weightpack.l2_norm is op.l2_norm\n"
        "assert t.unpack is oc.unpack and c.codec is oc and tr.PackedBlock is oc.PackedBlock\n"
        "assert t.__file__.startswith(%r)\n"
        "print('plug ok')\n") % (os.path.join(ROOT, "tests", "refsuite"), ref, os.path.join(ref, "weightpack"))
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=tmp_path)
    assert p.returncode == 0 and "plug ok" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]
