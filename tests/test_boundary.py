"""The C-ABI library and the host-side mirror of the reference interface
(no compute calls: these run without a GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import powersgd as O
from paper_1905_13727_b200 import _lib, catalogs, seeding
from paper_1905_13727_b200.compressor import (COMPRESSORS, CompressionContext, LowRank, PowerSGD,
                                              decode_cost, make_compressor)
from paper_1905_13727_b200.linalg import ContractViolation

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "psgd_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psgd_[a-z_0-9]+)\s*\(", text)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert set(names) == set(_lib.EXPORTS)
    for name in names:
        assert getattr(lib, name) is not None
    assert lib.psgd_version() >= 2


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    assert "sm_100a" in out.stdout


def test_invalid_arguments_are_reported_without_a_gpu():
    lib = _lib.load()
    h = ctypes.c_void_p()
    n = (ctypes.c_int64 * 1)(4)
    m = (ctypes.c_int64 * 1)(4)
    assert lib.psgd_plan_create(1, n, m, 0, 1, 0, ctypes.byref(h)) == _lib.PSGD_EINVAL
    assert b"rank" in lib.psgd_last_error()
    assert lib.psgd_plan_create(1, n, m, 2, 0, 0, ctypes.byref(h)) == _lib.PSGD_EINVAL
    assert lib.psgd_tree_mean(None, 2, 10, None, None) == _lib.PSGD_EINVAL
    assert lib.psgd_plan_destroy(None) == 0


def test_seeding_is_the_reference_stream():
    for labels in [("warm_start_init", 0), ("warm_start_init", 21), ("grad", 3, 1, 7)]:
        a = seeding.derive_rng(5, *labels).standard_normal(17)
        b = O.derive_rng(5, *labels).standard_normal(17)
        assert np.array_equal(a, b)
    for n, j, a in [(9, 1, 0), (512, 0, 0), (28869, 3, 0), (2, 1, 1), (7, 0, 2)]:
        assert np.array_equal(seeding.replacement_column(n, j, a), O.replacement_column(n, j, a))
    assert np.array_equal(seeding.warm_start_q(0, 4, 2304, 2),
                          O.CompressionContext(0, 4).param_rng("warm_start_init").standard_normal((2304, 2)))


def test_catalogs_mirror_reference():
    assert [(s.name, s.shape) for s in catalogs.RESNET18.params] == [(s.name, s.shape) for s in O.RESNET18]
    assert [(s.name, s.shape) for s in catalogs.LSTM.params] == [(s.name, s.shape) for s in O.LSTM]
    st = catalogs.stress()
    assert len(st.params) == 256 and sum(p.size for p in st.params) == 4_294_967_296


def test_compressor_accounting_matches_reference():
    ours, ref = PowerSGD(2), O.PowerSGD(2)
    for n, m in [(3, 7), (512, 4608), (10, 512), (64, 27), (5, 1)]:
        assert ours.effective_rank(n, m) == ref.effective_rank(n, m)
        assert ours.payload_bits(n, m) == ref.payload_bits(n, m)
        assert ours.compress_cost(n, m) == ref.compress_cost(n, m)
    assert PowerSGD.linear and PowerSGD.route == "allreduce" and PowerSGD.uses_error_feedback
    assert set(COMPRESSORS) == {"powersgd", "bestapprox", "unbiased"}
    for name, cls in (("bestapprox", O.BestApproximation), ("unbiased", O.UnbiasedRankK)):
        for r in (1, 2, 5):
            a, b = make_compressor(name, r), cls(r)
            assert a.linear and a.route == "allreduce" and a.uses_error_feedback
            for n, m in [(3, 7), (512, 4608), (64, 27)]:
                assert a.payload_bits(n, m) == b.payload_bits(n, m)
                assert a.compress_cost(n, m) == b.compress_cost(n, m)
    with pytest.raises(ContractViolation):
        make_compressor("topk")
    with pytest.raises(ContractViolation):
        make_compressor("powersgd", rank=0)
    assert decode_cost(LowRank(np.zeros((6, 2)), np.zeros((5, 2)))) == 2 * 6 * 5 * 2
    ctx = CompressionContext(3, 4, 5)
    assert np.array_equal(ctx.rng("x").standard_normal(3), O.derive_rng(3, "x", 4, 5).standard_normal(3))


def test_transfer_groups_cover_every_parameter_once():
    """pipeline.transfer_groups: small first and last groups, every parameter once."""
    from paper_1905_13727_b200 import catalogs
    from paper_1905_13727_b200.pipeline import transfer_groups
    for name in ("resnet18", "lstm"):
        specs = list(catalogs.get_catalog(name).params)
        total = sum(s.size for s in specs)
        for groups in (3, 4, 8, 12):
            gs = transfer_groups(specs, groups)
            flat = sorted(i for g in gs for i in g)
            assert flat == list(range(len(specs)))
            assert all(g == sorted(g) for g in gs)
            if name == "resnet18":
                sizes = [sum(specs[i].size for i in g) for g in gs]
                assert sizes[0] <= 0.1 * total and sizes[-1] <= 0.1 * total, sizes
