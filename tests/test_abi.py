"""CPU-side checks of the C ABI: the library loads (no GPU needed for dlopen)
and exports every symbol include/cnmf_b200.h declares, with matching ctypes
signatures; host-side helpers agree with the reference golden vectors."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cnmf_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cnmf_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_api():
    syms = declared_symbols()
    assert "cnmf_structured_compress" in syms and "cnmf_admm_run" in syms and "cnmf_select_spa" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    from paper_1505_04650_b200 import _lib

    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} has no ctypes signature"
    assert set(_lib.SIGNATURES) == set(declared_symbols())
    assert lib.cnmf_abi_version() == 1


def test_panel_ld_and_errors_without_gpu():
    from paper_1505_04650_b200 import _lib

    lib = _lib.load()
    assert [lib.cnmf_panel_ld(s) for s in (1, 20, 32, 33, 60, 64, 100, 128, 129)] == [32, 32, 32, 64, 64, 64, 128,
                                                                                      128, -1]
    # argument validation happens before any device work
    st = lib.cnmf_structured_compress(None, 0, 0, 0, 20, 4, 0, 0, None, None, 0, None)
    assert st == 1 and "non-empty" in _lib.last_error()


def test_child_seed_matches_reference(golden):
    from paper_1505_04650_b200 import _lib
    from paper_1505_04650_b200.rng import child_seed

    lib = _lib.load()
    tags = list(golden["child_seed_tags"])
    for (s, i), want in zip(golden["child_seed_in"], golden["child_seed_out"]):
        assert child_seed(int(s), tags[int(i)]) == int(want)
        assert lib.cnmf_child_seed(int(s), tags[int(i)].encode("utf-8")) == int(want)


def test_status_maps_to_reference_exceptions():
    from paper_1505_04650_b200 import _lib, errors

    with pytest.raises(errors.ArgumentError):
        _lib.check(1)
    with pytest.raises(errors.InfeasibleRankError):
        _lib.check(2)
    with pytest.raises(errors.RankDeficiencyError) as info:
        _lib.check(4, picks=[3, 1])
    assert info.value.picks == [3, 1]
    assert issubclass(errors.InfeasibleRankError, ValueError)


def test_config_rules_match_reference(golden):
    from paper_1505_04650_b200 import CompressionConfig, InfeasibleRankError, adjust_config

    got = [(c.r, c.r_ov) for c in (adjust_config(CompressionConfig(5, 10), 2000, 1000),
                                   adjust_config(CompressionConfig(5, 10), 2000, 12),
                                   adjust_config(CompressionConfig(30, 10), 2000, 1000))]
    assert np.array_equal(np.array(got), golden["adjust"])
    with pytest.raises(InfeasibleRankError):
        adjust_config(CompressionConfig(r=12), 50, 12)


def _parse_tables():
    text = open(os.path.join(ROOT, "paper_1505_04650_b200", "csrc", "ziggurat_tables.h")).read()

    def block(name):
        body = re.search(name + r"\[256\] = \{(.*?)\};", text, re.S).group(1)
        return [x.strip() for x in body.split(",") if x.strip()]

    ki = [int(x.rstrip("ULL"), 16) for x in block("kKi")]
    wi = [float.fromhex(x) for x in block("kWi")]
    fi = [float.fromhex(x) for x in block("kFi")]
    return ki, wi, fi


def test_ziggurat_tables_reproduce_numpy():
    """The committed device tables decode numpy's Philox stream exactly (the
    device kernel uses the same tables and decode order)."""
    import sys

    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import gen_ziggurat as gz

    ki, wi, fi = _parse_tables()
    for seed in (3, 99, 2**64 - 7):
        ref, raw = gz.numpy_stream(seed, 30000)
        got, _ = gz.decode(raw, 30000, ki, wi, fi)
        assert np.array_equal(got, ref)
