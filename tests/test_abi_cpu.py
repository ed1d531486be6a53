"""The C-ABI library loads without a GPU, exports every symbol the header
declares, and rejects bad arguments with the documented codes before any
CUDA call is made."""
import ctypes
import os
import re

import pytest

from paper_1611_02665_b200 import _abi
from paper_1611_02665_b200.errors import ConfigError, ContractError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "spo_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spo_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    return _abi.load()


def test_library_exports_every_header_symbol(lib):
    syms = header_symbols()
    assert len(syms) >= 8
    raw = ctypes.CDLL(_abi.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), s
    assert set(syms) == set(_abi.EXPORTS)


def test_abi_version(lib):
    assert lib.spo_abi_version() == 6
    assert lib.spo_eval_ratios_workspace_bytes(2, 0, 128, 32, 1000) > 1000 * 160 + 32 * 1000 * 10 * 8 - 1
    assert lib.spo_eval_ratios_workspace_bytes(2, 0, 96, 1, 1000) == -1  # 384-byte rows
    assert lib.spo_eval_workspace_bytes(2, 0, 0, 1000) >= 1000 * 160
    assert lib.spo_eval_workspace_bytes(2, 1, 0, 1000) >= 1000 * 304  # fp64 records
    assert lib.spo_eval_workspace_bytes(2, 0, 1, 1000) == 0  # strict: generic kernel only
    assert lib.spo_eval_workspace_bytes(9, 0, 0, 1000) == -1


def _eval(lib, **kw):
    a = dict(kind=2, dtype=0, mode=0, table=16, n3=(16, 16, 16), nb=64, n_tiles=1,
             dinv=(16.0,) * 3, delta=(1 / 16,) * 3, pos=16, n=10, out=16, ps=640, ss=64)
    a.update(kw)
    return lib.spo_eval(a["kind"], a["dtype"], a["mode"], a["table"], _abi.i32x3(a["n3"]), a["nb"],
                        a["n_tiles"], _abi.f64x3(a["dinv"]), _abi.f64x3(a["delta"]), a["pos"], a["n"],
                        a["out"], a["ps"], a["ss"], None, None, None, 0, None)


def test_eval_argument_validation(lib):
    assert _eval(lib, kind=7) == 1
    assert _eval(lib, dtype=3) == 1
    assert _eval(lib, mode=5) == 1
    assert _eval(lib, mode=1, dtype=1, nb=64, ps=640) == 3  # strict is fp32 only
    assert _eval(lib, nb=48) == 1                             # not a 128-byte row
    assert _eval(lib, n3=(3, 16, 16)) == 3                     # grid too small
    assert _eval(lib, table=8) == 1                            # misaligned
    assert _eval(lib, ss=32) == 1                              # streams overlap lanes
    assert _eval(lib, ps=320) == 1                             # positions overlap
    assert _eval(lib, n=0) == 0                                # empty batch: no-op
    assert _eval(lib, dinv=(0.0, 1.0, 1.0)) == 3
    assert b"positive" in lib.spo_last_error()
    # k-power table form (SPO_TABLE_KPOWER): FAST only
    assert _eval(lib, mode=1 | _abi.TABLE_KPOWER) == 3
    assert b"B-spline table form" in lib.spo_last_error()
    assert _eval(lib, mode=_abi.TABLE_KPOWER, n=0) == 0
    assert _eval(lib, mode=0x200) == 1                          # unknown flag
    assert lib.spo_eval_workspace_bytes(2, 0, _abi.TABLE_KPOWER, 1000) == lib.spo_eval_workspace_bytes(2, 0, 0, 1000)
    assert lib.spo_eval_path(2, 0, 1 | _abi.TABLE_KPOWER, _abi.i32x3((16, 16, 16)), 64, 1, 10, 0) == -1


def test_pack_kpower_validation(lib):
    n3 = _abi.i32x3((8, 8, 8))
    assert lib.spo_pack_kpower(5, 16, n3, 64, 1, 16, None) == 1     # dtype
    assert lib.spo_pack_kpower(0, 16, n3, 48, 1, 16, None) == 1     # row not 128-byte
    assert lib.spo_pack_kpower(0, None, n3, 64, 1, 16, None) == 1   # NULL
    assert lib.spo_pack_kpower(0, 8, n3, 64, 1, 16, None) == 1      # misaligned
    assert lib.spo_pack_kpower(0, 16, _abi.i32x3((8, 2, 8)), 64, 1, 16, None) == 3


def _eval_lanes(lib, limit, **kw):
    a = dict(kind=2, dtype=0, mode=0, table=16, n3=(16, 16, 16), nb=64, n_tiles=1,
             dinv=(16.0,) * 3, delta=(1 / 16,) * 3, pos=16, n=10, out=16, ps=640, ss=64)
    a.update(kw)
    return lib.spo_eval_lanes(a["kind"], a["dtype"], a["mode"], a["table"], _abi.i32x3(a["n3"]), a["nb"],
                              a["n_tiles"], _abi.f64x3(a["dinv"]), _abi.f64x3(a["delta"]), a["pos"], a["n"],
                              a["out"], a["ps"], a["ss"], limit, None, None, None, 0, None)


def test_eval_lanes_argument_validation(lib):
    assert _eval_lanes(lib, -1) == 1
    assert _eval_lanes(lib, 0) == 1                 # at least one lane
    assert _eval_lanes(lib, 65) == 1                # beyond the table's lanes
    assert _eval_lanes(lib, 40, ss=32) == 1         # streams overlap the stored lanes
    assert _eval_lanes(lib, 20, ss=20, ps=200, n=0) == 0  # empty batch: no-op
    assert _eval_lanes(lib, 20, ss=22) == 1         # strides must be multiples of 4 lanes
    assert b"multiples" in lib.spo_last_error()


def test_eval_path_selection(lib, monkeypatch):
    """spo_eval_path: the kernel spo_eval would run (no device needed)."""
    monkeypatch.delenv("SPO_LINE", raising=False)
    n3 = _abi.i32x3((64, 64, 64))
    big = 1 << 40
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 1048576, big) == 2   # >= 4 positions per cell: line
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 262144, big) == 3    # 0.3 .. 4 per cell: window
    assert lib.spo_eval_path(1, 0, 0, n3, 128, 32, 262144, big) == 3    # VGL too
    assert lib.spo_eval_path(0, 0, 0, n3, 128, 32, 786432, big) == 2    # V from 2.8 per cell: line
    assert lib.spo_eval_path(0, 0, 0, n3, 128, 32, 655360, big) == 3    # V 1.1 .. 2.8: the 2 x 1 window
    assert lib.spo_eval_path(0, 1, 0, n3, 64, 64, 983040, big) == 3     # fp64 V below 4 per cell: window
    assert lib.spo_eval_path(0, 1, 0, n3, 64, 64, 1048576, big) == 2    # fp64 V from 4: line
    assert lib.spo_eval_path(0, 0, 0, n3, 128, 32, 262144, big) == 3    # V 0.4 .. 1.1 per cell: 2 x 2 window
    assert lib.spo_eval_path(0, 0, 0, n3, 128, 32, 78643, big) == 1     # V below 0.3 per cell: TMA
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 60000, big) == 1     # sparser: per-position TMA
    assert lib.spo_eval_path(2, 0, 1, n3, 128, 32, 262144, big) == 0    # strict: generic
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 262144, 0) == 0      # no workspace: generic
    assert lib.spo_eval_path(2, 1, 0, n3, 64, 64, 262144, big) == 3     # fp64 too
    assert lib.spo_eval_path(2, 0, 0, n3, 96, 1, 262144, big) == 1      # rows not 512-byte multiples
    need = lib.spo_eval_workspace_bytes(2, 0, 0, 262144)
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 262144, need) == 3
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 262144, need - 1) == 1  # short workspace: TMA
    monkeypatch.setenv("SPO_LINE", "1")
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 262144, big) == 2
    monkeypatch.setenv("SPO_LINE", "2")
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 60000, big) == 3
    monkeypatch.setenv("SPO_LINE", "0")
    assert lib.spo_eval_path(2, 0, 0, n3, 128, 32, 262144, big) == 1
    assert lib.spo_eval_path(9, 0, 0, n3, 128, 32, 262144, big) == -1


def test_error_codes_map_to_reference_exceptions(lib):
    _eval(lib, kind=7)
    with pytest.raises(ContractError):
        _abi.check(1)
    with pytest.raises(ConfigError):
        _abi.check(3)


def test_pack_and_fill_validation(lib):
    n3 = _abi.i32x3((8, 8, 8))
    assert lib.spo_pack_table(0, 16, 16, 16, n3, 16, 30, 1, 16, None) == 1   # nb not 128 B
    assert lib.spo_pack_table(0, 16, 16, 64, n3, 16, 32, 2, 16, None) == 3   # tiles too small
    assert lib.spo_fill_uniform(16, 0, n3, 16, 32, 1, 16, None) == 3
    assert lib.spo_fill_normal_f64(16, 16, n3, 16, 8, 1, 16, None) == 1     # nb not 128 B


def test_oracle_library_builds_and_loads():
    import oracle

    L = oracle.lib()
    assert L.orc_abi_version() == 1
