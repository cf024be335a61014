"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/qigen_b200.h declares, and the host logic (config validation,
planner, Morton order, payload formula) matches the reference's fixtures."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2307_03738_b200 as q
from paper_2307_03738_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "qigen_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(qigen_\w+)\s*\(", text,
                                 flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "qigen_gemv" in syms and "qigen_quantize" in syms and len(syms) >= 18


def test_library_loads_and_exports_every_symbol():
    lib = _lib.lib()  # loads libqigen_b200.so (no device needed)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) <= set(_lib.SIGNATURES)
    assert lib.qigen_version() >= 100


def test_size_queries_without_gpu():
    lib = _lib.lib()
    # 4096x4096 4-bit: 256 panels x 16 supersteps x 4 uint4 x 32 lanes x 4 words
    assert lib.qigen_panel_words(4096, 4096, 4) == 4096 * 4096 * 4 // 32
    assert lib.qigen_panel_words(11008, 4096, 3) == 4096 * 11008 * 3 // 32
    assert lib.qigen_panel_params(4096, 4096, 128) == 256 * 32 * 16
    assert lib.qigen_panel_params(4096, 4096, 0) == 256 * 16
    # padding: K rounded to 256, N to 16
    assert lib.qigen_panel_words(100, 20, 2) == 2 * 1 * 2 * 32 * 4


def test_quant_config_validation():
    with pytest.raises(q.ConfigError):
        q.QuantConfig(bits=5)
    with pytest.raises(q.ConfigError):
        q.QuantConfig(bits=4, group_size=0)
    with pytest.raises(q.ConfigError):
        q.QuantConfig(4, 128).groups_for_rows(100)
    with pytest.raises(q.ConfigError):
        q.QuantConfig(4, None, "int8")
    assert q.QuantConfig(3, 64, "QUANTIZED").zero_mode is q.ZeroMode.QUANTIZED
    assert q.QuantConfig(3, None).groups_for_rows(4096) == 1
    assert q.pack_unit(3) == (32, 3) and q.pack_unit(2) == (16, 1) and q.pack_unit(4) == (8, 1)
    with pytest.raises(q.ConfigError):
        q.check_row_count(40, 3)


def test_plans_match_reference_fixtures(golden_plans):
    for p in golden_plans:
        hw = q.HardwareSpec(l1_bits=p.get("l1_bits", 262144), vregs=p.get("vregs", 16))
        cfg = q.QuantConfig(p["bits"], p["g"])
        if "error" in p:
            with pytest.raises(ValueError):
                q.plan(hw, cfg, tuple(p["dims"]))
        else:
            t = q.plan(hw, cfg, tuple(p["dims"]))
            assert [t.m_u, t.t_u, t.m_b, t.t_b] == p["plan"], p


def test_morton_and_block_order(golden_kats):
    for key, v in golden_kats["morton"].items():
        r, c = map(int, key.split(","))
        assert q.morton_index(r, c) == v
    assert [list(t) for t in q.block_order(2, 2)] == golden_kats["block_order_2x2"]
    # bijection on a 2^k x 2^k grid
    assert sorted(q.morton_index(r, c) for r in range(8) for c in range(8)) == list(range(64))


def test_register_tiles(golden_kats):
    assert list(q.select_register_tile(q.HardwareSpec(vregs=16))) == golden_kats["reg_tile_16"]
    assert list(q.select_register_tile(q.HardwareSpec(vregs=3))) == golden_kats["reg_tile_3"]
    with pytest.raises(q.PlanError):
        q.select_register_tile(q.HardwareSpec(vregs=2))


def test_hardware_spec_file(tmp_path):
    f = tmp_path / "hw.txt"
    f.write_text("l1_bits = 8192  # small\nvregs 8\n")
    hw = q.load_hardware_spec(f)
    assert hw.l1_bits == 8192 and hw.vregs == 8
    q.save_hardware_spec(hw, f)
    assert q.load_hardware_spec(f) == hw
    f.write_text("cache = 3\n")
    with pytest.raises(q.ConfigError):
        q.load_hardware_spec(f)


def test_payload_bits_formula(golden_kats):
    import torch
    cfg = q.QuantConfig(4, None, "quantized")
    pm = q.PackedMatrix(torch.zeros(4096 * 4096 // 8, dtype=torch.int32), 4096, 4096, cfg,
                        torch.ones(1, 4096), torch.zeros(1, 4096), q.TilePlan(3, 3, 24, 2040))
    assert list(pm.payload_bits()) == golden_kats["payload_bits_4096_b4_fc_q"]
    rep = q.memory_report(pm)
    assert rep["total_bits"] == 67_256_320
    assert abs(rep["ratio"] - 32 / 4) / 8 < 0.01
