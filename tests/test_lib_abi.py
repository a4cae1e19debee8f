"""Host-side checks of the boundary (no GPU needed): the C-ABI library builds,
loads, exports every symbol include/srt.h declares, and validates configs /
arguments on the host before touching a device."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2601_09083_b200 import build
    build.build()
    from paper_2601_09083_b200 import _lib
    return _lib.load()


def test_header_symbols_exported(lib):
    from paper_2601_09083_b200 import _lib
    hdr = (ROOT / "include" / "srt.h").read_text()
    declared = set(re.findall(r"SRT_API\s+[\w\s\*]*?\b(srt_\w+)\s*\(", hdr))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.srt_abi_version() == 1


def test_struct_layout_matches_header():
    from paper_2601_09083_b200._lib import SrtConfig, SrtDumpRecord, SrtCacheStats
    # srt_config: 8 x i32, double, 3 x i64, enum(int) -> 72 bytes with tail padding
    assert ctypes.sizeof(SrtConfig) == 72
    assert SrtConfig.min_path_score.offset == 32 and SrtConfig.node_capacity.offset == 40
    assert ctypes.sizeof(SrtDumpRecord) == 16 and ctypes.sizeof(SrtCacheStats) == 40


def _cfg(**kw):
    from paper_2601_09083_b200._lib import SrtConfig
    base = dict(vocab_size=100, max_prompts=2, max_depth=8, max_match_len=4, budget_max=8,
                budget_base=8, budget_slope_num=0, budget_slope_den=1, min_path_score=0.0,
                node_capacity=1024, hash_capacity=4096, slot_capacity=2048, logits_dtype=0)
    base.update(kw)
    return SrtConfig(**base)


@pytest.mark.parametrize("bad", [dict(vocab_size=1), dict(max_match_len=9), dict(max_match_len=33, max_depth=40),
                                 dict(budget_max=65), dict(budget_base=9), dict(budget_slope_den=0),
                                 dict(hash_capacity=3000), dict(hash_capacity=1024),
                                 dict(node_capacity=2), dict(logits_dtype=7),
                                 dict(min_path_score=-1.0)])
def test_invalid_config_rejected_on_host(lib, bad):
    h = ctypes.c_void_p()
    r = lib.srt_cache_create(ctypes.byref(_cfg(**bad)), None, ctypes.byref(h))
    assert r == 1 and not h.value  # SRT_ERR_INVALID_CONFIG, nothing allocated


def test_invalid_args_rejected_on_host(lib):
    assert lib.srt_insert(None, 1, None, None, 0, None, None, None, None, None) == 2
    assert lib.srt_cache_destroy(None, None) == 0
    assert lib.srt_noise_table(None, None) == 2
    assert lib.srt_cache_status(None, None, None, None) == 2


def test_product_package_does_not_import_oracle():
    """The product path never touches oracle/ (DESIGN.md §1)."""
    for p in (ROOT / "paper_2601_09083_b200").rglob("*"):
        if p.suffix in (".py", ".cu", ".cuh", ".h"):
            txt = p.read_text()
            assert "import oracle" not in txt and "from oracle" not in txt, p
            assert "srt_oracle" not in txt and "liboracle" not in txt, p
