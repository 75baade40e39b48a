"""The C-ABI library loads and exports every symbol include/ldpc_b200.h declares (no GPU calls)."""

import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "ldpc_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\**\s*(ldpc_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("ldpc_graph_create", "ldpc_decode", "ldpc_decoder_decode_host", "ldpc_phase_to_variable",
              "ldpc_count_errors", "ldpc_last_error"):
        assert s in syms


def test_library_exports_all_symbols():
    from paper_1609_01567_b200 import _native

    L = _native.load_library()
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert L.ldpc_abi_version() == 1


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch

    from paper_1609_01567_b200 import _native

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    try:
        _native.lib()
    except RuntimeError as e:
        assert "no CUDA device" in str(e)
    else:
        raise AssertionError("decoder must refuse to run without a CUDA device")
