"""The C-ABI library loads and exports every symbol include/ldpc_b200.h declares, and a plain-C client
builds against it (CPU); the C client decodes like the Python API (GPU)."""

import re

import pytest

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


def test_plain_c_client_compiles(tmp_path):
    # the C ABI is usable from C alone (no Python, no torch types): examples/c_api_demo.c builds
    import shutil
    import subprocess

    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no C compiler")
    lib_dir = ROOT / "paper_1609_01567_b200" / "_native"
    out = tmp_path / "c_api_demo"
    r = subprocess.run([gcc, "-O2", "-Wall", "-Werror", "-std=c11", f"-I{ROOT / 'include'}", "-o", str(out),
                        str(ROOT / "examples" / "c_api_demo.c"), f"-L{lib_dir}", "-lldpc_b200", "-lm"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_plain_c_client_matches_python(cuda, tmp_path):
    # run the C demo on the GPU and decode the same priors through the Python API
    import math
    import os
    import subprocess

    import numpy as np

    from conftest import PAIRS_14_7
    from paper_1609_01567_b200 import CodeTables, ParallelDecoder, ParityCheckMatrix

    lib_dir = ROOT / "paper_1609_01567_b200" / "_native"
    exe = tmp_path / "c_api_demo"
    subprocess.run(["gcc", "-O2", "-std=c11", f"-I{ROOT / 'include'}", "-o", str(exe),
                    str(ROOT / "examples" / "c_api_demo.c"), f"-L{lib_dir}", "-lldpc_b200", "-lm"], check=True)
    env = dict(os.environ, LD_LIBRARY_PATH=str(lib_dir))
    lines = subprocess.run([str(exe)], capture_output=True, text=True, env=env, check=True).stdout.splitlines()
    sigma2 = 0.5
    P = np.array([[1.0 / (1.0 + math.exp((-2.0 * (-1.0 + (1.6 if j in (f, f + 5) else 0.1 * ((j * 7 + f) % 5 - 2))))
                                          / sigma2)) for j in range(14)] for f in range(3)])
    with ParallelDecoder(CodeTables.from_matrix(ParityCheckMatrix(14, 7, PAIRS_14_7)), max_batch=3) as dec:
        res = dec.decode_priors(P, 50)
    assert len(lines) == 6
    for f, line in enumerate(lines[:3]):
        bits = "".join(str(int(b)) for b in res.estimates()[f])
        assert line == f"frame {f}: success={int(res.success[f])} iterations={int(res.iterations[f])} estimate={bits}"
    # observation input through the C ABI equals the Python decode_batch(Y, sigma2)
    Y = np.array([[-1.0 + (1.6 if j in (f, f + 5) else 0.1 * ((j * 7 + f) % 5 - 2)) for j in range(14)]
                  for f in range(3)])
    with ParallelDecoder(CodeTables.from_matrix(ParityCheckMatrix(14, 7, PAIRS_14_7)), max_batch=3) as dec:
        obs = dec.decode_batch(Y, sigma2, 50)
    for f, line in enumerate(lines[3:]):
        bits = "".join(str(int(b)) for b in obs.estimates()[f])
        assert line == (f"obs frame {f}: success={int(obs.success[f])} iterations={int(obs.iterations[f])} "
                        f"estimate={bits}")
