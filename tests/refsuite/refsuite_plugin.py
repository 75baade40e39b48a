"""pytest plugin for the vendored reference suite (tests/test_reference_suite.py).

Marks the one reference test that fails on the reference itself as a strict xfail:
test_serial.py:113-123 (TestValuesToVariable::test_degree_two_check_copies_other_message)
expects r == q of the other edge exactly, but serial.py:111 computes 1 - (0.5 + 0.5*(1 - 2q)),
which rounds.  This package reproduces serial.py:111, so the test fails
here for the same reason it fails on the reference.  Every test is also marked ``gpu``.
"""

import pytest

XFAIL = {
    "test_serial.py::TestValuesToVariable::test_degree_two_check_copies_other_message":
        "fails on the reference too: serial.py:111 rounds 1-(0.5+0.5*(1-2q)) != q",
}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the CUDA path")


def pytest_collection_modifyitems(config, items):
    for item in items:
        item.add_marker(pytest.mark.gpu)
        key = item.nodeid.split("/")[-1]
        if key in XFAIL:
            item.add_marker(pytest.mark.xfail(reason=XFAIL[key], strict=True))
