"""Copy the reference's own test suite (/root/reference/pkg/tests) to baseline/_ref_tests.

TEST INFRASTRUCTURE ONLY.  The copy is git-ignored (reference sources never enter the repo's
history) but travels to the GPU box with the working tree, where
tests/test_reference_suite.py runs it against this package through the ``edgeldpc`` alias in
tests/refsuite/.  Run by __graft_entry__.build() when /root/reference is present.
"""

from __future__ import annotations

import pathlib
import shutil

ROOT = pathlib.Path(__file__).resolve().parents[2]
SRC = pathlib.Path("/root/reference/pkg/tests")
DST = ROOT / "baseline" / "_ref_tests"


def vendor() -> pathlib.Path | None:
    if not SRC.is_dir():
        return None
    if DST.exists():
        shutil.rmtree(DST)
    shutil.copytree(SRC, DST, ignore=shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache"))
    return DST


if __name__ == "__main__":
    print(vendor())
