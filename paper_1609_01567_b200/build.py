"""Build libldpc_b200.so (sm_100a) in-tree: ``python -m paper_1609_01567_b200.build``."""

from __future__ import annotations

import os
import pathlib
import subprocess
import sys

HERE = pathlib.Path(__file__).resolve().parent


def build(jobs: int | None = None, verbose: bool = False) -> pathlib.Path:
    jobs = jobs or min(8, os.cpu_count() or 1)
    cmd = ["make", "-C", str(HERE / "csrc"), f"-j{jobs}"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        sys.stderr.write((out.stdout or "") + (out.stderr or ""))
        raise RuntimeError("native build failed")
    lib = HERE / "_native" / "libldpc_b200.so"
    if not lib.exists():
        raise RuntimeError(f"build did not produce {lib}")
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
