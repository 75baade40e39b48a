"""``edgeldpc`` alias of paper_1609_01567_b200, for running the reference's own test suite.

TEST INFRASTRUCTURE ONLY (tests/test_reference_suite.py).  The reference's tests import
``edgeldpc`` and ``edgeldpc.tables``; this shim points every public name and every submodule
of the reference package (edgeldpc/__init__.py:1-91) at this package, so the suite runs
unmodified against the B200 implementation.
"""

import sys

import paper_1609_01567_b200 as _impl
from paper_1609_01567_b200 import *  # noqa: F401,F403
from paper_1609_01567_b200 import channel as _channel
from paper_1609_01567_b200 import cli as _cli
from paper_1609_01567_b200 import codes as _codes
from paper_1609_01567_b200 import decoder as _decoder
from paper_1609_01567_b200 import tables as _tables

__all__ = list(_impl.__all__)
__version__ = _impl.__version__

# reference submodule -> the module of this package that holds its names
for _name, _mod in {"codes": _codes, "tables": _tables, "serial": _decoder, "engine": _decoder,
                    "rng": _channel, "channel": _channel, "cli": _cli}.items():
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
del _name, _mod
