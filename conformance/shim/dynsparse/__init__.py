"""`dynsparse` -> paper_2502_07590_b200 import shim (conformance runs only).

Maps the reference package name and every submodule its test suite imports onto this
repo's modules, so /root/reference/pkg/tests run unmodified against the B200 build:
`from dynsparse.selection import streaming_topk` resolves to
paper_2502_07590_b200.selection.streaming_topk (the device implementation).
"""

import importlib
import sys

from paper_2502_07590_b200 import *  # noqa: F401,F403
from paper_2502_07590_b200 import __all__, __version__  # noqa: F401

_MODULES = ("attention", "cpmodel", "cpsim", "dispatcher", "flops", "grid", "grouping",
            "predictor", "profiler", "selection", "serialize", "synthetic")
for _name in _MODULES:
    _mod = importlib.import_module(f"paper_2502_07590_b200.{_name}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod
