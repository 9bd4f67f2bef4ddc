"""Conformance-run hooks: put the `dynsparse` shim first on sys.path and mark the reference
tests whose expectations this build deliberately does not meet (documented deviations;
strict xfail, so a deviation that disappears fails the run until it is removed here)."""

import sys
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE / "shim"))

# test node id suffix -> reason
DEVIATIONS = {
}


def pytest_collection_modifyitems(config, items):
    for item in items:
        for key, reason in DEVIATIONS.items():
            if item.nodeid.endswith(key):
                item.add_marker(pytest.mark.xfail(reason=reason, strict=True))
