"""Run the reference's own unit suites (staged by ``stage.py``) against the
drop-in: ``import kapsm`` resolves to ``paper_2201_05024_b200`` and every
staged test is a GPU test (the package has no CPU fallback)."""

import os
import sys

import pytest

import paper_2201_05024_b200 as _pkg

sys.modules["kapsm"] = _pkg
for _name in ("apsm", "bench", "engine", "kernels", "modelio", "noma"):
    sys.modules[f"kapsm.{_name}"] = getattr(_pkg, _name)

_HERE = os.path.dirname(os.path.abspath(__file__))


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(_HERE):
            item.add_marker(pytest.mark.gpu)
