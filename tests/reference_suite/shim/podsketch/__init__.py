"""``podsketch`` -> ``paper_1905_05107_b200`` alias for subprocesses of the
staged reference suite (``python -m podsketch ...``, test_cli.py:392-406);
conftest.py puts this directory on PYTHONPATH."""

import importlib
import sys

import paper_1905_05107_b200 as _pkg
from paper_1905_05107_b200 import *  # noqa: F401,F403

for _name in ("baselines", "cli", "errors", "isma", "matcore", "merge", "ooc", "podio",
              "quality", "reporting", "sampling"):
    sys.modules[f"{__name__}.{_name}"] = importlib.import_module(f"paper_1905_05107_b200.{_name}")
__version__ = _pkg.__version__
