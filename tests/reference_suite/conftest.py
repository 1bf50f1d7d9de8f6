"""Run the reference package's own tests against the drop-in.

``stage.py`` copies ``/root/reference/pkg/tests`` (unmodified) into the
git-ignored ``_staged/``.  Here ``podsketch`` and its submodules are aliased
to ``paper_1905_05107_b200`` before those files are collected, and every
staged test is marked ``gpu``.  Tests that cannot apply to the drop-in are
deselected below, each with its reason.
"""

from __future__ import annotations

import importlib
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1905_05107_b200 as _pkg  # noqa: E402

SUBMODULES = ("baselines", "cli", "errors", "isma", "matcore", "merge", "ooc", "podio",
              "quality", "reporting", "sampling")
sys.modules["podsketch"] = _pkg
for _name in SUBMODULES:
    sys.modules[f"podsketch.{_name}"] = importlib.import_module(f"paper_1905_05107_b200.{_name}")

# subprocesses (python -m podsketch, test_cli.py:392-406) find the alias package
SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "shim")
os.environ["PYTHONPATH"] = os.pathsep.join(
    [SHIM, ROOT] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])

STAGED = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_staged")

#: reference tests that do not apply to the drop-in (node id substring -> reason)
EXCLUDED = {
    "TestPlots": "renders PNG figures; matplotlib is absent from this image",
    "plot": "PNG figures need matplotlib, absent from this image (reporting.render_plots); "
            "the reference's own run deselects them too (SURVEY.md section 0)",
    "report_and_plot": "writes PNG figures (matplotlib absent)",
    "rerenders": "re-renders PNG figures (matplotlib absent)",
}


def pytest_collection_modifyitems(config, items):
    keep, dropped = [], []
    for item in items:
        if not str(item.fspath).startswith(STAGED):
            keep.append(item)
            continue
        item.add_marker(pytest.mark.gpu)
        if any(key in item.nodeid for key in EXCLUDED):
            dropped.append(item)
        else:
            keep.append(item)
    if dropped:
        config.hook.pytest_deselected(items=dropped)
        items[:] = keep
