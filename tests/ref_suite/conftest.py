"""Runs the reference's own test suite (tests/ref_suite/test_*.py, vendored
UNCHANGED from /root/reference/pkg/tests) against the B200 package under the
reference's module name (compat/fastsum -> paper_2506_02219_b200).

This file replaces the reference's conftest.py: the same ``rng`` fixture
(seed 12345) and acceptance-gate summary hook (reference conftest.py:7-16),
plus the wiring for this repository:
  * ``compat/`` first on sys.path and on PYTHONPATH (acceptance criterion 10
    starts ``python -m fastsum.cli`` in a subprocess);
  * every test here is marked ``gpu`` (the package has no CPU fallback);
  * test_cli.py is not collected: the CLI is outside the hot path (tier
    framing); compat/fastsum/cli.py only covers what the gate drives.
"""

import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
COMPAT = os.path.join(ROOT, "compat")
for p in (ROOT, COMPAT, HERE):
    if p not in sys.path:
        sys.path.insert(0, p)
os.environ["PYTHONPATH"] = os.pathsep.join(
    [COMPAT, ROOT] + [p for p in os.environ.get("PYTHONPATH", "").split(os.pathsep) if p])

import _gate  # noqa: E402

collect_ignore = ["test_cli.py"]


def pytest_collection_modifyitems(config, items):
    for item in items:
        if str(item.fspath).startswith(HERE):
            item.add_marker(pytest.mark.gpu)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def pytest_terminal_summary(terminalreporter):
    if _gate.lines:
        terminalreporter.section("acceptance gate")
        for line in _gate.lines:
            terminalreporter.write_line(line)
