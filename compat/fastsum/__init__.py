"""``fastsum`` -> paper_2506_02219_b200: the drop-in under the reference's name.

Put ``compat/`` on ``sys.path`` (or PYTHONPATH) and unmodified reference code,
including the reference's own test suite (tests/ref_suite/), runs on the B200
path.  Every reference module name is the SAME module object as its
counterpart here (``fastsum.estimators is paper_2506_02219_b200.estimators``),
so private helpers and monkeypatching behave as in the reference:

    fastsum            paper_2506_02219_b200   (reference __init__.py:9-31)
    fastsum._core      ._core       fastsum.octree     .octree
    fastsum.types      .types       fastsum.kernels    .kernels
    fastsum.rng        .rng         fastsum.estimators .estimators
    fastsum.bench      .bench       fastsum.scene_io   .scene_io
    fastsum.meshes     .scenes (meshes.py:14-114 live there)
    fastsum.estimator_api .estimator_api

``fastsum.cli`` (compat/fastsum/cli.py) is a thin shim: the CLI is outside the
B200 hot path; it covers the two subcommands the reference's acceptance gate
drives (criterion 10: ``eval`` and ``sweep``).
"""

import importlib
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2506_02219_b200 as _impl  # noqa: E402
from paper_2506_02219_b200 import *  # noqa: E402,F401,F403
from paper_2506_02219_b200 import __all__, __version__  # noqa: E402,F401

_MODULES = {"_core": "_core", "types": "types", "octree": "octree", "kernels": "kernels",
            "rng": "rng", "estimators": "estimators", "bench": "bench",
            "scene_io": "scene_io", "meshes": "scenes", "estimator_api": "estimator_api"}

for _name, _target in _MODULES.items():
    _mod = importlib.import_module(f"paper_2506_02219_b200.{_target}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod


def __getattr__(name):
    return getattr(_impl, name)
