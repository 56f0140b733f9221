"""pytest plugin: run the reference's own test suite against this package.

Loaded with `-p alias_plugin` by tests/test_reference_suite.py.  Every
`tensorplace` module the reference tests import resolves to the module of
the same name in `paper_2111_00655_b200`; `tensorplace.oracle` (the
reference's exhaustive verifiers, a test utility) is the staged reference
file, executed on top of this package.  `tensorplace.cli` is out of scope
(DESIGN.md): its `main` skips the calling test.
"""

from __future__ import annotations

import importlib
import importlib.util
import os
import sys
import types

REPO = os.environ.get("CB_REPO_ROOT") or os.path.dirname(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))))
SUITE = os.environ.get("CB_REF_SUITE") or os.path.join(REPO, "oracle", "_ref", "suite")
sys.path.insert(0, REPO)

import paper_2111_00655_b200 as _pkg  # noqa: E402

MODULES = ("cost", "dp", "errors", "evolution", "graph", "matching", "patterns", "placement",
           "registry", "rules")

sys.modules["tensorplace"] = _pkg
for _m in MODULES:
    sys.modules["tensorplace." + _m] = importlib.import_module("paper_2111_00655_b200." + _m)

_spec = importlib.util.spec_from_file_location(
    "tensorplace.oracle", os.path.join(SUITE, "_tensorplace_oracle.py"))
_oracle = importlib.util.module_from_spec(_spec)
sys.modules["tensorplace.oracle"] = _oracle
_spec.loader.exec_module(_oracle)
_pkg.oracle = _oracle


def _cli_main(argv=None):
    import pytest
    pytest.skip("the reference CLI (tensorplace/cli.py) is out of scope for the hot path")


_cli = types.ModuleType("tensorplace.cli")
_cli.main = _cli_main
sys.modules["tensorplace.cli"] = _cli
_pkg.cli = _cli
