"""Stage the reference's own test suite for the drop-in check.

TEST INFRASTRUCTURE ONLY.  `stage()` copies the reference package's tests
(`/root/reference/pkg/tests/*.py`) and its exhaustive verifier module
(`pkg/src/tensorplace/oracle.py`, which the tests import as
`tensorplace.oracle`) into `oracle/_ref/suite/` -- git-ignored like every
`oracle/_ref` output, so nothing of the reference enters the history, but it
travels to the GPU box with the working tree, where `/root/reference` does
not exist.  `tests/test_reference_suite.py` runs the staged files with
`tests/refsuite/alias_plugin.py`, which makes `import tensorplace` resolve to
`paper_2111_00655_b200`.
"""

from __future__ import annotations

import glob
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
SUITE = os.path.join(HERE, "_ref", "suite")
REF_PKG = "/root/reference/pkg"


def stage(ref_pkg: str = REF_PKG) -> str | None:
    """Copy the suite when the reference is present; return the staged dir."""
    tests = os.path.join(ref_pkg, "tests")
    if not os.path.isdir(tests):
        return SUITE if os.path.isdir(SUITE) else None
    os.makedirs(SUITE, exist_ok=True)
    for src in glob.glob(os.path.join(tests, "*.py")):
        shutil.copyfile(src, os.path.join(SUITE, os.path.basename(src)))
    shutil.copyfile(os.path.join(ref_pkg, "src", "tensorplace", "oracle.py"),
                    os.path.join(SUITE, "_tensorplace_oracle.py"))
    return SUITE


if __name__ == "__main__":
    print(stage())
