"""The reference's own test suite, run against this package.

`oracle/ref_suite.py` stages `/root/reference/pkg/tests` (and the reference's
exhaustive verifier module) into the git-ignored `oracle/_ref/suite/`;
`tests/refsuite/alias_plugin.py` makes `import tensorplace` resolve to
`paper_2111_00655_b200`.  Each reference test module runs in a subprocess;
its junit report is checked here:

* on the GPU every reference test must pass, except the divergences listed
  in `DIVERGENCES` (each documented in DESIGN.md "Divergences") and the CLI
  tests, which skip (the CLI is out of scope);
* on CPU every failure must be the package's loud `DeviceUnavailableError`
  (the search has no CPU path) -- the host-side API (graph, patterns, rules,
  file formats, error texts) must pass as in the reference.
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import ref_suite  # noqa: E402  (test infrastructure)

SUITE = ref_suite.stage()
MODULES = ("test_graph", "test_patterns", "test_registry", "test_rules", "test_matching",
           "test_cost", "test_placement", "test_dp", "test_evolution", "test_oracle",
           "test_acceptance", "test_cli")

# reference test id -> why this package differs
DIVERGENCES: dict[str, str] = {
}

needs_suite = pytest.mark.skipif(
    SUITE is None or not os.path.exists(os.path.join(SUITE or "", "conftest.py")),
    reason="reference suite not staged (no /root/reference and no oracle/_ref/suite)")


def _run(module: str, tmp_path) -> list[tuple[str, str, str]]:
    """[(test id, outcome, message)] of one reference module."""
    xml = tmp_path / f"{module}.xml"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join(
        [os.path.join(ROOT, "tests", "refsuite"), SUITE, env.get("PYTHONPATH", "")])
    env["CB_REPO_ROOT"] = ROOT
    env["CB_REF_SUITE"] = SUITE
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-p", "alias_plugin", "-p", "no:cacheprovider",
         "--rootdir", SUITE, "-c", os.devnull, f"--junitxml={xml}", f"{module}.py"],
        cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    assert xml.exists(), proc.stdout[-3000:] + proc.stderr[-3000:]
    out = []
    for case in ET.parse(xml).getroot().iter("testcase"):
        tid = f"{module}::{case.get('name')}"
        outcome, msg = "passed", ""
        for tag in ("failure", "error", "skipped"):
            el = case.find(tag)
            if el is not None:
                outcome = tag
                msg = (el.get("message") or "") + "\n" + (el.text or "")
                break
        out.append((tid, outcome, msg))
    assert out, proc.stdout[-3000:]
    return out


@needs_suite
@pytest.mark.parametrize("module", MODULES)
def test_reference_module_host_side(module, tmp_path):
    """CPU: only device calls may fail, and only loudly."""
    from paper_2111_00655_b200 import _native
    if _native.device_available():
        pytest.skip("covered by the GPU variant")
    bad = [(t, m.strip().splitlines()[0] if m.strip() else "")
           for t, o, m in _run(module, tmp_path)
           if o in ("failure", "error") and "DeviceUnavailableError" not in m]
    assert not bad, bad


@pytest.mark.gpu
@needs_suite
@pytest.mark.parametrize("module", MODULES)
def test_reference_module_on_device(module, gpu, tmp_path):
    results = _run(module, tmp_path)
    bad = [(t, m.strip()[:400]) for t, o, m in results
           if o in ("failure", "error") and t not in DIVERGENCES]
    assert not bad, bad
    unexpected_pass = [t for t, o, _ in results if o == "passed" and t in DIVERGENCES]
    assert not unexpected_pass, f"listed as divergences but pass: {unexpected_pass}"
    skipped = [t for t, o, _ in results if o == "skipped"]
    if module != "test_cli":
        assert all(t.startswith("test_acceptance::test_0") for t in skipped), skipped
