"""The reference's OWN test-suite, run on the B200 receiver through the
kkmodem backend switch (paper_2108_07001_b200/kkmodem_backend.py, the
binding INTEGRATION.md §1 describes).

Each case runs pytest in a subprocess on kkmodem's tests (installed with the
reference package into baseline/_ref by tools/install_reference.py, which
`__graft_entry__.build()` calls; baseline/_ref travels to the GPU box) with
`-p paper_2108_07001_b200.kkmodem_backend`, so `kkmodem.rxdsp.RxPipeline`,
the functional stages and the names kkmodem/harness/runner.py:16-24 imported
are the GPU ones before the reference's test modules bind them.  Every
selected reference test must pass, unmodified.

Selected: tests/test_rxdsp.py (every receive-path unit test),
tests/test_harness.py (contiguity, diagnostics, run_single, sweeps, bench,
sustained; the CLI tests are excluded: they start `python -m kkmodem...`
subprocesses without the switch, and the plot test needs matplotlib), the
acceptance criteria (C1, C2 contiguity, C3 10,000 km CD, C4
KK, C5, C6 widely-linear, C7 formats x distances, C9, C10 sustained 2^26
samples, C11 bench stability, and C8 -- the nonlinear launch-power / CSPR
trade-offs, whose split-step spans run on the GPU through the switch's
kkmodem.channel.ssfm_span), and this repo's switch-behaviour checks
(tests/reference_switch/).
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "kkmodem_tests")

CASES = {
    "rxdsp": (["test_rxdsp.py"], None),
    "harness": (["test_harness.py"], "not TestCli"),
    # every criterion, C8 included (its 12 nonlinear links of 10 / 24 spans run
    # their split-step spans on the GPU: ~20 s instead of ~270 s on the CPU)
    "acceptance": (["test_acceptance.py"], None),
    "switch": ([os.path.join(REPO, "tests", "reference_switch", "test_switch_behaviour.py")], None),
    # the rest of kkmodem's unit tests, with the switch installed (they exercise
    # sigcore / txdsp / channel / frontend / metrics: the receiver must not disturb them)
    "other": (["test_sigcore.py", "test_txdsp.py", "test_channel.py", "test_frontend.py", "test_metrics.py"], None),
}


def _have_reference() -> bool:
    return os.path.isdir(os.path.join(REF, "kkmodem")) and os.path.isdir(REF_TESTS)


def run_reference_tests(files, kexpr, junit, timeout=2400):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, REPO] + ([env["PYTHONPATH"]] if env.get("PYTHONPATH") else []))
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/kkb200_numba_cache")
    paths = [f if os.path.isabs(f) else os.path.join(REF_TESTS, f) for f in files]
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "paper_2108_07001_b200.kkmodem_backend",
           "-p", "no:cacheprovider", "-c", os.devnull, "--rootdir", REF, f"--junitxml={junit}", *paths]
    if kexpr:
        cmd += ["-k", kexpr]
    return subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout, cwd=REF)


def _outcomes(junit):
    root = ET.parse(junit).getroot()
    out = {}
    for tc in root.iter("testcase"):
        name = f"{tc.get('classname')}::{tc.get('name')}"
        kind = "passed"
        for child in tc:
            if child.tag in ("failure", "error"):
                kind = "failed"
                break
            if child.tag == "skipped":
                kind = "skipped"
        out[name] = kind
    return out


@pytest.mark.parametrize("case", sorted(CASES))
def test_reference_suite_on_b200(case, tmp_path):
    if not _have_reference():
        pytest.fail("baseline/_ref (kkmodem + its tests) missing: run tools/install_reference.py "
                    "(__graft_entry__.build() does) in the container that has /root/reference")
    files, kexpr = CASES[case]
    junit = str(tmp_path / f"{case}.xml")
    r = run_reference_tests(files, kexpr, junit)
    assert os.path.exists(junit), r.stdout[-3000:] + r.stderr[-3000:]
    res = _outcomes(junit)
    bad = {k: v for k, v in res.items() if v != "passed"}
    print(f"{case}: {len(res)} reference tests, {len(res) - len(bad)} passed")
    for k in sorted(res):
        print(f"  {res[k]:7s} {k}")
    assert res, r.stdout[-3000:]
    assert not bad, f"{bad}\n{r.stdout[-6000:]}\n{r.stderr[-2000:]}"
    assert r.returncode == 0, r.stdout[-3000:]
