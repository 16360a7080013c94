"""Install the reference package `kkmodem` (and its test-suite) into
baseline/_ref -- test infrastructure for the drop-in switch
(paper_2108_07001_b200/kkmodem_backend.py).

baseline/_ref is git-ignored but travels to the GPU box with the repo
snapshot, so the reference's own tests can run there against the B200
receiver (tests/test_reference_suite.py).  Uses the base contract's offline
pip command (from a /tmp copy: /root/reference is read-only) and copies the
reference's pkg/tests next to the package as baseline/_ref/kkmodem_tests.
No-op when /root/reference is absent (the GPU box) or the install is current.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"
DEST = os.path.join(REPO, "baseline", "_ref")
TESTS = os.path.join(DEST, "kkmodem_tests")


def install(force: bool = False) -> str | None:
    if not os.path.isdir(REF):
        return DEST if os.path.isdir(os.path.join(DEST, "kkmodem")) else None
    if force or not os.path.isdir(os.path.join(DEST, "kkmodem")):
        tmp = "/tmp/kkmodem_pkg_copy"
        shutil.rmtree(tmp, ignore_errors=True)
        shutil.copytree(REF, tmp)
        subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                        "--find-links", "/opt/wheelhouse", "--no-deps", "--upgrade", "--target", DEST, tmp],
                       check=True, capture_output=True)
    src = os.path.join(REF, "tests")
    if force or not os.path.isdir(TESTS) or sorted(os.listdir(TESTS)) != sorted(
            f for f in os.listdir(src) if f.endswith(".py")) + (["__pycache__"] if os.path.isdir(
                os.path.join(TESTS, "__pycache__")) else []):
        shutil.rmtree(TESTS, ignore_errors=True)
        os.makedirs(TESTS)
        for f in os.listdir(src):
            if f.endswith(".py"):
                shutil.copy2(os.path.join(src, f), os.path.join(TESTS, f))
    return DEST


if __name__ == "__main__":
    print(install(force="--force" in sys.argv))
