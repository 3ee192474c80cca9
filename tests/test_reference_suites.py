"""The reference's own unit suites (tests/test_linalg.cpp, test_reduction.cpp,
test_pep.cpp, compiled in place by oracle/Makefile with a Catch2-compatible
shim):

* on the unmodified headers (CPU): the harness itself is sound;
* bound to libdrzg.so as INTEGRATION.md section 1 describes (GPU): the
  reference's linrec_eval and detail::sparse_steps call drzg_linrec_eval /
  drzg_sparse_steps, so its known-answer, associativity, sparse-vs-dense and
  chunk-vs-fresh-solve tests (test_linalg.cpp:294-357, test_reduction.cpp:
  297-402) run through the device kernels.
"""
import os
import subprocess

import pytest

from conftest import ROOT

HOST = os.path.join(ROOT, "oracle", "_ref", "ref_suite_host")
BOUND = os.path.join(ROOT, "oracle", "_ref", "ref_suite_bound")


def _run(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle where /root/reference exists)")
    out = subprocess.run([path], capture_output=True, text=True, timeout=1200)
    return out.returncode, out.stdout


def test_reference_suites_host():
    rc, out = _run(HOST)
    assert rc == 0, out[-3000:]
    assert "0 failed" in out.splitlines()[-1]


@pytest.mark.gpu
def test_reference_suites_bound_to_device():
    rc, out = _run(BOUND)
    assert rc == 0, out[-3000:]
    last = out.splitlines()[-1]
    assert "0 failed" in last and int(last.split()[0]) >= 30
