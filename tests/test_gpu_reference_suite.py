"""The reference's own test suite, run against the B200 drop-in.

tools/install_reference.sh installs the unmodified reference (convkit 0.1.0)
into baseline/_ref and stages its tests there (git-ignored; never committed).
The plugin tests/reference_rebind.py rebinds convkit.conv_twostage,
convkit.twostage.conv_twostage, convkit.bench.conv_twostage,
stage1_scalar_prods and stage2_sum to the drop-in before collection
(/root/reference/pkg/src/convkit/__init__.py:18-20, bench.py:25), so
test_twostage.py, test_acceptance.py, test_bench.py and test_cli.py exercise
the GPU engine — including the bitwise pins (criterion 1,
TestConvTwostage::test_matches_naive_bitwise) and the RunStats contract.
"""

from __future__ import annotations

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
SUITE = ["test_twostage.py", "test_acceptance.py", "test_bench.py", "test_cli.py"]


@pytest.mark.gpu
def test_reference_suite_passes_against_the_drop_in():
    tests = REF / "convkit_tests"
    if not (REF / "convkit").is_dir() or not tests.is_dir():
        pytest.skip("reference not staged in baseline/_ref (tools/install_reference.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests")]))
    r = subprocess.run([sys.executable, "-m", "pytest", *[str(tests / t) for t in SUITE], "-p", "reference_rebind",
                        "-q", "-p", "no:cacheprovider", "--rootdir", str(tests)],
                       cwd=str(tests), env=env, capture_output=True, text=True, timeout=1500)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    m = re.search(r"(\d+) passed", r.stdout)
    assert m and int(m.group(1)) >= 72, tail
    calls = re.search(r"drop-in calls \{'conv_twostage': (\d+), 'stage1_scalar_prods': (\d+), 'stage2_sum': (\d+)\}",
                      r.stdout)
    assert calls and int(calls.group(1)) > 100 and int(calls.group(2)) > 0 and int(calls.group(3)) > 0, tail
    print(tail[-600:])
