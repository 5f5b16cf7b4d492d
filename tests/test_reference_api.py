"""The reference's own per-diagram and splitting tests
(/root/reference/pkg/tests/test_bdd.py and test_split.py, 22 tests incl.
hypothesis properties against a brute-force enumerator) run unchanged
against this package through an import alias (tests/reference_alias.py:
``prodmatch.bdd`` -> paper_2310_08230_b200.bdd, ``prodmatch.splitting`` ->
paper_2310_08230_b200.splitting, ...).  Needs the reference checkout, which
exists in the build container only; skipped elsewhere."""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference checkout not present")
@pytest.mark.parametrize("name", ["test_bdd.py", "test_split.py"])
def test_reference_tests_pass_against_this_package(name, tmp_path):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ROOT, REF_TESTS]), NUMBA_CACHE_DIR=str(tmp_path))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "tests.reference_alias", "-p", "no:cacheprovider",
                        "--rootdir", str(tmp_path), "-c", os.devnull, os.path.join(REF_TESTS, name)],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "prodmatch" not in r.stderr
