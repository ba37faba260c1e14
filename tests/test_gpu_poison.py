"""Scratch-poisoning run (OEM_POISON=1: every workspace the library hands a kernel is first filled
with a NaN pattern): the cfg1 fit, a fold-mode CV fit, the logistic paths, the active-set solver
(its screened compact iterations for every family), the d rule, the two-panel weighted pass and
the sparse pass must still match the oracle, i.e. no kernel reads scratch it did not write in the
same call."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_poisoned_workspace_subprocess():
    env = dict(os.environ, OEM_POISON="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_path.py") + "::test_cfg1_lasso_path",
           os.path.join(ROOT, "tests", "test_gpu_path.py") + "::test_cfg3_fold_mode",
           os.path.join(ROOT, "tests", "test_gpu_cv.py"),
           os.path.join(ROOT, "tests", "test_gpu_logistic.py"),
           os.path.join(ROOT, "tests", "test_gpu_path.py") + "::test_active_set_solver",
           os.path.join(ROOT, "tests", "test_gpu_path.py") + "::test_screened_every_family",
           os.path.join(ROOT, "tests", "test_gpu_gram.py") + "::test_weighted_two_panel_parity",
           os.path.join(ROOT, "tests", "test_gpu_sparse.py") + "::test_sparse_gram_parity",
           "-k", "not full_size"]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
