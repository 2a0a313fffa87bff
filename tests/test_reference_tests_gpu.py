"""The reference's own test modules for the hot path, run UNMODIFIED against this package.

``__graft_entry__.build()`` (in the build container, where /root/reference exists) copies
the reference's tests/conftest.py, test_stats.py, test_threshold.py and test_estimators.py
into the git-ignored oracle/_ref/reftests together with a generated ``docthresh`` module that
re-exports paper_1210_3165_b200 -- so every ``from docthresh import ...`` in them binds to
the B200 implementation.  This test runs that directory as its own pytest session on the
GPU (/root/reference/pkg/tests/test_stats.py:137-173,
test_threshold.py:147-170)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

REFTESTS = os.path.join(ROOT, "oracle", "_ref", "reftests")


@pytest.mark.skipif(not os.path.isdir(REFTESTS),
                    reason="oracle/_ref/reftests not staged (run __graft_entry__.build() where "
                           "/root/reference exists)")
def test_reference_modules_pass_on_b200():
    env = dict(os.environ, PYTHONPATH=REFTESTS + os.pathsep + ROOT)
    res = subprocess.run([sys.executable, "-m", "pytest", "-v", "-p", "no:cacheprovider",
                          "--rootdir", REFTESTS, REFTESTS], capture_output=True, text=True,
                         timeout=1200, cwd=REFTESTS, env=env)
    tail = res.stdout[-3000:] + res.stderr[-2000:]
    assert res.returncode == 0, tail
    assert " failed" not in res.stdout, tail
    for mod in ("test_stats.py", "test_threshold.py", "test_estimators.py"):
        assert f"{mod}::" in res.stdout, f"{mod} not collected\n{tail}"
