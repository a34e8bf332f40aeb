"""The optional schedules and layouts never change a result.

The exact consult has switches that only move work around: the
leader-first schedule of a live wave on an empty table
(``HRPP_LEADER_FIRST``) and the grouping sort on a highest-priority stream
beside the early traversal (``HRPP_SORT_PRIO``).  Each is read once per
process, so the parity tests that compare waves with the reference's
goldens (hrpp/tracer.py:343-371) and with the oracle are re-run in a child
process with the switch on.
"""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SUBSET = ("wave_sequence_matches_reference or c1_frame_vs_oracle or "
          "very_long_key_segments_vs_oracle or table_clear_reuse_equals_fresh or "
          "deferred_commit_equals_direct")


def _rerun(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-m", "pytest", str(ROOT / "tests" / "test_gpu_parity.py"),
                        "-m", "gpu", "-x", "-q", "-k", SUBSET, "-p", "no:cacheprovider"],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:]


def test_leader_first_and_priority_sort_are_exact():
    _rerun({"HRPP_LEADER_FIRST": "2", "HRPP_SORT_PRIO": "1"})
