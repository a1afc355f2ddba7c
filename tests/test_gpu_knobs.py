"""GPU parity of the alternate scheduling paths behind the library's timing
knobs, against the CPU oracle: query sets of 8 consecutive tiles
(GJ_DEAL_BLOCK=8, reading R12's alternative), uniform (not guided) split plans
(GJ_PLAN_GUIDED=0) and the uniform estimator split (GJ_EST_UNIFORM=1).  The knobs
are read once per process, so the partition / batch / host-pipeline /
estimator cases of test_gpu_parity.py rerun in a child pytest; every assertion
there compares with oracle/brute.py or oracle/grid.py."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = "entity or batches or regrows or estimator or join_counts or work_counters or pairs_equal or filters_on_paper"


@pytest.mark.parametrize("knobs", [{"GJ_DEAL_BLOCK": "8"}, {"GJ_PLAN_GUIDED": "0", "GJ_EST_UNIFORM": "1"}],
                         ids=["deal_block_8", "uniform_plans"])
def test_scheduling_knobs_keep_parity(knobs):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, **knobs)
    env.pop("GJ_PARITY_REPORT", None)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-x", "-q", "-p", "no:cacheprovider", "-k", CASES],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
