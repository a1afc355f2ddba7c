"""GPU parity of the persistent tcgen05 join (gj_join_ws.cu, opt-in with
GJ_UMMA_WS=1) against the CPU oracle.

The kernel choice is read once per process, so the tcgen05 parity cases of
test_gpu_parity.py (paper shapes, every flag combination, near-boundary pairs,
the bound at its enable limit, exact-boundary lattices, degenerate inputs,
entity partitions, batches and the host pipeline) run again in a child pytest
with the persistent kernel selected, for two epilogue groupings (GJ_WS_EG: 8
or 4 warps read each accumulator block).  Every assertion of those
tests compares with oracle/brute.py or oracle/grid.py.
"""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ("filters_on_paper_shapes or pairs_equal or every_flag or near_boundary or enable_limit or lattice "
         "or degenerate or entity or batches or regrows or dimension_limit or join_counts")


@pytest.mark.parametrize("groups", [2, 4])
def test_persistent_kernel_parity(groups):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, GJ_UMMA_WS="1", GJ_WS_EG=str(groups))
    env.pop("GJ_PARITY_REPORT", None)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"), "-m", "gpu",
                        "-x", "-q", "-p", "no:cacheprovider", "-k", CASES],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in r.stdout and "failed" not in r.stdout, tail
