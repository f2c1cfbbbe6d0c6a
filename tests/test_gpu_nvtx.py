"""SPP_NVTX=1 (NVTX ranges per launch class and per setup / solve call, SURVEY 5 tracing) must not
change anything the solver computes: smoke() -- a 2D solve, a 1D solve and a 1D batch, each
checked against the oracle -- passes with the ranges on, with the iteration graphs and with the
host-driven loops."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("no_graph", ["0", "1"])
def test_smoke_with_nvtx_ranges(no_graph):
    env = dict(os.environ, SPP_NVTX="1")
    if no_graph == "1":
        env["SPP_NO_GRAPH"] = "1"
    p = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "SMOKE OK" in p.stdout, (p.stdout[-1000:], p.stderr[-3000:])
