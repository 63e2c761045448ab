"""The multi-GPU rank path of bench.py (x_3 slabs, one int64 all-gather of nnz, per-rank
CSR blocks chained through nnz_base) run as 2 ranks on ONE GPU over gloo (the only collective is the
nnz exchange; the kernels of the two ranks never wait on each other).  The concatenated blocks are
compared with the oracle: the pattern in full, values on sampled rows (rows independent)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle import STIFFNESS, Oracle
from parity_util import compare_rows, sample_rows
from wqinputs import Config

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("p,n_el", [(3, 12), (8, 10)])
def test_bench_rank_path_two_ranks(tmp_path, p, n_el):
    env = dict(os.environ, WQ_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--config", "C4", "--p", str(p), "--n-el", str(n_el), "--steps", "3", "--warmup", "3", "--no-sweep",
           "--no-e2e", "--no-cpu", "--dump-csr", str(tmp_path)]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["scaling"] == "weak"
    rps = [np.load(tmp_path / f"rank{r}_rp.npy") for r in range(2)]
    cols = [np.load(tmp_path / f"rank{r}_col.npy") for r in range(2)]
    vals = [np.load(tmp_path / f"rank{r}_val.npy") for r in range(2)]
    assert rps[0][0] == 0 and rps[1][0] == rps[0][-1]  # nnz_base from the all-gather
    rp = np.concatenate([rps[0][:-1], rps[1]])
    col, val = np.concatenate(cols), np.concatenate(vals)
    cfg = Config(f"C4p{p}e{n_el}", 3, p, n_el, "grid", 0.1)
    o = Oracle(p, cfg.knots(), cfg.ctrl())
    orp, ocol = o.pattern()
    assert np.array_equal(rp, orp) and np.array_equal(col, ocol)
    n = n_el + p
    rows = sample_rows(n, 3, p, k_random=16, seed=3)
    ptr, oc, ov, kappa, scale = o.rows(STIFFNESS, rows)
    gptr = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(rp[rows + 1] - rp[rows], out=gptr[1:])
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    compare_rows(rows, gptr, col[idx], val[idx], ptr, oc, ov, kappa, scale)
