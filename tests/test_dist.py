"""Multi-rank host logic on CPU (gloo, world_size 2): slab cuts, per-slab nnz,
all-gather of nnz and the exclusive-scan row_ptr base; the concatenated
per-rank row_ptr blocks equal the single-process pattern of the oracle
(P:537-548).  The CUDA kernels themselves are covered by
tests/test_gpu_parity.py::test_slabs_concatenate_bit_exact."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1605_01238_b200.dist import ni_1d, slab_cuts, slab_nnz


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, ns, p, out):
    import torch
    import torch.distributed as dist
    from paper_1605_01238_b200.dist import nnz_base
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cuts = slab_cuts(ns[-1], p, world)
    b, e = cuts[rank], cuts[rank + 1]
    local = slab_nnz(ns, p, b, e)
    base = nnz_base(local, dist)
    # per-rank row_ptr block from the closed form (what wq_pattern writes on the GPU)
    d = len(ns)
    rows = []
    L = [int(ni_1d(n, p).sum()) for n in ns]
    nis = [ni_1d(n, p) for n in ns]
    off = base
    for i3 in range(b, e):
        for r in range(int(np.prod(ns[:-1]))):
            idx = np.unravel_index(r, ns[:-1], order="F") if d > 1 else ()
            rows.append(off)
            nnz_row = int(np.prod([nis[l][idx[l]] for l in range(d - 1)])) * int(nis[-1][i3])
            off += nnz_row
    out[rank] = (rows, off, local, base)
    dist.destroy_process_group()


@pytest.mark.parametrize("ns,p", [([7, 6, 9], 2), ([10, 12], 3), ([11], 1)])
def test_slab_rowptr_two_ranks(ns, p):
    import oracle
    from wqinputs import uniform_open_knots
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, ns, p, out), nprocs=world, join=True)
    rp = []
    for r in range(world):
        rows, end, local, base = out[r]
        assert end - base == local
        rp += rows
    total = sum(out[r][2] for r in range(world))
    knots = [uniform_open_knots(p, n - p) for n in ns]
    o = oracle.Oracle(p, knots)
    orp, _ = o.pattern()
    assert np.array_equal(np.array(rp + [total]), orp)


def test_slab_cuts_balanced():
    from paper_1605_01238_b200.dist import plane_cost
    for n, p, w in [(104, 4, 8), (260, 4, 8), (110, 10, 4), (5, 2, 4)]:
        for balance in ("cost", "nnz"):
            cuts = slab_cuts(n, p, w, balance)
            assert cuts[0] == 0 and cuts[-1] == n and all(b < e for b, e in zip(cuts, cuts[1:]))
            nnz = [slab_nnz([n, n, n], p, b, e) for b, e in zip(cuts, cuts[1:])]
            assert sum(nnz) == slab_nnz([n, n, n], p, 0, n)
            wts = plane_cost(n, p) if balance == "cost" else ni_1d(n, p)
            per = [wts[b:e].sum() for b, e in zip(cuts, cuts[1:])]
            if n >= 8 * w:
                assert max(per) / min(per) < 1.1, (n, p, w, balance, per)


def test_plane_cost_counts():
    """#Q_i of reading R1 (interior 2p+1, boundary p+1+2i) against the oracle's point ranges."""
    import oracle
    from paper_1605_01238_b200.dist import nq_1d
    from wqinputs import uniform_open_knots
    for p, E in [(2, 9), (4, 12), (6, 15)]:
        D = oracle.Oracle(p, [uniform_open_knots(p, E)]).direction(0)
        assert np.array_equal(nq_1d(E + p, p), np.asarray(D["qlen"]))
