"""Host logic of the multi-GPU path on CPU (world_size 2, gloo): the U-scan partition of the
problems over ranks and the whole-job aggregation (sum of work / max of time over ranks).
DESIGN.md section 10: ranks are independent unfolds; there is no data-path collective."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch.distributed as dist

    import bench
    from workloads import u_scan_problem

    r, w, _ = bench.dist_init(None, backend="gloo")
    assert (r, w) == (rank, world)
    prob = u_scan_problem(1, rank, world)
    diag = prob.H0.to_dense().diagonal().real.copy()
    # each rank: its own work and time; the job: all work over the slowest rank's time
    nnz, steps, t = 1000 * (rank + 1), 10, 0.5 + rank
    value, tmax = bench.aggregate(nnz, steps, t, world)
    out[rank] = (prob.name, prob.H0.nnz, diag[5], value, tmax)
    dist.barrier()
    dist.destroy_process_group()


def test_u_scan_partition_and_aggregation_world2():
    world, port = 2, _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    (n0, z0, d0, v0, t0), (n1, z1, d1, v1, t1) = out[0], out[1]
    assert n0 != n1 and z0 == z1          # different U, same pattern size
    assert d0 != d1                        # the U-dependent diagonal differs
    assert t0 == t1 == 1.5                 # max over ranks
    assert v0 == v1 == pytest.approx((1000 + 2000) * 10 / 1.5)


def test_u_scan_single_rank_is_the_baseline_config():
    from workloads import config, u_scan_problem

    a, b = u_scan_problem(4, 0, 1), config(4)
    assert a.name == b.name and np.array_equal(a.H0.val, b.H0.val)
