"""Host-side multi-rank logic of bench.py on CPU with the gloo backend, world size 2
(the N>1 path: independent problem per rank, max-over-ranks step time)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import synth
    cfg = synth.CONFIGS["c256"]
    seed = bench.rank_instance_seed(cfg, rank)
    inst = synth.make_instance(cfg, m=4, n=4, l=4, seed=seed)
    t = bench.reduce_max(10.0 + rank, dist, torch.device("cpu"))
    out[rank] = (seed, int(inst.A.sum()), t)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_ranks_independent_problems_and_max_time():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    (s0, a0, t0), (s1, a1, t1) = out[0], out[1]
    assert s0 != s1                                   # different independent problems
    assert t0 == t1 == 11.0                           # both ranks see the slowest rank's time
