"""CPU, world_size 2 (gloo): the one-process-per-GPU plumbing of the
partitioned store (paper_2305_10863_b200/dist.py) and the routing contract
the device gather relies on — every reader's lookup table addresses its own
shard, the peers' shards (exchanged like IPC handles) and the host tier so
that out[i] == X[ids[i]]. The shards are materialised with the oracle here
(no GPU); the device path is covered by tests/test_gather_gpu.py.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, replicate, host_frac, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        import torch.distributed as dist

        from oracle.oracle import Oracle, topology_defaults
        from paper_2305_10863_b200 import dist as D

        r, w, local = D.init(backend="gloo")
        assert (r, w, local) == (rank, world, rank)
        o = Oracle()
        n, dim = 3000, 16
        rng = np.random.default_rng(7)  # same values on every rank
        values = rng.random(n)
        cap, rep, host = D.partition_capacities(n, world, replicate, host_frac)
        t = topology_defaults(gpus_per_server=world, nvlink_within_numa=1,
                              gpu_feature_capacity=cap, gpu_replicated_capacity=rep,
                              host_feature_capacity=host)
        lo, ids = o.plan_placement(values, t)
        x = o.features(n, dim)
        # this rank's shard: features with a copy at location `rank`, id order
        mine = np.array([f for f in range(n) if rank in ids[lo[f]:lo[f + 1]]], np.int64)
        shard = x[mine]
        host_rows = np.array([f for f in range(n) if world in ids[lo[f]:lo[f + 1]]], np.int64)
        shards = [None] * world
        dist.all_gather_object(shards, shard)  # stands in for the IPC handle exchange
        hb = D.exchange_bytes(bytes([rank]) * 64)
        assert [b[0] for b in hb] == list(range(world))
        loc, off = o.build_lookup_table(lo, ids, t, 0, rank)
        req = o.request_ids(11, rank, n, 2000)
        out = np.empty((len(req), dim), np.float32)
        for i, f in enumerate(req):
            l, of = int(loc[f]), int(off[f])
            out[i] = shards[l][of] if l < world else x[host_rows[of]]
        assert (out == x[req.astype(np.int64)]).all()
        # local rows really are local for this reader
        assert ((loc == rank) == np.isin(np.arange(n), mine)).all()
        m = D.max_over_ranks(float(rank + 1))
        ssum = D.sum_over_ranks(1.0)
        D.barrier()
        q.put((rank, "ok", m, ssum, float(np.mean(loc == rank))))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, "fail", traceback.format_exc(), 0, 0))


@pytest.mark.parametrize("replicate,host_frac", [(0.0, 0.0), (0.1, 0.0), (0.05, 0.2)])
def test_two_rank_partitioned_routing(replicate, host_frac):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, replicate, host_frac, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, a, b, frac in res:
        assert status == "ok", a
        assert a == 2.0 and b == 2.0
        assert frac >= 0.45 * (1 - host_frac)  # roughly half the table is local


def test_partition_capacities():
    from paper_2305_10863_b200.dist import partition_capacities

    cap, rep, host = partition_capacities(1000, 4, 0.1, 0.2)
    assert rep == 100 and cap == 100 + 175 and host == 1000
    cap, rep, host = partition_capacities(1000, 1)
    assert cap == 1000 and rep == 0
