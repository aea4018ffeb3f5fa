"""GPU, world_size 2, two processes: the one-process-per-GPU store path with
real CUDA IPC. Both ranks sit on cuda:0 here (one GPU per test box), so a
peer's shard is mapped with cudaIpcOpenMemHandle from the other process and
read one-sided by the gather kernel — the code path NVLink peers take on a
multi-GPU node — and the handles travel over torch.distributed (gloo, since
NCCL refuses two ranks on one device). Every rank's gather must return
X[ids] bit for bit, with rows served from its own shard, its peer's and the
host tier.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


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
        import torch
        import torch.distributed as dist

        from oracle.oracle import Oracle
        from paper_2305_10863_b200 import dist as D
        from paper_2305_10863_b200 import qvb

        D.init(backend="gloo")
        torch.cuda.set_device(0)
        o = Oracle()
        n, dim = 20000, 100
        values = np.random.default_rng(3).random(n)  # same on every rank
        topo = D.topology_for(qvb, n, world, replicate, host_frac)
        lo, ids = qvb.plan_placement(values, topo)
        store = D.build_store(qvb, lo, ids, dim, topo, rank, 0)  # IPC export / attach
        x = o.features(n, dim)
        req = o.request_ids(11, rank, n, 8192)
        out = store.gather_host(req)
        ok = bool((out == x[req.astype(np.int64)]).all())
        whole = bool((store.gather_host(np.arange(n, dtype=np.uint64)) == x).all())
        loc, _ = qvb.build_lookup_table(lo, ids, topo, 0, rank)
        fr = (float(np.mean(loc == rank)), float(np.mean((loc != rank) & (loc < world))),
              float(np.mean(loc == world)))
        D.barrier()
        store.close()
        q.put((rank, "ok", ok, whole, fr))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "fail", traceback.format_exc(), False, None))


@pytest.mark.parametrize("replicate,host_frac", [(0.0, 0.0), (0.1, 0.2)])
def test_two_process_ipc_gather(replicate, host_frac):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, replicate, host_frac, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, ok, whole, fr in res:
        assert status == "ok", ok
        assert ok and whole
        local, peer, host = fr
        assert peer > 0.2 and local > 0.2  # both shards really serve rows
        assert (host > 0.1) == (host_frac > 0)


def _p_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank), QVB_SEG_MB="4", QVB_F1_WINDOW="32")
    try:
        import torch
        import torch.distributed as dist

        from paper_2305_10863_b200 import dist as D
        from paper_2305_10863_b200 import qvb

        D.init(backend="gloo")
        torch.cuda.set_device(0)
        n, e = 2_400_000, 62_000_000
        g = qvb.DeviceGraph.synthetic(n, e, 7, False, False)
        p, sharded = D.sharded_access_prob(g, 3, 0)
        ref = g.access_prob(3)
        g.close()
        q.put((rank, "ok", bool((p.view(np.uint64) == ref.view(np.uint64)).all()) and sharded))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "fail", traceback.format_exc()))


def test_two_process_sharded_access_prob():
    """Two processes split the C2 sweeps by node chunks and all-gather P and
    the codes over torch.distributed after every sweep (gloo through host
    memory here, since both share the box's one GPU; NCCL in place on a
    multi-GPU node): both end with the single-GPU answer bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, ok in res:
        assert status == "ok" and ok is True, ok
