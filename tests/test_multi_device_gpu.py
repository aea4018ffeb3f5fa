"""Feature partitions across REAL devices (run when >= 2 GPUs are visible;
skipped on the one-GPU test boxes): the paths a multi-B200 node takes and a
single device cannot — P2P access between two CUDA devices
(qvb_store_attach_local_peer's cudaDeviceEnablePeerAccess branch), CUDA IPC
between processes that own different devices over NCCL (dist.init's NCCL
branch) — each checked bit for bit against the restatement.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _gpus():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs2 = pytest.mark.skipif(_gpus() < 2, reason="needs >= 2 visible GPUs (one-GPU box)")


@needs2
@pytest.mark.parametrize("host", [False, True])
def test_cross_device_stores_one_process(qvb, oracle, host):
    g = min(_gpus(), 8)
    n, dim = 40000, 128
    t = qvb.Topology.with_defaults(gpus_per_server=g, nvlink_within_numa=1,
                                   gpu_feature_capacity=n // (2 * g) if host else n // g + 1,
                                   host_feature_capacity=n)
    v = np.random.default_rng(4).random(n)
    lo, ids = qvb.plan_placement(v, t)
    stores = [qvb.FeatureStore(lo, ids, dim, t, reader=r, device=r) for r in range(g)]
    for r, st in enumerate(stores):
        for p in range(g):
            if p != r:
                st.attach_local_peer(p, stores[p])  # P2P between devices r and p
    x = oracle.features(n, dim)
    for r, st in enumerate(stores):
        req = oracle.request_ids(11, 100 + r, n, 200_000)
        assert (st.gather_host(req) == oracle.gather(x, req)).all()
        d = torch.from_numpy(req.view(np.int64)).to(f"cuda:{r}")
        out = torch.empty((len(req), dim), dtype=torch.float32, device=f"cuda:{r}")
        st.gather(d, out)
        st.check_error()
        assert (out.cpu().numpy() == oracle.gather(x, req)).all()
    for st in stores:
        st.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    try:
        import torch.distributed as dist

        from oracle.oracle import Oracle
        from paper_2305_10863_b200 import dist as D
        from paper_2305_10863_b200 import qvb

        D.init()  # NCCL: one process per device
        assert dist.get_backend() == "nccl"
        o = Oracle()
        n, dim = 30000, 100
        topo = D.topology_for(qvb, n, world, 0.1, 0.1)
        lo, ids = qvb.plan_placement(np.random.default_rng(3).random(n), topo)
        store = D.build_store(qvb, lo, ids, dim, topo, rank, rank)
        x = o.features(n, dim)
        req = o.request_ids(11, rank, n, 100_000)
        ok = bool((store.gather_host(req) == x[req.astype(np.int64)]).all())
        mx = D.max_over_ranks(float(rank))
        D.barrier()
        store.close()
        q.put((rank, "ok", ok and mx == world - 1))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "fail", traceback.format_exc()))


@needs2
def test_nccl_ranks_ipc_gather():
    world = min(_gpus(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, ok in res:
        assert status == "ok" and ok is True, ok


def test_device_count_reported(qvb):
    """Runs everywhere: the library sees the devices torch sees."""
    assert qvb.device_count() == torch.cuda.device_count()


def _sharded_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank), QVB_SEG_MB="4", QVB_F1_WINDOW="32")
    try:
        import torch.distributed as dist

        from paper_2305_10863_b200 import dist as D
        from paper_2305_10863_b200 import qvb

        D.init()  # NCCL, one process per device: in-place all-gathers over NVLink
        g = qvb.DeviceGraph.synthetic(2_400_000, 62_000_000, 7, False, False, device=rank)
        p, sharded = D.sharded_access_prob(g, 3, rank)
        ref = g.access_prob(3)
        g.close()
        q.put((rank, "ok", bool((p.view(np.uint64) == ref.view(np.uint64)).all()) and sharded))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, "fail", traceback.format_exc()))


@needs2
def test_nccl_sharded_access_prob():
    world = min(_gpus(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, status, ok in res:
        assert status == "ok" and ok is True, ok
