"""One-process-per-GPU plumbing for the partitioned feature store.

The gather shards naturally: every rank serves its own batch,
reading one-sided from its own HBM, from peer shards over NVLink/NVSwitch
(CUDA IPC mappings) and from host pinned memory. There is no collective on
the data path; torch.distributed only carries the setup (IPC handle
exchange), barriers and the max-over-ranks timing reduction.
"""
from __future__ import annotations

import math
import os

import torch
import torch.distributed as dist


def env_rank():
    """(rank, world, local_rank) from the torchrun environment (1 process = 1 GPU)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shared_gpu() -> bool:
    """QVB_SHARE_GPU=1 (testing on a one-GPU box): every rank runs on the
    same device; peers are still separate processes mapped with CUDA IPC, and
    the setup collectives go over gloo (NCCL refuses two ranks on one GPU)."""
    return os.environ.get("QVB_SHARE_GPU", "0") == "1"


def device_index(local_rank: int) -> int:
    if shared_gpu() and torch.cuda.is_available():
        return local_rank % torch.cuda.device_count()
    return local_rank


def init(backend: str | None = None):
    rank, world, local = env_rank()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() and not shared_gpu() else "gloo"
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend=backend, **kw)
    return rank, world, local


def is_dist() -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1


def barrier() -> None:
    if is_dist():
        dist.barrier()


def exchange_bytes(b: bytes) -> list[bytes]:
    """All-gather one small byte string per rank (rank order)."""
    if not is_dist():
        return [b]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, b)
    return out


def max_over_ranks(x: float) -> float:
    if not is_dist():
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    if not is_dist():
        return x
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def partition_capacities(n: int, world: int, replicate: float = 0.0, host_frac: float = 0.0):
    """GPU capacities (records) that force the SURVEY §8(d) C5 layout on one
    server of `world` GPUs: the hottest `replicate`·n rows on every GPU, the
    coldest `host_frac`·n rows in host memory, the rest LPT-partitioned.
    Returns (gpu_feature_capacity, gpu_replicated_capacity, host_capacity)."""
    rep = int(round(replicate * n))
    host = int(round(host_frac * n))
    rest = max(0, n - rep - host)
    part = math.ceil(rest / world)
    return rep + part, rep, n


def topology_for(qvb, n: int, world: int, replicate: float = 0.0, host_frac: float = 0.0):
    cap, rep, host = partition_capacities(n, world, replicate, host_frac)
    return qvb.Topology.with_defaults(servers=1, numa_per_server=1, gpus_per_server=world,
                                      nvlink_within_numa=1 if world > 1 else 0,
                                      gpu_feature_capacity=cap,
                                      gpu_replicated_capacity=rep if world > 1 else 0,
                                      host_feature_capacity=host, disk_feature_capacity=0)


def build_store(qvb, loc_offsets, loc_ids, dim: int, topo, rank: int, local_rank: int,
                features=None):
    """This rank's FeatureStore with every peer shard attached (IPC)."""
    store = qvb.FeatureStore(loc_offsets, loc_ids, dim, topo, reader=rank, features=features,
                             device=local_rank)
    handles = exchange_bytes(store.export_handle())
    for peer, h in enumerate(handles):
        if peer != rank:
            store.attach_peer(peer, h)
    barrier()
    return store


class _DevView:
    """A device pointer as a torch tensor (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def allgather_exchange(rank: int, world: int, device: int):
    """The exchange step of the row-sharded P pass: after each
    sweep, every rank's chunk of P_j (f64) and of the codes the next sweep
    gathers (u32) is all-gathered IN PLACE into every rank's buffers — one
    ncclAllGather per array over NVLink/NVSwitch, ordered on the library's
    stream. With gloo (ranks sharing one GPU in tests) the chunks travel
    through host memory."""

    def exchange(layer, p_ptr, codes_ptr, chunk, stream_ptr):
        ext = torch.cuda.ExternalStream(stream_ptr, device=device) if stream_ptr else \
            torch.cuda.default_stream(device)
        with torch.cuda.device(device), torch.cuda.stream(ext):
            for ptr, ts in ((p_ptr, "<f8"), (codes_ptr, "<i4")):  # codes: u32 bits as i32
                if not ptr:
                    continue
                whole = torch.as_tensor(_DevView(ptr, world * chunk, ts), device=f"cuda:{device}")
                mine = whole[rank * chunk:(rank + 1) * chunk]
                if dist.get_backend() == "nccl":
                    dist.all_gather_into_tensor(whole, mine)
                else:  # gloo: host staging (functional multi-rank tests on one GPU)
                    host = mine.cpu()
                    parts = [torch.empty_like(host) for _ in range(world)]
                    dist.all_gather(parts, host)
                    whole.copy_(torch.cat(parts).to(whole.device))

    return exchange


def sharded_access_prob(graph, layers: int, device: int, out=None, stream=None):
    """P(n, layers) with the sweeps split over the ranks (one process per
    GPU, each holding the graph): bit-identical to the single-GPU call."""
    rank, world = (dist.get_rank(), dist.get_world_size()) if is_dist() else (0, 1)
    return graph.access_prob_sharded(layers, rank, world, allgather_exchange(rank, world, device),
                                     out=out, stream=stream)
