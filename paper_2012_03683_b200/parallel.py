"""Multi-GPU plumbing: one process per GPU, torch.distributed
for the host-side collectives (NCCL on GPUs, gloo on CPU in the tests).

Two ways the registration path shards:

* independent frame pairs / sequence chains (C3, C5): each rank registers its
  own pairs or chains; no data-path collective. `shard_range`, `chain_spans`,
  `rank_spans`, `register_sequence_distributed` (the chain partition is the
  one `kreg_register_sequence_chains` uses, so a distributed run reproduces
  the single-GPU chained run pair for pair).
* source-row sharding of one large pair (C4): every rank registers the
  replicated target X against its Morton-contiguous rows of the source Z; after
  every device round the replicated host loop combines F, the gradient and the
  pair counts (sum) and the displacements (max) through `TorchCollective`, a
  kreg_collective_fn callback (include/kreg_b200.h) running one all-reduce per
  kind. All ranks see identical totals, so they take identical decisions and
  stay in lockstep (`register_clouds_sharded`).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .types import Isometry, PointCloud, SequenceResult, compose


# ------------------------------------------------------------------ ranks
def world_info():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None):
    """Initialise torch.distributed when WORLD_SIZE > 1 (MASTER_ADDR defaults to
    127.0.0.1). Backend: NCCL when CUDA is available, else gloo."""
    rank, world, local = world_info()
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if not dist.is_initialized():
            if backend is None:
                backend = "nccl" if torch.cuda.is_available() else "gloo"
            if backend == "nccl":
                torch.cuda.set_device(local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group(backend)
    return rank, world, local


def _device():
    import torch
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def barrier():
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def reduce_scalar(x: float, op: str = "max") -> float:
    """max / sum of a host scalar over all ranks (identity without a group)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------- partitions
def shard_range(n: int, rank: int, world: int):
    """Balanced contiguous [begin, end) share of n items."""
    return n * rank // world, n * (rank + 1) // world


def chain_spans(n_frames: int, n_chains: int):
    """Pair spans [(begin, end)) of the chains of a sequence of n_frames frames,
    exactly as kreg_register_sequence_chains partitions them (capi.cpp);
    adjacent chains share one frame."""
    m = n_frames - 1
    if m < 1:
        raise ValueError("register_sequence: need at least 2 frames")
    nc = max(1, min(n_chains, m))
    return [(m * c // nc, m * (c + 1) // nc) for c in range(nc)]


def rank_spans(spans, rank: int, world: int):
    """Contiguous block of chains for one rank."""
    b, e = shard_range(len(spans), rank, world)
    return list(spans[b:e])


def morton_order(points: np.ndarray) -> np.ndarray:
    """Order of points along a 63-bit Morton curve over their bounding box (the
    engine's own spatial order), so row shards are spatially compact."""
    p = np.asarray(points, dtype=np.float64)
    if len(p) == 0:
        return np.zeros(0, dtype=np.int64)
    lo = p.min(axis=0)
    span = float((p.max(axis=0) - lo).max())
    s = (2 ** 21 - 1) / span if span > 0 else 0.0
    q = np.clip(((p - lo) * s), 0, 2 ** 21 - 1).astype(np.uint64)

    def spread(v):
        v = v & np.uint64(0x1FFFFF)
        for sh, m in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                      (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
            v = (v | (v << np.uint64(sh))) & np.uint64(m)
        return v

    key = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(key, kind="stable")


def shard_rows(Z: PointCloud, rank: int, world: int) -> PointCloud:
    """This rank's Morton-contiguous rows of the source cloud."""
    if world > Z.size():
        raise ValueError("row sharding needs at least one source row per rank")
    order = morton_order(Z.positions)
    b, e = shard_range(Z.size(), rank, world)
    rows = np.sort(order[b:e])
    feats = Z.features[rows] if Z.schema.total_dim else None
    return PointCloud(Z.positions[rows], Z.schema, feats)


# ------------------------------------------------------------- collective
class TorchCollective:
    """kreg_collective_fn over torch.distributed (CUDA tensors under NCCL, CPU
    under gloo), in place on the engine's host arrays. Keep the object alive
    while the engine may call it.

    deterministic=True (default): ONE all_gather of every rank's [sums, maxes]
    and the sums added in rank order on every rank, so the totals are
    bitwise independent of the collective's algorithm (ring / tree / NVLS) and
    equal on all ranks. deterministic=False: a SUM all_reduce of `sums` and a
    MAX all_reduce of `maxes` (two collectives, the backend's summation
    order)."""

    def __init__(self, group=None, deterministic: bool = True):
        from . import api
        self.group = group
        self.deterministic = deterministic
        self.calls = 0
        self.seconds = 0.0  # host wall time inside the callback (per-round collective latency)
        self.c_fn = api.COLLECTIVE_FN(self._call)

    def _call(self, user, sums, n_sums, maxes, n_maxes):
        import time
        t0 = time.perf_counter()
        try:
            import torch
            import torch.distributed as dist
            dev = _device()
            s = np.ctypeslib.as_array(sums, shape=(n_sums,)) if n_sums > 0 else np.zeros(0)
            m = np.ctypeslib.as_array(maxes, shape=(n_maxes,)) if n_maxes > 0 else np.zeros(0)
            if self.deterministic:
                world = dist.get_world_size(self.group)
                t = torch.from_numpy(np.concatenate([s, m])).to(dev)
                out = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(out, t, group=self.group)
                parts = np.stack([o.cpu().numpy() for o in out])  # [world, n_sums + n_maxes]
                tot = parts[0, :n_sums].copy()
                for r in range(1, world):  # fixed rank order
                    tot = tot + parts[r, :n_sums]
                if n_sums > 0:
                    s[:] = tot
                if n_maxes > 0:
                    m[:] = parts[:, n_sums:].max(axis=0)
            else:
                for host, op in ((s, dist.ReduceOp.SUM), (m, dist.ReduceOp.MAX)):
                    if host.size == 0:
                        continue
                    t = torch.from_numpy(host.copy()).to(dev)
                    dist.all_reduce(t, op=op, group=self.group)
                    host[:] = t.cpu().numpy()
            self.calls += 1
            self.seconds += time.perf_counter() - t0
            return 0
        except Exception:  # surfaced by the engine as a failed call
            return 1


class NcclCollective:
    """The collective as NCCL calls inside the engine (kreg_ctx_set_nccl: no
    host callback): rank 0 creates the ncclUniqueId, torch.distributed
    broadcasts it, and every rank's context joins one communicator on first
    use. deterministic=True: one ncclAllGather + rank-order sums (bitwise
    independent of NCCL's algorithm), else ncclAllReduce (sum, max)."""

    native = True

    def __init__(self, group=None, deterministic: bool = True):
        import torch.distributed as dist
        from . import api
        self.group = group
        self.deterministic = deterministic
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            api._check(api.lib().kreg_nccl_unique_id(uid))
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        self.uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        self._attached = set()

    def attach(self, ctx):
        from . import api
        if id(ctx) not in self._attached:  # one communicator per context
            api._check(api.lib().kreg_ctx_set_nccl(ctx.h, self.uid, self.rank, self.world, int(self.deterministic)))
            self._attached.add(id(ctx))

    def calls(self, ctx) -> int:
        from . import api
        return int(api.lib().kreg_ctx_nccl_calls(ctx.h))


# ------------------------------------------------------------- front ends
def register_clouds_sharded(X: PointCloud, Z: PointCloud, initial, params, config, ctx=None, group=None,
                            deterministic: bool = True):
    """register_clouds(X, Z, ...) with Z's rows sharded over the ranks (C4).
    Every rank returns the same RegistrationResult (TorchCollective modes)."""
    from . import api
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    Zr = shard_rows(Z, rank, world) if world > 1 else Z
    coll = TorchCollective(group, deterministic) if world > 1 else None
    return api.register_clouds_rows(X, Zr, Z.size(), initial, params, config, ctx=ctx, collective=coll)


def assemble_sequence(n_frames: int, parts) -> SequenceResult:
    """Merge per-rank [(pair, relative12, fallback, converged, indicator,
    iterations), ...] into one SequenceResult (trajectory composed as
    registration.cpp:226)."""
    m = n_frames - 1
    rel = [Isometry() for _ in range(m)]
    fb = np.zeros(m, dtype=np.uint8)
    cv = np.zeros(m, dtype=np.uint8)
    fi = np.zeros(m)
    it = np.zeros(m, dtype=np.int32)
    for part in parts:
        for p, r12, f, c, ind, n in part:
            rel[p] = Isometry.from12(np.asarray(r12))
            fb[p], cv[p], fi[p], it[p] = f, c, ind, n
    traj = [Isometry()]
    for k in range(m):
        traj.append(compose(traj[-1], rel[k]))
    return SequenceResult(relative=rel, trajectory=traj, fallback=fb, converged=cv, final_indicator=fi,
                          iterations=it)


def register_sequence_distributed(frames, params, config, n_chains: int, ctx=None, group=None) -> SequenceResult:
    """register_sequence over n_chains chains (C5), the chains split into one
    contiguous block per rank; every rank returns the assembled result."""
    from . import api
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    spans = chain_spans(len(frames), n_chains)
    mine = rank_spans(spans, rank, world)
    part = []
    if mine:
        res = api.register_sequence_spans(frames, mine, params, config, ctx=ctx)
        for b, e in mine:
            for p in range(b, e):
                part.append((p, res.relative[p].as12().tolist(), int(res.fallback[p]), int(res.converged[p]),
                             float(res.final_indicator[p]), int(res.iterations[p])))
    parts = [part]
    if world > 1:
        parts = [None] * world
        dist.all_gather_object(parts, part, group=group)
    return assemble_sequence(len(frames), parts)


__all__ = ["world_info", "init", "barrier", "reduce_scalar", "shard_range", "chain_spans", "rank_spans",
           "morton_order", "shard_rows", "TorchCollective", "register_clouds_sharded", "assemble_sequence",
           "register_sequence_distributed"]
