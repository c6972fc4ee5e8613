"""Ray-sharded multi-GPU driver.

Rays are independent, so the path shards with no data-path collective: every
rank replicates the mesh, builds its own BVH on its GPU (rsi_build), and
intersects the contiguous ray slice [floor(r N / W), floor((r+1) N / W)).  The
only collective is the final gather of the per-ray outputs to rank 0 in ray
order (north_star: "NCCL over NVLink is used only to gather the per-ray
outputs").  The gather pads every slice to ceil(N / W) rows and uses one
dist.gather per output field (NCCL over NVLink on GPUs, gloo in the CPU
tests), then trims the padding on rank 0.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

# output fields per mode, in rsi_outputs_t order
FIELDS = {"boolean": ("hit",), "intercept_count": ("count",), "barycentric": ("tri", "t", "dist", "point")}


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice of rank `rank` out of `world` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def gather_outputs(local: dict, n_total: int, group=None, dst: int = 0) -> dict | None:
    """Gather per-ray outputs of every rank's slice to rank `dst` in ray order
    (one dist.gather per output field: NCCL point-to-point over NVLink on GPUs,
    gloo in the CPU tests).  Slices are padded to ceil(N / W) rows.  Returns the
    full arrays on `dst` and None on the other ranks."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per = -(-n_total // world)
    lo, hi = shard_range(n_total, rank, world)
    out = {}
    for k in sorted(local):
        t = local[k]
        if t.shape[0] != hi - lo:
            raise ValueError(f"{k}: slice has {t.shape[0]} rows, expected {hi - lo}")
        dev = t.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
        pad = torch.zeros((per,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        pad[: hi - lo] = t
        bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
        dist.gather(pad, bufs, dst=dst, group=group)
        if rank == dst:
            out[k] = torch.cat([bufs[r][: shard_range(n_total, r, world)[1] - shard_range(n_total, r, world)[0]]
                                for r in range(world)], 0)
    return out if rank == dst else None


class PendingGather:
    """An in-flight gather (GatherPipeline.start): `wait()` makes the caller's
    stream wait for it (NCCL: a device-side wait, the host does not block) and
    returns the full outputs on the destination rank, None elsewhere."""

    def __init__(self, works, recv, n_total, world, rank, dst):
        self.works, self.recv, self.n_total, self.world, self.rank, self.dst = works, recv, n_total, world, rank, dst

    def wait(self):
        for w in self.works:
            w.wait()
        self.works = []
        if self.rank != self.dst:
            return None
        # slices are padded to ceil(N / W) rows: drop the padding (a view when none)
        per = -(-self.n_total // self.world)
        out = {}
        for k, buf in self.recv.items():
            if per * self.world == self.n_total:
                out[k] = buf[: self.n_total]
            else:
                out[k] = torch.cat([buf[r * per: r * per + (shard_range(self.n_total, r, self.world)[1]
                                                          - shard_range(self.n_total, r, self.world)[0])]
                                    for r in range(self.world)], 0)
        return out


class GatherPipeline:
    """Asynchronous ordered gather of per-ray outputs into receive buffers
    allocated once (weak-scaling steps: the gather of step k overlaps the
    build + traversal of step k+1, as the NCCL work runs on its own stream).
    Each slot owns its receive buffers; `start` waits for the slot's previous
    gather before reusing them.  Slices of ceil(N / W) rows are sent in place
    when no padding is needed (the equal-slice case), else through a padded copy."""

    def __init__(self, slots: int = 2, group=None, dst: int = 0):
        self.group, self.dst = group, dst
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.slots = [None] * slots
        self.recv = [None] * slots

    def start(self, slot: int, local: dict, n_total: int) -> PendingGather:
        if self.slots[slot] is not None:
            self.slots[slot].wait()
        per = -(-n_total // self.world)
        lo, hi = shard_range(n_total, self.rank, self.world)
        nccl = dist.get_backend(self.group) == "nccl"
        def fits(buf, t):
            return (buf is not None and buf.shape[0] == per * self.world and buf.shape[1:] == t.shape[1:]
                    and buf.dtype == t.dtype)

        if self.rank == self.dst and (self.recv[slot] is None or set(self.recv[slot]) != set(local) or
                                      not all(fits(self.recv[slot][k], t) for k, t in local.items())):
            self.recv[slot] = {k: torch.empty((per * self.world,) + tuple(t.shape[1:]), dtype=t.dtype,
                                              device=t.device if nccl else torch.device("cpu"))
                               for k, t in local.items()}
        works = []
        for k in sorted(local):
            t = local[k]
            if t.shape[0] != hi - lo:
                raise ValueError(f"{k}: slice has {t.shape[0]} rows, expected {hi - lo}")
            if not nccl:
                t = t.cpu()
            if hi - lo != per:
                pad = torch.zeros((per,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                pad[: hi - lo] = t
                t = pad
            bufs = list(self.recv[slot][k].split(per)) if self.rank == self.dst else None
            works.append(dist.gather(t.contiguous(), bufs, dst=self.dst, group=self.group, async_op=True))
        self.slots[slot] = PendingGather(works, self.recv[slot], n_total, self.world, self.rank, self.dst)
        return self.slots[slot]

    def drain(self):
        for i, pg in enumerate(self.slots):
            if pg is not None:
                pg.wait()
                self.slots[i] = None


# per-ray output fields: dtype and columns (rsi_outputs_t)
FIELD_SPEC = {"hit": (torch.uint8, 1), "count": (torch.int32, 1), "tri": (torch.int32, 1),
              "t": (torch.float32, 1), "dist": (torch.float32, 1), "point": (torch.float32, 3)}


class PeerOutputs:
    """The fused alternative to the gather: every rank's
    traversal epilogue writes its slice of the per-ray outputs STRAIGHT INTO
    RANK 0's buffers over NVLink (peer-mapped symmetric memory), so no separate
    collective moves them; `complete()` is a device-side barrier across the
    ranks on the current stream (each rank's kernel precedes it in stream
    order, and the barrier's release/acquire makes the peer writes visible on
    rank 0).  Every rank allocates the same symmetric buffers; only rank 0's
    are written.  Correct by construction: each rank writes the disjoint rows
    [floor(r N / W), floor((r+1) N / W)) of the full arrays, exactly the rows
    the gather would place there.  A step is begin() -> traversal into
    outputs() -> complete(): begin() holds every rank's writes until rank 0's
    stream has passed its uses of the previous result() (enqueued before its
    own begin()), so the buffers can be reused step after step.  Opt-in (bench --fused-gather); the default
    multi-GPU path is GatherPipeline."""

    def __init__(self, n_total: int, mode: str, device, group=None):
        import torch.distributed._symmetric_memory as symm
        self.group = group if group is not None else dist.group.WORLD
        self.world = dist.get_world_size(self.group)
        self.rank = dist.get_rank(self.group)
        self.n_total = n_total
        lo, hi = shard_range(n_total, self.rank, self.world)
        self.local, self.slices, self._handles = {}, {}, []
        self._steps = 0
        for f in FIELDS[mode]:
            dtype, cols = FIELD_SPEC[f]
            buf = symm.empty(n_total * cols, dtype=dtype, device=device)
            hdl = symm.rendezvous(buf, self.group)
            remote = hdl.get_buffer(0, (n_total * cols,), dtype)  # rank 0's buffer, mapped here
            shape = (n_total, cols) if cols > 1 else (n_total,)
            self.local[f] = buf.view(shape)
            self.slices[f] = remote.view(shape)[lo:hi]
            self._handles.append(hdl)

    def outputs(self) -> dict:
        """Output tensors for rsi_intersect: this rank's rows of rank 0's arrays.
        Call `begin()` before the step that writes them."""
        return self.slices

    def begin(self):
        """Device-side barrier before a step's peer writes (write-after-read):
        no rank overwrites rank 0's rows while rank 0 may still be consuming
        the previous step's result() on its stream.  Skipped for the first
        step (nothing to protect yet)."""
        if self._steps > 0:
            self._handles[0].barrier(channel=1)

    def complete(self):
        """Device-side barrier of all ranks on the current stream: afterwards
        rank 0's arrays hold every rank's rows."""
        self._handles[0].barrier(channel=0)
        self._steps += 1

    def result(self) -> dict | None:
        """The full outputs on rank 0 (valid after complete()), None elsewhere."""
        return self.local if self.rank == 0 else None


def intersect_sharded(vertices: torch.Tensor, triangles: torch.Tensor, start: torch.Tensor, end: torch.Tensor,
                      mode: str = "boolean", options=None, group=None, intersect_fn=None) -> dict:
    """Replicated build + sharded intersect + gather.  `start`/`end` are the
    FULL ray arrays (any device; this rank's slice is moved to its GPU).
    `intersect_fn(vertices, triangles, s, e, mode) -> dict` defaults to the
    CUDA path (rsi_build + rsi_intersect on the current device)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = start.shape[0]
    lo, hi = shard_range(n, rank, world)
    if intersect_fn is None:
        from . import rsi
        dev = torch.device("cuda", torch.cuda.current_device())
        V, T = vertices.to(dev), triangles.to(dev)
        s, e = start[lo:hi].to(dev), end[lo:hi].to(dev)
        with rsi.rsi_build(V, T, options) as h:
            local = rsi.rsi_intersect(h, s, e, mode)
    else:
        local = intersect_fn(vertices, triangles, start[lo:hi], end[lo:hi], mode)
    local = {k: local[k] for k in FIELDS[mode] if k in local}
    return gather_outputs(local, n, group)  # full outputs on rank 0, None elsewhere
