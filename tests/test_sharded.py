"""-m "not gpu": the multi-GPU host logic (ray sharding + ordered gather) on CPU
with the gloo backend, world_size 2.  The per-rank intersect is a stand-in
(the CPU oracle on the rank's slice, test infrastructure), so what is checked
is exactly the sharding and reassembly the NCCL path uses."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2305_01867_b200.sharded import FIELDS, shard_range


def test_shard_range_partitions():
    for n in (0, 1, 2, 7, 10, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_fn(V, T, S, E, mode):
    r = oracle.run(V.numpy(), T.numpy(), S.numpy(), E.numpy(), flags=False)
    out = {"hit": torch.from_numpy(r["hit"]), "count": torch.from_numpy(r["count"]),
           "tri": torch.from_numpy(r["tri"]), "t": torch.from_numpy(r["t"].astype(np.float32)),
           "dist": torch.from_numpy(r["dist"].astype(np.float32)),
           "point": torch.from_numpy(r["point"].astype(np.float32))}
    return {k: out[k] for k in FIELDS[mode]}


def _worker(rank, world, port, n_rays, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_01867_b200.sharded import intersect_sharded
        V, T, S, E, _ = synth.workload("cube", n_rays, seed=5)
        V, T, S, E = (torch.from_numpy(a) for a in (V, T, S, E))
        res = {}
        for mode in ("boolean", "barycentric", "intercept_count"):
            g = intersect_sharded(V, T, S, E, mode, intersect_fn=_oracle_fn)
            if rank == 0:
                res[mode] = {k: v.numpy() for k, v in g.items()}
            else:
                assert g is None
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_rays", [1, 1001])
def test_gloo_world2_gather_matches_single_process(n_rays):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_rays, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    V, T, S, E, _ = synth.workload("cube", n_rays, seed=5)
    ref = oracle.run(V, T, S, E, flags=False)
    assert (res["boolean"]["hit"] == ref["hit"]).all()
    assert (res["intercept_count"]["count"] == ref["count"]).all()
    assert (res["barycentric"]["tri"] == ref["tri"]).all()
    m = ref["tri"] >= 0
    np.testing.assert_allclose(res["barycentric"]["point"][m], ref["point"][m], atol=1e-6)


def _pipe_worker(rank, world, port, n_rays, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_01867_b200.sharded import GatherPipeline
        pipe = GatherPipeline(slots=2)
        got = []
        for step in range(4):  # 4 steps over 2 slots: every slot is reused once
            V, T, S, E, _ = synth.workload("cube", n_rays, seed=10 + step)
            lo, hi = shard_range(n_rays, rank, world)
            loc = _oracle_fn(*(torch.from_numpy(a) for a in (V, T, S[lo:hi], E[lo:hi])), "barycentric")
            pending = pipe.start(step % 2, loc, n_rays)
            if step % 2 == 1:  # collect the two steps in flight
                for pg in prev, pending:
                    r = pg.wait()
                    if rank == 0:
                        got.append({k: v.clone().numpy() for k, v in r.items()})
                    else:
                        assert r is None
            prev = pending
        pipe.drain()
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_rays", [1000, 1001])
def test_gloo_world2_pipelined_gather(n_rays):
    """GatherPipeline (the bench's overlapped gather): asynchronous gathers into
    reused receive buffers give each step's outputs in ray order (equal and
    padded slices)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_worker, args=(r, 2, port, n_rays, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(got) == 4
    for step in range(4):
        V, T, S, E, _ = synth.workload("cube", n_rays, seed=10 + step)
        ref = oracle.run(V, T, S, E, flags=False)
        assert (got[step]["tri"] == ref["tri"]).all()
        m = ref["tri"] >= 0
        np.testing.assert_allclose(got[step]["point"][m], ref["point"][m], atol=1e-6)


def _pipe_modes_worker(rank, world, port, n_rays, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2305_01867_b200.sharded import GatherPipeline
        pipe = GatherPipeline(slots=2)
        V, T, S, E, _ = synth.workload("cube", n_rays, seed=21)
        lo, hi = shard_range(n_rays, rank, world)
        got = []
        for step, mode in enumerate(("boolean", "barycentric", "intercept_count", "barycentric", "boolean")):
            loc = _oracle_fn(*(torch.from_numpy(a) for a in (V, T, S[lo:hi], E[lo:hi])), mode)
            r = pipe.start(step % 2, loc, n_rays).wait()  # slots change field sets between modes
            if rank == 0:
                got.append((mode, {k: v.clone().numpy() for k, v in r.items()}))
        pipe.drain()
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


def test_gloo_world2_pipeline_mode_switch():
    """A GatherPipeline slot reused by a different mode (other fields) reallocates
    its receive buffers; every step's gathered outputs equal the oracle's."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pipe_modes_worker, args=(r, 2, port, 777, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    V, T, S, E, _ = synth.workload("cube", 777, seed=21)
    ref = oracle.run(V, T, S, E, flags=False)
    for mode, out in got:
        if mode == "boolean":
            assert (out["hit"] == ref["hit"]).all()
        elif mode == "intercept_count":
            assert (out["count"] == ref["count"]).all()
        else:
            assert (out["tri"] == ref["tri"]).all()
