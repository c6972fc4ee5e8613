"""-m gpu: the ray-sharded multi-process path with the
REAL CUDA path on every rank.  Two processes share cuda:0 (the GPU box has one
device) and gather over gloo; with >= 2 visible devices each rank takes its own
GPU and the gather runs over NCCL.  The gathered outputs are compared element
by element with the CPU oracle (boolean / intercept_count / nearest id exact,
t / dist / point within the north_star tolerances), on ragged slices."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    ndev = torch.cuda.device_count()
    dev = torch.device("cuda", rank % ndev)
    torch.cuda.set_device(dev)
    if ndev >= world:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:  # ranks share a device: gloo gather (host staging)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return dev


def _np(d):
    return {k: v.cpu().numpy().copy() for k, v in d.items()}


def _sharded_worker(rank, world, port, workload, n_rays, seed, q):
    try:
        _init(rank, world, port)
        from paper_2305_01867_b200 import rsi
        from paper_2305_01867_b200.sharded import intersect_sharded
        V, T, S, E, _ = synth.workload(workload, n_rays, seed=seed)
        V, T, S, E = (torch.from_numpy(a) for a in (V, T, S, E))
        res = {}
        launches0 = rsi.rsi_launch_count()
        for mode in ("boolean", "barycentric", "intercept_count"):
            g = intersect_sharded(V, T, S, E, mode)  # intersect_fn=None: the CUDA path
            if rank == 0:
                res[mode] = _np(g)
            else:
                assert g is None
        res["launches"] = rsi.rsi_launch_count() - launches0
        q.put((rank, res))
    except BaseException as e:  # surface the failure in the parent
        q.put((rank, repr(e)))
        raise
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, res = q.get(timeout=600)
        assert not isinstance(res, str), f"rank {rank}: {res}"
        got[rank] = res
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return got


def _check_modes(res, ref, S, E):
    assert (res["boolean"]["hit"] == ref["hit"]).all()
    assert (res["intercept_count"]["count"] == ref["count"]).all()
    b = res["barycentric"]
    assert (b["tri"] == ref["tri"]).all()
    m = ref["tri"] >= 0
    dn = np.linalg.norm(E.astype(np.float64) - S, axis=1)
    assert np.all(np.abs(b["t"][m] - ref["t"][m]) <= 1e-5)
    assert np.all(np.abs(b["dist"][m] - ref["dist"][m]) <= 1e-5 * np.maximum(dn[m], 1e-30))
    scale = np.maximum(np.abs(S).max(1), np.abs(E).max(1))[m]
    assert np.all(np.abs(b["point"][m] - ref["point"][m]).max(1) <= 1e-5 * np.maximum(scale, 1e-30))
    assert np.all(np.isnan(b["t"][~m]))


@pytest.mark.parametrize("world,workload,n_rays", [(2, "sphere", 1), (2, "sphere", 1001), (2, "sphere", 100_003),
                                                   (3, "terrain", 20_011)])
def test_intersect_sharded_cuda_vs_oracle(world, workload, n_rays):
    """intersect_sharded with the CUDA path on every rank: replicated build,
    contiguous ragged slices, gather to rank 0 in ray order == the oracle."""
    got = _spawn(_sharded_worker, world, workload, n_rays, 31)
    V, T, S, E, _ = synth.workload(workload, n_rays, seed=31)
    ref = oracle.run(V, T, S, E, flags=False)
    _check_modes(got[0], ref, S, E)
    for r in range(world):  # every rank ran the library's kernels (no fallback)
        assert got[r]["launches"] > 0


def _pipe_worker(rank, world, port, n_rays, q):
    try:
        dev = _init(rank, world, port)
        from paper_2305_01867_b200 import rsi
        from paper_2305_01867_b200.sharded import FIELDS, GatherPipeline, shard_range
        V, T, _, _, _ = synth.workload("sphere", 8, seed=0)
        Vd, Td = torch.from_numpy(V).to(dev), torch.from_numpy(T).to(dev)
        lo, hi = shard_range(n_rays, rank, world)
        pipe = GatherPipeline(slots=2)
        got = []
        with rsi.rsi_build(Vd, Td) as h:
            pending = []
            modes = ("barycentric", "barycentric", "boolean", "intercept_count", "barycentric", "boolean")
            outs = [None, None]
            for step, mode in enumerate(modes):  # 6 steps over 2 slots: each slot reused, fields change
                _, _, S, E, _ = synth.workload("sphere", n_rays, seed=100 + step)
                Sd, Ed = torch.from_numpy(S[lo:hi]).to(dev), torch.from_numpy(E[lo:hi]).to(dev)
                rsi.rsi_rebuild(h, Vd, Td)
                outs[step % 2] = rsi.rsi_intersect(h, Sd, Ed, mode)
                pending.append((mode, pipe.start(step % 2, {f: outs[step % 2][f] for f in FIELDS[mode]}, n_rays)))
                if step % 2 == 1:  # two gathers in flight, then collect both
                    for m, pg in pending:
                        r = pg.wait()
                        if rank == 0:
                            got.append((m, _np(r)))
                        else:
                            assert r is None
                    pending = []
            pipe.drain()
        q.put((rank, got))
    except BaseException as e:
        q.put((rank, repr(e)))
        raise
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("n_rays", [1000, 100_003])
def test_gather_pipeline_cuda_slot_reuse_vs_oracle(n_rays):
    """GatherPipeline (the bench's overlapped gather) on the CUDA path at W=2:
    asynchronous gathers into reused receive slots, mode switches, every step's
    gathered outputs == the oracle's."""
    got = _spawn(_pipe_worker, 2, n_rays)[0]
    assert len(got) == 6
    V, T, _, _, _ = synth.workload("sphere", 8, seed=0)
    for step, (mode, out) in enumerate(got):
        _, _, S, E, _ = synth.workload("sphere", n_rays, seed=100 + step)
        ref = oracle.run(V, T, S, E, flags=False)
        if mode == "boolean":
            assert (out["hit"] == ref["hit"]).all(), step
        elif mode == "intercept_count":
            assert (out["count"] == ref["count"]).all(), step
        else:
            assert (out["tri"] == ref["tri"]).all(), step
            m = ref["tri"] >= 0
            assert np.all(np.abs(out["t"][m] - ref["t"][m]) <= 1e-5), step
