"""GPU: the sample-sort device steps (b2s_sample_regular, b2s_select_splitters,
b2s_bucket_bounds, b2s_merge) bit-identical to their CPU restatements, and the
whole pipeline with G emulated ranks on one device (the exchange done by
slicing; no rank waits on another) equal to the oracle's sort. Plus the
torch.distributed path itself over NCCL at world size 1."""
import os
import socket

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from cpu_ops import CpuOps, to_np, to_t  # noqa: E402
from paper_1105_6040_b200.device import Context  # noqa: E402
from test_sample_sort_gloo import make_input  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def dev(x):
    return to_t(x).cuda()


def host(t):
    return to_np(t.cpu())


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("kind,dt,with_vals", [("uniform", np.uint32, False),
                                               ("uniform", np.int32, True),
                                               ("uniform", np.uint64, True),
                                               ("equal", np.int32, True),
                                               ("zipf", np.int32, False),
                                               ("sorted", np.int64, False),
                                               ("reverse", np.int32, False)])
def test_emulated_ranks(ctx, world, kind, dt, with_vals):
    n = 200_003
    full = make_input(kind, n, dt)
    sizes = oracle.plan_partition(n, world)
    cpu = CpuOps()
    shards, vshards, samples = [], [], []
    off = 0
    for r in range(world):
        sh = dev(full[off: off + sizes[r]])
        v = dev(np.arange(off, off + sizes[r], dtype=np.uint32)) if with_vals else None
        sk, sv = ctx.sort(sh, vals=v)
        shards.append(sk)
        vshards.append(sv)
        smp = ctx.sample_regular(sk, r, 64)
        assert np.array_equal(host(smp), host(cpu.sample(sk.cpu(), r, 64)))
        samples.append(smp)
        off += sizes[r]
    allsmp = torch.cat(samples)
    spl = ctx.select_splitters(allsmp, world)
    assert np.array_equal(host(spl), host(cpu.select(allsmp.cpu(), world)))
    bounds = []
    for r in range(world):
        b = ctx.bucket_bounds(shards[r], r, spl, world)
        assert np.array_equal(b.cpu().numpy(), cpu.bounds(shards[r].cpu(), r, spl.cpu(), world).numpy())
        bounds.append(b.cpu().tolist())
    outs, vouts = [], []
    for dst in range(world):
        runs = [shards[g][bounds[g][dst]: bounds[g][dst + 1]] for g in range(world)]
        vr = [vshards[g][bounds[g][dst]: bounds[g][dst + 1]] for g in range(world)] if with_vals else None
        if sum(r.numel() for r in runs) == 0:
            continue
        k, v = ctx.merge([r.contiguous() for r in runs],
                         vals=[x.contiguous() for x in vr] if vr else None)
        outs.append(host(k))
        if with_vals:
            vouts.append(host(v))
    got = np.concatenate(outs)
    if with_vals:
        ek, ev = oracle.stable_sort_kv(full, np.arange(n, dtype=np.uint32))
        assert np.array_equal(got, ek) and np.array_equal(np.concatenate(vouts), ev)
    else:
        assert np.array_equal(got, oracle.sort(full))
    assert max(len(o) for o in outs) <= 2 * n / world + 64 * world


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_distributed_path_nccl_world1(ctx, transport):
    import torch.distributed as dist

    from paper_1105_6040_b200.sample_sort import SampleSorter
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        keys = ctx.gen_keys(1 << 20, 3, torch.int32, shift=33)
        vals = torch.arange(1 << 20, dtype=torch.int32, device="cuda")
        sorter = SampleSorter(ctx, force_exchange=True, transport=transport)
        k, v = sorter.sort(keys, vals)
        assert sorter.verify(k, keys)
        ek, ev = oracle.stable_sort_kv(keys.cpu().numpy(), np.arange(1 << 20, dtype=np.uint32))
        assert np.array_equal(k.cpu().numpy(), ek)
        assert np.array_equal(v.cpu().numpy().view(np.uint32), ev)
        assert set(sorter.last_phase_ms) >= {"local_sort", "splitters", "exchange", "merge"}
    finally:
        dist.destroy_process_group()


def _p2p_rank(rank, world, port, kind, dt, with_vals, n, q):
    """One rank of the pull-exchange test: its own process and context on the
    one GPU; peers' sorted shards are mapped through CUDA IPC and read by this
    rank's merge kernel. Host collectives (gloo) order the steps: no kernel
    waits on another rank."""
    import torch.distributed as dist

    from paper_1105_6040_b200.device import Context
    from paper_1105_6040_b200.sample_sort import SampleSorter
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx = Context(0)
        full = make_input(kind, n, dt)
        sizes = oracle.plan_partition(n, world)
        off = sum(sizes[:rank])
        keys = dev(full[off: off + sizes[rank]])
        vals = dev(np.arange(off, off + sizes[rank], dtype=np.uint32)) if with_vals else None
        sorter = SampleSorter(ctx, transport="p2p")
        outs = []
        for _ in range(2):  # the second sort reuses the mapped buffers
            k, v = sorter.sort(keys, vals)
            outs.append((host(k), host(v) if v is not None else None))
        res = [None] * world
        dist.all_gather_object(res, outs)
        if rank == 0:
            q.put(res)
        dist.barrier()
        ctx.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind,dt,with_vals", [("uniform", np.int32, True),
                                               ("equal", np.uint64, True),
                                               ("zipf", np.int32, False)])
def test_p2p_pull_exchange_processes(world, kind, dt, with_vals):
    """The p2p transport across `world` processes on the one GPU (CUDA IPC
    works between processes on the same device): each rank's bucket is pulled
    from every peer's exported shard by its merge kernel."""
    import torch.multiprocessing as mp
    n = 300_007
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_p2p_rank, args=(r, world, port, kind, dt, with_vals, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, t0 = None, time.time()
    while res is None:
        try:
            res = q.get(timeout=2)
        except queue.Empty:
            bad = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if bad or time.time() - t0 > 300:
                for p in procs:
                    p.kill()
                pytest.fail(f"rank processes failed: exit codes {[p.exitcode for p in procs]}")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full = make_input(kind, n, dt)
    for it in range(2):
        got = np.concatenate([res[r][it][0] for r in range(world)])
        if with_vals:
            ek, ev = oracle.stable_sort_kv(full, np.arange(n, dtype=np.uint32))
            assert np.array_equal(got, ek)
            assert np.array_equal(np.concatenate([res[r][it][1] for r in range(world)]).view(np.uint32), ev)
        else:
            assert np.array_equal(got, oracle.sort(full))
