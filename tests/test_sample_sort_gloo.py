"""CPU, world_size 2 and 3 over gloo: the multi-rank sample sort host logic
(paper_1105_6040_b200/sample_sort.py) with the device steps replaced by their
CPU restatements (tests/cpu_ops.py). The ranks' outputs concatenated in rank
order must equal the oracle's sort of the whole input -- the array the
reference's scatter_merge_sort gathers at its master
(P/src/parallel_sort.cpp:246-248) -- including stability of the payload,
skewed inputs and empty shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def make_input(kind, n, dt, seed=1):
    z = oracle.gen_data_np(n, seed)
    if kind == "uniform":
        x = z
    elif kind == "equal":
        x = np.full(n, 12345, dtype=np.uint64)
    elif kind == "sorted":
        x = np.arange(n, dtype=np.uint64)
    elif kind == "reverse":
        x = np.arange(n, dtype=np.uint64)[::-1].copy()
    elif kind == "zipf":  # heavy duplicates: a handful of values dominate
        r = (z >> np.uint64(11)).astype(np.float64) / 2.0 ** 53
        x = np.floor(1.0 / np.maximum(r, 1e-9) ** 0.8).astype(np.uint64) % np.uint64(1 << 20)
    else:
        raise ValueError(kind)
    if dt == np.int32:
        return (x >> np.uint64(33)).astype(np.int32) if kind == "uniform" else x.astype(np.int32)
    if dt == np.uint32:
        return (x >> np.uint64(32)).astype(np.uint32) if kind == "uniform" else x.astype(np.uint32)
    if dt == np.int64:
        return x.view(np.int64) if kind == "uniform" else x.astype(np.int64)
    return x.astype(np.uint64)


def _worker(rank, world, port, cases, result_dir):
    import sys
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    from cpu_ops import CpuOps, to_np, to_t

    from paper_1105_6040_b200.sample_sort import SampleSorter

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for ci, (kind, n, dt, with_vals, samples) in enumerate(cases):
            full = make_input(kind, n, dt)
            sizes = oracle.plan_partition(n, world)  # P/src/parallel_sort.cpp:26-38
            off = sum(sizes[:rank])
            shard = full[off: off + sizes[rank]]
            vals = np.arange(off, off + sizes[rank], dtype=np.uint32)
            sorter = SampleSorter(group=None, samples_per_rank=samples, ops=CpuOps())
            k, v = sorter.sort(to_t(shard), to_t(vals) if with_vals else None)
            ok = sorter.verify(k, to_t(shard))
            np.save(os.path.join(result_dir, f"c{ci}_r{rank}_k.npy"), to_np(k))
            if with_vals:
                np.save(os.path.join(result_dir, f"c{ci}_r{rank}_v.npy"), to_np(v))
            np.save(os.path.join(result_dir, f"c{ci}_r{rank}_meta.npy"),
                    np.array([int(ok)] + list(sorter.last_bucket_sizes), dtype=np.int64))
    finally:
        dist.destroy_process_group()


CASES = [
    ("uniform", 50_000, np.uint32, False, 64),
    ("uniform", 40_001, np.int32, True, 64),
    ("uniform", 30_000, np.uint64, True, 64),
    ("uniform", 20_000, np.int64, False, 16),
    ("equal", 30_000, np.int32, True, 64),
    ("sorted", 30_000, np.int32, False, 64),
    ("reverse", 30_000, np.int32, False, 64),
    ("zipf", 50_000, np.int32, True, 64),
    ("uniform", 1, np.uint32, False, 64),   # empty shard on the other ranks
    ("uniform", 0, np.uint32, False, 64),
]


@pytest.mark.parametrize("world", [2, 3])
def test_sample_sort_gloo(tmp_path, world):
    port = _free_port()
    mp.spawn(_worker, args=(world, port, CASES, str(tmp_path)), nprocs=world, join=True)
    for ci, (kind, n, dt, with_vals, _) in enumerate(CASES):
        full = make_input(kind, n, dt)
        ks = [np.load(tmp_path / f"c{ci}_r{r}_k.npy") for r in range(world)]
        metas = [np.load(tmp_path / f"c{ci}_r{r}_meta.npy") for r in range(world)]
        assert all(m[0] == 1 for m in metas), (kind, n, "verify() failed")
        got = np.concatenate(ks)
        if with_vals:
            ek, ev = oracle.stable_sort_kv(full, np.arange(n, dtype=np.uint32))
            gv = np.concatenate([np.load(tmp_path / f"c{ci}_r{r}_v.npy") for r in range(world)])
            assert np.array_equal(got, ek) and np.array_equal(gv, ev), (kind, n, dt)
        else:
            assert np.array_equal(got, oracle.sort(full)), (kind, n, dt)
        # load balance: regular sampling with compound keys bounds every bucket
        sizes = [len(k) for k in ks]
        if n >= 1000:
            assert max(sizes) <= 2 * n / world + 64 * world, (kind, sizes)
