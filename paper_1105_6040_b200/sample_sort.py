"""Multi-GPU sample sort: the B200 replacement of the reference's
scatter / odd-even exchange / gather across ranks.

The reference (P/src/parallel_sort.cpp:166-254) scatters contiguous blocks
(plan_partition, :26-38), sorts each block, then runs p odd-even merge_split
phases (:217-244) -- p full-block exchanges -- and gathers at rank 0
(:246-248). Here every GPU is one process (torch.distributed, NCCL over
NVLink/NVSwitch) holding its contiguous shard, and the global order is reached
with exactly ONE data exchange:

  1. local stable radix sort of the shard                     (b2s_sort)
  2. s regular samples (key, rank, position) of the sorted shard (b2s_sample_regular)
  3. all-gather of the samples                                 (NCCL all_gather)
  4. splitter i = sample of rank i*m/G in (key, rank, pos) order (b2s_select_splitters)
  5. bucket bounds: local keys ordered before each splitter    (b2s_bucket_bounds)
  6. counts exchange, then the variable all-to-all of keys     (NCCL all_to_all)
  7. stable k-way merge of the G received runs                 (b2s_merge)

transport="p2p" fuses 6 and 7: the local sort writes into the context's
IPC-exported buffer (b2s_exchange_buffer), the ranks all-gather their bucket
bounds and buffer handles (a few hundred bytes), and each rank's merge kernel
reads its slice of every peer's sorted shard straight over NVLink
(b2s_open_peer + b2s_merge on peer pointers): no receive buffer, no separate
all-to-all, the exchange overlaps the merge tile by tile. A stream-ordered
all-reduce after the merge keeps every rank from re-sorting into its buffer
while peers still read it.

Bucket r (the output on rank r) is the r-th slice of the global order, so the
ranks' outputs concatenated in rank order are the sorted input -- the array the
reference gathers at its master. Because records compare as (key, rank,
position), equal keys (all-equal or Zipf inputs) still split evenly and the
result is stable by global index, which the key/value configuration needs.

The step kernels are the CUDA C-ABI functions (CudaOps). The host logic takes
an `ops` object so that the gloo tests can drive it on CPU with the oracle.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

_WIRE = {torch.uint32: torch.int32, torch.uint64: torch.int64, torch.int32: torch.int32,
         torch.int64: torch.int64}


def _wire(t: torch.Tensor) -> torch.Tensor:
    """Bit-identical view with a dtype every collective backend carries."""
    return t.view(_WIRE[t.dtype]) if t.dtype in (torch.uint32, torch.uint64) else t


class CudaOps:
    """The device steps, all through libb200sort.so (no CPU fallback)."""

    def __init__(self, ctx):
        self.ctx = ctx

    def sort(self, keys, vals):
        return self.ctx.sort(keys, vals=vals)

    def sample(self, sorted_keys, rank, s):
        return self.ctx.sample_regular(sorted_keys, rank, s)

    def select(self, samples, nparts):
        return self.ctx.select_splitters(samples, nparts)

    def bounds(self, sorted_keys, rank, splitters, nparts):
        return self.ctx.bucket_bounds(sorted_keys, rank, splitters, nparts)

    def merge(self, runs, vals):
        return self.ctx.merge(runs, vals=vals)

    def sort_into(self, keys, vals, out, vals_out):
        return self.ctx.sort(keys, out=out, vals=vals, vals_out=vals_out)

    def check(self, keys):
        return self.ctx.check_sorted(keys)


class SampleSorter:
    """Sorts a key (or key/uint32-value) array sharded over the ranks of a
    process group; returns this rank's bucket of the global order."""

    def __init__(self, ctx=None, group=None, samples_per_rank: int = 64, ops=None,
                 force_exchange: bool = False, transport: str = "nccl"):
        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown transport {transport!r} (nccl or p2p)")
        if transport == "p2p" and ctx is None:
            raise ValueError("the p2p transport needs a device context")
        self.ctx = ctx
        self.transport = transport
        self.group = group
        self.force_exchange = force_exchange
        self.samples = samples_per_rank
        self.ops = ops if ops is not None else CudaOps(ctx)
        self.last_phase_ms = {}
        self.last_bucket_sizes = []
        self._timing = ctx is not None and ops is None
        self._hinfo = None  # p2p: (handle, payload offset) and its device copy

    @property
    def rank(self) -> int:
        return dist.get_rank(self.group)

    @property
    def world(self) -> int:
        return dist.get_world_size(self.group)

    def sort(self, keys: torch.Tensor, vals: torch.Tensor | None = None):
        if self.transport == "p2p":
            return self._sort_p2p(keys, vals)
        rank, world = self.rank, self.world
        ev = _Events(self._timing)
        ev.mark("start")
        skeys, svals = self.ops.sort(keys, vals)
        ev.mark("local_sort")
        if world == 1 and not self.force_exchange:
            self.last_bucket_sizes = [skeys.numel()]
            ev.finish(self)
            return skeys, svals

        samples = self.ops.sample(skeys, rank, self.samples)
        gathered = torch.empty((world * self.samples, 2), dtype=samples.dtype,
                               device=samples.device)
        dist.all_gather_into_tensor(_wire(gathered), _wire(samples.contiguous()),
                                    group=self.group)
        splitters = self.ops.select(gathered, world)
        bounds = self.ops.bounds(skeys, rank, splitters, world)
        ev.mark("splitters")

        send_counts = (bounds[1:] - bounds[:-1]).to(torch.int64)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        counts = torch.stack([send_counts, recv_counts]).cpu()  # NCCL needs host split sizes
        send, recv = counts[0].tolist(), counts[1].tolist()
        total = sum(recv)
        rkeys = torch.empty(total, dtype=skeys.dtype, device=skeys.device)
        dist.all_to_all_single(_wire(rkeys), _wire(skeys), recv, send, group=self.group)
        rvals = None
        if svals is not None:
            rvals = torch.empty(total, dtype=svals.dtype, device=svals.device)
            dist.all_to_all_single(_wire(rvals), _wire(svals), recv, send, group=self.group)
        ev.mark("exchange")

        runs = list(torch.split(rkeys, recv))
        vruns = list(torch.split(rvals, recv)) if rvals is not None else None
        if total == 0:
            out_k, out_v = rkeys, rvals
        else:
            out_k, out_v = self.ops.merge(runs, vruns)
        ev.mark("merge")
        self.last_bucket_sizes = recv
        ev.finish(self)
        return out_k, out_v

    def p2p_available(self) -> tuple[bool, str]:
        """Collective probe of the p2p transport: every rank exports its buffer
        and maps every peer's. All ranks get the same answer (False when any
        rank failed), plus this rank's error text."""
        world, dev = self.world, torch.device("cuda", self.ctx.device)
        gloo = dist.get_backend(self.group) == "gloo"
        err = ""
        try:
            _, handle = self.ctx.exchange_buffer(256)
        except Exception as e:  # noqa: BLE001 - reported, decided collectively
            handle, err = bytes(64), str(e)
        mine = torch.frombuffer(bytearray(handle), dtype=torch.int64)
        allh = torch.empty(world * 8, dtype=torch.int64, device="cpu" if gloo else dev)
        dist.all_gather_into_tensor(allh, mine if gloo else mine.to(dev), group=self.group)
        allh = allh.cpu().view(world, 8)
        if not err:
            for r in range(world):
                if r != self.rank:
                    try:
                        self.ctx.open_peer(allh[r].numpy().tobytes())
                    except Exception as e:  # noqa: BLE001
                        err = str(e)
                        break
        ok = torch.tensor([0 if err else 1], dtype=torch.int32, device="cpu" if gloo else dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=self.group)
        return bool(ok.item()), err

    def _sort_p2p(self, keys: torch.Tensor, vals: torch.Tensor | None):
        rank, world = self.rank, self.world
        ctx = self.ctx
        gloo = dist.get_backend(self.group) == "gloo"  # functional tests: host collectives
        ev = _Events(self._timing)
        ev.mark("start")
        n, kb = keys.numel(), keys.element_size()
        voff = (n * kb + 255) // 256 * 256
        base, handle = ctx.exchange_buffer(max(voff + (4 * n if vals is not None else 0), 256))
        skeys = ctx.view(base, n, keys.dtype)
        svals = ctx.view(base + voff, n, vals.dtype) if vals is not None else None
        self.ops.sort_into(keys, vals, skeys, svals)
        ev.mark("local_sort")

        samples = self.ops.sample(skeys, rank, self.samples)
        gathered = torch.empty((world * self.samples, 2), dtype=samples.dtype,
                               device=samples.device)
        if gloo:
            g = gathered.cpu()
            dist.all_gather_into_tensor(_wire(g), _wire(samples.cpu()), group=self.group)
            gathered.copy_(g)
        else:
            dist.all_gather_into_tensor(_wire(gathered), _wire(samples.contiguous()),
                                        group=self.group)
        splitters = self.ops.select(gathered, world)
        bounds = self.ops.bounds(skeys, rank, splitters, world)
        ev.mark("splitters")

        # every rank's bounds, buffer handle and payload offset: world x (G+1+8+1),
        # gathered on the device; the host reads the result once per step (the
        # merge takes host pointers and lengths). The handle part is uploaded
        # only when this rank's buffer or payload offset changed.
        hkey = (handle, voff)
        if self._hinfo is None or self._hinfo[0] != hkey:
            hdl = torch.frombuffer(bytearray(handle), dtype=torch.int64)
            self._hinfo = (hkey, torch.cat([hdl, torch.tensor([voff])]).to(keys.device))
        if gloo:
            info = torch.cat([bounds.to(torch.int64).cpu(), self._hinfo[1].cpu()])
            allinfo = torch.empty(world * info.numel(), dtype=torch.int64)
            dist.all_gather_into_tensor(allinfo, info, group=self.group)
        else:
            info = torch.cat([bounds.to(torch.int64), self._hinfo[1]])
            allinfo = torch.empty(world * info.numel(), dtype=torch.int64, device=keys.device)
            dist.all_gather_into_tensor(allinfo, info, group=self.group)
            allinfo = allinfo.cpu()
        allinfo = allinfo.view(world, -1)
        rows = allinfo.tolist()
        ptrs, vptrs, lens = [], [], []
        for r, row in enumerate(rows):
            lo, hi = row[rank], row[rank + 1]
            h = allinfo[r, world + 1:world + 9].numpy().tobytes()
            peer = base if r == rank else ctx.open_peer(h)
            ptrs.append(peer + lo * kb)
            vptrs.append(peer + row[world + 9] + lo * 4)
            lens.append(hi - lo)
        total = sum(lens)
        ev.mark("exchange")

        out_k = torch.empty(total, dtype=keys.dtype, device=keys.device)
        out_v = torch.empty(total, dtype=vals.dtype, device=keys.device) if vals is not None else None
        if total:
            ctx.merge_ptrs(keys.dtype, ptrs, lens, out_k,
                           vptrs if vals is not None else None, out_v)
        ev.mark("merge")
        # release: nobody re-sorts into its buffer before every peer has read it
        if gloo:
            torch.cuda.synchronize(keys.device)
            dist.barrier(group=self.group)
        else:
            flag = torch.zeros(1, dtype=torch.int32, device=keys.device)
            dist.all_reduce(flag, group=self.group)
        self.last_bucket_sizes = lens
        ev.finish(self)
        return out_k, out_v

    def verify(self, out_keys: torch.Tensor, in_keys: torch.Tensor | None = None) -> bool:
        """Global check of bench::verify_output's gate (P/src/bench.cpp:95-104):
        every bucket sorted, bucket boundaries ordered across ranks, and (when
        the input shard is given) the multiset of all outputs equals that of
        all inputs."""
        world = self.world
        inv, _, ms_out = self.ops.check(out_keys)
        n = out_keys.numel()
        first = out_keys[:1] if n else out_keys.new_zeros(1)
        last = out_keys[-1:] if n else out_keys.new_zeros(1)
        info = torch.tensor([inv, n, _u2i(ms_out), _u2i(self.ops.check(in_keys)[2]) if
                             in_keys is not None else 0], dtype=torch.int64)
        edge = torch.cat([_wire(first).to(torch.int64), _wire(last).to(torch.int64)])
        dev = out_keys.device
        allinfo = [torch.empty_like(info, device=dev) for _ in range(world)]
        alledge = [torch.empty_like(edge, device=dev) for _ in range(world)]
        dist.all_gather(allinfo, info.to(dev), group=self.group)
        dist.all_gather(alledge, edge.to(dev), group=self.group)
        allinfo = [t.cpu().tolist() for t in allinfo]
        alledge = [t.cpu().tolist() for t in alledge]
        if any(i[0] != 0 for i in allinfo):
            return False
        signed = out_keys.dtype in (torch.int32, torch.int64)
        prev = None
        for (inv_r, n_r, _, _), (f, l) in zip(allinfo, alledge):
            if n_r == 0:
                continue
            f, l = _ordered(f, out_keys.dtype, signed), _ordered(l, out_keys.dtype, signed)
            if prev is not None and prev > f:
                return False
            prev = l
        if in_keys is not None:
            m = (1 << 64) - 1
            if sum(i[2] & m for i in allinfo) & m != sum(i[3] & m for i in allinfo) & m:
                return False
        return True


def _u2i(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def _ordered(v: int, dtype, signed: bool) -> int:
    bits = 32 if dtype in (torch.int32, torch.uint32) else 64
    v &= (1 << bits) - 1
    if signed and v >= 1 << (bits - 1):
        v -= 1 << bits
    return v


class _Events:
    """CUDA-event phase timer on torch's current stream (no-op on CPU)."""

    def __init__(self, on: bool):
        self.on = on and torch.cuda.is_available()
        self.ev = []

    def mark(self, name):
        if self.on:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev.append((name, e))

    def finish(self, sorter):
        if not self.on or len(self.ev) < 2:
            return
        self.ev[-1][1].synchronize()
        sorter.last_phase_ms = {self.ev[i][0]: self.ev[i - 1][1].elapsed_time(self.ev[i][1])
                                for i in range(1, len(self.ev))}
