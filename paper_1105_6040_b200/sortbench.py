"""The reference's sort entry points, re-implemented on the B200 C ABI.

Same names, argument meaning and error behaviour as sortbench's
``kernels`` / ``parallel`` / ``bench`` functions on the hot path
(P/include/sortbench/sort_core.hpp, parallel_sort.hpp, bench.hpp), so code
and tests written against the reference read the same here. Arrays are int64
(``Element``, P/include/sortbench/element.hpp:10) numpy arrays -- the
reference's host ``std::vector<int64_t>`` -- or CUDA tensors of any supported
key width. Every sort/merge runs as CUDA kernels through libb200sort.so; there
is no CPU path. The C++ shims with the exact reference signatures live in
include/sortbench_b200/ (see INTEGRATION.md).
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import default_context
from .errors import ConfigError, ProgrammingError, VerificationError

Element = np.int64


class Algorithm(enum.Enum):
    """parallel::Algorithm (P/include/sortbench/parallel_sort.hpp:14). On the
    GPU all three select the same radix sort: the output of any correct sort
    of integers is identical."""
    bubble = 0
    merge = 1
    quick = 2


def to_string(algorithm: Algorithm) -> str:
    return algorithm.name


def algorithm_from_string(name: str) -> Algorithm:
    """P/src/parallel_sort.cpp:18-24."""
    try:
        return Algorithm[name]
    except KeyError:
        raise ConfigError(f"unknown algorithm '{name}' (expected bubble, merge or quick)") from None


class KeepHalf(enum.Enum):
    low = 0
    high = 1


@dataclass
class PartitionPlan:
    n: int = 0
    procs: int = 1
    sizes: list = field(default_factory=list)


def plan_partition(n: int, p: int) -> PartitionPlan:
    """P/src/parallel_sort.cpp:26-38, via b2s_plan_partition."""
    if p < 1:
        raise ConfigError("partition needs at least one process")
    sizes = (ctypes.c_uint64 * p)()
    _lib.check(_lib.lib().b2s_plan_partition(n, p, sizes))
    return PartitionPlan(n=n, procs=p, sizes=[int(s) for s in sizes])


@dataclass
class PhaseSchedule:
    procs: int = 1
    partners: list = field(default_factory=list)  # [phase][rank]

    def phases(self) -> int:
        return len(self.partners)

    def partner(self, phase: int, rank: int) -> int:
        return self.partners[phase][rank]


def build_schedule(p: int) -> PhaseSchedule:
    """The p-phase odd-even pairing, P/src/parallel_sort.cpp:40-55."""
    if p < 1:
        raise ConfigError("schedule needs at least one process")
    rows = []
    for phase in range(p):
        row = [-1] * p
        for r in range(0 if phase % 2 == 0 else 1, p - 1, 2):
            row[r], row[r + 1] = r + 1, r
        rows.append(row)
    return PhaseSchedule(procs=p, partners=rows)


def _as_host_int64(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.int64))


def _sort_inplace(block, lo: int, hi: int) -> None:
    """Sorts block[lo:hi] in place on the GPU."""
    if hi - lo < 2:
        return
    view = block[lo:hi]
    if isinstance(block, np.ndarray) and not view.flags.c_contiguous:
        raise ValueError("block must be contiguous")
    default_context(_device_of(block)).sort(view, out=view)


def _device_of(x) -> int:
    if isinstance(x, np.ndarray):
        return 0
    return x.device.index or 0


# -- kernels:: (P/include/sortbench/sort_core.hpp) ---------------------------

def bubble_sort(block) -> None:
    """kernels::bubble_sort (P/src/sort_core.cpp:23-36): sorts the block in place."""
    _sort_inplace(block, 0, len(block))


def merge_sort(block, first: int, last: int, scratch=None) -> None:
    """kernels::merge_sort over the inclusive range [first, last]
    (P/src/sort_core.cpp:98-106); first >= last is a no-op. `scratch` is the
    reference's host buffer and is unused by the GPU path."""
    if first >= last:
        return
    if first < 0 or last >= len(block):
        raise ProgrammingError(f"merge_sort range [{first}, {last}] out of range "
                               f"size={len(block)}")
    _sort_inplace(block, first, last + 1)


def quick_sort(block, start: int, length: int) -> None:
    """kernels::quick_sort on [start, start+length) (P/src/sort_core.cpp:135-144);
    an out-of-range segment raises ProgrammingError as the reference does.
    The reference takes size_t, so a negative start or length (which Python
    slicing would wrap around) is out of range too."""
    if start < 0 or length < 0 or start + length > len(block):
        raise ProgrammingError(f"quick_sort segment out of range: start={start} "
                               f"length={length} size={len(block)}")
    _sort_inplace(block, start, start + length)


def merge_runs(run_a, run_b):
    """kernels::merge_runs (P/src/sort_core.cpp:38-62): a fresh merged run,
    ties taken from run_a first."""
    if isinstance(run_a, np.ndarray) or isinstance(run_b, np.ndarray) or isinstance(run_a, list):
        a, b = _as_host_int64(run_a), _as_host_int64(run_b)
    else:
        a, b = run_a, run_b
    if len(a) + len(b) == 0:
        return a[:0].copy()
    out, _ = default_context(_device_of(a)).merge([a, b])
    return out


def is_sorted(seq) -> bool:
    """kernels::is_sorted (P/src/sort_core.cpp:146-151), checked on the GPU."""
    n = len(seq)
    if n < 2:
        return True
    x = seq
    if isinstance(seq, (list, tuple)):
        x = _as_host_int64(seq)
    if isinstance(x, np.ndarray):
        import torch
        x = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    inv, _, _ = default_context(_device_of(x)).check_sorted(x)
    return inv == 0


# -- parallel:: (P/include/sortbench/parallel_sort.hpp) ----------------------

@dataclass
class PaddedBlock:
    """A phase block padded with `virtuals` top sentinels
    (P/include/sortbench/parallel_sort.hpp:56-65)."""
    reals: np.ndarray = field(default_factory=lambda: np.empty(0, dtype=np.int64))
    virtuals: int = 0

    def width(self) -> int:
        return len(self.reals) + self.virtuals


def merge_split(mine, theirs, keep: KeepHalf):
    """parallel::merge_split (P/src/parallel_sort.cpp:107-113): the lowest or
    highest |mine| elements of mine U theirs."""
    return merge_split_padded(PaddedBlock(_as_host_int64(mine), 0),
                              PaddedBlock(_as_host_int64(theirs), 0), keep).reals


def merge_split_padded(mine: PaddedBlock, theirs: PaddedBlock, keep: KeepHalf) -> PaddedBlock:
    """parallel::merge_split_padded (P/src/parallel_sort.cpp:115-134) on the
    GPU. As in the reference the kept width is mine.width()."""
    m = _as_host_int64(mine.reals)
    t = _as_host_int64(theirs.reals)
    reals, virt = default_context(0).merge_split_padded(m, mine.virtuals, t, theirs.virtuals,
                                                        keep == KeepHalf.high)
    return PaddedBlock(np.asarray(reals, dtype=np.int64).copy(), int(virt))


def select_kernel(algorithm: Algorithm):
    """parallel::select_kernel (P/src/parallel_sort.cpp:157-164): a callable
    with KernelFn's (block, scratch) shape that sorts the block in place."""
    if not isinstance(algorithm, Algorithm):
        raise ConfigError("unknown algorithm id")

    def kernel(block, scratch=None):
        _sort_inplace(block, 0, len(block))

    kernel.__name__ = f"{algorithm.name}_kernel_b200"
    return kernel


@dataclass
class WorldOptions:
    """runtime::WorldOptions (P/include/sortbench/runtime.hpp:60-66). On one
    GPU `procs` is the partition count; core_slots/mode/weights emulate CPU
    cores and message costs of the paper's MPI runs and do not apply."""
    procs: int = 1
    core_slots: int = 1
    mode: str = "counted"
    latency_weight: int = 1000
    bandwidth_weight: int = 1


@dataclass
class SortOutcome:
    sorted: object = None
    procs: int = 1
    device_ms: float = 0.0


def scatter_merge_sort(algorithm: Algorithm, data, options: WorldOptions) -> SortOutcome:
    """parallel::scatter_merge_sort (P/src/parallel_sort.cpp:166-254) on one
    GPU: plan_partition scatter, a local radix sort per partition, and a
    merge-path merge of the p sorted runs (b2s_partitioned_sort)."""
    p = options.procs
    if p < 1:
        raise ConfigError("partition needs at least one process")
    select_kernel(algorithm)  # validates the algorithm like the reference
    host = not hasattr(data, "is_cuda")
    x = _as_host_int64(data) if host else data
    if len(x) == 0:
        return SortOutcome(sorted=x.copy() if host else x.clone(), procs=p)
    out, _ = default_context(_device_of(x)).partitioned_sort(x, p)
    return SortOutcome(sorted=out, procs=p)


# -- bench:: (P/include/sortbench/bench.hpp) -----------------------------------

def gen_data(n: int, seed: int, device: bool = False):
    """bench::gen_data (P/src/bench.cpp:57-71), generated on the GPU
    (b2s_gen_keys, bit-identical). Returns int64 numpy unless device=True."""
    import torch
    ctx = default_context(0)
    t = ctx.gen_keys(n, seed, torch.int64, shift=0)
    if device:
        return t
    torch.cuda.synchronize()
    return t.cpu().numpy()


def verify_output(input_data, output) -> None:
    """bench::verify_output (P/src/bench.cpp:95-104): raises VerificationError
    unless output is sorted and a permutation of input. The checks run on the
    GPU: inversion count + multiset hash (b2s_check_sorted), then exact
    equality with an independent sort of the input (torch.sort, CUB's), the
    reference's std::sort(copy(input)) comparison."""
    import torch

    def dev(x):
        return torch.from_numpy(_as_host_int64(x)).cuda() if not hasattr(x, "is_cuda") else x

    a, b = dev(input_data), dev(output)
    if a.numel() != b.numel():
        raise VerificationError("run produced output that is not the sorted input")
    ctx = default_context(_device_of(a))
    inv, _, ms_out = ctx.check_sorted(b)
    _, _, ms_in = ctx.check_sorted(a)
    if inv != 0 or ms_in != ms_out:
        raise VerificationError("run produced output that is not the sorted input")
    if not torch.equal(_independent_sort(a), b):
        raise VerificationError("run produced output that is not the sorted input")


def _independent_sort(a):
    """The ascending order of a device tensor by torch.sort (not this
    library): unsigned keys are sorted through an order-preserving signed view."""
    import torch
    if a.dtype in (torch.uint32, torch.uint64):
        signed = torch.int32 if a.dtype == torch.uint32 else torch.int64
        flip = torch.tensor(-(1 << (8 * a.element_size() - 1)), dtype=signed, device=a.device)
        s = torch.sort(a.view(signed) ^ flip)[0] ^ flip
        return s.view(a.dtype)
    return torch.sort(a)[0]
