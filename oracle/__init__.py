"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 partitioned sort.

Two checkers live here, both used only by tests/, ``__graft_entry__.smoke()``
and bench.py's CPU-baseline legs (never by the product path):

* ``port``: ``oracle/oracle.c`` -- a plain-C restatement of the reference's
  path (gen_data, plan_partition, merge_sort, merge_runs, merge_split_padded,
  scatter_merge_sort; see the file:line citations in that file).
* ``ref``: ``oracle/_ref/libsortbench_ref.so`` -- the unmodified reference
  library compiled from /root/reference/proj/src by ``oracle/build_ref.sh``,
  behind ``oracle/ref_driver.cpp``'s C ABI.

The port is pinned against the reference through the golden fixtures in
``tests/golden`` (written by ``tests/golden/make_golden.py`` from ``ref``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_p = ctypes.c_void_p

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def build() -> None:
    """Compile liboracle.so (and the reference library when its sources exist)."""
    subprocess.run(["bash", os.path.join(HERE, "build_ref.sh")], check=True)


def _load(name: str):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        build()
    return ctypes.CDLL(path)


_port = None
_ref = None


def port():
    global _port
    if _port is None:
        lib = _load("liboracle.so")
        lib.orc_gen_data.argtypes = [_u64, _u64, _u64, _p]
        lib.orc_plan_partition.argtypes = [_u64, ctypes.c_int, _p]
        lib.orc_plan_partition.restype = ctypes.c_int
        lib.orc_build_schedule.argtypes = [ctypes.c_int, _p]
        lib.orc_scatter_merge_sort.argtypes = [_p, _u64, ctypes.c_int, _p]
        lib.orc_scatter_merge_sort.restype = ctypes.c_int
        for t in ("i64", "u64", "i32", "u32"):
            getattr(lib, f"orc_sort_{t}").argtypes = [_p, _u64]
            getattr(lib, f"orc_sort_{t}").restype = ctypes.c_int
            getattr(lib, f"orc_stable_sort_kv_{t}").argtypes = [_p, _p, _u64]
            getattr(lib, f"orc_stable_sort_kv_{t}").restype = ctypes.c_int
            getattr(lib, f"orc_merge_runs_{t}").argtypes = [_p, _u64, _p, _u64, _p]
            getattr(lib, f"orc_merge_sort_{t}").argtypes = [_p, _i64, _i64, _p]
        lib.orc_merge_split.argtypes = [_p, _u64, _p, _u64, ctypes.c_int, _p]
        lib.orc_merge_split_padded.argtypes = [_p, _u64, _u64, _p, _u64, _u64,
                                               ctypes.c_int, _p, _p, _p]
        lib.orc_is_sorted_i64.argtypes = [_p, _u64]
        lib.orc_is_sorted_i64.restype = ctypes.c_int
        lib.orc_fingerprint_u64.argtypes = [_p, _u64]
        lib.orc_fingerprint_u64.restype = _u64
        _port = lib
    return _port


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libsortbench_ref.so"))


def ref():
    """The reference library itself (compiled from /root/reference)."""
    global _ref
    if _ref is None:
        lib = _load("libsortbench_ref.so")
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_gen_data.argtypes = [_u64, _u64, _p]
        lib.ref_plan_partition.argtypes = [_u64, ctypes.c_int, _p]
        lib.ref_plan_partition.restype = ctypes.c_int
        lib.ref_scatter_merge_sort.argtypes = [ctypes.c_int, _p, _u64, ctypes.c_int,
                                               ctypes.c_int, ctypes.c_int, _p, _p]
        lib.ref_scatter_merge_sort.restype = ctypes.c_int
        lib.ref_kernel_sort.argtypes = [ctypes.c_int, _p, _u64]
        lib.ref_kernel_sort.restype = ctypes.c_int
        lib.ref_merge_sort_range.argtypes = [_p, _u64, _i64, _i64]
        lib.ref_merge_sort_range.restype = ctypes.c_int
        lib.ref_quick_sort_range.argtypes = [_p, _u64, _u64, _u64]
        lib.ref_quick_sort_range.restype = ctypes.c_int
        lib.ref_merge_runs.argtypes = [_p, _u64, _p, _u64, _p]
        lib.ref_merge_split_padded.argtypes = [_p, _u64, _u64, _p, _u64, _u64,
                                               ctypes.c_int, _p, _p, _p]
        for f in ("ref_acceptance1_cases", "ref_random_oracle_cases"):
            getattr(lib, f).argtypes = [ctypes.c_int, _p, _p, _p, _p]
        lib.ref_kernel_oracle_cases.argtypes = [ctypes.c_int, _p, _p]
        lib.ref_std_sort.argtypes = [_p, _u64]
        lib.ref_run_id.argtypes = [ctypes.c_int, _u64, ctypes.c_int, ctypes.c_int, _u64,
                                   ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
        lib.ref_run_benchmark.argtypes = [ctypes.c_int, _u64, ctypes.c_int, ctypes.c_int, _u64,
                                          ctypes.c_int, ctypes.c_int] + [ctypes.c_char_p, _u64, _p] * 3
        lib.ref_run_benchmark.restype = ctypes.c_int
        lib.ref_to_chars_general.argtypes = [ctypes.c_double, ctypes.c_char_p]
        _ref = lib
    return _ref


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ---------------------------------------------------------------------------
# numpy restatements (vectorised; same streams as oracle.c)

def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def gen_data(n: int, seed: int, first: int = 0) -> np.ndarray:
    """bench::gen_data (P/src/bench.cpp:57-71) as int64: mix(seed + (i+1)*gamma)."""
    out = np.empty(n, dtype=np.int64)
    port().orc_gen_data(first, n, seed, _ptr(out))
    return out


def gen_data_np(n: int, seed: int, first: int = 0) -> np.ndarray:
    """Vectorised numpy form of gen_data (uint64 words)."""
    i = np.arange(first + 1, first + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(np.uint64(seed) + i * GAMMA)


def fingerprint(x: np.ndarray) -> int:
    """Order-sensitive fingerprint sum_i mix(x_i ^ mix(i+1)) mod 2^64 over the
    64-bit sign-preserving widening of x (matches orc_fingerprint_u64)."""
    if x.dtype in (np.int32, np.int64):
        w = x.astype(np.int64).view(np.uint64)
    else:
        w = x.astype(np.uint64)
    idx = np.arange(1, w.size + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return int(np.sum(_mix(w ^ _mix(idx)), dtype=np.uint64))


def fingerprint_chunked(x: np.ndarray, first: int = 0, chunk: int = 1 << 25) -> int:
    """fingerprint() of x computed in chunks (2^31-key outputs), x occupying
    positions first.. of the sequence."""
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for a in range(0, x.size, chunk):
            part = x[a: a + chunk]
            if part.dtype in (np.int32, np.int64):
                w = part.astype(np.int64).view(np.uint64)
            else:
                w = part.astype(np.uint64)
            idx = np.arange(first + a + 1, first + a + 1 + w.size, dtype=np.uint64)
            total = total + np.sum(_mix(w ^ _mix(idx)), dtype=np.uint64)
    return int(total)


def multiset_hash(x: np.ndarray, chunk: int = 1 << 25) -> int:
    """Order-independent sum_i mix(w_i) (b2s_check_sorted's multiset hash)."""
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for a in range(0, x.size, chunk):
            part = x[a: a + chunk]
            w = part.astype(np.int64).view(np.uint64) if part.dtype in (np.int32, np.int64) \
                else part.astype(np.uint64)
            total = total + np.sum(_mix(w), dtype=np.uint64)
    return int(total)


def gen_keys(n: int, seed: int, dtype, shift: int = 0, chunk: int = 1 << 25) -> np.ndarray:
    """(T)(z_i >> shift) over gen_data's stream (P/src/bench.cpp:57-71), the
    BASELINE configs' inputs (cfg2: u32 >> 32, cfg3: i32 >> 33, cfg5: u64),
    generated in chunks."""
    out = np.empty(n, dtype=dtype)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        z = gen_data_np(m, seed, first=a) >> np.uint64(shift)
        out[a: a + m] = z.astype(dtype) if np.dtype(dtype).itemsize == 4 else z.view(dtype)
    return out


def zipf_thresholds(values: int = 1 << 20, s: float = 1.2) -> np.ndarray:
    """Integer inverse-CDF table of Zipf(s) over `values` ranks (SURVEY.md
    8(d), cfg4a): T[r] = floor(CDF(r) * 2^53) with the weights (r+1)^-s summed
    in rank order in float64; T[-1] = 2^53. Rank r is drawn for
    u = z >> 11 (53 bits) when T[r-1] <= u < T[r], so the draw itself is
    integer arithmetic and bit-identical wherever the table is the same."""
    w = np.power(np.arange(1, values + 1, dtype=np.float64), -s)
    cdf = np.cumsum(w)
    t = np.floor(cdf / cdf[-1] * float(1 << 53)).astype(np.uint64)
    t[-1] = np.uint64(1 << 53)
    return t


def zipf_keys(n: int, seed: int, thresholds: np.ndarray, dtype=np.int32,
              chunk: int = 1 << 25) -> np.ndarray:
    """key_i = min r with (z_i >> 11) < T[r] (the rank is the key)."""
    out = np.empty(n, dtype=dtype)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        u = gen_data_np(m, seed, first=a) >> np.uint64(11)
        out[a: a + m] = np.searchsorted(thresholds, u, side="right").astype(dtype)
    return out


# ---------------------------------------------------------------------------
# port (C restatement) wrappers

_SUFFIX = {np.dtype(np.int64): "i64", np.dtype(np.uint64): "u64",
           np.dtype(np.int32): "i32", np.dtype(np.uint32): "u32"}


def plan_partition(n: int, p: int) -> list[int]:
    sizes = np.zeros(max(p, 1), dtype=np.uint64)
    if port().orc_plan_partition(n, p, _ptr(sizes)) != 0:
        raise ValueError("partition needs at least one process")
    return [int(s) for s in sizes]


def sort(keys: np.ndarray) -> np.ndarray:
    """Merge-sort restatement (ascending, stable) of any supported key width."""
    out = np.ascontiguousarray(keys).copy()
    if getattr(port(), f"orc_sort_{_SUFFIX[out.dtype]}")(_ptr(out), out.size) != 0:
        raise MemoryError("oracle sort allocation failed")
    return out


def stable_sort_kv(keys: np.ndarray, vals: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    k = np.ascontiguousarray(keys).copy()
    v = np.ascontiguousarray(vals, dtype=np.uint32).copy()
    fn = getattr(port(), f"orc_stable_sort_kv_{_SUFFIX[k.dtype]}")
    if fn(_ptr(k), _ptr(v), k.size) != 0:
        raise MemoryError("oracle kv sort allocation failed")
    return k, v


def merge_runs(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, dtype=a.dtype)
    out = np.empty(a.size + b.size, dtype=a.dtype)
    getattr(port(), f"orc_merge_runs_{_SUFFIX[a.dtype]}")(_ptr(a), a.size, _ptr(b), b.size,
                                                         _ptr(out))
    return out


def merge_kway(runs: list[np.ndarray]) -> np.ndarray:
    """Stable k-way merge, ties to the lower run index: left fold of merge_runs."""
    if not runs:
        return np.empty(0, dtype=np.int64)
    acc = np.ascontiguousarray(runs[0])
    for r in runs[1:]:
        acc = merge_runs(acc, r)
    return acc


def merge_split(mine: np.ndarray, theirs: np.ndarray, keep_high: bool) -> np.ndarray:
    mine = np.ascontiguousarray(mine, dtype=np.int64)
    theirs = np.ascontiguousarray(theirs, dtype=np.int64)
    out = np.empty(mine.size, dtype=np.int64)
    port().orc_merge_split(_ptr(mine), mine.size, _ptr(theirs), theirs.size,
                           int(keep_high), _ptr(out))
    return out


def merge_split_padded(mine, mine_virt, theirs, theirs_virt, keep_high):
    mine = np.ascontiguousarray(mine, dtype=np.int64)
    theirs = np.ascontiguousarray(theirs, dtype=np.int64)
    width = mine.size + mine_virt
    out = np.empty(max(width, 1), dtype=np.int64)
    nr = ctypes.c_uint64()
    nv = ctypes.c_uint64()
    port().orc_merge_split_padded(_ptr(mine), mine.size, mine_virt, _ptr(theirs),
                                  theirs.size, theirs_virt, int(keep_high), _ptr(out),
                                  ctypes.addressof(nr), ctypes.addressof(nv))
    return out[: nr.value].copy(), nv.value


def scatter_merge_sort(data: np.ndarray, p: int) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.int64)
    out = np.empty(data.size, dtype=np.int64)
    rc = port().orc_scatter_merge_sort(_ptr(data), data.size, p, _ptr(out))
    if rc == -1:
        raise ValueError("partition needs at least one process")
    if rc != 0:
        raise MemoryError("oracle allocation failed")
    return out


# ---------------------------------------------------------------------------
# reference-library wrappers (oracle/_ref)

ALGOS = {"bubble": 0, "merge": 1, "quick": 2}


def ref_scatter_merge_sort(data: np.ndarray, p: int, algo: str = "merge", cores: int = 1,
                           wall: bool = False) -> tuple[np.ndarray, float]:
    data = np.ascontiguousarray(data, dtype=np.int64)
    out = np.empty(data.size, dtype=np.int64)
    secs = ctypes.c_double(0.0)
    rc = ref().ref_scatter_merge_sort(ALGOS[algo], _ptr(data), data.size, p, cores,
                                      int(wall), _ptr(out), ctypes.addressof(secs))
    if rc != 0:
        raise RuntimeError(f"reference failed ({rc}): {ref().ref_last_error().decode()}")
    return out, secs.value


def ref_gen_data(n: int, seed: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    ref().ref_gen_data(n, seed, _ptr(out))
    return out


def ref_run_id(algo: str, n: int, procs: int, cores: int, seed: int, mode: str = "wall",
               reps: int = 1) -> str:
    """bench::run_id of the reference (P/src/bench.cpp:30-50)."""
    out = ctypes.create_string_buffer(17)
    ref().ref_run_id(ALGOS[algo], n, procs, cores, seed, int(mode == "wall"), reps, out)
    return out.value.decode()


def ref_run_benchmark(algo: str, n: int, procs: int, cores: int, seed: int = 1,
                      mode: str = "wall", reps: int = 1) -> tuple[str, str, str]:
    """bench::run_benchmark of the reference plus its exports: (experiment-1
    CSV row, trace JSONL, trace summary JSON)."""
    caps = [4096, 64 << 20, 1 << 20]
    bufs = [ctypes.create_string_buffer(c) for c in caps]
    lens = [ctypes.c_uint64() for _ in caps]
    args = []
    for b, c, ln in zip(bufs, caps, lens):
        args += [b, c, ctypes.addressof(ln)]
    rc = ref().ref_run_benchmark(ALGOS[algo], n, procs, cores, seed, int(mode == "wall"), reps,
                                 *args)
    if rc != 0:
        raise RuntimeError(f"reference failed: {ref().ref_last_error().decode()}")
    return tuple(b.value.decode() for b in bufs)


def ref_to_chars_general(v: float) -> str:
    """std::to_chars(general) -- the reference's format_double for finite values."""
    out = ctypes.create_string_buffer(64)
    ref().ref_to_chars_general(v, out)
    return out.value.decode()
