"""Python handle on the C ABI: a per-device context that sorts torch CUDA
tensors (device pointers, asynchronous on torch's current stream) or numpy
arrays (host pointers, B2S_HOST: copies inside the call, synchronous).

PyTorch is plumbing here (device memory, streams); every compute step is a
kernel in libb200sort.so.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import B2S_DEVICE, B2S_HOST, check, lib

try:  # torch is optional for host-only use
    import torch
except ImportError:  # pragma: no cover
    torch = None

_NP_DTYPES = {np.dtype(np.int32): _lib.B2S_I32, np.dtype(np.uint32): _lib.B2S_U32,
              np.dtype(np.int64): _lib.B2S_I64, np.dtype(np.uint64): _lib.B2S_U64}


def _torch_dtypes():
    return {torch.int32: _lib.B2S_I32, torch.uint32: _lib.B2S_U32,
            torch.int64: _lib.B2S_I64, torch.uint64: _lib.B2S_U64}


def dtype_code(x) -> int:
    if isinstance(x, np.ndarray):
        try:
            return _NP_DTYPES[x.dtype]
        except KeyError:
            raise TypeError(f"unsupported key dtype {x.dtype}") from None
    try:
        return _torch_dtypes()[x.dtype]
    except KeyError:
        raise TypeError(f"unsupported key dtype {x.dtype}") from None


def _is_host(x) -> bool:
    return isinstance(x, np.ndarray)


def _ptr(x) -> int | None:
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data if x.size else None
    return x.data_ptr() if x.numel() else None


def _check_1d(x, name):
    if isinstance(x, np.ndarray):
        if x.ndim != 1 or not x.flags.c_contiguous:
            raise ValueError(f"{name} must be a contiguous 1-D array")
    elif x is not None:
        if x.dim() != 1 or not x.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 1-D tensor")
        if not x.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (or pass a numpy array)")


@dataclass
class Timing:
    hist_ms: float
    pass_ms: list
    passes_executed: int
    passes_possible: int
    copy_ms: float
    merge_ms: float
    merge_rounds: int
    total_ms: float


class Context:
    """One b2s_ctx: bound to one CUDA device, used by one thread at a time."""

    def __init__(self, device: int = 0):
        self.device = device
        h = ctypes.c_void_p()
        check(lib().b2s_create(device, ctypes.byref(h)))
        self._h = h

    # -- lifetime -----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().b2s_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self):
        return self._h

    def _bind_stream(self, stream=None) -> None:
        if stream is None and torch is not None and torch.cuda.is_available():
            stream = torch.cuda.current_stream(self.device)
        if stream is None:
            return  # keep the context's own stream (no torch / no CUDA torch)
        s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        check(lib().b2s_set_stream(self._h, s or None))

    def synchronize(self) -> None:
        check(lib().b2s_synchronize(self._h))

    @property
    def lane_ordered_atomics(self) -> bool:
        """True when keys are ranked by lane-ordered shared atomics (the probe
        at context creation passed), False on the ballot-matching fallback."""
        return lib().b2s_lane_ordered_atomics(self._h) == 1

    def enable_timing(self, on: bool = True) -> None:
        check(lib().b2s_enable_timing(self._h, int(on)))

    def timing(self) -> Timing:
        t = _lib.b2s_timing()
        check(lib().b2s_get_timing(self._h, ctypes.byref(t)))
        return Timing(t.hist_ms, list(t.pass_ms)[: t.passes_executed], t.passes_executed,
                      t.passes_possible, t.copy_ms, t.merge_ms, t.merge_rounds, t.total_ms)

    # -- local sort -----------------------------------------------------------
    def sort(self, keys, out=None, vals=None, vals_out=None, stream=None):
        """Sorts `keys` ascending (stable; `vals` is a uint32 payload permuted
        with the keys). Returns (out, vals_out); out may be `keys` (in place)."""
        _check_1d(keys, "keys")
        host = _is_host(keys)
        if out is None:
            out = np.empty_like(keys) if host else torch.empty_like(keys)
        if vals is not None and vals_out is None:
            vals_out = np.empty_like(vals) if host else torch.empty_like(vals)
        self._validate_pair(keys, out, vals, vals_out)
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_sort(self._h, dtype_code(keys), _ptr(keys), _ptr(out), _ptr(vals),
                             _ptr(vals_out), _numel(keys), B2S_HOST if host else B2S_DEVICE))
        return out, vals_out

    def sort_batch(self, keys_list, outs=None, vals_list=None, vals_outs=None):
        """Sorts a list of equally sized host (numpy) arrays with the uploads,
        sorts and downloads of consecutive arrays overlapped (b2s_sort_batch)."""
        if not keys_list:
            return [], None
        n = _numel(keys_list[0])
        code = dtype_code(keys_list[0])
        for x in keys_list:
            if not _is_host(x) or _numel(x) != n or dtype_code(x) != code:
                raise ValueError("sort_batch takes equally sized host arrays of one dtype")
        if outs is None:
            outs = [np.empty_like(x) for x in keys_list]
        if vals_list is not None and vals_outs is None:
            vals_outs = [np.empty_like(v) for v in vals_list]
        c = len(keys_list)
        ki = (ctypes.c_void_p * c)(*[_ptr(x) for x in keys_list])
        ko = (ctypes.c_void_p * c)(*[_ptr(x) for x in outs])
        vi = (ctypes.c_void_p * c)(*[_ptr(v) for v in vals_list]) if vals_list is not None else None
        vo = (ctypes.c_void_p * c)(*[_ptr(v) for v in vals_outs]) if vals_outs is not None else None
        check(lib().b2s_sort_batch(self._h, code, ki, ko, vi, vo, n, c, B2S_HOST))
        return outs, vals_outs

    def partitioned_sort(self, keys, p: int, out=None, vals=None, vals_out=None, stream=None):
        """scatter / local sort / merge on this device with p partitions."""
        _check_1d(keys, "keys")
        host = _is_host(keys)
        if out is None:
            out = np.empty_like(keys) if host else torch.empty_like(keys)
        if vals is not None and vals_out is None:
            vals_out = np.empty_like(vals) if host else torch.empty_like(vals)
        self._validate_pair(keys, out, vals, vals_out)
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_partitioned_sort(self._h, dtype_code(keys), _ptr(keys), _ptr(out),
                                         _ptr(vals), _ptr(vals_out), _numel(keys), int(p),
                                         B2S_HOST if host else B2S_DEVICE))
        return out, vals_out

    def odd_even_sort(self, keys, p: int, out=None, stream=None):
        """The reference's p-phase odd-even merge-split sort on this device
        (b2s_odd_even_sort), for comparison with partitioned_sort."""
        _check_1d(keys, "keys")
        host = _is_host(keys)
        if out is None:
            out = np.empty_like(keys) if host else torch.empty_like(keys)
        self._validate_pair(keys, out, None, None)
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_odd_even_sort(self._h, dtype_code(keys), _ptr(keys), _ptr(out), _numel(keys),
                                      int(p), B2S_HOST if host else B2S_DEVICE))
        return out

    def merge(self, runs, vals=None, out=None, vals_out=None, stream=None):
        """Stable k-way merge of sorted runs (ties to the lower run index)."""
        if len(runs) == 0:
            raise ValueError("merge needs at least one run")
        for r in runs:
            _check_1d(r, "run")
        host = _is_host(runs[0])
        total = sum(_numel(r) for r in runs)
        code = dtype_code(runs[0])
        for r in runs:
            if dtype_code(r) != code or _is_host(r) != host:
                raise TypeError("all runs must share dtype and memory space")
        if out is None:
            out = (np.empty(total, dtype=runs[0].dtype) if host
                   else torch.empty(total, dtype=runs[0].dtype, device=runs[0].device))
        if vals is not None and vals_out is None:
            vals_out = (np.empty(total, dtype=np.uint32) if host
                        else torch.empty(total, dtype=vals[0].dtype, device=vals[0].device))
        k = len(runs)
        rp = (ctypes.c_void_p * k)(*[_ptr(r) for r in runs])
        ln = (ctypes.c_uint64 * k)(*[_numel(r) for r in runs])
        vp = (ctypes.c_void_p * k)(*[_ptr(v) for v in vals]) if vals is not None else None
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_merge(self._h, code, rp, vp, ln, k, _ptr(out), _ptr(vals_out),
                              B2S_HOST if host else B2S_DEVICE))
        return out, vals_out

    def merge_split_padded(self, mine, mine_virtuals: int, theirs, theirs_virtuals: int,
                           keep_high: bool, stream=None):
        """The reference's padded merge-split on the device; returns (reals, virtuals)."""
        host = _is_host(mine)
        width = _numel(mine) + mine_virtuals
        out = (np.empty(max(width, 1), dtype=mine.dtype) if host
               else torch.empty(max(width, 1), dtype=mine.dtype, device=mine.device))
        nr, nv = ctypes.c_uint64(), ctypes.c_uint64()
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_merge_split_padded(
            self._h, dtype_code(mine), _ptr(mine), _numel(mine), mine_virtuals, _ptr(theirs),
            _numel(theirs), theirs_virtuals, int(keep_high), _ptr(out), ctypes.byref(nr),
            ctypes.byref(nv), B2S_HOST if host else B2S_DEVICE))
        return out[: nr.value], nv.value

    # -- multi-GPU pull exchange ------------------------------------------------
    def exchange_buffer(self, nbytes: int):
        """(device pointer, 64-byte IPC handle) of this context's exported
        buffer, grown to at least `nbytes`."""
        p = ctypes.c_void_p()
        h = ctypes.create_string_buffer(64)
        check(lib().b2s_exchange_buffer(self._h, nbytes, ctypes.byref(p), h))
        return p.value, h.raw

    def open_peer(self, handle: bytes) -> int:
        """Device pointer of a peer's exported buffer (mapped once per handle)."""
        if len(handle) != 64:
            raise ValueError("an IPC handle is 64 bytes")
        p = ctypes.c_void_p()
        check(lib().b2s_open_peer(self._h, ctypes.create_string_buffer(handle, 64), ctypes.byref(p)))
        return p.value

    def close_peers(self) -> None:
        check(lib().b2s_close_peers(self._h))

    def view(self, ptr: int, n: int, dtype):
        """A torch tensor over n elements of device memory at `ptr` (no copy;
        the memory belongs to this context)."""
        wire = {torch.uint32: torch.int32, torch.uint64: torch.int64}.get(dtype, dtype)
        code = {torch.int32: "<i4", torch.int64: "<i8"}[wire]
        holder = _CudaArray(ptr, n, code)
        t = torch.as_tensor(holder, device=f"cuda:{self.device}")
        return t.view(dtype) if wire is not dtype else t

    def merge_ptrs(self, dtype, ptrs, lens, out, vptrs=None, vals_out=None, stream=None):
        """k-way merge of device runs given as raw pointers (peer memory
        included) into the device tensor `out`."""
        k = len(ptrs)
        rp = (ctypes.c_void_p * k)(*[p if n else None for p, n in zip(ptrs, lens)])
        ln = (ctypes.c_uint64 * k)(*lens)
        vp = ((ctypes.c_void_p * k)(*[p if n else None for p, n in zip(vptrs, lens)])
              if vptrs is not None else None)
        self._bind_stream(stream)
        check(lib().b2s_merge(self._h, _torch_dtypes()[dtype], rp, vp, ln, k, _ptr(out),
                              _ptr(vals_out), B2S_DEVICE))
        return out, vals_out

    # -- sample sort steps (device tensors) -----------------------------------
    def sample_regular(self, sorted_keys, rank: int, samples: int, out=None, stream=None):
        """(samples, 2) uint64 tensor of (order key, rank<<40 | position) records."""
        if out is None:
            out = torch.empty((samples, 2), dtype=torch.uint64, device=sorted_keys.device)
        self._bind_stream(stream)
        check(lib().b2s_sample_regular(self._h, dtype_code(sorted_keys), _ptr(sorted_keys),
                                       _numel(sorted_keys), rank, samples, _ptr(out)))
        return out

    def select_splitters(self, samples, nparts: int, out=None, stream=None):
        count = samples.shape[0]
        if out is None:
            out = torch.empty((max(nparts - 1, 1), 2), dtype=torch.uint64, device=samples.device)
        self._bind_stream(stream)
        check(lib().b2s_select_splitters(self._h, _ptr(samples), count, nparts, _ptr(out)))
        return out

    def bucket_bounds(self, sorted_keys, rank: int, splitters, nparts: int, out=None,
                      stream=None):
        if out is None:
            out = torch.empty(nparts + 1, dtype=torch.int64, device=sorted_keys.device)
        self._bind_stream(stream)
        check(lib().b2s_bucket_bounds(self._h, dtype_code(sorted_keys), _ptr(sorted_keys),
                                      _numel(sorted_keys), rank, _ptr(splitters), nparts,
                                      _ptr(out)))
        return out

    # -- generation / verification -------------------------------------------
    def gen_keys(self, n: int, seed: int, dtype, shift: int = 0, first: int = 0, out=None,
                 stream=None):
        """bench::gen_data's stream on the device: key_i = (T)(z_{first+i} >> shift)."""
        if out is None:
            out = torch.empty(n, dtype=dtype, device=f"cuda:{self.device}")
        if _is_host(out):
            check(lib().b2s_gen_keys(self._h, dtype_code(out), first, n, seed, shift, _ptr(out),
                                     B2S_HOST))
            return out
        self._bind_stream(stream)
        check(lib().b2s_gen_keys(self._h, dtype_code(out), first, n, seed, shift, _ptr(out),
                                 B2S_DEVICE))
        return out

    def gen_zipf(self, n: int, seed: int, thresholds, dtype=None, first: int = 0, out=None,
                 stream=None):
        """cfg4a's Zipf keys on the device: key_i = #{r : thresholds[r] <= z_{first+i} >> 11}
        (thresholds: ascending uint64 numpy array, see workloads.zipf_thresholds)."""
        t = np.ascontiguousarray(thresholds, dtype=np.uint64)
        if out is None:
            out = torch.empty(n, dtype=dtype or torch.int32, device=f"cuda:{self.device}")
        host = _is_host(out)
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_gen_zipf(self._h, dtype_code(out), first, n, seed, t.ctypes.data,
                                 t.size, _ptr(out), B2S_HOST if host else B2S_DEVICE))
        return out

    def check_sorted(self, keys, stream=None):
        """(adjacent inversions, order-sensitive fingerprint, multiset hash)."""
        inv, fp, ms = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        host = _is_host(keys)
        if not host:
            self._bind_stream(stream)
        check(lib().b2s_check_sorted(self._h, dtype_code(keys), _ptr(keys), _numel(keys),
                                     ctypes.byref(inv), ctypes.byref(fp), ctypes.byref(ms),
                                     B2S_HOST if host else B2S_DEVICE))
        return inv.value, fp.value, ms.value

    # -- helpers ----------------------------------------------------------------
    @staticmethod
    def _validate_pair(keys, out, vals, vals_out):
        _check_1d(out, "out")
        if _numel(out) != _numel(keys) or dtype_code(out) != dtype_code(keys):
            raise ValueError("out must match keys in size and dtype")
        if _is_host(out) != _is_host(keys):
            raise ValueError("keys and out must live in the same memory space")
        if (vals is None) != (vals_out is None):
            raise ValueError("vals and vals_out go together")
        if vals is not None:
            _check_1d(vals, "vals")
            _check_1d(vals_out, "vals_out")
            if _numel(vals) != _numel(keys) or _numel(vals_out) != _numel(keys):
                raise ValueError("vals must match keys in size")
            for v in (vals, vals_out):
                if isinstance(v, np.ndarray):
                    ok = v.dtype in (np.uint32, np.int32)
                else:
                    ok = v.dtype in (torch.int32, torch.uint32)
                if not ok:
                    raise TypeError("the payload is 32-bit (uint32 / int32)")


class _CudaArray:
    """__cuda_array_interface__ of a raw device range, for torch.as_tensor."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def _numel(x) -> int:
    return int(x.size) if isinstance(x, np.ndarray) else int(x.numel())


_default = {}


def default_context(device: int = 0) -> Context:
    """A lazily created per-device context for the module-level helpers."""
    ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        _default[device] = ctx
    return ctx


@dataclass
class MultiTiming:
    local_sort_ms: float
    splitters_ms: float
    exchange_merge_ms: float
    total_ms: float
    transport: str
    max_bucket: int
    min_bucket: int


class MultiContext:
    """One b2s_multi: the sample sort over several GPUs in this process, one
    host thread per rank inside the library (b2s_sample_sort). `devices` may
    repeat a device (emulated ranks)."""

    TRANSPORTS = {"auto": _lib.B2S_XCHG_AUTO, "p2p": _lib.B2S_XCHG_P2P, "nccl": _lib.B2S_XCHG_NCCL}

    def __init__(self, devices):
        self.devices = [int(d) for d in devices]
        arr = (ctypes.c_int * len(self.devices))(*self.devices)
        h = ctypes.c_void_p()
        check(lib().b2s_create_multi(len(self.devices), arr, ctypes.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().b2s_destroy_multi(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def info(self) -> dict:
        r, p, n, v = (ctypes.c_int() for _ in range(4))
        check(lib().b2s_multi_info(self._h, ctypes.byref(r), ctypes.byref(p), ctypes.byref(n),
                                   ctypes.byref(v)))
        return {"ranks": r.value, "p2p": bool(p.value), "nccl": bool(n.value),
                "nccl_version": v.value}

    def set_transport(self, name: str) -> None:
        check(lib().b2s_multi_set_transport(self._h, self.TRANSPORTS[name]))

    def timing(self) -> MultiTiming:
        t = _lib.b2s_multi_timing()
        check(lib().b2s_multi_get_timing(self._h, ctypes.byref(t)))
        names = {_lib.B2S_XCHG_P2P: "p2p", _lib.B2S_XCHG_NCCL: "nccl"}
        return MultiTiming(t.local_sort_ms, t.splitters_ms, t.exchange_merge_ms, t.total_ms,
                           names.get(t.transport, "?"), t.max_bucket, t.min_bucket)

    def sample_sort(self, shards, vals=None, outs=None, out_vals=None, capacity=None,
                    samples_per_gpu: int = 64):
        """Sorts the shards (one per rank: CUDA tensors on that rank's device,
        or numpy arrays) into buckets. Returns (buckets, bucket_vals): bucket
        r holds the r-th slice of the global ascending order; with a payload
        the order is stable by global index (shard order)."""
        G = len(self.devices)
        if len(shards) != G:
            raise ValueError(f"need {G} shards")
        host = _is_host(shards[0])
        code = dtype_code(shards[0])
        for x in shards:
            _check_1d(x, "shard")
            if _is_host(x) != host or dtype_code(x) != code:
                raise ValueError("shards must share dtype and memory kind")
        outs_given = outs
        counts = [_numel(x) for x in shards]
        total = sum(counts)
        if capacity is None:
            # regular sampling bounds a bucket by ~2 N / G; the slack covers
            # the sample granularity
            capacity = [min(total, 2 * (total // G) + 2 * samples_per_gpu * G + 1024)] * G
        if outs is None:
            outs = [np.empty(capacity[r], dtype=shards[0].dtype) if host else
                    torch.empty(capacity[r], dtype=shards[r].dtype, device=f"cuda:{self.devices[r]}")
                    for r in range(G)]
        if vals is not None and out_vals is None:
            out_vals = [np.empty(capacity[r], dtype=np.uint32) if host else
                        torch.empty(capacity[r], dtype=vals[r].dtype,
                                    device=f"cuda:{self.devices[r]}") for r in range(G)]
        P = ctypes.c_void_p * G
        U = ctypes.c_uint64 * G
        oc = U()
        st = lib().b2s_sample_sort(
            self._h, code, P(*[_ptr(x) for x in shards]),
            P(*[_ptr(v) for v in vals]) if vals is not None else None, U(*counts),
            P(*[_ptr(o) for o in outs]), P(*[_ptr(o) for o in out_vals]) if out_vals is not None else None,
            U(*capacity), oc, int(samples_per_gpu), B2S_HOST if host else B2S_DEVICE)
        if st == _lib.B2S_EINVAL and b"exceeds out_capacity" in lib().b2s_last_error() and \
                capacity != [total] * G and outs_given is None:
            # a bucket outgrew the default capacity (far from regular
            # sampling's bound): retry with room for everything
            return self.sample_sort(shards, vals, None, None, [total] * G, samples_per_gpu)
        check(st)
        sizes = [int(oc[r]) for r in range(G)]
        buckets = [outs[r][: sizes[r]] for r in range(G)]
        bvals = [out_vals[r][: sizes[r]] for r in range(G)] if out_vals is not None else None
        return buckets, bvals
