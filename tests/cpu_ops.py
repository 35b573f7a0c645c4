"""TEST INFRASTRUCTURE: CPU restatements of the sample-sort device steps
(b2s_sample_regular / b2s_select_splitters / b2s_bucket_bounds / b2s_merge /
b2s_sort / b2s_check_sorted semantics) so the multi-rank host logic in
paper_1105_6040_b200/sample_sort.py can be exercised with the gloo backend on
CPU. Sorting and merging go through the C oracle."""
import numpy as np
import torch

import oracle

EMPTY = np.uint64(0xFFFFFFFFFFFFFFFF)
_NP = {torch.int32: np.int32, torch.uint32: np.uint32, torch.int64: np.int64,
       torch.uint64: np.uint64}
_VIEW = {torch.uint32: (torch.int32, np.uint32), torch.uint64: (torch.int64, np.uint64)}


def to_np(t: torch.Tensor) -> np.ndarray:
    if t.dtype in _VIEW:
        wire, npd = _VIEW[t.dtype]
        return t.view(wire).numpy().view(npd)
    return t.numpy()


def to_t(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        return torch.from_numpy(a.view(np.int32)).view(torch.uint32)
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64)).view(torch.uint64)
    return torch.from_numpy(a)


def ord_bits(a: np.ndarray) -> np.ndarray:
    if a.dtype == np.int32:
        return (a.view(np.uint32) ^ np.uint32(0x80000000)).astype(np.uint64)
    if a.dtype == np.int64:
        return a.view(np.uint64) ^ np.uint64(1 << 63)
    return a.astype(np.uint64)


class CpuOps:
    def sort(self, keys, vals):
        k = to_np(keys)
        if vals is None:
            return to_t(oracle.sort(k)), None
        sk, sv = oracle.stable_sort_kv(k, to_np(vals).view(np.uint32))
        return to_t(sk), to_t(sv.view(np.int32)).view(vals.dtype) if vals.dtype == torch.int32 \
            else to_t(sv)

    def sample(self, sorted_keys, rank, s):
        k = to_np(sorted_keys)
        n = k.size
        out = np.empty((s, 2), dtype=np.uint64)
        if n == 0:
            out[:] = EMPTY
            return to_t(out)
        pos = ((2 * np.arange(s, dtype=np.uint64) + 1) * np.uint64(n)) // np.uint64(2 * s)
        out[:, 0] = ord_bits(k)[pos.astype(np.int64)]
        out[:, 1] = (np.uint64(rank) << np.uint64(40)) | pos
        return to_t(out)

    def select(self, samples, nparts):
        s = to_np(samples)
        order = np.lexsort((s[:, 1], s[:, 0]))
        s = s[order]
        v = int(np.sum(s[:, 1] != EMPTY))
        out = np.empty((max(nparts - 1, 1), 2), dtype=np.uint64)
        for i in range(nparts - 1):
            r = ((i + 1) * v) // nparts
            out[i] = s[min(r, v - 1)] if v > 0 else (EMPTY, EMPTY)
        return to_t(out)

    def bounds(self, sorted_keys, rank, splitters, nparts):
        k = ord_bits(to_np(sorted_keys))
        sp = to_np(splitters)
        b = np.zeros(nparts + 1, dtype=np.int64)
        b[nparts] = k.size
        for i in range(1, nparts):
            key, tag = sp[i - 1]
            if tag == EMPTY:
                b[i] = k.size
                continue
            srank = int(tag >> np.uint64(40))
            if rank < srank:
                b[i] = np.searchsorted(k, key, side="right")
            elif rank > srank:
                b[i] = np.searchsorted(k, key, side="left")
            else:
                b[i] = int(tag & np.uint64((1 << 40) - 1))
        return torch.from_numpy(b)

    def merge(self, runs, vals):
        ks = [to_np(r) for r in runs]
        if vals is None:
            return to_t(oracle.merge_kway(ks)), None
        vs = [to_np(v).view(np.uint32) for v in vals]
        # stable by key with ties in run order == stable sort of the concatenation
        k, v = oracle.stable_sort_kv(np.concatenate(ks), np.concatenate(vs))
        return to_t(k), to_t(v.view(np.int32)).view(vals[0].dtype) if vals[0].dtype == torch.int32 \
            else to_t(v)

    def check(self, keys):
        k = to_np(keys)
        inv = int(np.sum(k[1:] < k[:-1])) if k.size > 1 else 0
        w = k.astype(np.int64).view(np.uint64) if k.dtype in (np.int32, np.int64) else \
            k.astype(np.uint64)
        with np.errstate(over="ignore"):
            ms = int(np.sum(oracle._mix(w), dtype=np.uint64))
        return inv, oracle.fingerprint(k), ms
