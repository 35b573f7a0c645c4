"""The BASELINE.json workloads as device-generated inputs (synthetic stand-ins
for the paper's unstated data). Every key stream is
bench::gen_data's splitmix64 sequence (P/src/bench.cpp:57-71, seed 1 unless
stated), generated on the GPU bit-identically to the host generator.

  cfg1  N=2^20 int32 (z >> 33), p=4 partitioned sort
  cfg2  N=2^28 uint32 (z >> 32), one local sort
  cfg3  N=2^31 int32 (z >> 33), sharded over G GPUs (plan_partition)
  cfg4  N=2^27 int32: (a) Zipf s=1.2 over 2^20 ranks, (b) ascending,
        (c) descending, (d) all equal
  cfg5  N=2^28 (uint64 z, uint32 index) pairs, stable
"""
from __future__ import annotations

import numpy as np

ZIPF_VALUES = 1 << 20
ZIPF_S = 1.2
CONST_KEY = 7


def zipf_thresholds(values: int = ZIPF_VALUES, s: float = ZIPF_S) -> np.ndarray:
    """Integer inverse-CDF table of Zipf(s) over `values` ranks: T[r] =
    floor(CDF(r) * 2^53) with the weights (r+1)^-s summed in rank order in
    float64 and T[-1] = 2^53. b2s_gen_zipf draws rank r for u = z >> 11 when
    T[r-1] <= u < T[r]; the draw is integer-only, so a host draw from the same
    table gives the same bytes."""
    w = np.power(np.arange(1, values + 1, dtype=np.float64), -s)
    cdf = np.cumsum(w)
    t = np.floor(cdf / cdf[-1] * float(1 << 53)).astype(np.uint64)
    t[-1] = np.uint64(1 << 53)
    return t


def cfg4_keys(ctx, kind: str, n: int = 1 << 27, seed: int = 1, first: int = 0,
              total: int | None = None):
    """cfg4's skewed / structured int32 inputs on ctx's device: keys
    first..first+n-1 of a stream of `total` keys (default n), so a shard of a
    sharded input is its slice of the global stream."""
    import torch
    dev = f"cuda:{ctx.device}"
    total = n if total is None else total
    if kind == "zipf":
        return ctx.gen_zipf(n, seed, zipf_thresholds(), torch.int32, first=first)
    if kind == "ascending":  # key i = i
        return torch.arange(first, first + n, dtype=torch.int32, device=dev)
    if kind == "descending":  # key i = total - 1 - i
        hi = total - 1 - first
        return torch.arange(hi, hi - n, -1, dtype=torch.int32, device=dev)
    if kind == "equal":
        return torch.full((n,), CONST_KEY, dtype=torch.int32, device=dev)
    raise ValueError(kind)
