"""Writes tests/golden/fullsize.json: order-sensitive fingerprints of the
sorted output of every BASELINE.json configuration at its FULL size, computed
on the CPU from the same seeded bytes the GPU sorts.

    python tests/golden/make_fullsize.py          (build container, ~10 min, ~40 GB RAM)

Expected outputs come from a CPU sort of the generated input (numpy's sort,
and numpy's stable argsort for the key/value config). Where the reference
library fits in host memory it is run as well, and its output must give the
same fingerprint:

  cfg2   2^28 uint32 (gen_data >> 32)         reference scatter_merge_sort(merge, p=8) on the
                                              int64 widening: checked
  cfg3   2^31 int32 (gen_data >> 33), G=1      numpy only (the reference needs ~90 GB at 2^31,
                                              SURVEY.md 8(d)); bit-identical by the cfg2 check
  cfg4a  2^27 int32 Zipf(1.2) over 2^20 ranks  reference checked
  cfg4b-d ascending / descending / all-equal   closed form, reference checked for (b)
  cfg5   2^28 (uint64 key, uint32 index)       keys: reference on the order-preserving int64
                                              image k ^ 2^63; payload: stable argsort (the
                                              reference has no payload; its tie rule is
                                              P/src/sort_core.cpp:46,77)

Fingerprints are oracle.fingerprint (sum_i mix(w_i ^ mix(i+1)) over the 64-bit
widening, = b2s_check_sorted's); the payload is fingerprinted the same way as a
uint32 array. Every config also records the input's multiset hash.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fullsize.json")


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def ref_fp(keys_i64: np.ndarray, unmap=None) -> int:
    out, secs = oracle.ref_scatter_merge_sort(keys_i64, 8, "merge", cores=8, wall=True)
    if unmap is not None:
        out = unmap(out)
    fp = oracle.fingerprint_chunked(out)
    log(f"  reference scatter_merge_sort(merge, p=8): {secs:.1f} s")
    return fp


def entry(name, keys, sorted_keys, **extra):
    e = {"config": name, "n": int(keys.size), "dtype": str(keys.dtype),
         "input_multiset": str(oracle.multiset_hash(keys)),
         "fp": str(oracle.fingerprint_chunked(sorted_keys)),
         "multiset": str(oracle.multiset_hash(sorted_keys))}
    e.update(extra)
    assert e["input_multiset"] == e["multiset"], name
    return e


def main() -> None:
    if not oracle.ref_available():
        oracle.build()
    rows = []

    log("cfg2: 2^28 uint32")
    k = oracle.gen_keys(1 << 28, 1, np.uint32, shift=32)
    s = np.sort(k)
    e = entry("cfg2", k, s, seed=1, shift=32, source="numpy sort")
    assert str(ref_fp(k.astype(np.int64))) == e["fp"]
    e["reference_checked"] = True
    rows.append(e)
    del k, s

    log("cfg3 G=1: 2^31 int32")
    k = oracle.gen_keys(1 << 31, 1, np.int32, shift=33)
    ms_in = oracle.multiset_hash(k)
    k.sort()
    rows.append({"config": "cfg3", "n": 1 << 31, "dtype": "int32", "seed": 1, "shift": 33,
                 "input_multiset": str(ms_in), "fp": str(oracle.fingerprint_chunked(k)),
                 "multiset": str(oracle.multiset_hash(k)), "source": "numpy sort",
                 "reference_checked": False})
    del k

    n4 = 1 << 27
    t = oracle.zipf_thresholds(1 << 20, 1.2)
    log("cfg4a: Zipf")
    k = oracle.zipf_keys(n4, 1, t)
    s = np.sort(k)
    e = entry("cfg4a", k, s, seed=1, zipf_values=1 << 20, zipf_s=1.2,
              thresholds_fp=str(oracle.fingerprint(t)), source="numpy sort")
    assert str(ref_fp(k.astype(np.int64))) == e["fp"]
    e["reference_checked"] = True
    rows.append(e)
    log("cfg4b-d")
    k = np.arange(n4, dtype=np.int32)
    e = entry("cfg4b", k, k, source="closed form (ascending i)")
    assert str(ref_fp(k.astype(np.int64))) == e["fp"]
    e["reference_checked"] = True
    rows.append(e)
    kd = k[::-1].copy()
    rows.append(entry("cfg4c", kd, k, source="closed form (descending n-1-i)",
                      reference_checked=False))
    kc = np.full(n4, 7, dtype=np.int32)
    rows.append(entry("cfg4d", kc, kc, value=7, source="closed form (all equal 7)",
                      reference_checked=False))
    del k, kd, kc

    log("cfg5: 2^28 (uint64, uint32 index)")
    n5 = 1 << 28
    k = oracle.gen_keys(n5, 1, np.uint64)
    order = np.argsort(k, kind="stable")
    sk = k[order]
    sv = order.astype(np.uint32)
    e = entry("cfg5", k, sk, seed=1, source="numpy stable argsort",
              payload_fp=str(oracle.fingerprint_chunked(sv)))
    del order, sv
    top = np.uint64(1 << 63)
    img = (k ^ top).view(np.int64)
    assert str(ref_fp(img, unmap=lambda o: o.view(np.uint64) ^ top)) == e["fp"]
    e["reference_checked"] = True
    rows.append(e)

    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_fullsize.py", "configs": rows}, f, indent=1)
    log("wrote", OUT)


if __name__ == "__main__":
    main()
