#!/usr/bin/env python3
"""Regenerate the reference's missing codec fixtures (proj/tests/codec_test.cpp
:286-322 reads them from tests/data/, which the reference does not ship --
SURVEY.md §8c) WITH THE REFERENCE ITSELF (oracle/_ref, its own encoders and
writers), into tests/golden/ref_data/.  The unmodified codec_test then runs
against the drop-in (make ref_tests), so the drop-in's decoders and encoders
are pinned to bytes the reference produced.  Test infrastructure only.

  python oracle/make_ref_data.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "ref_data")


def main():
    from oracle import ref_oracle
    ro = ref_oracle()
    if ro is None:
        sys.exit("oracle/_ref not built (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    m = 48
    idx = np.array([1, 7, 12, 30, 47], np.uint64)  # 5 entries over M = 48 (codec_test.cpp:290)
    val = np.array([1.5, -2.0, 3.25, 0.5, -7.0], np.float32)
    files = {"tensor_m48.zspt": ro.write_sparse(m, idx, val),
             "coo64_m48.bin": ro.write_framed("coo", m, idx, val, coo_bits=64),
             "bitmap_m48.bin": ro.write_framed("bitmap", m, idx, val),
             "block8_m48.bin": ro.write_framed("tensor_block", m, idx, val, block_size=8)}
    # server 0's slice under HashUniverseTable(48, 3, 2024) (codec_test.cpp:297-301)
    own = ro.partition_of(idx, 2024, 3) == 0
    files["hashbitmap_s0_seed2024_m48.bin"] = ro.write_framed("hash_bitmap", m, idx[own], val[own],
                                                              n=3, pseed=2024, server=0)
    files["hashbitmap_s0_expected.zspt"] = ro.write_sparse(m, idx[own], val[own])
    for name, data in files.items():
        with open(os.path.join(OUT, name), "wb") as f:
            f.write(bytes(data))
        print(f"{name}: {len(data)} bytes")


if __name__ == "__main__":
    main()
