"""In-process XRS (qk_xrs_swap_local): 2^R slices of 2^(N-R) amplitudes on one
device, swapped in place by k_slab_swap; reports HBM GB/s (every swapped
amplitude is read and written on both sides: 64 B per swapped pair).
python tools/xrsbench.py N R"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_14697_b200 as qk

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1
region = n - R
sl = [qk.State(n, R, r, region, 0) for r in range(1 << R)]
for S in range(1, R + 1):
    pairs = [(region - S + j, region + j) for j in range(S)]  # AIO-staged: the top S in-rank positions
    qk.xrs_swap(sl, pairs)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        qk.xrs_swap(sl, pairs)
        best = min(best, time.perf_counter() - t0)
    swapped = (1 << R) * (1 << region) * (1 - 2.0 ** -S) / 2  # unordered pairs of amplitudes
    print(f"N={n} R={R} S={S}: {best * 1e3:8.2f} ms, {64 * swapped / best / 1e9:7.0f} GB/s HBM "
          f"(16 B/amp x (1-2^-S) per slice = {16 * (1 << region) * (1 - 2.0 ** -S) / best / 1e9:6.0f} GB/s per rank per direction)",
          flush=True)
