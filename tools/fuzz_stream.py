"""Randomized parity sweep of the stream kernels against the oracle (GPU).

usage: python tools/fuzz_stream.py [first_seed] [last_seed]
Runs tests/test_gpu_stream.py's random-shape check for every seed in the range, plus a
long-read variant (reads up to 1,023: striped team/sequential modes, second-stage FP64).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_stream as T  # noqa: E402
from paper_2411_11547_b200 import _native  # noqa: E402

a = int(sys.argv[1]) if len(sys.argv) > 1 else 5
b = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ctx = _native.Context(0)
for seed in range(a, b + 1):
    T.test_random_batches_all_modes_against_oracle(ctx, seed)
    rng = np.random.default_rng(5000 + seed)
    spec = []
    for _ in range(int(rng.integers(1, 6))):
        reads = [int(x) for x in rng.integers(200, 1024, size=int(rng.integers(1, 5)))]
        haps = [int(x) for x in rng.integers(1, 2048, size=int(rng.integers(1, 6)))]
        spec.append((reads, haps, ["random", "derived", "degenerate"][int(rng.integers(0, 3))]))
    T._check(ctx, T._flat(rng, spec))
    print("seed %d ok" % seed, flush=True)
