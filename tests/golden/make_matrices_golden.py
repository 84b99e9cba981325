"""Generate the DP-matrix fixtures by running the REFERENCE's forward_matrices
(reference.py:150-156) on a handful of pairs.  Build container only:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_matrices_golden.py

Writes tests/golden/matrices.npz: per case the read tracks, haplotype, scale and the
reference's M, I, D (float64, (m+1) x (n+1)); tests/test_gpu_api.py compares the GPU
k_matrices bit for bit.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from pairhmm import Haplotype, ReadRecord  # noqa: E402
from pairhmm.datagen import generate_verification_pairs  # noqa: E402
from pairhmm.reference import forward_matrices  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(1234)
    cases = []
    for b in generate_verification_pairs(6, seed=99, max_read_len=120, max_hap_len=160):
        cases.append((b.reads[0], b.haps[0], 0))
    # hand-built edges: N bases, q = 0 / 93 tracks, gcp 0, 1 x 1, scale 120
    m, n = 17, 23
    bases = rng.integers(0, 5, m).astype(np.int8)
    hap = rng.integers(0, 5, n).astype(np.int8)
    q = lambda lo, hi: rng.integers(lo, hi + 1, m).astype(np.uint8)   # noqa: E731
    cases.append((ReadRecord(bases, q(0, 93), q(20, 93), q(20, 93), q(0, 40)), Haplotype(hap), 0))
    cases.append((ReadRecord(bases, q(0, 93), q(30, 45), q(30, 45), np.zeros(m, np.uint8)), Haplotype(hap), 120))
    cases.append((ReadRecord(np.array([4], np.int8), np.array([0], np.uint8), np.array([93], np.uint8),
                             np.array([93], np.uint8), np.array([10], np.uint8)), Haplotype(np.array([2], np.int8)), 0))
    out = {}
    for i, (r, h, s) in enumerate(cases):
        mat = forward_matrices(r, h, s)
        for k, v in (("bases", r.bases), ("bq", r.base_qual), ("iq", r.ins_qual), ("dq", r.del_qual),
                     ("gq", r.gcp_qual), ("hap", h.bases), ("M", mat.M), ("I", mat.I), ("D", mat.D)):
            out["%d_%s" % (i, k)] = np.asarray(v)
        out["%d_scale" % i] = np.array(s)
    out["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(OUT, "matrices.npz"), **out)
    print("wrote %d cases" % len(cases))


if __name__ == "__main__":
    main()
