"""Generate the golden parity fixtures by running the REFERENCE package itself.

Run in the build container only (needs /root/reference and numba):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

For every fixture it stores the flat inputs (same layout as the engine C-ABI)
and the reference's own outputs:
  ref_f32 / ref_f32_kind : pairhmm.run(batches, default_configs("f32"))   (pipeline.py:77)
  ref_f64 / ref_f64_kind : pairhmm.run(batches, default_configs("f64"))
kind codes: 0 ok, 1 numeric-overflow, 2 config-too-small, 3 degenerate-transition.
Inputs come from pairhmm.datagen (datagen.py:78-158) with the SURVEY §8(d)
seeds (prefixes of the c1..c4 configs: generation is sequential per batch, so
a smaller num_batches yields a prefix of the full config) plus hand-built edge
cases.  The fixtures are consumed by tests/ only; nothing at run time reads
/root/reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

import pairhmm  # noqa: E402  (the reference)
from pairhmm import Batch, Haplotype, ReadRecord, default_configs, encode_bases, run  # noqa: E402
from pairhmm.datagen import generate_synthetic, generate_verification_pairs  # noqa: E402
from pairhmm.prob import LOG10_2, PHRED_TO_PROB  # noqa: E402

from oracle.oracle import Flat  # noqa: E402  (flattening helper only)

SEED = 20240811
OUT = os.path.dirname(os.path.abspath(__file__))
KIND_CODE = {"numeric-overflow": 1, "config-too-small": 2, "degenerate-transition": 3}


def ref_outputs(batches, precision):
    scores, report = run(batches, default_configs(precision), workers=os.cpu_count())
    kind = np.zeros(scores.shape[0], np.uint8)
    for gid, k in report.errors:
        kind[gid] = KIND_CODE[k]
    return scores, kind, report.total_cells


def save(name, batches, params):
    flat = Flat.from_batches(batches)
    f32, k32, cells32 = ref_outputs(batches, "f32")
    f64, k64, cells64 = ref_outputs(batches, "f64")
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **flat.as_dict(),
                        ref_f32=f32, ref_f32_kind=k32, ref_f64=f64, ref_f64_kind=k64,
                        ref_cells=np.array([cells32, cells64], np.int64),
                        params=np.array(json.dumps(params)))
    print("%-16s pairs=%6d f32-flagged=%5d f64-flagged=%5d cells=%d"
          % (name, f32.shape[0], int((k32 == 1).sum()), int((k64 == 1).sum()), cells32))


def gen(name, *args, **kw):
    batches = generate_synthetic(*args, **kw)
    params = {"args": list(args), "kw": kw}
    save(name, batches, params)


def edge_batches():
    def read(bases, bq=30, iq=40, dq=40, gq=10):
        codes = encode_bases(bases)
        m = codes.shape[0]

        def track(q):
            return np.full(m, q, np.uint8) if np.isscalar(q) else np.asarray(q, np.uint8)
        return ReadRecord(codes, track(bq), track(iq), track(dq), track(gq))

    def hap(bases):
        return Haplotype(encode_bases(bases))

    rng = np.random.default_rng(SEED + 99)

    def rand_bases(n, alphabet="ACGT"):
        return "".join(alphabet[i] for i in rng.integers(0, len(alphabet), n))

    batches = [
        # hand cases test_reference.py:14-30 (log10 0.81 / log10 0.03)
        Batch((read("A", 10, 40, 40, 10),), (hap("A"), hap("C"))),
        # N handling on both sides, m = n = 1 .. 3
        Batch((read("N", 20), read("NNN", 93, 40, 40, 10), read("ANA", 20)),
              (hap("N"), hap("ACG"), hap("NNNN"))),
        # degenerate read (ins=del=0) next to a good one in the same batch
        Batch((read("ACG", iq=0, dq=0), read("ACGT")), (hap("ACGTT"), hap("CG"))),
        # read too long for the default configs (1025 > 1024) and one at the edge (1024)
        Batch((read(rand_bases(1025)), read(rand_bases(1024), bq=35)),
              (hap(rand_bases(1030)),)),
        # extreme qualities: gcp 0 (beta = 0), q 93 everywhere, q 0 base quality
        Batch((read(rand_bases(40), bq=0, iq=30, dq=30, gq=0),
               read(rand_bases(37), bq=93, iq=93, dq=93, gq=93),
               read(rand_bases(64), bq=rng.integers(0, 94, 64), iq=rng.integers(4, 94, 64),
                    dq=rng.integers(4, 94, 64), gq=rng.integers(0, 94, 64))),
              (hap(rand_bases(50)), hap(rand_bases(1)), hap(rand_bases(300, "ACGTN")))),
        # read longer than the haplotype and vice versa, exact lane-product lengths
        Batch((read(rand_bases(8)), read(rand_bases(32)), read(rand_bases(255)),
               read(rand_bases(256)), read(rand_bases(257)), read(rand_bases(511)),
               read(rand_bases(512)), read(rand_bases(513))),
              (hap(rand_bases(7)), hap(rand_bases(256)), hap(rand_bases(513)))),
    ]
    return batches


def main():
    np.savez_compressed(os.path.join(OUT, "prob_tables.npz"), phred_to_prob=PHRED_TO_PROB,
                        log10_2=np.float64(LOG10_2))
    gen("c1_derived", 10, 25, 4, 100, 150, SEED, mode="derived", base_qual=30,
        indel_qual=45, gcp_qual=10)
    gen("c1_independent", 10, 25, 4, 100, 150, SEED, mode="independent", base_qual=30,
        indel_qual=45, gcp_qual=10)
    gen("c2_prefix", 8, 16, 4, 250, 250, SEED + 1, mode="derived")
    gen("c3_prefix", 8, 64, 8, (50, 250), (100, 600), SEED + 2, mode="derived")
    gen("c4_prefix", 2, 8, 4, (512, 1024), (1024, 2048), SEED + 3, mode="derived")
    gen("c4_underflow", 1, 8, 4, (512, 1024), (1024, 2048), SEED + 3, mode="derived",
        mutation_rate=0.10, base_qual=(10, 11))
    gen("short_mixed", 40, 6, 5, (1, 40), (1, 60), SEED + 5, mode="derived")
    save("verify_pairs", generate_verification_pairs(300, SEED),
         {"generate_verification_pairs": [300, SEED]})
    save("edge", edge_batches(), {"hand": "edge_batches()"})


if __name__ == "__main__":
    main()
