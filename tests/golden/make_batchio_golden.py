"""Generate the batch-text-format fixtures by running the REFERENCE package itself.

Run in the build container only (needs /root/reference):

    python tests/golden/make_batchio_golden.py

For every case of CASES it stores the file text and the reference's own outcome of
pairhmm.batchio.parse_batch_file (batchio.py:50-108): either the ParseError message or
the parsed batches (flat arrays, as lists); plus the reference's write_batch_file and
write_scores output for a generated batch list.  tests/test_batchio.py consumes
tests/golden/batchio.json; nothing at run time reads /root/reference.
"""
from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from pairhmm.batchio import parse_batch_file, write_batch_file, write_scores  # noqa: E402
from pairhmm.datagen import generate_synthetic  # noqa: E402
from pairhmm.errors import PairHmmError  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

GOOD = "# comment line\nBATCH 1 1\nREAD ACG III III III III\n\nHAP ACGT\n"
CASES = {
    # the reference's own test_io.py cases
    "minimal": GOOD,
    "header_fields": "BATCH 1\nREAD A I I I I\nHAP A\n",
    "header_int": "BATCH x 1\nREAD A I I I I\nHAP A\n",
    "no_header": "READ A I I I I\n",
    "qual_len": "BATCH 1 1\nREAD ACG II III III III\nHAP A\n",
    "read_base": "BATCH 1 1\nREAD AXG III III III III\nHAP A\n",
    "hap_base": "BATCH 1 1\nREAD ACG III III III III\nHAP AXGT\n",
    "missing_read": "BATCH 2 1\nREAD ACG III III III III\nHAP ACGT\n",
    "eof": "BATCH 1 2\nREAD ACG III III III III\nHAP ACGT\n",
    "read_fields": "BATCH 1 1\nREAD ACG III III III\nHAP ACGT\n",
    # further edges (the native reader hands all but the canonical ones to the slow path)
    "empty": "",
    "only_comments": "# a\n\n   \n# b\n",
    "no_trailing_newline": "BATCH 1 1\nREAD ACGTN !!!!! ~~~~~ +++++ 55555\nHAP ACGTNNA",
    "crlf": "BATCH 1 2\r\nREAD AC II II II II\r\nHAP A\r\nHAP CG\r\n",
    "lone_cr": "BATCH 1 1\rREAD AC II II II II\rHAP A\r",
    "tabs_and_spaces": "  BATCH\t2   1 \nREAD\tAC II II II II   \n \tREAD G I I I I\nHAP  T\n",
    "plus_count": "BATCH +1 1\nREAD A I I I I\nHAP A\n",
    "underscore_count": "BATCH 1_0 1\n" + "READ A I I I I\n" * 10 + "HAP A\n",
    "zero_count": "BATCH 0 1\nHAP A\n",
    "negative_count": "BATCH 1 -1\nREAD A I I I I\n",
    "lowercase_base": "BATCH 1 1\nREAD acg III III III III\nHAP ACG\n",
    "qual_del": "BATCH 1 1\nREAD AC I\x7f II II II\nHAP A\n",
    "qual_space_like": "BATCH 1 1\nREAD AC I\x1f II II II\nHAP A\n",
    "qual_unicode": "BATCH 1 1\nREAD AC I\u00e9 II II II\nHAP A\n",
    "unicode_space": "BATCH\u20031 1\nREAD A\u00a0I I I I\nHAP A\n",
    "bom": "\ufeffBATCH 1 1\nREAD A I I I I\nHAP A\n",
    "hap_fields": "BATCH 1 1\nREAD A I I I I\nHAP A C\n",
    "wrong_record": "BATCH 1 1\nREAD A I I I I\nREAD A I I I I\n",
    "comment_inside": "BATCH 2 1\nREAD A I I I I\n# note\nREAD C I I I I\nHAP AC\n",
    "hash_not_first": "BATCH 1 1\nREAD A I I I I\nHAP A#C\n",
    "trailing_text": "BATCH 1 1\nREAD A I I I I\nHAP A\nBATCH\n",
}


def outcome(text):
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False, encoding="utf-8", newline="") as f:
        f.write(text)
        path = f.name
    try:
        batches = parse_batch_file(path)
    except PairHmmError as exc:
        return {"error": type(exc).__name__, "message": str(exc)}
    finally:
        os.unlink(path)
    reads = [r for b in batches for r in b.reads]
    haps = [h for b in batches for h in b.haps]
    cat = lambda xs: np.concatenate(xs).tolist() if xs else []   # noqa: E731
    return {"batch_reads": [len(b.reads) for b in batches], "batch_haps": [len(b.haps) for b in batches],
            "read_len": [r.length for r in reads], "hap_len": [h.length for h in haps],
            "read_bases": cat([r.bases for r in reads]), "bq": cat([r.base_qual for r in reads]),
            "iq": cat([r.ins_qual for r in reads]), "dq": cat([r.del_qual for r in reads]),
            "gq": cat([r.gcp_qual for r in reads]), "hap_bases": cat([h.bases for h in haps])}


class _Report:
    total_cells, wall_seconds, gcups = 987654321, 0.1234567, 8.0000004


def main():
    out = {"cases": {name: {"text": text, "outcome": outcome(text)} for name, text in CASES.items()}}
    batches = generate_synthetic(3, 5, 3, (1, 40), (1, 60), seed=77, mode="derived")
    with tempfile.TemporaryDirectory() as d:
        write_batch_file(os.path.join(d, "b.txt"), batches)
        n = sum(b.num_items for b in batches)
        rng = np.random.default_rng(5)
        scores = -rng.random(n) * 100.0
        scores[[0, 7, 11]] = [0.0, -0.0000004, -0.0000005]
        scores[[4, 9]] = np.nan
        errors = [(4, "numeric-overflow"), (20, "degenerate-transition")]
        write_scores(os.path.join(d, "s.txt"), batches, scores, errors, _Report())
        out["writer"] = {"gen": [3, 5, 3, [1, 40], [1, 60], 77, "derived"],
                         "batch_file": open(os.path.join(d, "b.txt")).read(),
                         "scores": [None if np.isnan(v) else float(v) for v in scores],
                         "errors": errors, "report": [_Report.total_cells, _Report.wall_seconds, _Report.gcups],
                         "score_file": open(os.path.join(d, "s.txt")).read()}
    with open(os.path.join(OUT, "batchio.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", os.path.join(OUT, "batchio.json"))


if __name__ == "__main__":
    main()
