"""Batch text format (batchio.py) and the CLI against the reference's own behaviour:
tests/golden/batchio.json holds what the reference's parse_batch_file / write_batch_file /
write_scores produce (tests/golden/make_batchio_golden.py ran the reference), including
the exact ParseError messages; the CLI cases mirror the reference's test_io.py::TestCli.
"""
import json
import os

import numpy as np
import pytest

from conftest import ROOT
from paper_2411_11547_b200 import batchio, datagen
from paper_2411_11547_b200.cli import main
from paper_2411_11547_b200.errors import DataError, ParseError
from paper_2411_11547_b200.model import FlatBatches

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "batchio.json")))


def _write(tmp_path, text, name="b.txt"):
    path = tmp_path / name
    with open(path, "w", encoding="utf-8", newline="") as f:
        f.write(text)
    return str(path)


@pytest.mark.parametrize("name", sorted(GOLD["cases"]))
def test_parse_matches_reference(tmp_path, name):
    case = GOLD["cases"][name]
    path = _write(tmp_path, case["text"])
    want = case["outcome"]
    if "error" in want:
        with pytest.raises(ParseError) as err:
            batchio.parse_batch_file_flat(path)
        assert str(err.value) == want["message"]
        with pytest.raises(ParseError):
            batchio.parse_batch_file(path)
        return
    f = batchio.parse_batch_file_flat(path)
    assert np.diff(f.batch_read_off).tolist() == want["batch_reads"]
    assert np.diff(f.batch_hap_off).tolist() == want["batch_haps"]
    assert f.read_len.tolist() == want["read_len"] and f.hap_len.tolist() == want["hap_len"]
    for k in ("read_bases", "bq", "iq", "dq", "gq", "hap_bases"):
        assert getattr(f, k).tolist() == want[k], k
    batches = batchio.parse_batch_file(path)
    assert [len(b.reads) for b in batches] == want["batch_reads"]


def test_writers_match_reference_bytes(tmp_path):
    w = GOLD["writer"]
    nb, nr, nh, rl, hl, seed, mode = w["gen"]
    flat = datagen.generate_synthetic_flat(nb, nr, nh, tuple(rl), tuple(hl), seed, mode=mode)
    bpath = str(tmp_path / "b.txt")
    batchio.write_batch_file(bpath, flat)
    assert open(bpath).read() == w["batch_file"]
    # the Batch-object form writes the same bytes
    batchio.write_batch_file(bpath, flat.to_batches())
    assert open(bpath).read() == w["batch_file"]

    class Rep:
        total_cells, wall_seconds, gcups = w["report"]

    scores = np.array([np.nan if v is None else v for v in w["scores"]])
    errors = [tuple(e) for e in w["errors"]]
    spath = str(tmp_path / "s.txt")
    batchio.write_scores(spath, flat, scores, errors, Rep())
    assert open(spath).read() == w["score_file"]
    lines = [l for l in w["score_file"].splitlines() if not l.startswith("#")]
    assert batchio.format_score_lines(flat, scores, errors) == lines


def test_round_trip_large_flat(tmp_path):
    flat = datagen.workload("c3", num_batches=16)
    path = str(tmp_path / "c3.txt")
    batchio.write_batch_file(path, flat)
    back = batchio.parse_batch_file_flat(path)
    for k in FlatBatches.FIELDS:
        assert np.array_equal(getattr(back, k), getattr(flat, k)), k


def test_phred_strings():
    q = np.array([0, 10, 40, 93], np.uint8)
    assert batchio.decode_phred_string(batchio.encode_phred_string(q)).tolist() == q.tolist()
    with pytest.raises(DataError, match="position 2"):
        batchio.decode_phred_string("I I")


def test_missing_file_is_os_error(tmp_path):
    with pytest.raises(OSError):
        batchio.parse_batch_file_flat(str(tmp_path / "nope.txt"))


def test_from_batches_native_equals_numpy_path():
    flat = datagen.workload("c3", num_batches=5)
    batches = flat.to_batches()
    a = FlatBatches.from_batches(batches)
    for k in FlatBatches.FIELDS:
        assert np.array_equal(getattr(a, k), getattr(flat, k)), k

    class Rec:                           # duck-typed, list-backed: the numpy fallback path
        def __init__(self, r):
            self.bases, self.base_qual, self.ins_qual = list(r.bases), list(r.base_qual), list(r.ins_qual)
            self.del_qual, self.gcp_qual, self.length = list(r.del_qual), list(r.gcp_qual), r.length

    class Hap:
        def __init__(self, h):
            self.bases, self.length = list(h.bases), h.length

    class Duck:
        def __init__(self, b):
            self.reads, self.haps = [Rec(r) for r in b.reads], [Hap(h) for h in b.haps]

    d = FlatBatches.from_batches([Duck(b) for b in batches])
    for k in FlatBatches.FIELDS:
        assert np.array_equal(getattr(d, k), getattr(flat, k)), k


class TestCliCpu:
    def test_gen_writes_the_reference_stream(self, tmp_path):
        out = str(tmp_path / "d.txt")
        assert main(["gen", "--output", out, "--batches", "3", "--reads", "5", "--haps", "3",
                     "--read-len", "1:40", "--hap-len", "1:60", "--seed", "77"]) == 0
        assert open(out).read() == GOLD["writer"]["batch_file"]

    def test_usage_errors_exit_one(self):
        with pytest.raises(SystemExit) as err:
            main(["align"])
        assert err.value.code == 1
        with pytest.raises(SystemExit) as err:
            main(["frobnicate"])
        assert err.value.code == 1

    def test_missing_input_is_a_data_error(self, tmp_path):
        assert main(["align", "--input", str(tmp_path / "nope.txt"), "--output", str(tmp_path / "o.txt")]) == 2

    def test_malformed_input_is_a_data_error(self, tmp_path):
        bad = _write(tmp_path, "BATCH 1 1\nREAD AXG III III III III\nHAP ACGT\n")
        assert main(["align", "--input", bad, "--output", str(tmp_path / "o.txt")]) == 2

    def test_bad_config_is_a_data_error(self, tmp_path):
        data = str(tmp_path / "d.txt")
        main(["gen", "--output", data])
        assert main(["align", "--input", data, "--output", str(tmp_path / "o.txt"), "--configs", "3:x"]) == 2


@pytest.mark.gpu
class TestCliGpu:
    def test_gen_align_verify_bench(self, tmp_path, capsys):
        data = str(tmp_path / "d.txt")
        out = str(tmp_path / "s.txt")
        assert main(["gen", "--output", data, "--batches", "2", "--reads", "4", "--haps", "2",
                     "--read-len", "10:40", "--hap-len", "20:60", "--seed", "3"]) == 0
        assert main(["align", "--input", data, "--output", out]) == 0
        lines = [l for l in open(out) if not l.startswith("#")]
        assert len(lines) == 16
        assert main(["verify", "--pairs", "40", "--max-len", "64", "--seed", "2"]) == 0
        assert main(["bench", "--fixed-len", "32", "--reads", "4", "--haps", "2", "--batches", "1"]) == 0
        assert "gcups=" in capsys.readouterr().out

    def test_align_scores_equal_the_oracle(self, tmp_path):
        from oracle import oracle
        data = str(tmp_path / "d.txt")
        out = str(tmp_path / "s.txt")
        main(["gen", "--output", data, "--batches", "6", "--reads", "8", "--haps", "3", "--seed", "8",
              "--read-len", "10:200", "--hap-len", "50:400"])
        assert main(["align", "--input", data, "--output", out]) == 0
        flat = batchio.parse_batch_file_flat(data)
        ref, kind = oracle.score(oracle.Flat(**flat.as_dict()), "f32")
        got = [l.split()[3] for l in open(out) if not l.startswith("#")]
        for g, r, k in zip(got, ref, kind):
            if k == 0:
                assert abs(float(g) - r) <= 1e-4 * abs(r) + 1e-6
            else:
                assert g.startswith("ERROR:")

    def test_align_f64_matches_f32_closely(self, tmp_path):
        data = str(tmp_path / "d.txt")
        main(["gen", "--output", data, "--seed", "12", "--read-len", "10:100", "--hap-len", "120:200"])
        vals = {}
        for precision in ("f32", "f64"):
            out = str(tmp_path / (precision + ".txt"))
            main(["align", "--input", data, "--output", out, "--precision", precision])
            vals[precision] = [float(l.split()[3]) for l in open(out) if not l.startswith("#")]
        assert max(abs(a - b) for a, b in zip(vals["f32"], vals["f64"])) <= 1e-3

    def test_verify_long_pairs_batched_f64(self, capsys):
        # 1,000 pairs up to 1,024 x 1,024 with the FP64 retry: every pair within tolerance
        assert main(["verify", "--pairs", "1000", "--max-len", "1024", "--seed", "5", "--retry-f64",
                     "--tol", "1e-4"]) == 0
        assert "failures=0" in capsys.readouterr().out
