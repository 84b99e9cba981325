import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
GOLDEN = sorted(os.path.splitext(os.path.basename(p))[0]
                for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
                if "prob_tables" not in p and "matrices" not in p)   # pair-score fixtures only
SEED = 20240811


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA engine parity / API tests)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    return np.load(os.path.join(GOLDEN_DIR, name + ".npz"))


def golden_flat(z):
    from paper_2411_11547_b200.model import FlatBatches
    return FlatBatches(**{f: z[f] for f in FlatBatches.FIELDS})


@pytest.fixture
def rng():
    return np.random.default_rng(SEED)


@pytest.fixture(scope="session")
def engine():
    """The CUDA engine context (GPU tests only; fails loudly without a device)."""
    from paper_2411_11547_b200 import _native
    from paper_2411_11547_b200.build import build_native
    build_native()
    return _native.context(0)


def make_read(bases, base_q=30, ins_q=40, del_q=40, gcp_q=10):
    from paper_2411_11547_b200 import ReadRecord, encode_bases
    codes = encode_bases(bases)
    m = codes.shape[0]

    def track(q):
        return np.full(m, q, dtype=np.uint8) if np.isscalar(q) else np.asarray(q)
    return ReadRecord(codes, track(base_q), track(ins_q), track(del_q), track(gcp_q))


def make_hap(bases):
    from paper_2411_11547_b200 import Haplotype, encode_bases
    return Haplotype(encode_bases(bases))


def random_pair(rng, m, n, mutation_rate=0.01, base_q=(10, 41), indel_q=(30, 46), gcp_q=10):
    """Read derived from a random haplotype (the reference's tests/conftest.py recipe)."""
    from paper_2411_11547_b200 import Haplotype, ReadRecord
    hap = rng.integers(0, 4, size=n, dtype=np.int8)
    if m <= n:
        start = int(rng.integers(0, n - m + 1))
        read = hap[start:start + m].copy()
    else:
        read = np.concatenate([hap, rng.integers(0, 4, size=m - n, dtype=np.int8)])
    hits = rng.random(m) < mutation_rate
    if hits.any():
        read[hits] = (read[hits] + rng.integers(1, 4, size=int(hits.sum()))) % 4
    rec = ReadRecord(read, rng.integers(*base_q, size=m), rng.integers(*indel_q, size=m),
                     rng.integers(*indel_q, size=m), np.full(m, gcp_q))
    return rec, Haplotype(hap)
