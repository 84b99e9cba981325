"""Multi-GPU sharding host logic (shards.py) on CPU: cost-balanced contiguous cuts and
rebased sub-batches; the GPU test runs two shard contexts on one device."""
import numpy as np
import pytest

from paper_2411_11547_b200 import datagen
from paper_2411_11547_b200.shards import batch_costs, cut_points, sub_flat


def test_cut_points_balance_cost_and_cover_all_batches():
    flat = datagen.workload("c3", num_batches=40)
    costs = batch_costs(flat)
    assert costs.shape == (40,) and np.all(costs > 0)
    for parts in (1, 2, 3, 4, 8):
        cuts = cut_points(costs, parts)
        assert cuts[0] == 0 and cuts[-1] == 40 and np.all(np.diff(cuts) >= 0)
        shares = np.array([costs[a:b].sum() for a, b in zip(cuts[:-1], cuts[1:])])
        assert shares.sum() == pytest.approx(costs.sum())
        assert shares.max() <= costs.sum() / parts + costs.max() + 1e-9


def test_sub_flat_rebases_and_preserves_pairs():
    flat = datagen.workload("c3", num_batches=12)
    pr, ph = flat.pair_index()
    cuts = cut_points(batch_costs(flat), 3)
    got = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        s = sub_flat(flat, int(a), int(b))
        assert s.read_off[0] == 0 and s.hap_off[0] == 0 and s.batch_read_off[0] == 0
        spr, sph = s.pair_index()
        got.append((s.read_len[spr], s.hap_len[sph],
                    [bytes(s.read_bases[s.read_off[r]:s.read_off[r + 1]]) for r in spr[:5]]))
    m = np.concatenate([g[0] for g in got])
    n = np.concatenate([g[1] for g in got])
    assert np.array_equal(m, flat.read_len[pr]) and np.array_equal(n, flat.hap_len[ph])


@pytest.mark.gpu
def test_sharded_run_equals_single_device():
    from paper_2411_11547_b200 import default_configs, run
    flat = datagen.workload("c3", num_batches=24)
    a, ra = run(flat, default_configs("f32"), retry_f64=True)
    b, rb = run(flat, default_configs("f32"), retry_f64=True, devices=[0, 0, 0])
    assert np.array_equal(a, b, equal_nan=True)
    assert ra.total_cells == rb.total_cells and ra.errors == rb.errors and ra.retried == rb.retried
