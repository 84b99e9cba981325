"""Multi-GPU sharding host logic (shards.py) on CPU: bin-stratified cost-balanced read
deal, shard extraction with global ids, and the gather; the GPU test runs three shard
contexts on one device."""
import numpy as np
import pytest

from paper_2411_11547_b200 import datagen
from paper_2411_11547_b200.shards import (TILING_WIDTHS, make_shard, plan_shards, read_costs,
                                          shards)


def _pairs(flat):
    pr, ph = flat.pair_index()
    return pr, ph


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_plan_balances_cost_and_bins(parts):
    flat = datagen.workload("c3", num_batches=64)
    cost, key = read_costs(flat)
    owner = plan_shards(flat, parts)
    assert owner.shape == (flat.num_reads,) and owner.min() >= 0 and owner.max() < parts
    loads = np.bincount(owner, weights=cost, minlength=parts)
    assert loads.sum() == pytest.approx(cost.sum())
    # within about one read per bin of the mean
    nbins = np.unique(key).shape[0]
    assert loads.max() - loads.min() <= cost.max() * max(2, nbins // parts + 2)
    assert loads.max() <= cost.sum() / parts * 1.05
    # every GPU gets the same mix of tiling-width classes (within one read per bin)
    for k in np.unique(key):
        cnt = np.bincount(owner[key == k], minlength=parts)
        assert cnt.max() - cnt.min() <= 1


def test_cost_counts_padding_to_the_tiling_width():
    flat = datagen.workload("c3", num_batches=4)
    cost, _ = read_costs(flat)
    m = flat.read_len
    W = TILING_WIDTHS[np.searchsorted(TILING_WIDTHS, m + 1)]
    rb = np.repeat(np.arange(flat.num_batches), np.diff(flat.batch_read_off))
    hsum = np.add.reduceat(flat.hap_len, flat.batch_hap_off[:-1])[rb]
    assert np.all(cost >= W * hsum) and np.all(cost < W * (hsum + 64))


@pytest.mark.parametrize("parts", [2, 3, 5])
def test_shards_partition_the_pairs_and_keep_contents(parts):
    flat = datagen.workload("c3", num_batches=20)
    pr, ph = _pairs(flat)
    got = shards(flat, parts)
    gids = np.concatenate([s.gids for s in got])
    assert np.array_equal(np.sort(gids), np.arange(flat.num_pairs))
    for s in got:
        f = s.flat
        assert f.read_off[0] == 0 and f.hap_off[0] == 0 and f.batch_read_off[0] == 0
        spr, sph = f.pair_index()
        assert np.array_equal(f.read_len[spr], flat.read_len[pr[s.gids]])
        assert np.array_equal(f.hap_len[sph], flat.hap_len[ph[s.gids]])
        # same bases and qualities for a sample of pairs
        for i in range(0, f.num_pairs, max(1, f.num_pairs // 7)):
            gr, gh, lr, lh = pr[s.gids[i]], ph[s.gids[i]], spr[i], sph[i]
            for a, b in ((f.read_bases, flat.read_bases), (f.bq, flat.bq), (f.gq, flat.gq)):
                assert np.array_equal(a[f.read_off[lr]:f.read_off[lr + 1]],
                                      b[flat.read_off[gr]:flat.read_off[gr + 1]])
            assert np.array_equal(f.hap_bases[f.hap_off[lh]:f.hap_off[lh + 1]],
                                  flat.hap_bases[flat.hap_off[gh]:flat.hap_off[gh + 1]])


def test_sharded_oracle_scores_gather_bit_identical():
    """Shard, score every shard with the CPU oracle, gather by global id: bitwise equal to
    scoring the unsharded batch list (pairs are independent)."""
    from oracle import oracle
    flat = datagen.workload("c3", num_batches=6)
    ref, kind = oracle.score(oracle.Flat(**flat.as_dict()), "f32")
    out = np.full(flat.num_pairs, -1.0)
    ok = np.zeros(flat.num_pairs, np.int64)
    for s in shards(flat, 3):
        v, k = oracle.score(oracle.Flat(**s.flat.as_dict()), "f32")
        out[s.gids] = v
        ok[s.gids] = k
    assert np.array_equal(out, ref, equal_nan=True) and np.array_equal(ok, kind)


def test_empty_shard_when_more_gpus_than_reads():
    flat = datagen.workload("c1", num_batches=1)          # 25 reads
    owner = plan_shards(flat, 32)
    s = make_shard(flat, owner, 31)
    assert s.flat.num_pairs == 0 and s.gids.shape == (0,)


@pytest.mark.gpu
def test_sharded_run_equals_single_device():
    from paper_2411_11547_b200 import default_configs, run
    flat = datagen.workload("c3", num_batches=24)
    a, ra = run(flat, default_configs("f32"), retry_f64=True)
    b, rb = run(flat, default_configs("f32"), retry_f64=True, devices=[0, 0, 0])
    assert np.array_equal(a, b, equal_nan=True)
    assert ra.total_cells == rb.total_cells and ra.errors == rb.errors and ra.retried == rb.retried


def test_check_budget_first_item_matches_per_item_definition():
    """partition.check_budget (O(reads)) raises for the same first item, with the same
    estimate, as the per-item definition (partition.py:40-45 / item_bytes)."""
    from paper_2411_11547_b200 import default_configs
    from paper_2411_11547_b200.errors import BudgetError
    from paper_2411_11547_b200.partition import check_budget, item_bytes
    flat = datagen.workload("c3", num_batches=30)
    cfgs = default_configs("f32")
    est, _ = item_bytes(flat, cfgs)
    for budget in (int(est.max()), int(np.percentile(est, 99.9)), int(np.percentile(est, 50)), 100):
        over = np.flatnonzero(est > budget)
        if over.size == 0:
            check_budget(flat, cfgs, budget)
            continue
        with pytest.raises(BudgetError) as err:
            check_budget(flat, cfgs, budget)
        assert str(err.value) == ("work item %d alone needs ~%d bytes, over the %d-byte budget"
                                  % (over[0], est[over[0]], budget))


def test_host_gather_scatter_matches_numpy():
    """HostGather.put (libphmm_host.so streaming scatter over ascending global-id runs)
    writes exactly what numpy fancy assignment writes, for run-structured and scattered
    ids; out-of-range ids raise."""
    import os
    from paper_2411_11547_b200.shards import HostGather
    rng = np.random.default_rng(7)
    n = 5000
    name = "phmm_test_scatter_%d" % os.getpid()
    g = HostGather(name, n, create=True)
    try:
        for gids in (np.arange(100, 900, dtype=np.int64),
                     np.sort(rng.choice(n, 1200, replace=False)).astype(np.int64),
                     np.concatenate([np.arange(10, 30), np.arange(40, 41), np.arange(4000, 4999)]).astype(np.int64)):
            sc = rng.random(gids.shape[0])
            st = rng.integers(0, 255, gids.shape[0]).astype(np.uint8)
            want_sc, want_st = g.scores.copy(), g.status.copy()
            want_sc[gids] = sc
            want_st[gids] = st
            g.put(gids, sc, st)
            assert np.array_equal(g.scores, want_sc) and np.array_equal(g.status, want_st)
        with pytest.raises(IndexError):
            g.put(np.array([n], np.int64), np.zeros(1), np.zeros(1, np.uint8))
    finally:
        g.close()
