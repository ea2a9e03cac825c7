"""The reference's benchmark harness API (bench.hpp) on the device heap:
the batch plan against the reference's own run_workload, CSV columns, and
(GPU) verified + timed rows."""
import io

import numpy as np
import pytest

from oracle import oracle as O
from paper_1906_06504_b200 import Variant
from paper_1906_06504_b200 import workload as W


@pytest.mark.parametrize("k,workers,pct", [(64, 4, 100), (64, 4, 70), (16, 3, 20), (1, 2, 50)])
def test_plan_batches_covers_keys(k, workers, pct):
    spec = W.WorkloadSpec(k=k, workers=workers, total_keys=100_003, full_batch_pct=pct, seed=5)
    lens = W.plan_batches(spec)
    assert int(lens.sum()) == spec.total_keys
    assert lens.min() >= 1 and lens.max() <= k
    if pct == 100:
        assert (lens == k).sum() >= len(lens) - workers  # only share tails are short


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("pct", [100, 60, 20])
def test_plan_batches_matches_reference_batch_count(pct):
    """Every planned batch is one counted insert in the reference's
    run_workload, so its insert counter equals our plan's batch count."""
    spec = W.WorkloadSpec(k=32, workers=3, total_keys=50_000, full_batch_pct=pct, seed=9,
                          op_pattern=W.OpPattern.InsDelPairs)
    out = np.zeros(7, np.float64)
    st = O.ref().ref_run_workload(0, spec.k, spec.workers, spec.total_keys, 0, 1, 0, pct, spec.seed, out)
    assert st == 0
    assert int(out[5]) == len(W.plan_batches(spec))  # every planned batch is one counted insert


def test_csv_columns_match_reference_writer():
    row = W.BenchRow(W.WorkloadSpec(), 1.5, 10, 6.66667, 2.25, None)

    class C:
        merges, early_stops, max_partial_len = 7, 3, 12
    row.counters = C()
    buf = io.StringIO()
    W.write_csv(buf, [row])
    lines = buf.getvalue().splitlines()
    assert lines[0] == W.CSV_HEADER
    assert lines[1] == "td,64,4,1000000,random,insall,0,100,1,1.5,10,6.66667,2.25,7,3,12"


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [Variant.TD, Variant.BU])
@pytest.mark.parametrize("pattern", [W.OpPattern.InsertAllThenDeleteAll, W.OpPattern.InsDelPairs])
def test_run_workload_rows(variant, pattern):
    spec = W.WorkloadSpec(variant=variant, k=64, workers=4, total_keys=200_000, op_pattern=pattern,
                          initial_levels=5, full_batch_pct=80, seed=3)
    row = W.run_workload(spec)  # raises if the verified pass fails
    n_batches = len(W.plan_batches(spec))
    assert row.counters.inserts == n_batches
    # (deletes that find the heap empty are not counted, as in the
    # reference; concurrency decides how many do)
    assert row.ops == row.counters.inserts + row.counters.deletes and row.ops_per_second > 0
    buf = io.StringIO()
    W.write_csv(buf, [row])
    assert len(buf.getvalue().splitlines()) == 2


@pytest.mark.gpu
@pytest.mark.skipif(not O.ref_available(), reason="reference library not built")
@pytest.mark.parametrize("pct", [100, 60, 20])
def test_run_workload_op_count_matches_reference(pct):
    """Same spec on the device and in the reference's run_workload: the
    counted ops (counter semantics replayed exactly in test_gpu_heap) agree,
    so the two plans agree batch for batch."""
    spec = W.WorkloadSpec(variant=Variant.BU, k=32, workers=3, total_keys=50_000, full_batch_pct=pct, seed=9,
                          op_pattern=W.OpPattern.InsDelPairs)
    out = np.zeros(7, np.float64)
    assert O.ref().ref_run_workload(1, spec.k, spec.workers, spec.total_keys, 0, 1, 0, pct, spec.seed, out) == 0
    assert W.run_workload(spec).counters.inserts == int(out[5])
