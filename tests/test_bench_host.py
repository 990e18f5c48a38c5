"""Host-side logic of bench.py (no GPU): which committed ncu summary the line's `traffic` and
issue-fraction fields come from, and that they parse."""
import os

import bench


def test_current_summary_is_read_first():
    paths = bench.ncu_summaries()
    cur = open(os.path.join(bench.ROOT, "profiles", "ncu_current.txt")).read().strip()
    assert paths and os.path.basename(paths[0]) == cur


def test_summary_metrics_parse():
    issue, src = bench.ncu_metric("generate_kernel", "smsp__issue_active.avg.pct_of_peak_sustained_active")
    assert issue is not None and 0.0 < issue <= 100.0 and src.startswith("profiles/")
    tensor, _ = bench.ncu_metric("crss_mma_sp_kernel", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    assert tensor is not None and 0.0 < tensor <= 100.0
    for k in ("crss_mma_sp_kernel", "generate_kernel"):
        t, tsrc = bench.ncu_traffic(k)
        assert t is not None and t > 0 and "ncu" in tsrc


def test_missing_kernel_gives_none():
    assert bench.ncu_metric("no_such_kernel", "gpu__time_duration.sum") == (None, None)
    assert bench.ncu_traffic("no_such_kernel") == (None, None)
