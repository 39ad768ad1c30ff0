"""Host-side logic of bench.py (no GPU): the roofline peak and the N-rank launcher's
refusal when fewer GPUs than --gpus are visible."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

PEAKS = {"bf16_tflops": 1680.5, "bf16_tflops_sustained": 1448.3, "clocks_under_load": {"sm_mhz_median": 1395.0}}


def test_tensor_peak_follows_the_runs_clock_record():
    capped = {"sm_mhz": 1237, "sm_max_mhz": 1965, "reasons": ["sw_power_cap"]}
    p, note, ref = bench.tensor_peak(PEAKS, "measured", capped, False)
    assert p == pytest.approx(1448.3) and "1448.3" in note
    assert ref["burst"] == 1680.5 and ref["sustained"] == 1448.3
    # context: the nominal 8,192 FLOP/clk/SM x 148 SMs at the run's clock
    assert ref["nominal_at_run_clock"] == pytest.approx(8192 * 148 * 1237e6 / 1e12)
    # FP8: x 2 (nominal fp8:bf16 dense ratio), references too
    p8, _, ref8 = bench.tensor_peak(PEAKS, "measured", capped, True)
    assert p8 == pytest.approx(2 * p) and ref8["burst"] == pytest.approx(2 * 1680.5)
    assert ref8["nominal_at_run_clock"] == pytest.approx(2 * ref["nominal_at_run_clock"])
    # below max clock with no reason recorded: still the sustained rate
    assert bench.tensor_peak(PEAKS, "measured", {"sm_mhz": 1500, "sm_max_mhz": 1965, "reasons": []},
                             False)[0] == pytest.approx(1448.3)
    # a short run at the maximum clock, never throttled: the burst rate
    pb, nb, _ = bench.tensor_peak(PEAKS, "measured", {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []}, False)
    assert pb == pytest.approx(1680.5) and "burst" in nb
    # no clock record: sustained, and no nominal figure
    pn, _, refn = bench.tensor_peak(PEAKS, "measured", {}, False)
    assert pn == pytest.approx(1448.3) and refn["nominal_at_run_clock"] is None


def test_self_launch_refuses_more_ranks_than_gpus():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "ASYNCEP_BENCH_DEVICE")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                       text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 2
    assert "--gpus 4" in r.stderr and r.stdout.strip() == ""
