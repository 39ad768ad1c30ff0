"""Host-side logic of bench.py (no GPU): the clock-aware roofline peak and the N-rank launcher's
refusal when fewer GPUs than --gpus are visible."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

PEAKS = {"bf16_tflops": 1680.5, "bf16_tflops_sustained": 1448.3, "clocks_under_load": {"sm_mhz_median": 1395.0}}


def test_tensor_peak_scales_with_the_run_clock():
    p, note, ref = bench.tensor_peak(PEAKS, "measured", 1237, False)
    assert p == pytest.approx(1448.3 * 1237 / 1395.0, rel=1e-12)
    assert ref == {"burst": 1680.5, "sustained": 1448.3} and "1237" in note
    # at the sustained measurement's own clock the peak is the sustained figure
    assert bench.tensor_peak(PEAKS, "measured", 1395, False)[0] == pytest.approx(1448.3)
    # never above the burst figure, however high the clock
    assert bench.tensor_peak(PEAKS, "measured", 1965, False)[0] == pytest.approx(1680.5)
    # FP8: x 2 (nominal fp8:bf16 dense ratio), references too
    p8, _, ref8 = bench.tensor_peak(PEAKS, "measured", 1237, True)
    assert p8 == pytest.approx(2 * p) and ref8["burst"] == pytest.approx(2 * 1680.5)
    # no clock record: the sustained figure
    assert bench.tensor_peak(PEAKS, "measured", None, False)[0] == pytest.approx(1448.3)


def test_self_launch_refuses_more_ranks_than_gpus():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "ASYNCEP_BENCH_DEVICE")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], capture_output=True,
                       text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 2
    assert "--gpus 4" in r.stderr and r.stdout.strip() == ""
