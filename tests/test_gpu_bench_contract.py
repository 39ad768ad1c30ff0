"""bench.py's JSON line keeps the driver's contract (keys, types, consistency), on a small run."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # exactly one JSON line
    return json.loads(lines[0])


@pytest.mark.parametrize("fp8", [False, True], ids=["bf16", "fp8"])
def test_bench_line_contract(fp8):
    d = run_bench("--layers", "2", "--tokens", "4096", "--steps", "2", "--warmup", "3", "--no-cpu-baseline",
                  *(["--fp8"] if fp8 else []))
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["dtype"] == ("fp8_e4m3" if fp8 else "bf16") and d["data"] == "synthetic"
    assert "workload" in d["config"] and d["config"]["tokens_per_gpu"] == 4096
    # value = tokens of the timed steps / device time
    assert abs(d["value"] - 4096 * 1e3 / d["ms_per_step"]) / d["value"] < 1e-6
    rf = d["roofline"]
    assert rf["bound"] == "tensor" and rf["unit"] == "TFLOP/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9 and 0 < rf["frac"] < 1.5
    ck = d["clocks"]
    assert ck["sm_max_mhz"] > 0 and isinstance(ck["reasons"], list)
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 4096 * 4096 * 2 and e["d2h_bytes_per_step"] == 4096 * 4096 * 2
    # our kernels launched inside the timed region: 7 per BF16 layer, 9 per FP8 layer
    assert d["gpu_launches"] == 2 * 2 * (9 if fp8 else 7)


def test_bench_self_launches_two_ranks_on_one_gpu():
    """`bench.py --gpus 2` without torchrun launches the two ranks itself (here both on GPU 0 with a
    gloo control plane, ASYNCEP_BENCH_DEVICE / _BACKEND): one JSON line from rank 0, both peer-copy
    transports probed and timed, exposed AllGather = gathered - resident wall with the gathered
    output bitwise equal to the resident stack's."""
    env = dict(os.environ, ASYNCEP_BENCH_DEVICE="0", ASYNCEP_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--layers", "3",
                        "--tokens", "4096", "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                       timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch_tokens"] == 8192
    tr = d["gather_transports"]
    assert set(tr) == {"copy_kernel", "copy_engine"}
    for v in tr.values():
        assert v["probe"]["gbs"] > 0 and v["ms_per_step"] > 0
    assert d["config"]["gather"].split(" ")[0] in tr
    ex = d["exposed_ag"]
    assert ex["output_bitwise_equal_resident"] is True
    assert ex["step_ms_gathered"] > 0 and ex["step_ms_resident"] > 0
    assert d["saturation_T"]["ag_bandwidth_source"].startswith("probed")
