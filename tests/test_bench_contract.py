"""The reference arm of bench.py (the CPU oracle, tier framing) runs on a CPU host and prints
exactly one JSON line on stdout carrying the driver's contract keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout  # nothing but the JSON line on stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"] == "gpt3-1b"


def test_roofline_classes():
    """bench.roofline picks the dominant class (tensor-bound when it has FLOPs); roofline_hbm lists
    only FLOP-free classes, largest time first, achieved = algorithmic bytes / time."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    ks = {"gemm_fwd": {"launches": 10, "ms": 20.0, "flops": 2e13, "bytes": 1e9},
          "layernorm": {"launches": 4, "ms": 2.0, "flops": 0, "bytes": 8e9},
          "embed": {"launches": 2, "ms": 0.5, "flops": 0, "bytes": 1e9},
          "misc": {"launches": 0, "ms": 0.0, "flops": 0, "bytes": 0}}
    r = bench.roofline(ks, 25.0, 1, 1400.0, 6500.0, "measured")
    assert r["kernel"] == "gemm_fwd" and r["bound"] == "tensor"
    assert abs(r["achieved"] - 1000.0) < 1e-9  # 2e12 FLOP per launch / 2 ms
    h = bench.roofline_hbm(ks, 25.0, 1, 6500.0, "measured")
    assert [x["kernel"] for x in h] == ["layernorm", "embed"]
    assert abs(h[0]["achieved"] - 4000.0) < 1e-9  # 8e9 B / 2 ms
    assert abs(h[0]["frac"] - 4000.0 / 6500.0) < 1e-12
