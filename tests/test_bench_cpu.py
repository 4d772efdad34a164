"""CPU checks of bench.py's contract pieces that need no GPU: the reference arm (the fp64
oracle timed on the host) prints one JSON line with the keys the driver reads, and the
CPU-baseline sampler reports what it ran."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "2", "--warmup", "1", "--ref-seconds", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    cb = line["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and "passes" in cb["sample"]


def test_cpu_sample_uses_its_budget():
    sys.path.insert(0, ROOT)
    import bench
    import agcn_inputs as gen
    w = gen.make_config("c1")
    cb, t = bench.cpu_sample_gflops(w, w.X(), 0.3)
    assert t >= 0.27 and cb["value"] > 0 and cb["unit"] == "GFLOP/s"
