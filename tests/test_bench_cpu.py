"""The reference arm of bench.py runs on CPU (the oracle on a bounded
sample) and prints one JSON line with the keys the driver reads; checked on
a small square variant so it finishes in seconds."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--rows", "256",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, cwd=ROOT,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Gcells/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_gpus_flag_fails_loudly_without_enough_gpus():
    """`bench.py --gpus 2` outside torchrun launches the ranks itself -- and on
    a box with fewer GPUs (this CPU container: none) it must refuse, not time
    one GPU and report n_gpus = 1."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1", "--warmup",
                          "3"], capture_output=True, text=True, cwd=ROOT, timeout=600, env=env)
    assert out.returncode == 2, (out.returncode, out.stderr[-1000:])
    assert "--gpus 2" in out.stderr
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                         capture_output=True, text=True, cwd=ROOT, timeout=600, env=env)
    assert out.returncode == 2 and "WORLD_SIZE=2" in out.stderr


def test_gen_only_cfg4_variant():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gen-only", "--config", "cfg4", "--rows",
                          "512"], capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-1000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["config"] == "cfg4" and d["cells"] == 512 * 512 and abs(d["nodata_frac"] - 0.3) < 0.1
