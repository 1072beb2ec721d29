"""`bench.py --gpus N` run without torchrun launches N ranks itself (one process
per GPU, torch.distributed.run on 127.0.0.1); CPU-only probe of the launcher."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_2_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--ranks-probe"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 for x in lines)


def test_reference_arm_line():
    """`bench.py --impl reference` (the CPU oracle port of the reference's path,
    timed on the host cores) prints one JSON line with the GPU arm's metric and
    config, the cpu_baseline / e2e objects, and an ms_per_step that is the wall
    time of the work it actually did (the sample), next to the extrapolation."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "tok/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert 0 < line["ms_per_step"] < line["ms_per_full_step_extrapolated"]
    import bench
    assert line["metric"] == bench.METRIC and line["config"]["workload"] == bench.WORKLOAD
