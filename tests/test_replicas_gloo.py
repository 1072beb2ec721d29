"""N>1 path on CPU: two gloo ranks each serve their round-robin shard of one
bursty trace on their own engine (cost-model clock; on GPUs the same code runs
with a DeviceModel per rank).  Each replica's event log must equal a
single-process run of the same shard, and the union report must be the merge
of the per-shard reports."""
import json
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = os.path.join(ROOT, "tests", "golden", "example.json")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _serve_shard(rank, world):
    from paper_2506_02006_b200 import _core, morphsim as M
    from paper_2506_02006_b200.replicas import shard_trace
    doc = {k: v for k, v in json.load(open(CFG)).items() if k != "sequence_file"}
    cfg = M.config_from_json(doc)
    cfg["workload"]["synth"].update(total_ms=12000, burst_start_ms=2000, burst_len_ms=4000)
    trace = shard_trace(M.resolve_workload(cfg), rank, world)
    out = _core.run_simulation(M._engine_dict(cfg), M.arm_spec(cfg, "static-full"), trace, int(cfg["seed"]))
    return json.loads(out["report_json"]), out["log"]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep, log = _serve_shard(rank, world)
    t = torch.tensor([rep["sim_end_ms"]], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max-over-ranks timing
    gathered = [None] * world
    dist.all_gather_object(gathered, (rep, log))
    if rank == 0:
        q.put((gathered, float(t.item())))
    dist.destroy_process_group()


def test_two_replicas_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2506_02006_b200.replicas import merge_reports
    for r in range(world):
        rep, log = _serve_shard(r, world)  # same shard, single process
        assert gathered[r][1] == log
        assert gathered[r][0] == rep
    merged = merge_reports([g[0] for g in gathered])
    assert merged["requests"]["total"] == sum(g[0]["requests"]["total"] for g in gathered)
    assert merged["sim_end_ms"] == tmax
    assert merged["p95_ttft_ms"] is not None
