"""Multi-GPU = independent replicas: requests of one trace go
round-robin to G GPUs; each replica runs its own engine, arena, layer table,
KV pool and controller.  No collective sits on the data path -- the only
cross-rank traffic is gathering reports and the max-over-ranks timing.
"""
from __future__ import annotations

from . import _core


def shard_trace(trace, rank: int, world: int):
    """Request i -> replica i mod world (arrival times unchanged)."""
    out = _core.Trace()
    out.events = [e for i, e in enumerate(trace.events) if i % world == rank]
    out.source_label = f"{trace.source_label}[{rank}/{world}]"
    return out


def merge_reports(reports: list) -> dict:
    """Union view over replicas: P95 over the union of requests, sums of counts."""
    ttft, tpot = [], []
    done = total = unserv = slo = tokens = 0
    decode_tokens = 0.0
    decode_ms = []
    end = 0.0
    for r in reports:
        for p in r["per_request"]:
            ttft.append(p["ttft_ms"])
            if p["tpot_ms"] is not None:
                tpot.append(p["tpot_ms"])
        done += r["requests"]["completed"]
        total += r["requests"]["total"]
        unserv += r["requests"]["unserviceable"]
        slo += r["slo"]["violations"]
        tokens += r["exposure"]["tokens_total"]
        end = max(end, r["sim_end_ms"])
        dev = r.get("device", {})
        decode_tokens += dev.get("decode_tokens", 0.0)
        decode_ms.append(dev.get("decode_ms", 0.0))
    p95 = _core.percentile_nearest_rank(ttft, 95.0)
    return {
        "replicas": len(reports), "requests": {"completed": done, "total": total, "unserviceable": unserv},
        "p95_ttft_ms": p95, "p95_tpot_ms": _core.percentile_nearest_rank(tpot, 95.0),
        "slo_violations": slo, "tokens_total": tokens, "sim_end_ms": end,
        "throughput_rps": done / (end / 1000.0) if end > 0 else 0.0,
        "decode_tokens": decode_tokens, "decode_ms_max_over_replicas": max(decode_ms) if decode_ms else 0.0,
    }
