"""Serving runs on the B200: the morphsim engine driving a DeviceModel.

Builds an engine config whose ledger matches the device's physical pages (a
KV block = one arena page; layer_bytes = page-rounded image sizes from
ms_layer_pages), so the reference attach arithmetic (engine.cpp:273,
floor(freed / block_bytes)) and the arena agree exactly.
"""
from __future__ import annotations

import os

from . import morphsim as M
from .device import DeviceModel, layer_pages

GIB = 1 << 30
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sequence_file(num_layers: int) -> str:
    """LIS swap order produced offline by the reference profiler (configs/)."""
    p = os.path.join(ROOT, "configs", f"sequence_lis_{num_layers}.json")
    if not os.path.exists(p):
        p = os.path.join(ROOT, "configs", f"sequence_front_to_back_{num_layers}.json")
        M.save_sequence(M.baseline_sequence("front_to_back", num_layers), p)
    return p


def device_config(dev: DeviceModel, workload: dict, *, budget_gib: float = 24.0, reserve_gib: float = 4.0,
                  slo_ms: float = 2000.0, seed: int = 7, controller: dict | None = None) -> dict:
    shape = dev.shape
    pb = dev.page_bytes
    p16, p8, p4, p3 = (layer_pages(shape, b) for b in (16, 8, 4, 3))
    budget = int(budget_gib * GIB)
    if budget // pb > dev.desc.arena_pages:
        raise ValueError(f"budget {budget_gib} GiB exceeds the device arena ({dev.desc.arena_pages} pages)")
    cfg = {
        "seed": seed,
        "slo_ms": slo_ms,
        "model": {"num_layers": shape["L"],
                  "layer_bytes": {"full": p16 * pb, "q8": p8 * pb, "q4": p4 * pb, "q3": p3 * pb}},
        "kv": {"block_tokens": 16, "block_bytes": pb, "static_capacity_blocks": 0},
        "budget": {"device_bytes": budget, "reserve_bytes": int(reserve_gib * GIB)},
        "toy": {"num_layers": shape["L"]},
        "workload": workload,
        "sequence_file": sequence_file(shape["L"]),
    }
    if controller:
        cfg["controller"] = controller
    return cfg


def serve(dev: DeviceModel, cfg: dict, arm: str = "morph-performance", clock: str = "wall", trace=None):
    """Runs one arm on the GPU (real clock by default); returns (report, event_log).
    trace: this replica's shard of the workload (replicas.shard_trace)."""
    rep, log, _ = M.run_arm_full(cfg, arm, device=dev, clock=clock, trace=trace)
    return rep, log


def summary(rep: dict) -> dict:
    d = rep.get("device", {})
    return {
        "requests": rep["requests"],
        "p50_ttft_ms": rep["ttft_ms"]["p50"], "p95_ttft_ms": rep["ttft_ms"]["p95"],
        "p95_tpot_ms": rep["tpot_ms"]["p95"], "mean_tpot_ms": rep["tpot_ms"]["mean"],
        "slo_violations": rep["slo"]["violations"], "throughput_rps": rep["throughput_rps"],
        "sim_end_ms": rep["sim_end_ms"],
        "swap_events": rep["morph"]["swap_events"], "restore_events": rep["morph"]["restore_events"],
        "peak_quantized_layers": rep["morph"]["peak_quantized_layers"],
        "kv_static_blocks": rep["kv"]["static_capacity_blocks"], "kv_peak_blocks": rep["kv"]["peak_capacity_blocks"],
        "preemptions": rep["requests"]["preemptions"],
        "decode_tok_s": d.get("decode_tokens", 0.0) / (d["decode_ms"] / 1e3) if d.get("decode_ms") else None,
        "prefill_tok_s": d.get("prefill_tokens", 0) / (d["prefill_ms"] / 1e3) if d.get("prefill_ms") else None,
        "prefill_ms_total": d.get("prefill_ms"),
        "device_busy_ms": d.get("busy_ms"), "decode_steps": d.get("decode_steps"),
        "swap_upload_ms_total": d.get("swap_upload_ms"),
        "decode_steps_overlapping_uploads": d.get("decode_steps_overlap"),
        "exposed_swap_stall_ms_per_token": d.get("exposed_stall_ms_per_token"),
        # step time above the no-upload step model, as a fraction of all decode time
        "exposed_swap_stall_frac_of_decode": (d["exposed_swap_stall_ms"] / d["decode_ms"]
                                              if d.get("decode_ms") else None),
        "host_gap_ms": d.get("host_gap_ms"), "graph_captures": d.get("graph_captures"),
    }
