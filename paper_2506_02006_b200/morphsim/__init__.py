"""Drop-in ``morphsim`` API over the B200 host runtime.

Mirrors the reference package (proj/python/morphsim/__init__.py:1-73 and the
experiment layer proj/src/experiment.cpp): JSON configs with the same
defaults and validation, the same arms, ``run_arm`` / ``sweep`` /
``config_fingerprint`` returning the same report schema, plus the trace and
KV-pool objects.  The engine underneath is the C++ host runtime
(``paper_2506_02006_b200._core``) and, when ``device=`` is given, every
prefill / decode step / layer swap / KV resize also runs on the B200 through
include/morphserve.h.

Out of scope: the offline LIS profiler and the
CLI.  ``load_sequence`` consumes the sequence files the reference profiler
writes; ``baseline_sequence`` covers the front-to-back / back-to-front /
random orders.
"""
from __future__ import annotations

import copy
import json as _json
import os

from .. import _core

TraceEvent = _core.TraceEvent
Trace = _core.Trace
KvConfig = _core.KvConfig
KvBlockPool = _core.KvBlockPool
parse_trace = _core.parse_trace
serialize_trace = _core.serialize_trace
downscale = _core.downscale
synth_burst = _core.synth_burst
synth_gamma = _core.synth_gamma

ARMS = ("static-full", "static-quant", "morph-accuracy", "morph-performance")
GIB = 1 << 30


def _gib(x: float) -> int:
    return int(round(x * GIB))


# --------------------------------------------------------------- defaults
def _controller_defaults(mode: str, num_layers: int) -> dict:
    return dict(_core.controller_defaults(mode, num_layers))


def default_config() -> dict:
    """ExperimentConfig defaults (reference experiment.hpp:26-60 + struct defaults)."""
    return {
        "seed": 7,
        "downscale": 1.0,
        "quant_bits": 4,
        "slo_ms": 2000.0,
        "monitor_tick_ms": 100.0,
        "model": {"num_layers": 32,
                  "layer_bytes": {"full": _gib(0.4), "q8": _gib(0.2), "q4": _gib(0.1), "q3": _gib(0.075)}},
        "kv": {"block_tokens": 16, "block_bytes": 2 * 1024 * 1024, "static_capacity_blocks": 0},
        "budget": {"device_bytes": 24 * GIB, "reserve_bytes": 4 * GIB},
        "cost": {"prefill_ms_per_token": 0.02,
                 "decode_ms_per_layer": {"full": 0.3, "q8": 0.24, "q4": 0.18, "q3": 0.15},
                 "attn_ms_per_kv_block": 0.00005, "pcie_gib_per_s": 26.0, "swap_fixed_overhead_ms": 2.0,
                 "max_batch_tokens": 100000},
        "toy": {"seed": 7, "num_layers": 32, "hidden_dim": 16, "calibration_vectors": 32, "bits": 4,
                "random_baseline_seed": 1234, "weights": {"alpha1": 0.25, "alpha2": 0.25, "beta": 0.5}},
    }


class Config(dict):
    """A resolved experiment config (defaults applied, validated)."""


def _resolved(config) -> "Config":
    return config if isinstance(config, Config) else config_from_json(config)


def _merge(dst: dict, src: dict, keys) -> None:
    for k in keys:
        if k in src:
            dst[k] = src[k]


def config_from_json(doc) -> dict:
    """Resolved config (defaults applied, validated) -- reference experiment.cpp:88-179."""
    if isinstance(doc, str):
        doc = _json.loads(doc)
    cfg = default_config()
    _merge(cfg, doc, ["seed", "downscale", "quant_bits", "slo_ms", "monitor_tick_ms"])
    if "model" in doc:
        m = doc["model"]
        _merge(cfg["model"], m, ["num_layers"])
        if "layer_bytes" in m:
            _merge(cfg["model"]["layer_bytes"], m["layer_bytes"], ["full", "q8", "q4", "q3"])
    if "kv" in doc:
        _merge(cfg["kv"], doc["kv"], ["block_tokens", "block_bytes", "static_capacity_blocks"])
    if "budget" in doc:
        _merge(cfg["budget"], doc["budget"], ["device_bytes", "reserve_bytes"])
    if "cost" in doc:
        c = doc["cost"]
        _merge(cfg["cost"], c, ["prefill_ms_per_token", "attn_ms_per_kv_block", "pcie_gib_per_s",
                                "swap_fixed_overhead_ms", "max_batch_tokens"])
        if "decode_ms_per_layer" in c:
            _merge(cfg["cost"]["decode_ms_per_layer"], c["decode_ms_per_layer"], ["full", "q8", "q4", "q3"])
    L = cfg["model"]["num_layers"]
    ctl = {"accuracy": _controller_defaults("accuracy", L), "performance": _controller_defaults("performance", L)}
    keys = ["kv_trigger", "kv_low", "queue_trigger_ms", "hold_ms", "max_swapped_layers", "swap_step",
            "telemetry_window_ms", "target_bits"]
    for mode in ("accuracy", "performance"):
        if "controller" in doc and mode in doc["controller"]:
            _merge(ctl[mode], doc["controller"][mode], keys)
        ctl[mode]["target_bits"] = cfg["quant_bits"]
    cfg["controller"] = ctl
    if "toy" in doc:
        t = doc["toy"]
        _merge(cfg["toy"], t, ["seed", "num_layers", "hidden_dim", "calibration_vectors", "bits",
                               "random_baseline_seed"])
        if "weights" in t:
            _merge(cfg["toy"]["weights"], t["weights"], ["alpha1", "alpha2", "beta"])
    w = doc.get("workload", {})
    cfg["workload"] = {}
    if "trace_file" in w:
        cfg["workload"]["trace_file"] = w["trace_file"]
    if "synth" in w:
        s = {"seed": 0, "base_rps": 1.0, "burst_rps": 1.0, "burst_start_ms": 0, "burst_len_ms": 0, "total_ms": 0,
             "prompt_tokens": 1, "output_tokens": 1}
        _merge(s, w["synth"], list(s))
        cfg["workload"]["synth"] = s
    if "gamma" in w:  # extension: Gamma-renewal bursty arrivals (BASELINE.json config 3)
        g = {"seed": 0, "rps": 1.0, "shape": 0.25, "total_ms": 0, "prompt_tokens": 1, "output_tokens": 1}
        _merge(g, w["gamma"], list(g))
        cfg["workload"]["gamma"] = g
    if "sequence_file" in doc:
        cfg["sequence_file"] = doc["sequence_file"]
    validate(cfg)
    return Config(cfg)


def _engine_dict(cfg: dict) -> dict:
    lb = cfg["model"]["layer_bytes"]
    dm = cfg["cost"]["decode_ms_per_layer"]
    return {
        "num_layers": cfg["model"]["num_layers"],
        "layer_bytes": [lb["full"], lb["q8"], lb["q4"], lb["q3"]],
        "block_tokens": cfg["kv"]["block_tokens"], "block_bytes": cfg["kv"]["block_bytes"],
        "static_capacity_blocks": cfg["kv"]["static_capacity_blocks"],
        "device_bytes": cfg["budget"]["device_bytes"], "reserve_bytes": cfg["budget"]["reserve_bytes"],
        "prefill_ms_per_token": cfg["cost"]["prefill_ms_per_token"],
        "decode_ms_per_layer": [dm["full"], dm["q8"], dm["q4"], dm["q3"]],
        "attn_ms_per_kv_block": cfg["cost"]["attn_ms_per_kv_block"],
        "pcie_gib_per_s": cfg["cost"]["pcie_gib_per_s"],
        "swap_fixed_overhead_ms": cfg["cost"]["swap_fixed_overhead_ms"],
        "max_batch_tokens": cfg["cost"]["max_batch_tokens"],
        "slo_ms": cfg["slo_ms"], "monitor_tick_ms": cfg["monitor_tick_ms"],
    }


def validate(cfg: dict) -> None:
    """reference experiment.cpp:56-86 (ValueError == std::invalid_argument)."""
    e = _engine_dict(cfg)
    lb = e["layer_bytes"]
    if e["num_layers"] < 1:
        raise ValueError("model: num_layers must be >= 1")
    if any(b < 1 for b in lb):
        raise ValueError("model: layer byte sizes must be positive")
    if not (lb[0] >= lb[1] >= lb[2] >= lb[3]):
        raise ValueError("model: layer bytes must be non-increasing with precision")
    dm = e["decode_ms_per_layer"]
    if not (e["prefill_ms_per_token"] > 0):
        raise ValueError("cost: prefill rate must be > 0")
    if any(not (x > 0) for x in dm) or not (dm[0] >= dm[1] >= dm[2] >= dm[3]):
        raise ValueError("cost: decode cost must be positive and non-increasing as precision drops")
    if not (e["attn_ms_per_kv_block"] > 0) or not (e["pcie_gib_per_s"] > 0) or not (e["swap_fixed_overhead_ms"] > 0):
        raise ValueError("cost: attention, pcie and swap terms must be > 0")
    if e["max_batch_tokens"] < 1:
        raise ValueError("cost: max_batch_tokens must be >= 1")
    if not (e["slo_ms"] > 0) or not (e["monitor_tick_ms"] > 0):
        raise ValueError("engine: slo_ms and monitor tick must be > 0")
    if e["device_bytes"] < 1 or e["reserve_bytes"] < 0:
        raise ValueError("engine: invalid budget")
    if e["block_tokens"] < 1 or e["block_bytes"] < 1:
        raise ValueError("engine: invalid kv block geometry")
    L = e["num_layers"]
    acc, perf = cfg["controller"]["accuracy"], cfg["controller"]["performance"]
    _core.validate_controller(acc, L)
    _core.validate_controller(perf, L)
    if acc["max_swapped_layers"] > perf["max_swapped_layers"]:
        raise ValueError("accuracy mode may not swap more layers than performance mode")
    if acc["kv_trigger"] < perf["kv_trigger"]:
        raise ValueError("accuracy mode kv trigger must be >= performance mode's")
    if cfg["quant_bits"] not in (8, 4, 3):
        raise ValueError("quant_bits must be one of 8, 4, 3")
    if not (cfg["downscale"] > 0):
        raise ValueError("downscale factor must be > 0")
    w = cfg.get("workload", {})
    n = sum(k in w for k in ("trace_file", "synth", "gamma"))
    if n == 0:
        raise ValueError("workload requires either trace_file or synth parameters")
    if n > 1:
        raise ValueError("workload must name exactly one of trace_file or synth")
    t = cfg["toy"]
    if t["num_layers"] < 1 or t["hidden_dim"] < 2 or t["calibration_vectors"] < 1:
        raise ValueError("invalid toy model parameters")
    tw = t["weights"]
    if min(tw.values()) < 0 or all(v == 0 for v in tw.values()):
        raise ValueError("LIS weights must be non-negative and not all zero")
    if t["bits"] not in (8, 4, 3):
        raise ValueError("toy bits must be one of 8, 4, 3")


# ---------------------------------------------------------- fingerprint
def _jnum(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, int):
        return str(v)
    r = repr(float(v))
    if "e" in r:  # nlohmann: mantissa + 'e' + sign + 2-digit exponent
        mant, ex = r.split("e")
        sign = "-" if ex.startswith("-") else "+"
        ex = ex.lstrip("+-").rjust(2, "0")
        return f"{mant}e{sign}{ex}"
    return r


def _canon(x) -> str:
    if isinstance(x, dict):
        return "{" + ",".join(_json.dumps(k) + ":" + _canon(x[k]) for k in sorted(x)) + "}"
    if isinstance(x, (list, tuple)):
        return "[" + ",".join(_canon(v) for v in x) + "]"
    if isinstance(x, str):
        return _json.dumps(x)
    return _jnum(x)


def canonical_config(cfg: dict) -> str:
    """config_to_json + compact dump (reference experiment.cpp:193-253)."""
    c = copy.deepcopy(dict(cfg))
    for mode in ("accuracy", "performance"):
        c["controller"][mode] = {k: c["controller"][mode][k] for k in
                                 ["kv_trigger", "kv_low", "queue_trigger_ms", "hold_ms", "max_swapped_layers",
                                  "swap_step", "telemetry_window_ms", "target_bits"]}
    for k in ("downscale", "slo_ms", "monitor_tick_ms"):
        c[k] = float(c[k])
    for k in ("prefill_ms_per_token", "attn_ms_per_kv_block", "pcie_gib_per_s", "swap_fixed_overhead_ms"):
        c["cost"][k] = float(c["cost"][k])
    for k in c["cost"]["decode_ms_per_layer"]:
        c["cost"]["decode_ms_per_layer"][k] = float(c["cost"]["decode_ms_per_layer"][k])
    for mode in ("accuracy", "performance"):
        for k in ("kv_trigger", "kv_low", "queue_trigger_ms", "hold_ms", "telemetry_window_ms"):
            c["controller"][mode][k] = float(c["controller"][mode][k])
    for k in c["toy"]["weights"]:
        c["toy"]["weights"][k] = float(c["toy"]["weights"][k])
    if "synth" in c.get("workload", {}):
        for k in ("base_rps", "burst_rps"):
            c["workload"]["synth"][k] = float(c["workload"]["synth"][k])
    return _canon(c)


def fnv1a64(data: str) -> int:
    h = 0xCBF29CE484222325
    for b in data.encode():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def config_fingerprint(config) -> str:
    return f"{fnv1a64(canonical_config(_resolved(config))):016x}"


# ------------------------------------------------------------ sequences
def load_sequence(path: str) -> dict:
    """Swap-order file written by the reference profiler (profiler.cpp:216-257)."""
    try:
        with open(path) as f:
            doc = _json.load(f)
    except OSError as e:
        raise RuntimeError(f"cannot open sequence file: {path}") from e
    except ValueError as e:
        raise RuntimeError(f"malformed sequence file {path}: {e}") from e
    try:
        order = [int(x) for x in doc["order"]]
        lis = [float(x) for x in doc["per_step_lis"]]
        bits = int(doc["bits"])
        kind = doc["provenance"]
        declared = int(doc["L"])
    except (KeyError, TypeError, ValueError) as e:
        raise RuntimeError(f"malformed sequence file {path}: {e}") from e
    if declared != len(order):
        raise RuntimeError("sequence file L does not match order length")
    if sorted(order) != list(range(len(order))):
        raise RuntimeError(f"sequence file {path} is not a permutation of [0, L)")
    if len(lis) != len(order):
        raise RuntimeError(f"sequence file {path} has mismatched per_step_lis length")
    return {"order": order, "per_step_lis": lis, "bits": bits, "kind": kind,
            "weights": doc.get("weights", {}), "random_seed": doc.get("random_seed", 0)}


def baseline_sequence(kind: str, num_layers: int, seed: int = 0, bits: int = 4) -> dict:
    if num_layers < 1:
        raise ValueError("baseline_sequence: num_layers must be >= 1")
    order = list(range(num_layers))
    if kind == "back_to_front":
        order.reverse()
    elif kind == "random":
        order = _mt_shuffle(order, seed)
    elif kind != "front_to_back":
        raise ValueError(f"unknown sequence kind: {kind}")
    return {"order": order, "per_step_lis": [0.0] * num_layers, "bits": bits, "kind": kind,
            "weights": {"alpha1": 0.25, "alpha2": 0.25, "beta": 0.5}, "random_seed": seed}


def _mt_shuffle(v, seed: int):
    """Fisher-Yates with the reference Rng (random.hpp:34-50: mt19937_64 + rejection)."""
    mt = _MT19937_64(seed)
    v = list(v)
    for i in range(len(v), 1, -1):
        n = i
        limit = 0xFFFFFFFFFFFFFFFF - 0xFFFFFFFFFFFFFFFF % n
        while True:
            x = mt.next()
            if x < limit:
                break
        j = x % n
        v[i - 1], v[j] = v[j], v[i - 1]
    return v


class _MT19937_64:
    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def next(self) -> int:
        if self.i >= 312:
            for k in range(312):
                y = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                x = self.mt[(k + 156) % 312] ^ (y >> 1)
                if y & 1:
                    x ^= 0xB5026F5AA96619E9
                self.mt[k] = x
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def save_sequence(seq: dict, path: str) -> None:
    doc = {"version": 1, "L": len(seq["order"]), "bits": seq.get("bits", 4),
           "weights": seq.get("weights", {"alpha1": 0.25, "alpha2": 0.25, "beta": 0.5}),
           "provenance": seq.get("kind", "front_to_back"), "order": list(seq["order"]),
           "per_step_lis": list(seq.get("per_step_lis", [0.0] * len(seq["order"])))}
    if doc["provenance"] == "random":
        doc["random_seed"] = seq.get("random_seed", 0)
    with open(path, "w") as f:
        f.write(_json.dumps(doc, indent=2) + "\n")


# -------------------------------------------------------------- workloads
def resolve_workload(cfg: dict):
    w = cfg["workload"]
    if "trace_file" in w:
        t = parse_trace(w["trace_file"])
    elif "synth" in w:
        s = w["synth"]
        t = synth_burst(s["seed"], s["base_rps"], s["burst_rps"], s["burst_start_ms"], s["burst_len_ms"],
                        s["total_ms"], s["prompt_tokens"], s["output_tokens"])
    else:
        g = w["gamma"]
        t = synth_gamma(g["seed"], g["rps"], g["shape"], g["total_ms"], g["prompt_tokens"], g["output_tokens"])
    if cfg["downscale"] != 1.0:
        t = downscale(t, cfg["downscale"])
    return t


def arm_spec(cfg: dict, arm: str) -> dict:
    """reference experiment.cpp:292-315."""
    L = cfg["model"]["num_layers"]
    if arm == "static-full":
        return {"label": arm, "initial_bits": 16, "controller": None, "sequence": None}
    if arm == "static-quant":
        return {"label": arm, "initial_bits": cfg["quant_bits"], "controller": None, "sequence": None}
    if arm in ("morph-accuracy", "morph-performance"):
        mode = "accuracy" if arm == "morph-accuracy" else "performance"
        ctl = dict(cfg["controller"][mode])
        ctl["enabled"] = True
        ctl["mode"] = mode
        if "sequence_file" not in cfg:
            raise ValueError("morph arm requires sequence_file in the config")
        seq = load_sequence(cfg["sequence_file"])
        if len(seq["order"]) != L:
            raise ValueError("swap sequence layer count does not match engine model")
        return {"label": arm, "initial_bits": 16, "controller": ctl, "sequence": seq["order"]}
    raise ValueError(f"unknown arm: {arm}")


def _run(cfg: dict, arm: str, device=None, clock: str = "virtual", record: bool = False, trace=None):
    spec = arm_spec(cfg, arm)
    if trace is None:
        trace = resolve_workload(cfg)
    dev_ptr, vocab = 0, 0
    if device is not None:
        dev_ptr = device.h.value if hasattr(device.h, "value") else int(device.h)
        vocab = device.shape["V"]
    out = _core.run_simulation(_engine_dict(cfg), spec, trace, int(cfg["seed"]), dev_ptr, vocab, clock, record)
    report = _json.loads(out["report_json"])
    report["fingerprint"] = config_fingerprint(cfg)
    if record:
        report["device_calls"] = out.get("device_calls", [])
    return report, out["log"], out["timeline_csv"]


def run_arm(config, arm: str, out_dir: str = "", device=None, clock: str = "virtual") -> dict:
    """Serves the configured workload under one arm; returns the report dict.

    device: a ``paper_2506_02006_b200.device.DeviceModel`` -- every step runs on
    the GPU.  clock: "virtual" (reference cost model durations, bit-exact event
    log), "device" (measured GPU durations advance a simulated clock) or
    "wall" (real clock: arrivals released on time, swaps polled at event
    boundaries while decode continues).
    """
    cfg = _resolved(config)
    report, log, timeline = _run(cfg, arm, device, clock)
    if out_dir:
        os.makedirs(out_dir, exist_ok=True)
        with open(os.path.join(out_dir, f"report_{arm}.json"), "w") as f:
            f.write(_json.dumps(report, indent=2) + "\n")
        with open(os.path.join(out_dir, f"timeline_{arm}.csv"), "w") as f:
            f.write(timeline)
        with open(os.path.join(out_dir, f"events_{arm}.log"), "w") as f:
            f.write(log)
    return report


def run_arm_full(config, arm: str, device=None, clock: str = "virtual", record: bool = False, trace=None):
    """(report, event_log_text, timeline_csv) -- for parity checks; record=True
    adds report["device_calls"] (every prefill/decode launch with its rows and
    the per-layer precision at launch) for replay against the CPU oracle.
    trace: serve this Trace instead of the config's workload (e.g. one
    replica's round-robin shard, replicas.shard_trace).  clock: "virtual",
    "device" (GPU-time simulation) or "wall" (real clock, swaps overlapped)."""
    return _run(_resolved(config), arm, device, clock, record, trace)


def sweep(config, rps_list, arms) -> dict:
    """Homogeneous-rate sweep (reference experiment.cpp:372-402)."""
    cfg = config_from_json(config)
    if not rps_list:
        raise ValueError("sweep requires a non-empty rps list")
    if "synth" not in cfg["workload"]:
        raise ValueError("sweep requires synth workload parameters")
    if any(not (r > 0) for r in rps_list):
        raise ValueError("sweep rates must be > 0")
    rows, sat = [], {}
    for arm in arms:
        first = None
        for rps in rps_list:
            point = Config(copy.deepcopy(dict(cfg)))
            point["workload"]["synth"]["base_rps"] = rps
            point["workload"]["synth"]["burst_rps"] = rps
            rep, _, _ = _run(point, arm)
            p95 = rep["ttft_ms"]["p95"]
            rows.append({"rps": rps, "arm": arm, "p95_ttft_ms": p95, "slo_violations": rep["slo"]["violations"],
                         "throughput_rps": rep["throughput_rps"]})
            if first is None and p95 is not None and p95 > cfg["slo_ms"]:
                first = rps
        sat[arm] = first
    return {"rows": rows, "saturation_rps": sat}


__all__ = [
    "TraceEvent", "Trace", "KvConfig", "KvBlockPool", "parse_trace", "serialize_trace", "downscale",
    "synth_burst", "synth_gamma", "config_from_json", "config_fingerprint", "canonical_config", "load_sequence",
    "save_sequence", "baseline_sequence", "resolve_workload", "arm_spec", "run_arm", "run_arm_full", "sweep",
]
