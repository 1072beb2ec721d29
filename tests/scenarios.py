"""Small engine scenarios shared by the parity tests and tests/golden/make_golden.py.

Each mirrors a case of the reference's own engine tests
(proj/tests/test_engine.cpp) expressed as a morphsim JSON config + arm.
"""
import os

MiB = 1 << 20
GiB = 1 << 30
TRACES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "traces")


def small_config(trace, **over):
    """test_engine.cpp:16-30 small_config()."""
    cfg = {
        "seed": 5,
        "model": {"num_layers": 2, "layer_bytes": {"full": 512 * MiB, "q8": 256 * MiB, "q4": 128 * MiB,
                                                   "q3": 96 * MiB}},
        "kv": {"block_tokens": 16, "block_bytes": 2 * MiB, "static_capacity_blocks": 1024},
        "budget": {"device_bytes": 8 * GiB, "reserve_bytes": 1 * GiB},
        "cost": {"prefill_ms_per_token": 0.05, "decode_ms_per_layer": {"full": 0.3, "q8": 0.24, "q4": 0.18,
                                                                         "q3": 0.15},
                 "attn_ms_per_kv_block": 0.0001},
        "slo_ms": 2000.0,
        "toy": {"num_layers": 2},
        "workload": {"trace_file": os.path.join(TRACES, trace)},
    }
    for k, v in over.items():
        if isinstance(v, dict) and isinstance(cfg.get(k), dict):
            cfg[k] = {**cfg[k], **v}
        else:
            cfg[k] = v
    return cfg


def _morph8(trace, ctl, **over):
    return small_config(
        trace,
        model={"num_layers": 8, "layer_bytes": {"full": 128 * MiB, "q8": 64 * MiB, "q4": 32 * MiB, "q3": 24 * MiB}},
        kv={"block_tokens": 16, "block_bytes": 2 * MiB, "static_capacity_blocks": 40},
        budget={"device_bytes": 4 * GiB, "reserve_bytes": 512 * MiB},
        controller={"performance": ctl, "accuracy": {"kv_trigger": 0.95, "max_swapped_layers": 2}},
        toy={"num_layers": 8}, **over)


SCENARIOS = {
    # test_engine.cpp:316-374
    "pressure": (_morph8("pressure.csv", {"kv_trigger": 0.6, "kv_low": 0.5, "hold_ms": 200.0,
                                          "max_swapped_layers": 4, "swap_step": 2},
                         cost={"prefill_ms_per_token": 0.05, "attn_ms_per_kv_block": 0.00005}),
                 "morph-performance"),
    # test_engine.cpp:376-416 (swaps land mid-step)
    "step_boundary": (_morph8("step_boundary.csv", {"kv_trigger": 0.6, "kv_low": 0.3, "max_swapped_layers": 8,
                                                    "swap_step": 2},
                              cost={"prefill_ms_per_token": 0.05,
                                    "decode_ms_per_layer": {"full": 1.0, "q8": 0.8, "q4": 0.6, "q3": 0.5},
                                    "attn_ms_per_kv_block": 0.0001}),
                      "morph-performance"),
    # test_engine.cpp:418-476 (deferred detach before restore)
    "deferred_detach": (small_config(
        "deferred_detach.csv",
        model={"num_layers": 4, "layer_bytes": {"full": 96 * MiB, "q8": 48 * MiB, "q4": 24 * MiB, "q3": 18 * MiB}},
        kv={"block_tokens": 16, "block_bytes": 2 * MiB, "static_capacity_blocks": 30},
        budget={"device_bytes": 640 * MiB, "reserve_bytes": 64 * MiB},
        cost={"prefill_ms_per_token": 0.05, "decode_ms_per_layer": {"full": 2.0, "q8": 1.8, "q4": 1.6, "q3": 1.5},
              "attn_ms_per_kv_block": 0.0001},
        controller={"performance": {"kv_trigger": 0.7, "kv_low": 0.5, "hold_ms": 100.0, "max_swapped_layers": 1,
                                    "swap_step": 1},
                    "accuracy": {"kv_trigger": 0.95, "max_swapped_layers": 1}},
        toy={"num_layers": 4}), "morph-performance"),
    # test_engine.cpp:216-244
    "preempt": (small_config("preempt.csv", kv={"block_tokens": 16, "block_bytes": 2 * MiB,
                                                 "static_capacity_blocks": 6}), "static-full"),
    # test_engine.cpp:259-280
    "fifo": (small_config("fifo.csv", kv={"block_tokens": 16, "block_bytes": 2 * MiB, "static_capacity_blocks": 8}),
             "static-full"),
    # test_engine.cpp:246-257
    "unserviceable": (small_config("unserviceable.csv", kv={"block_tokens": 16, "block_bytes": 2 * MiB,
                                                             "static_capacity_blocks": 8}), "static-full"),
    # test_engine.cpp:173-205
    "mixed_quant": (small_config("mixed.csv"), "static-quant"),
}
