"""Host runtime parity: the C++ engine / KV pool / controller driven through the
drop-in morphsim API must reproduce the reference simulator byte for byte
(event logs, timelines, reports) -- SURVEY 8(a) rows a2-a10, a13.

Golden logs/reports were produced by the unmodified reference
(tests/golden/make_golden.py); when oracle/_ref is built the same runs are
also compared live.
"""
import hashlib
import json
import os
import tempfile

import pytest

import oracle as O
from paper_2506_02006_b200 import morphsim as M
from tests.scenarios import SCENARIOS

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REF_CFG = os.path.join(GOLD, "example.json")


def _with_sequence(cfg, arm, d):
    cfg = dict(cfg)
    if arm.startswith("morph"):
        path = os.path.join(d, "seq.json")
        M.save_sequence(M.baseline_sequence("front_to_back", cfg["model"]["num_layers"]), path)
        cfg["sequence_file"] = path
    return cfg


@pytest.mark.parametrize("name", sorted(SCENARIOS))
def test_scenario_matches_golden(name, tmp_path):
    cfg, arm = SCENARIOS[name]
    cfg = _with_sequence(cfg, arm, str(tmp_path))
    rep, log, _ = M.run_arm_full(cfg, arm)
    gold = json.load(open(os.path.join(GOLD, "engine_index.json")))[name]
    assert hashlib.sha256(log.encode()).hexdigest() == gold["sha256"]
    assert log == open(os.path.join(GOLD, f"engine_{name}.log")).read()
    rep.pop("device")
    rep.pop("fingerprint")
    assert rep == gold["report"]


needs_ref = pytest.mark.skipif(not O.have_ref_core(), reason="oracle/_ref not built (make -C oracle ref)")


def _ref_run(ref, cfg, arm, d):
    rep = json.loads(ref.run_arm(json.dumps(cfg), arm, d))
    return rep, open(os.path.join(d, f"events_{arm}.log")).read(), open(os.path.join(d, f"timeline_{arm}.csv")).read()


@needs_ref
def test_acceptance_burst_all_arms_bit_exact(tmp_path):
    """The reference acceptance burst (configs/example.json, LIS sequence)."""
    ref = O.ref_core()
    seq = str(tmp_path / "seq.json")
    model = ref.build_model(7, 32, 16)
    ref.save_sequence(ref.greedy_sequence(model, ref.calibration_batch(ref.calibration_seed(7), 32, 16)), seq)
    cfg = json.load(open(REF_CFG))
    cfg["sequence_file"] = seq
    for arm in M.ARMS:
        r_ref, log_ref, tl_ref = _ref_run(ref, cfg, arm, str(tmp_path / arm))
        rep, log, tl = M.run_arm_full(cfg, arm)
        rep.pop("device")
        assert log == log_ref, arm
        assert tl == tl_ref, arm
        assert rep == r_ref, arm


@needs_ref
def test_random_scenarios_bit_exact(tmp_path):
    """30 random engines x 4 arms (reference test_engine.cpp:518-587 style)."""
    import numpy as np
    ref = O.ref_core()
    rng = np.random.default_rng(987654321)
    MiB = 1 << 20
    for sc in range(30):
        L = int(rng.integers(2, 9))
        full = int(rng.integers(32, 128)) * MiB
        bt = int(8 << rng.integers(0, 3))
        bb = int(MiB << rng.integers(0, 3))
        cap = int(rng.integers(8, 72))
        dev = L * full + 64 * MiB + cap * bb + int(rng.integers(0, 128)) * MiB
        rows, t = [], 0
        for _ in range(int(rng.integers(5, 25))):
            t += int(rng.integers(0, 50))
            rows.append((t, int(rng.integers(1, 200)), int(rng.integers(1, 60))))
        tr = tmp_path / f"t{sc}.csv"
        tr.write_text("".join(f"{a},{p},{o}\n" for a, p, o in rows))
        cfg = {"seed": 42, "model": {"num_layers": L, "layer_bytes": {"full": full, "q8": full // 2, "q4": full // 4,
                                                                         "q3": full // 8}},
               "kv": {"block_tokens": bt, "block_bytes": bb, "static_capacity_blocks": cap},
               "budget": {"device_bytes": dev, "reserve_bytes": 64 * MiB},
               "cost": {"prefill_ms_per_token": float(0.01 + 0.1 * rng.random()), "attn_ms_per_kv_block": 0.0001},
               "toy": {"num_layers": L}, "workload": {"trace_file": str(tr)}}
        seq = tmp_path / f"s{sc}.json"
        ref.save_sequence(ref.baseline_sequence("front_to_back", L, 0, 4), str(seq))
        cfg["sequence_file"] = str(seq)
        for arm in M.ARMS:
            r_ref, log_ref, tl_ref = _ref_run(ref, cfg, arm, str(tmp_path / f"{sc}_{arm}"))
            rep, log, tl = M.run_arm_full(cfg, arm)
            rep.pop("device")
            assert log == log_ref, (sc, arm)
            assert tl == tl_ref, (sc, arm)
            assert rep == r_ref, (sc, arm)


@needs_ref
def test_fingerprint_and_sweep_match_reference():
    ref = O.ref_core()
    cfg = json.load(open(REF_CFG))
    cfg.pop("sequence_file")
    assert M.config_fingerprint(cfg) == ref.config_fingerprint(json.dumps(cfg))
    cfg["workload"]["synth"].update(total_ms=8000, burst_start_ms=1000, burst_len_ms=2000)
    ours = M.sweep(cfg, [8, 24, 40], ["static-full", "static-quant"])
    theirs = json.loads(ref.sweep(json.dumps(cfg), [8.0, 24.0, 40.0], ["static-full", "static-quant"]))
    assert ours["rows"] == theirs["rows"]
    assert ours["saturation_rps"] == theirs["saturation_rps"]


def test_validation_errors_are_value_errors():
    cfg = json.load(open(REF_CFG))
    bad = json.loads(json.dumps(cfg))
    bad["controller"]["accuracy"]["max_swapped_layers"] = 20
    with pytest.raises(ValueError):
        M.config_from_json(bad)
    bad = json.loads(json.dumps(cfg))
    bad["quant_bits"] = 5
    with pytest.raises(ValueError):
        M.config_from_json(bad)
    bad = json.loads(json.dumps(cfg))
    bad["workload"]["trace_file"] = "x.csv"
    with pytest.raises(ValueError):
        M.config_from_json(bad)
    with pytest.raises(ValueError):
        M.run_arm({k: v for k, v in cfg.items() if k != "sequence_file"}, "morph-performance")


def test_morph_without_pressure_equals_static_full(tmp_path):
    """Reference test_engine.cpp:297-314 / acceptance criterion 7."""
    cfg, _ = SCENARIOS["mixed_quant"]
    cfg = _with_sequence(cfg, "morph-performance", str(tmp_path))
    a = M.run_arm(cfg, "static-full")
    b = M.run_arm(cfg, "morph-performance")
    for r in (a, b):
        r.pop("arm")
    assert a == b


def test_trace_tools():
    t = M.synth_burst(9, 10, 40, 500, 500, 2000, 32, 8)
    assert len(t.events) > 0
    again = M.synth_burst(9, 10, 40, 500, 500, 2000, 32, 8)
    assert [e.arrival_ms for e in again.events] == [e.arrival_ms for e in t.events]
    tr = M.Trace()
    tr.events = [M.TraceEvent(0, 8, 4), M.TraceEvent(10, 8, 4), M.TraceEvent(20, 8, 4)]
    assert [e.arrival_ms for e in M.downscale(tr, 4.75).events] == [0, 48, 95]  # test_workload.cpp:91-101
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "t.csv")
        M.serialize_trace(t, p)
        back = M.parse_trace(p)
        assert [(e.arrival_ms, e.prompt_tokens, e.output_tokens) for e in back.events] == \
               [(e.arrival_ms, e.prompt_tokens, e.output_tokens) for e in t.events]
    g = M.synth_gamma(101, 20.0, 0.25, 60000, 256, 64)
    gaps = [b.arrival_ms - a.arrival_ms for a, b in zip(g.events, g.events[1:])]
    import numpy as np
    cv = float(np.std(gaps) / np.mean(gaps))
    assert 1.5 < cv < 2.6  # shape 0.25 => CV 2
    assert 0.6 < len(g.events) / (20.0 * 60) < 1.4


@needs_ref
def test_trace_generators_match_reference():
    ref = O.ref_core()
    for args in [(9, 10.0, 40.0, 500, 500, 2000, 32, 8), (101, 6.0, 33.0, 5000, 12000, 40000, 512, 256),
                 (3, 4.0, 4.0, 0, 0, 4000, 64, 16)]:
        a = [(e.arrival_ms, e.prompt_tokens, e.output_tokens) for e in M.synth_burst(*args).events]
        b = [(e.arrival_ms, e.prompt_tokens, e.output_tokens) for e in ref.synth_burst(*args).events]
        assert a == b
    seq_ref = ref.baseline_sequence("random", 32, 1234, 4).order
    assert M.baseline_sequence("random", 32, 1234)["order"] == list(seq_ref)
