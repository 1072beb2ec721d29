"""The serving engine driving the B200 (virtual clock): the event log / block
tables must be byte-identical to the CPU-only run (and to the reference when
oracle/_ref is built), and every token the GPU generated -- across prefills,
re-prefills after preemption, continuous-batching decode steps, layer swaps to
W4 and back, KV attach/detach -- must be what the CPU oracle predicts when it
replays the same launches with the same per-layer precision (teacher forced;
near ties within the bf16 logit tolerance are allowed and counted).
"""
import json
import os

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

TINY = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024)
PB = 16 * 4 * 2 * 2 * 64 * 2  # page = one KV block (all layers) = 32 KiB


def tiny_config(trace_path, seq_path, static_blocks=40):
    return {
        "seed": 11,
        "model": {"num_layers": 4, "layer_bytes": {"full": 48 * PB, "q8": 16 * PB, "q4": 16 * PB, "q3": 16 * PB}},
        "kv": {"block_tokens": 16, "block_bytes": PB, "static_capacity_blocks": static_blocks},
        "budget": {"device_bytes": (4 * 48 + static_blocks + 40) * PB, "reserve_bytes": 40 * PB},
        "cost": {"prefill_ms_per_token": 0.05, "attn_ms_per_kv_block": 0.0001},
        "controller": {"performance": {"kv_trigger": 0.6, "kv_low": 0.4, "hold_ms": 50.0, "max_swapped_layers": 2,
                                       "swap_step": 1},
                       "accuracy": {"kv_trigger": 0.9, "max_swapped_layers": 1}},
        "toy": {"num_layers": 4},
        "workload": {"trace_file": trace_path},
        "sequence_file": seq_path,
    }


def _replay_on_oracle(cfg, dev, calls, min_checked=300, shape=TINY):
    """Replays every recorded device launch on the CPU oracle with the same
    per-layer precision; every generated token must match (near ties allowed)."""
    from paper_2506_02006_b200 import morphsim as M
    from paper_2506_02006_b200 import _core
    from paper_2506_02006_b200.morphsim import resolve_workload
    trace = resolve_workload(M.config_from_json(cfg))
    n_req = len(trace.events)
    hist = {r: dev.hist_read(r, 0, trace.events[r].prompt_tokens + trace.events[r].output_tokens)
            for r in range(n_req)}
    for r in range(n_req):
        P = trace.events[r].prompt_tokens
        assert np.array_equal(hist[r][:P], np.array(_core.synthetic_prompt(cfg["seed"], r, P, shape["V"])))
    model = O.RefModel(dict(shape, max_pos=256), 7)
    seqs, checked, ties = {}, 0, []
    bits_now = [16] * 4

    def set_bits(bits):
        for l, b in enumerate(bits):
            if bits_now[l] != b:
                model.set_precision(l, b)
                bits_now[l] = b

    for c in calls:
        set_bits(c["bits"])
        if c["kind"] == "P":
            r, n = c["reqs"][0], c["pos"][0]
            seqs[r] = model.new_seq(256)  # (re-)prefill rebuilds the whole KV
            nxt, lg = model.prefill(seqs[r], hist[r][:n])
            pairs = [(r, n, nxt, lg)]
        else:
            toks = [hist[r][p] for r, p in zip(c["reqs"], c["pos"])]
            for r, p in zip(c["reqs"], c["pos"]):
                assert O.lib().ref_seq_len(seqs[r]) == p  # KV footprint = position of the input token
            nxt, lg = model.forward([seqs[r] for r in c["reqs"]], toks)
            pairs = [(r, p + 1, nxt[i], lg[i]) for i, (r, p) in enumerate(zip(c["reqs"], c["pos"]))]
        for r, at, rtok, rlog in pairs:
            if at >= len(hist[r]):
                continue
            g = int(hist[r][at])
            checked += 1
            if g != int(rtok):
                margin = float(rlog[rtok] - rlog[g])
                assert margin <= 2e-3 * float(np.max(np.abs(rlog))), (c, r, at, margin)
                ties.append((r, at, margin))
    assert checked >= min_checked
    assert len(ties) <= 0.02 * checked, ties
    model.close()




@pytest.fixture(scope="module")
def setup(tmp_path_factory):
    from paper_2506_02006_b200 import morphsim as M
    from paper_2506_02006_b200.device import DeviceModel, layer_pages
    assert layer_pages(TINY, 16) == 48 and layer_pages(TINY, 4) == 16
    d = tmp_path_factory.mktemp("eng")
    trace = d / "trace.csv"
    trace.write_text("".join(f"{i * 3},{40 + (i % 3) * 8},{24 + (i % 4) * 4}\n" for i in range(14)) +
                     "".join(f"{400 + i * 40},{32},{16}\n" for i in range(6)))
    seq = str(d / "seq.json")
    M.save_sequence(M.baseline_sequence("back_to_front", 4), seq)
    cfg = tiny_config(str(trace), seq)
    dev = DeviceModel(TINY, max_batch=32, max_prefill_tokens=128, max_pos=128, arena_pages=(4 * 48 + 40 + 40) + 32)
    dev.weights_synthetic(7)
    yield M, cfg, dev
    dev.close()


def test_device_backed_run_is_bit_exact_and_tokens_match_oracle(setup):
    M, cfg, dev = setup
    rep_cpu, log_cpu, tl_cpu = M.run_arm_full(cfg, "morph-performance")
    rep, log, tl = M.run_arm_full(cfg, "morph-performance", device=dev, record=True)
    assert log == log_cpu and tl == tl_cpu
    calls = rep.pop("device_calls")
    for r in (rep, rep_cpu):
        r.pop("device")
    assert rep == rep_cpu
    assert rep["morph"]["swap_events"] >= 1 and rep["kv"]["peak_capacity_blocks"] > 40
    assert "KV_ATTACH" in log
    if O.have_ref_core():
        ref = O.ref_core()
        import tempfile
        with tempfile.TemporaryDirectory() as td:
            r_ref = json.loads(ref.run_arm(json.dumps(cfg), "morph-performance", td))
            assert open(os.path.join(td, "events_morph-performance.log")).read() == log
        rep.pop("fingerprint")
        r_ref.pop("fingerprint")
        assert rep == r_ref

    _replay_on_oracle(cfg, dev, calls)


def test_device_clock_run_measures_real_time(setup):
    M, cfg, dev = setup
    rep, log, _ = M.run_arm_full(cfg, "morph-performance", device=dev, clock="device")
    assert rep["requests"]["completed"] == rep["requests"]["total"]
    d = rep["device"]
    assert d["decode_steps"] > 0 and d["decode_ms"] > 0 and d["prefill_ms"] > 0
    # durations in the log are the measured GPU times, not the cost model's
    assert rep["ttft_ms"]["p95"] is not None


def test_wall_clock_run_overlaps_swaps_and_matches_oracle(setup):
    """ClockMode::kWall: arrivals released on the wall clock, swaps polled at
    event boundaries (never waited on), every generated token still what the
    oracle predicts for the precision each launch ran at."""
    M, cfg, dev = setup
    rep, log, _ = M.run_arm_full(cfg, "morph-performance", device=dev, clock="wall", record=True)
    calls = rep.pop("device_calls")
    assert rep["requests"]["completed"] == rep["requests"]["total"]
    d = rep["device"]
    assert d["decode_steps"] > 0 and d["host_gap_ms"] >= 0.0 and d["exposed_stall_ms_per_token"] >= 0.0
    if rep["morph"]["swap_events"]:
        assert "done_at=poll" in log and "SWAP_DONE" in log
    # wall-clock TTFT includes the (real) arrival spacing: the last arrival is at 600 ms
    assert rep["sim_end_ms"] >= 600.0
    _replay_on_oracle(cfg, dev, calls, min_checked=200)


def test_swap_commit_keeps_captured_graphs():
    """Page tables are read from device memory: a swap commit does not drop the
    captured decode graphs; returning to a precision vector already captured
    replays its graph (no new capture) and still matches the oracle."""
    from paper_2506_02006_b200.device import DeviceModel
    dev = DeviceModel(TINY, max_batch=4, max_prefill_tokens=64, max_pos=128, arena_pages=300)
    ref = O.RefModel(dict(TINY, max_pos=128), 7)
    try:
        dev.weights_synthetic(7)
        dev.hist_reserve(2, 128)
        dev.kv_attach(0, 16)
        table = np.arange(16, dtype=np.int64).reshape(2, 8)
        prompts = (np.arange(2 * 16, dtype=np.int32).reshape(2, 16) * 53) % TINY["V"]
        seqs = [ref.new_seq(128) for _ in range(2)]
        toks = []
        for b in range(2):
            dev.hist_write(b, 0, prompts[b])
            toks.append(dev.prefill(b, 16, table[b])[0])
            ref.prefill(seqs[b], prompts[b])
        toks = np.array(toks, np.int32)
        pos = np.full(2, 16, np.int32)

        def steps(k):
            nonlocal toks, pos
            for _ in range(k):
                got, lg = dev.decode(np.arange(2), pos, table, tokens=toks, want_logits=True)
                rt, rl = ref.forward(seqs, toks)
                for b in range(2):
                    assert np.max(np.abs(lg[b] - rl[b])) <= 2e-2 * np.max(np.abs(rl[b]))
                toks = rt.astype(np.int32)
                pos = pos + 1

        def swap(layer, bits):
            t = dev.swap_begin(layer, bits)
            dev.swap_wait(t)
            dev.swap_commit(t)
            ref.set_precision(layer, bits)

        # a step shape is captured on its second sighting per staging slot (ring of 3)
        steps(6)
        c0 = dev.lib.ms_graph_captures(dev.h)
        swap(0, 4)
        steps(6)
        c1 = dev.lib.ms_graph_captures(dev.h)
        swap(0, 16)
        steps(6)
        c2 = dev.lib.ms_graph_captures(dev.h)
        assert c1 > c0 and c2 == c1, (c0, c1, c2)
    finally:
        ref.close()
        dev.close()


@pytest.mark.parametrize("bits", [8, 3])
def test_engine_swaps_to_q8_and_q3_levels(tmp_path, bits):
    """Controller target_bits 8 / 3 (config quant_bits, reference
    experiment.cpp:92,139-140; toy_model.hpp:26): the engine's swaps upload
    real Q8 / Q3 images and carve what they free into KV blocks; the event log
    stays byte-identical to the CPU-only run and every generated token is what
    the oracle predicts at that precision.  Tiny shape with 4 KV heads: 64 KiB
    pages hold three 16640-B Q8 chunks, so a Q8 layer is smaller than BF16."""
    from paper_2506_02006_b200 import morphsim as M
    from paper_2506_02006_b200.device import DeviceModel, layer_pages, page_bytes
    shape = dict(TINY, KVH=4)
    pb = page_bytes(shape)
    pages = {b: layer_pages(shape, b) for b in (16, 8, 4, 3)}
    assert pages[16] > pages[8] > pages[4] == pages[3]
    trace = tmp_path / "trace.csv"
    trace.write_text("".join(f"{i * 3},{40 + (i % 3) * 8},{24 + (i % 4) * 4}\n" for i in range(14)) +
                     "".join(f"{400 + i * 40},{32},{16}\n" for i in range(6)))
    seq = str(tmp_path / "seq.json")
    M.save_sequence(M.baseline_sequence("back_to_front", 4), seq)
    static = 40
    cfg = tiny_config(str(trace), seq, static_blocks=static)
    cfg["quant_bits"] = bits  # both controller modes' target_bits
    cfg["model"]["layer_bytes"] = {k: pages[b] * pb for k, b in (("full", 16), ("q8", 8), ("q4", 4), ("q3", 3))}
    cfg["kv"]["block_bytes"] = pb
    cfg["budget"] = {"device_bytes": (4 * pages[16] + static + 40) * pb, "reserve_bytes": 40 * pb}
    dev = DeviceModel(shape, max_batch=32, max_prefill_tokens=128, max_pos=128,
                      arena_pages=4 * pages[16] + static + 40 + 64, variants=(16, bits, 4))
    try:
        dev.weights_synthetic(7)
        rep_cpu, log_cpu, _ = M.run_arm_full(cfg, "morph-performance")
        rep, log, _ = M.run_arm_full(cfg, "morph-performance", device=dev, record=True)
        assert log == log_cpu
        calls = rep.pop("device_calls")
        assert rep["morph"]["swap_events"] >= 1 and "KV_ATTACH" in log
        assert any(b == bits for c in calls for b in c["bits"])
        _replay_on_oracle(cfg, dev, calls, min_checked=150, shape=shape)
    finally:
        dev.close()
