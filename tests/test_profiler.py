"""Offline layer profiler: the GPU restatement of the
reference LIS profile (proj/src/profiler.cpp:41-139) against its CPU oracle
(oracle.lis_greedy over the Llama-style reference model)."""
import numpy as np
import pytest

import oracle as O

CFG = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024, max_pos=128)
PROMPTS = [((np.arange(24, dtype=np.int32) * 37 + 5 * i) % 1024).astype(np.int32) for i in range(3)]


def test_oracle_lis_greedy_properties(oracle_lib):
    # alpha1 only: the order is LTS descending, ties to the lowest index (profiler.cpp:125-130)
    r = O.lis_greedy(CFG, 7, PROMPTS, weights={"alpha1": 1.0, "alpha2": 0.0, "beta": 0.0})
    lts = np.array(r["lts"])
    assert r["order"] == sorted(range(CFG["L"]), key=lambda j: (-lts[j], j))
    assert np.allclose(r["per_step_lis"], lts[r["order"]])
    # scores are cosines
    assert all(0.0 < x <= 1.0 + 1e-12 for x in r["lts"] + r["lrs"])
    # the GPU module imports without a device (no CUDA work at import time)
    from paper_2506_02006_b200.profiler import DEFAULT_WEIGHTS
    assert DEFAULT_WEIGHTS == {"alpha1": 0.25, "alpha2": 0.25, "beta": 0.5}  # profiler.hpp:13-15


@pytest.mark.gpu
def test_gpu_profile_matches_oracle():
    from paper_2506_02006_b200.device import DeviceModel
    from paper_2506_02006_b200.profiler import GpuProfiler

    ref = O.lis_greedy(CFG, 7, PROMPTS)
    dev = DeviceModel({k: v for k, v in CFG.items() if k != "max_pos"}, max_batch=4, max_prefill_tokens=64,
                      max_pos=128, arena_pages=512)
    try:
        dev.weights_synthetic(7)
        prof = GpuProfiler(dev, PROMPTS)
        got = prof.greedy_sequence()
        prof.close()
    finally:
        dev.close()
    np.testing.assert_allclose(got["lts"], ref["lts"], atol=1e-4)
    np.testing.assert_allclose(got["lrs"], ref["lrs"], atol=1e-4)
    np.testing.assert_allclose(got["per_step_lis"], ref["per_step_lis"], atol=1e-4)
    assert got["order"] == ref["order"]


def test_committed_gpu_sequence_loads():
    # configs/sequence_gpu_lis_32.json: tools/gpu_profile.py --shape 7b on a B200
    import os

    from paper_2506_02006_b200 import morphsim as M
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs",
                        "sequence_gpu_lis_32.json")
    seq = M.load_sequence(path)
    assert sorted(seq["order"]) == list(range(32))
    assert len(seq["per_step_lis"]) == 32
