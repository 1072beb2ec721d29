"""KV block pool (KVResizer bookkeeping): reference KATs (proj/tests/test_kvpool.cpp)
and op-by-op identity with the compiled reference pool under a random fuzz."""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2506_02006_b200 import _core as C

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pool(blocks, bt=16):
    return C.KvBlockPool(C.KvConfig(bt, 2 << 20, blocks))


def test_golden_sequence_survey_a9():
    g = json.load(open(os.path.join(GOLD, "kvpool.json")))[0]
    p = pool(g["capacity"])
    for op in g["ops"]:
        if op[0] == "alloc":
            if not p.is_admitted(op[1]):
                p.admit(op[1])
            assert p.alloc_for_tokens(op[1], op[2]) == op[3]
        elif op[0] == "attach":
            assert p.attach_blocks(op[1]) == op[2]
        elif op[0] == "release":
            assert p.release(op[1]) == op[2]
        elif op[0] == "detach":
            assert list(p.detach_blocks(op[1])) == op[2]
    assert p.take_retired() == [3, 2, 1]  # detach removes the free-stack top, not the attached ids
    p.check_invariants()


def test_ceiling_and_in_block_growth():
    p = pool(64)
    p.admit(1)
    assert len(p.alloc_for_tokens(1, 512)) == 32
    q = pool(8)
    q.admit(1)
    assert len(q.alloc_for_tokens(1, 17)) == 2
    assert q.alloc_for_tokens(1, 1) == []
    assert len(q.alloc_for_tokens(1, 14)) == 0
    assert len(q.alloc_for_tokens(1, 1)) == 1


def test_all_or_nothing_and_errors():
    p = pool(2)
    p.admit(1)
    p.admit(2)
    assert p.alloc_for_tokens(2, 1) is not None
    assert p.alloc_for_tokens(1, 48) is None
    assert p.free_blocks() == 1 and p.tokens_of(1) == 0
    with pytest.raises(ValueError):
        p.admit(1)
    with pytest.raises(ValueError):
        p.alloc_for_tokens(99, 1)
    with pytest.raises(ValueError):
        p.attach_blocks(0)
    with pytest.raises(ValueError):
        p.detach_blocks(1)


def test_deferred_detach_absorbs_releases():
    p = pool(5)
    p.attach_blocks(10)
    p.admit(1)
    p.alloc_for_tokens(1, 12 * 16)
    assert p.detach_blocks(10) == (3, 7, 12)
    assert p.pending_detach_blocks() == 7
    p.release(1)
    assert p.pending_detach_blocks() == 0 and p.capacity_blocks() == 5 and p.free_blocks() == 5
    assert len(p.take_retired()) == 10
    p.check_invariants()


def test_lifo_preemption():
    p = pool(16)
    for r in (10, 11, 12):
        p.admit(r)
        p.alloc_for_tokens(r, 16)
    assert p.preempt_victim() == 12
    assert p.preempt_victim(lambda r: r == 10) == 10
    assert p.preempt_victim() == 11
    assert p.preempt_victim() is None


@pytest.mark.skipif(not O.have_ref_core(), reason="oracle/_ref not built")
def test_fuzz_identical_to_reference():
    ref = O.ref_core()
    a, b = pool(64, 8), ref.KvBlockPool(ref.KvConfig(8, 2 << 20, 64))
    rng = np.random.default_rng(2024)
    admitted, nxt = [], 0
    for step in range(20000):
        roll = int(rng.integers(0, 100))
        if roll < 30:
            a.admit(nxt); b.admit(nxt); admitted.append(nxt); nxt += 1
        elif roll < 60 and admitted:
            r = admitted[int(rng.integers(0, len(admitted)))]
            n = 1 + int(rng.integers(0, 64))
            assert a.alloc_for_tokens(r, n) == b.alloc_for_tokens(r, n)
        elif roll < 75 and admitted:
            r = admitted.pop(int(rng.integers(0, len(admitted))))
            assert a.release(r) == b.release(r)
        elif roll < 85:
            n = 1 + int(rng.integers(0, 32))
            assert a.attach_blocks(n) == b.attach_blocks(n)
        elif roll < 95:
            can = a.attached_extra_blocks() - a.pending_detach_blocks()
            if can > 0:
                n = 1 + int(rng.integers(0, can))
                assert tuple(a.detach_blocks(n)) == tuple(b.detach_blocks(n))
        assert a.capacity_blocks() == b.capacity_blocks()
        assert a.free_blocks() == b.free_blocks()
        if step % 256 == 0:
            a.check_invariants()
            for r in admitted:
                assert a.tokens_of(r) == b.tokens_of(r) and a.blocks_of(r) == b.blocks_of(r)
