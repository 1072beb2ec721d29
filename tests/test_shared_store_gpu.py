"""One box-wide host copy of the variant store for all replica processes
(ms_variant_register): local rank 0 builds the packed BF16 / W4
images into POSIX shared memory, rank 1 registers the same memory as
pre-packed and skips the build.  Both replicas must hold byte-identical
images (equal to a context that built its own store), swap a layer to W4 from
them, and decode the same greedy tokens (2 processes on one GPU, gloo)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

pytestmark = pytest.mark.gpu

TINY = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _decode(dev):
    dev.hist_reserve(1, 64)
    dev.kv_attach(0, 4)
    table = np.arange(4, dtype=np.int64)[None, :]
    dev.hist_write(0, 0, np.arange(20, dtype=np.int32) * 7)
    tok = dev.prefill(0, 20, table[0])[0]
    t = dev.swap_begin(1, 4)
    dev.swap_wait(t)
    dev.swap_commit(t)
    out = [tok]
    pos = np.array([20], np.int32)
    for _ in range(6):
        nxt, _ = dev.decode(np.zeros(1, np.int32), pos, table)
        out.append(int(nxt[0]))
        pos += 1
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_02006_b200.replicas import replica_device
    key = f"test_{port}"
    dev, store = replica_device(TINY, local_rank=rank, world=world, barrier=dist.barrier, key=key, device=0,
                                max_batch=4, max_prefill_tokens=64, max_pos=64, arena_pages=300)
    imgs = [dev.variant_image(l, b) for l in range(TINY["L"]) for b in (16, 4)]
    toks = _decode(dev)
    dev.close()
    dist.barrier()
    if rank == 0:
        store.unlink()
    gathered = [None] * world
    dist.all_gather_object(gathered, (toks, [int(np.frombuffer(i.tobytes(), np.uint64).sum()) for i in imgs]))
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


def test_shared_variant_store_two_replicas():
    from paper_2506_02006_b200.device import DeviceModel
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    own = DeviceModel(TINY, max_batch=4, max_prefill_tokens=64, max_pos=64, arena_pages=300)
    try:
        own.weights_synthetic(7)
        sums = [int(np.frombuffer(own.variant_image(l, b).tobytes(), np.uint64).sum())
                for l in range(TINY["L"]) for b in (16, 4)]
        toks = _decode(own)
    finally:
        own.close()
    for g in gathered:
        assert g[1] == sums
        assert g[0] == toks
