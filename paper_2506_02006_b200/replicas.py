"""Multi-GPU = independent replicas: requests of one trace go
round-robin to G GPUs; each replica runs its own engine, arena, layer table,
KV pool and controller.  No collective sits on the data path -- the only
cross-rank traffic is gathering reports and the max-over-ranks timing.
"""
from __future__ import annotations

import os

import numpy as np

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


class SharedVariantStore:
    """One host copy of every layer's packed BF16 and W4 images for all the
    replica processes of a box, in POSIX shared
    memory (/dev/shm).  Local rank 0 registers it with prefilled=False and
    builds the images (ms_weights_synthetic packs into it); after `barrier()`
    the other ranks register the same memory with prefilled=True and skip the
    build.  Every context page-locks its mapping (cudaHostRegister), so the
    uploads stream from the same physical pages."""

    def __init__(self, key: str, nbytes_per_layer: int, layers: int):
        self.path = f"/dev/shm/morphserve_{key}"
        self.per_layer = nbytes_per_layer
        self.layers = layers
        self.arr = None

    def create(self):
        if os.path.exists(self.path):
            os.unlink(self.path)
        self.arr = np.memmap(self.path, dtype=np.uint8, mode="w+", shape=(self.per_layer * self.layers,))
        return self

    def attach(self):
        self.arr = np.memmap(self.path, dtype=np.uint8, mode="r+", shape=(self.per_layer * self.layers,))
        return self

    def register(self, dev, prefilled: bool):
        base = self.arr.ctypes.data
        n16, n4 = dev.variant_bytes(16), dev.variant_bytes(4)
        assert n16 + n4 == self.per_layer
        for l in range(self.layers):
            off = l * self.per_layer
            dev.variant_register(l, 16, base + off, n16, prefilled)
            dev.variant_register(l, 4, base + off + n16, n4, prefilled)

    def unlink(self):
        if os.path.exists(self.path):
            os.unlink(self.path)


def replica_device(shape: dict, *, local_rank: int, world: int, barrier, key: str, seed: int = 7,
                   device: int | None = None, **kw):
    """A DeviceModel with synthetic weights on GPU `device` (default: the local
    rank); at world > 1 its variant store is the box-wide shared copy (built
    once by local rank 0)."""
    from .device import DeviceModel
    dev = DeviceModel(shape, device=local_rank if device is None else device, **kw)
    if world <= 1:
        dev.weights_synthetic(seed)
        return dev, None
    store = SharedVariantStore(key, dev.variant_bytes(16) + dev.variant_bytes(4), shape["L"])
    if local_rank == 0:
        store.create().register(dev, prefilled=False)
        dev.weights_synthetic(seed)
        barrier()
    else:
        barrier()
        store.attach().register(dev, prefilled=True)
        dev.weights_synthetic(seed)
    return dev, store
