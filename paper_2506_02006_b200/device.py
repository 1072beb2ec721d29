"""Python handle on one B200 device context (libmorphserve.so, include/morphserve.h).

This is the model-runner / LayerSwapper / KV-resizer surface the host runtime
drives; every method is one C-ABI call.  Shapes follow the
BASELINE.json configs:

    TINY      Llama-style L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024 (config 1)
    LLAMA2_7B L=32, d=4096, H=KVH=32, hd=128, ffn=11008, V=32000      (config 2)
    LLAMA3_8B L=32, d=4096, H=32, KVH=8, hd=128, ffn=14336, V=128256  (config 3/5)
    LLAMA2_13B L=40, d=5120, H=KVH=40, hd=128, ffn=13824, V=32000     (config 4)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N

TINY = dict(L=4, d=256, H=4, KVH=2, hd=64, ffn=768, V=1024)
LLAMA2_7B = dict(L=32, d=4096, H=32, KVH=32, hd=128, ffn=11008, V=32000)
LLAMA3_8B = dict(L=32, d=4096, H=32, KVH=8, hd=128, ffn=14336, V=128256, theta=500000.0)
LLAMA2_13B = dict(L=40, d=5120, H=40, KVH=40, hd=128, ffn=13824, V=32000)


def model_desc(shape: dict, *, max_batch: int, max_prefill_tokens: int, max_pos: int,
               arena_pages: int, eps: float = 1e-5) -> N.ModelDesc:
    return N.ModelDesc(shape["L"], shape["d"], shape["H"], shape["KVH"], shape["hd"], shape["ffn"],
                       shape["V"], 16, max_batch, max_prefill_tokens, max_pos, eps,
                       float(shape.get("theta", 10000.0)), arena_pages)


def page_bytes(shape: dict) -> int:
    return 16 * shape["L"] * shape["KVH"] * 2 * shape["hd"] * 2


def layer_pages(shape: dict, bits: int) -> int:
    d = model_desc(shape, max_batch=1, max_prefill_tokens=1, max_pos=16, arena_pages=1)
    return N.lib().ms_layer_pages(C.byref(d), bits)


@dataclass
class SwapTicket:
    layer: int
    bits: int
    ticket: int


class DeviceModel:
    """One device context: arena, layer table, variant store, streams, steps."""

    def __init__(self, shape: dict, *, device: int = 0, max_batch: int = 64, max_prefill_tokens: int = 2048,
                 max_pos: int = 4096, arena_pages: int, eps: float = 1e-5, variants=(16, 4)):
        self.shape = dict(shape)
        self.desc = model_desc(shape, max_batch=max_batch, max_prefill_tokens=max_prefill_tokens,
                               max_pos=max_pos, arena_pages=arena_pages, eps=eps)
        self.lib = N.lib()
        h = C.c_void_p()
        N.check(self.lib.ms_ctx_create(device, C.byref(self.desc), C.byref(h)))
        self.h = h
        self.max_blocks = (max_pos + 15) // 16
        self.page_bytes = self.lib.ms_page_bytes(C.byref(self.desc))
        # precision levels of the variant store (BF16 and Q4 always; Q8 / Q3 on request)
        for bits in variants:
            self.variant_enable(bits)

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            self.lib.ms_ctx_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        N.check(self.lib.ms_sync(self.h))

    # -- weights
    def weights_synthetic(self, seed: int):
        N.check(self.lib.ms_weights_synthetic(self.h, seed))

    def upload(self, layer: int, which: int, arr_bf16: np.ndarray):
        a = np.ascontiguousarray(arr_bf16, np.uint16)
        N.check(self.lib.ms_weights_upload(self.h, layer, which, a.ctypes.data, a.size))

    def finalize(self):
        N.check(self.lib.ms_weights_finalize(self.h))

    def variant_enable(self, bits: int):
        """Add the `bits` level (16, 8, 4, 3) to the pinned variant store (ms_variant_enable)."""
        N.check(self.lib.ms_variant_enable(self.h, bits))

    def variant_bytes(self, bits: int) -> int:
        return int(self.lib.ms_variant_bytes(self.h, bits))

    def variant_register(self, layer: int, bits: int, addr: int, nbytes: int, prefilled: bool):
        """Use caller-owned host memory at `addr` as the layer's variant image
        (ms_variant_register); before weights_synthetic / finalize."""
        N.check(self.lib.ms_variant_register(self.h, layer, bits, C.c_void_p(addr), nbytes, int(prefilled)))

    def variant_image(self, layer: int, bits: int) -> np.ndarray:
        n = self.lib.ms_variant_bytes(self.h, bits)
        out = np.empty(n, np.uint8)
        N.check(self.lib.ms_variant_export(self.h, layer, bits, out.ctypes.data, n))
        return out

    # -- LayerSwapper
    def swap_begin(self, layer: int, bits: int) -> SwapTicket:
        t = C.c_uint64()
        N.check(self.lib.ms_swap_begin(self.h, layer, bits, C.byref(t)))
        return SwapTicket(layer, bits, t.value)

    def set_stream(self, stream_ptr: int | None):
        """Order steps after / before the caller's CUDA stream (ms_set_stream)."""
        N.check(self.lib.ms_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def swap_begin_peer(self, layer: int, bits: int, src: "DeviceModel") -> SwapTicket:
        """Swap with the image copied from another context that holds the layer at
        `bits` (ms_swap_begin_peer: device to device / NVLink instead of host PCIe)."""
        t = C.c_uint64()
        N.check(self.lib.ms_swap_begin_peer(self.h, layer, bits, src.h, C.byref(t)))
        return SwapTicket(layer, bits, t.value)

    def swap_done(self, t: SwapTicket) -> bool:
        d = C.c_int()
        N.check(self.lib.ms_swap_poll(self.h, t.ticket, C.byref(d)))
        return bool(d.value)

    def swap_wait(self, t: SwapTicket) -> float:
        ms = C.c_float()
        N.check(self.lib.ms_swap_wait(self.h, t.ticket, C.byref(ms)))
        return ms.value

    def swap_commit(self, t: SwapTicket) -> int:
        freed = C.c_int64()
        N.check(self.lib.ms_swap_commit(self.h, t.ticket, C.byref(freed)))
        return freed.value

    def layer_bits(self, layer: int) -> int:
        return self.lib.ms_layer_bits(self.h, layer)

    # -- KV resizer
    def kv_attach(self, first_id: int, n: int):
        N.check(self.lib.ms_kv_attach(self.h, first_id, n))

    def kv_detach(self, ids):
        a = np.ascontiguousarray(ids, np.int64)
        N.check(self.lib.ms_kv_detach(self.h, N.i64p(a), a.size))

    def free_pages(self) -> int:
        return self.lib.ms_free_pages(self.h)

    def page_of(self, block_id: int) -> int:
        return self.lib.ms_kv_page_of(self.h, block_id)

    def kv_export(self, block_id: int) -> np.ndarray:
        """One block's KV page (bf16 as u16): [L][KVH][2][16][hd]."""
        s = self.shape
        out = np.empty((s["L"], s["KVH"], 2, 16, s["hd"]), np.uint16)
        N.check(self.lib.ms_kv_export(self.h, block_id, out.ctypes.data, out.nbytes))
        return out

    # -- token history
    def hist_reserve(self, slots: int, max_len: int):
        N.check(self.lib.ms_hist_reserve(self.h, slots, max_len))

    def hist_write(self, slot: int, offset: int, tokens):
        a = np.ascontiguousarray(tokens, np.int32)
        N.check(self.lib.ms_hist_write(self.h, slot, offset, N.i32p(a), a.size))

    def hist_read(self, slot: int, offset: int, n: int) -> np.ndarray:
        out = np.empty(n, np.int32)
        N.check(self.lib.ms_hist_read(self.h, slot, offset, N.i32p(out), n))
        return out

    # -- steps
    def prefill(self, slot: int, n_tokens: int, block_ids, want_logits: bool = False):
        ids = np.ascontiguousarray(block_ids, np.int64)
        nxt = C.c_int32()
        logits = np.empty(self.shape["V"], np.float32) if want_logits else None
        N.check(self.lib.ms_prefill(self.h, slot, n_tokens, N.i64p(ids), ids.size, C.byref(nxt),
                                    N.f32p(logits)))
        return nxt.value, logits

    def prefill_trace(self, slot: int, n_tokens: int, block_ids, want_logits: bool = True):
        """Prefill that also returns the residual stream entering every layer and
        leaving the last one: ([L+1, n, d] fp32, last-token logits)."""
        ids = np.ascontiguousarray(block_ids, np.int64)
        h = np.empty((self.shape["L"] + 1, n_tokens, self.shape["d"]), np.float32)
        logits = np.empty(self.shape["V"], np.float32) if want_logits else None
        N.check(self.lib.ms_prefill_trace(self.h, slot, n_tokens, N.i64p(ids), ids.size, N.f32p(h), N.f32p(logits)))
        return h, logits

    def decode(self, slots, positions, block_table, tokens=None, want_next: bool = True,
               want_logits: bool = False):
        slots = np.ascontiguousarray(slots, np.int32)
        pos = np.ascontiguousarray(positions, np.int32)
        bt = np.ascontiguousarray(block_table, np.int64)
        n = slots.size
        tok = np.ascontiguousarray(tokens, np.int32) if tokens is not None else None
        b = N.DecodeBatch(n, N.i32p(slots), N.i32p(pos), N.i32p(tok), N.i64p(bt), bt.shape[1])
        nxt = np.empty(n, np.int32) if want_next else None
        logits = np.empty((n, self.shape["V"]), np.float32) if want_logits else None
        N.check(self.lib.ms_decode_step(self.h, C.byref(b), N.i32p(nxt), N.f32p(logits)))
        return nxt, logits

    def decode_submit(self, slots, positions, block_table, tokens=None):
        """Enqueue a decode step (ms_decode_submit); collect its tokens later."""
        slots = np.ascontiguousarray(slots, np.int32)
        pos = np.ascontiguousarray(positions, np.int32)
        bt = np.ascontiguousarray(block_table, np.int64)
        tok = np.ascontiguousarray(tokens, np.int32) if tokens is not None else None
        b = N.DecodeBatch(slots.size, N.i32p(slots), N.i32p(pos), N.i32p(tok), N.i64p(bt), bt.shape[1])
        N.check(self.lib.ms_decode_submit(self.h, C.byref(b)))

    def decode_collect(self) -> np.ndarray:
        """Next tokens of the oldest submitted step (waits for it)."""
        out = np.empty(self.desc.max_batch, np.int32)
        n = C.c_int32()
        N.check(self.lib.ms_decode_collect(self.h, N.i32p(out), C.byref(n)))
        return out[: n.value].copy()

    def last_step_ms(self) -> float:
        ms = C.c_float()
        N.check(self.lib.ms_last_step_ms(self.h, C.byref(ms)))
        return ms.value

    def kv_fill_synthetic(self, block_ids, seed: int):
        a = np.ascontiguousarray(block_ids, np.int64)
        N.check(self.lib.ms_kv_fill_synthetic(self.h, N.i64p(a), a.size, seed))

    # -- instrumentation
    def launch_count(self) -> int:
        return self.lib.ms_launch_count(self.h)

    def timer_start(self):
        N.check(self.lib.ms_timer_start(self.h))

    def timer_stop(self) -> float:
        ms = C.c_float()
        N.check(self.lib.ms_timer_stop(self.h, C.byref(ms)))
        return ms.value

    PK_NAMES = ["embed", "gemm_qkv", "gemm_qkv_w4", "qkv_post", "attn", "gemm_o", "gemm_o_w4", "norm", "gemm_gu",
                "gemm_gu_w4", "silu", "gemm_down", "gemm_down_w4", "lm_head", "argmax"]

    def prof_kernels(self, enable: bool):
        N.check(self.lib.ms_prof_kernels(self.h, int(enable)))

    def prof_kernels_read(self) -> dict:
        """{category: (total ms, launches)} since prof_kernels(True)."""
        k = len(self.PK_NAMES)
        ms = (C.c_float * k)()
        n = (C.c_int64 * k)()
        N.check(self.lib.ms_prof_kernels_read(self.h, ms, n))
        return {name: (float(ms[i]), int(n[i])) for i, name in enumerate(self.PK_NAMES) if n[i]}

    def prof_attention(self, enable: bool):
        N.check(self.lib.ms_prof_attention(self.h, int(enable)))

    def prof_attention_read(self):
        ms = C.c_float()
        n = C.c_int64()
        N.check(self.lib.ms_prof_attention_read(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value
