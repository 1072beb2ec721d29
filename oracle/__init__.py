"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference legs may import this package, and only as the checker.  The product
(``paper_2506_02006_b200``) never imports it; the product's native path fails
loudly when its CUDA library is missing instead of falling back to anything here.

Two oracles live here:

* ``ref_core()`` -- the UNMODIFIED reference simulator (``/root/reference/proj``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/`` (its own pybind11
  ``_core`` module).  Bit-exact target for KV block allocation, block tables,
  swap decisions / event logs, attach arithmetic and the metric definitions.
* ``libref_llama`` (``oracle/ref_llama.c``) -- a C restatement of the g128
  quantizer (reference ``proj/src/toy_model.cpp:40-60``) plus this repo's
  Llama-style decoder contract, which the reference does not have (SURVEY 8(c):
  logits / attention / GEMM numerics are "parity unpinned" against the
  reference; they are pinned by the frozen fixtures in ``tests/golden``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_lib", "libref_llama.so")
_REF_DIR = os.path.join(_HERE, "_ref")
_lib = None

# tensor ids, mirrored from ref_llama.c
T_EMBED, T_NORMF, T_LMHEAD = 0, 1, 2
W_NORM1, W_QKV, W_O, W_NORM2, W_GU, W_DOWN = 0, 1, 2, 3, 4, 5


def build(ref: bool = False) -> None:
    """Builds oracle/_lib (and oracle/_ref when asked and /root/reference exists)."""
    targets = ["lib"] + (["ref"] if ref and os.path.isdir("/root/reference/proj/src") else [])
    subprocess.check_call(["make", "-s", "-C", _HERE, *targets])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        u16p = np.ctypeslib.ndpointer(np.uint16, flags="C")
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
        i8p = np.ctypeslib.ndpointer(np.int8, flags="C")
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C")
        i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
        L.ref_gen_weight.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_double, C.c_double, u16p]
        L.ref_quantize_groups.argtypes = [u16p, C.c_int64, C.c_int64, C.c_int, C.c_int, i8p, f64p, u16p]
        L.ref_dequant_w4.argtypes = [i8p, u16p, C.c_int64, C.c_int64, C.c_int, u16p]
        L.ref_pack_bf16.argtypes = [u16p, C.c_int64, C.c_int64, u16p]
        L.ref_pack_w4.argtypes = [i8p, u16p, C.c_int64, C.c_int64, u8p]
        L.ref_pack_w8.argtypes = [i8p, u16p, C.c_int64, C.c_int64, u8p]
        L.ref_gemm_bf16.argtypes = [u16p, u16p, C.c_int64, C.c_int64, C.c_int64, f32p]
        L.ref_rmsnorm.argtypes = [f32p, u16p, C.c_int64, C.c_int64, C.c_float, u16p]
        L.ref_attention.argtypes = [f32p, u16p, u16p, C.c_int, C.c_int, C.c_int, C.c_int, u16p, f32p]
        L.ref_rope_table.argtypes = [C.c_int, C.c_int, C.c_double, f32p, f32p]
        L.ref_model_create.argtypes = [C.c_void_p, C.c_uint64]
        L.ref_model_create.restype = C.c_void_p
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_model_set_precision.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_model_tensor.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_model_tensor.restype = C.POINTER(C.c_uint16)
        L.ref_seq_create.argtypes = [C.c_void_p, C.c_int]
        L.ref_seq_create.restype = C.c_void_p
        L.ref_seq_destroy.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_seq_len.argtypes = [C.c_void_p]
        L.ref_seq_k.argtypes = [C.c_void_p, C.c_int]
        L.ref_seq_k.restype = C.POINTER(C.c_uint16)
        L.ref_seq_v.argtypes = [C.c_void_p, C.c_int]
        L.ref_seq_v.restype = C.POINTER(C.c_uint16)
        L.ref_forward.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), i32p, C.c_int, C.c_void_p, i32p]
        L.ref_prefill.argtypes = [C.c_void_p, C.c_void_p, i32p, C.c_int, C.c_void_p]
        L.ref_prefill.restype = C.c_int32
        L.ref_prefill_trace.argtypes = [C.c_void_p, C.c_void_p, i32p, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_prefill_trace.restype = C.c_int32
        L.ref_prefill_rows.argtypes = [C.c_void_p, C.c_void_p, i32p, C.c_int, C.c_void_p, C.c_int, C.c_void_p,
                                       C.c_void_p]
        L.ref_prefill_rows.restype = C.c_int32
        L.ref_seq_set_len.argtypes = [C.c_void_p, C.c_int]
        L.ref_seq_fill_pages.argtypes = [C.c_void_p, C.c_void_p, np.ctypeslib.ndpointer(np.int64, flags="C"),
                                         C.c_int, C.c_uint64]
        L.ref_num_threads.restype = C.c_int
        _lib = L
    return _lib


def ref_core():
    """The compiled reference simulator's pybind11 module (oracle/_ref/_core)."""
    if _REF_DIR not in sys.path:
        sys.path.insert(0, _REF_DIR)
    import _core  # noqa: PLC0415  (the reference's own module name)
    return _core


def have_ref_core() -> bool:
    return any(f.startswith("_core") and f.endswith(".so") for f in os.listdir(_REF_DIR)) \
        if os.path.isdir(_REF_DIR) else False


# ---------------------------------------------------------------- helpers
def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u >> 16) & 1) + 0x7FFF
    out = ((u + r) >> 16).astype(np.uint16)
    out[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)
    return out


def gen_weight(seed: int, tensor: int, n: int, scale: float, offset: float = 0.0) -> np.ndarray:
    out = np.empty(n, np.uint16)
    lib().ref_gen_weight(seed, tensor, n, scale, offset, out)
    return out


def quantize_groups(w_bf16: np.ndarray, group: int = 128, bits: int = 4):
    """-> (codes int8 [N,K], scales fp64 [N,K/g], scales bf16 [N,K/g])"""
    w = np.ascontiguousarray(w_bf16, np.uint16)
    N, K = w.shape
    codes = np.empty((N, K), np.int8)
    s64 = np.empty((N, K // group), np.float64)
    s16 = np.empty((N, K // group), np.uint16)
    lib().ref_quantize_groups(w, N, K, group, bits, codes, s64, s16)
    return codes, s64, s16


def dequant_w4(codes: np.ndarray, scales_bf16: np.ndarray) -> np.ndarray:
    """bf16(code * float(scale_bf16)) per g128 group (every quantised level: 8, 4, 3 bits)."""
    N, K = codes.shape
    out = np.empty((N, K), np.uint16)
    lib().ref_dequant_w4(np.ascontiguousarray(codes), np.ascontiguousarray(scales_bf16), N, K, 128, out)
    return out


def pack_bf16(w_bf16: np.ndarray) -> np.ndarray:
    N, K = w_bf16.shape
    out = np.empty(N * K, np.uint16)
    lib().ref_pack_bf16(np.ascontiguousarray(w_bf16), N, K, out)
    return out


def pack_w4(codes: np.ndarray, scales_bf16: np.ndarray) -> np.ndarray:
    N, K = codes.shape
    out = np.empty((N // 128) * (K // 128) * 8448, np.uint8)
    lib().ref_pack_w4(np.ascontiguousarray(codes), np.ascontiguousarray(scales_bf16), N, K, out)
    return out


def pack_w8(codes: np.ndarray, scales_bf16: np.ndarray) -> np.ndarray:
    N, K = codes.shape
    out = np.empty((N // 128) * (K // 128) * 16640, np.uint8)
    lib().ref_pack_w8(np.ascontiguousarray(codes), np.ascontiguousarray(scales_bf16), N, K, out)
    return out


def pack_quant(codes: np.ndarray, scales_bf16: np.ndarray, bits: int) -> np.ndarray:
    """Device image of a quantised matrix: W8 chunks for 8 bits, 4-bit containers for 4 and 3 bits."""
    return pack_w8(codes, scales_bf16) if bits == 8 else pack_w4(codes, scales_bf16)


def gemm_bf16(W: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Y[b,n] = sum_k W[n,k] X[b,k], fp64 accumulation, fp32 result."""
    N, K = W.shape
    B = X.shape[0]
    Y = np.empty((B, N), np.float32)
    lib().ref_gemm_bf16(np.ascontiguousarray(W), np.ascontiguousarray(X), B, N, K, Y)
    return Y


def rmsnorm(h: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    B, d = h.shape
    out = np.empty((B, d), np.uint16)
    lib().ref_rmsnorm(np.ascontiguousarray(h, np.float32), np.ascontiguousarray(w), B, d, eps, out)
    return out


def attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, H: int, KVH: int, hd: int):
    """q [H*hd] f32; k,v [ctx, KVH, hd] bf16 -> (o bf16 [H*hd], o f32 [H*hd])."""
    ctx = k.shape[0]
    o16 = np.empty(H * hd, np.uint16)
    o32 = np.empty(H * hd, np.float32)
    lib().ref_attention(np.ascontiguousarray(q, np.float32), np.ascontiguousarray(k),
                        np.ascontiguousarray(v), ctx, H, KVH, hd, o16, o32)
    return o16, o32


def rope_table(max_pos: int, hd: int, theta: float):
    c = np.empty((max_pos, hd // 2), np.float32)
    s = np.empty((max_pos, hd // 2), np.float32)
    lib().ref_rope_table(max_pos, hd, theta, c, s)
    return c, s


class _Cfg(C.Structure):
    _fields_ = [("L", C.c_int), ("d", C.c_int), ("H", C.c_int), ("KVH", C.c_int), ("hd", C.c_int),
                ("ffn", C.c_int), ("V", C.c_int), ("max_pos", C.c_int), ("eps", C.c_float),
                ("theta", C.c_double)]


class RefModel:
    """Llama-style CPU model with the same synthetic weights as the GPU path."""

    def __init__(self, cfg: dict, seed: int):
        self.cfg = dict(cfg)
        c = _Cfg(cfg["L"], cfg["d"], cfg["H"], cfg["KVH"], cfg["hd"], cfg["ffn"], cfg["V"],
                 cfg["max_pos"], cfg.get("eps", 1e-5), cfg.get("theta", 10000.0))
        self._c = c
        self.h = lib().ref_model_create(C.byref(c), seed)
        self.seqs = []

    def close(self):
        if self.h:
            for s in self.seqs:
                lib().ref_seq_destroy(self.h, s)
            lib().ref_model_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_precision(self, layer: int, bits: int):
        lib().ref_model_set_precision(self.h, layer, bits)

    def tensor(self, layer: int, which: int, shape) -> np.ndarray:
        p = lib().ref_model_tensor(self.h, layer, which)
        n = int(np.prod(shape))
        return np.ctypeslib.as_array(p, shape=(n,)).reshape(shape).copy()

    def new_seq(self, cap: int):
        s = lib().ref_seq_create(self.h, cap)
        self.seqs.append(s)
        return s

    def seq_kv(self, s, layer: int, length: int):
        c = self.cfg
        n = length * c["KVH"] * c["hd"]
        k = np.ctypeslib.as_array(lib().ref_seq_k(s, layer), shape=(n,)).reshape(length, c["KVH"], c["hd"]).copy()
        v = np.ctypeslib.as_array(lib().ref_seq_v(s, layer), shape=(n,)).reshape(length, c["KVH"], c["hd"]).copy()
        return k, v

    def forward(self, seqs, tokens, want_logits: bool = True):
        B = len(seqs)
        arr = (C.c_void_p * B)(*seqs)
        toks = np.ascontiguousarray(tokens, np.int32)
        nxt = np.empty(B, np.int32)
        logits = np.empty((B, self.cfg["V"]), np.float32) if want_logits else None
        lib().ref_forward(self.h, arr, toks, B,
                          logits.ctypes.data_as(C.c_void_p) if want_logits else None, nxt)
        return nxt, logits

    def prefill_trace(self, s, tokens):
        """Prefill returning the residual stream entering each layer and leaving
        the last one: [L+1, n, d] fp32 (oracle of ms_prefill_trace)."""
        toks = np.ascontiguousarray(tokens, np.int32)
        tr = np.empty((self.cfg["L"] + 1, len(toks), self.cfg["d"]), np.float32)
        lib().ref_prefill_trace(self.h, s, toks, len(toks), None, tr.ctypes.data_as(C.c_void_p))
        return tr

    def prefill_rows(self, s, tokens, rows=None, want_logits: bool = True, want_trace: bool = False):
        """Batched prefill (bit-identical to ``prefill`` / ``prefill_trace``).
        ``rows``: token rows carried through the last layer (sorted, unique;
        must contain the last token for logits).  Returns (next, logits,
        trace [L+1, n, d] or None; in the last layer slice only ``rows`` are
        defined)."""
        toks = np.ascontiguousarray(tokens, np.int32)
        n = len(toks)
        r = None if rows is None else np.ascontiguousarray(np.unique(np.asarray(rows, np.int32)))
        logits = np.empty(self.cfg["V"], np.float32) if want_logits else None
        tr = np.zeros((self.cfg["L"] + 1, n, self.cfg["d"]), np.float32) if want_trace else None
        nxt = lib().ref_prefill_rows(self.h, s, toks, n, None if r is None else r.ctypes.data_as(C.c_void_p),
                                     0 if r is None else len(r),
                                     logits.ctypes.data_as(C.c_void_p) if want_logits else None,
                                     tr.ctypes.data_as(C.c_void_p) if want_trace else None)
        return int(nxt), logits, tr

    def seq_fill_pages(self, s, page_index, seed: int):
        """Fill the sequence's KV cache with the device's synthetic fill
        (ms_kv_fill_synthetic): block j = the page_index[j]-th page of the fill
        list; sets the sequence length to 16 * len(page_index)."""
        pi = np.ascontiguousarray(page_index, np.int64)
        lib().ref_seq_fill_pages(self.h, s, pi, len(pi), seed)
        lib().ref_seq_set_len(s, 16 * len(pi))

    def seq_set_len(self, s, n: int):
        lib().ref_seq_set_len(s, n)

    def prefill(self, s, tokens, want_logits: bool = True):
        toks = np.ascontiguousarray(tokens, np.int32)
        logits = np.empty(self.cfg["V"], np.float32) if want_logits else None
        nxt = lib().ref_prefill(self.h, s, toks, len(toks),
                                logits.ctypes.data_as(C.c_void_p) if want_logits else None)
        return int(nxt), logits


# ------------------------------------------------------- layer profiler oracle
def _cos64(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0.0 or nb == 0.0:
        return 1.0 if na == nb else 0.0
    return float(np.dot(a, b) / (na * nb))


def lis_greedy(cfg: dict, seed: int, prompts, bits: int = 4, weights=None) -> dict:
    """CPU restatement of the layer-importance profile (reference
    proj/src/profiler.cpp:41-139: LTS, LRS, MDS, greedy argmax with ties to the
    lowest index) over the Llama-style oracle model; the oracle of
    paper_2506_02006_b200.profiler.GpuProfiler.greedy_sequence."""
    w = {"alpha1": 0.25, "alpha2": 0.25, "beta": 0.5}
    w.update(weights or {})
    m = RefModel(cfg, seed)
    L = cfg["L"]
    try:
        def traces(q):
            for l in range(L):
                m.set_precision(l, bits if l in q else 16)
            out = []
            for p in prompts:
                s = m.new_seq(len(p) + 1)
                out.append(m.prefill_trace(s, p))
            return out
        full = traces(set())
        lts = [float(np.mean([_cos64(h[p + 1], h[p]) for h in full])) for p in range(L)]
        lrs = []
        for p in range(L):
            qt = traces({p})
            lrs.append(float(np.mean([_cos64(f[p + 1], q[p + 1]) for f, q in zip(full, qt)])))
        quant, order, per_step = set(), [], []
        base = [h[L] for h in full]
        for _ in range(L):
            best, best_score, best_final = -1, -np.inf, None
            for j in range(L):
                if j in quant:
                    continue
                cand = [h[L] for h in traces(quant | {j})]
                mds = float(np.mean([_cos64(b, c) for b, c in zip(base, cand)]))
                lis = w["alpha1"] * lts[j] + w["alpha2"] * lrs[j] + w["beta"] * mds
                if lis > best_score:
                    best, best_score, best_final = j, lis, cand
            order.append(best)
            per_step.append(best_score)
            quant.add(best)
            base = best_final
        return {"order": order, "per_step_lis": per_step, "bits": bits, "kind": "lis_greedy", "weights": w,
                "lts": lts, "lrs": lrs}
    finally:
        m.close()
