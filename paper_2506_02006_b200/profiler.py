"""Offline layer-importance profiler on the B200.

The reference computes MorphServe's swap order with its fp64 toy model
(proj/src/profiler.cpp:41-139).  This module runs the same algorithm on the real
Llama-style model with the production kernels and emits the same sequence JSON
(profiler.cpp:198-214 via morphsim.save_sequence), which the engine consumes
unchanged (experiment.cpp:307-310):

    LTS[p]    mean over the calibration set of cos(output of layer p, its input)
              with every layer at full precision            (profiler.cpp:41-54)
    LRS[p]    mean cos(output of layer p at full precision, output of layer p
              with ITS weights quantized, on the same input) (profiler.cpp:56-79)
    MDS(Q, j) mean cos(final output with layers Q quantized, final output with
              Q + {j} quantized)                             (profiler.cpp:81-103)
    greedy:   L rounds; each picks argmax_j alpha1*LTS[j] + alpha2*LRS[j] +
              beta*MDS(Q, j), ties to the lowest index       (profiler.cpp:106-139)

"Output of layer p" is the residual stream leaving the decoder block (the
toy model's h + tanh(Wh + b) becomes the Llama block here); the final output is
the residual stream after the last block.  Each calibration sample is one prompt
prefilled through ms_prefill_trace; precision changes go through the
LayerSwapper (upload + token-boundary commit), so the profile sees exactly the
dequantised weights decode will use.  Cosines accumulate in fp64 over the
flattened [tokens x hidden] activations.
"""
from __future__ import annotations

import numpy as np

from .device import DeviceModel

DEFAULT_WEIGHTS = {"alpha1": 0.25, "alpha2": 0.25, "beta": 0.5}  # profiler.hpp:13-15


def _cos(a: np.ndarray, b: np.ndarray) -> float:
    a = a.astype(np.float64).ravel()
    b = b.astype(np.float64).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0.0 or nb == 0.0:
        return 1.0 if na == nb else 0.0
    return float(np.dot(a, b) / (na * nb))


class GpuProfiler:
    """Drives one DeviceModel over a calibration set of prompts."""

    def __init__(self, dev: DeviceModel, prompts, bits: int = 4):
        self.dev = dev
        self.prompts = [np.ascontiguousarray(p, np.int32) for p in prompts]
        if not self.prompts:
            raise ValueError("profiler: calibration batch is empty")
        self.bits = bits
        self.L = dev.shape["L"]
        self.max_n = max(len(p) for p in self.prompts)
        nb = (self.max_n + 15) // 16
        self.block_ids = np.arange(1 << 20, (1 << 20) + nb, dtype=np.int64)
        dev.kv_attach(int(self.block_ids[0]), nb)
        dev.hist_reserve(1, self.max_n + 2)
        self.forwards = 0

    def close(self):
        self.dev.kv_detach(self.block_ids.tolist())

    def _set(self, quantized: set):
        """Brings every layer to its target precision through the LayerSwapper."""
        for l in range(self.L):
            want = self.bits if l in quantized else 16
            if self.dev.layer_bits(l) != want:
                t = self.dev.swap_begin(l, want)
                self.dev.swap_wait(t)
                self.dev.swap_commit(t)

    def _trace(self, p: np.ndarray) -> np.ndarray:
        self.dev.hist_write(0, 0, p)
        h, _ = self.dev.prefill_trace(0, len(p), self.block_ids, want_logits=False)
        self.forwards += 1
        return h

    def traces(self, quantized: set):
        self._set(quantized)
        return [self._trace(p) for p in self.prompts]

    def layer_transformation_scores(self, full_traces=None):
        tr = full_traces or self.traces(set())
        return [float(np.mean([_cos(h[p + 1], h[p]) for h in tr])) for p in range(self.L)]

    def layer_replacement_scores(self, full_traces=None):
        tr = full_traces or self.traces(set())
        out = []
        for p in range(self.L):
            # only layer p quantized: its input equals the full-precision trace's
            qt = self.traces({p})
            out.append(float(np.mean([_cos(f[p + 1], q[p + 1]) for f, q in zip(tr, qt)])))
        return out

    def greedy_sequence(self, weights: dict | None = None) -> dict:
        w = dict(DEFAULT_WEIGHTS, **(weights or {}))
        if min(w.values()) < 0 or not any(w.values()):
            raise ValueError("greedy_sequence: weights must be non-negative and not all zero")
        full = self.traces(set())
        lts = self.layer_transformation_scores(full)
        lrs = self.layer_replacement_scores(full)
        quantized: set = set()
        order, per_step, mds_log = [], [], []
        base = [h[self.L] for h in full]
        for _ in range(self.L):
            best, best_score, best_final = -1, -np.inf, None
            for j in range(self.L):
                if j in quantized:
                    continue
                cand = [h[self.L] for h in self.traces(quantized | {j})]
                mds = float(np.mean([_cos(b, c) for b, c in zip(base, cand)]))
                lis = w["alpha1"] * lts[j] + w["alpha2"] * lrs[j] + w["beta"] * mds
                if lis > best_score:  # ties resolve to the lowest index
                    best, best_score, best_final = j, lis, cand
            order.append(best)
            per_step.append(best_score)
            quantized.add(best)
            base = best_final  # the next round's baseline: Q + {best}
            mds_log.append(best_score)
        self._set(set())
        return {"order": order, "per_step_lis": per_step, "bits": self.bits, "kind": "lis_greedy", "weights": w,
                "lts": lts, "lrs": lrs}
