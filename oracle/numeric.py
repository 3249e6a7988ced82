"""CPU numeric oracle for the hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker; the product path never imports it.

The reference (/root/reference/proj) is a discrete-event simulator: its GPU is
the latency formula oracle_latency (perf_model.cpp:56-96) and it computes no
attention outputs, logits or KV bytes. This module therefore restates the
*semantics* the reference's BatchPlan encodes
as a plain fp32 Llama-style decoder over a KV store keyed by (request,
position):

  * decode entry (P=1, C): query position C-1, keys [0, C)      (scheduler.cpp:187-192)
  * prefill entry (P, C): queries [C, C+P), keys [0, C+P), causal (scheduler.cpp:151)
  * recompute entry: the positions of the re-materialized pages  (kv_cache.cpp:76-107)
  * online entries form a prefix of the plan                     (scheduler.cpp:183-317)

Numeric parity is therefore builder-pinned, not reference-pinned ("parity
unpinned" for logits/attention in the sense of the task statement); the
control-plane parity (page tables, checkpoint byte volumes, scheduling
decisions) is pinned by the compiled reference itself (oracle/Makefile).

Weights and teacher-forced token ids come from the same splitmix64 hashes as
paper_2410_01228_b200/csrc/common.cuh (mix64 = rng.hpp:11-16 of the reference),
so both sides see identical bf16 parameters.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _u64(x) -> np.ndarray:
    return np.asarray(x, dtype=np.uint64)


def mix64(x) -> np.ndarray:
    """splitmix64 finalizer (reference rng.hpp:11-16)."""
    with np.errstate(over="ignore"):
        x = _u64(x) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def token_id(seed: int, req, pos, vocab: int) -> np.ndarray:
    """Teacher-forced synthetic id(req, pos)."""
    with np.errstate(over="ignore"):
        inner = _u64(req) * np.uint64(0x100000001B3) + _u64(pos)
        h = mix64(np.uint64(seed) ^ mix64(inner))
    return (h % np.uint64(vocab)).astype(np.int64)


def hash_uniform(seed: int, tensor: int, idx) -> np.ndarray:
    """Uniform in [-1, 1) as float32, bit-identical to csk::hash_uniform."""
    with np.errstate(over="ignore"):
        t = np.uint64(tensor) * np.uint64(0x9E3779B97F4A7C15)
        h = mix64(np.uint64(seed) ^ mix64(t ^ mix64(_u64(idx))))
    top = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return top.astype(np.float32) * np.float32(1.0 / 8388608.0)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even), returned as float32."""
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16) << np.uint64(16)
    return b.astype(np.uint32).view(np.float32)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return (bf16_round(x).view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bf16_bits(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << np.uint32(16)).view(np.float32)


TENSOR_EMB, TENSOR_LM, TENSOR_FINAL_NORM = 1, 2, 3
W_ATTN_NORM, W_QKV, W_O, W_MLP_NORM, W_GU, W_D = 0, 1, 2, 3, 4, 5


def _tid(layer: int, which: int) -> int:
    return 1000 + layer * 16 + which


@dataclass
class ModelShape:
    num_layers: int = 2
    hidden: int = 256
    n_heads: int = 4
    n_kv_heads: int = 4
    head_dim: int = 64
    ffn: int = 512
    vocab: int = 1024
    rope_theta: float = 10000.0
    rms_eps: float = 1e-5
    weight_seed: int = 1
    token_seed: int = 1

    @classmethod
    def from_cfg(cls, cfg) -> "ModelShape":
        return cls(cfg.num_layers, cfg.hidden, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.ffn, cfg.vocab,
                   cfg.rope_theta, cfg.rms_eps, cfg.weight_seed, cfg.token_seed)


def _matrix(seed: int, tensor: int, rows: int, cols: int, scale: float, offset: float) -> np.ndarray:
    idx = np.arange(rows * cols, dtype=np.uint64)
    u = hash_uniform(seed, tensor, idx)
    v = (np.float32(offset) + (np.float32(scale) * u).astype(np.float32)).astype(np.float32)
    return bf16_round(v).reshape(rows, cols)


class Weights:
    """Unsharded random-init weights, identical to the engine's (csrc/engine.cu)."""

    def __init__(self, s: ModelShape):
        self.s = s
        ws = np.float32(np.float32(0.02) * np.float32(1.7320508))  # 0.02f * 1.7320508f
        seed = s.weight_seed
        H, D = s.hidden, s.head_dim
        self.emb = _matrix(seed, TENSOR_EMB, s.vocab, H, ws, 0.0)
        self.lm_head = _matrix(seed, TENSOR_LM, s.vocab, H, ws, 0.0)
        self.final_norm = _matrix(seed, TENSOR_FINAL_NORM, 1, H, 0.1, 1.0)[0]
        self.attn_norm, self.mlp_norm, self.wqkv, self.wo, self.wgu, self.wd = [], [], [], [], [], []
        for l in range(s.num_layers):
            self.attn_norm.append(_matrix(seed, _tid(l, W_ATTN_NORM), 1, H, 0.1, 1.0)[0])
            self.mlp_norm.append(_matrix(seed, _tid(l, W_MLP_NORM), 1, H, 0.1, 1.0)[0])
            self.wqkv.append(_matrix(seed, _tid(l, W_QKV), (s.n_heads + 2 * s.n_kv_heads) * D, H, ws, 0.0))
            self.wo.append(_matrix(seed, _tid(l, W_O), H, s.n_heads * D, ws, 0.0))
            self.wgu.append(_matrix(seed, _tid(l, W_GU), 2 * s.ffn, H, ws, 0.0))
            self.wd.append(_matrix(seed, _tid(l, W_D), H, s.ffn, ws, 0.0))


def rmsnorm(x: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    ms = np.mean(x.astype(np.float32) ** 2, axis=-1, keepdims=True)
    return (x / np.sqrt(ms + np.float32(eps))).astype(np.float32) * w


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """Rotate-half RoPE over the last axis; x [T, H, D], pos [T]."""
    D = x.shape[-1]
    half = D // 2
    j = np.arange(half, dtype=np.float32)
    inv = np.power(np.float32(theta), np.float32(-2.0) * j / np.float32(D)).astype(np.float32)
    ang = pos.astype(np.float32)[:, None] * inv[None, :]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1).astype(np.float32)


@dataclass
class Entry:
    """coserve::BatchEntry (perf_model.hpp:15-21) plus recompute positions."""
    request_id: int
    compute_tokens: int
    context_tokens: int
    kind: int = 0  # 0 prefill, 1 decode, 2 recompute (EntryKind order)
    online: bool = False
    positions: Optional[List[int]] = None  # recompute only


def entry_positions(e: Entry) -> np.ndarray:
    if e.kind == 1:
        return np.array([e.context_tokens - 1], dtype=np.int64)
    if e.kind == 0:
        return np.arange(e.context_tokens, e.context_tokens + e.compute_tokens, dtype=np.int64)
    assert e.positions is not None and len(e.positions) == e.compute_tokens
    return np.array(e.positions, dtype=np.int64)


class KVStore:
    """K/V per (request, layer) indexed by absolute position (bf16 values)."""

    def __init__(self, s: ModelShape):
        self.s = s
        self.k: Dict[Tuple[int, int], np.ndarray] = {}
        self.v: Dict[Tuple[int, int], np.ndarray] = {}

    def _ensure(self, req: int, layer: int, n: int):
        key = (req, layer)
        cur = self.k.get(key)
        if cur is None or cur.shape[0] < n:
            cap = max(n, 16 if cur is None else 2 * cur.shape[0])
            nk = np.zeros((cap, self.s.n_kv_heads, self.s.head_dim), np.float32)
            nv = np.zeros_like(nk)
            if cur is not None:
                nk[: cur.shape[0]] = cur
                nv[: cur.shape[0]] = self.v[key]
            self.k[key], self.v[key] = nk, nv
        return self.k[key], self.v[key]

    def write(self, req: int, layer: int, pos: np.ndarray, k: np.ndarray, v: np.ndarray):
        K, V = self._ensure(req, layer, int(pos.max()) + 1)
        K[pos] = k
        V[pos] = v

    def read(self, req: int, layer: int, n: int):
        K, V = self._ensure(req, layer, n)
        return K[:n], V[:n]


class Oracle:
    """fp32 forward with bf16 storage points matching the engine's tensors."""

    def __init__(self, s: ModelShape, weights: Optional[Weights] = None, mimic_bf16: bool = True):
        self.s = s
        self.w = weights or Weights(s)
        self.kv = KVStore(s)
        self.mimic = mimic_bf16
        self.last_attn: Optional[np.ndarray] = None  # [T, Hq*D] of the last layer

    def _r(self, x):
        return bf16_round(x) if self.mimic else x.astype(np.float32)

    def forward(self, entries: Sequence[Entry]) -> np.ndarray:
        """Runs one plan; returns logits [n_entries, vocab] (fp32) of each
        entry's last row, and updates the KV store for every query position."""
        s, w = self.s, self.w
        H, D, Hq, Hkv = s.hidden, s.head_dim, s.n_heads, s.n_kv_heads
        G = Hq // Hkv
        pos_list = [entry_positions(e) for e in entries]
        rows = np.concatenate(pos_list)
        reqs = np.concatenate([np.full(len(p), e.request_id, np.int64) for e, p in zip(entries, pos_list)])
        ids = token_id(s.token_seed, reqs, rows, s.vocab)
        x = w.emb[ids].astype(np.float32)
        starts = np.cumsum([0] + [len(p) for p in pos_list])
        scale = np.float32(1.0 / np.sqrt(D))
        add = None
        for l in range(s.num_layers):
            if add is not None:
                x = self._r(x + add)
            xn = self._r(rmsnorm(x, w.attn_norm[l], s.rms_eps))
            qkv = self._r(xn @ w.wqkv[l].T)
            q = qkv[:, : Hq * D].reshape(-1, Hq, D)
            k = qkv[:, Hq * D: (Hq + Hkv) * D].reshape(-1, Hkv, D)
            v = qkv[:, (Hq + Hkv) * D:].reshape(-1, Hkv, D)
            q = self._r(rope(q, rows, s.rope_theta))
            k = self._r(rope(k, rows, s.rope_theta))
            for e, i0, i1 in zip(entries, starts[:-1], starts[1:]):
                self.kv.write(e.request_id, l, rows[i0:i1], k[i0:i1], v[i0:i1])
            attn = np.zeros((len(rows), Hq, D), np.float32)
            for e, i0, i1 in zip(entries, starts[:-1], starts[1:]):
                p = rows[i0:i1]
                kv_len = int(p.max()) + 1
                K, V = self.kv.read(e.request_id, l, kv_len)
                qe = q[i0:i1].reshape(-1, Hkv, G, D)  # [P, Hkv, G, D]; head h = kvh*G + g
                Kt = np.ascontiguousarray(K.transpose(1, 2, 0))  # [Hkv, D, kv]
                sc = np.matmul(qe.transpose(1, 2, 0, 3), Kt[:, None]) * scale  # [Hkv, G, P, kv]
                mask = np.arange(kv_len)[None, :] > p[:, None]
                sc = np.where(mask[None, None], -np.inf, sc).astype(np.float32)
                sc = sc - sc.max(axis=-1, keepdims=True)
                pr = np.exp(sc)
                pr /= pr.sum(axis=-1, keepdims=True)
                o = np.matmul(pr, np.ascontiguousarray(V.transpose(1, 0, 2))[:, None])  # [Hkv, G, P, D]
                attn[i0:i1] = o.transpose(2, 0, 1, 3).reshape(-1, Hq, D)
            attn = self._r(attn.reshape(-1, Hq * D))
            self.last_attn = attn
            o = self._r(attn @ w.wo[l].T)
            x = self._r(x + o)
            xn = self._r(rmsnorm(x, w.mlp_norm[l], s.rms_eps))
            gu = self._r(xn @ w.wgu[l].T)
            g, u = gu[:, : s.ffn], gu[:, s.ffn:]
            act = self._r(g / (1.0 + np.exp(-g)) * u)
            add = self._r(act @ w.wd[l].T)
        x = self._r(x + add)
        last = starts[1:] - 1
        xl = self._r(rmsnorm(x[last], w.final_norm, s.rms_eps))
        return (xl @ w.lm_head.T).astype(np.float32)


def online_prefix_ok(entries: Sequence[Entry]) -> bool:
    seen_off = False
    for e in entries:
        if e.online and seen_off:
            return False
        seen_off |= not e.online
    return True
