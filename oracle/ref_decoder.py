"""numpy fp32 Llama-style decoder -- TEST INFRASTRUCTURE ONLY (parity UNPINNED).

The reference has no transformer arithmetic, so
this restatement follows the public Llama-3 architecture and the
*interface/semantics* of the reference model plug-in (models.py:85-200):
``start`` = init_state, ``predict`` = next_token (pure), ``extend`` =
advance, ``crop`` = rollback, ``verify`` = verify_tokens (pure).  It plugs
into the restated engines in specdec_oracle.py.

Evaluation order mirrors the CUDA kernels so fp32 differences are rounding
only:  norm(x) W^T = rsqrt(mean(x^2)+eps) * ((x*g) W^T);  K/V are rounded to
the cache dtype before use;  first-index argmax with eos optionally masked
(models.py:256-261 analog).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .specdec_oracle import coin_token, mix64, rho_threshold


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bfloat16, returned as float32."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


@dataclass
class TfShape:
    vocab: int
    d: int
    layers: int
    heads: int
    kv_heads: int
    head_dim: int
    ffn: int
    eos: int = 2
    exclude_eos: bool = True
    eps: float = 1e-5
    theta: float = 500000.0
    kv_bf16: bool = False
    # bf16-faithful mode: round activations to bf16 exactly where the tcgen05 kernels do
    # (normed GEMM inputs bf16(h*g), attention output, SiLU*up product); accumulation fp32
    act_bf16: bool = False
    # float64 accumulation in every matmul (rounded to fp32 at the same points): a second
    # summation order, i.e. the fp32 noise floor the GPU parity tolerance is measured against
    acc64: bool = False


@dataclass
class DecState:
    prompt_len: int
    tokens: list
    k: list = field(default_factory=list)   # per layer [kv_heads, n, hd]
    v: list = field(default_factory=list)
    last_logits: np.ndarray | None = None


class RefDecoder:
    """fp32 decoder over host weights (names as paper_2410_17375_b200.models.weight_names)."""

    def __init__(self, shape: TfShape, weights: dict, tied: bool):
        self.s = shape
        self.w = {k: np.ascontiguousarray(v, dtype=np.float32) for k, v in weights.items()}
        self.lm = self.w["embed"] if tied else self.w["lm_head"]
        self.eos_token = shape.eos
        half = shape.head_dim // 2
        self.inv_freq = 1.0 / (shape.theta ** (np.arange(0, half, dtype=np.float64) * 2.0 / shape.head_dim))

    # ------------------------------------------------------------ arithmetic
    def _rope(self, x: np.ndarray, pos: np.ndarray) -> np.ndarray:
        """x [m, heads, hd], rotate_half convention, fp32 tables from float64 angles."""
        half = self.s.head_dim // 2
        ang = pos[:, None].astype(np.float64) * self.inv_freq[None, :]
        c = np.cos(ang).astype(np.float32)[:, None, :]
        s = np.sin(ang).astype(np.float32)[:, None, :]
        x1, x2 = x[..., :half], x[..., half:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)

    def _act(self, a):
        return bf16_round(a) if self.s.act_bf16 else a

    def _mm(self, x, W):
        if self.s.acc64:
            return (x.astype(np.float64) @ W.T.astype(np.float64)).astype(np.float32)
        return x @ W.T

    def _normed_matmul(self, h, g, W):
        inv = 1.0 / np.sqrt((h * h).mean(axis=1, keepdims=True) + np.float32(self.s.eps))
        return self._mm(self._act(h * g[None, :]), W) * inv.astype(np.float32)

    def _cast_kv(self, a):
        return bf16_round(a) if self.s.kv_bf16 else a

    def forward(self, st: DecState, toks, commit: bool = True) -> np.ndarray:
        """Forward `toks` at positions len(kv).. ; returns logits [m, vocab].

        commit=False leaves the state untouched (teacher forcing on scratch)."""
        s, w = self.s, self.w
        m = len(toks)
        n0 = st.k[0].shape[1] if st.k else 0
        pos = np.arange(n0, n0 + m)
        h = w["embed"][np.asarray(toks)].astype(np.float32)
        H, KV, hd = s.heads, s.kv_heads, s.head_dim
        grp = H // KV
        newk, newv = [], []
        for l in range(s.layers):
            p = f"layers.{l}."
            qkv = self._normed_matmul(h, w[p + "attn_norm"], w[p + "wqkv"])
            q = self._rope(qkv[:, : H * hd].reshape(m, H, hd), pos)
            k = self._cast_kv(self._rope(qkv[:, H * hd:(H + KV) * hd].reshape(m, KV, hd), pos))
            v = self._cast_kv(qkv[:, (H + KV) * hd:].reshape(m, KV, hd))
            kk = np.concatenate([st.k[l], k.transpose(1, 0, 2)], axis=1) if st.k else k.transpose(1, 0, 2)
            vv = np.concatenate([st.v[l], v.transpose(1, 0, 2)], axis=1) if st.v else v.transpose(1, 0, 2)
            newk.append(kk)
            newv.append(vv)
            scale = np.float32(1.0 / np.sqrt(np.float32(hd)))
            out = np.empty((m, H, hd), dtype=np.float32)
            for hh in range(H):
                g = hh // grp
                sc = (q[:, hh, :] @ kk[g].T) * scale                     # [m, n0+m]
                mask = np.arange(n0 + m)[None, :] > pos[:, None]
                sc = np.where(mask, -np.inf, sc)
                sc = np.exp(sc - sc.max(axis=1, keepdims=True))
                sc = sc / sc.sum(axis=1, keepdims=True)
                out[:, hh, :] = sc @ vv[g]
            h = h + self._mm(self._act(out.reshape(m, H * hd)), w[p + "wo"])
            x = self._act(h * w[p + "mlp_norm"][None, :])
            inv = (1.0 / np.sqrt((h * h).mean(axis=1, keepdims=True) + np.float32(s.eps))).astype(np.float32)
            gg = self._mm(x, w[p + "wgate"]) * inv
            uu = self._mm(x, w[p + "wup"]) * inv
            a = self._act((gg / (1.0 + np.exp(-gg))) * uu)
            h = h + self._mm(a, w[p + "wdown"])
        logits = self._normed_matmul(h, w["final_norm"], self.lm)
        self.scratch = (newk, newv)   # the KV this forward produced (ref_models reuses it on advance)
        if commit:
            st.k, st.v = newk, newv
            st.tokens.extend(int(t) for t in toks)
            st.last_logits = logits[-1]
        return logits

    def argmax(self, logits: np.ndarray) -> int:
        z = np.array(logits, dtype=np.float32, copy=True)
        if self.s.exclude_eos:
            z[self.s.eos] = -np.inf
        return int(np.argmax(z))  # numpy returns the first maximal index

    # -------------------------------------------- model interface (oracle)
    def start(self, prompt) -> DecState:
        st = DecState(len(prompt), [])
        self.forward(st, list(prompt))
        return st

    def predict(self, st: DecState) -> int:
        return self.argmax(st.last_logits)

    def extend(self, st: DecState, toks) -> None:
        self.forward(st, list(toks))

    def crop(self, st: DecState, n: int) -> None:
        if not st.prompt_len <= n <= len(st.tokens):
            raise ValueError("rollback out of range")
        if n == len(st.tokens):
            return
        last = st.tokens[n - 1]
        st.tokens = st.tokens[: n - 1]
        st.k = [k[:, : n - 1] for k in st.k]
        st.v = [v[:, : n - 1] for v in st.v]
        self.forward(st, [last])

    def verify(self, st: DecState, cands) -> list:
        preds = [self.predict(st)]
        if len(cands) > 1:
            lg = self.forward(st, list(cands[:-1]), commit=False)
            preds += [self.argmax(r) for r in lg]
        return preds


@dataclass
class CoinState:
    inner: DecState
    hashes: list

    @property
    def tokens(self):
        return self.inner.tokens

    @property
    def prompt_len(self):
        return self.inner.prompt_len


class CanonCoinDraft:
    """AgreementDraft restated: coin on the prefix hash, canonical token while
    on the canonical path, own greedy token off it (models.py:271-314 +
    SURVEY.md section 0.4).  Mirrors csrc/protocol.cu coin_pick."""

    def __init__(self, model: RefDecoder, canon: list, rho: float, coin_seed: int):
        self.m, self.canon, self.thr, self.seed = model, list(canon), rho_threshold(rho), coin_seed
        self.always = rho >= 1.0
        self.eos_token = model.eos_token
        self.vocab, self.eos, self.excl = model.s.vocab, model.s.eos, model.s.exclude_eos

    def _push(self, st: CoinState, toks):
        for t in toks:
            st.hashes.append(mix64(st.hashes[-1] ^ t))

    def start(self, prompt):
        st = CoinState(self.m.start(prompt), [mix64(self.seed)])
        self._push(st, prompt)
        return st

    def _on_path(self, toks) -> bool:
        n = len(toks)
        return n < len(self.canon) and toks == self.canon[:n]

    def predict(self, st: CoinState) -> int:
        n = len(st.tokens)
        if self._on_path(st.tokens):
            agreed = self.canon[n]
            if self.always:
                return agreed
            return coin_token(st.hashes[n], agreed, self.thr, self.vocab, self.eos, self.excl)
        return self.m.predict(st.inner)

    def extend(self, st, toks):
        self.m.extend(st.inner, toks)
        self._push(st, toks)

    def crop(self, st, n):
        self.m.crop(st.inner, n)
        del st.hashes[n + 1:]

    def verify(self, st, cands):
        out, toks = [], list(st.tokens)
        hs = list(st.hashes)
        base = self.m.verify(st.inner, cands)
        for j, c in enumerate(cands):
            n = len(toks)
            if n < len(self.canon) and toks == self.canon[:n]:
                a = self.canon[n]
                out.append(a if self.always else coin_token(hs[n], a, self.thr, self.vocab, self.eos, self.excl))
            else:
                out.append(base[j])
            toks.append(c)
            hs.append(mix64(hs[-1] ^ c))
        return out


def uniform_weights_like(shapes: dict, seed: int, std: float = 0.02) -> dict:
    """Host twin of amusd_fill_uniform for small models (splitmix64 counter stream)."""
    out = {}
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    for i, (name, shp) in enumerate(shapes.items()):
        n = int(np.prod(shp))
        if name.endswith("norm"):
            out[name] = np.ones(shp, dtype=np.float32)
            continue
        sub = (seed * 0x9E3779B97F4A7C15 + (i + 1) * 0xD1B54A32D192ED03) & ((1 << 64) - 1)
        x = (np.arange(n, dtype=np.uint64) + np.uint64(sub)) & M
        with np.errstate(over="ignore"):
            z = x + np.uint64(0x9E3779B97F4A7C15)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        u = (z >> np.uint64(40)).astype(np.float32) * np.float32(1.0 / 16777216.0)
        scale = np.float32(std * np.sqrt(3.0))
        out[name] = (scale * (np.float32(2.0) * u - np.float32(1.0))).reshape(shp).astype(np.float32)
    return out
