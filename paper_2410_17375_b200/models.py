"""Device models behind the reference's model plug-in interface.

The reference's compute boundary is ``MockModel`` (pkg/src/specdec/models.py:85-200):
``init_state / next_token / advance / rollback / verify_tokens`` over a
``ModelState`` owned by exactly one model.  ``CudaModel`` keeps that interface
and semantics (purity of ``next_token``/``verify_tokens``, crop range,
validation, ownership) while the state -- token prefix, KV cache or hash
chain -- lives in HBM and every prediction is computed by libamusd kernels.

Bs=1 by design: a device model holds ONE live sequence; ``init_state`` starts
a new one and invalidates older ``ModelState`` handles.

Families
--------
HashChainModel / AgreementDraftModel / make_agreement_pair
    splitmix64 hash-chain test doubles computed on the GPU,
    bit-identical to models.py:203-314.
TransformerModel
    Llama-style decoder (RMSNorm, RoPE theta=500000, GQA, SwiGLU), fp32 or
    bf16 weights, random-init or caller-provided.
AgreementDraft
    wraps a draft TransformerModel with the reference's agreement coin
    keyed on the prefix hash (models.py:271-314).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field, replace
from typing import Sequence

import torch

from . import _lib as L
from .errors import InvalidInputError

__all__ = [
    "ModelState", "CudaModel", "HashChainModel", "AgreementDraftModel", "ScriptedModel", "make_agreement_pair",
    "TransformerConfig", "TransformerModel", "AgreementDraft", "device_stream",
]


def device_stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def settle(device) -> None:
    """Wait for allocation/initialisation work torch queued on its current stream.

    Device buffers are created with torch (zero fills, weight init) on the
    current stream, but the decode loops run on their own non-blocking
    streams; without this a late fill could land on live state."""
    torch.cuda.current_stream(device).synchronize()


@dataclass
class ModelState:
    """Handle on a model's device-resident sequence (models.py:58-82)."""
    prompt_length: int
    owner: "CudaModel" = field(repr=False, compare=False)
    generation: int = 0

    @property
    def prefix_length(self) -> int:
        self.owner._check_owner(self)
        out = C.c_int()
        L.check(L.load().amusd_prefix_length(self.owner._h, C.byref(out)))
        return out.value


class CudaModel:
    """MockModel-compatible base over a libamusd model handle."""

    coin_mode = L.COIN_NONE
    agreement_rho = None
    coin_seed = 0

    def __init__(self, vocab_size: int, eos_token: int, device=None):
        if vocab_size < 2:
            raise InvalidInputError(f"vocab_size must be >= 2, got {vocab_size}")
        if not 0 <= eos_token < vocab_size:
            raise InvalidInputError(f"eos_token must be in [0, {vocab_size}), got {eos_token}")
        self.vocab_size = vocab_size
        self.eos_token = eos_token
        self.device = torch.device(device if device is not None else "cuda")
        self._h = C.c_void_p()
        self._generation = 0
        self._fresh = None  # prompt of an untouched init_state (lets engines skip a second prefill)
        self._lib = L.load()

    # ------------------------------------------------------------ lifecycle
    def init_state(self, prompt: Sequence[int]) -> ModelState:
        """Fresh state conditioned on ``prompt`` (models.py:109-118); prefill on the GPU."""
        if len(prompt) == 0:
            raise InvalidInputError("prompt must be non-empty")
        self._validate_tokens(prompt)
        arr = L.int_array(prompt)
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_init_state(self._h, arr, len(prompt), device_stream(self.device)))
        self._generation += 1
        self._fresh = tuple(prompt)
        st = ModelState(len(prompt), self, self._generation)
        st.prompt = list(prompt)
        return st

    def next_token(self, state: ModelState) -> int:
        """Greedy prediction for position prefix_length + 1; no logical mutation (models.py:120-123)."""
        self._check_owner(state)
        out = C.c_int32()
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_next_token(self._h, C.byref(out), device_stream(self.device)))
        return int(out.value)

    def advance(self, state: ModelState, tokens: Sequence[int]) -> None:
        """Extend the prefix (models.py:125-131); the forward happens lazily on the GPU."""
        self._check_owner(state)
        if len(tokens) == 0:
            raise InvalidInputError("advance requires at least one token")
        self._validate_tokens(tokens)
        self._fresh = None
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_advance(self._h, L.int_array(tokens), len(tokens), device_stream(self.device)))

    def rollback(self, state: ModelState, position: int) -> None:
        """Crop to ``position`` tokens: a cache-length truncate (models.py:133-149)."""
        self._check_owner(state)
        self._fresh = None
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_rollback(self._h, int(position), device_stream(self.device)))

    def verify_tokens(self, state: ModelState, candidates: Sequence[int]) -> list:
        """Teacher-forced predictions for every candidate position (models.py:151-169)."""
        self._check_owner(state)
        if len(candidates) == 0:
            raise InvalidInputError("verify_tokens requires at least one candidate")
        self._validate_tokens(candidates)
        out = (C.c_int32 * len(candidates))()
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_verify_tokens(self._h, L.int_array(candidates), len(candidates), out,
                                                  device_stream(self.device)))
        return [int(v) for v in out]

    # ---------------------------------------------------------- validation
    def _validate_tokens(self, tokens: Sequence[int]) -> None:
        for tok in tokens:  # models.py:191-196
            if not isinstance(tok, int) or not 0 <= tok < self.vocab_size:
                raise InvalidInputError(f"token {tok!r} out of vocabulary range [0, {self.vocab_size})")

    def _check_owner(self, state: ModelState) -> None:
        if not isinstance(state, ModelState) or state.owner is not self:
            raise InvalidInputError("state belongs to a different model")
        if state.generation != self._generation:
            raise InvalidInputError("state was superseded by a newer init_state (device models hold one sequence)")

    @property
    def handle(self):
        return self._h

    def set_max_grid(self, sms: int) -> None:
        """Cap the persistent forward's grid at `sms` CTAs (0 = all SMs): models sharing one GPU
        whose forwards wait on each other (tensor-parallel ranks, co-located drafts) must be
        co-resident."""
        L.check(self._lib.amusd_model_set_max_grid(self._h, int(sms)))

    def kernels_per_forward(self) -> int:
        raise NotImplementedError

    def __del__(self):
        try:
            if self._h:
                L.load().amusd_model_destroy(self._h)
        except Exception:
            pass


class HashChainModel(CudaModel):
    """Greedy next token = h_n mod V over the splitmix64 chain (models.py:203-268), on the GPU."""

    def __init__(self, seed: int, vocab_size: int, eos_token: int, exclude_eos: bool = False,
                 max_seq: int = 4096, device=None, _rho: float = -1.0):
        super().__init__(vocab_size, eos_token, device)
        if exclude_eos and vocab_size < 3:
            raise InvalidInputError("exclude_eos requires vocab_size >= 3")
        self.seed = seed & ((1 << 64) - 1)
        self.exclude_eos = exclude_eos
        self.max_seq = max_seq
        nbytes = self._lib.amusd_hash_state_bytes(max_seq)
        self._state = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        L.check(self._lib.amusd_hash_create(C.byref(self._h), self.seed, vocab_size, eos_token, int(exclude_eos),
                                            float(_rho), max_seq, C.c_void_p(self._state.data_ptr()), nbytes))
        settle(self.device)

    def kernels_per_forward(self) -> int:
        return 1


class AgreementDraftModel(HashChainModel):
    """Draft member of an agreement pair (models.py:271-314): same chain,
    agrees with probability rho via the prefix-keyed coin."""

    def __init__(self, seed: int, agreement_rho: float, vocab_size: int, eos_token: int,
                 exclude_eos: bool = False, max_seq: int = 4096, device=None):
        if not 0.0 <= agreement_rho <= 1.0:
            raise InvalidInputError(f"agreement_rho must be in [0, 1], got {agreement_rho}")
        super().__init__(seed, vocab_size, eos_token, exclude_eos, max_seq, device, _rho=agreement_rho)
        self.agreement_rho = agreement_rho


class ScriptedModel(CudaModel):
    """Prediction depends only on the absolute position (models.py:317-346), on the GPU:
    ``script[i]`` is the token at 1-based absolute position ``i + 1`` (cycling), and
    ``eos_position`` forces ``eos_token`` there -- the reference's eos edge-case model."""

    def __init__(self, script: Sequence[int], vocab_size: int, eos_token: int, eos_position: int | None = None,
                 max_seq: int = 4096, device=None):
        super().__init__(vocab_size, eos_token, device)
        if len(script) == 0:
            raise InvalidInputError("script must contain at least one token")
        self._validate_tokens(script)
        if eos_position is not None and eos_position < 1:
            raise InvalidInputError(f"eos_position must be >= 1, got {eos_position}")
        self.script = list(script)
        self.eos_position = eos_position
        nbytes = self._lib.amusd_scripted_state_bytes(max_seq, len(script))
        self._state = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        settle(self.device)
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_scripted_create(C.byref(self._h), L.int_array(script), len(script), vocab_size,
                                                    eos_token, eos_position or 0, max_seq,
                                                    C.c_void_p(self._state.data_ptr()), nbytes,
                                                    device_stream(self.device)))

    def kernels_per_forward(self) -> int:
        return 1


def make_agreement_pair(seed: int, rho: float, vocab_size: int, eos_token: int, exclude_eos: bool = False,
                        max_seq: int = 4096, device=None):
    """(draft, verify) with per-position agreement rho (models.py:349-365)."""
    if not 0.0 <= rho <= 1.0:
        raise InvalidInputError(f"rho must be in [0, 1], got {rho}")
    verify = HashChainModel(seed, vocab_size, eos_token, exclude_eos, max_seq, device)
    draft = AgreementDraftModel(seed, rho, vocab_size, eos_token, exclude_eos, max_seq, device)
    return draft, verify


# ---------------------------------------------------------------- transformer

@dataclass(frozen=True)
class TransformerConfig:
    """Llama-style decoder shape."""
    vocab_size: int
    d_model: int
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn: int
    max_seq: int = 1024
    dtype: str = "bf16"
    eos_token: int = 2
    exclude_eos: bool = True
    norm_eps: float = 1e-5
    rope_theta: float = 500000.0
    tied: bool = False
    use_tensor_cores: bool = True

    # presets (vocab 32000 / eos 2 pinned from the reference CLI defaults, cli.py:72-81)
    @classmethod
    def tiny_draft(cls, **kw):
        return cls(**{**dict(vocab_size=32000, d_model=256, n_layers=2, n_heads=4, n_kv_heads=2, head_dim=64,
                             ffn=768, tied=True, max_seq=512), **kw})

    @classmethod
    def tiny_verify(cls, **kw):
        return cls(**{**dict(vocab_size=32000, d_model=512, n_layers=4, n_heads=8, n_kv_heads=4, head_dim=64,
                             ffn=1536, tied=True, max_seq=512), **kw})

    @classmethod
    def llama_1b(cls, **kw):  # Llama-3.2-1B shape
        return cls(**{**dict(vocab_size=128256, d_model=2048, n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64,
                             ffn=8192, tied=True), **kw})

    @classmethod
    def llama_8b(cls, **kw):  # Llama-3.1-8B shape
        return cls(**{**dict(vocab_size=128256, d_model=4096, n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128,
                             ffn=14336, tied=False), **kw})

    @classmethod
    def llama_70b(cls, **kw):  # Llama-3.1-70B shape
        return cls(**{**dict(vocab_size=128256, d_model=8192, n_layers=80, n_heads=64, n_kv_heads=8, head_dim=128,
                             ffn=28672, tied=False), **kw})

    @property
    def qkv_rows(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def param_count(self) -> int:
        d, hd = self.d_model, self.head_dim
        per_layer = self.qkv_rows * d + d * self.n_heads * hd + 3 * d * self.ffn + 2 * d
        head = 0 if self.tied else self.vocab_size * d
        return self.vocab_size * d + head + self.n_layers * per_layer + d

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    def step_weight_bytes(self) -> int:
        """Algorithmic weight bytes one forward streams (embedding rows excluded, LM head included)."""
        d, hd = self.d_model, self.head_dim
        per_layer = self.qkv_rows * d + d * self.n_heads * hd + 3 * d * self.ffn + 2 * d
        return (self.n_layers * per_layer + self.vocab_size * d + d) * self.elem_bytes

    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * self.elem_bytes


def rope_tables(cfg: TransformerConfig):
    """fp32 cos/sin [max_seq][head_dim/2], computed in float64 (HF rotate_half convention)."""
    half = cfg.head_dim // 2
    inv = 1.0 / (cfg.rope_theta ** (torch.arange(0, half, dtype=torch.float64) * 2.0 / cfg.head_dim))
    ang = torch.arange(cfg.max_seq, dtype=torch.float64)[:, None] * inv[None, :]
    return torch.cos(ang).float(), torch.sin(ang).float()


def weight_names(cfg: TransformerConfig) -> list:
    names = ["embed", "final_norm"] + ([] if cfg.tied else ["lm_head"])
    for l in range(cfg.n_layers):
        names += [f"layers.{l}.{n}" for n in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate", "wup", "wdown")]
    return names


def weight_shape(cfg: TransformerConfig, name: str) -> tuple:
    d = cfg.d_model
    leaf = name.split(".")[-1]
    return {
        "embed": (cfg.vocab_size, d), "lm_head": (cfg.vocab_size, d), "final_norm": (d,),
        "attn_norm": (d,), "mlp_norm": (d,), "wqkv": (cfg.qkv_rows, d), "wo": (d, cfg.n_heads * cfg.head_dim),
        "wgate": (cfg.ffn, d), "wup": (cfg.ffn, d), "wdown": (d, cfg.ffn),
    }[leaf]


def synthetic_weight(config: TransformerConfig, i: int, name: str, tdt, seed: int, std: float, device):
    """Weight `name` (index i of weight_names) of the seeded synthetic model, filled on the GPU:
    uniform with the given std from a splitmix64 counter stream (amusd_fill_uniform), norms = 1."""
    t = torch.empty(weight_shape(config, name), dtype=tdt, device=device)
    if name.endswith("norm"):
        t.fill_(1.0)
    else:
        sub = (seed * 0x9E3779B97F4A7C15 + (i + 1) * 0xD1B54A32D192ED03) & ((1 << 64) - 1)
        dt = L.BF16 if tdt == torch.bfloat16 else L.F32
        with torch.cuda.device(device):
            L.check(L.load().amusd_fill_uniform(C.c_void_p(t.data_ptr()), dt, t.numel(), sub,
                                                std * math.sqrt(3.0), device_stream(device)))
    return t


class TransformerModel(CudaModel):
    """Llama-style decoder whose forwards are libamusd CUDA kernels."""

    def __init__(self, config: TransformerConfig, weights: dict | None = None, seed: int = 0,
                 device=None, init_std: float = 0.02, keep_row_major: bool = True, prefill: bool = True):
        super().__init__(config.vocab_size, config.eos_token, device)
        if config.dtype not in ("bf16", "fp32"):
            raise InvalidInputError(f"dtype must be 'bf16' or 'fp32', got {config.dtype!r}")
        if config.n_layers > L.MAX_LAYERS:
            raise InvalidInputError("too many layers")
        self.config = config
        self.seed = seed
        tdt = torch.bfloat16 if config.dtype == "bf16" else torch.float32
        self._synth = None
        if weights is None:
            weights = self._synthetic(tdt, seed, init_std)
            self._synth = (tdt, seed, init_std)
        else:
            weights = {k: v.to(device=self.device, dtype=tdt).contiguous() for k, v in weights.items()}
        for n in weight_names(config):
            if n not in weights:
                raise InvalidInputError(f"missing weight {n}")
            if tuple(weights[n].shape) != weight_shape(config, n):
                raise InvalidInputError(f"weight {n} has shape {tuple(weights[n].shape)}, "
                                        f"expected {weight_shape(config, n)}")
        self.weights = weights
        cos, sin = rope_tables(config)
        self.rope_cos, self.rope_sin = cos.to(self.device), sin.to(self.device)
        cfg = L.TfConfig(vocab=config.vocab_size, d_model=config.d_model, n_layers=config.n_layers,
                         n_heads=config.n_heads, n_kv_heads=config.n_kv_heads, head_dim=config.head_dim,
                         ffn=config.ffn, max_seq=config.max_seq, dtype=L.BF16 if config.dtype == "bf16" else L.F32,
                         eos_token=config.eos_token, exclude_eos=int(config.exclude_eos), norm_eps=config.norm_eps,
                         use_tensor_cores=int(config.use_tensor_cores))
        w = L.TfWeights()
        p = lambda t: C.c_void_p(t.data_ptr())
        w.embed = p(weights["embed"])
        w.lm_head = p(weights["embed"] if config.tied else weights["lm_head"])
        w.final_norm = p(weights["final_norm"])
        w.rope_cos, w.rope_sin = p(self.rope_cos), p(self.rope_sin)
        for l in range(config.n_layers):
            for leaf in ("attn_norm", "wqkv", "wo", "mlp_norm", "wgate", "wup", "wdown"):
                getattr(w, leaf)[l] = weights[f"layers.{l}.{leaf}"].data_ptr()
        self._cfg_c, self._w_c = cfg, w
        nbytes = self._lib.amusd_tf_state_bytes(C.byref(cfg))
        self._state = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        L.check(self._lib.amusd_tf_create(C.byref(self._h), C.byref(cfg), C.byref(w),
                                          C.c_void_p(self._state.data_ptr()), nbytes))
        settle(self.device)
        self.row_major = True
        self._prefill = None
        if prefill and config.dtype == "bf16" and config.use_tensor_cores and config.max_seq >= 128:
            self.set_prefill(True)
        if not keep_row_major:
            self.release_row_major()

    def set_prefill(self, on: bool) -> None:
        """Attach (or detach) the compute-bound prompt prefill: init_state of
        >= 64-position prompts runs as dense tcgen05 GEMMs over all prompt tokens plus a causal
        attention instead of 16-row decode forwards.  Workspace ~ max_seq x (d, ffn, qkv) HBM."""
        if not on:
            L.check(self._lib.amusd_model_set_prefill(self._h, None, 0, 0))
            self._prefill = None
            return
        n = self.config.max_seq
        nbytes = self._lib.amusd_prefill_bytes(self._h, n)
        if nbytes == 0:
            raise InvalidInputError("this model has no prefill path")
        buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_model_set_prefill(self._h, C.c_void_p(buf.data_ptr()), nbytes, n))
        self._prefill = buf

    def release_row_major(self) -> None:
        """Free the row-major layer weights (the persistent forward streams only its
        tile-contiguous copy): halves the model's HBM (8B: 16 GB).  Only the persistent
        path stays selectable; ``host_weights`` regenerates synthetic weights by seed."""
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_model_release_row_major(self._h))
        keep = {"embed", "final_norm"} | {n for n in self.weights if n.endswith("norm")}
        self._dropped = [n for n in self.weights if n not in keep]
        for n in self._dropped:
            del self.weights[n]
        self.row_major = False
        torch.cuda.empty_cache()
    def _synthetic_one(self, i: int, n: str, tdt, seed: int, std: float):
        return synthetic_weight(self.config, i, n, tdt, seed, std, self.device)

    def _synthetic(self, tdt, seed: int, std: float) -> dict:
        """Deterministic random init on the GPU: uniform with the given std, norms = 1."""
        return {n: self._synthetic_one(i, n, tdt, seed, std) for i, n in enumerate(weight_names(self.config))}

    PATHS = {"persistent": L.PATH_PERSISTENT, "kernels": L.PATH_KERNELS, "simt": L.PATH_SIMT,
             "decode": L.PATH_DECODE, "cluster": L.PATH_CLUSTER}

    def set_path(self, path: str) -> None:
        """Select the forward implementation: 'persistent' (one tcgen05 launch per forward,
        default), 'decode' (one persistent SIMT GEMV launch per forward -- the draft's path:
        its forwards carry 1-2 rows), 'kernels' (per-kernel tcgen05) or 'simt'.  Sessions
        capture the path when they first launch an engine."""
        if path not in self.PATHS:
            raise InvalidInputError(f"unknown forward path {path!r}")
        if path == "decode" and getattr(self, "_decode_w", None) is None:
            nbytes = self._lib.amusd_decode_bytes(self._h)
            if nbytes == 0:
                raise InvalidInputError("this model's shapes do not take the decode forward")
            buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            with torch.cuda.device(self.device):
                L.check(self._lib.amusd_model_set_decode(self._h, C.c_void_p(buf.data_ptr()), nbytes))
            self._decode_w = buf   # decode-layout weights (~ the model's weight bytes), owned here
        if path == "cluster" and getattr(self, "_cluster_w", None) is None:
            nbytes = self._lib.amusd_cluster_bytes(self._h)
            if nbytes == 0:
                raise InvalidInputError("this model's shapes do not take the cluster decode forward")
            buf = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            with torch.cuda.device(self.device):
                L.check(self._lib.amusd_model_set_cluster(self._h, C.c_void_p(buf.data_ptr()), nbytes))
            self._cluster_w = buf
        L.check(self._lib.amusd_model_set_path(self._h, self.PATHS[path]))
        self.path = path

    def kernels_per_forward(self) -> int:
        c = self.config
        tc = c.dtype == "bf16" and c.use_tensor_cores
        if tc and getattr(self, "path", "persistent") in ("persistent", "decode", "cluster"):
            return 1
        return 1 + 5 * c.n_layers + 2

    def last_logits(self, rows: int = 1):
        """fp32 logits of the last `rows` forwarded rows of the latest API forward (parity/debug)."""
        out = torch.empty((rows, self.vocab_size), dtype=torch.float32)
        with torch.cuda.device(self.device):
            L.check(self._lib.amusd_last_logits(self._h, C.cast(out.data_ptr(), C.POINTER(C.c_float)), rows,
                                                device_stream(self.device)))
        return out

    def host_weights(self) -> dict:
        """fp32 numpy copies of every weight (for the CPU oracle / baseline).  Released
        synthetic weights are regenerated one at a time by the same device fill."""
        out = {}
        for i, n in enumerate(weight_names(self.config)):
            if n in self.weights:
                out[n] = self.weights[n].float().cpu().numpy()
            elif self._synth is not None:
                out[n] = self._synthetic_one(i, n, *self._synth).float().cpu().numpy()
            else:
                raise InvalidInputError(f"weight {n} was released (keep_row_major=False) and is not synthetic")
        return out


class AgreementDraft:
    """A draft TransformerModel plus the reference's agreement coin.

    While the draft's prefix equals the verify model's canonical greedy path,
    it publishes the canonical token with probability rho (coin
    ``splitmix64(h ^ AGREE_SALT) < rho * 2**64`` on the prefix hash h, seeded
    with ``coin_seed``) and otherwise the reference's "different token"
    draw -- exactly AgreementDraftModel's acceptance model (models.py:271-314),
    so rho is a controlled input.  Off the canonical path it publishes its own
    greedy token.  The draft forward always runs in full (real cost).  The
    engines compute the canonical path with the verify model on the GPU.

    MockModel methods delegate to the wrapped model (raw greedy tokens).
    """

    coin_mode = L.COIN_CANON

    def __init__(self, model: TransformerModel, rho: float, coin_seed: int = 1234):
        if not 0.0 <= rho <= 1.0:
            raise InvalidInputError(f"rho must be in [0, 1], got {rho}")
        self.model = model
        self.agreement_rho = rho
        self.coin_seed = coin_seed & ((1 << 64) - 1)

    def __getattr__(self, name):
        return getattr(self.model, name)
