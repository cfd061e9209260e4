"""B200-native AMUSD: asynchronous draft/verify speculative decoding on sm_100a.

Drop-in for the reference ``specdec`` decode path (pkg/src/specdec/__init__.py:71-122):
same entry points, config/result types, trace schema and error types; the
models' forwards, the accept/rollback logic and the draft<->verify mailbox
run as CUDA kernels from ``libamusd.so`` (include/amusd.h).
"""
from .errors import (
    ConfigError,
    InvalidInputError,
    InvalidRollbackError,
    ProtocolViolationError,
    SimulatorError,
    SpecDecError,
)
from .metrics import (
    ACTOR_DRAFT,
    ACTOR_VERIFY,
    DecodeStats,
    DecodeTrace,
    TraceEvent,
    busy_intervals,
    overlap_ms,
    summarize,
    trace_to_csv,
)
from .coordination import RollbackRequest, SharedDecodeState, TokenBuffer

__version__ = "0.1.0"


_LAZY = ("engines", "models")


def __getattr__(name):
    # device-facing modules import torch/libamusd lazily so that the pure host
    # pieces (errors, metrics, coordination) import without a GPU stack.
    import importlib
    if name.startswith("_"):  # private submodules (_lib) resolve through the import system
        raise AttributeError(name)
    if name in _LAZY:
        return importlib.import_module(f"{__name__}.{name}")
    for mod in _LAZY:
        m = importlib.import_module(f"{__name__}.{mod}")
        if name in m.__dict__:
            return m.__dict__[name]
    raise AttributeError(name)


__all__ = [
    "ACTOR_DRAFT", "ACTOR_VERIFY", "AgreementDraft", "AgreementDraftModel", "ConfigError", "CudaAsyncExecutor",
    "CudaModel", "DecodeConfig", "DecodeResult", "DecodeStats", "DecodeTrace", "DeviceSession", "HashChainModel",
    "InvalidInputError", "InvalidRollbackError", "ModelState", "ProtocolViolationError", "RollbackRequest",
    "ScriptedModel", "SharedDecodeState", "SimulatorError", "SpecDecError", "TokenBuffer", "TraceEvent", "TransformerConfig",
    "TransformerModel", "busy_intervals", "canonical_path", "decode_autoregressive", "decode_speculative_async",
    "decode_speculative_sync", "find_mismatch", "finalize_tokens", "make_agreement_pair", "overlap_ms",
    "summarize", "trace_to_csv",
]
