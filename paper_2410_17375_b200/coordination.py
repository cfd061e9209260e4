"""Host view of the draft/verify coordination record.

On the GPU the record is the HBM mailbox written by the protocol kernels
(csrc/internal.h ``MailboxHdr``; include/amusd.h).  This class keeps the
reference's host-side API (pkg/src/specdec/coordination.py:114-275) so the
executor plug-in contract holds: an executor leaves the verified stream in
``shared.V`` through ``publish_verified`` and the engine reads it back with
``verified_tokens()`` (engines.py:558-560).  After a device run the executor
mirrors the final mailbox state into this object.
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import InvalidInputError, ProtocolViolationError


@dataclass(frozen=True)
class RollbackRequest:
    """Correction notice: ``target`` = absolute position of the correction token (coordination.py:102-111)."""
    target: int
    correction_token: int


class TokenBuffer:
    """Append-only token list with a published length (coordination.py:39-99)."""

    def __init__(self, name: str, allow_truncate: bool = False) -> None:
        self.name = name
        self._tokens: list = []
        self._allow_truncate = allow_truncate

    def __len__(self) -> int:
        return len(self._tokens)

    def append(self, token: int) -> None:
        self._tokens.append(token)

    def extend(self, tokens) -> None:
        self._tokens.extend(tokens)

    def truncate_to(self, count: int) -> None:
        if not self._allow_truncate:
            raise ProtocolViolationError(f"buffer {self.name} is append-only")
        if not 0 <= count <= len(self._tokens):
            raise InvalidInputError(f"cannot truncate {self.name} of length {len(self._tokens)} to {count}")
        del self._tokens[count:]

    def token_at(self, index: int) -> int:
        if not 0 <= index < len(self._tokens):
            raise InvalidInputError(f"index {index} outside published range of {self.name}")
        return self._tokens[index]

    def read_range(self, start: int, stop: int) -> list:
        if not 0 <= start <= stop <= len(self._tokens):
            raise InvalidInputError(f"range [{start}, {stop}) outside published range of {self.name}")
        return self._tokens[start:stop]

    def snapshot(self) -> list:
        return list(self._tokens)


class SharedDecodeState:
    """Frontiers, buffers, rollback slot and completion flag (coordination.py:114-275)."""

    def __init__(self, prompt_length: int, max_new_tokens: int, max_draft_lead: int | None = None) -> None:
        if prompt_length < 1:
            raise InvalidInputError(f"prompt_length must be >= 1, got {prompt_length}")
        if max_new_tokens < 1:
            raise InvalidInputError(f"max_new_tokens must be >= 1, got {max_new_tokens}")
        if max_draft_lead is not None and max_draft_lead < 1:
            raise InvalidInputError(f"max_draft_lead must be >= 1 when set, got {max_draft_lead}")
        self.prompt_length = prompt_length
        self.max_new_tokens = max_new_tokens
        self.max_draft_lead = max_draft_lead
        self.D = TokenBuffer("D", allow_truncate=True)
        self.V = TokenBuffer("V")
        self._p_d = self._p_v = prompt_length
        self._rollback: RollbackRequest | None = None
        self._complete = False
        self.rollback_acks = 0

    p_d = property(lambda self: self._p_d)
    p_v = property(lambda self: self._p_v)
    verified_count = property(lambda self: self._p_v - self.prompt_length)
    draft_lead = property(lambda self: self._p_d - self._p_v)
    pending_rollback = property(lambda self: self._rollback)

    @property
    def lead_capped(self) -> bool:
        return self.max_draft_lead is not None and self.draft_lead >= self.max_draft_lead

    def rollback_pending(self) -> bool:
        return self._rollback is not None

    def is_complete(self) -> bool:
        return self._complete

    def verified_tokens(self) -> list:
        return self.V.snapshot()

    # draft side
    def publish_draft_token(self, token: int) -> None:
        self.D.append(token)
        self._p_d += 1

    # verify side
    def read_draft_window(self) -> list:
        if self._rollback is not None:
            raise ProtocolViolationError("read_draft_window during pending rollback")
        return self.D.read_range(self._p_v - self.prompt_length, self._p_d - self.prompt_length)

    def publish_verified(self, tokens: list) -> None:
        if self._rollback is not None:
            raise ProtocolViolationError("publish_verified during pending rollback")
        if len(tokens) == 0:
            raise InvalidInputError("publish_verified requires at least one token")
        self.V.extend(tokens)
        self._p_v += len(tokens)

    def request_rollback(self, request: RollbackRequest) -> None:
        if self._rollback is not None:
            raise ProtocolViolationError("rollback requested while one is already pending")
        if request.target != self._p_v:
            raise ProtocolViolationError(f"rollback target {request.target} does not match p_v {self._p_v}")
        if len(self.V) == 0 or self.V.token_at(len(self.V) - 1) != request.correction_token:
            raise ProtocolViolationError("correction token must be published to V before requesting rollback")
        self._rollback = request

    def signal_completion(self) -> None:
        if self._complete:
            raise ProtocolViolationError("completion signaled twice")
        self._complete = True

    def mirror_device(self, D: list, p_d: int) -> None:
        """Adopt the draft frontier reported by the device mailbox after a run."""
        self.D = TokenBuffer("D", allow_truncate=True)
        self.D.extend(D)
        self._p_d = p_d
