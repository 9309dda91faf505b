"""Synthetic output-token fill on the GPU (emu_token_fill).

Restates the token part of ``EmulatorEngine._apply_outcome``
(/root/reference/pkg/src/serve_emu/engine.py:464-483) for a batch of scheduled
entries: a prefill entry emits a token only when its chunk completes the
prompt, a decode entry always emits, and the emitted id is the request's
token index (``generated`` before the step; SPEC.md: token k of request r has
id k, pinned by the server test's [0, 1, 2]).
"""
from __future__ import annotations

from . import _lib


def token_fill(is_prefill, chunk, prefill_progress, prompt_len, generated, target_len, *, out_ids=None,
               out_finished=None):
    """CUDA tensors in, (ids int32 [-1 = no token], finished uint8) CUDA tensors out."""
    torch = _lib.require_cuda()
    cols = [is_prefill.to(torch.uint8), chunk.to(torch.int32), prefill_progress.to(torch.int32),
            prompt_len.to(torch.int32), generated.to(torch.int32), target_len.to(torch.int32)]
    cols = [c.contiguous() for c in cols]
    n = cols[0].numel()
    if any(c.numel() != n or not c.is_cuda for c in cols):
        raise ValueError("token_fill needs equal-length CUDA tensors")
    ids = out_ids if out_ids is not None else torch.empty(n, dtype=torch.int32, device=cols[0].device)
    fin = out_finished if out_finished is not None else torch.empty(n, dtype=torch.uint8, device=cols[0].device)
    _lib.check(_lib.lib().emu_token_fill(*[_lib.ptr(c) for c in cols], n, _lib.ptr(ids), _lib.ptr(fin),
                                         _lib.stream_ptr()))
    return ids, fin
