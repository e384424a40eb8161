"""Coherent decode attention over the replicated context cache (host side of
exf_coherent_attention, include/exflow_c.h). SURVEY §8(f) rank 1.

No CPU fallback: the call goes through libexflow_b200.so or raises. torch is
plumbing only (device buffers, the current stream).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def coherent_attention(q: torch.Tensor, seq: torch.Tensor, ctx_len: torch.Tensor,
                       k: torch.Tensor, v: torch.Tensor, scale: float | None = None,
                       out: torch.Tensor | None = None,
                       workspace: torch.Tensor | None = None) -> torch.Tensor:
    """q [N][H][Dh] bf16, seq [N] int32, ctx_len [S] int32, k/v [S][H][C][Dh]
    bf16 (all on the same CUDA device) -> out [N][H][Dh] bf16."""
    N, H, Dh = q.shape
    S, Hk, Cap, Dk = k.shape
    if (Hk, Dk) != (H, Dh) or v.shape != k.shape:
        raise _capi.ExflowInvalidArgument("coherent_attention: q/k/v shape mismatch")
    for t in (q, k, v):
        if t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise _capi.ExflowInvalidArgument("coherent_attention: contiguous bf16 q/k/v required")
    if seq.dtype != torch.int32 or ctx_len.dtype != torch.int32:
        raise _capi.ExflowInvalidArgument("coherent_attention: int32 seq/ctx_len required")
    if scale is None:
        scale = Dh ** -0.5
    if out is None:
        out = torch.empty_like(q)
    lib = _capi.load()
    ws_bytes = lib.exf_coherent_attention_workspace_bytes(N, H, Dh, Cap)
    if ws_bytes and (workspace is None or workspace.numel() * workspace.element_size() < ws_bytes):
        # any contents: the call zeroes its arrival counters on the stream
        workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=q.device)
    stream = torch.cuda.current_stream(q.device).cuda_stream
    _capi.call("exf_coherent_attention", _ptr(q), _ptr(seq), _ptr(ctx_len), _ptr(k), _ptr(v),
               N, S, H, Dh, Cap, C.c_float(scale), _ptr(workspace) if ws_bytes else None,
               _ptr(out), C.c_void_p(stream))
    return out


def kv_append(k_new: torch.Tensor, v_new: torch.Tensor, seq: torch.Tensor,
              k_caches, v_caches, ctx_lens, overflow: torch.Tensor | None = None) -> None:
    """Append one token per sequence to every replica of the context cache.

    k_new/v_new [N][H][Dh] bf16, seq [N] int32 (distinct); k_caches/v_caches
    lists of [S][H][C][Dh] bf16 replicas (replica 0 local; the others may be
    CUDA-IPC peer tensors), ctx_lens the matching [S] int32 lengths.
    """
    N, H, Dh = k_new.shape
    S, Hk, Cap, Dk = k_caches[0].shape
    if (Hk, Dk) != (H, Dh) or v_new.shape != k_new.shape:
        raise _capi.ExflowInvalidArgument("kv_append: shape mismatch")
    for t in [k_new, v_new, *k_caches, *v_caches]:
        if t.dtype != torch.bfloat16 or not t.is_contiguous() or t.shape[-1] != Dh:
            raise _capi.ExflowInvalidArgument("kv_append: contiguous bf16 tensors required")
    R = len(k_caches)
    if len(v_caches) != R or len(ctx_lens) != R:
        raise _capi.ExflowInvalidArgument("kv_append: replica lists differ in length")
    ks = (C.c_void_p * R)(*[t.data_ptr() for t in k_caches])
    vs = (C.c_void_p * R)(*[t.data_ptr() for t in v_caches])
    cs = (C.c_void_p * R)(*[t.data_ptr() for t in ctx_lens])
    stream = torch.cuda.current_stream(k_new.device).cuda_stream
    _capi.call("exf_kv_append", _ptr(k_new), _ptr(v_new), _ptr(seq), N, S, H, Dh, Cap, R,
               ks, vs, cs, _ptr(overflow), C.c_void_p(stream))


def export_replica(t: torch.Tensor):
    """(64-byte CUDA-IPC handle, byte offset) of a device tensor's buffer."""
    h = (C.c_char * 64)()
    off = C.c_int64()
    _capi.call("exf_ipc_export", _ptr(t), h, C.byref(off))
    return bytes(h), off.value


class _Cai:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def import_replica(handle: bytes, offset: int, shape, dtype: torch.dtype) -> torch.Tensor:
    """Map a peer's buffer on the current device (NVLink peer access). The
    returned tensor aliases the peer's HBM; pass it to kv_append as a replica.
    Release with close_replica(t, offset)."""
    h = (C.c_char * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _capi.call("exf_ipc_import", h, offset, C.byref(p))
    if dtype == torch.bfloat16:
        return torch.as_tensor(_Cai(p.value, shape, "<i2"), device="cuda").view(torch.bfloat16)
    if dtype == torch.int32:
        return torch.as_tensor(_Cai(p.value, shape, "<i4"), device="cuda")
    raise _capi.ExflowInvalidArgument("import_replica: bf16 or int32 buffers only")


def close_replica(t: torch.Tensor, offset: int) -> None:
    _capi.call("exf_ipc_close", C.c_void_p(t.data_ptr()), offset)
