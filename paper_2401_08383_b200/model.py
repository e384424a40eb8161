"""Context-coherent expert-parallel MoE decode layer (one handle per rank).

Python mirror of the exf_model_* C-ABI (include/exflow_c.h). Device memory
and multi-process plumbing come from torch (tensors for inputs/outputs,
torch.distributed to exchange the 64-byte CUDA-IPC handles); every kernel is
the hand-written sm_100a code in libexflow_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _capi

PHASE_BEGIN, PHASE_DISPATCH, PHASE_FFN, PHASE_GATHER_SEND, PHASE_GATHER_WAIT, PHASE_FUSED, \
    PHASE_COMBINE_SEND, PHASE_COMBINE_WAIT, PHASE_ATTN = range(9)
EP_COHERENT, EP_VANILLA = 0, 1  # include/exflow_c.h EXF_EP_*
DTYPE_BF16, DTYPE_F32 = 0, 1    # include/exflow_c.h EXF_DTYPE_*


@dataclass
class MoeModelConfig:
    """Value struct in the style of SynthConfig (proj/include/exflow/synth.hpp:13-23)."""
    num_experts: int = 8
    num_layers: int = 4
    d_model: int = 512
    d_ffn: int = 2048
    top_k: int = 1
    tokens_per_gpu: int = 256
    world_size: int = 1
    rank: int = 0
    seed: int = 0
    init_std: float = 0.02
    gate_affinity: float = 0.0
    # EP_COHERENT (ExFlow) or EP_VANILLA (dispatch + combine back home every
    # layer, proj/src/sim.cpp:60-64)
    ep_mode: int = 0
    # DTYPE_BF16 (tcgen05 path) or DTYPE_F32 (fp32 mode: fp32 weights, states,
    # gate and SIMT FFN; the north star's 1e-5 bar)
    dtype: int = 0
    # coherent attention block before every MoE layer (bf16): heads (0 = off),
    # replicated context capacity per sequence, prompt length written by
    # context_setup() (the setup AllGather)
    attn_heads: int = 0
    context_len: int = 0
    context_prefix: int = 0

    @property
    def capacity(self) -> int:
        return self.tokens_per_gpu * self.world_size

    @property
    def np_dtype(self):
        """Host element type of rows/weights: uint16 bf16 bits or float32."""
        return np.float32 if self.dtype == DTYPE_F32 else np.uint16

    def home_tokens(self, rank: Optional[int] = None) -> np.ndarray:
        r = self.rank if rank is None else rank
        return r + self.world_size * np.arange(self.tokens_per_gpu)

    def _c(self) -> _capi.ModelConfigC:
        return _capi.ModelConfigC(self.num_experts, self.num_layers, self.d_model, self.d_ffn,
                                  self.top_k, self.tokens_per_gpu, self.world_size, self.rank,
                                  self.seed, self.init_std, self.gate_affinity, self.ep_mode,
                                  self.dtype, self.attn_heads, self.context_len, self.context_prefix)


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        return None
    return int(getattr(stream, "cuda_stream", stream))


class MoeModel:
    """One rank of the ExFlow decode layer stack."""

    def __init__(self, config: MoeModelConfig, assign: np.ndarray):
        self.config = config
        self.assign = np.ascontiguousarray(assign, dtype=np.int32)
        if self.assign.shape != (config.num_layers, config.num_experts):
            raise _capi.ExflowInvalidArgument("placement must be [L][E]")
        self._h = C.c_void_p()
        cfg = config._c()
        _capi.call("exf_model_create", C.byref(cfg), self.assign.ctypes.data, C.byref(self._h))

    # ------------------------------------------------------------ wiring
    @property
    def handle(self) -> int:
        return self._h.value

    def ipc_handle(self) -> bytes:
        buf = (C.c_uint8 * 64)()
        _capi.call("exf_model_ipc_handle", self._h, buf)
        return bytes(buf)

    def connect(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(handles)
        if len(blob) != 64 * self.config.world_size:
            raise _capi.ExflowInvalidArgument("need one 64-byte IPC handle per rank")
        arr = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _capi.call("exf_model_connect", self._h, arr)

    @staticmethod
    def connect_local(models: Sequence["MoeModel"]) -> None:
        arr = (C.c_void_p * len(models))(*[m.handle for m in models])
        _capi.call("exf_model_connect_local", arr, len(models))

    # ------------------------------------------------------------ execution
    def step(self, x_in, stream=None) -> None:
        """x_in: torch cuda bf16 tensor [B][d] of this rank's home tokens."""
        _capi.call("exf_model_step", self._h, x_in.data_ptr(), _stream_ptr(stream))

    def phase(self, phase: int, layer: int = 0, x_in=None, stream=None) -> None:
        _capi.call("exf_model_step_phase", self._h, phase, layer,
                   None if x_in is None else x_in.data_ptr(), _stream_ptr(stream))

    def capture(self, x_in, stream) -> None:
        _capi.call("exf_model_capture", self._h, x_in.data_ptr(), _stream_ptr(stream))

    def replay(self, stream) -> None:
        _capi.call("exf_model_replay", self._h, _stream_ptr(stream))

    def output_ptr(self) -> int:
        p = C.c_void_p()
        _capi.call("exf_model_output", self._h, C.byref(p))
        return p.value

    def output(self):
        """torch [G*B][d] view (bf16, or fp32 in fp32 mode) of the context-AllGather
        output (token-id order)."""
        import torch
        cfg = self.config
        n = cfg.capacity * cfg.d_model
        f32 = cfg.dtype == DTYPE_F32
        holder = _CudaArray(self.output_ptr(), (cfg.capacity, cfg.d_model), "<f4" if f32 else "<i2")
        t = torch.as_tensor(holder, device="cuda")
        assert t.numel() == n
        return t if f32 else t.view(torch.bfloat16)

    def check(self) -> None:
        _capi.call("exf_model_check", self._h)

    def set_forced_routes(self, routes: Optional[np.ndarray]) -> None:
        if routes is None:
            _capi.call("exf_model_set_forced_routes", self._h, None)
            return
        r = np.ascontiguousarray(routes, dtype=np.int32)
        if r.shape != (self.config.capacity, self.config.num_layers):
            raise _capi.ExflowInvalidArgument("forced routes must be [G*B][L]")
        _capi.call("exf_model_set_forced_routes", self._h, r.ctypes.data)

    # ------------------------------------------------------------ statistics
    def routes(self) -> np.ndarray:
        out = np.empty((self.config.capacity, self.config.num_layers), np.int32)
        _capi.call("exf_model_read_routes", self._h, out.ctypes.data)
        return out

    def save_trace(self, path) -> None:
        """Emit the routes of the last step as an EXFLOW-TRACE v1 file (the
        format the reference CLI reads, proj/src/trace.cpp:152-168). Rows are
        token ids; with G > 1 merge every rank's routes first (dist.merge_routes)
        and use traceio.save_trace directly."""
        from . import traceio
        traceio.save_trace(path, self.routes(), self.config.num_experts)

    def crossed(self) -> np.ndarray:
        out = np.empty(self.config.num_layers, np.int64)
        _capi.call("exf_model_read_crossed", self._h, out.ctypes.data)
        return out

    def affinity_counts(self) -> np.ndarray:
        E = self.config.num_experts
        out = np.empty((self.config.num_layers - 1, E, E), np.int64)
        _capi.call("exf_affinity_snapshot", self._h, out.ctypes.data)
        return out

    def reset_stats(self) -> None:
        _capi.call("exf_model_reset_stats", self._h)

    def resident(self, which: int):
        cfg = self.config
        x = np.empty((cfg.capacity, cfg.d_model), cfg.np_dtype)
        meta = np.empty((cfg.capacity, 2), np.int32)
        n = C.c_int32()
        _capi.call("exf_model_read_resident", self._h, which, x.ctypes.data, meta.ctypes.data,
                   C.byref(n))
        return x[:n.value], meta[:n.value]

    def expert_weights(self, layer: int, expert: int):
        cfg = self.config
        dt = cfg.np_dtype
        w1 = np.empty((cfg.d_ffn, cfg.d_model), dt)
        b1 = np.empty(cfg.d_ffn, dt)
        w2 = np.empty((cfg.d_model, cfg.d_ffn), dt)
        b2 = np.empty(cfg.d_model, dt)
        _capi.call("exf_model_read_expert", self._h, layer, expert, w1.ctypes.data,
                   b1.ctypes.data, w2.ctypes.data, b2.ctypes.data)
        return w1, b1, w2, b2

    def expert_storage(self, layer: int, slot: int):
        """torch int16 (bf16 bits; float32 in fp32 mode) views of local weight slot `slot` of `layer`:
        (W1 [d_ffn][d], b1 [d_ffn], W2 [d][d_ffn], b2 [d]) -- device memory of
        this model, for expert migration (migrate.py)."""
        import torch
        cfg = self.config
        ptrs = [C.c_void_p() for _ in range(4)]
        _capi.call("exf_model_expert_storage", self._h, layer, slot, *[C.byref(p) for p in ptrs])
        shapes = [(cfg.d_ffn, cfg.d_model), (cfg.d_ffn,), (cfg.d_model, cfg.d_ffn), (cfg.d_model,)]
        ts = "<f4" if cfg.dtype == DTYPE_F32 else "<i2"
        return tuple(torch.as_tensor(_CudaArray(p.value, sh, ts), device="cuda") for p, sh in zip(ptrs, shapes))

    def set_placement(self, assign: np.ndarray) -> None:
        """Install a new [L][E] placement (same table on every rank, weights
        already in their new slots: see migrate.py)."""
        a = np.ascontiguousarray(assign, dtype=np.int32)
        if a.shape != (self.config.num_layers, self.config.num_experts):
            raise _capi.ExflowInvalidArgument("placement must be [L][E]")
        _capi.call("exf_model_set_placement", self._h, a.ctypes.data)
        self.assign = a

    # ------------------------------------------------------------ attention block
    def context_setup(self, stream=None, phase: int = 0) -> None:
        """Setup AllGather of the replicated context (every rank must call it);
        phase 1/2 = publish/wait halves for lock-step ranks in one stream."""
        _capi.call("exf_model_context_setup_phase", self._h, phase, _stream_ptr(stream))

    def kv_rows(self, layer: int, seq: int, pos0: int, count: int):
        """(K, V) rows of this rank's replica: [count][H][Dh] bf16 bits each."""
        cfg = self.config
        H, Dh = cfg.attn_heads, cfg.d_model // max(cfg.attn_heads, 1)
        k = np.empty((count, H, Dh), np.uint16)
        v = np.empty((count, H, Dh), np.uint16)
        _capi.call("exf_model_read_kv", self._h, layer, seq, pos0, count, k.ctypes.data, v.ctypes.data)
        return k, v

    def kv_len(self, layer: int) -> np.ndarray:
        out = np.empty(self.config.capacity, np.int32)
        _capi.call("exf_model_read_kv_len", self._h, layer, out.ctypes.data)
        return out

    def attn_weights(self, layer: int):
        """(Wqkv [3d][d], bqkv [3d], Wo [d][d], bo [d]) bf16 bits."""
        d = self.config.d_model
        wqkv = np.empty((3 * d, d), np.uint16)
        bqkv = np.empty(3 * d, np.uint16)
        wo = np.empty((d, d), np.uint16)
        bo = np.empty(d, np.uint16)
        _capi.call("exf_model_read_attn", self._h, layer, wqkv.ctypes.data, bqkv.ctypes.data,
                   wo.ctypes.data, bo.ctypes.data)
        return wqkv, bqkv, wo, bo

    def gate_weights(self, layer: int) -> np.ndarray:
        cfg = self.config
        wg = np.empty((cfg.num_experts, cfg.d_model), cfg.np_dtype)
        _capi.call("exf_model_read_gate", self._h, layer, wg.ctypes.data)
        return wg

    def launches_per_step(self) -> int:
        return int(_capi.load().exf_model_launches_per_step(self._h))

    def describe(self) -> dict:
        import json
        buf = C.create_string_buffer(512)
        _capi.call("exf_model_describe", self._h, buf, 512)
        return json.loads(buf.value.decode())

    def close(self) -> None:
        if self._h:
            _capi.call("exf_model_destroy", self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _CudaArray:
    """__cuda_array_interface__ over a raw device pointer (int16 view of bf16)."""

    def __init__(self, ptr: int, shape, typestr: str = "<i2"):
        self.__cuda_array_interface__ = {"data": (ptr, False), "shape": tuple(shape),
                                         "typestr": typestr, "version": 3, "strides": None}
