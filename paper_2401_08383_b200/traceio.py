"""EXFLOW-TRACE v1 text I/O for routing traces (host side).

Mirrors the reference's trace format and its error behaviour
(proj/include/exflow/trace.hpp:39-56, parser proj/src/trace.cpp:72-150,
writer :152-168, RoutingTrace::validate :48-70): a GPU run's routes
(`MoeModel.routes()`, [tokens][layers] int32) can be saved in the format the
reference CLI reads, and a reference trace can drive the model's forced
routing or the replay kernels.

Format: optional blank / '#' comment lines anywhere; first content line
`EXFLOW-TRACE v1`; then `E <experts> L <layers>` (E >= 1, L >= 2); then one
line per token with L whitespace-separated expert ids in [0, E).
"""
from __future__ import annotations

import os
import re
from typing import Tuple

import numpy as np

MAGIC = "EXFLOW-TRACE v1"
_INT = re.compile(r"-?[0-9]+")  # std::from_chars(long): optional '-', decimal digits only
_LONG_MIN, _LONG_MAX = -(1 << 63), (1 << 63) - 1


class ParseError(RuntimeError):
    """Malformed EXFLOW-TRACE input (proj/include/exflow/trace.hpp:39-43: a
    std::runtime_error whose message carries the offending line number)."""


def _parse_int(tok: str, line_no: int) -> int:
    if not _INT.fullmatch(tok):
        raise ParseError(f"invalid token '{tok}' at line {line_no}")
    v = int(tok)
    if v < _LONG_MIN or v > _LONG_MAX:  # from_chars: result_out_of_range
        raise ParseError(f"invalid token '{tok}' at line {line_no}")
    return v


def parse_trace(text: str) -> Tuple[np.ndarray, int]:
    """Text -> (paths [T][L] int32, num_experts). Raises ParseError with the
    reference's messages (proj/src/trace.cpp:72-140)."""
    magic = dims = False
    E = L = 0
    rows = []
    for line_no, line in enumerate(text.split("\n"), start=1):
        if line.endswith("\r"):
            line = line[:-1]
        if line.strip() == "" or line[0] == "#":
            continue
        if not magic:
            if line != MAGIC:
                raise ParseError(f"missing or unsupported EXFLOW-TRACE header at line {line_no}")
            magic = True
            continue
        fields = line.split()
        if not dims:
            if len(fields) != 4 or fields[0] != "E" or fields[2] != "L":
                raise ParseError(f"expected 'E <experts> L <layers>' at line {line_no}")
            E = _parse_int(fields[1], line_no)
            L = _parse_int(fields[3], line_no)
            if E < 1:
                raise ParseError(f"E must be >= 1, got {E} at line {line_no}")
            if L < 2:
                raise ParseError(f"L must be >= 2, got {L} at line {line_no}")
            dims = True
            continue
        if len(fields) != L:
            raise ParseError(f"path length {len(fields)} != L={L} at line {line_no}")
        row = []
        for f in fields:
            v = _parse_int(f, line_no)
            if v < 0 or v >= E:
                raise ParseError(f"expert id {v} out of range [0,{E}) at line {line_no}")
            row.append(v)
        rows.append(row)
    if not magic:
        raise ParseError("missing or unsupported EXFLOW-TRACE header at line 1")
    if not dims:
        raise ParseError("missing 'E <experts> L <layers>' line")
    if not rows:
        raise ParseError("trace contains no token paths")
    return np.asarray(rows, np.int32).reshape(len(rows), L), E


def validate_trace(paths: np.ndarray, num_experts: int) -> None:
    """RoutingTrace::validate (proj/src/trace.cpp:48-70): ValueError (the
    reference's std::invalid_argument) with the same messages."""
    paths = np.asarray(paths)
    if num_experts < 1:
        raise ValueError(f"num_experts must be >= 1, got {num_experts}")
    if paths.ndim != 2 or paths.shape[1] < 2:
        raise ValueError(f"num_layers must be >= 2, got {paths.shape[1] if paths.ndim == 2 else 0}")
    if paths.shape[0] < 1:
        raise ValueError("trace contains no token paths")
    if (paths < 0).any() or (paths >= num_experts).any():
        raise ValueError(f"expert id out of range [0,{num_experts})")


def serialize_trace(paths: np.ndarray, num_experts: int) -> str:
    """write_trace (proj/src/trace.cpp:152-165): header, dims, one line per token."""
    validate_trace(paths, num_experts)
    paths = np.asarray(paths)
    out = [MAGIC, f"E {num_experts} L {paths.shape[1]}"]
    out += [" ".join(str(int(v)) for v in row) for row in paths]
    return "\n".join(out) + "\n"


def save_trace(path: str | os.PathLike, paths: np.ndarray, num_experts: int) -> None:
    text = serialize_trace(paths, num_experts)
    try:
        with open(path, "wb") as f:
            f.write(text.encode())
    except OSError as e:
        raise RuntimeError(f"cannot write trace file: {os.fspath(path)}") from e


def load_trace(path: str | os.PathLike) -> Tuple[np.ndarray, int]:
    try:
        with open(path, "rb") as f:
            text = f.read().decode()
    except OSError as e:
        raise RuntimeError(f"cannot open trace file: {os.fspath(path)}") from e
    return parse_trace(text)
