"""Host ingestion: the reference CLI's "id weight" text (cli.py:60-70) into
numpy arrays / CSR batches for the GPU engine.

`parse_weighted_text` runs the native parser (pmh_parse_weighted_text in
libpmh.so, no device work) and, for any input outside its well-formed
grammar, the exact line-by-line restatement `read_weighted_lines`, so the
result -- or the exception -- is the reference's.  `read_sets_csr` packs one
set per text/file into a CSRBatch, validated like WeightedSet
(sketch.py:82-90) unless validate=False.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib
from .datagen import CSRBatch
from .errors import EmptyInputError, InvalidParamsError


def read_weighted_lines(stream):
    """cli._read_weighted_lines (cli.py:60-70): list of (id, weight)."""
    entries = []
    for line in stream:
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        parts = line.split()
        eid = int(parts[0], 0)
        weight = float(parts[1]) if len(parts) > 1 else 1.0
        entries.append((eid, weight))
    return entries


def _python_path(data: bytes):
    entries = read_weighted_lines(data.decode().splitlines())
    ids = np.array([e for e, _ in entries], np.uint64)   # negative ids raise like WeightedSet
    w = np.array([x for _, x in entries], np.float64)
    return ids, w


def parse_weighted_text(data) -> tuple:
    """Text (bytes or str) -> (ids uint64[n], weights float64[n])."""
    if isinstance(data, str):
        data = data.encode()
    data = bytes(data)
    # universal newlines: a bare CR is a line break for the reference
    if b"\r" in data and b"\r" in data.replace(b"\r\n", b""):
        return _python_path(data)
    cap = data.count(b"\n") + 1
    ids = np.empty(cap, np.uint64)
    w = np.empty(cap, np.float64)
    n = _lib.load().pmh_parse_weighted_text(data, len(data), ids.ctypes.data, w.ctypes.data, cap)
    if n < 0:
        return _python_path(data)
    return ids[:n].copy(), w[:n].copy()


def read_weighted_file(path) -> tuple:
    """A file of "id weight" lines ('-' is not special here) -> (ids, weights)."""
    with open(path, "rb") as f:
        return parse_weighted_text(f.read())


def _validate(ids, w, s):
    if ids.size == 0:
        raise EmptyInputError(f"set {s} has no entries")
    if not np.all(np.isfinite(w)) or not np.all(w > 0):
        raise InvalidParamsError(f"set {s}: weights must be finite and > 0")
    if np.unique(ids).size != ids.size:
        raise InvalidParamsError(f"set {s}: duplicate ids")


def read_sets_csr(sources, validate: bool = True, name: str = "text") -> CSRBatch:
    """One set per source (a path, or bytes/str text) -> CSRBatch."""
    parts = []
    for s, src in enumerate(sources):
        if isinstance(src, (bytes, bytearray)) or (isinstance(src, str) and not os.path.exists(src)
                                                   and ("\n" in src or " " in src)):
            ids, w = parse_weighted_text(src)
        else:
            ids, w = read_weighted_file(src)
        if validate:
            _validate(ids, w, s)
        parts.append((ids, w))
    sizes = np.array([p[0].size for p in parts], np.int64)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ids = np.concatenate([p[0] for p in parts]) if parts else np.zeros(0, np.uint64)
    w = np.concatenate([p[1] for p in parts]) if parts else np.zeros(0, np.float64)
    return CSRBatch(ids, w, off, name)


def format_signature(components) -> str:
    """The CLI's output: one component per line (cli.py:99-103)."""
    return "\n".join(str(int(c)) for c in components) + "\n"

