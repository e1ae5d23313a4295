"""``rs-tensor-container v1`` files (reference
``container.py:23-208``): byte-compatible reader and writer for the reference
tensor and for RS tensors, so results move between this package and the
reference in either direction.

Format: the magic line, then sections ``tag (8 ASCII bytes, space padded) |
payload length (u64 LE) | payload``.  Arrays are C-order little-endian f8 (i8
for particle indices); one ``META`` section is JSON with sorted keys.  The
section order below is the reference's, so identical tensors give identical
bytes (the writer is deterministic).  Device arrays are copied to the host.
"""

from __future__ import annotations

import json
import struct

import numpy as np

from .errors import ParseError
from .formats import CCT, CanonicalTensor, RSCanonical, RSTucker, TuckerTensor, to_host
from .particles import Box3, Grid3
from .quadrature import QuadratureRule, RadialKernel, ReferenceCanonical

MAGIC = b"rs-tensor-container v1\n"
_HEAD = struct.Struct("<8sQ")


# ---------------------------------------------------------------- sections
def encode_sections(sections) -> bytes:
    """``[(tag, payload), ...]`` -> container bytes."""
    parts = [MAGIC]
    for tag, payload in sections:
        raw = tag.encode("ascii")
        if len(raw) > 8:
            raise ParseError(f"section tag longer than 8 bytes: {tag!r}")
        parts.append(_HEAD.pack(raw.ljust(8), len(payload)))
        parts.append(payload)
    return b"".join(parts)


def decode_sections(blob: bytes, where: str = "<bytes>") -> dict:
    """Container bytes -> ``{tag: payload}`` in file order."""
    if not blob.startswith(MAGIC):
        raise ParseError(f"{where}: not an rs-tensor container (bad magic)")
    out, pos = {}, len(MAGIC)
    while pos < len(blob):
        if pos + _HEAD.size > len(blob):
            raise ParseError(f"{where}: truncated section header at byte {pos}")
        tag, size = _HEAD.unpack_from(blob, pos)
        pos += _HEAD.size
        if pos + size > len(blob):
            raise ParseError(f"{where}: truncated section {tag!r}")
        out[tag.decode("ascii").rstrip(" ")] = blob[pos:pos + size]
        pos += size
    return out


def _f8(a) -> bytes:
    return np.ascontiguousarray(to_host(a), dtype="<f8").tobytes()


def _i8(a) -> bytes:
    return np.ascontiguousarray(to_host(a), dtype="<i8").tobytes()


def _meta(d: dict) -> bytes:
    return json.dumps(d, sort_keys=True).encode("ascii")


def _arr(sec: dict, tag: str, dtype: str, shape=None) -> np.ndarray:
    if tag not in sec:
        raise ParseError(f"container lacks section {tag!r}")
    a = np.frombuffer(sec[tag], dtype=dtype).astype(np.float64 if dtype == "<f8" else np.int64)
    return a.reshape(shape) if shape is not None else a


def _read(path) -> dict:
    with open(path, "rb") as fh:
        blob = fh.read()
    sec = decode_sections(blob, str(path))
    if "META" not in sec:
        raise ParseError(f"{path}: no META section")
    return sec


def _write(path, sections) -> None:
    with open(path, "wb") as fh:
        fh.write(encode_sections(sections))


# ------------------------------------------------------- reference tensor
def reference_sections(ref: ReferenceCanonical) -> list:
    rule = ref.rule
    meta = {"type": "reference", "grid_n": ref.grid.n, "grid_b": ref.grid.box.half_width,
            "doubled": ref.doubled, "entry_rule": ref.entry_rule,
            "split_index": ref.split_index, "kernel": rule.kernel.kind, "lam": rule.kernel.lam,
            "M": rule.M, "C0": rule.C0, "h_M": rule.h_M, "r_range": list(rule.r_range),
            "symmetric_folded": rule.symmetric_folded, "rank": ref.R}
    return [("META", _meta(meta)), ("QNOD", _f8(rule.nodes)), ("QWTS", _f8(rule.weights)),
            ("TWTS", _f8(ref.tensor.weights)), ("SIDE", _f8(ref.tensor.factors[0]))]


def write_reference(ref: ReferenceCanonical, path) -> None:
    _write(path, reference_sections(ref))


def read_reference(path) -> ReferenceCanonical:
    sec = _read(path)
    m = json.loads(sec["META"].decode("ascii"))
    if m.get("type") != "reference":
        raise ParseError(f"{path}: container holds {m.get('type')!r}, not a reference")
    rule = QuadratureRule(kernel=RadialKernel(m["kernel"], m["lam"]), M=m["M"], C0=m["C0"],
                          h_M=m["h_M"], nodes=_arr(sec, "QNOD", "<f8"),
                          weights=_arr(sec, "QWTS", "<f8"), r_range=tuple(m["r_range"]),
                          symmetric_folded=m["symmetric_folded"])
    n = m["grid_n"]
    side = np.ascontiguousarray(_arr(sec, "SIDE", "<f8", (n, m["rank"])))
    return ReferenceCanonical(tensor=CanonicalTensor(_arr(sec, "TWTS", "<f8"), (side,) * 3),
                              rule=rule, grid=Grid3(n, Box3(m["grid_b"])), doubled=m["doubled"],
                              entry_rule=m["entry_rule"], split_index=m["split_index"])


# ------------------------------------------------------------- RS tensors
def rs_sections(rs) -> list:
    if isinstance(rs, RSCanonical):
        fmt = "canonical"
    elif isinstance(rs, RSTucker):
        fmt = "tucker"
    else:
        raise ParseError(f"cannot serialize {type(rs).__name__}")
    sh = rs.short
    meta = {"type": "rs", "long_format": fmt, "grid_n": rs.grid.n,
            "grid_b": rs.grid.box.half_width, "gamma": int(sh.gamma),
            "overlap_policy": sh.overlap_policy, "max_overlap": sh.max_overlap,
            "local_rank": sh.local.rank, "local_size": sh.local.mode_sizes[0],
            "count": int(sh.centers.shape[0])}
    if fmt == "canonical":
        meta["long_rank"] = rs.long.rank
        long_secs = [("LWTS", _f8(rs.long.weights))] + \
            [(f"LV{l}", _f8(rs.long.factors[l])) for l in range(3)]
    else:
        meta["tucker_ranks"] = list(rs.long.ranks)
        long_secs = [("CORE", _f8(rs.long.core))] + \
            [(f"TF{l}", _f8(rs.long.factors[l])) for l in range(3)]
    return ([("META", _meta(meta))] + long_secs + [("U0WT", _f8(sh.local.weights))] +
            [(f"U0V{l}", _f8(sh.local.factors[l])) for l in range(3)] +
            [("CTRS", _i8(sh.centers)), ("CWTS", _f8(sh.weights))])


def write_rs(rs, path) -> None:
    _write(path, rs_sections(rs))


def read_rs(path):
    """RS tensor from a container (the Tucker long part lives on the device)."""
    sec = _read(path)
    m = json.loads(sec["META"].decode("ascii"))
    if m.get("type") != "rs":
        raise ParseError(f"{path}: container holds {m.get('type')!r}, not an RS tensor")
    n, size, r0 = m["grid_n"], m["local_size"], m["local_rank"]
    grid = Grid3(n, Box3(m["grid_b"]))
    local = CanonicalTensor(_arr(sec, "U0WT", "<f8"),
                            tuple(_arr(sec, f"U0V{l}", "<f8", (size, r0)) for l in range(3)))
    short = CCT(local=local, gamma=m["gamma"], centers=_arr(sec, "CTRS", "<i8", (m["count"], 3)),
                weights=_arr(sec, "CWTS", "<f8"), mode_sizes=(n, n, n),
                overlap_policy=m["overlap_policy"], max_overlap=m["max_overlap"])
    if m["long_format"] == "canonical":
        r = m["long_rank"]
        long = CanonicalTensor(_arr(sec, "LWTS", "<f8"),
                               tuple(_arr(sec, f"LV{l}", "<f8", (n, r)) for l in range(3)))
        return RSCanonical(long=long, short=short, grid=grid)
    r1, r2, r3 = m["tucker_ranks"]
    long = TuckerTensor(_arr(sec, "CORE", "<f8", (r1, r2, r3)),
                        tuple(_arr(sec, f"TF{l}", "<f8", (n, r)) for l, r in enumerate((r1, r2, r3))))
    return RSTucker(long=long, short=short, grid=grid)
