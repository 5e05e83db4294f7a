"""`mct` JSON blobs for MC tensors (serialize.hpp:40-76), the reference's
on-disk format: component bit patterns as fixed-width lowercase hex strings
(4 / 8 / 16 digits for binary16 / 32 / 64), component index fastest, elements
row-major, so a round trip is bit-exact.  Works on device or host tensors
(a device tensor is copied to the host once); files written with the
reference's `write_json_file` layout (2-space indent, trailing newline)."""
from __future__ import annotations

import json

import numpy as np
import torch

_TAG = {torch.float16: ("b16", np.uint16, 4), torch.float32: ("b32", np.uint32, 8),
        torch.float64: ("b64", np.uint64, 16)}
_BY_NAME = {v[0]: (k, v[1], v[2]) for k, v in _TAG.items()}


def mct_to_json(x: torch.Tensor) -> dict:
    """x: (*shape, nc) tensor of binary16/32/64 components."""
    if x.dtype not in _TAG:
        raise ValueError(f"mct_to_json: unsupported component dtype {x.dtype}")
    name, ut, width = _TAG[x.dtype]
    bits = x.detach().contiguous().cpu().numpy().view(ut).ravel()
    return {"format": "mct", "version": 1, "precision": name, "shape": list(x.shape[:-1]),
            "nc": int(x.shape[-1]), "data": [format(int(b), f"0{width}x") for b in bits]}


def mct_from_json(j: dict, precision: str, device="cpu") -> torch.Tensor:
    """The reference's checks and messages (serialize.hpp:58-76)."""
    if not isinstance(j, dict) or j.get("format", "") != "mct":
        raise ValueError("mct_from_json: not an mct blob")
    if j.get("precision", "") != precision:
        raise ValueError(f"mct_from_json: precision tag '{j.get('precision', '')}' does not match requested "
                         f"{precision}")
    dtype, ut, _ = _BY_NAME[precision]
    shape = [int(d) for d in j["shape"]]
    nc = int(j["nc"])
    data = j["data"]
    if len(data) != int(np.prod(shape, dtype=np.int64)) * nc:
        raise ValueError("mct_from_json: data length mismatch")
    bits = np.array([int(h, 16) for h in data], dtype=ut)
    return torch.from_numpy(bits.view(_np_float(dtype)).reshape(*shape, nc)).to(device)


def _np_float(dtype):
    return {torch.float16: np.float16, torch.float32: np.float32, torch.float64: np.float64}[dtype]


def dumps(j: dict, indent: int = 2) -> str:
    """The text of the reference's Json::dump(2) as the nlohmann build it links
    emits it (checked byte for byte in tests/test_oracle_pin.py): object keys
    sorted, 2-space indent, ": " after keys, arrays of numbers inline as
    "[2,3]", other arrays one element per line."""
    def num(v):
        return isinstance(v, (int, float)) and not isinstance(v, bool)

    def go(v, lvl):
        pad, inner = " " * (indent * lvl), " " * (indent * (lvl + 1))
        if isinstance(v, dict):
            if not v:
                return "{}"
            items = [f"{inner}{json.dumps(k)}: {go(v[k], lvl + 1)}" for k in sorted(v)]
            return "{\n" + ",\n".join(items) + "\n" + pad + "}"
        if isinstance(v, (list, tuple)):
            if not v:
                return "[]"
            if all(num(e) for e in v):
                return "[" + ",".join(json.dumps(e) for e in v) + "]"
            return "[\n" + ",\n".join(inner + go(e, lvl + 1) for e in v) + "\n" + pad + "]"
        return json.dumps(v)

    return go(j, 0)


def write_json_file(path: str, j: dict) -> None:
    with open(path, "w") as f:
        f.write(dumps(j) + "\n")


def read_json_file(path: str) -> dict:
    with open(path) as f:
        return json.load(f)
