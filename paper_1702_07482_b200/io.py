"""Model and image files of the reference, so trained models and images move
between the reference and this package unchanged.

Restates the formats of the reference's io.py:
  * model file v1 (io.py:133-210): a "specklediff-model 1" header, one
    `key value` line per field, per stage a `beta` line plus `coeff` and
    `weight` rows, reals as C99 hex floats so the round trip is bit-exact,
    an `end` marker; unknown versions are rejected;
  * images (io.py:32-128): FGRID (plain-text doubles, `repr` round trip) and
    portable graymaps P2/P5 with 8- or 16-bit samples (writing clamps to
    [0, peak] and rounds).
Pure host code: nothing here is on the accelerated path.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .diffusion import DiffusionModel, StageParams
from .imageops import as_image
from .influence import RbfGrid

MODEL_MAGIC = "specklediff-model"
MODEL_FORMAT_VERSION = 1
IMAGE_SUFFIXES = (".pgm", ".fgrid")


# ------------------------------------------------------------------ models

def _hx(v) -> str:
    return float(v).hex()


def save_model(model: DiffusionModel, path) -> None:
    head = [
        ("filter_size", str(model.filter_size)),
        ("num_filters", str(model.num_filters)),
        ("stages", str(model.num_stages)),
        ("looks", str(model.looks)),
        ("value_range", _hx(model.value_range)),
        ("variant", model.variant),
        ("floor", _hx(model.floor)),
        ("rbf_count", str(model.rbf.count)),
        ("rbf_radius", _hx(model.rbf.radius)),
        ("rbf_bandwidth", _hx(model.rbf.gamma)),
        ("generator", model.generator),
        ("seed", str(model.seed)),
        ("metadata", json.dumps(model.metadata, sort_keys=True)),
    ]
    out = [f"{MODEL_MAGIC} {MODEL_FORMAT_VERSION}"]
    out += [f"{k} {v}" for k, v in head]
    for t, st in enumerate(model.stages):
        out.append(f"stage {t}")
        out.append(f"beta {_hx(st.beta)}")
        out += ["coeff " + " ".join(map(_hx, row)) for row in st.coeffs]
        out += ["weight " + " ".join(map(_hx, row)) for row in st.weights]
    out.append("end")
    Path(path).write_text("\n".join(out) + "\n")


class _Lines:
    def __init__(self, path):
        self.path = path
        self._it = (ln for ln in Path(path).read_text().splitlines() if ln.strip())

    def next(self):
        return next(self._it, None)

    def field(self, key: str) -> str:
        ln = self.next()
        if ln is None or not ln.startswith(key + " "):
            raise ValueError(f"{self.path}: expected '{key}' entry")
        return ln[len(key) + 1:]


def load_model(path) -> DiffusionModel:
    rd = _Lines(path)
    head = (rd.next() or "").split()
    if len(head) != 2 or head[0] != MODEL_MAGIC:
        raise ValueError(f"{path}: not a model file")
    if int(head[1]) != MODEL_FORMAT_VERSION:
        raise ValueError(f"{path}: unsupported model format version {head[1]}")
    m = int(rd.field("filter_size"))
    nk = int(rd.field("num_filters"))
    T = int(rd.field("stages"))
    looks = int(rd.field("looks"))
    value_range = float.fromhex(rd.field("value_range"))
    variant = rd.field("variant")
    floor = float.fromhex(rd.field("floor"))
    count = int(rd.field("rbf_count"))
    radius = float.fromhex(rd.field("rbf_radius"))
    bandwidth = float.fromhex(rd.field("rbf_bandwidth"))
    generator = rd.field("generator")
    seed = int(rd.field("seed"))
    metadata = json.loads(rd.field("metadata"))
    stages = []
    for t in range(T):
        if rd.field("stage") != str(t):
            raise ValueError(f"{path}: stage blocks out of order")
        beta = float.fromhex(rd.field("beta"))
        coeffs = np.array([[float.fromhex(v) for v in rd.field("coeff").split()]
                           for _ in range(nk)])
        weights = np.array([[float.fromhex(v) for v in rd.field("weight").split()]
                            for _ in range(nk)])
        stages.append(StageParams(beta=beta, coeffs=coeffs, weights=weights))
    if rd.next() != "end":
        raise ValueError(f"{path}: missing end marker")
    return DiffusionModel(stages=stages, filter_size=m, looks=looks,
                          value_range=value_range,
                          rbf=RbfGrid(count=count, radius=radius, bandwidth=bandwidth),
                          variant=variant, floor=floor, generator=generator,
                          seed=seed, metadata=metadata)


# ------------------------------------------------------------------ images

def load_image(path) -> np.ndarray:
    path = Path(path)
    data = path.read_bytes()
    if data[:5] == b"FGRID":
        return _read_fgrid(data.decode("ascii"), path)
    if data[:2] in (b"P2", b"P5"):
        return _read_pgm(data, path)
    raise ValueError(f"{path}: unsupported image format")


def save_image(img, path, peak: float = 255.0) -> None:
    img = as_image(img)
    path = Path(path)
    if path.suffix == ".fgrid":
        save_fgrid(img, path)
    elif path.suffix == ".pgm":
        save_pgm(img, path, peak)
    else:
        raise ValueError(f"{path}: unsupported image suffix")


def _read_fgrid(text: str, path) -> np.ndarray:
    tok = text.split()
    try:
        if len(tok) < 3 or tok[0] != "FGRID":
            raise ValueError
        w, h = int(tok[1]), int(tok[2])
    except ValueError as exc:
        raise ValueError(f"{path}: malformed FGRID header") from exc
    vals = tok[3:]
    if len(vals) != w * h:
        raise ValueError(f"{path}: expected {w * h} values, got {len(vals)}")
    return np.array(vals, dtype=np.float64).reshape(h, w)


def save_fgrid(img: np.ndarray, path) -> None:
    h, w = img.shape
    rows = [" ".join(repr(float(v)) for v in r) for r in img]
    Path(path).write_text(f"FGRID {w} {h}\n" + "\n".join(rows) + "\n")


def _read_pgm(data: bytes, path) -> np.ndarray:
    tokens, pos = [], 0
    while len(tokens) < 4:                      # magic, width, height, maxval
        while pos < len(data) and data[pos:pos + 1].isspace():
            pos += 1
        if data[pos:pos + 1] == b"#":           # comment to end of line
            while pos < len(data) and data[pos:pos + 1] != b"\n":
                pos += 1
            continue
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        if start == pos:
            raise ValueError(f"{path}: truncated graymap header")
        tokens.append(data[start:pos])
    try:
        w, h, maxval = (int(t) for t in tokens[1:4])
    except ValueError as exc:
        raise ValueError(f"{path}: malformed graymap header") from exc
    if w < 1 or h < 1 or not 1 <= maxval <= 65535:
        raise ValueError(f"{path}: unsupported graymap geometry/depth")
    if tokens[0] == b"P2":
        vals = data[pos:].split()
        if len(vals) != w * h:
            raise ValueError(f"{path}: truncated graymap data")
        arr = np.array([int(v) for v in vals], dtype=np.float64)
    else:
        raw = data[pos + 1:]                    # one whitespace after maxval
        dt = np.dtype(">u2") if maxval > 255 else np.dtype("u1")
        if len(raw) < w * h * dt.itemsize:
            raise ValueError(f"{path}: truncated graymap data")
        arr = np.frombuffer(raw[:w * h * dt.itemsize], dtype=dt).astype(np.float64)
    if arr.size and arr.max() > maxval:
        raise ValueError(f"{path}: sample exceeds declared maxval")
    return arr.reshape(h, w)


def save_pgm(img: np.ndarray, path, peak: float = 255.0) -> None:
    if not peak > 0:
        raise ValueError("peak must be positive")
    maxval = int(round(peak))
    if not 1 <= maxval <= 65535:
        raise ValueError(f"peak {peak} not representable in a graymap")
    q = np.minimum(np.rint(np.clip(img, 0.0, peak)).astype(np.uint32), maxval)
    dt = np.dtype(">u2") if maxval > 255 else np.dtype("u1")
    hdr = f"P5 {img.shape[1]} {img.shape[0]} {maxval}\n".encode("ascii")
    Path(path).write_bytes(hdr + q.astype(dt).tobytes())
